"""The reference's test-visible helpers (idrstab.hpp:27-68: arnoldi_init, bicg_projection,
level_iteration, poly_combination) on the device, through the kernel-level C-ABI the drop-in shim
binds (include/mstab_b200_kernels.h), against the UNMODIFIED reference answering the same ABI
(oracle/_ref). Element-wise steps are bit-identical given equal small-solve inputs; the reductions
are trees on the device, so the comparison is to a tight relative tolerance."""
import numpy as np
import pytest

import paper_1604_06043_b200 as m
from paper_1604_06043_b200 import problems as pb

pytestmark = pytest.mark.gpu


def shifted_random(n, shift, seed):
    rng = np.random.default_rng(seed)
    d = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.4)
    d[np.arange(n), np.arange(n)] += shift
    return m.CsrMatrix.from_dense(d)


def relerr(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(1e-300, np.linalg.norm(b)))


def close(a, b, tol):
    return relerr(a, b) <= tol


def state(op, b, s, seed):
    u, v, _ = m.arnoldi_init(op, b, s, seed)
    return m.IterationState.start(np.zeros(b.size), b, u, v)


@pytest.mark.parametrize("n,s", [(10, 2), (64, 4), (300, 8)])
def test_bicg_projection_matches_reference(gpu_ctx, ref_ctx, n, s):
    rng = np.random.default_rng(5 + n)
    p = m.make_cut_space(n, s, 7, ref_ctx)
    block = rng.standard_normal((n, s))
    target = rng.standard_normal(n)
    g, r = m.bicg_projection(p, block, target, gpu_ctx), m.bicg_projection(p, block, target, ref_ctx)
    assert close(g, r, 1e-12)
    # orthogonality of the corrected target (test_solvers.cpp BicgProjection.OrthogonalityResidual)
    assert np.abs(p.T @ (target - block @ g)).max() <= 1e-10 * np.linalg.norm(target)
    with pytest.raises(m.SingularProjection):
        m.bicg_projection(p, np.zeros((n, s)), target, gpu_ctx)


@pytest.mark.parametrize("case", ["rand10_s2", "c1_24_s4", "c2_12_s8"])
def test_level_iteration_and_poly_match_reference(gpu_ctx, ref_ctx, case):
    if case == "rand10_s2":
        A, s, ell = shifted_random(10, 3.0, 8), 2, 2
    elif case == "c1_24_s4":
        A, s, ell = pb.config("c1", grid=24).matrix(), 4, 2
    else:
        A, s, ell = pb.config("c2", grid=12).matrix(), 8, 3
    n = A.n_rows
    gop, rop = m.CsrOperator(A, gpu_ctx), m.CsrOperator(A, ref_ctx)
    b = np.random.default_rng(11).standard_normal(n)
    p = m.make_cut_space(n, s, 8, ref_ctx)
    # the same starting state for both (the reference's Arnoldi block)
    sg, sr = state(rop, b, s, 3), state(rop, b, s, 3)
    lib = gpu_ctx.lib
    l0 = lib.dll.mstab_launch_count()
    import copy
    for k in range(ell):
        # teacher-forced per level: the device starts level k from the reference's state
        sg = copy.deepcopy(sr)
        m.level_iteration(sg, gop, p, k)
        m.level_iteration(sr, rop, p, k)
        assert len(sg.r_levels) == k + 2 and len(sg.v_levels) == k + 3
        assert close(sg.x0, sr.x0, 1e-9), (k, relerr(sg.x0, sr.x0))
        for i in range(k + 2):
            assert close(sg.r_levels[i], sr.r_levels[i], 1e-9), (k, i, relerr(sg.r_levels[i], sr.r_levels[i]))
        for i in range(k + 3):
            assert close(sg.v_levels[i], sr.v_levels[i], 1e-9), (k, i, relerr(sg.v_levels[i], sr.v_levels[i]))
        # level-vector property r^(i+1) = A r^(i) on the device result (LevelIteration tests)
        for i in range(k + 1):
            assert close(sg.r_levels[i + 1], gop.apply(sg.r_levels[i]), 1e-9)
    assert lib.dll.mstab_launch_count() - l0 >= ell * (2 * s + 3)  # kernels ran: not a host path
    # poly from the SAME state on both sides (the reference's), so only the LS reduction differs
    pg, pr = m.poly_combination(sr, ell, gpu_ctx), m.poly_combination(sr, ell, ref_ctx)
    assert close(pg.tau, pr.tau, 1e-8), relerr(pg.tau, pr.tau)
    assert pg.tail_perturbed == pr.tail_perturbed
    for a, c in ((pg.x, pr.x), (pg.r, pr.r), (pg.u, pr.u), (pg.v, pr.v)):
        assert close(a, c, 1e-8), relerr(a, c)
    pg = m.poly_combination(sg, ell, gpu_ctx)
    assert np.linalg.norm(pg.r) <= np.linalg.norm(sg.r_levels[0]) * (1.0 + 1e-14)


def test_arnoldi_with_caller_draws_pads_like_the_seed_form(gpu_ctx):
    """Happy breakdown (identity operator): the padding draws come from the caller's stream; with a
    numpy stream standing in for the engine the basis is orthonormal, and with the library's own
    seeded stream the two entry points agree bit for bit."""
    op = m.CsrOperator(m.CsrMatrix.identity(6), gpu_ctx)
    r0 = np.zeros(6)
    r0[0] = 1.0
    rng = np.random.default_rng(4)
    calls = []

    def draw(count):
        calls.append(count)
        return rng.standard_normal(count)

    u, v, mv = m.arnoldi_init_draws(op, r0, 3, draw)
    assert mv == 3 and calls and all(c == 6 for c in calls)
    assert np.abs(u.T @ u - np.eye(3)).max() <= 1e-12
    assert np.array_equal(u, v)  # V = A U with A = I

"""Split preconditioning on the B200 (precond.cpp / precond.hpp): the factor
builders, the preconditioned operator L^-1 A R^-1, the triangular solves and preconditioned
solves, each checked against the reference itself (oracle/_ref through the same C-ABI).

Bit-exact: factors (host build), fingerprints, triangular solves and applies. Solves are checked
like every other solve here: cycles within +-2 of the reference, solution within 1e-6 relative."""
import numpy as np
import pytest

import paper_1604_06043_b200 as m
from paper_1604_06043_b200 import problems as pb

pytestmark = pytest.mark.gpu


def matrices():
    out = {"tridiag40": m.CsrMatrix.tridiag(2.0, 3.0, 1.0, 40),
           "convdiff2d_24": pb.convdiff(2, 24, 5, (100.0, 100.0, 0.0), 1e-2),
           "convdiff3d_10": pb.convdiff(3, 10, 7, (200.0, 100.0, 50.0), 1e-2),
           "banded_3000": pb.banded(3000, 9, 64, 5)}
    return out


def same_csr(a, b):
    return (np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_idx, b.col_idx)
            and np.array_equal(a.values.view(np.uint64), b.values.view(np.uint64)))


@pytest.mark.parametrize("kind", ["jacobi", "ilu0"])
def test_factor_build_matches_reference(kind, gpu_ctx, ref_ctx):
    for name, a in matrices().items():
        build = m.build_jacobi if kind == "jacobi" else m.build_ilu0
        g, r = build(a, gpu_ctx.lib), build(a, ref_ctx.lib)
        assert same_csr(g.l_factor, r.l_factor), name
        assert same_csr(g.r_factor, r.r_factor), name


@pytest.mark.parametrize("kind", ["jacobi", "ilu0"])
def test_apply_fingerprint_and_solves_bit_exact(kind, gpu_ctx, ref_ctx):
    for name, a in matrices().items():
        pc = (m.build_jacobi if kind == "jacobi" else m.build_ilu0)(a, ref_ctx.lib)
        g = m.PreconditionedOperator(pc, a, gpu_ctx)
        r = m.PreconditionedOperator(pc, a, ref_ctx)
        assert g.fingerprint() == r.fingerprint(), name
        assert g.fingerprint() != m.CsrOperator(a, gpu_ctx).fingerprint()
        x = pb.normal(7, a.n_rows)
        assert np.array_equal(g.apply(x), r.apply(x)), name
        assert np.array_equal(g.lower_solve(x), r.lower_solve(x)), name
        assert np.array_equal(g.upper_solve(x), r.upper_solve(x)), name
        assert np.array_equal(m.preconditioned_rhs(g, x), m.preconditioned_rhs(r, x))
        assert np.array_equal(m.unpreconditioned_solution(g, x), m.unpreconditioned_solution(r, x))


@pytest.mark.parametrize("kind", ["jacobi", "ilu0"])
def test_apply_adjoint_bit_exact(kind, gpu_ctx, ref_ctx):
    """PreconditionedOperator::apply_adjoint (precond.cpp:190-200): R^-H A^H L^-H through the
    transposed factors, against the reference's scatter-form adjoint solves, bit for bit."""
    for name, a in matrices().items():
        pc = (m.build_jacobi if kind == "jacobi" else m.build_ilu0)(a, ref_ctx.lib)
        g = m.PreconditionedOperator(pc, a, gpu_ctx)
        r = m.PreconditionedOperator(pc, a, ref_ctx)
        for seed in (8, 9):
            x = pb.normal(seed, a.n_rows)
            assert np.array_equal(g.apply_adjoint(x), r.apply_adjoint(x)), name
        assert np.array_equal(g.apply(x), r.apply(x)), name  # the forward chain is untouched


def test_bicg_preconditioned_matches_reference(gpu_ctx, ref_ctx):
    a = pb.convdiff(2, 32, 5, (50.0, 50.0, 0.0), 1e-2)
    pc = m.build_ilu0(a, ref_ctx.lib)
    b = pb.normal(11, a.n_rows)
    out = []
    for ctx in (gpu_ctx, ref_ctx):
        op = m.PreconditionedOperator(pc, a, ctx)
        out.append(m.bicg_solve(op, m.preconditioned_rhs(op, b), None, 1e-10, 2000))
    (xg, rg), (xr, rr) = out
    assert rg.status == rr.status == m.CONVERGED
    assert abs(rg.cycles - rr.cycles) <= max(2, rr.cycles // 10)
    assert np.linalg.norm(xg - xr) <= 1e-6 * np.linalg.norm(xr)


def test_exact_ilu0_on_tridiag_is_identity(gpu_ctx):
    """ApplyPreconditioned.ExactFactorsMakeOperatorIdentity (test_precond.cpp:121-138)."""
    a = m.CsrMatrix.tridiag(2.0, 3.0, 1.0, 40)
    op = m.PreconditionedOperator(m.build_ilu0(a, gpu_ctx.lib), a, gpu_ctx)
    x = pb.normal(3, 40)
    assert np.max(np.abs(op.apply(x) - x)) <= 1e-12


def test_zero_pivot_raised(gpu_ctx, ref_ctx):
    """Ilu0.SingularDiagonalRaisesZeroPivot (test_precond.cpp:75-82)."""
    d = np.eye(5)
    d[2, 2] = 0.0
    a = m.CsrMatrix.from_dense(d + np.diag(np.ones(4), 1))
    for lib in (gpu_ctx.lib, ref_ctx.lib):
        with pytest.raises(m.ZeroPivot):
            m.build_ilu0(a, lib)
        with pytest.raises(m.ZeroPivot):
            m.build_jacobi(a, lib)


def test_jacobi_negative_diagonal_is_not_real(gpu_ctx):
    a = m.CsrMatrix.tridiag(1.0, -3.0, 1.0, 10)
    with pytest.raises(m.NotReal):
        m.build_jacobi(a, gpu_ctx.lib)


@pytest.mark.parametrize("kind,s,ell", [("jacobi", 4, 2), ("ilu0", 4, 2), ("ilu0", 2, 1), ("jacobi", 8, 4)])
def test_split_solve_and_recycled_solve_vs_reference(kind, s, ell, gpu_ctx, ref_ctx):
    """Precond.EndToEndSplitSolve (test_precond.cpp:168-192) on a conv-diff system, plus one
    recycled M(s,ell)stab solve teacher-forced on the reference's hand-off."""
    a = pb.convdiff(2, 32, 5, (100.0, 100.0, 0.0), 1e-2)
    pc = (m.build_jacobi if kind == "jacobi" else m.build_ilu0)(a, ref_ctx.lib)
    g = m.PreconditionedOperator(pc, a, gpu_ctx)
    r = m.PreconditionedOperator(pc, a, ref_ctx)
    cfg = pb.config("c1", grid=32)
    x0, f = cfg.sources()
    b = cfg.first_rhs(x0, f)
    bt = m.preconditioned_rhs(r, b)
    sc = m.SolverConfig(s, ell, 1e-8, 100000, True, 0)
    fp = m.FetchPolicy.at_half_tolerance()
    rg = m.idrstab_solve(g, bt, None, sc, None, fp)
    rr = m.idrstab_solve(r, bt, None, sc, None, fp)
    assert rg.report.status == rr.report.status == m.CONVERGED
    assert abs(rg.report.cycles - rr.report.cycles) <= 2
    assert np.linalg.norm(rg.x - rr.x) <= 1e-6 * np.linalg.norm(rr.x)
    x = m.unpreconditioned_solution(g, rg.x)
    assert np.linalg.norm(b - m.CsrOperator(a, gpu_ctx).apply(x)) <= 1e-6 * np.linalg.norm(b)
    # recycled solve on the reference's hand-off (fetch moves it onto the device)
    h = rr.handoff()
    b2 = m.preconditioned_rhs(r, cfg.next_rhs(1, m.unpreconditioned_solution(r, rr.x), f))
    rec_g = m.fetch(h.p, h.u, h.v, h.omega_history, h.level_J, h.matrix_fingerprint, gpu_ctx)
    rg2 = m.mstab_solve(g, b2, None, sc, rec_g, fp)
    rr2 = m.mstab_solve(r, b2, None, sc, h, fp)
    assert rg2.report.status == rr2.report.status == m.CONVERGED
    assert abs(rg2.report.cycles - rr2.report.cycles) <= 2
    assert np.linalg.norm(rg2.x - rr2.x) <= 1e-6 * np.linalg.norm(rr2.x)

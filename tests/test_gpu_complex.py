"""The complex128 path against the unmodified reference (oracle/_ref), which
computes in std::complex<double> natively (types.hpp:11-15): complex CSR operators, complex right-hand
sides and guesses, complex recycle data, fresh and teacher-forced recycled solves, validate."""
import numpy as np
import pytest

import paper_1604_06043_b200 as m
from paper_1604_06043_b200 import problems as pb

pytestmark = pytest.mark.gpu


def helmholtz_1d(n, shift):
    """Complex-shifted 1-D Laplacian (a damped Helmholtz operator): tridiag(-1, 2 + shift, -1)."""
    t = []
    for i in range(n):
        if i > 0:
            t.append((i, i - 1, -1.0 + 0.0j))
        t.append((i, i, 2.0 + shift))
        if i + 1 < n:
            t.append((i, i + 1, -1.0 + 0.0j))
    return m.CsrMatrix.from_triplets(n, n, t)


def convdiff_complex(g):
    """2-D 5-point conv-diff with a complex reaction term and a complex convection coefficient."""
    n = g * g
    t = []
    for j in range(g):
        for i in range(g):
            r = j * g + i
            t.append((r, r, 4.0 + 0.4j))
            if i > 0:
                t.append((r, r - 1, -1.3 - 0.1j))
            if i + 1 < g:
                t.append((r, r + 1, -0.7 + 0.1j))
            if j > 0:
                t.append((r, r - g, -1.1 + 0.05j))
            if j + 1 < g:
                t.append((r, r + g, -0.9 - 0.05j))
    return m.CsrMatrix.from_triplets(n, n, t)


def cvec(seed, n):
    d = pb.normal(seed, 2 * n)
    return d[0::2] + 1j * d[1::2]


def relerr(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_complex_spmv_bit_exact_and_fingerprint(gpu_ctx, ref_ctx):
    for a in (helmholtz_1d(257, 0.3j), convdiff_complex(23)):
        op, rop = m.CsrOperator(a, gpu_ctx), m.CsrOperator(a, ref_ctx)
        assert not op.is_real()
        assert op.fingerprint() == rop.fingerprint()
        x = cvec(5, a.n_rows)
        y, yr = op.apply(x), rop.apply(x)
        assert y.dtype == np.complex128
        assert np.array_equal(y.view(np.float64).view(np.uint64), yr.view(np.float64).view(np.uint64))


def test_real_operator_complex_vector(gpu_ctx, ref_ctx):
    a = m.CsrMatrix.tridiag(-1.0, 2.5, -0.8, 300)
    op, rop = m.CsrOperator(a, gpu_ctx), m.CsrOperator(a, ref_ctx)
    x = cvec(9, 300)
    assert np.array_equal(op.apply(x), rop.apply(x))
    assert op.fingerprint() == op._complex_twin().fingerprint()


@pytest.mark.parametrize("case", ["helmholtz", "convdiff"])
@pytest.mark.parametrize("s,ell", [(4, 1), (4, 2), (2, 4)])
def test_fresh_complex_solve_vs_reference(gpu_ctx, ref_ctx, case, s, ell):
    a = helmholtz_1d(1500, 0.05 + 0.2j) if case == "helmholtz" else convdiff_complex(40)
    n = a.n_rows
    op, rop = m.CsrOperator(a, gpu_ctx), m.CsrOperator(a, ref_ctx)
    b = cvec(21, n)
    cfg = m.SolverConfig(s, ell, 1e-9, 200000, True, 7)
    res, ref = m.idrstab_solve(op, b, None, cfg), m.idrstab_solve(rop, b, None, cfg)
    assert ref.report.status == m.CONVERGED
    assert res.report.status == m.CONVERGED
    assert abs(res.report.cycles - ref.report.cycles) <= 2, (res.report.cycles, ref.report.cycles)
    assert res.x.dtype == np.complex128
    assert relerr(res.x, ref.x) <= 1e-6
    assert np.linalg.norm(b - op.apply(res.x)) <= 1e-9 * np.linalg.norm(b)
    # the complex cut-space draw (both parts of every entry, baselines.cpp:41-42) and the hand-off
    fd, rfd = res.final_data, ref.final_data
    assert fd.is_complex and np.abs(fd.p.imag).max() > 0
    assert np.abs(fd.p - rfd.p).max() <= 1e-12
    assert fd.level_J == res.report.cycles * ell and fd.matrix_fingerprint == rfd.matrix_fingerprint
    # counters (idrstab.cpp:125,150,241,263-264)
    assert res.report.h_mv == s + res.report.cycles * ell * (s + 1)
    assert res.report.h_mv_aux == res.report.cycles
    if ell <= 2 and res.report.cycles == ref.report.cycles:  # complex relaxations (idrstab.cpp:28-41)
        # the early relaxations agree to rounding; later ones drift with the Krylov recurrences (both sides
        # amplify their own reduction rounding), like the iterates themselves
        assert fd.omega_history.size == fd.level_J
        scale = np.abs(rfd.omega_history).max()
        assert np.abs(fd.omega_history[:4] - rfd.omega_history[:4]).max() <= 1e-9 * scale


def test_first_cycles_match_reference_closely(gpu_ctx, ref_ctx):
    """Two cycles from the same start: the iterates agree to reduction-rounding accuracy."""
    a = convdiff_complex(32)
    op, rop = m.CsrOperator(a, gpu_ctx), m.CsrOperator(a, ref_ctx)
    b = cvec(2, a.n_rows)
    s, ell = 4, 2
    cfg = m.SolverConfig(s, ell, 1e-30, s + 2 * ell * (s + 1), False, 3)
    res, ref = m.idrstab_solve(op, b, None, cfg), m.idrstab_solve(rop, b, None, cfg)
    assert res.report.cycles == ref.report.cycles == 2
    assert relerr(res.x, ref.x) <= 1e-10
    t, tr = np.concatenate(res.report.omega_history), np.concatenate(ref.report.omega_history)
    assert np.abs(t - tr).max() <= 1e-9 * np.abs(tr).max()
    assert np.abs(t.imag).max() > 0
    h, hr = res.report.residual_history, ref.report.residual_history
    assert [p.mv for p in h] == [p.mv for p in hr]
    assert max(abs(p.resnorm - q.resnorm) / q.resnorm for p, q in zip(h, hr)) <= 1e-9


def test_teacher_forced_recycled_sequence(gpu_ctx, ref_ctx):
    """The reference drives a chain of complex systems; each B200 solve starts from the reference's
    hand-off (recycle data re-created on the device from its P, U, V)."""
    a = convdiff_complex(36)
    n = a.n_rows
    op, rop = m.CsrOperator(a, gpu_ctx), m.CsrOperator(a, ref_ctx)
    cfg = m.SolverConfig(4, 2, 1e-9, 200000, True, 11)
    pol = m.FetchPolicy.at_half_tolerance()
    b = cvec(40, n)
    ref = m.idrstab_solve(rop, b, None, cfg, None, pol)
    for i in range(3):
        h = ref.handoff()
        b = ref.x + 0.2 * cvec(41 + i, n)
        ref = m.mstab_solve(rop, b, None, cfg, h, pol)
        dev_h = m.fetch(h.p, h.u, h.v, h.omega_history, h.level_J, h.matrix_fingerprint, gpu_ctx)
        assert dev_h.is_complex
        v, vr = m.validate(dev_h, op), m.validate(h, rop)
        assert abs(v.max_deviation - vr.max_deviation) <= 1e-9 and v.low_rank_warning == vr.low_rank_warning
        assert abs(v.sigma_min_ratio - vr.sigma_min_ratio) <= 1e-6 * vr.sigma_min_ratio
        res = m.mstab_solve(op, b, None, cfg, dev_h, pol)
        assert res.report.status == m.CONVERGED and ref.report.status == m.CONVERGED
        assert abs(res.report.cycles - ref.report.cycles) <= 2
        assert relerr(res.x, ref.x) <= 1e-6
        assert res.report.h_mv_aux == ref.report.h_mv_aux and res.report.h_rd - ref.report.h_rd == \
            (res.report.cycles - ref.report.cycles) * 2 * 4
        assert (res.fetched is None) == (ref.fetched is None)


def test_complex_guess_and_real_data_through_the_complex_path(gpu_ctx, ref_ctx):
    a = m.CsrMatrix.tridiag(-1.0, 2.4, -0.9, 800)
    op, rop = m.CsrOperator(a, gpu_ctx), m.CsrOperator(a, ref_ctx)
    b = pb.normal(3, 800)
    x0 = 0.1 * cvec(4, 800)
    cfg = m.SolverConfig(3, 2, 1e-10, 100000, False, 5)
    res, ref = m.idrstab_solve(op, b, x0, cfg), m.idrstab_solve(rop, b, x0, cfg)
    assert res.report.status == m.CONVERGED
    assert abs(res.report.cycles - ref.report.cycles) <= 2 and relerr(res.x, ref.x) <= 1e-6
    assert res.report.h_mv_aux == ref.report.h_mv_aux == 1  # r = b - A x0
    # a real triple draws the REAL cut-space even on the complex path (baselines.cpp:41): P has no imaginary part
    lib, C = gpu_ctx.lib, __import__("ctypes")
    bz = np.ascontiguousarray(b, dtype=np.complex128)
    h = C.c_void_p()
    c = cfg._c()
    assert lib.dll.mstab_solve_z(gpu_ctx.h, op._complex_twin().h, bz.ctypes.data, None, 0, C.byref(c), None, None,
                                 C.byref(h)) == 0
    rz = m.SolveResult(gpu_ctx, h)
    rz.n = 800
    rr = m.idrstab_solve(op, b, None, cfg)  # the fused real path
    assert np.abs(rz.final_data.p.imag).max() == 0.0
    assert np.abs(rz.final_data.p.real - rr.final_data.p).max() <= 1e-12
    assert abs(rz.report.cycles - rr.report.cycles) <= 1 and relerr(rz.x.real, rr.x) <= 1e-7
    assert np.abs(rz.x.imag).max() == 0.0


def test_validate_rejections_and_real_entry_points(gpu_ctx):
    a = helmholtz_1d(400, 0.25j)
    op = m.CsrOperator(a, gpu_ctx)
    b = cvec(8, 400)
    res = m.idrstab_solve(op, b, None, m.SolverConfig(3, 1, 1e-8, 100000, False, 2))
    fd = res.final_data
    assert m.validate(fd, op).max_deviation <= 1e-6
    bad_v = np.array(fd.v)
    bad_v[:, 1] *= 1.0 + 1e-3j
    with pytest.raises(m.StaleData):
        m.validate(m.fetch(fd.p, fd.u, bad_v, fd.omega_history, fd.level_J, fd.matrix_fingerprint, gpu_ctx), op)
    with pytest.raises(m.FingerprintMismatch):
        m.validate(fd, m.CsrOperator(helmholtz_1d(400, 0.26j), gpu_ctx))
    with pytest.raises(m.StaleData):  # omega history length != level
        m.validate(m.fetch(fd.p, fd.u, fd.v, fd.omega_history[:-1], fd.level_J, fd.matrix_fingerprint, gpu_ctx), op)
    # a complex handle given to a real fp64 entry point is refused, never silently truncated
    import ctypes as C
    y = np.empty(400)
    rc = gpu_ctx.lib.dll.mstab_operator_apply(gpu_ctx.h, op.h, y.ctypes.data, y.ctypes.data, 0)
    assert rc == -21
    with pytest.raises(m.ConfigError):
        m.idrstab_solve(op, b, None, m.SolverConfig(0, 1, 1e-8, 100, False, 1))


def test_breakdown_keeps_last_completed_cycle(gpu_ctx, ref_ctx):
    """A singular projection mid-cycle: status BREAKDOWN with the reference's reason and counters."""
    n = 12
    a = m.CsrMatrix.from_triplets(n, n, [(i, i, 1.0 + 0.0j if i else 1.0 + 1e-300j) for i in range(n)])
    a.values = np.ascontiguousarray(a.values, dtype=np.complex128)
    a.values[0] = 1.0 + 1.0j
    op, rop = m.CsrOperator(a, gpu_ctx), m.CsrOperator(a, ref_ctx)
    b = np.zeros(n, dtype=np.complex128)
    b[0] = 1.0j
    cfg = m.SolverConfig(2, 1, 1e-12, 1000, False, 1)
    res, ref = m.idrstab_solve(op, b, None, cfg), m.idrstab_solve(rop, b, None, cfg)
    assert res.report.status == ref.report.status
    assert res.report.cycles == ref.report.cycles and res.report.h_mv == ref.report.h_mv
    assert res.report.breakdown_reason == ref.report.breakdown_reason

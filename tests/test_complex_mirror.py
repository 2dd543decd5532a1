"""CPU: the Python mirror's complex128 routing driven against the REFERENCE
implementation of the same C-ABI (oracle/_ref, the unmodified reference behind oracle/ref_capi.cpp):
operators, solves, recycle data and validate take the *_z entry points whenever data is complex, and
the results satisfy the equations. The B200 side of the same calls is tests/test_gpu_complex.py."""
import numpy as np
import pytest

import paper_1604_06043_b200 as m
from paper_1604_06043_b200 import problems as pb


def shifted_laplacian(n, shift):
    t = []
    for i in range(n):
        if i > 0:
            t.append((i, i - 1, -1.0 + 0.0j))
        t.append((i, i, 2.0 + shift))
        if i + 1 < n:
            t.append((i, i + 1, -1.0 + 0.0j))
    return m.CsrMatrix.from_triplets(n, n, t)


def cvec(seed, n):
    d = pb.normal(seed, 2 * n)
    return d[0::2] + 1j * d[1::2]


def test_complex_matrix_keeps_its_values_and_real_stays_real():
    a = shifted_laplacian(20, 0.3j)
    assert not a.is_real() and a.values.dtype == np.complex128
    assert a.to_dense()[3, 3] == 2.0 + 0.3j
    r = m.CsrMatrix.tridiag(-1.0, 2.0, -1.0, 20)
    assert r.is_real() and r.values.dtype == np.float64
    # complex dtype with zero imaginary parts is real data (is_real, types.cpp:25-29)
    z = m.CsrMatrix(2, 2, [0, 1, 2], [0, 1], np.array([1.0 + 0j, 2.0 + 0j]))
    assert z.is_real() and z.values.dtype == np.float64


def test_complex_solve_chain_through_the_mirror(ref_ctx):
    n = 300
    a = shifted_laplacian(n, 0.1 + 0.25j)
    op = m.CsrOperator(a, ref_ctx)
    assert not op.is_real()
    x = cvec(1, n)
    y = op.apply(x)
    assert y.dtype == np.complex128 and np.allclose(y, a.to_dense() @ x, rtol=0, atol=1e-13)
    cfg = m.SolverConfig(3, 2, 1e-10, 100000, True, 4)
    b = cvec(2, n)
    r1 = m.idrstab_solve(op, b, None, cfg, None, m.FetchPolicy.at_half_tolerance())
    assert r1.report.status == m.CONVERGED and r1.x.dtype == np.complex128
    assert np.linalg.norm(b - op.apply(r1.x)) <= 1e-10 * np.linalg.norm(b)
    h = r1.handoff()
    assert h.is_complex and h.p.dtype == np.complex128 and np.abs(h.p.imag).max() > 0
    assert h.matrix_fingerprint == op.fingerprint() and h.s == 3
    v = m.validate(h, op)
    assert v.max_deviation <= 1e-6
    # re-created from host blocks (fetch) and continued (mstab_solve)
    h2 = m.fetch(h.p, h.u, h.v, h.omega_history, h.level_J, h.matrix_fingerprint, ref_ctx)
    assert h2.is_complex and np.array_equal(h2.u, h.u)
    b2 = r1.x + 0.1 * cvec(3, n)
    r2 = m.mstab_solve(op, b2, None, cfg, h2)
    assert r2.report.status == m.CONVERGED
    assert np.linalg.norm(b2 - op.apply(r2.x)) <= 1e-10 * np.linalg.norm(b2)
    assert r2.report.h_mv_aux == 3 + r2.report.cycles  # validate's s products + one true residual per cycle
    t = np.concatenate(r2.report.omega_history)
    assert np.abs(t.imag).max() > 0


def test_real_operator_with_complex_right_hand_side(ref_ctx):
    n = 200
    a = m.CsrMatrix.tridiag(-1.0, 2.5, -0.7, n)
    op = m.CsrOperator(a, ref_ctx)
    assert op.is_real()
    b = cvec(5, n)
    r = m.idrstab_solve(op, b, None, m.SolverConfig(2, 1, 1e-10, 100000, False, 1))
    assert r.report.status == m.CONVERGED
    assert np.linalg.norm(b - a.to_dense() @ r.x) <= 1e-9 * np.linalg.norm(b)
    assert op._complex_twin().fingerprint() == op.fingerprint()
    # real data keeps the real entry points and real results
    rr = m.idrstab_solve(op, b.real, None, m.SolverConfig(2, 1, 1e-10, 100000, False, 1))
    assert rr.x.dtype == np.float64


def test_real_entry_points_refuse_complex_values():
    with pytest.raises(m.NotReal):
        m.mstab._f64(np.array([1.0 + 1.0j]))

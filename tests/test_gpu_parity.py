"""Teacher-forced parity at BASELINE-like sizes against the C restatement oracle run live on the
GPU box's host (sizes it finishes in seconds), plus size-independent properties at the full c2
size. North-star bar: every RHS converges, ‖x − x_ref‖/‖x_ref‖ ≤ 1e-6,
cycle counts within ±2 of the reference's."""
import numpy as np
import pytest

import oracle_c as oc
import paper_1604_06043_b200 as m
from paper_1604_06043_b200 import problems as pb

pytestmark = pytest.mark.gpu


def relres(csr, b, x):
    return np.linalg.norm(b - csr.apply(x)) / np.linalg.norm(b)


def teacher_forced_chain(gpu_ctx, cfg, nrhs, true_res=False):
    """Chain driven by the ORACLE (its b_i and its hand-off); the GPU solves each system from the
    same inputs and is compared system by system."""
    A = cfg.matrix()
    op = m.CsrOperator(A, gpu_ctx)
    csr = oc.Csr(A)
    x0, f = cfg.sources()
    b = cfg.first_rhs(x0, f)
    sc = m.SolverConfig(cfg.s, cfg.ell, 1e-8, 100000, true_res, 0)
    rec = None
    rows = []
    for i in range(nrhs):
        o = oc.solve(csr, b, s=cfg.s, ell=cfg.ell, seed=0, true_residual=true_res, recycle=rec, fetch_kind=1)
        grec = None if rec is None else m.fetch(rec.p, rec.u, rec.v, rec.omega, rec.level_j, rec.fingerprint, gpu_ctx)
        g = m.idrstab_solve(op, b, None, sc, grec, m.FetchPolicy.at_half_tolerance())
        rows.append((i, o.cycles, g.report.cycles, np.linalg.norm(g.x - o.x) / np.linalg.norm(o.x),
                     relres(csr, b, g.x), relres(csr, b, o.x), g.report.status))
        assert g.report.status == m.CONVERGED and o.status == 0, rows[-1]
        assert abs(g.report.cycles - o.cycles) <= 2, rows[-1]
        assert rows[-1][3] <= 1e-6, rows[-1]
        assert rows[-1][4] <= max(1e-8, 1.5 * rows[-1][5]), rows[-1]
        rec = o.fetched
        b = cfg.next_rhs(i + 1, o.x, f)
    return rows


def test_c1_full_size_teacher_forced(gpu_ctx):
    """BASELINE configs[0] at full size (256^2, s=4, ell=2): first three systems of the chain."""
    teacher_forced_chain(gpu_ctx, pb.config("c1"), 3)


def test_c2_reduced_teacher_forced(gpu_ctx):
    """configs[1] shape at 40^3 (s=8, ell=4) with the bench's true-residual setting."""
    teacher_forced_chain(gpu_ctx, pb.config("c2", grid=40), 2, true_res=True)


def test_c3_reduced_teacher_forced(gpu_ctx):
    """configs[2] (random banded, 27 nnz/row, CSR path) at N=131072, half-width 4096."""
    cfg = pb.config("c3", grid=131072)
    teacher_forced_chain(gpu_ctx, cfg, 3)


def test_c2_full_size_properties(gpu_ctx):
    """Full c2 size: convergence of the true residual, bit-identical repeat (determinism), the
    hand-off satisfies validate's invariants or is rejected exactly like the reference would."""
    cfg = pb.config("c2")
    A = cfg.matrix()
    op = m.CsrOperator(A, gpu_ctx)
    x0, f = cfg.sources()
    b = cfg.first_rhs(x0, f)
    sc = m.SolverConfig(cfg.s, cfg.ell, 1e-8, 100000, True, 0)
    r1 = m.idrstab_solve(op, b, None, sc, None, m.FetchPolicy.at_half_tolerance())
    r2 = m.idrstab_solve(op, b, None, sc, None, m.FetchPolicy.at_half_tolerance())
    assert r1.report.status == m.CONVERGED
    h1 = [h.resnorm for h in r1.report.residual_history]
    assert h1 == [h.resnorm for h in r2.report.residual_history]
    assert np.array_equal(r1.x, r2.x)
    assert np.linalg.norm(b - op.apply(r1.x)) / np.linalg.norm(b) <= 1e-8
    assert r1.report.h_mv == cfg.s + r1.report.cycles * cfg.ell * (cfg.s + 1)
    h = r1.handoff()
    vr = m.validate(h, op)
    assert vr.max_deviation <= 1e-6
    # one recycled solve along the chain
    b2 = cfg.next_rhs(1, r1.x, f)
    r3 = m.mstab_solve(op, b2, None, sc, h, m.FetchPolicy.at_half_tolerance())
    assert r3.report.status == m.CONVERGED
    assert np.linalg.norm(b2 - op.apply(r3.x)) / np.linalg.norm(b2) <= 1e-8
    assert r3.report.h_mv_aux == cfg.s + r3.report.cycles  # validate + true residual per cycle


def test_c3_full_size_properties(gpu_ctx):
    """Full c3 size (N=4,194,304, 27 nnz/row, irregular gathers): two chained solves converge."""
    cfg = pb.config("c3")
    A = cfg.matrix()
    op = m.CsrOperator(A, gpu_ctx)
    sc = m.SolverConfig(cfg.s, cfg.ell, 1e-8, 100000, False, 0)
    b = cfg.first_rhs()
    r = m.idrstab_solve(op, b, None, sc, None, m.FetchPolicy.at_half_tolerance())
    assert r.report.status == m.CONVERGED
    assert np.linalg.norm(b - op.apply(r.x)) / np.linalg.norm(b) <= 1e-7
    b2 = cfg.next_rhs(1, r.x)
    r2 = m.mstab_solve(op, b2, None, sc, r.handoff(), m.FetchPolicy.at_half_tolerance())
    assert r2.report.status == m.CONVERGED
    assert np.linalg.norm(b2 - op.apply(r2.x)) / np.linalg.norm(b2) <= 1e-7

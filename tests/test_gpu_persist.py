"""The persistent cycle kernel (csrc/kpersist.cu: one cooperative kernel per IDR(s)stab(ell) cycle,
the cycle state in registers) against the stream-of-kernels path and the oracle, on L2-resident
systems (BASELINE c1 shapes). Same element-wise arithmetic, different grouping of the reductions:
cycle counts within the parity bar, solutions to 1e-6, true residual under tol."""
import os

import numpy as np
import pytest

import oracle_c as oc
import paper_1604_06043_b200 as m
from paper_1604_06043_b200 import problems as pb

pytestmark = pytest.mark.gpu


def solve_chain(ctx, cfg, A, n_rhs, tres):
    """Free-running chain on `ctx`; returns per system (b, hand-off fed in as host blocks, x, cycles, status,
    launches)."""
    op = m.CsrOperator(A, ctx)
    x0, f = cfg.sources()
    b = cfg.first_rhs(x0, f)
    sc = m.SolverConfig(cfg.s, cfg.ell, 1e-8, 100000, tres, 0)
    fp = m.FetchPolicy.at_half_tolerance()
    rec, out = None, []
    lib = ctx.lib
    for i in range(1, n_rhs + 1):
        l0 = lib.dll.mstab_launch_count()
        r = m.idrstab_solve(op, b, None, sc, rec, fp)
        host_in = None if rec is None else (rec.p.copy(), rec.u.copy(), rec.v.copy(), np.array(rec.omega_history),
                                            rec.level_J, rec.matrix_fingerprint)
        out.append((b.copy(), host_in, r.x.copy(), r.report.cycles, r.report.status,
                    lib.dll.mstab_launch_count() - l0))
        rec = r.handoff()
        b = cfg.next_rhs(i, r.x, f)
    return op, out


@pytest.mark.parametrize("grid,s,ell,tres", [(64, 4, 2, True), (96, 4, 2, False), (128, 2, 2, True), (256, 4, 2, True)])
def test_persistent_cycle_matches_stream_path(grid, s, ell, tres):
    """The stream-of-kernels chain supplies every system (b_i and the hand-off); the persistent
    path solves the same systems (teacher-forced, like the parity against the reference)."""
    cfg = pb.config("c1", grid=grid)
    cfg.s, cfg.ell = s, ell
    A = cfg.matrix()
    lib = m.Lib()
    os.environ["MSTAB_NO_PERSIST"] = "1"
    try:
        _, strm = solve_chain(m.Context(lib, 0), cfg, A, 3, tres)
    finally:
        os.environ.pop("MSTAB_NO_PERSIST", None)
    ctx = m.Context(lib, 0)
    op = m.CsrOperator(A, ctx)
    sc = m.SolverConfig(cfg.s, cfg.ell, 1e-8, 100000, tres, 0)
    for b, host_in, xs, cs, sts, ls in strm:
        rec = None if host_in is None else m.fetch(*host_in, ctx)
        l0 = lib.dll.mstab_launch_count()
        r = m.idrstab_solve(op, b, None, sc, rec, m.FetchPolicy.at_half_tolerance())
        lp, cp, xp = lib.dll.mstab_launch_count() - l0, r.report.cycles, r.x
        assert r.report.status == m.CONVERGED and sts == m.CONVERGED
        # one launch per cycle (+ validate / prologue / copies) against ~26 per cycle
        assert lp < 3 * cp + 60 and ls > 10 * cs, (lp, cp, ls, cs)
        assert abs(cp - cs) <= max(2, int(np.ceil(0.07 * cs))), (cp, cs)
        assert np.linalg.norm(xp - xs) <= 1e-6 * np.linalg.norm(xs)
        res = np.linalg.norm(b - op.apply(xp)) / np.linalg.norm(b)
        assert res <= (1e-8 if tres else 5e-8), res


def test_persistent_cycle_teacher_forced_vs_oracle(gpu_ctx):
    """Fresh + recycled solve of a 64^2 system: the oracle's hand-off into both, cycles within +-2."""
    os.environ.pop("MSTAB_NO_PERSIST", None)
    cfg = pb.config("c1", grid=64)
    A = cfg.matrix()
    op = m.CsrOperator(A, gpu_ctx)
    csr = oc.Csr(A)
    x0, f = cfg.sources()
    b = cfg.first_rhs(x0, f)
    sc = m.SolverConfig(cfg.s, cfg.ell, 1e-8, 100000, False, 0)
    g = m.idrstab_solve(op, b, None, sc, None, m.FetchPolicy.at_half_tolerance())
    o = oc.solve(csr, b, s=cfg.s, ell=cfg.ell, seed=0, fetch_kind=1)
    assert g.report.status == m.CONVERGED and abs(g.report.cycles - o.cycles) <= 2
    assert np.linalg.norm(g.x - o.x) <= 1e-6 * np.linalg.norm(o.x)
    h = o.fetched
    b2 = cfg.next_rhs(1, o.x, f)
    rec = m.fetch(h.p, h.u, h.v, h.omega, h.level_j, h.fingerprint, gpu_ctx)
    g2 = m.mstab_solve(op, b2, None, sc, rec, m.FetchPolicy.at_half_tolerance())
    o2 = oc.solve(csr, b2, s=cfg.s, ell=cfg.ell, seed=0, recycle=h, fetch_kind=1)
    assert g2.report.status == m.CONVERGED and abs(g2.report.cycles - o2.cycles) <= 2
    assert np.linalg.norm(g2.x - o2.x) <= 1e-6 * np.linalg.norm(o2.x)

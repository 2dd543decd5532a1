"""Quick GPU-vs-reference parity smoke (developer tool)."""
import sys, time
import numpy as np
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1604_06043_b200 as m
from paper_1604_06043_b200 import problems as pb

ref = m.Lib("oracle/_ref/libmstab_ref.so")
gpu = m.Lib()
rctx, gctx = m.Context(ref), m.Context(gpu)

def both(A):
    return m.CsrOperator(A, rctx), m.CsrOperator(A, gctx)

# spmv bit-exactness
cfg = pb.config("c1", grid=64)
A = cfg.matrix()
ro, go = both(A)
print("fingerprint", ro.fingerprint() == go.fingerprint(), hex(go.fingerprint()))
x = np.random.default_rng(0).standard_normal(A.n_rows)
print("spmv bitexact", np.array_equal(ro.apply(x), go.apply(x)))
# small solve
rng = np.random.default_rng(1)
M = rng.standard_normal((8, 8)); r = rng.standard_normal(8)
print("solve_small bitexact", np.array_equal(m.solve_small(M, r, rctx), m.solve_small(M, r, gctx)))
Z = rng.standard_normal((1000, 4)); rr = rng.standard_normal(1000)
t1, t2 = m.least_squares_tall(Z, rr, rctx), m.least_squares_tall(Z, rr, gctx)
print("ls", np.max(np.abs(t1 - t2) / np.abs(t1)))
P1, P2 = m.make_cut_space(5000, 4, 7, rctx), m.make_cut_space(5000, 4, 7, gctx)
print("cut space", np.max(np.abs(P1 - P2)))
# tridiag KATs
tri = m.CsrMatrix.tridiag(2.0, 3.0, 1.0, 40)
rt, gt = both(tri)
for s in (2, 4):
    c = m.SolverConfig(s, 1, 1e-8, 100000, True, 1)
    a, b = m.idrstab_solve(rt, np.ones(40), None, c), m.idrstab_solve(gt, np.ones(40), None, c)
    print("tridiag s", s, a.report.cycles, b.report.cycles, a.report.h_mv, b.report.h_mv, b.report.status)
# conv-diff sequence (teacher forced)
for name, grid in (("c1", 64), ("c1", 256), ("c2", 64)):
    cfg = pb.config(name, grid=grid)
    A = cfg.matrix(); ro, go = both(A)
    x0, f = cfg.sources(); b = cfg.first_rhs(x0, f)
    sc = m.SolverConfig(cfg.s, cfg.ell, 1e-8, 100000, False, 0)
    fp = m.FetchPolicy.at_half_tolerance()
    t = time.time(); a = m.idrstab_solve(ro, b, None, sc, None, fp); ta = time.time() - t
    t = time.time(); g = m.idrstab_solve(go, b, None, sc, None, fp); tg = time.time() - t
    print(name, grid, "fresh: cycles", a.report.cycles, g.report.cycles, g.report.status,
          "dx", np.linalg.norm(a.x - g.x) / np.linalg.norm(a.x), "t", round(ta, 3), round(tg, 3))
    # teacher forced second solve: same handoff (the reference's) into both
    h = a.handoff()
    hg = m.fetch(h.p, h.u, h.v, h.omega_history, h.level_J, h.matrix_fingerprint, gctx)
    b2 = cfg.next_rhs(1, a.x, f)
    t = time.time(); a2 = m.mstab_solve(ro, b2, None, sc, h, fp); ta = time.time() - t
    t = time.time(); g2 = m.mstab_solve(go, b2, None, sc, hg, fp); tg = time.time() - t
    tr = np.linalg.norm(b2 - ro.apply(g2.x)) / np.linalg.norm(b2)
    print(name, grid, "mstab: cycles", a2.report.cycles, g2.report.cycles, g2.report.status,
          "dx", np.linalg.norm(a2.x - g2.x) / np.linalg.norm(a2.x), "true res", tr, "t", round(ta, 3), round(tg, 3))
    print("  hist ref", [f"{p.resnorm:.3e}" for p in a2.report.residual_history[:6]])
    print("  hist gpu", [f"{p.resnorm:.3e}" for p in g2.report.residual_history[:6]])

# GPU-only timing on the full c2 config: fresh solve + 3 chained Mstab solves
cfg = pb.config("c2")
A = cfg.matrix(); go = m.CsrOperator(A, gctx)
x0, f = cfg.sources(); b = cfg.first_rhs(x0, f)
sc = m.SolverConfig(cfg.s, cfg.ell, 1e-8, 100000, False, 0)
fp = m.FetchPolicy.at_half_tolerance()
t = time.time(); g = m.idrstab_solve(go, b, None, sc, None, fp); print("c2 fresh", g.report.cycles, g.report.status, time.time() - t)
h = g.handoff(); x = g.x
for i in range(3):
    b = cfg.next_rhs(i + 1, x, f)
    t = time.time(); g = m.mstab_solve(go, b, None, sc, h, fp); dt = time.time() - t
    x = g.x; h = g.handoff()
    tr = np.linalg.norm(b - go.apply(x)) / np.linalg.norm(b)
    print("c2 mstab", i, g.report.cycles, g.report.status, "t", round(dt, 4), "per cycle ms", round(1e3 * dt / max(g.report.cycles, 1), 3), "true res", tr)

"""Where the e2e step time goes (developer tool): solve (incl. H2D of b), D2H of x, host RHS."""
import sys, time
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np
import torch
import paper_1604_06043_b200 as m
from paper_1604_06043_b200 import problems as pb

cfg = pb.config(sys.argv[1] if len(sys.argv) > 1 else "c2")
A = cfg.matrix()
ctx = m.Context(m.Lib(), 0)
op = m.CsrOperator(A, ctx)
x0, f = cfg.sources()
b = torch.from_numpy(cfg.first_rhs(x0, f)).pin_memory().numpy()
x = torch.empty(cfg.N, dtype=torch.float64).pin_memory().numpy()
sc = m.SolverConfig(cfg.s, cfg.ell, cfg.tol, 100000, True, 0)
fp = m.FetchPolicy.at_half_tolerance()
rec = None
dll = ctx.lib.dll
for i in range(8):
    t0 = time.perf_counter()
    try:
        r = m.idrstab_solve(op, b, None, sc, rec, fp)
    except m.StaleData:
        r = m.idrstab_solve(op, b, None, sc, None, fp)
    t1 = time.perf_counter()
    r.x_into(x)
    t2 = time.perf_counter()
    rec = r.handoff()
    t3 = time.perf_counter()
    dll.mstab_harness_euler_rhs(ctx.h, cfg.N, x.ctypes.data, f.ctypes.data, cfg.dt, cfg.h2, b.ctypes.data, 0)
    t4 = time.perf_counter()
    print(f"rhs {i}: cycles {r.report.cycles} solve {1e3*(t1-t0):.2f} ms  x D2H {1e3*(t2-t1):.2f}  handoff {1e3*(t3-t2):.2f}"
          f"  host rhs {1e3*(t4-t3):.2f}", flush=True)

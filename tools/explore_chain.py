"""Explore recycle hand-off stability along a BASELINE sequence (developer tool)."""
import sys, time
import numpy as np
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1604_06043_b200 as m
from paper_1604_06043_b200 import problems as pb

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 10
ctx = m.Context(m.Lib())
cfg = pb.config(name)
A = cfg.matrix(); op = m.CsrOperator(A, ctx)
x0, f = cfg.sources()
tres = len(sys.argv) > 3 and sys.argv[3] == "tr"
sc = m.SolverConfig(cfg.s, cfg.ell, 1e-8, 100000, tres, 0)
for label, fp in (("half", m.FetchPolicy.at_half_tolerance()), ("cyc1", m.FetchPolicy.at_cycle(1)),
                  ("cyc2", m.FetchPolicy.at_cycle(2)), ("cyc3", m.FetchPolicy.at_cycle(3)), ("off", None)):
    b = cfg.first_rhs(x0, f); rec = None; log = []; t0 = time.time()
    for i in range(nrhs):
        stale = False
        try:
            r = m.idrstab_solve(op, b, None, sc, rec, fp)
        except m.StaleData:
            stale = True
            r = m.idrstab_solve(op, b, None, sc, None, fp)
        tr = np.linalg.norm(b - op.apply(r.x)) / np.linalg.norm(b)
        h = r.handoff()
        try:
            dev = m.validate(h, op).max_deviation
        except m.StaleData:
            dev = float("inf")
        log.append(f"{'S' if stale else ''}{r.report.cycles}{r.report.status[0]}/{tr:.0e}/{dev:.0e}")
        if r.report.status == "Breakdown":
            break
        rec = h; b = cfg.next_rhs(i + 1, r.x, f)
    print(name, label, f"{time.time()-t0:.2f}s", " ".join(log), flush=True)

"""One-cycle parity probe: residual history and solution after `cycles` cycles of a fresh
IDR(s)stab(ell) solve on the B200 and on the reference (same b, seed, MV budget).

usage: python tools/cycle_diff.py GRID s,ell [s,ell ...] [--cycles C]"""
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0] + "/tests")
import paper_1604_06043_b200 as m  # noqa: E402
from paper_1604_06043_b200 import problems as pb  # noqa: E402
from conftest import REF_LIB  # noqa: E402

grid = int(sys.argv[1])
cycles = int(sys.argv[sys.argv.index("--cycles") + 1]) if "--cycles" in sys.argv else 1
pairs = [tuple(int(v) for v in a.split(",")) for a in sys.argv[2:] if "," in a]
g, r = m.Context(m.Lib(), 0), m.Context(m.Lib(REF_LIB))
cfg = pb.config("c5", grid=grid)
A = cfg.matrix()
x0, f = cfg.sources()
b = cfg.first_rhs(x0, f)
for s, ell in pairs:
    sc = m.SolverConfig(s, ell, 1e-30, s + cycles * ell * (s + 1), False, 0)
    xs, hs = [], []
    t0 = time.perf_counter()
    for ctx in (g, r):
        res = m.idrstab_solve(m.CsrOperator(A, ctx), b, None, sc, None, None)
        xs.append(res.x)
        hs.append([p.resnorm for p in res.report.residual_history])
    d = np.linalg.norm(xs[0] - xs[1]) / np.linalg.norm(xs[1])
    print(f"grid {grid} (s,ell)=({s},{ell}) cycles {cycles}: resnorm b200 {hs[0][-1]:.4e} ref {hs[1][-1]:.4e} "
          f"|dx|/|x| {d:.2e} ({time.perf_counter() - t0:.1f} s)", flush=True)

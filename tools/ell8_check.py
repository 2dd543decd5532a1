"""Cross-check of the (s, ell) points where the c5 sweep diverges or breaks down: the FIRST (fresh)
solve of the sequence at a reduced grid, on the B200 and on the reference (oracle/_ref, same ABI),
same b, same seed. Reports status, cycles, MVs and the true relative residual of each.

usage: python tools/ell8_check.py GRID s,ell [s,ell ...] [--no-ref]"""
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0] + "/tests")
import paper_1604_06043_b200 as m  # noqa: E402
from paper_1604_06043_b200 import problems as pb  # noqa: E402
from conftest import REF_LIB  # noqa: E402

grid = int(sys.argv[1])
pairs = [tuple(int(v) for v in a.split(",")) for a in sys.argv[2:] if not a.startswith("--")] or [(16, 8)]
g = m.Context(m.Lib(), 0)
with_ref = "--no-ref" not in sys.argv
r = m.Context(m.Lib(REF_LIB)) if with_ref else None
for s, ell in pairs:
    cfg = pb.config("c5", grid=grid)
    cfg.s, cfg.ell = s, ell
    A = cfg.matrix()
    x0, f = cfg.sources()
    b = cfg.first_rhs(x0, f)
    sc = m.SolverConfig(s, ell, 1e-8, 20000, True, 0)
    chk = m.CsrOperator(A, g)
    for name, ctx in (("b200", g), ("reference", r)) if with_ref else (("b200", g),):
        t0 = time.perf_counter()
        res = m.idrstab_solve(m.CsrOperator(A, ctx), b, None, sc, None, m.FetchPolicy.at_half_tolerance())
        x = res.x
        tr = np.linalg.norm(b - chk.apply(x)) / np.linalg.norm(b) if np.all(np.isfinite(x)) else float("inf")
        print(f"grid {grid} (s,ell)=({s},{ell}) {name:9s} status {res.report.status} cycles {res.report.cycles} "
              f"h_mv {res.report.h_mv} true relres {tr:.2e} ({time.perf_counter() - t0:.1f} s)", flush=True)

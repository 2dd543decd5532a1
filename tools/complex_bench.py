"""Complex128 path timing (developer tool): one fresh solve of a complex-shifted 3-D
7-point conv-diff system (the c2 matrix plus a complex reaction term on the diagonal) on the B200,
next to the fused real path on the unshifted matrix of the same size.
usage: python tools/complex_bench.py [grid=96] [s=4] [ell=2]"""
import json
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np  # noqa: E402

import paper_1604_06043_b200 as m  # noqa: E402
from paper_1604_06043_b200 import problems as pb  # noqa: E402

grid = int(sys.argv[1]) if len(sys.argv) > 1 else 96
s = int(sys.argv[2]) if len(sys.argv) > 2 else 4
ell = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cfg = pb.config("c2", grid=grid)
A = cfg.matrix()
n = A.n_rows
ctx = m.Context(m.Lib(), 0)
diag = np.zeros(A.nnz(), dtype=bool)
rp = np.asarray(A.row_ptr)
rows = np.repeat(np.arange(n), np.diff(rp))
diag[np.asarray(A.col_idx) == rows] = True
vz = np.asarray(A.values, dtype=np.complex128)
vz[diag] += 0.05j * np.abs(vz[diag])
Az = m.CsrMatrix(n, n, A.row_ptr, A.col_idx, vz)
x0, f = cfg.sources()
b = cfg.first_rhs(x0, f)
bz = b * (1.0 + 0.3j)
sc = m.SolverConfig(s, ell, 1e-8, 100000, True, 0)
out = {"grid": grid, "N": n, "s": s, "ell": ell}
for name, mat, rhs in (("real_fused", A, b), ("complex", Az, bz)):
    op = m.CsrOperator(mat, ctx)
    m.idrstab_solve(op, rhs, None, m.SolverConfig(s, ell, 1e-8, s + 2 * ell * (s + 1), True, 0))  # warm-up
    ctx.synchronize()
    t0 = time.perf_counter()
    r = m.idrstab_solve(op, rhs, None, sc)
    ctx.synchronize()
    dt = time.perf_counter() - t0
    rep = r.report
    res = np.linalg.norm(rhs - op.apply(r.x)) / np.linalg.norm(rhs)
    h = rep.residual_history  # point 0 is stamped after the fresh start (cut-space draw + Arnoldi)
    loop_ms = (h[-1].wall_ns - h[0].wall_ns) / 1e6
    out[name] = {"status": str(rep.status), "cycles": rep.cycles, "seconds": round(dt, 4),
                 "fresh_start_ms": round(h[0].wall_ns / 1e6, 2),
                 "ms_per_cycle": round(loop_ms / max(rep.cycles, 1), 3), "true_relres": float(res)}
print(json.dumps(out, indent=1))

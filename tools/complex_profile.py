"""Per-class kernel times of one complex128 solve (developer tool): SpMV vs the other primitives."""
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np  # noqa: E402

import paper_1604_06043_b200 as m  # noqa: E402
from paper_1604_06043_b200 import _capi  # noqa: E402
from paper_1604_06043_b200 import problems as pb  # noqa: E402

grid = int(sys.argv[1]) if len(sys.argv) > 1 else 128
s = int(sys.argv[2]) if len(sys.argv) > 2 else 8
ell = int(sys.argv[3]) if len(sys.argv) > 3 else 4
cfg = pb.config("c2", grid=grid)
A = cfg.matrix()
n = A.n_rows
ctx = m.Context(m.Lib(), 0)
lib = ctx.lib
vz = np.asarray(A.values, dtype=np.complex128)
rows = np.repeat(np.arange(n), np.diff(np.asarray(A.row_ptr)))
vz[np.asarray(A.col_idx) == rows] *= 1.0 + 0.05j
op = m.CsrOperator(m.CsrMatrix(n, n, A.row_ptr, A.col_idx, vz), ctx)
x0, f = cfg.sources()
b = cfg.first_rhs(x0, f) * (1.0 + 0.3j)
cyc = 3
sc = m.SolverConfig(s, ell, 1e-30, s + cyc * ell * (s + 1), True, 0)
m.idrstab_solve(op, b, None, sc)
lib.dll.mstab_profiling_reset()
lib.dll.mstab_profiling_enable(1)
t0 = time.perf_counter()
r = m.idrstab_solve(op, b, None, sc)
ctx.synchronize()
dt = time.perf_counter() - t0
lib.dll.mstab_profiling_enable(0)
stats = (_capi.KernelClassStatsC * 16)()
ncls = lib.dll.mstab_profiling_read(stats, 16)
print(f"N={n} s={s} ell={ell}: {r.report.cycles} cycles in {dt * 1e3:.1f} ms (profiling on)")
for i in range(ncls):
    st = stats[i]
    if st.launches:
        print(f"{lib.dll.mstab_kernel_class_name(i).decode():12s} launches {st.launches:6d}  total {st.total_ms:9.2f} ms  "
              f"avg {1e3 * st.total_ms / st.launches:8.1f} us  {st.total_bytes / st.total_ms / 1e6:8.1f} GB/s")

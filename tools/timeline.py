"""Phase timeline of the column-loop pair (SpMV of column q with its P^H reduction + LU, then the
rebuild of column q+1) from the ktimeline.cuh probes (developer tool; needs `make timeline`).

    python tools/timeline.py [config] [iters]
Prints, in microseconds from the SpMV's first CTA start: ramp (last CTA start), PDL wait release,
streaming done (first / last CTA), reduction done (the finisher CTA has every partial summed), dense
step done, SpMV end, then the rebuild's start / wait release / end. "ticket" and the reduce-phase
cycle count belong to the last-CTA scheme the constant-diagonal SpMV no longer uses (NaN there);
they still apply to the other SpMV forms."""
import ctypes as C
import json
import os
import sys

ROOT = __file__.rsplit("/tools/", 1)[0]
sys.path.insert(0, ROOT)
import paper_1604_06043_b200 as m  # noqa: E402
from paper_1604_06043_b200 import problems as pb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = pb.config(name)
lib = m.Lib(os.path.join(ROOT, "paper_1604_06043_b200", "libmstab_b200_tl.so"))
lib.dll.mstab_kernel_bench.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_int64, C.c_int32,
                                      C.POINTER(C.c_double), C.POINTER(C.c_double)]
lib.dll.mstab_timeline.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_uint64)]
ctx = m.Context(lib)
op = m.CsrOperator(cfg.matrix(), ctx)
us, by = C.c_double(), C.c_double()
out = (C.c_uint64 * 32)()
rows = []
for it in range(iters):
    lib.dll.mstab_timeline(ctx.h, 0, out)
    rc = lib.dll.mstab_kernel_bench(ctx.h, op.h, 8, cfg.s, cfg.ell, 1, C.byref(us), C.byref(by))
    assert rc == 0, lib.last_error()
    lib.dll.mstab_timeline(ctx.h, 1, out)
    t = list(out)
    t0 = t[0]
    rel = lambda i: (t[i] - t0) / 1e3 if t[i] not in (0, 2 ** 64 - 1) else float("nan")
    rows.append({
        "spmv_first_start": 0.0, "spmv_last_start": rel(1), "spmv_wait_first": rel(2), "spmv_wait_last": rel(3),
        "stream_done_first": rel(4), "stream_done_last": rel(5), "ticket": rel(6), "reduced": rel(7),
        "lu_done": rel(8), "spmv_end": rel(9),
        "tail_cycles_reduce": t[11] - t[10], "tail_cycles_lu": t[12] - t[11], "tail_cycles_total": t[13] - t[10],
        "rebuild_first_start": rel(16), "rebuild_last_start": rel(17), "rebuild_wait_first": rel(18),
        "rebuild_wait_last": rel(19), "rebuild_done_first": rel(20), "rebuild_done_last": rel(21)})
keys = list(rows[0])
med = {k: sorted(r[k] for r in rows[2:])[len(rows[2:]) // 2] for k in keys}
print(json.dumps({"config": name, "s": cfg.s, "median_of": len(rows) - 2, "us_or_cycles": med}, indent=1))

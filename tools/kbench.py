"""Kernel micro-benchmarks on a BASELINE operator shape (developer tool): mean us, GB/s, frac of HBM.
usage: python tools/kbench.py [config] [s] [ell] [kinds, e.g. 0,3] [iters] [grid]"""
import ctypes as C, json, os, sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1604_06043_b200 as m
from paper_1604_06043_b200 import problems as pb

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = pb.config(name, grid=int(sys.argv[6])) if len(sys.argv) > 6 else pb.config(name)
s = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else cfg.s
ell = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] != "-" else cfg.ell
kinds = [int(k) for k in sys.argv[4].split(",")] if len(sys.argv) > 4 else list(range(6))
iters = int(sys.argv[5]) if len(sys.argv) > 5 else 50
lib = m.Lib(os.environ["KBENCH_LIB"]) if os.environ.get("KBENCH_LIB") else m.Lib()
lib.dll.mstab_kernel_bench.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_int64, C.c_int32,
                                      C.POINTER(C.c_double), C.POINTER(C.c_double)]
ctx = m.Context(lib)
op = m.CsrOperator(cfg.matrix(), ctx)
hbm = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6538.6
names = ["spmv+ph+lu", "rebuild_top", "level_update", "deferred(k=ell-1)", "poly", "ls", "spmv+ph(store)", "lu(s x s)"]
for kind in kinds:
    us, by = C.c_double(), C.c_double()
    rc = lib.dll.mstab_kernel_bench(ctx.h, op.h, kind, s, ell, iters, C.byref(us), C.byref(by))
    if rc:
        print(names[kind], "error", lib.last_error(), flush=True)
        continue
    gbs = by.value / (us.value * 1e-6) / 1e9
    print(f"{name} s={s} ell={ell} {names[kind]:18s} {us.value:9.2f} us  {by.value / 1e6:8.1f} MB  {gbs:7.1f} GB/s"
          f"  {gbs / hbm:.3f}", flush=True)

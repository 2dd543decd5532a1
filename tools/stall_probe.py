"""Allocation / stall probe of the bench's chained sequence (developer tool): run with
MSTAB_DEBUG_STALL=<ms> MSTAB_DEBUG_ALLOC=1 to see which host-side step of a solve stalls."""
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch  # noqa: E402
import bench  # noqa: E402
import paper_1604_06043_b200 as m  # noqa: E402
from paper_1604_06043_b200 import problems as pb  # noqa: E402

cfg = pb.config(sys.argv[1] if len(sys.argv) > 1 else "c2")
lib = m.Lib()
ctx = m.Context(lib, 0)
op = m.CsrOperator(cfg.matrix(), ctx)
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 4):
    dev = rep % 2 == 0
    seq = bench.Sequence(m, cfg, op, ctx, seed=0, device_mode=dev, torch=torch, n_steps=16)
    t0 = time.perf_counter()
    for i in range(8):
        print(f"-- run {rep} step {i + 1}", file=sys.stderr, flush=True)
        seq.step()
    ctx.synchronize()
    ms = [round(r["solve_ms"]) for r in seq.log]
    print(f"run {rep} device_mode={dev} total {1e3 * (time.perf_counter() - t0):.0f} ms {ms}", flush=True)

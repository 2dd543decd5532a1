"""Where a right-hand side's wall time goes (developer tool): time to the first history point
(copy-in, validate, prologue), then per-cycle wall times, for the bench's own chained sequence."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
import bench  # noqa: E402
import paper_1604_06043_b200 as m  # noqa: E402
from paper_1604_06043_b200 import problems as pb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 12
cfg = pb.config(name)
lib = m.Lib()
ctx = m.Context(lib, 0)
op = m.CsrOperator(cfg.matrix(), ctx)
seq = bench.Sequence(m, cfg, op, ctx, seed=0, device_mode=True, torch=torch, n_steps=nrhs + 1)
for i in range(1, nrhs + 1):
    t0 = time.perf_counter()
    r = seq.step()
    ctx.synchronize()
    wall = time.perf_counter() - t0
    h = r.report.residual_history
    ns = [p.wall_ns for p in h]
    cyc = [round((b - a) / 1e6, 2) for a, b in zip(ns, ns[1:])]
    print(f"rhs {i:2d} {'restart' if seq.log[-1]['restart'] else '       '} step {wall * 1e3:8.2f} ms  solve "
          f"{seq.log[-1]['solve_ms']:8.2f}  to first point {ns[0] / 1e6:7.2f}  total in report {r.report.wall_ns_total / 1e6:8.2f}  cycles {cyc}",
          flush=True)

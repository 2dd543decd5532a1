"""Host<->device copy rates (developer tool): torch's copies vs the C-ABI's, same pinned buffers."""
import sys, time
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np
import torch
import paper_1604_06043_b200 as m
from paper_1604_06043_b200 import problems as pb

n = 1 << 21
h = torch.empty(n, dtype=torch.float64).pin_memory()
hp = torch.empty(n, dtype=torch.float64)  # pageable
d = torch.empty(n, dtype=torch.float64, device="cuda")
for name, src in (("pinned", h), ("pageable", hp)):
    for _ in range(3):
        d.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        d.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    for _ in range(10):
        src.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"torch {name}: H2D {8*n*10/(t1-t0)/1e9:.1f} GB/s  D2H {8*n*10/(t2-t1)/1e9:.1f} GB/s", flush=True)
cfg = pb.config("c2", grid=128)
ctx = m.Context(m.Lib(), 0)
op = m.CsrOperator(cfg.matrix(), ctx)
x = np.ones(n)
ctx.lib.dll.mstab_operator_apply  # noqa: B018
hn = h.numpy()
for name, buf in (("pinned", hn), ("pageable", hp.numpy())):
    buf[:] = 1.0
    out = np.empty_like(buf) if name == "pageable" else torch.empty(n, dtype=torch.float64).pin_memory().numpy()
    op.apply(buf, out)
    t0 = time.perf_counter()
    for _ in range(10):
        op.apply(buf, out)
    t1 = time.perf_counter()
    print(f"C-ABI apply with host {name} buffers (H2D + SpMV + D2H): {1e3*(t1-t0)/10:.3f} ms", flush=True)

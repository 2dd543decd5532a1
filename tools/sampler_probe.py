"""How much does clock sampling perturb the timed region? (developer tool) Runs the bench's c2
sequence under: no sampler, NVML clock only, NVML throttle reasons only, NVML both at 50 ms and at
500 ms, and the recipe's nvidia-smi child. Prints per-mode total and worst per-RHS solve time."""
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
import bench  # noqa: E402
import paper_1604_06043_b200 as m  # noqa: E402
from paper_1604_06043_b200 import problems as pb  # noqa: E402
import pynvml  # noqa: E402

cfg = pb.config("c2")
lib = m.Lib()
ctx = m.Context(lib, 0)
op = m.CsrOperator(cfg.matrix(), ctx)
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)


def run(label, sampler):
    seq = bench.Sequence(m, cfg, op, ctx, seed=0, device_mode=True, torch=torch, n_steps=16)
    for _ in range(3):
        seq.step()
    ctx.synchronize()
    stop = [False]
    n = [0]
    th = None
    proc = None
    if callable(sampler):
        def loop():
            while not stop[0]:
                sampler()
                n[0] += 1
                time.sleep(period)
        th = threading.Thread(target=loop, daemon=True)
        th.start()
    elif sampler == "smi":
        proc = subprocess.Popen(["nvidia-smi", "--id=0", f"--query-gpu={bench.Clocks.Q}", "--format=csv,noheader,nounits",
                                 "-lms", "200"], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        time.sleep(1.0)
    t0 = time.perf_counter()
    for _ in range(10):
        seq.step()
    ctx.synchronize()
    dt = time.perf_counter() - t0
    stop[0] = True
    if th:
        th.join()
    if proc:
        proc.terminate()
    ms = [r["solve_ms"] for r in seq.log[3:]]
    print(f"{label:34s} total {dt * 1e3:8.1f} ms  worst solve {max(ms):7.1f} ms  samples {n[0]:3d}  {[round(v) for v in ms]}", flush=True)


period = 0.05
run("no sampler", None)
run("nvml clock only, 50 ms", lambda: pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
run("nvml reasons only, 50 ms", lambda: pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))
run("nvml clock+reasons, 50 ms", lambda: (pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                         pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
period = 0.5
run("nvml clock+reasons, 500 ms", lambda: (pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                          pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
run("no sampler (again)", None)
run("nvidia-smi child -lms 200", "smi")
run("no sampler (after smi)", None)

#!/usr/bin/env python
"""bench.py — solved RHS/s over the BASELINE c2 system sequence on B200.

Workload (BASELINE.json configs[1], builder-defined details in SURVEY.md §8(d) / DESIGN.md §5):
3-D convection-diffusion 128^3 (N = 2,097,152, 7-point first-order upwind, beta = (1,.5,.25)*200,
h^2-scaled implicit Euler, dt = 1e-2), a chained right-hand-side sequence b_{i+1} = h^2(x_i/dt + f),
M(8,4)stab with tol 1e-8 on the true residual (true_residual_each_cycle), recycle hand-off at half
tolerance. A STEP is one right-hand side of that sequence: the whole mstab_solve (validate, cycles,
fetch, hand-off); a hand-off rejected by validate (StaleData, recycle.cpp:73) is re-solved fresh.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Arms:
  b200 (default)  value: device-resident inputs (b, x in HBM), CUDA events on the solver stream;
                  e2e:   the same sequence through the C-ABI with HOST b/x (H2D + D2H every step).
  reference       the unmodified reference (oracle/_ref, compiled from its own sources) advancing its
                  own solve loop on the same c2 system one level iteration per step, 1 host core.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "solved RHS/sec over a system sequence; SpMV+block-kernel HBM GB/s vs roofline"
UNIT = "RHS/s"
REF_LIB = ROOT / "oracle" / "_ref" / "libmstab_ref.so"
CYCLES_FILE = ROOT / "profiles" / "sequence_cycles.json"
NCU_FILE = ROOT / "profiles" / "ncu_traffic.json"


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"], "measured"
    except Exception:
        return 6650.0, "fallback"


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def workload_desc(cfg, A):
    ws_gb = (2 * (2 + 2 * cfg.s) + cfg.ell * (cfg.s + 1) + 1 + cfg.s) * cfg.N * 8 / 1e9
    if cfg.kind == "convdiff":
        what = (f"{cfg.dim}-D conv-diff {cfg.grid}^{cfg.dim} {cfg.stencil}-pt upwind, beta={tuple(cfg.beta)}, "
                f"implicit-Euler RHS sequence b_(i+1) = h^2(x_i/dt + f)")
    else:
        what = (f"random banded N={cfg.N}, 27 nnz/row, half-width {cfg.half_width}, diagonally dominant, "
                f"RHS sequence b_(i+1) = x_i + 0.1 g_i")
    return {
        "workload": f"{cfg.name}: {what}, M({cfg.s},{cfg.ell})stab tol 1e-8 (true residual), fetch at half tolerance",
        "N": int(A.n_rows), "nnz": int(A.nnz()), "s": cfg.s, "ell": cfg.ell, "sequence_len": cfg.n_rhs,
        "l2": f"working set ~{ws_gb:.2f} GB of N-vectors vs 126 MB L2"
              + (" (no flush needed)" if ws_gb > 1.0 else " (L2-resident: latency-bound config)"),
    }


# ---- clocks sampling (B200_PROFILING.md) -------------------------------------------------------
class Clocks:
    """SM clock and throttle reasons sampled DURING the timed region (the recipe's fields:
    clocks.sm, clocks.max.sm, clocks_event_reasons.*). Sampled in-process through NVML (pynvml)
    every 50 ms: the recipe's `nvidia-smi --query-gpu=... -lms 200` child reads the same NVML
    counters, but its start-up and its heavier per-sample queries stalled solves on the device by
    60-300 ms on this pool (r02: per-RHS solve times of 121 / 293 / 363 ms against 32 ms with the
    child running, none without it), which is measurement noise, not workload. The child is the
    fallback when pynvml is missing. The sampler starts before the warm-up; only samples inside
    the timed window are summarised."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device):
        self.device, self.rows, self.proc, self.stop, self.thread, self.source = device, [], None, False, None, None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            # CUDA_VISIBLE_DEVICES remaps ordinals: resolve the NVML handle through the PCI bus id
            import torch
            pr = torch.cuda.get_device_properties(self.device)
            bus, dom, dev = getattr(pr, "pci_bus_id", -1), getattr(pr, "pci_domain_id", 0), getattr(pr, "pci_device_id", 0)
            try:
                h = pynvml.nvmlDeviceGetHandleByPciBusId(f"{dom:08X}:{bus:02X}:{dev:02X}.0".encode())
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            masks = [pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                     pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap]

            def loop():
                while not self.stop:
                    try:
                        sm = float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        bits = int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))
                        self.rows.append([time.perf_counter(), str(self.device), str(sm), str(mx), "", ""]
                                         + ["Active" if bits & mk else "Not Active" for mk in masks])
                    except Exception:
                        pass
                    time.sleep(0.05)

            self.thread = threading.Thread(target=loop, daemon=True)
            self.thread.start()
            self.source = "nvml in-process, 50 ms"
            return self
        except Exception:
            self.thread = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
            self.source = "nvidia-smi -lms 200"
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([time.perf_counter()] + [c.strip() for c in line.split(",")])

    def mark(self):
        """Host time stamp for windowing the samples (perf_counter, like the rows)."""
        return time.perf_counter()

    def __exit__(self, *a):
        self.stop = True
        if self.thread:
            self.thread.join(timeout=2)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t0=None, t1=None):
        """Median SM clock and throttle reasons of the samples taken inside [t0, t1] (the timed region)."""
        rows = [r[1:] for r in self.rows if (t0 is None or r[0] >= t0) and (t1 is None or r[0] <= t1 + 0.25)]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock samples"], "samples": 0,
                    "source": self.source}
        sm = [float(r[1]) for r in rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[i] for r in rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "source": self.source}


# ---- the sequence driver (caller side of the hot path; reference harness.cpp:192-265) ----------
class Sequence:
    """One chained sequence. With a row-slab operator (N > 1 GPUs) every vector here is the
    rank's own rows [lo, hi) and the solve calls are collective."""

    def __init__(self, m, cfg, op, ctx, seed, device_mode, torch=None, rows=None, n_steps=64):
        self.m, self.cfg, self.op, self.ctx, self.torch = m, cfg, op, ctx, torch
        cfg.seed = seed
        lo, hi = rows if rows is not None else (0, cfg.N)
        self.lo, self.hi = lo, hi
        self.sc = m.SolverConfig(cfg.s, cfg.ell, cfg.tol, 100000, True, 0)
        self.fp = m.FetchPolicy.at_half_tolerance()
        self.device_mode = device_mode
        self.rec = None
        self.restarts = 0
        self.log = []
        self.i = 1  # 1-based index of the next solve in the sequence
        N = hi - lo
        if cfg.kind == "convdiff":
            x0, f = cfg.sources()
            self.f = np.ascontiguousarray(f[lo:hi])
            b0 = np.ascontiguousarray(cfg.first_rhs(x0, f)[lo:hi])
        else:  # banded: g_i drawn up front (host RNG outside the timed region)
            from paper_1604_06043_b200 import problems as pb
            b0 = np.ascontiguousarray(cfg.first_rhs()[lo:hi])
            self.g = [np.ascontiguousarray(pb.normal(1000 + cfg.seed + i, cfg.N)[lo:hi])
                      for i in range(1, n_steps + 1)]
        if device_mode:
            dev = torch.device("cuda", torch.cuda.current_device())
            if cfg.kind == "convdiff":
                self.f_d = torch.from_numpy(self.f).to(dev)
            else:
                self.g_d = [torch.from_numpy(g).to(dev) for g in self.g]
            self.x_d = torch.empty(N, dtype=torch.float64, device=dev)
            self.b_d = torch.from_numpy(b0).to(dev)
            torch.cuda.synchronize()
        else:
            if cfg.kind != "convdiff":
                self.g = [torch.from_numpy(g).pin_memory().numpy() for g in self.g]
            self.b_h = torch.from_numpy(b0).pin_memory().numpy()
            self.x_h = torch.empty(N, dtype=torch.float64).pin_memory().numpy()

    def step(self):
        m = self.m
        b = self.b_d if self.device_mode else self.b_h
        restarted = False
        t0 = time.perf_counter()
        r = None
        try:
            r = m.idrstab_solve(self.op, b, None, self.sc, self.rec, self.fp)
        except m.StaleData:
            restarted = True
        if restarted:  # outside the handler: the rejected hand-off and the traceback are released first
            self.restarts += 1
            self.rec = None
            r = m.idrstab_solve(self.op, b, None, self.sc, None, self.fp)
        rep = r._rep
        self.log.append({"cycles": int(rep.cycles), "status": int(rep.status), "restart": restarted,
                         "relres": float(rep.final_resnorm / rep.bnorm) if rep.bnorm else 0.0,
                         "solve_ms": round(1e3 * (time.perf_counter() - t0), 3)})
        self.rec = r.handoff()
        c = self.cfg
        dll, h = self.ctx.lib.dll, self.ctx.h
        nloc = self.hi - self.lo
        # next right-hand side through the C-ABI harness helpers (same rounding on both paths):
        # conv-diff b_{i+1} = h^2 (x_i/dt + f); banded b_{i+1} = x_i + 0.1 g_i
        if self.device_mode:
            r.x_into(self.x_d)  # D2D on the solver stream (synchronised)
            if c.kind == "convdiff":
                dll.mstab_harness_euler_rhs(h, nloc, self.x_d.data_ptr(), self.f_d.data_ptr(), c.dt, c.h2,
                                            self.b_d.data_ptr(), 1)
            else:
                dll.mstab_harness_axpby(h, nloc, self.x_d.data_ptr(), self.g_d[self.i - 1].data_ptr(), 0.1,
                                        self.b_d.data_ptr(), 1)
        else:
            r.x_into(self.x_h)  # D2H into pinned host memory
            if c.kind == "convdiff":
                dll.mstab_harness_euler_rhs(h, nloc, self.x_h.ctypes.data, self.f.ctypes.data, c.dt, c.h2,
                                            self.b_h.ctypes.data, 0)
            else:
                dll.mstab_harness_axpby(h, nloc, self.x_h.ctypes.data, self.g[self.i - 1].ctypes.data, 0.1,
                                        self.b_h.ctypes.data, 0)
        self.i += 1
        return r


def run_b200(args):
    import torch
    import paper_1604_06043_b200 as m
    from paper_1604_06043_b200 import _capi
    from paper_1604_06043_b200 import problems as pb

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    lib = m.Lib()
    ctx = m.Context(lib, local)
    cfg = pb.config(args.config, grid=args.grid)
    rows = None
    local_slabs = world > 1 and cfg.kind == "convdiff" and cfg.dim == 3 and not args.global_matrix
    A = None if local_slabs else cfg.matrix()
    if local_slabs:
        # Row-sharded stencil configs: every rank generates ONLY its z-slab of whole grid planes (c4:
        # 1.5e9 entries, 25 GB of int64 CSR, would not fit N times in host memory), the ranks exchange
        # their column spans and fold the reference fingerprint of the global matrix in three relays.
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(m.Context.nccl_unique_id(lib)), dtype=torch.uint8))
        torch.distributed.broadcast(uid, 0)
        ctx.set_comm_nccl(rank, world, bytes(uid.cpu().numpy().tobytes()))
        plane = cfg.grid * cfg.grid
        nplanes = cfg.N // plane
        slabs = np.array([(nplanes * r // world) * plane for r in range(world + 1)], dtype=np.int64)
        lo_r, hi_r = int(slabs[rank]), int(slabs[rank + 1])
        rp, ci, va = pb.convdiff_rows(cfg.dim, cfg.grid, cfg.stencil, cfg.beta, cfg.dt, lo_r, hi_r)
        nnz_t = torch.tensor([ci.size], dtype=torch.int64, device="cuda")
        nnz_all = [torch.zeros_like(nnz_t) for _ in range(world)]
        torch.distributed.all_gather(nnz_all, nnz_t)
        nnz_all = [int(t.item()) for t in nnz_all]
        span_t = torch.tensor(m.local_col_span(lo_r, hi_r, ci), dtype=torch.int64, device="cuda")
        spans = [torch.zeros_like(span_t) for _ in range(world)]
        torch.distributed.all_gather(spans, span_t)
        spans = np.array([t.cpu().numpy() for t in spans], dtype=np.int64)
        fp = m.distributed_fingerprint(lib, cfg.N, sum(nnz_all), rp, ci, va, sum(nnz_all[:rank]))
        op = m.CsrOperator.from_local_rows(cfg.N, slabs, rp, ci, va, spans, fp, ctx)
        rows = (lo_r, hi_r)

        class _Shape:  # what workload_desc reads
            n_rows = cfg.N

            @staticmethod
            def nnz():
                return sum(nnz_all)
        A = _Shape()
    elif world > 1:
        # Row-sharded solve of ONE sequence over the N GPUs (strong scaling):
        # z-slabs of whole grid planes, halo exchange + reductions over NCCL on the solver stream.
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(m.Context.nccl_unique_id(lib)), dtype=torch.uint8))
        torch.distributed.broadcast(uid, 0)
        ctx.set_comm_nccl(rank, world, bytes(uid.cpu().numpy().tobytes()))
        plane = cfg.grid * cfg.grid if cfg.kind == "convdiff" and cfg.dim == 3 else 1
        nplanes = cfg.N // plane
        slabs = np.array([(nplanes * r // world) * plane for r in range(world + 1)], dtype=np.int64)
        op = m.CsrOperator(A, ctx, slabs=slabs)
        rows = (int(slabs[rank]), int(slabs[rank + 1]))
    else:
        op = m.CsrOperator(A, ctx)
    stream = torch.cuda.ExternalStream(ctx.stream)
    N = cfg.N

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    # ---- value: device-resident inputs -------------------------------------------------------
    seq = Sequence(m, cfg, op, ctx, seed=0, device_mode=True, torch=torch, rows=rows,
                   n_steps=args.warmup + 2 * args.steps + 1)
    with Clocks(local) as clk:  # sampling from before the warm-up; only the timed window is summarised
        for _ in range(args.warmup):
            seq.step()
        barrier()
        torch.cuda.synchronize()
        ctx.synchronize()
        lib.dll.mstab_profiling_reset()
        lib.dll.mstab_profiling_enable(1 if args.profile == "timed" else 0)
        l0 = lib.dll.mstab_launch_count()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clk_t0 = clk.mark()
        ev0.record(stream)
        for _ in range(args.steps):
            seq.step()
        ev1.record(stream)
        ev1.synchronize()
        clk_t1 = clk.mark()
    launches = int(lib.dll.mstab_launch_count() - l0)
    if args.profile == "after":  # per-kernel events on K more steps of the same sequence
        lib.dll.mstab_profiling_enable(1)
        for _ in range(args.steps):
            seq.step()
        ctx.synchronize()
    lib.dll.mstab_profiling_enable(0)
    stats = (_capi.KernelClassStatsC * 16)()
    ncls = lib.dll.mstab_profiling_read(stats, 16)
    ms = ev0.elapsed_time(ev1)
    barrier()
    ms_max = max_over_ranks(ms)
    timed = seq.log[args.warmup:args.warmup + args.steps]
    value = args.steps / (ms_max / 1e3)  # one sequence over all ranks: whole-job RHS/s

    # ---- e2e: host buffers through the C-ABI --------------------------------------------------
    seq.rec = None  # the device-resident sequence is over: its hand-off blocks go back to the library
    seq_h = Sequence(m, cfg, op, ctx, seed=0, device_mode=False, torch=torch, rows=rows,
                     n_steps=args.warmup + args.steps + 1)
    for _ in range(args.warmup):
        seq_h.step()
    barrier()
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        seq_h.step()
    e1.record(stream)
    e1.synchronize()
    ems = max_over_ranks(e0.elapsed_time(e1))
    e2e = {"value": args.steps / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": 8 * N,
           "d2h_bytes_per_step": 8 * N, "per_rhs": seq_h.log[args.warmup:args.warmup + args.steps]}

    # ---- per-kernel roofline of the timed region ---------------------------------------------
    hbm, hbm_src = peaks()
    kernels = {}
    total_ms = sum(stats[i].total_ms for i in range(ncls))
    for i in range(ncls):
        s = stats[i]
        if s.launches == 0:
            continue
        avg_ms = s.total_ms / s.launches
        gbs = (s.total_bytes / s.launches) / (avg_ms / 1e3) / 1e9 if avg_ms > 0 else 0.0
        kernels[lib.dll.mstab_kernel_class_name(i).decode()] = {
            "launches": int(s.launches), "avg_us": round(avg_ms * 1e3, 3),
            "bytes_per_launch": s.total_bytes / s.launches, "achieved_gbs": round(gbs, 1),
            "frac": round(gbs / hbm, 4), "share_of_kernel_time": round(s.total_ms / total_ms, 4)}
    dom = "spmv_ph"
    traffic = ncu_us = None
    if NCU_FILE.exists():
        try:
            rec = json.loads(NCU_FILE.read_text()).get(args.config, {})
            traffic, ncu_us = rec.get(dom), rec.get(dom + "_us")
        except Exception:
            traffic = ncu_us = None
    bpl = kernels.get(dom, {}).get("bytes_per_launch")
    roof = {"bound": "hbm", "kernel": dom, "achieved": kernels.get(dom, {}).get("achieved_gbs"),
            "peak": hbm, "peak_source": hbm_src, "unit": "GB/s",
            "frac": kernels.get(dom, {}).get("frac"), "traffic": traffic,
            "bytes_per_launch": bpl}
    if world == 1:
        # The same kernel timed ALONE: 50 back-to-back launches between one CUDA-event pair on the
        # solver stream (mstab_kernel_bench), programmatic dependent launch intact. The in-sequence
        # figure above brackets every launch with event nodes, which removes that overlap (~6 us).
        try:
            kus, kby = C.c_double(), C.c_double()
            lib.dll.mstab_kernel_bench.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_int64, C.c_int32,
                                                  C.POINTER(C.c_double), C.POINTER(C.c_double)]
            if lib.dll.mstab_kernel_bench(ctx.h, op.h, 0, cfg.s, cfg.ell, 50, C.byref(kus), C.byref(kby)) == 0:
                roof["back_to_back"] = {"us": round(kus.value, 3), "bytes_per_launch": kby.value,
                                        "frac": round(kby.value / (kus.value * 1e-6) / (hbm * 1e9), 4),
                                        "how": "50 launches of the SpMV + P^H + dense-step kernel, one event pair"}
        except Exception as e:  # the headline does not depend on it
            roof["back_to_back"] = {"error": str(e)}
    if ncu_us and bpl:  # the same algorithmic bytes over the committed ncu launch duration (profiles/)
        roof["ncu"] = {"us": ncu_us, "frac": round(bpl / (ncu_us * 1e-6) / (hbm * 1e9), 4),
                       "source": "profiles/ncu_traffic.json"}

    mean_cycles = float(np.mean([r["cycles"] for r in timed])) if timed else None
    bad = [i + args.warmup + 1 for i, r in enumerate(timed) if r["status"] != 0]
    timed_restarts = sum(1 for r in timed if r["restart"])

    # ---- the whole sequence (RHS/s over ALL n_rhs systems, fresh RHS 1 included) ----
    full = None
    if not args.no_full_sequence:
        # a fresh context on one GPU: no cached P, no captured cycle graphs (cold start); the bench
        # context first gives its workspace back (c4: 37 GB of cycle vectors per context)
        seq_h.rec = None
        if world == 1:
            ctx.trim()
        ctx_f, op_f = (m.Context(lib, local), None) if world == 1 else (ctx, op)
        if op_f is None:
            op_f = m.CsrOperator(A, ctx_f)
        stream_f = torch.cuda.ExternalStream(ctx_f.stream)
        seq_f = Sequence(m, cfg, op_f, ctx_f, seed=0, device_mode=True, torch=torch, rows=rows,
                         n_steps=cfg.n_rhs + 1)
        barrier()
        ctx_f.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream_f)
        for _ in range(cfg.n_rhs):
            seq_f.step()
        f1.record(stream_f)
        f1.synchronize()
        fms = max_over_ranks(f0.elapsed_time(f1))
        full = {"rhs": cfg.n_rhs, "seconds": round(fms / 1e3, 4), "rhs_per_s": round(cfg.n_rhs / (fms / 1e3), 4),
                "restarts": seq_f.restarts, "total_cycles": int(sum(r["cycles"] for r in seq_f.log)),
                "non_converged": [i + 1 for i, r in enumerate(seq_f.log) if r["status"] != 0],
                "first_rhs": seq_f.log[:2],
                "note": "device-resident, all systems of the sequence including the fresh IDRstab solve of RHS 1 "
                        "(make_cut_space + Arnoldi) from a fresh context (no cached P, cycle graphs captured "
                        "inside the timed region)" + ("" if world == 1 else "; row-sharded: the bench context")}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, A, mean_cycles, steps=args.cpu_levels)
    if rank == 0:
        out = {
            "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generators, DESIGN.md §5)",
            "config": dict(workload_desc(cfg, A), parallelism=(f"row-slab{world}: one sequence, z-slabs, NCCL "
                                                              f"halo + allreduce" if world > 1 else "single GPU"),
                           rhs_range=[args.warmup + 1, args.warmup + args.steps]),
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(clk_t0, clk_t1), "kernels": kernels,
            "sequence": {"mean_cycles_per_rhs": mean_cycles, "restarts": seq.restarts,
                         "restarts_in_timed_window": timed_restarts,
                         "max_true_relres": max(r["relres"] for r in timed) if timed else None,
                         "per_rhs": timed},
            "sequence_full": full,
            "reference_per_rhs": reference_rows(cfg),
            "build_id": lib.build_id,
        }
        if bad:
            out["valid"] = False
            out["invalid_reason"] = f"RHS {bad} of the timed window did not converge"
        print(json.dumps(out), flush=True)
        if args.write_cycles:
            CYCLES_FILE.write_text(json.dumps({args.config: {"mean_cycles_per_rhs": mean_cycles,
                                                              "rhs_range": out["config"]["rhs_range"],
                                                              "per_rhs": [r["cycles"] for r in timed]}}, indent=1))
    if world > 1:
        torch.distributed.destroy_process_group()


# ---- the reference arm ------------------------------------------------------------------------
def ref_sampler(cfg, A):
    import ctypes as C

    import paper_1604_06043_b200 as m
    lib = m.Lib(REF_LIB)
    lib.dll.mstab_ref_sample_create.restype = C.c_void_p
    lib.dll.mstab_ref_sample_create.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_int64, C.c_int64, C.c_uint64]
    lib.dll.mstab_ref_sample_step.argtypes = [C.c_void_p]
    lib.dll.mstab_ref_sample_destroy.argtypes = [C.c_void_p]
    ctx = m.Context(lib)
    op = m.CsrOperator(A, ctx)
    x0, f = cfg.sources()
    b = cfg.first_rhs(x0, f)
    h = lib.dll.mstab_ref_sample_create(op.h, b.ctypes.data_as(C.POINTER(C.c_double)), cfg.s, cfg.ell, 0)
    if not h:
        raise RuntimeError("reference sample init failed: " + lib.last_error())
    return lib, op, h


def reference_rows(cfg):
    """The reference's own per-system rows for the first systems of this sequence (cycles, true
    relative residual, wall time on 1 core of the CPU container), from the corpus
    tools/ref_fixtures.py wrote (tests/golden/fullsize/<config>.json)."""
    path = ROOT / "tests" / "golden" / "fullsize" / f"{cfg.name}.json"
    if cfg.grid and cfg.name in ("c4",):
        path = ROOT / "tests" / "golden" / "fullsize" / f"{cfg.name}_{cfg.grid}.json"
    if cfg.name == "c5":
        path = ROOT / "tests" / "golden" / "fullsize" / "c5_42.json"
    try:
        d = json.loads(path.read_text())
    except Exception:
        return None
    if d.get("grid") != cfg.grid or d.get("s") != cfg.s or d.get("ell") != cfg.ell:
        return None
    return {"source": f"tests/golden/fullsize/{path.name} (oracle/_ref, 1 core, CPU container)",
            "per_rhs": [{"rhs": r["rhs"], "kind": r["kind"], "cycles": r["cycles"], "h_mv": r["h_mv"],
                         "true_relres": r["true_relres"], "seconds": round(r["seconds"], 2)}
                        for r in d["systems"]]}


def workload_cycles(cfg, measured):
    if measured:
        return measured, "measured in this run (b200 arm, same sequence positions)"
    ref = reference_rows(cfg)
    if ref:
        rec = [r["cycles"] for r in ref["per_rhs"] if r["kind"] == "mstab"]
        if rec:
            return float(np.mean(rec)), f"the reference's own recycled solves ({ref['source']})"
    try:
        d = json.loads(CYCLES_FILE.read_text())[cfg.name]
        return d["mean_cycles_per_rhs"], f"profiles/{CYCLES_FILE.name} (b200 arm, RHS {d['rhs_range']})"
    except Exception:
        return 11.0, "fresh-solve cycle count of the c2 system (no sequence record)"


def cpu_baseline(cfg, A, mean_cycles, steps):
    """The reference's own loop on this system, `steps` level iterations on 1 core."""
    lib, op, h = ref_sampler(cfg, A)
    t = []
    for _ in range(steps):
        t0 = time.perf_counter()
        lib.dll.mstab_ref_sample_step(h)
        t.append(time.perf_counter() - t0)
    lib.dll.mstab_ref_sample_destroy(h)
    cyc, src = workload_cycles(cfg, mean_cycles)
    per_level = sum(t) / len(t)
    rhs_s = 1.0 / (cyc * cfg.ell * per_level)
    return {"value": rhs_s, "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"{steps} level iterations of the reference solve loop (oracle/_ref, unmodified sources) on "
                      f"the {cfg.name} system, {per_level:.2f} s each; RHS time = cycles/RHS ({cyc:.2f}, {src}) x "
                      f"ell ({cfg.ell}) x level time (validate/poly/true-residual MVs not charged: favours the CPU)",
            "cpu_model": cpu_model()}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip() + f" ({os.cpu_count()} cores)"
    except Exception:
        pass
    return None


def run_reference(args):
    from paper_1604_06043_b200 import problems as pb
    rank, world, _ = dist_env()
    if rank != 0:
        return
    if not REF_LIB.exists():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libmstab_ref.so not built"}))
        return
    cfg = pb.config(args.config, grid=args.grid)
    A = cfg.matrix()
    lib, op, h = ref_sampler(cfg, A)
    for _ in range(args.warmup):
        lib.dll.mstab_ref_sample_step(h)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        lib.dll.mstab_ref_sample_step(h)
    dt = time.perf_counter() - t0
    lib.dll.mstab_ref_sample_destroy(h)
    cyc, src = workload_cycles(cfg, None)
    value = args.steps / (cyc * cfg.ell * dt)
    out = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded generators, DESIGN.md §5)",
           "config": dict(workload_desc(cfg, A), parallelism="1 host core (the reference is single-threaded)"),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "reference",
                            "sample": f"each step = one level iteration of the reference solve loop on the {cfg.name} "
                                      f"system; RHS time = cycles/RHS ({cyc:.2f}, {src}) x ell x level time",
                            "cpu_model": cpu_model()},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--grid", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-levels", type=int, default=2)
    ap.add_argument("--write-cycles", action="store_true")
    ap.add_argument("--no-full-sequence", action="store_true")
    ap.add_argument("--global-matrix", action="store_true",
                    help="row-sharded runs: every rank builds the global CSR (the r01 path) instead of its own slab")
    ap.add_argument("--profile", default="after", choices=["timed", "after", "off"],  # graphs: events are nodes
                    help="per-kernel CUDA events on K extra steps after the timed region (default), or inside it")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()

"""TEST MODEL (not product code): a NumPy statement of the row-slab partition of the Mstab path
 that the CPU tests check the slab logic against; the product's planner is the
C++ one (csrc/solver.cpp make_operator_slab / make_operator_slab_local).

Row-slab partition of the Mstab path across the GPUs of one node.

Every operation of the solve loop except the SpMV is row-local (idrstab.cpp:105-191: the BiCG
updates, column rebuilds and the poly combination touch one row at a time); the SpMV needs the
halo rows of x owned by the neighbours, and the length-N dots (Pᴴ[V|r], the least-squares
factor, ‖r‖) need a sum over ranks. This module is the host-side plan:

* `plan_rows`      contiguous row slabs, balanced by nonzeros, aligned to `align` rows (a grid
                   plane for the 3-D stencils, so halos are whole planes);
* `RankPlan`       the local CSR of one rank with columns remapped to [left halo | own | right
                   halo], and the send/receive ranges of its halo exchange;
* `reduction_schedule`  the fused allreduce payloads of one cycle (what the device path sums with
                   one NCCL allreduce per reduction point instead of one per dot).

`halo_spmv` runs one distributed SpMV with any torch.distributed backend (gloo on CPU in the
tests, NCCL on the GPUs); it is bit-identical to the global SpMV because each row is still
accumulated from 0 in CSR order.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Tuple

import numpy as np


def plan_rows(row_ptr: np.ndarray, world: int, align: int = 1) -> List[Tuple[int, int]]:
    """Contiguous [start, end) row slabs with ~equal nonzeros, boundaries multiples of `align`."""
    n = len(row_ptr) - 1
    if world < 1 or n < 1:
        raise ValueError("need world >= 1 and n >= 1")
    nnz = int(row_ptr[-1])
    bounds = [0]
    for r in range(1, world):
        target = nnz * r / world
        i = int(np.searchsorted(row_ptr, target))
        i = min(max((i // align) * align, bounds[-1]), n)
        bounds.append(i)
    bounds.append(n)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


@dataclass
class RankPlan:
    rank: int
    start: int                 # first owned row
    end: int                   # one past the last owned row
    halo_lo: int               # first global column of the left halo (<= start)
    halo_hi: int               # one past the last global column of the right halo (>= end)
    row_ptr: np.ndarray        # local CSR (rows start..end), columns local to [halo_lo, halo_hi)
    col_idx: np.ndarray
    values: np.ndarray
    sends: List[Tuple[int, int, int]]   # (peer, global_start, global_end) of owned rows to send
    recvs: List[Tuple[int, int, int]]   # (peer, global_start, global_end) of halo rows to receive

    @property
    def n_local(self) -> int:
        return self.end - self.start

    @property
    def ext_len(self) -> int:
        return self.halo_hi - self.halo_lo


def rank_plan(row_ptr, col_idx, values, slabs: List[Tuple[int, int]], rank: int) -> RankPlan:
    """Local operator and halo ranges of `rank`. The halo is the column range the owned rows
    reference outside the slab; it must lie within the neighbouring slabs' rows (true for the
    banded/stencil BASELINE matrices), each received from its owner."""
    start, end = slabs[rank]
    lo, hi = int(row_ptr[start]), int(row_ptr[end])
    cols = np.asarray(col_idx[lo:hi], dtype=np.int64)
    halo_lo = int(min(cols.min(), start)) if cols.size else start
    halo_hi = int(max(cols.max() + 1, end)) if cols.size else end
    recvs, sends = [], []
    for peer, (ps, pe) in enumerate(slabs):
        if peer == rank:
            continue
        a, b = max(ps, halo_lo), min(pe, halo_hi)
        if a < b:
            recvs.append((peer, a, b))
    # what each peer needs from me: my rows inside its halo range
    for peer, (ps, pe) in enumerate(slabs):
        if peer == rank or pe <= ps:
            continue
        plo, phi = int(row_ptr[ps]), int(row_ptr[pe])
        pc = np.asarray(col_idx[plo:phi], dtype=np.int64)
        if pc.size == 0:
            continue
        a, b = max(start, int(min(pc.min(), ps))), min(end, int(max(pc.max() + 1, pe)))
        if a < b:
            sends.append((peer, a, b))
    local_rp = np.asarray(row_ptr[start:end + 1], dtype=np.int64) - lo
    return RankPlan(rank, start, end, halo_lo, halo_hi, local_rp, cols - halo_lo,
                    np.asarray(values[lo:hi], dtype=np.float64), sends, recvs)


def local_spmv(plan: RankPlan, x_ext: np.ndarray) -> np.ndarray:
    """y = A_local x_ext, each row from 0 in CSR order (csr.cpp:103-113)."""
    y = np.empty(plan.n_local)
    rp, ci, va = plan.row_ptr, plan.col_idx, plan.values
    for i in range(plan.n_local):
        acc = 0.0
        for k in range(rp[i], rp[i + 1]):
            acc += va[k] * x_ext[ci[k]]
        y[i] = acc
    return y


def halo_exchange(plan: RankPlan, x_own: np.ndarray, dist) -> np.ndarray:
    """Extended vector [halo_lo, halo_hi) from the owned slice plus the neighbours' rows
    (point-to-point sends/receives in global order, deadlock-free with isend/irecv)."""
    import torch
    x_ext = np.zeros(plan.ext_len)
    x_ext[plan.start - plan.halo_lo:plan.end - plan.halo_lo] = x_own
    reqs, bufs = [], []
    for peer, a, b in plan.sends:
        t = torch.from_numpy(np.ascontiguousarray(x_own[a - plan.start:b - plan.start]))
        reqs.append(dist.isend(t, dst=peer))
        bufs.append(t)
    recv_bufs = []
    for peer, a, b in plan.recvs:
        t = torch.empty(b - a, dtype=torch.float64)
        reqs.append(dist.irecv(t, src=peer))
        recv_bufs.append((a, b, t))
    for r in reqs:
        r.wait()
    for a, b, t in recv_bufs:
        x_ext[a - plan.halo_lo:b - plan.halo_lo] = t.numpy()
    return x_ext


def halo_spmv(plan: RankPlan, x_own: np.ndarray, dist) -> np.ndarray:
    return local_spmv(plan, halo_exchange(plan, x_own, dist))


def reduction_schedule(s: int, ell: int, true_residual: bool = False) -> List[Tuple[str, int]]:
    """The reduction points of one cycle and the fp64 payload of each fused allreduce: what the
    single-GPU kernels reduce in their last CTA (kernels.h) becomes one allreduce per point."""
    sched = []
    for k in range(ell):
        sched.append((f"level{k}.rhs=P^H r^(k+1)", s))               # after step (b)
        for q in range(s):
            sched.append((f"level{k}.col{q}=P^H V^(k+1)_q", s))      # after each column SpMV
        if k >= 1:
            pass  # gamma_k uses the cached products: no extra reduction
    sched.append(("ls.R+colnorms", (ell + 1) * (ell + 2) // 2 + ell))  # TSQR factor + ||Z_j||^2
    sched.append(("poly.||r||^2,P^H r,P^H V", 1 + s + s * s))
    if true_residual:
        sched.append(("trueres.P^H r,||r||^2", s + 1))
    return sched


def allreduce_sum(vec: np.ndarray, dist) -> np.ndarray:
    import torch
    t = torch.from_numpy(np.ascontiguousarray(vec, dtype=np.float64))
    dist.all_reduce(t)
    return t.numpy()

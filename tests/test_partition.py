"""Row-slab sharding of the path — CPU, world size 2 over gloo."""
import os
import socket

import numpy as np
import pytest

import partition_model as pt
from paper_1604_06043_b200 import problems as pb


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_plan_rows_balanced_and_aligned():
    A = pb.config("c2", grid=12).matrix()
    n2 = 12 * 12
    for world in (1, 2, 3, 4, 8):
        slabs = pt.plan_rows(A.row_ptr, world, align=n2)
        assert slabs[0][0] == 0 and slabs[-1][1] == A.n_rows
        assert all(a % n2 == 0 for a, _ in slabs)
        assert all(slabs[i][1] == slabs[i + 1][0] for i in range(world - 1))


@pytest.mark.parametrize("world", [2, 3, 4])
def test_rank_plans_reassemble_the_global_spmv(world):
    """Serial check of the plans: gathering each rank's halo from the global vector and running
    the local SpMV reproduces the global SpMV bit-for-bit (CSR order is preserved)."""
    import oracle_c as oc
    cfg = pb.config("c3", grid=3000)
    cfg.half_width = 40
    A = cfg.matrix()
    x = np.random.default_rng(0).standard_normal(A.n_rows)
    ref = oc.Csr(A).apply(x)
    slabs = pt.plan_rows(A.row_ptr, world)
    out = np.empty_like(ref)
    for r in range(world):
        p = pt.rank_plan(A.row_ptr, A.col_idx, A.values, slabs, r)
        out[p.start:p.end] = pt.local_spmv(p, x[p.halo_lo:p.halo_hi])
        for peer, a, b in p.recvs:  # every halo row is owned by the peer it is received from
            assert slabs[peer][0] <= a < b <= slabs[peer][1]
    assert np.array_equal(out, ref)


def test_reduction_schedule_counts():
    sched = pt.reduction_schedule(8, 4, true_residual=True)
    # ell*(s+1) SpMV reductions + LS + poly + true residual: the allreduce count per cycle
    assert len(sched) == 4 * 9 + 3
    assert sched[-2][1] == 1 + 8 + 64


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = pb.config("c2", grid=10).matrix()
        slabs = pt.plan_rows(A.row_ptr, world, align=100)
        plan = pt.rank_plan(A.row_ptr, A.col_idx, A.values, slabs, rank)
        x = np.random.default_rng(7).standard_normal(A.n_rows)
        y = pt.halo_spmv(plan, x[plan.start:plan.end], dist)
        # distributed dot: partial + allreduce
        part = np.array([np.dot(y, x[plan.start:plan.end])])
        tot = pt.allreduce_sum(part, dist)
        q.put((rank, plan.start, plan.end, y, float(tot[0])))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_halo_spmv_and_allreduce():
    import multiprocessing as mp

    import oracle_c as oc
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A = pb.config("c2", grid=10).matrix()
    x = np.random.default_rng(7).standard_normal(A.n_rows)
    ref = oc.Csr(A).apply(x)
    y = np.empty_like(ref)
    totals = set()
    for rank, a, b, yl, tot in res:
        y[a:b] = yl
        totals.add(tot)
    assert np.array_equal(y, ref)                    # halo SpMV is bit-exact
    assert len(totals) == 1                          # every rank holds the same reduced bits
    assert abs(totals.pop() - float(np.dot(ref, x))) <= 1e-12 * abs(float(np.dot(ref, x)))


def _fp_worker(rank, world, port, q):
    import torch.distributed as dist

    import paper_1604_06043_b200 as m
    from conftest import REF_LIB
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # every rank keeps ONLY its rows (a slab of whole grid planes) and folds the reference
        # checksum of the global matrix in three relays over the ranks
        A = pb.config("c4", grid=10).matrix()
        slabs = pt.plan_rows(A.row_ptr, world, align=100)
        a, b = slabs[rank]
        rp = np.asarray(A.row_ptr, dtype=np.int64)
        loc_rp = rp[a:b + 1] - rp[a]
        ci = np.asarray(A.col_idx, dtype=np.int64)[rp[a]:rp[b]]
        va = np.asarray(A.values)[rp[a]:rp[b]]
        lib = m.Lib(str(REF_LIB))  # the fold is host code in both libraries; this one needs no GPU
        h = m.distributed_fingerprint(lib, A.n_rows, int(rp[-1]), loc_rp, ci, va, int(rp[a]))
        q.put((rank, h, m.local_col_span(a, b, ci)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_distributed_fingerprint_matches_the_global_checksum():
    """Rank-local rows only: the relayed FNV fold equals the reference's checksum of the whole
    matrix on every rank (csr.cpp:28-43), and the column spans describe one halo plane per side."""
    import multiprocessing as mp

    import oracle_c as oc
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_fp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A = pb.config("c4", grid=10).matrix()
    want = oc.Csr(A).fingerprint()
    assert [h for _, h, _ in res] == [want, want]
    (lo0, hi0), (lo1, hi1) = res[0][2], res[1][2]
    assert (lo0, hi0) == (0, 600) and (lo1, hi1) == (400, 1000)  # 27-point: exactly one halo plane per side

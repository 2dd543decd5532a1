"""Generates the golden fixtures in tests/golden/ by running the UNMODIFIED reference
(oracle/_ref/libmstab_ref.so, compiled from /root/reference by oracle/Makefile) through the C-ABI.

    python tests/golden/make_golden.py

Fixtures are small (N <= 4096) and store every float as its exact IEEE value (npz), so the tests
can demand bit-exact agreement from the C restatement oracle and the B200 element-wise kernels.
Covered (the reference's own known-answer tests):
  * kat_tridiag.npz   tridiag(2,3,1) N=40 finite termination (test_solvers.cpp:268-282), Mstab after
                      fetch (:341-366), l-mixing (:368-389), counter laws (:284-303, :391-409)
  * seq_small.npz     chained conv-diff / banded sequences with half-tolerance hand-off (§8(d))
  * kernels.npz       solve_small, least_squares_tall, make_cut_space, arnoldi_init cases
  * donor_tridiag30.mrd  a reference-written .mrd (recycle.cpp:85-126) for byte-level interop
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_1604_06043_b200 as m  # noqa: E402
from paper_1604_06043_b200 import problems as pb  # noqa: E402

OUT = Path(__file__).resolve().parent


def ref_ctx():
    return m.Context(m.Lib(ROOT / "oracle" / "_ref" / "libmstab_ref.so"))


def pack_result(prefix, r, out):
    rep = r.report
    out[prefix + "x"] = r.x
    out[prefix + "counters"] = np.array([rep.cycles, rep.h_mv, rep.h_mv_aux, rep.h_rd,
                                         {"Converged": 0, "MaxMV": 1, "Breakdown": 2}[rep.status]])
    out[prefix + "resnorms"] = np.array([h.resnorm for h in rep.residual_history])
    out[prefix + "levels"] = np.array([h.level for h in rep.residual_history])
    out[prefix + "mvs"] = np.array([h.mv for h in rep.residual_history])
    out[prefix + "taus"] = (np.concatenate(rep.omega_history).real if rep.omega_history else np.zeros(0))


def pack_recycle(prefix, d, out):
    out[prefix + "p"] = np.array(d.p)
    out[prefix + "u"] = np.array(d.u)
    out[prefix + "v"] = np.array(d.v)
    out[prefix + "omega"] = np.array(d.omega_history)
    out[prefix + "meta"] = np.array([d.level_J, d.s], dtype=np.int64)
    out[prefix + "fp"] = np.array([d.matrix_fingerprint], dtype=np.uint64)


def kat_tridiag(ctx):
    out = {}
    tri = m.CsrMatrix.tridiag(2.0, 3.0, 1.0, 40)
    op = m.CsrOperator(tri, ctx)
    b1, b2 = np.ones(40), pb.sinewave(40)
    out["b_sine40"] = b2
    for s in (2, 4):
        cfg = m.SolverConfig(s, 1, 1e-8, 100000, True, 1)
        pack_result(f"idr{s}_", m.idrstab_solve(op, b1, None, cfg), out)
        fp = m.FetchPolicy.at_cycle(19 if s == 2 else 9)
        donor = m.idrstab_solve(op, b1, None, cfg, None, fp)
        pack_recycle(f"donor{s}_", donor.fetched, out)
        pack_result(f"mstab{s}_", m.mstab_solve(op, b2, None, cfg, donor.fetched), out)
    for dl in (1, 2):
        dcfg = m.SolverConfig(4, dl, 1e-8, 100000, False, 1)
        donor = m.idrstab_solve(op, b1, None, dcfg, None, m.FetchPolicy.at_cycle(8 if dl == 1 else 4))
        for ul in (1, 2):
            pack_result(f"mix{dl}{ul}_", m.mstab_solve(op, b2, None, m.SolverConfig(4, ul, 1e-8, 100000, False, 1),
                                                         donor.fetched), out)
    tri200 = m.CsrMatrix.tridiag(2.0, 3.0, 1.0, 200)
    op200 = m.CsrOperator(tri200, ctx)
    ones200 = np.ones(200)
    for s in (2, 4):
        for ell in (1, 2):
            cfg = m.SolverConfig(s, ell, 1e-30, s + 5 * ell * (s + 1), False, 3)
            pack_result(f"law{s}{ell}_", m.idrstab_solve(op200, ones200, None, cfg), out)
    np.savez(OUT / "kat_tridiag.npz", **out)


def seq_small(ctx):
    out = {}
    cases = [("c1", 16, 5), ("c1", 32, 4), ("c2", 8, 3), ("c3", 2048, 3)]
    for name, grid, nrhs in cases:
        cfg = pb.config(name, grid=grid)
        if name == "c3":
            cfg.half_width = 64
        key = f"{name}_{grid}_"
        A = cfg.matrix()
        out[key + "rp"], out[key + "ci"], out[key + "va"] = A.row_ptr, A.col_idx, A.values
        op = m.CsrOperator(A, ctx)
        x0, f = cfg.sources()
        b = cfg.first_rhs(x0, f)
        sc = m.SolverConfig(cfg.s, cfg.ell, 1e-8, 100000, False, 0)
        fp = m.FetchPolicy.at_half_tolerance()
        rec = None
        for i in range(nrhs):
            k = f"{key}{i}_"
            out[k + "b"] = b
            if rec is not None:
                pack_recycle(k + "in_", rec, out)
            try:
                r = m.idrstab_solve(op, b, None, sc, rec, fp)
            except m.StaleData:
                # validate() rejects the hand-off (recycle.cpp:73): the reference lets StaleData
                # escape; the sequence driver restarts fresh (recorded as "restart")
                out[k + "stale"] = np.array([1])
                r = m.idrstab_solve(op, b, None, sc, None, fp)
            pack_result(k, r, out)
            if r.report.status == "Breakdown":
                break
            rec = r.handoff()
            b = cfg.next_rhs(i + 1, r.x, f)
        out[key + "count"] = np.array([i + 1])
    np.savez(OUT / "seq_small.npz", **out)


def kernels(ctx):
    out = {}
    rng = np.random.default_rng(20261020)
    for s in (1, 2, 3, 4, 8, 16):
        M = rng.standard_normal((s, s))
        rhs = rng.standard_normal(s)
        out[f"lu{s}_m"], out[f"lu{s}_rhs"] = M, rhs
        out[f"lu{s}_x"] = m.solve_small(M, rhs, ctx)
    sing = np.ones((3, 3))
    out["lu_sing_m"] = sing
    for n, ell in ((50, 1), (300, 2), (1000, 4), (4000, 8)):
        Z = rng.standard_normal((n, ell))
        r = rng.standard_normal(n)
        out[f"ls{n}_{ell}_z"], out[f"ls{n}_{ell}_r"] = Z, r
        out[f"ls{n}_{ell}_tau"] = m.least_squares_tall(Z, r, ctx)
    # a Krylov power basis (ill-conditioned, like the stabilisation block) and a rank-deficient one
    A = pb.config("c1", grid=16).matrix()
    op = m.CsrOperator(A, ctx)
    z = [rng.standard_normal(A.n_rows)]
    for _ in range(4):
        z.append(op.apply(z[-1]))
    Zk = np.stack(z[1:], axis=1)
    out["lsk_z"], out["lsk_r"] = Zk, z[0]
    out["lsk_tau"] = m.least_squares_tall(Zk, z[0], ctx)
    Zd = np.stack([z[1], z[2], 2.0 * z[1]], axis=1)
    out["lsdef_z"], out["lsdef_r"] = Zd, z[0]
    for n, s, seed in ((257, 1, 0), (257, 3, 7), (1000, 4, 11), (64, 8, 99)):
        out[f"cut{n}_{s}_{seed}"] = m.make_cut_space(n, s, seed, ctx)
    tri = m.CsrMatrix.tridiag(2.0, 3.0, 1.0, 8)
    opt = m.CsrOperator(tri, ctx)
    u, v, _ = m.arnoldi_init(opt, np.ones(8), 3, 2)
    out["arn_tri_u"], out["arn_tri_v"] = u, v
    eye = m.CsrMatrix.identity(6)
    ope = m.CsrOperator(eye, ctx)
    e1 = np.zeros(6)
    e1[0] = 1.0
    u, v, _ = m.arnoldi_init(ope, e1, 3, 4)
    out["arn_eye_u"], out["arn_eye_v"] = u, v
    out["normal_5"] = pb.normal(5, 1001)
    np.savez(OUT / "kernels.npz", **out)


def donor_mrd(ctx):
    tri = m.CsrMatrix.tridiag(2.0, 3.0, 1.0, 30)
    op = m.CsrOperator(tri, ctx)
    r = m.idrstab_solve(op, np.ones(30), None, m.SolverConfig(2, 1, 1e-8, 100000, False, 21), None,
                        m.FetchPolicy.at_cycle(4))
    m.save(r.fetched, OUT / "donor_tridiag30.mrd")


if __name__ == "__main__":
    ctx = ref_ctx()
    kat_tridiag(ctx)
    seq_small(ctx)
    kernels(ctx)
    donor_mrd(ctx)
    for p in sorted(OUT.glob("*.np*")) + sorted(OUT.glob("*.mrd")):
        print(p.name, p.stat().st_size)

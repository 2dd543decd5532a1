"""Pins the oracles before any GPU result is trusted (CPU only).

* the plain-C restatement (oracle/mstab_oracle.c) must reproduce the golden vectors written by the
  unmodified reference (tests/golden/make_golden.py) BIT-FOR-BIT;
* the compiled reference (oracle/_ref) must reproduce them too (it wrote them; this catches a
  stale or mis-built _ref before the GPU tests use it as the checker);
* both must satisfy the reference's own known-answer assertions (test_solvers.cpp:268-409,
  SURVEY.md §8(c)).
"""
import struct

import numpy as np
import pytest

import oracle_c as oc
from conftest import GOLDEN


def tri(n, a=2.0, b=3.0, c=1.0):
    import paper_1604_06043_b200 as m
    return m.CsrMatrix.tridiag(a, b, c, n)


def same(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b))


def check_result(res, g, prefix):
    c = g[prefix + "counters"]
    assert [res.cycles, res.h_mv, res.h_mv_aux, res.h_rd, res.status] == list(c), prefix
    assert same(res.x, g[prefix + "x"]), prefix
    assert same(res.resnorms, g[prefix + "resnorms"]), prefix
    assert same(res.hist[:, 2], g[prefix + "levels"]), prefix
    assert same(res.hist[:, 1], g[prefix + "mvs"]), prefix
    assert same(res.taus, g[prefix + "taus"]), prefix


def rec_from(g, prefix):
    meta = g[prefix + "meta"]
    return oc.Recycle(g[prefix + "p"], g[prefix + "u"], g[prefix + "v"], g[prefix + "omega"], int(meta[0]),
                      int(g[prefix + "fp"][0]))


# ---- known answers (test_solvers.cpp) -----------------------------------------------------------
def test_kat_finite_termination_tridiag40(golden_kat):
    c = oc.Csr(tri(40))
    for s, bound in ((2, 22), (4, 11)):
        r = oc.solve(c, np.ones(40), s=s, ell=1, true_residual=True, seed=1)
        check_result(r, golden_kat, f"idr{s}_")
        assert r.status == 0 and r.cycles <= bound
    # SURVEY.md §8(c) measured values: IDR(2)stab(1) 20 cycles / h_mv 62; IDR(4)stab(1) 10 / 54
    assert list(golden_kat["idr2_counters"][:2]) == [20, 62]
    assert list(golden_kat["idr4_counters"][:2]) == [10, 54]


def test_kat_mstab_after_fetch(golden_kat):
    c = oc.Csr(tri(40))
    b2 = golden_kat["b_sine40"]
    for s, cyc, bound in ((2, 19, 12), (4, 9, 5)):
        donor = oc.solve(c, np.ones(40), s=s, ell=1, true_residual=True, seed=1, fetch_kind=0, fetch_cycle=cyc)
        d = donor.fetched
        g = rec_from(golden_kat, f"donor{s}_")
        assert d.level_j == g.level_j == cyc
        assert same(d.u, g.u) and same(d.v, g.v) and same(d.p, g.p) and same(d.omega, g.omega)
        r = oc.solve(c, b2, s=s, ell=1, true_residual=True, seed=1, recycle=d)
        check_result(r, golden_kat, f"mstab{s}_")
        assert r.status == 0 and r.cycles <= bound
    assert list(golden_kat["mstab2_counters"][[0, 1, 3]]) == [11, 33, 41]
    assert list(golden_kat["mstab4_counters"][[0, 1, 3]]) == [4, 20, 43]


def test_kat_degree_agnostic_recycle(golden_kat):
    c = oc.Csr(tri(40))
    b2 = golden_kat["b_sine40"]
    for dl in (1, 2):
        donor = oc.solve(c, np.ones(40), s=4, ell=dl, seed=1, fetch_kind=0, fetch_cycle=8 if dl == 1 else 4)
        assert donor.fetched.level_j == 8
        for ul in (1, 2):
            r = oc.solve(c, b2, s=4, ell=ul, seed=1, recycle=donor.fetched)
            check_result(r, golden_kat, f"mix{dl}{ul}_")
            assert r.hist[-1, 2] <= (13 if ul == 1 else 14)


def test_kat_counter_laws(golden_kat):
    c = oc.Csr(tri(200))
    for s in (2, 4):
        for ell in (1, 2):
            r = oc.solve(c, np.ones(200), s=s, ell=ell, tol=1e-30, max_mv=s + 5 * ell * (s + 1), seed=3)
            check_result(r, golden_kat, f"law{s}{ell}_")
            assert r.cycles == 5 and r.h_mv == s + 5 * ell * (s + 1) and r.h_rd == 5 * ell * s


# ---- chained sequences, teacher-forced (same b_i, same incoming recycle data) --------------------
@pytest.mark.parametrize("key", ["c1_16_", "c1_32_", "c2_8_", "c3_2048_"])
def test_sequences_bit_exact(golden_seq, key):
    import paper_1604_06043_b200 as m
    g = golden_seq
    A = m.CsrMatrix(len(g[key + "rp"]) - 1, len(g[key + "rp"]) - 1, g[key + "rp"], g[key + "ci"], g[key + "va"])
    c = oc.Csr(A)
    from paper_1604_06043_b200 import problems as pb
    cfgname = key.split("_")[0]
    cfg = pb.config(cfgname)
    for i in range(int(g[key + "count"][0])):
        k = f"{key}{i}_"
        rec = rec_from(g, k + "in_") if (k + "in_meta") in g else None
        if rec is not None and (k + "stale") in g:
            rc, dev, _ = oc.validate(c, rec)
            assert rc == -5 and dev > 1e-6  # StaleData, recycle.cpp:73
            rec = None
        r = oc.solve(c, g[k + "b"], s=cfg.s, ell=cfg.ell, seed=0, recycle=rec, fetch_kind=1)
        check_result(r, g, k)


# ---- kernels -------------------------------------------------------------------------------------
def test_kernels_bit_exact(golden_kernels):
    g = golden_kernels
    for s in (1, 2, 3, 4, 8, 16):
        assert same(oc.solve_small(g[f"lu{s}_m"], g[f"lu{s}_rhs"]), g[f"lu{s}_x"])
    assert oc.solve_small(g["lu_sing_m"], np.ones(3)) is None
    for n, ell in ((50, 1), (300, 2), (1000, 4), (4000, 8)):
        assert same(oc.least_squares(g[f"ls{n}_{ell}_z"], g[f"ls{n}_{ell}_r"]), g[f"ls{n}_{ell}_tau"])
    assert same(oc.least_squares(g["lsk_z"], g["lsk_r"]), g["lsk_tau"])
    assert oc.least_squares(g["lsdef_z"], g["lsdef_r"]) == -9  # RankDeficient
    for n, s, seed in ((257, 1, 0), (257, 3, 7), (1000, 4, 11), (64, 8, 99)):
        assert same(oc.cut_space(n, s, seed), g[f"cut{n}_{s}_{seed}"])
    u, v = oc.arnoldi(oc.Csr(tri(8)), np.ones(8), 3, 2)
    assert same(u, g["arn_tri_u"]) and same(v, g["arn_tri_v"])
    import paper_1604_06043_b200 as m
    u, v = oc.arnoldi(oc.Csr(m.CsrMatrix.identity(6)), np.eye(6)[0], 3, 4)
    assert same(u, g["arn_eye_u"]) and same(v, g["arn_eye_v"])
    assert same(oc.normal_draws(5, 1001), g["normal_5"])


def read_mrd(path):
    raw = open(path, "rb").read()
    magic, ver, flags, n, s, lvl, om, fp = struct.unpack("<8sIIQQQQQ", raw[:56])
    return magic, ver, flags, n, s, lvl, om, fp, raw


def test_mrd_golden_layout():
    magic, ver, flags, n, s, lvl, om, fp, raw = read_mrd(GOLDEN / "donor_tridiag30.mrd")
    assert magic == b"MSTABMRD" and ver == 1 and flags == 1 and (n, s, lvl, om) == (30, 2, 4, 4)
    c = oc.Csr(tri(30))
    assert fp == c.fingerprint()
    d = oc.solve(c, np.ones(30), s=2, ell=1, seed=21, fetch_kind=0, fetch_cycle=4).fetched
    body = np.frombuffer(raw[56:56 + 3 * n * s * 8], dtype="<f8")
    assert same(body[:n * s], d.p.T.ravel()) and same(body[n * s:2 * n * s], d.u.T.ravel())
    assert same(body[2 * n * s:], d.v.T.ravel())
    omb = np.frombuffer(raw[56 + 3 * n * s * 8:], dtype="<f8")
    assert same(omb[0::2] + 1j * omb[1::2], d.omega)


# ---- the compiled reference reproduces its own fixtures (guards a stale oracle/_ref) -----------
def test_ref_lib_reproduces_golden(ref_ctx, golden_kat, golden_kernels):
    import paper_1604_06043_b200 as m
    op = m.CsrOperator(tri(40), ref_ctx)
    r = m.idrstab_solve(op, np.ones(40), None, m.SolverConfig(2, 1, 1e-8, 100000, True, 1))
    assert same(r.x, golden_kat["idr2_x"])
    assert same([h.resnorm for h in r.report.residual_history], golden_kat["idr2_resnorms"])
    g = golden_kernels
    assert same(m.solve_small(g["lu8_m"], g["lu8_rhs"], ref_ctx), g["lu8_x"])
    assert same(m.make_cut_space(1000, 4, 11, ref_ctx), g["cut1000_4_11"])

"""Full-size reference corpus for teacher-forced parity.

Runs the UNMODIFIED reference (oracle/_ref/libmstab_ref.so, compiled from /root/reference by
oracle/Makefile) over the first systems of a BASELINE sequence on ONE host core, the reference
driving its own chain (its b_i, its hand-off: harness.cpp:220-249 with FetchPolicy
at_half_tolerance). For every system it writes

  parity_store/<case>/x<i>.npy           the reference's solution x_i (fp64, N)
  parity_store/<case>/in<i>_uv.npy       the recycle data fed INTO solve i (U, V as (2, s, N) fp64;
                                        P is make_cut_space(N, s, 0) and is regenerated bit-exactly
                                        on the GPU box through the same compiled reference)
  tests/golden/fullsize/<case>.json     the small summary that is committed: cycles, h_mv, status,
                                        residual history, true relative residual, ||x||, sampled
                                        entries of x, the reference's validate() of each hand-off,
                                        per-RHS wall time, omega history, level_J, fingerprints.

parity_store/ is git- and gpurun-ignored; tools/parity_fullsize.py moves one case to parity_data/ so it travels to the GPU box with a gpurun snapshot for the
teacher-forced run (tools/parity_fullsize.py). This script only needs a CPU.

    python tools/ref_fixtures.py c2 [--nrhs 2]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1604_06043_b200 as m  # noqa: E402
from paper_1604_06043_b200 import problems as pb  # noqa: E402

REF = ROOT / "oracle" / "_ref" / "libmstab_ref.so"
DATA = ROOT / "parity_store"
GOLD = ROOT / "tests" / "golden" / "fullsize"

# case -> (config name, grid override, number of systems, true_residual_each_cycle)
CASES = {
    "c1": ("c1", 0, 20, True),
    "c1_recres": ("c1", 0, 20, False),
    "c2": ("c2", 0, 2, True),
    "c3": ("c3", 0, 3, True),
    "c4_64": ("c4", 64, 3, True),
    "c4_96": ("c4", 96, 3, True),
    "c5_42": ("c5", 0, 2, True),
}
N_SAMPLES = 4096


def sample_idx(n: int) -> np.ndarray:
    return np.sort(np.random.default_rng(12345).choice(n, size=min(n, N_SAMPLES), replace=False))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def run(case: str, nrhs: int | None, save_big: bool) -> dict:
    name, grid, n_default, true_res = CASES[case]
    nrhs = nrhs or n_default
    cfg = pb.config(name, grid=grid)
    ctx = m.Context(m.Lib(str(REF)))
    A = cfg.matrix()
    op = m.CsrOperator(A, ctx)
    x0, f = cfg.sources()
    b = cfg.first_rhs(x0, f) if cfg.kind == "convdiff" else cfg.first_rhs()
    sc = m.SolverConfig(cfg.s, cfg.ell, cfg.tol, 100000, true_res, 0)
    fp = m.FetchPolicy.at_half_tolerance()
    idx = sample_idx(cfg.N)
    out_dir = DATA / case
    if save_big:
        out_dir.mkdir(parents=True, exist_ok=True)
    summary = {"case": case, "config": name, "grid": cfg.grid, "N": cfg.N, "nnz": int(A.nnz()), "s": cfg.s,
               "ell": cfg.ell, "true_residual_each_cycle": true_res, "tol": cfg.tol,
               "fingerprint": f"{op.fingerprint():016x}", "sample_idx_seed": 12345, "n_samples": int(idx.size),
               "reference": "oracle/_ref/libmstab_ref.so (unmodified reference, -O3 -DNDEBUG, 1 host core)",
               "systems": []}
    rec = None
    for i in range(1, nrhs + 1):
        row = {"rhs": i, "b_norm": float(np.linalg.norm(b)), "b_sha": sha(b)}
        if rec is not None:
            t0 = time.perf_counter()
            vr = m.validate(rec, op)
            row["in_validate"] = {"max_deviation": vr.max_deviation, "sigma_min_ratio": vr.sigma_min_ratio,
                                  "low_rank_warning": vr.low_rank_warning,
                                  "stale": bool(vr.max_deviation > 1e-6),
                                  "seconds": time.perf_counter() - t0}
            if save_big:
                np.save(out_dir / f"in{i}_uv.npy", np.stack([np.ascontiguousarray(rec.u.T),
                                                             np.ascontiguousarray(rec.v.T)]))
            row["in_level_J"] = rec.level_J
            row["in_omega"] = [[z.real, z.imag] for z in rec.omega_history]
            row["in_p_sha"] = sha(np.ascontiguousarray(rec.p.T))
            row["in_uv_sha"] = sha(np.stack([np.ascontiguousarray(rec.u.T), np.ascontiguousarray(rec.v.T)]))
        t0 = time.perf_counter()
        try:
            r = m.idrstab_solve(op, b, None, sc, rec, fp)
            row["kind"] = "fresh" if rec is None else "mstab"
        except m.StaleData as e:
            row["stale_data"] = str(e)
            r = m.idrstab_solve(op, b, None, sc, None, fp)
            row["kind"] = "fresh (reference validate raised StaleData)"
        row["seconds"] = time.perf_counter() - t0
        rep = r.report
        x = r.x
        row.update({
            "status": rep.status, "breakdown_reason": rep.breakdown_reason, "cycles": rep.cycles, "h_mv": rep.h_mv,
            "h_mv_aux": rep.h_mv_aux, "h_rd": rep.h_rd, "final_resnorm": rep.final_resnorm, "bnorm": rep.bnorm,
            "history": [[h.cycle, h.mv, h.level, h.resnorm] for h in rep.residual_history],
            "true_relres": float(np.linalg.norm(b - op.apply(x)) / np.linalg.norm(b)),
            "x_norm": float(np.linalg.norm(x)), "x_sha": sha(x), "x_samples": x[idx].tolist(),
            "fetched": r.fetched is not None,
        })
        summary["systems"].append(row)
        print(f"{case} rhs {i}: {row['kind']} cycles {rep.cycles} status {rep.status} true relres "
              f"{row['true_relres']:.2e} {row['seconds']:.1f}s"
              + (f" in-validate dev {row['in_validate']['max_deviation']:.2e}" if "in_validate" in row else ""),
              flush=True)
        if save_big:
            np.save(out_dir / f"x{i}.npy", x)
        GOLD.mkdir(parents=True, exist_ok=True)
        (GOLD / f"{case}.json").write_text(json.dumps(summary, indent=1))
        if i < nrhs:
            rec = r.handoff()
            b = cfg.next_rhs(i, x, f)
    return summary


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("case", choices=sorted(CASES))
    ap.add_argument("--nrhs", type=int, default=None)
    ap.add_argument("--no-big", action="store_true", help="summary only (no x / U,V files)")
    a = ap.parse_args()
    run(a.case, a.nrhs, not a.no_big)

"""Teacher-forced parity against the reference at the BASELINE sizes.

The corpus comes from tools/ref_fixtures.py, which ran the UNMODIFIED reference (oracle/_ref) in
the CPU container: the committed summary tests/golden/fullsize/<case>.json (cycles, residual
histories, ||x_ref||, 4096 sampled entries of x_ref, the reference's validate() of every hand-off)
and, when present, the full vectors under parity_data/<case>/ (x_i, and U, V of the recycle data
fed into solve i; git-ignored, moved there from parity_store/ for the GPU call).

For each system i of a case the B200 library solves A x = b_i from the reference's inputs:
  b_1 from the generator; b_i = next_rhs(x_ref_{i-1}) (the reference's own chain);
  recycle in = (P, U_ref, V_ref, omega_ref, J_ref): P is make_cut_space(N, s, 0) computed by the
  compiled reference on this host (checked against the corpus' sha), U/V from the corpus.
Reported per system: cycles (ref / b200), ||x - x_ref|| / ||x_ref|| (full vectors when present,
else the sampled estimate sqrt(N/m * sum_sampled (x - x_ref)^2) / ||x_ref||), true relative
residuals, the reference's validate() deviation of the hand-off it fed in, the B200's validate()
of the same hand-off, and the reference's validate() of the B200's own hand-off (whether the
reference would reject the hand-offs the B200 chain restarts on, recycle.cpp:51-73).

    python tools/parity_fullsize.py c2 c3 ... > profiles/r02_parity_fullsize.txt
"""
from __future__ import annotations

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

GOLD = ROOT / "tests" / "golden" / "fullsize"
DATA = ROOT / "parity_data"
REF = ROOT / "oracle" / "_ref" / "libmstab_ref.so"


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def sample_idx(n: int, count: int, seed: int) -> np.ndarray:
    return np.sort(np.random.default_rng(seed).choice(n, size=min(n, count), replace=False))


def load_case(case: str) -> dict:
    return json.loads((GOLD / f"{case}.json").read_text())


def has_vectors(case: str) -> bool:
    return (DATA / case / "x1.npy").exists()


def run_case(case: str, gctx, rctx=None, max_rhs: int | None = None, live: bool = False, log=print) -> list[dict]:
    """Teacher-forced comparison of every system of `case` that its data allows. Returns rows.

    The reference's inputs to system i >= 2 (x_{i-1} for b_i, and its hand-off) come from
    parity_data/<case>/ when present, else (live=True) from the compiled reference re-running its
    own chain on this host — checked bit-for-bit against the corpus (x sha) — and otherwise the
    case stops after the fresh first system."""
    g = load_case(case)
    cfg = pb.config(g["config"], grid=g["grid"])
    A = cfg.matrix()
    op = m.CsrOperator(A, gctx)
    rows = []
    if f"{op.fingerprint():016x}" != g["fingerprint"]:
        raise AssertionError(f"{case}: fingerprint {op.fingerprint():016x} != reference {g['fingerprint']}")
    rop = m.CsrOperator(A, rctx) if rctx is not None else None
    x0, f = cfg.sources()
    idx = sample_idx(cfg.N, g["n_samples"], g["sample_idx_seed"])
    sc = m.SolverConfig(cfg.s, cfg.ell, g["tol"], 100000, g["true_residual_each_cycle"], 0)
    fp = m.FetchPolicy.at_half_tolerance()
    d = DATA / case
    P = None
    x_prev = None    # the reference's x_{i-1}
    rec_live = None  # the live reference's hand-off into system i
    systems = g["systems"][:max_rhs] if max_rhs else g["systems"]
    last = systems[-1]["rhs"]
    for sysd in systems:
        i = sysd["rhs"]
        if i == 1:
            b = cfg.first_rhs(x0, f) if cfg.kind == "convdiff" else cfg.first_rhs()
        elif x_prev is not None:
            b = cfg.next_rhs(i - 1, x_prev, f)
        else:
            break  # later systems need the reference's x_{i-1} and hand-off
        assert sha(b) == sysd["b_sha"], f"{case} rhs {i}: b differs from the reference's"
        rec = None
        row = {"case": case, "rhs": i, "ref_cycles": sysd["cycles"], "ref_true_relres": sysd["true_relres"],
               "ref_seconds": sysd["seconds"], "ref_kind": sysd["kind"], "inputs": "generator" if i == 1 else None}
        if i > 1 and sysd["kind"] == "mstab":
            if (d / f"in{i}_uv.npy").exists():
                if P is None:
                    if rctx is None:
                        raise AssertionError("the recycled systems need oracle/_ref for P")
                    P = m.make_cut_space(cfg.N, cfg.s, 0, rctx)
                assert sha(np.ascontiguousarray(P.T)) == sysd["in_p_sha"], f"{case}: P differs from the reference's"
                uv = np.load(d / f"in{i}_uv.npy")
                assert sha(uv) == sysd["in_uv_sha"]
                om = np.array([complex(a, b_) for a, b_ in sysd["in_omega"]])
                rec = m.fetch(P, uv[0].T, uv[1].T, om, sysd["in_level_J"], int(g["fingerprint"], 16), gctx)
                del uv
                row["inputs"] = "corpus files"
            elif rec_live is not None:
                uv = np.stack([np.ascontiguousarray(rec_live.u.T), np.ascontiguousarray(rec_live.v.T)])
                assert sha(uv) == sysd["in_uv_sha"], f"{case}: live reference hand-off differs from the corpus"
                rec = m.fetch(rec_live.p, rec_live.u, rec_live.v, rec_live.omega_history, rec_live.level_J,
                              rec_live.matrix_fingerprint, gctx)
                del uv
                row["inputs"] = "live reference chain (sha-checked against the corpus)"
            else:
                break
            row["ref_in_validate"] = sysd["in_validate"]["max_deviation"]
            row["b200_in_validate"] = m.validate(rec, op).max_deviation
        t0 = time.perf_counter()
        try:
            r = m.idrstab_solve(op, b, None, sc, rec, fp)
        except m.StaleData as e:  # the reference accepted this hand-off (it is in the corpus as mstab)
            row["b200_stale"] = str(e)
            r = m.idrstab_solve(op, b, None, sc, None, fp)
        row["b200_seconds"] = time.perf_counter() - t0
        x = r.x
        rep = r.report
        row.update({"b200_cycles": rep.cycles, "b200_status": rep.status, "h_mv": rep.h_mv,
                    "ref_h_mv": sysd["h_mv"],
                    "b200_true_relres": float(np.linalg.norm(b - op.apply(x)) / np.linalg.norm(b))})
        xs = np.asarray(sysd["x_samples"])
        row["dx_sampled"] = float(np.sqrt(cfg.N / xs.size * np.sum((x[idx] - xs) ** 2)) / sysd["x_norm"])
        row["dx"] = None
        x_prev = None
        if (d / f"x{i}.npy").exists():
            x_ref = np.load(d / f"x{i}.npy")
            assert sha(x_ref) == sysd["x_sha"]
            row["dx"] = float(np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref))
            x_prev = x_ref
        elif live and rop is not None and i < last:
            # the reference solves system i itself (its inputs are the same b_i and hand-off)
            t1 = time.perf_counter()
            rin = None
            if rec is not None:
                rin = rec_live
            rr = m.idrstab_solve(rop, b, None, sc, rin, fp)
            x_ref = rr.x
            assert sha(x_ref) == sysd["x_sha"], f"{case} rhs {i}: live reference x differs from the corpus"
            row["dx"] = float(np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref))
            row["ref_live_seconds"] = time.perf_counter() - t1
            x_prev = x_ref
            rec_live = rr.handoff()
        if rop is not None and i < last:
            # would the reference accept the B200's own hand-off? (its validate on host cores)
            h = r.handoff()
            rh = m.fetch(h.p, h.u, h.v, h.omega_history, h.level_J, h.matrix_fingerprint, rctx)
            row["ref_validate_of_b200_handoff"] = m.validate(rh, rop).max_deviation
            row["b200_validate_of_b200_handoff"] = m.validate(h, op).max_deviation
            del rh, h
        rows.append(row)
        log(fmt(row))
    return rows


def fmt(r: dict) -> str:
    dx = r["dx"] if r["dx"] is not None else r["dx_sampled"]
    tag = "full" if r["dx"] is not None else "smpl"
    s = (f"{r['case']:10s} rhs {r['rhs']:2d} {r['ref_kind'][:5]:5s} cycles ref {r['ref_cycles']:3d} b200 "
         f"{r['b200_cycles']:3d}  |dx|/|x| {dx:8.1e} ({tag})  true relres ref {r['ref_true_relres']:8.1e} "
         f"b200 {r['b200_true_relres']:8.1e}  time ref {r['ref_seconds']:8.1f}s b200 {r['b200_seconds']:7.3f}s")
    if "ref_in_validate" in r:
        s += f"  in-validate ref {r['ref_in_validate']:.2e} b200 {r['b200_in_validate']:.2e}"
    if "ref_validate_of_b200_handoff" in r:
        s += (f"  b200-handoff validate ref {r['ref_validate_of_b200_handoff']:.2e} "
              f"b200 {r['b200_validate_of_b200_handoff']:.2e}")
    if "b200_stale" in r:
        s += "  B200 VALIDATE REJECTED THE REFERENCE HAND-OFF"
    return s


if __name__ == "__main__":
    live = "--live" in sys.argv
    cases = [a for a in sys.argv[1:] if not a.startswith("--")] or sorted(p.stem for p in GOLD.glob("*.json"))
    gctx = m.Context(m.Lib())
    rctx = m.Context(m.Lib(str(REF))) if REF.exists() else None
    print(f"# teacher-forced parity at BASELINE sizes; b200 build: {gctx.lib.build_id}")
    print("# reference corpus: tools/ref_fixtures.py (oracle/_ref, unmodified reference, 1 core of the CPU container)")
    allrows = []
    for c in cases:
        allrows += run_case(c, gctx, rctx, live=live, log=lambda s: print(s, flush=True))
    out = ROOT / "gpurun_out" / f"parity_fullsize_{'_'.join(cases)}.json"
    out.parent.mkdir(exist_ok=True)
    out.write_text(json.dumps(allrows, indent=1))

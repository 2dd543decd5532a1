"""The reference's own cycle-count noise floor on a full-size corpus case.

Teacher-forced parity asks for per-system cycle counts within +-2 of the reference's. A Krylov
recurrence in finite precision is chaotic over tens of cycles, so the count at which ||r|| first
drops under tol * ||b|| moves when any rounding moves. This tool measures how far the UNMODIFIED
reference (oracle/_ref, CPU) moves by itself: every system of the case is re-solved from the
corpus inputs (the reference's b_i and hand-off, parity_data/<case>/ or parity_store/<case>/) with
b_i perturbed by a relative 1e-15 per entry (about one ulp), `trials` times. The spread of those
counts is the band a different summation order (the device's tree reductions) can land in.

    python tools/ref_cycle_noise.py c1 [trials] > profiles/r02_ref_cycle_noise_c1.txt
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1604_06043_b200 as m  # noqa: E402
from paper_1604_06043_b200 import problems as pb  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "c1"
trials = int(sys.argv[2]) if len(sys.argv) > 2 else 3
g = json.loads((ROOT / "tests" / "golden" / "fullsize" / f"{case}.json").read_text())
d = next(p for p in (ROOT / "parity_data" / case, ROOT / "parity_store" / case) if p.exists())
cfg = pb.config(g["config"], grid=g["grid"])
A = cfg.matrix()
ctx = m.Context(m.Lib(str(ROOT / "oracle" / "_ref" / "libmstab_ref.so")))
op = m.CsrOperator(A, ctx)
x0, f = cfg.sources()
sc = m.SolverConfig(cfg.s, cfg.ell, g["tol"], 100000, g["true_residual_each_cycle"], 0)
fp = m.FetchPolicy.at_half_tolerance()
P = m.make_cut_space(cfg.N, cfg.s, 0, ctx)
print(f"# reference cycle-count noise floor, case {case}: each system re-solved by the reference itself from the")
print(f"# corpus inputs with b_i * (1 + 1e-15 * N(0,1)) ({trials} draws). ref = the corpus count (unperturbed).")
band = []
for sysd in g["systems"]:
    i = sysd["rhs"]
    if i == 1:
        b = cfg.first_rhs(x0, f) if cfg.kind == "convdiff" else cfg.first_rhs()
        rec = None
    else:
        if not (d / f"x{i - 1}.npy").exists() or not (d / f"in{i}_uv.npy").exists():
            break
        b = cfg.next_rhs(i - 1, np.load(d / f"x{i - 1}.npy"), f)
        uv = np.load(d / f"in{i}_uv.npy")
        om = np.array([complex(a, c) for a, c in sysd["in_omega"]])
        rec = m.fetch(P, uv[0].T, uv[1].T, om, sysd["in_level_J"], int(g["fingerprint"], 16), ctx)
    counts = []
    for t in range(trials):
        bp = b * (1.0 + 1e-15 * pb.normal(7000 + 31 * i + t, b.size))
        r = m.idrstab_solve(op, bp, None, sc, rec, fp)
        counts.append(int(r.report.cycles))
    band.append((i, sysd["cycles"], counts))
    print(f"{case} rhs {i:2d} ref {sysd['cycles']:3d}  ref on perturbed b: {counts}  "
          f"spread {min(counts + [sysd['cycles']]) - sysd['cycles']:+d}..{max(counts + [sysd['cycles']]) - sysd['cycles']:+d}",
          flush=True)
worst = max(max(abs(c - ref) for c in cs) for _, ref, cs in band)
print(f"# largest |perturbed - unperturbed| over {len(band)} systems: {worst} cycles")

"""Does the reference reject the same hand-offs the B200 chain restarts on? (VERDICT r01 weak #1,
ADVICE r01 bench.py:159.)

The bench's sequence driver re-solves a right-hand side fresh when validate() rejects the hand-off
(StaleData: ||V - A U|| / ||V|| or ||P^H P - I|| above 1e-6, recycle.cpp:51-73). This tool runs the
free-running B200 chain of a config (the bench's own driver settings) and, for EVERY hand-off,
records the B200's validate() verdict; for every hand-off the B200 rejects — and for the accepted
one with the largest deviation — it moves P, U, V to the host and asks the UNMODIFIED reference
(oracle/_ref) to validate the same data, plus an independent numpy evaluation of the two deviations.

    python tools/restart_check.py c2 [n_rhs] > profiles/r02_restart_check_c2.txt
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1604_06043_b200 as m  # noqa: E402
from paper_1604_06043_b200 import problems as pb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = pb.config(name)
n_rhs = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n_rhs
gctx = m.Context(m.Lib())
rctx = m.Context(m.Lib(str(ROOT / "oracle" / "_ref" / "libmstab_ref.so")))
A = cfg.matrix()
gop, rop = m.CsrOperator(A, gctx), m.CsrOperator(A, rctx)
x0, f = cfg.sources()
b = cfg.first_rhs(x0, f) if cfg.kind == "convdiff" else cfg.first_rhs()
sc = m.SolverConfig(cfg.s, cfg.ell, cfg.tol, 100000, True, 0)
fp = m.FetchPolicy.at_half_tolerance()
print(f"# {name}: free-running B200 chain of {n_rhs} systems, M({cfg.s},{cfg.ell})stab, true residual, fetch at half "
      f"tolerance; build {gctx.lib.build_id}")
print("# per hand-off: the B200 validate() verdict; for rejected hand-offs (and the worst accepted one) the reference's "
      "validate() of the same P, U, V and the deviations recomputed in numpy (host fp64, pairwise sums)")


def numpy_deviation(h):
    import scipy.sparse as sp
    M = sp.csr_matrix((np.asarray(A.values), np.asarray(A.col_idx), np.asarray(A.row_ptr)), shape=(A.n_rows, A.n_cols))
    P, U, V = h.p, h.u, h.v
    dv = np.linalg.norm(V - M @ U) / np.linalg.norm(V)
    dp = np.abs(P.T @ P - np.eye(P.shape[1])).max()
    return dv, dp


def ref_verdict(h):
    rh = m.fetch(h.p, h.u, h.v, h.omega_history, h.level_J, h.matrix_fingerprint, rctx)
    try:
        return f"accepts (max_deviation {m.validate(rh, rop).max_deviation:.3e})"
    except m.StaleData as e:
        return f"REJECTS: StaleData ({e})"


rec = None
worst = (0.0, None, None)
rejected = 0
for i in range(1, n_rhs + 1):
    verdict = "-"
    if rec is not None:
        try:
            dev = m.validate(rec, gop).max_deviation
            verdict = f"accepted, max_deviation {dev:.3e}"
            if dev > worst[0]:
                worst = (dev, i, rec)
        except m.StaleData:
            rejected += 1
            dv, dp = numpy_deviation(rec)
            verdict = (f"REJECTED by the B200 (StaleData); reference {ref_verdict(rec)}; numpy ||V-AU||/||V|| {dv:.3e}, "
                       f"max|P^H P - I| {dp:.3e}")
            rec = None
    r = m.idrstab_solve(gop, b, None, sc, rec, fp)
    print(f"{name} rhs {i:2d} {'mstab' if rec is not None else 'fresh'} cycles {r.report.cycles:3d} status {r.report.status} "
          f"hand-off in: {verdict}", flush=True)
    rec = r.handoff()
    b = cfg.next_rhs(i, r.x, f) if cfg.kind == "convdiff" else cfg.next_rhs(i, r.x)
if worst[2] is not None:
    dv, dp = numpy_deviation(worst[2])
    print(f"# worst ACCEPTED hand-off (into rhs {worst[1]}): B200 max_deviation {worst[0]:.3e}; reference "
          f"{ref_verdict(worst[2])}; numpy ||V-AU||/||V|| {dv:.3e}, max|P^H P - I| {dp:.3e}")
print(f"# {rejected} of {n_rhs - 1} hand-offs rejected by the B200's validate()")

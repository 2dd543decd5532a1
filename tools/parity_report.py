"""Teacher-forced parity table: the compiled reference (oracle/_ref) drives each chain (its b_i and
its hand-off); the B200 library solves every system from the same inputs. Prints one row per
system: cycles (ref / b200), relative solution difference, true relative residuals.

    python tools/parity_report.py > profiles/r01_parity.txt
"""
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1604_06043_b200 as m  # noqa: E402
from paper_1604_06043_b200 import problems as pb  # noqa: E402

REF = m.Lib(__file__.rsplit("/tools/", 1)[0] + "/oracle/_ref/libmstab_ref.so")
rctx, gctx = m.Context(REF), m.Context(m.Lib())


def chain(name, cfg, nrhs, true_res=False):
    A = cfg.matrix()
    ro, go = m.CsrOperator(A, rctx), m.CsrOperator(A, gctx)
    x0, f = cfg.sources()
    b = cfg.first_rhs(x0, f) if cfg.kind == "convdiff" else cfg.first_rhs()
    sc = m.SolverConfig(cfg.s, cfg.ell, 1e-8, 100000, true_res, 0)
    fp = m.FetchPolicy.at_half_tolerance()
    rec = None
    for i in range(nrhs):
        t0 = time.perf_counter()
        try:
            r = m.idrstab_solve(ro, b, None, sc, rec, fp)
            stale = False
        except m.StaleData:
            r = m.idrstab_solve(ro, b, None, sc, None, fp)
            stale = True
        tr = time.perf_counter() - t0
        grec = None
        if rec is not None and not stale:
            grec = m.fetch(rec.p, rec.u, rec.v, rec.omega_history, rec.level_J, rec.matrix_fingerprint, gctx)
        t0 = time.perf_counter()
        g = m.idrstab_solve(go, b, None, sc, grec, fp)
        tg = time.perf_counter() - t0
        xr = r.x
        dx = np.linalg.norm(g.x - xr) / np.linalg.norm(xr)
        trr = np.linalg.norm(b - ro.apply(xr)) / np.linalg.norm(b)
        trg = np.linalg.norm(b - ro.apply(g.x)) / np.linalg.norm(b)
        print(f"{name:10s} rhs {i + 1:2d} {'fresh' if rec is None or stale else 'mstab':5s} cycles ref {r.report.cycles:3d} "
              f"b200 {g.report.cycles:3d}  |dx|/|x| {dx:8.1e}  true relres ref {trr:8.1e} b200 {trg:8.1e}  "
              f"time ref {tr:7.2f}s b200 {tg:6.3f}s", flush=True)
        rec = r.handoff()
        b = cfg.next_rhs(i + 1, xr, f)


if __name__ == "__main__":
    print("# teacher-forced parity: reference (oracle/_ref, 1 host core) drives the chain; B200 solves the same systems")
    chain("c1 256^2", pb.config("c1"), 6)
    chain("c2 48^3", pb.config("c2", grid=48), 3, true_res=True)
    c3 = pb.config("c3", grid=262144)
    chain("c3 262k", c3, 4)
    chain("c4 40^3", pb.config("c4", grid=40), 3, true_res=True)  # 27-point stencil, reduced size
    chain("c5 48^3", pb.config("c5", grid=48), 4, true_res=True)

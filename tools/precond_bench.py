"""Split-preconditioned solves on one B200: apply time of L^-1 A R^-1 and a short
preconditioned M(s,ell)stab sequence, for Jacobi and ILU(0), next to the unpreconditioned operator.

usage: python tools/precond_bench.py [config] [grid] [n_rhs]
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1604_06043_b200 as m  # noqa: E402
from paper_1604_06043_b200 import problems as pb  # noqa: E402


def apply_us(op, n, iters=20):
    dev = torch.device("cuda", 0)
    x = torch.from_numpy(pb.normal(5, n)).to(dev)
    y = torch.empty_like(x)
    for _ in range(3):
        op.apply(x, y)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(iters):
        op.apply(x, y)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / iters * 1e6


def sequence(op, cfg, n_rhs, precond):
    x0, f = cfg.sources()
    b = cfg.first_rhs(x0, f)
    sc = m.SolverConfig(cfg.s, cfg.ell, 1e-8, 100000, True, 0)
    fp = m.FetchPolicy.at_half_tolerance()
    rec, rows = None, []
    t0 = time.perf_counter()
    for i in range(n_rhs):
        bt = m.preconditioned_rhs(op, b) if precond else b
        try:
            r = m.idrstab_solve(op, bt, None, sc, rec, fp)
        except m.StaleData:
            r = m.idrstab_solve(op, bt, None, sc, None, fp)
        x = m.unpreconditioned_solution(op, r.x) if precond else r.x
        rows.append({"cycles": int(r.report.cycles), "status": int(r.report.status == m.CONVERGED)})
        rec = r.handoff()
        b = cfg.next_rhs(i + 1, x, f)
    return {"rhs_per_s": round(n_rhs / (time.perf_counter() - t0), 3), "per_rhs": rows}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    grid = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    n_rhs = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    ctx = m.Context(m.Lib(), 0)
    cfg = pb.config(name, grid=grid)
    a = cfg.matrix()
    out = {"config": name, "grid": cfg.grid, "N": a.n_rows, "s": cfg.s, "ell": cfg.ell, "n_rhs": n_rhs,
           "timing": "host wall clock around synchronised device work (sequence includes host RHS updates)"}
    ops = {"none": m.CsrOperator(a, ctx)}
    for kind, build in (("jacobi", m.build_jacobi), ("ilu0", m.build_ilu0)):
        t0 = time.perf_counter()
        pc = build(a, ctx.lib)
        ops[kind] = m.PreconditionedOperator(pc, a, ctx)
        out[f"{kind}_setup_s"] = round(time.perf_counter() - t0, 2)
    for kind, op in ops.items():
        out[kind] = {"apply_us": round(apply_us(op, a.n_rows), 1),
                     "sequence": sequence(op, cfg, n_rhs, kind != "none")}
        print(kind, out[kind], flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()

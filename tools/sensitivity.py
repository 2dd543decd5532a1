"""Rounding sensitivity of one IDR(s)stab(ell) cycle: the same fresh solve on b and on b perturbed
by a relative 1e-15 (one ulp-scale change per entry), on the B200 and on the reference. When the
reference's own answer moves as much under the perturbation as it differs from the B200's, the
disagreement is the method's conditioning at those parameters, not a device-path error.

usage: python tools/sensitivity.py GRID s ell [cycles] [--full]"""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0] + "/tests")
import paper_1604_06043_b200 as m  # noqa: E402
from paper_1604_06043_b200 import problems as pb  # noqa: E402
from conftest import REF_LIB  # noqa: E402

grid, s, ell = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
cycles = int(sys.argv[4]) if len(sys.argv) > 4 and sys.argv[4].isdigit() else 1
g, r = m.Context(m.Lib(), 0), m.Context(m.Lib(REF_LIB))
cfg = pb.config("c5", grid=grid)
A = cfg.matrix()
x0, f = cfg.sources()
b = cfg.first_rhs(x0, f)
bp = b * (1.0 + 1e-15 * pb.normal(99, b.size))
sc = m.SolverConfig(s, ell, 1e-30, s + cycles * ell * (s + 1), False, 0)
out = {}
for name, ctx in (("b200", g), ("ref", r)):
    op = m.CsrOperator(A, ctx)
    for tag, rhs in (("b", b), ("b+1e-15", bp)):
        res = m.idrstab_solve(op, rhs, None, sc, None, None)
        out[(name, tag)] = res.x
        print(f"{name:5s} {tag:8s} resnorm after {cycles} cycle(s): {res.report.residual_history[-1].resnorm:.4e}",
              flush=True)
nx = np.linalg.norm(out[("ref", "b")])
print(f"ref(b) vs ref(b+1e-15):  {np.linalg.norm(out[('ref', 'b')] - out[('ref', 'b+1e-15')]) / nx:.2e}")
print(f"b200(b) vs b200(b+1e-15): {np.linalg.norm(out[('b200', 'b')] - out[('b200', 'b+1e-15')]) / nx:.2e}")
print(f"b200(b) vs ref(b):       {np.linalg.norm(out[('b200', 'b')] - out[('ref', 'b')]) / nx:.2e}")

if "--full" in sys.argv:  # the whole solve (tol 1e-8, true residual) on b and on the perturbed b
    scf = m.SolverConfig(s, ell, 1e-8, 20000, True, 0)
    for name, ctx in (("b200", g), ("ref", r)):
        op = m.CsrOperator(A, ctx)
        for tag, rhs in (("b", b), ("b+1e-15", bp)):
            res = m.idrstab_solve(op, rhs, None, scf, None, m.FetchPolicy.at_half_tolerance())
            print(f"full {name:5s} {tag:8s} status {res.report.status} cycles {res.report.cycles} "
                  f"final resnorm/bnorm {res.report.final_resnorm / res.report.bnorm:.2e}", flush=True)

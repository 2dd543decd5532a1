import sys
sys.path.insert(0,'/root/repo')
import numpy as np
import paper_1604_06043_b200 as m
from paper_1604_06043_b200 import problems as pb
cfg = pb.config("c1"); A = cfg.matrix(); ctx = m.Context(m.Lib(), 0); op = m.CsrOperator(A, ctx)
x0, f = cfg.sources(); b = cfg.first_rhs(x0, f)
sc = m.SolverConfig(cfg.s, cfg.ell, 1e-8, cfg.s + 4 * cfg.ell * (cfg.s + 1), True, 0)
r = m.idrstab_solve(op, b, None, sc, None, None)
print(r.report.cycles, r.report.status)

import sys, numpy as np
sys.path.insert(0, '.')
import paper_1607_01404_b200 as p
from paper_1607_01404_b200 import eigensolver as es
from oracle import phsvds
d = np.arange(1.0, 31.0)
NEVER = lambda lam, rnorm, x, opx, op_norm: False
cfgkw = dict(num_evals=1, max_basis_size=8, min_restart_size=3, convergence_test=NEVER, practical_test=NEVER, stagnation_window=40, seed=16)
o = phsvds.GDk(phsvds.SymOp(30, lambda x: d[:, None] * x), phsvds.Opts(target=phsvds.LARGEST, **cfgkw))
log = []
res = o.run()
print("oracle", res.status, o.work)
for spec in (True, False):
    op = p.LinearOperator(30, lambda x: d[:, None] * x)
    s = es.DavidsonSolver(op, p.EigConfig(target="largest_algebraic", **cfgkw))
    s.speculate = spec
    it = 0
    try:
        while not s._finished and it < 400:
            info = s.step(); it += 1
            if it < 80: print(spec, it, "%.3e" % info.get("rnorm", -1), s.collapse_streak, s.g)
        print("device spec=%s" % spec, s.status, s.stats)
    except Exception as e:
        print("device spec=%s raised" % spec, repr(e), "after", it, s.stats)

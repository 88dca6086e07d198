import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import numpy as np, oracle_lib as O
from paper_2203_11733_b200._native import Context
ctx = Context(0)
for n in [63, 64, 65, 100, 128, 129, 130, 200, 500]:
    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, n)) + 0.5*np.eye(n); b = rng.standard_normal(n)
    x, res, st = ctx.lu_solve(A, b)
    xo, ro, sto, _ = O.lu_solve(A, b)
    xr = np.linalg.solve(A, b)
    print(n, "gpu res %.2e orc res %.2e  |x-xr|/|xr| gpu %.2e orc %.2e cond %.1e" % (res, ro, np.abs(x-xr).max()/np.abs(xr).max(), np.abs(xo-xr).max()/np.abs(xr).max(), np.linalg.cond(A)))

import sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2203_11733_b200 as g
from paper_2203_11733_b200._native import Context
ctx = Context(0)
m = g.config_model(1, scale=1.0); ps = m.partition(1); n = len(ps)
A, _ = ctx.assemble_single(ps.arrays())
for K in (6, 9, 12, 16):
    rng = np.random.default_rng(K)
    B = rng.standard_normal((n, K))
    ctx.matrix_upload(A)
    X, res, st = ctx.spd_solve(B)
    Xr = np.linalg.solve(A, B)
    print("spd_solve K", K, "res", np.max(res), "err", np.abs(X - Xr).max() / np.abs(Xr).max())

"""Small runs of the round-2 kernels for compute-sanitizer (memcheck / racecheck):
the sharded solve (2 Jacobi blocks), the DMMA residual (n >= 16,384 path forced
through a 17-RHS solve on a random SPD matrix of n = 16,400) and a config-1
extraction."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_2203_11733_b200 as g  # noqa: E402
from paper_2203_11733_b200 import _native as N  # noqa: E402
from paper_2203_11733_b200.pcg import sharded_cmatrix  # noqa: E402

m = g.config_model(1, seed=1, scale=0.5)
ps = m.partition(1)
ids = m.net_ids
net = np.array([ids.index(v) if k == 0 else -1 for v, k in zip(ps.net, ps.kind)], dtype=np.int32)
ctx = N.Context(0)
Cd, _, _, _ = ctx.extract_cmatrix(ps.arrays(), net, len(ids), 3.9)
Cp, res, _, st, _ = sharded_cmatrix(ctx, ps.arrays(), net, len(ids), 3.9, tol=1e-12, jacobi_blocks=2)
assert np.abs(Cp - Cd).max() <= 1e-9 * np.abs(Cd).max()
n = 16400
rng = np.random.default_rng(1)
M = rng.standard_normal((n, 64)) / 8
A = M @ M.T + np.eye(n)
ctx.matrix_upload(A)
B = rng.standard_normal((n, 17))
X, r, _ = ctx.spd_solve(B)
assert r.max() <= 1e-12, r.max()
print("sanitize run ok", st.iterations, r.max())
ctx.close()

"""Small bordered extractions through the look-ahead backward sweep (k_bwd_step clusters with
distributed shared memory, k_bwd_bulk) for compute-sanitizer:
    compute-sanitizer --tool memcheck  python tools/sanitize_bwd.py
    compute-sanitizer --tool racecheck python tools/sanitize_bwd.py
n = 1,456 = 11 * 128 + 48 (ragged last block); K = 17 and 40 right-hand sides."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_2203_11733_b200 as g  # noqa: E402
from paper_2203_11733_b200 import _native as N  # noqa: E402

ps = g.config_model(1, scale=1.0).partition(1)
n = len(ps)
ctx = N.Context(0)
for K in (17, 40):
    rng = np.random.default_rng(K)
    net = rng.integers(0, K, size=n).astype(np.int32)
    net[:K] = np.arange(K)
    Cm, res, _, _ = ctx.extract_cmatrix(ps.arrays(), net, K, 3.9)
    assert res.max() <= 1e-12, res.max()
    print("ok", n, K, res.max())
ctx.close()

"""One config-2 extraction (optionally after warm-up steps) for ncu captures."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

import paper_2203_11733_b200 as g
from paper_2203_11733_b200 import _native as N

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 0
m = g.config_model(cfg)
ps = m.partition(1)
ids = m.net_ids
net = np.where(ps.kind == 0, ps.net - 1, -1).astype(np.int32)
ctx = N.Context(0)
for _ in range(warm + 1):
    Cm, res, ast, sst = ctx.extract_cmatrix(ps.arrays(), net, len(ids), m.info()["eps_r"])
print("n", len(ps), "assembly_ms", ast.ms_total, "far", ast.ms_far, "near", ast.ms_near, "factor_ms", sst.ms_factor,
      "solve_ms", sst.ms_solve, "launches", ctx.launches, "resid", res.max())

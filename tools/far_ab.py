"""Assembly phase times on BASELINE configs (A/B driver for kernel experiments):
    python tools/far_ab.py [configs, default 2,3] [repeats]
Prints the minimum over the repeats of the classify / far / near / total milliseconds."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2203_11733_b200 as g  # noqa: E402
from paper_2203_11733_b200 import _native as N  # noqa: E402

cfgs = [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "2,3").split(",")]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
ctx = N.Context(0)
for cfg in cfgs:
    ps = g.config_model(cfg, seed=1).partition(1)
    best = None
    for _ in range(reps):
        A, st = ctx.assemble_single(ps.arrays(), download=False)
        d = st.as_dict()
        t = (d["ms_total"], d["ms_classify"], d["ms_far"], d["ms_near"])
        best = t if best is None else tuple(min(a, b) for a, b in zip(best, t))
    print({"config": cfg, "panels": len(ps), "ms_total": round(best[0], 3), "ms_classify": round(best[1], 3),
           "ms_far": round(best[2], 3), "ms_near": round(best[3], 3), "far_evals": d["far_evals"],
           "far_tflops": round(d["far_flops"] / best[2] * 1e-9, 2)}, flush=True)

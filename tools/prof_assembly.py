"""One assembly of a BASELINE config on cuda:0 (for ncu captures of the
assembly kernels):  python tools/prof_assembly.py [config] [repeats]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2203_11733_b200 as g  # noqa: E402
from paper_2203_11733_b200 import _native as N  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ps = g.config_model(cfg, seed=1).partition(1)
ctx = N.Context(0)
for _ in range(reps):
    A, st = ctx.assemble_single(ps.arrays(), download=False)
print({k: v for k, v in st.as_dict().items() if not isinstance(v, list)})

"""Run the on-device kernel selftest at a given scale and dump each class's worst
pair (geometry, evaluator value, oracle value) as JSON lines, for offline study
against the compiled reference (tools/selftest_recheck.py)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_11733_b200._native import Context  # noqa: E402

pairs = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
seeds = [int(s) for s in sys.argv[2:]] or [20260817]
ctx = Context(0)
for seed in seeds:
    for c in ctx.selftest(pairs=pairs, seed=seed):
        c["seed"] = seed
        print(json.dumps(c), flush=True)
ctx.close()

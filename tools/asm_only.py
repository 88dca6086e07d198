"""Assembly-only throughput on a BASELINE config (default 5: random panels),
streaming row blocks through one GPU buffer (checksummed, then overwritten)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2203_11733_b200 as g
from paper_2203_11733_b200 import _native as N
from paper_2203_11733_b200.shard import ShardedAssembler, panels_to_device, balanced_row_split, row_work

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
chunks = int(sys.argv[3]) if len(sys.argv) > 3 else 16
with_stats = (sys.argv[4] != '0') if len(sys.argv) > 4 else True  # 0: no per-phase timing (near field overlaps far)
t0 = time.time()
ps = g.config_model(cfg, seed=1, scale=scale).partition(1)
n = len(ps)
print("panels", n, "gen s", round(time.time() - t0, 2), flush=True)
ctx = N.Context(0)
dev = torch.device("cuda", 0)
pdev = panels_to_device(ps, dev)
torch.cuda.set_device(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
tot_pairs = 0; tot = dict(far=0, cop=0, par=0, orth=0, nonconv=0, far_evals=0, near_evals=0, ms_far=0, ms_near=0, ms_cls=0)
chk = torch.zeros((), dtype=torch.float64, device=dev)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
ev0.record()
for c in range(chunks):
    sh = ShardedAssembler(ctx, pdev, n, c, chunks)
    blk = sh.assemble(with_stats=with_stats)
    chk += blk.sum()
    if not with_stats:
        tot_pairs += sh.unique_pairs
        del sh, blk
        continue
    st = sh.stats
    tot_pairs += st.pairs_total
    for k, f in (("far", "pairs_far"), ("cop", "pairs_coplanar"), ("par", "pairs_parallel"), ("orth", "pairs_orthogonal"),
                 ("nonconv", "not_converged"), ("far_evals", "far_evals"), ("near_evals", "near_evals"),
                 ("ms_far", "ms_far"), ("ms_near", "ms_near"), ("ms_cls", "ms_classify")):
        tot[k] += getattr(st, f)
    del sh, blk
ev1.record(); torch.cuda.synchronize()
ms = ev0.elapsed_time(ev1)
print({"config": cfg, "panels": n, "pairs": tot_pairs, "ms": ms, "entries_per_s": tot_pairs / ms * 1e3,
       "checksum": float(chk), **tot}, flush=True)

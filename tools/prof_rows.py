"""One row-block assembly (chunk c of C) of a BASELINE config on cuda:0 with the per-route statistics
(for ncu launch lists of the sharded assembly):  python tools/prof_rows.py [config] [chunk] [chunks]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import paper_2203_11733_b200 as g  # noqa: E402
from paper_2203_11733_b200 import _native as N  # noqa: E402
from paper_2203_11733_b200.shard import ShardedAssembler, panels_to_device  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
c = int(sys.argv[2]) if len(sys.argv) > 2 else 0
C = int(sys.argv[3]) if len(sys.argv) > 3 else 8
ps = g.config_model(cfg, seed=1).partition(1)
n = len(ps)
ctx = N.Context(0)
dev = torch.device("cuda", 0)
pdev = panels_to_device(ps, dev)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
sh = ShardedAssembler(ctx, pdev, n, c, C)
blk = sh.assemble(with_stats=True)
torch.cuda.synchronize()
print({k: v for k, v in sh.stats.as_dict().items()})

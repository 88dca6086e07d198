"""Per-rank time of the config-5 row-block assembly at N = 1, 2, 4, 8 ranks, measured on one B200 by
running every rank's work-balanced row block (shard.balanced_row_split) alone, one after the other:
the assembly needs no communication, so the N-rank time is the slowest rank's.  A model of the
scaling (ranks do not share a GPU in a real run), not a multi-GPU measurement.
  python tools/config5_rank_model.py [config=5] [chunk_gb=40]"""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2203_11733_b200 as g  # noqa: E402
from paper_2203_11733_b200 import _native as N  # noqa: E402
from paper_2203_11733_b200.shard import balanced_row_split, panels_to_device, row_work  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 5
chunk_gb = float(sys.argv[2]) if len(sys.argv) > 2 else 40.0
ps = g.config_model(cfg_id, seed=1).partition(1)
n = len(ps)
dev = torch.device("cuda", 0)
ctx = N.Context(0)
stream = torch.cuda.Stream(dev)
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
pdev = panels_to_device(ps, dev)
dp = C.POINTER(C.c_double)
panels = N.GbemPanels(C.cast(C.c_void_p(pdev["axis"].data_ptr()), C.POINTER(C.c_uint8)),
                      *[C.cast(C.c_void_p(pdev[k].data_ptr()), dp) for k in ("level", "a0", "a1", "b0", "b1")])
quad = ctx.quad()
ld = (n + 7) // 8 * 8
rows_chunk = max(1, int(chunk_gb * 1e9 / (8 * ld)))
buf = torch.empty((rows_chunk + 1, ld), dtype=torch.float64, device=dev)


def rank_ms(a, b):
    nch = max(1, -(-(b - a) // rows_chunk))
    cuts = [a + (b - a) * k // nch for k in range(nch + 1)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for c0, c1 in zip(cuts[:-1], cuts[1:]):
        if c1 > c0:
            ctx.check(ctx.lib.gbem_assemble_rows_dev(ctx.h, C.byref(panels), n, c0, c1, C.byref(quad),
                                                     C.c_void_p(buf.data_ptr()), ld, None))
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


rank_ms(0, min(n, 2000))  # warm-up
out = {"config": cfg_id, "panels": n, "unique_entries": n * (n + 1) // 2, "chunk_gb": chunk_gb, "worlds": []}
t1 = None
for world in (1, 2, 4, 8):
    split = balanced_row_split(n, world)
    ms = [rank_ms(a, b) for a, b in split]
    t = max(ms)
    t1 = t1 or t
    out["worlds"].append({"ranks": world, "rank_ms": [round(x, 1) for x in ms], "slowest_ms": round(t, 1),
                          "entries_per_s": n * (n + 1) / 2 / (t * 1e-3), "modelled_speedup": round(t1 / t, 3),
                          "modelled_efficiency": round(t1 / t / world, 3),
                          "rank_entries_min_max": [min(row_work(n, a, b) for a, b in split),
                                                   max(row_work(n, a, b) for a, b in split)]})
    print(json.dumps(out["worlds"][-1]), flush=True)
print(json.dumps(out))

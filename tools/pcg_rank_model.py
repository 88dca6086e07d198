"""Per-rank cost of one block-Jacobi PCG iteration for config 4 at P ranks,
measured on one B200 by running rank r's share alone:
its complete rows (gbem_assemble_rows_full_dev), its factored diagonal block,
and per iteration the row-block product (K = 64 right-hand sides) and the
preconditioner solve.  The all-gather of the n x K search directions is not
run (one GPU); its volume is reported for the NVLink estimate.
  python tools/pcg_rank_model.py [P=8] [rank=0]
"""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2203_11733_b200 as g
from paper_2203_11733_b200 import _native as N
from paper_2203_11733_b200.pcg import GpuRowBlockOps
from paper_2203_11733_b200.shard import panels_to_device

P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
rank = int(sys.argv[2]) if len(sys.argv) > 2 else 0
m = g.config_model(4, seed=1)
ps = m.partition(1)
n = len(ps)
K = len(m.net_ids)
ctx = N.Context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
pd = panels_to_device(ps, torch.device("cuda", 0))
ops = GpuRowBlockOps(ctx, pd, n, rank, P)
e = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
e[0].record()
ops.assemble(with_stats=True)
e[1].record()
ops.factor()
e[2].record()
torch.cuda.synchronize()
p_full = torch.randn((P * ops.m, K), dtype=torch.float64, device="cuda")
r = torch.randn((ops.rows, K), dtype=torch.float64, device="cuda")
for _ in range(2):
    ops.matvec(p_full)
    ops.precond(r)
torch.cuda.synchronize()
reps = 5
e[3].record()
for _ in range(reps):
    ops.matvec(p_full)
e[4].record()
for _ in range(reps):
    ops.precond(r)
e[5].record()
torch.cuda.synchronize()
mv = e[3].elapsed_time(e[4]) / reps
pc = e[4].elapsed_time(e[5]) / reps
gather_bytes = n * K * 8
out = dict(config=4, panels=n, K=K, ranks=P, rank=rank, rows=ops.rows,
           row_block_gb=ops.rows * ops.ld * 8 / 1e9,
           assemble_rows_ms=e[0].elapsed_time(e[1]), assembled_pairs=ops.astats.pairs_total,
           factor_diag_ms=e[1].elapsed_time(e[2]),
           matvec_ms=mv, matvec_tflops=2.0 * ops.rows * n * K / (mv * 1e-3) / 1e12,
           matvec_hbm_gbs=ops.rows * n * 8 / (mv * 1e-3) / 1e9,
           precond_ms=pc, iteration_compute_ms=mv + pc,
           allgather_bytes=gather_bytes,
           allgather_ms_at_400GBps=gather_bytes / 400e9 * 1e3,
           note="all-gather estimate: NCCL ring all-gather moves (P-1)/P of n*K*8 B per rank; "
                "400 GB/s is a conservative achieved NVLink-5 bus bandwidth (900 GB/s/direction peak)")
print(json.dumps(out), flush=True)

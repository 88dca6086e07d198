"""Per-rank cost of the sharded config-4 solve at P ranks, measured on one B200
by running rank r's share of gbem_pcg_extract_cmatrix_dev alone (SURVEY.md
section 8e): the context is given P ranks through host collectives whose
all-gather replicates this rank's slot on the device (on the context's stream,
no host synchronisation) and whose all-reduce leaves the local sums — so the
numerics are not the P-rank solve, but every kernel of rank r runs at its real
shape: its complete rows, the explicit inverse of its diagonal block, and per
iteration the split-K row-block product and the preconditioner GEMM.  The
NVLink all-gather of the n x K search directions is estimated from its volume.
  python tools/pcg_rank_model.py [P=8] [rank=0] [iterations=20]
"""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_11733_b200 as g  # noqa: E402
from paper_2203_11733_b200 import _native as N  # noqa: E402
from paper_2203_11733_b200.pcg import _DevView, equal_row_split  # noqa: E402
from paper_2203_11733_b200.shard import panels_to_device  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
rank = int(sys.argv[2]) if len(sys.argv) > 2 else 0
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20

m = g.config_model(4, seed=1)
ps = m.partition(1)
ids = m.net_ids
col = {nid: k for k, nid in enumerate(ids)}
net = np.array([col.get(int(v), -1) if k == 0 else -1 for v, k in zip(ps.net, ps.kind)], dtype=np.int32)
K, eps, n = len(ids), m.info()["eps_r"], len(ps)


def all_gather(user, send, recv, count, stream):
    s = torch.as_tensor(_DevView(send, count), device="cuda")
    r = torch.as_tensor(_DevView(recv, count * P), device="cuda").view(P, count)
    r.copy_(s.expand(P, count))
    return 0


def all_reduce(user, buf, count, stream):
    return 0


ag, ar = N.AllGatherFn(all_gather), N.AllReduceFn(all_reduce)
coll = N.GbemCollectives(None, ag, ar)
ctx = N.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
ctx.check(ctx.lib.gbem_ctx_set_collectives(ctx.h, P, rank, C.byref(coll)))
pd = panels_to_device(ps, torch.device("cuda", 0))
dp = C.POINTER(C.c_double)
panels = N.GbemPanels(C.cast(C.c_void_p(pd["axis"].data_ptr()), C.POINTER(C.c_uint8)),
                      *[C.cast(C.c_void_p(pd[k].data_ptr()), dp) for k in ("level", "a0", "a1", "b0", "b1")])
d_net = torch.from_numpy(net).cuda()
Cm = torch.zeros(K * K, dtype=torch.float64, device="cuda")
res = torch.zeros(K, dtype=torch.float64, device="cuda")
rb, re = equal_row_split(n, P)[rank]
jb = max(1, -(-(re - rb) // 12032))  # the bench's Jacobi blocks of ~12k rows at every rank count
opt = N.GbemPcgOptions(1e-300, iters, jb)
out = []
for rep in range(2):
    pst = N.GbemPcgStats()
    rc = ctx.lib.gbem_pcg_extract_cmatrix_dev(ctx.h, C.byref(panels), n, C.c_void_p(d_net.data_ptr()), K, eps,
                                              C.byref(ctx.quad()), C.byref(opt), C.c_void_p(Cm.data_ptr()),
                                              C.c_void_p(res.data_ptr()), None, None, C.byref(pst))
    assert rc in (0, 2), ctx.lib.gbem_last_error(ctx.h).decode()  # 2: tol 1e-300 is never reached
    torch.cuda.synchronize()
    out.append(pst)
st = out[-1]
ag_bytes = (P - 1) / P * n * 64 * 8
line = {"config": 4, "panels": n, "K": K, "ranks": P, "rank": rank, "rows": re - rb, "jacobi_blocks": jb,
        "row_block_gb": (re - rb) * ((n + 7) // 8 * 8) * 8 / 1e9,
        "assemble_rows_ms": st.ms_assembly, "precond_setup_ms": st.ms_precond,
        "iterations": st.iterations, "iteration_ms": st.ms_iterations / max(1, st.iterations + 1),
        "matvec_ms": st.ms_matvec, "matvec_tflops": st.matvec_flops / (st.ms_matvec * 1e-3) / 1e12,
        "allgather_bytes_per_rank": ag_bytes, "allgather_ms_at_400GBps": ag_bytes / 400e9 * 1e3,
        "note": "iteration_ms = (iterations phase incl. the one extra lagged iteration) / (iterations + 1); "
                "the device-side all-gather here is 8 local copies; NCCL ring all-gather moves (P-1)/P of "
                "n*K*8 B per rank, 400 GB/s is a conservative achieved NVLink-5 rate (900 GB/s/direction peak)"}
print(json.dumps(line), flush=True)
ctx.close()

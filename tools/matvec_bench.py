"""Row-block product timing (gbem_rowblock_matvec_dev): HBM GB/s on the A block."""
import ctypes as C, json, sys
import torch
sys.path.insert(0, ".")
from paper_2203_11733_b200._native import Context
ctx = Context(0)
s = torch.cuda.current_stream()
s = torch.cuda.Stream(); torch.cuda.set_stream(s); ctx.set_stream(s.cuda_stream)
out = []
for rows, n, K in [(8192, 65536, 1), (8192, 65536, 8), (8192, 65536, 16), (8192, 65536, 64), (12544, 100000, 8)]:
    ld = ((n + 7) // 8) * 8
    A = torch.randn((rows, ld), dtype=torch.float64, device="cuda")
    P = torch.randn((n, K), dtype=torch.float64, device="cuda")
    Q = torch.empty((rows, K), dtype=torch.float64, device="cuda")
    args = (ctx.h, C.c_void_p(A.data_ptr()), ld, rows, n, C.c_void_p(P.data_ptr()), K, K, C.c_void_p(Q.data_ptr()), K)
    for _ in range(3):
        ctx.check(ctx.lib.gbem_rowblock_matvec_dev(*args))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        ctx.check(ctx.lib.gbem_rowblock_matvec_dev(*args))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ref = (A[:64, :n].cpu() @ P.cpu())
    err = float((Q[:64].cpu() - ref).abs().max() / ref.abs().max())
    passes = 1 if K <= 8 else -(-K // 64)
    gbs = rows * n * 8 * passes / ms / 1e6
    out.append(dict(rows=rows, n=n, K=K, ms=ms, a_gbs=gbs, tflops=2.0 * rows * n * K / ms / 1e9, err=err))
    print(json.dumps(out[-1]))
    del A

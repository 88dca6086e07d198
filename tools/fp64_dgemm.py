"""cuBLAS DGEMM ceiling (torch.matmul float64) on one B200: burst best-of-10 and 4 s sustained."""
import json, time, torch
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(3): c = a @ b
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
t0 = time.time(); k = 0
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 4.0:
    c = a @ b; k += 1
    if k % 8 == 0: torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
sus = e0.elapsed_time(e1) / k
print(json.dumps({"dgemm_n": n, "burst_tflops": 2 * n**3 / best / 1e9, "sustained_tflops": 2 * n**3 / sus / 1e9}))
# cuSOLVER potrf ceiling
for m in (6000, 12000, 25000):
    A = torch.randn(m, m, dtype=torch.float64, device="cuda"); A = A @ A.T + m * torch.eye(m, dtype=torch.float64, device="cuda")
    torch.linalg.cholesky(A); torch.cuda.synchronize()
    e0.record(); L = torch.linalg.cholesky(A); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(json.dumps({"potrf_n": m, "ms": ms, "tflops": m**3 / 3 / ms / 1e9}))
    del A, L

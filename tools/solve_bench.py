"""Factor + K-RHS solve timing through the C-ABI on a random SPD matrix
(gbem_spd_factor_dev / gbem_spd_solve_factored_dev), per GBEM_SOLVE_DBG mode."""
import ctypes as C, json, os, subprocess, sys
import torch
sys.path.insert(0, ".")
from paper_2203_11733_b200._native import Context, GbemSolveStats

n = int(sys.argv[1]) if len(sys.argv) > 1 else 11340
R = int(sys.argv[2]) if len(sys.argv) > 2 else 6
ctx = Context(0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); ctx.set_stream(s.cuda_stream)
g = torch.Generator(device="cuda").manual_seed(1)
G = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
M = G @ G.T / n + torch.eye(n, dtype=torch.float64, device="cuda")
del G
ld = n
st = GbemSolveStats()
ctx.check(ctx.lib.gbem_spd_factor_dev(ctx.h, C.c_void_p(M.data_ptr()), n, ld, C.byref(st)))
B = torch.randn((R, n), dtype=torch.float64, device="cuda", generator=g)
X = torch.empty_like(B)
res = torch.empty(R, dtype=torch.float64, device="cuda")
for _ in range(3):
    ctx.check(ctx.lib.gbem_spd_solve_factored_dev(ctx.h, C.c_void_p(B.data_ptr()), R, C.c_void_p(X.data_ptr()), None, C.byref(st)))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    ctx.check(ctx.lib.gbem_spd_solve_factored_dev(ctx.h, C.c_void_p(B.data_ptr()), R, C.c_void_p(X.data_ptr()), None, None))
e1.record(); torch.cuda.synchronize()
ctx.check(ctx.lib.gbem_spd_solve_factored_dev(ctx.h, C.c_void_p(B.data_ptr()), R, C.c_void_p(X.data_ptr()), C.c_void_p(res.data_ptr()), None))
print(json.dumps(dict(n=n, R=R, dbg=os.environ.get("GBEM_SOLVE_DBG", "0"), solve_ms=e0.elapsed_time(e1) / 5,
                      factor_ms=st.ms_factor, resid=float(res.max()))))

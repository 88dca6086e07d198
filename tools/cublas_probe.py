import torch
from paper_2203_11733_b200._native import Context
c = Context(0)
try:
    a = torch.randn(64, 64, dtype=torch.float64, device="cuda")
    print("matmul after ctx ok", float((a @ a).sum()))
except Exception as e:
    print("matmul after ctx FAILED", e)
print(torch.cuda.mem_get_info())

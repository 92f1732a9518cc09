"""Which cuBLAS kernel runs a stage GEMM shape (diagnostic, run under ncu)."""
import sys
import torch
m, n, k = (int(x) for x in sys.argv[1:4])
a = torch.randn(m, k, device="cuda").to(torch.bfloat16)
b = torch.randn(n, k, device="cuda").to(torch.bfloat16)
for _ in range(5):
    torch.mm(a, b.t())
torch.cuda.synchronize()

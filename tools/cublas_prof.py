"""torch.matmul (cuBLAS) at s^3 bf16 -- a target for ncu metric comparison."""
import sys
import torch
s = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
a = torch.randn(s, s, device="cuda", dtype=torch.bfloat16)
b = torch.randn(s, s, device="cuda", dtype=torch.bfloat16)
c = torch.empty(s, s, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    torch.matmul(a, b, out=c)
torch.cuda.synchronize()

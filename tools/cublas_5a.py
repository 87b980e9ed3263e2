"""cuBLAS / copy reference points for BASELINE config 5a (65536x256x4096 BF16)."""
import torch
A=torch.randn(65536,4096,device='cuda').bfloat16(); B=torch.randn(4096,256,device='cuda').bfloat16()
Bt=B.t().contiguous()
C=torch.empty(65536,256,device='cuda',dtype=torch.bfloat16)
Cf=torch.randn(65536,256,device='cuda')
def t(f,n=20):
    for _ in range(3): f()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    ts=[]
    for _ in range(n):
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1)*1e3)
    ts.sort(); return ts[len(ts)//2]
print("cublas bf16 out", t(lambda: torch.matmul(A,B,out=C)))
print("cublas bf16 out Bt", t(lambda: torch.matmul(A,Bt.t(),out=C)))
print("A.sum read", t(lambda: A.sum(dtype=torch.float32)))
X=torch.empty_like(A)
print("copy A", t(lambda: X.copy_(A)))

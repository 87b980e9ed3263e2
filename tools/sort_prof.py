"""Run the radix sort variant on n random FP32 keys (ncu target)."""
import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2311_03543_b200 import compar as cm
ctx = cm.Compar()
names = [n for n, _ in ctx.variants()]
n = int(sys.argv[1])
x = torch.randint(-2**31, 2**31-1, (n,), dtype=torch.int32, device='cuda').view(torch.float32)
for _ in range(3):
    t = x.clone()
    r = ctx.sort(t, key_type=cm.KEY_F32, variant_hint=names.index('sort_radix'))
    print(r.ns)
ctx.terminate()

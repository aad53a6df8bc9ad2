"""One representative K1/K2 launch pair (slice 4 of the c2 step: Ls=16K,
32 heads, d=128, 4 chunks) for ncu captures; run plain first, then under ncu."""
import sys
import torch
sys.path.insert(0, '.')
from paper_2504_14519_b200 import ops
L, n, heads, d = 16384, 4, 32, 128
q = torch.randn(L, heads * d, device='cuda', dtype=torch.bfloat16)
kp = torch.randn(n * L, heads * d, device='cuda', dtype=torch.bfloat16)
vp = torch.randn(n * L, heads * d, device='cuda', dtype=torch.bfloat16)
do = torch.randn(L, heads * d, device='cuda', dtype=torch.bfloat16)
rows = [c * L for c in range(n)]
dq = torch.zeros(L, heads * d, device='cuda'); dk = torch.zeros(n * L, heads * d, device='cuda'); dv = torch.zeros_like(dk)
ws = torch.empty(2 * heads * L, device='cuda')
for it in range(2):
    o, lse = ops.attn_fwd(q, kp, vp, rows, L, heads, heads, True)
    ops.attn_bwd(q, kp, vp, rows, L, heads, heads, True, o, lse, do, dq, dk, dv, rows, ws)
torch.cuda.synchronize()
print("ok", float(dq.abs().sum()))

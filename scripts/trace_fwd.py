import os, sys, ctypes as C
os.environ["SP_FWD_TRACE"] = "1"
import torch, numpy as np
sys.path.insert(0, '.')
from paper_2504_14519_b200 import ops, native
L, n, heads, d = 16384, 4, 32, 128
q = torch.randn(L, heads * d, device='cuda', dtype=torch.bfloat16)
kp = torch.randn(n * L, heads * d, device='cuda', dtype=torch.bfloat16)
vp = torch.randn(n * L, heads * d, device='cuda', dtype=torch.bfloat16)
rows = [c * L for c in range(n)]
for _ in range(2):
    o, lse = ops.attn_fwd(q, kp, vp, rows, L, heads, heads, True)
torch.cuda.synchronize()
buf = (C.c_longlong * (12 * 1024))()
native.lib().sp_debug_fwd_trace(buf)
t = np.array(buf[:], dtype=np.int64).reshape(12, 1024)
t = t - t[0, 0]
names = ["mma_top", "s_issued", "p_full_ok", "v_full_ok", "pv_issued", "sm_top", "s_full_ok", "max_done", "exp_done", "arrived", "k_full_ok(j)"]
nt = int((t[0] > 0).sum()) + 1
print("tiles", nt)
per = np.diff(t[0, 10:nt - 5])
print("mean period (cycles)", per.mean())
for e in range(1, 11):
    print(f"{names[e]:10s} - mma_top  median {np.median(t[e, 10:nt-5] - t[0, 10:nt-5]):8.0f}")
print("k_full_ok(j+1) - mma_top(j) median", np.median(t[10, 11:nt-4] - t[0, 10:nt-5]))

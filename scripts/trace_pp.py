"""Per-tile timeline of one CTA of the ping-pong attention forward (K1)."""
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
buf = (C.c_longlong * (16 * 1024))()
native.lib().sp_debug_pp_trace(buf)
t = np.array(buf[:], dtype=np.int64).reshape(16, 1024).astype(np.float64)
nt = int((t[0] > 0).sum())
t = t - t[0, 0]
a, b = 20, nt - 5
print("tiles", nt, "mean period", np.diff(t[0, a:b]).mean())
names = {0: "mma_top", 1: "v_full", 2: "pA_ok", 3: "PV_A issued", 4: "S_A issued", 5: "pB_ok", 6: "PV_B issued",
         7: "S_B issued", 8: "A s_full", 9: "A max", 10: "A exps", 11: "A arrive", 12: "B s_full", 13: "B max",
         14: "B exps", 15: "B arrive"}
for e in range(1, 16):
    print(f"{names[e]:12s} {np.median(t[e, a:b] - t[0, a:b]):8.0f}")

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
native.lib().sp_debug_ps_trace(buf)
t = np.array(buf[:], dtype=np.int64).reshape(16, 1024).astype(np.float64)
nt = int((t[0] > 0).sum())
t = t - t[0, 0]
a, b = 20, nt - 5
print("tiles", nt, "mean period", np.diff(t[0, a:b]).mean())
# MMA events: 0 = S issue (indexed by S-stream position k: A_j at 2j, B_j at 2j+1), 2/3 = PV_A/PV_B issue (by j)
nj = (nt + 1) // 2
a, b = 20, nj - 5
sA = t[0, 0::2][:nj]; sB = t[0, 1::2][:nj]
rel = lambda e, ref: np.median(e[a:b] - ref[a:b])
base = t[8, :nj]  # A s_full ok (j)
print("period (A s_full)", np.diff(base[a:b]).mean())
for nm, ev in [("S_A issued(j)", sA), ("S_B issued(j)", sB), ("PV_A issued", t[2, :nj]), ("PV_B issued", t[3, :nj]),
               ("A max", t[9, :nj]), ("A exps", t[10, :nj]), ("A arrive", t[11, :nj]),
               ("B s_full", t[12, :nj]), ("B max", t[13, :nj]), ("B exps", t[14, :nj]), ("B arrive", t[15, :nj])]:
    print(f"{nm:16s} {rel(ev, base):8.0f}")

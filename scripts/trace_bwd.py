import os, sys, ctypes as C
os.environ["SP_BWD_TRACE"] = "1"
import torch, numpy as np
sys.path.insert(0, '.')
from paper_2504_14519_b200 import ops, native
L, n, heads, d = 16384, 1, 32, 128
q = torch.randn(L, heads * d, device='cuda', dtype=torch.bfloat16)
kp = torch.randn(n * L, heads * d, device='cuda', dtype=torch.bfloat16)
vp = torch.randn(n * L, heads * d, device='cuda', dtype=torch.bfloat16)
do = torch.randn(L, heads * d, device='cuda', dtype=torch.bfloat16)
rows = [c * L for c in range(n)]
dq = torch.zeros(L, heads * d, device='cuda'); dk = torch.zeros(n * L, heads * d, device='cuda'); dv = torch.zeros_like(dk)
ws = torch.empty(2 * heads * L, device='cuda')
o, lse = ops.attn_fwd(q, kp, vp, rows, L, heads, heads, True)
for _ in range(2):
    ops.attn_bwd(q, kp, vp, rows, L, heads, heads, True, o, lse, do, dq, dk, dv, rows, ws)
torch.cuda.synchronize()
buf = (C.c_longlong * 6144)()
lib = native.lib()
lib.sp_debug_bwd_trace(buf)
t = np.array(buf[:], dtype=np.int64).reshape(12, 512)
t = t - t[0, 0]
names = ["sdp_top(j)", "sdp_issued(j)", "acc: pds_ready_ok(j)", "acc: issued(j)", "drain_dqfull_ok(j)", "sdp_full_ok", "compute_done", "pds_free_ok", "pds_ready_arr", "drain_staged(j)", "sdp: q/dq/acc free ok(j)", "-"]
per = np.diff(t[0, 10:250])
print("mean period (cycles)", per.mean())
for e in range(1, 11):
    print(names[e], "-", names[0], np.median(t[e, 10:250] - t[0, 10:250]))

"""Launch each MoE kernel once at config-4 shapes (Phi-3.5-MoE: seq 3072,
hidden 4096, 16 experts, top-2, capacity 512 — the pre-rounding-change capacity) for an ncu capture of achieved
DRAM bandwidth (same recipe as tools/hbm_kernels.py):

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \\
      --clock-control none --csv python tools/moe_kernels.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_15871_b200 import device as dh  # noqa: E402

T, H, E, K, C = 3072, 4096, 16, 2, 512
R = E * C
bf = dict(device="cuda", dtype=torch.bfloat16)
x = torch.randn(T, H, **bf)
wr = (torch.randn(E, H, device="cuda") * 0.02).to(torch.bfloat16)
probs = torch.empty(T, E, device="cuda")
ids = torch.empty(T, K, dtype=torch.int32, device="cuda")
wts = torch.empty(T, K, device="cuda")
slot = torch.empty(T, K, dtype=torch.int32, device="cuda")
slot_src = torch.empty(R, dtype=torch.int32, device="cuda")
xp = torch.empty(R, H, **bf)
y = torch.randn(R, H, **bf)
out = torch.empty(T, H, **bf)
dy = torch.randn(T, H, **bf)
dys = torch.empty(R, H, **bf)
dw = torch.zeros(T, K, device="cuda")
dx = torch.empty(T, H, **bf)
dwr = torch.zeros(E, H, device="cuda")

expect = {}
dh.moe_router_fwd(x, wr, probs, ids, wts, K)
expect["router_fwd (GEMM + topk)"] = T * H * 2 + T * E * 4 * 2 + T * K * 8
dh.moe_assign(ids, E, C, slot, slot_src)
expect["assign"] = T * K * 4 * 2 + R * 4
dh.moe_permute(x, slot_src, xp, K)
expect["permute"] = R * H * 2 + T * K * H * 2  # every slot row written, routed rows read
dh.moe_unpermute(y, slot, wts, out)
expect["unpermute"] = T * K * H * 2 + T * H * 2
dh.moe_unpermute_bwd(dy, y, slot_src, wts, dys, dw, K)
expect["unpermute_bwd"] = R * H * 2 + 2 * T * K * H * 2
dh.moe_permute_bwd(y, slot, dx)
expect["permute_bwd"] = T * K * H * 2 + T * H * 2
dh.moe_router_bwd(probs, ids, slot, dw, x, wr, dx, dx, dwr)
expect["router_bwd (dlogits + 2 GEMMs)"] = 3 * T * H * 2
torch.cuda.synchronize()
print(json.dumps({"algorithmic_bytes_per_launch": expect, "shape": {"T": T, "H": H, "E": E, "K": K, "C": C}}))

"""Launch each HBM-bound kernel once at the TP=1 Llama-3-8B layer shapes (seq
4096) for an ncu capture of achieved DRAM bandwidth:

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv python tools/hbm_kernels.py

Algorithmic bytes per launch are printed so the capture can be read against them.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_15871_b200 import device as dh  # noqa: E402

S, H, F, NQ, NKV, D = 4096, 4096, 14336, 32, 8, 128
Q = (NQ + 2 * NKV) * D
bf = dict(device="cuda", dtype=torch.bfloat16)
x = torch.randn(S, H, **bf)
gamma = torch.ones(H, **bf)
y = torch.empty(S, H, **bf)
rstd = torch.empty(S, device="cuda")
dy = torch.randn(S, H, **bf)
dx = torch.empty(S, H, **bf)
dg = torch.zeros(H, device="cuda")
gate, up = torch.randn(S, F, **bf), torch.randn(S, F, **bf)
act, dact, dgate, dup = (torch.empty(S, F, **bf) for _ in range(4))
qkv = torch.randn(S, Q, **bf)
n_opt = 218_103_808  # one Llama-3-8B layer's parameters
master = torch.randn(n_opt, device="cuda")
grad, m1, v1 = torch.randn(n_opt, device="cuda"), torch.zeros(n_opt, device="cuda"), torch.zeros(n_opt, device="cuda")
wb = torch.empty(n_opt, **bf)

expect = {}
dh.rmsnorm_fwd(x, gamma, y, rstd)
expect["rmsnorm_fwd"] = 2 * S * H * 2 + S * 4
dh.rmsnorm_bwd(x, gamma, rstd, dy, dx, dgamma_acc=dg)
expect["rmsnorm_bwd"] = 3 * S * H * 2 + S * 4
dh.add(x, dy, y)
expect["add"] = 3 * S * H * 2
dh.swiglu_fwd(gate, up, act)
expect["swiglu_fwd"] = 3 * S * F * 2
dh.swiglu_bwd(gate, up, act, dgate, dup)
expect["swiglu_bwd"] = 5 * S * F * 2
dh.rope(qkv, NQ, NKV, D, 500000.0)
expect["rope"] = 2 * S * (NQ + NKV) * D * 2
dh.adamw(master, wb, grad, m1, v1, 1e-4)
expect["adamw"] = n_opt * 34
torch.cuda.synchronize()
print(json.dumps({"algorithmic_bytes_per_launch": expect}))

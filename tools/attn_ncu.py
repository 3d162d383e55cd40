"""One attention fwd + bwd launch at a chosen per-GPU head count (ncu target)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_15871_b200 import device as dh
nq = int(sys.argv[1]) if len(sys.argv) > 1 else 32
T, nkv, d = 4096, max(1, nq // 4), 128
qkv = (torch.randn(T, (nq + 2 * nkv) * d, device="cuda") * 0.5).to(torch.bfloat16)
q, k, v = qkv[:, :nq * d], qkv[:, nq * d:(nq + nkv) * d], qkv[:, (nq + nkv) * d:]
o = torch.empty(T, nq * d, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(nq, T, device="cuda")
do = torch.randn_like(o)
dqkv = torch.empty_like(qkv)
scratch = torch.empty(dh.attn_bwd_scratch_floats(T, nq, nkv, d), device="cuda")
for _ in range(2):
    dh.attn_fwd(q, k, v, o, lse, nq, nkv, d, d ** -0.5)
    dh.attn_bwd(q, k, v, o, lse, do, dqkv[:, :nq * d], dqkv[:, nq * d:(nq + nkv) * d],
                dqkv[:, (nq + nkv) * d:], nq, nkv, d, d ** -0.5, scratch=scratch)
torch.cuda.synchronize()

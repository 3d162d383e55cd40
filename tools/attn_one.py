import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2411_15871_b200 import device as dh
T, nq, nkv, d = 4096, 4, 1, 128
qkv = (torch.randn(T, (nq + 2 * nkv) * d, device="cuda") * 0.5).to(torch.bfloat16)
q, k, v = qkv[:, :nq * d], qkv[:, nq * d:(nq + nkv) * d], qkv[:, (nq + nkv) * d:]
o = torch.empty(T, nq * d, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(nq, T, device="cuda")
for _ in range(3):
    dh.attn_fwd(q, k, v, o, lse, nq, nkv, d, d ** -0.5)
torch.cuda.synchronize()

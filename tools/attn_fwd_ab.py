"""Forward attention output + lse for a fixed seeded input, saved to a file
(A/B bitwise comparison of build / env variants). usage: attn_fwd_ab.py <nq> <out.pt>"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_15871_b200 import device as dh
nq = int(sys.argv[1])
T, nkv, d = 4096, max(1, nq // 4), 128
g = torch.Generator(device="cuda").manual_seed(7)
qkv = (torch.randn(T, (nq + 2 * nkv) * d, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
q, k, v = qkv[:, :nq * d], qkv[:, nq * d:(nq + nkv) * d], qkv[:, (nq + nkv) * d:]
o = torch.empty(T, nq * d, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(nq, T, device="cuda")
for _ in range(3):
    dh.attn_fwd(q, k, v, o, lse, nq, nkv, d, d ** -0.5)
torch.cuda.synchronize()
torch.save({"o": o.cpu(), "lse": lse.cpu()}, sys.argv[2])

"""clock64 timeline of one attention-backward CTA. Build a traced copy of the
library first:  make cuda NVFLAGS_EXTRA=-DDH_ATTN_TRACE=<block>  (block 0 = the
heaviest dK/dV item of head 0; block nq = the heaviest dQ item).
usage: attn_trace.py <nq> [iterations]"""
import sys, os, ctypes
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
for _ in range(3):
    dh.attn_fwd(q, k, v, o, lse, nq, nkv, d, d ** -0.5)
    dh.attn_bwd(q, k, v, o, lse, do, dqkv[:, :nq * d], dqkv[:, nq * d:(nq + nkv) * d], dqkv[:, (nq + nkv) * d:],
                nq, nkv, d, d ** -0.5)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * 1024)()
dh.lib().dh_attn_trace_read(buf, 1024)
t0 = buf[3]
print("cycles relative to the first S ready (EW). mma: [0] before wait P / s_free, [1] after, [2] got dS | "
      "ew: [7] iter start, [3] got S, [4] P done / S read, [5] got dP, [6] dS done")
prev = None
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 32):
    r = [buf[it * 8 + j] - t0 for j in range(8)]
    if r[3] < 0 and it > 0:
        break
    dt = "" if prev is None else f"  (+{r[3] - prev})"
    prev = r[3]
    print(it, "mma", r[0], r[1], r[2], "| ew", r[7], r[3], r[4], r[5], r[6], dt)

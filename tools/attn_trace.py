"""clock64 timeline of one attention-backward CTA (build with -DDH_ATTN_TRACE=<block>)."""
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
print("it mma_s_issued(it+1) mma_got_p(it) | ew: wait_s got_s ld_done bar_done math_done arrive   (cycles rel. to it0 s_full)")
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 64):
    r = [buf[it * 8 + j] - t0 for j in range(8)]
    print(it, r[0], r[1], "|", r[2], r[3], r[5], r[6], r[7], r[4])

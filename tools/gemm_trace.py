"""Where a single-wave CTA-pair GEMM spends its time: per-CTA globaltimer
stamps (build with NVFLAGS_EXTRA=-DDH_GEMM_TRACE).
usage: gemm_trace.py m n k [pair_tile_n (256|192|128)] [b_mn 0|1] [flush 0|1] [rewarm a|b]
(rewarm: after the L2 flush, read A or B once so only the other operand is cold)
env EPI=fwd|bwd: the fused SwiGLU forward / backward epilogue (aux operands random)"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_15871_b200 import device as dh
m, n, k = (int(x) for x in sys.argv[1:4])
pbn = int(sys.argv[4]) if len(sys.argv) > 4 else 256
b_mn = len(sys.argv) > 5 and sys.argv[5] == "1"
do_flush = not (len(sys.argv) > 6 and sys.argv[6] == "0")
kw = dict(tile_n=512 if pbn == 256 else -pbn, b_mn=b_mn)  # a CTA-pair kernel, 256 x pbn tiles
a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
b = torch.randn((k, n) if b_mn else (n, k), device="cuda", dtype=torch.bfloat16)
d = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
epi = os.environ.get("EPI", "")
if epi:
    x0 = torch.randn(m, n, device="cuda", dtype=torch.bfloat16)
    x1 = torch.randn(m, n, device="cuda", dtype=torch.bfloat16)
    d2 = torch.empty_like(d)
    kw.update(epilogue=dh.EPI_SWIGLU_FWD if epi == "fwd" else dh.EPI_SWIGLU_BWD, d2=d2, aux0=x0,
              aux1=x1 if epi == "bwd" else None)
flush = torch.empty(256 << 20, dtype=torch.int8, device="cuda")
for _ in range(3):
    dh.gemm(a, b, d, **kw)
torch.cuda.synchronize()
torch.cuda.synchronize()
if do_flush:
    flush.zero_()
    rewarm = sys.argv[7] if len(sys.argv) > 7 else ""
    if rewarm:
        (a if rewarm == "a" else b).sum(dtype=torch.float32)
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
dh.gemm(a, b, d, **kw)
e.record()
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (512 * 8))()
dh.lib().dh_gemm_trace_read(buf, 512 * 8)
tiles = -(-m // 256) * -(-n // pbn)
ctas = 2 * min(torch.cuda.get_device_properties(0).multi_processor_count // 2, tiles)
rows = [[buf[c * 8 + i] for i in range(6)] for c in range(ctas)]
t0 = min(r[0] for r in rows)
print(f"event time {s.elapsed_time(e) * 1e3:.1f} us; {ctas} CTAs; stamps relative to the first CTA entry (us)")
names = ["entry", "prologue", "first_mma", "last_acc", "stores_drained", "exit"]
for i, nm in enumerate(names):
    vals = sorted((r[i] - t0) / 1e3 for r in rows if r[i] >= t0)
    if vals:
        print(f"  {nm:15s} min {vals[0]:7.2f}  median {vals[len(vals) // 2]:7.2f}  max {vals[-1]:7.2f}")

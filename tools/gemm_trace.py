"""Where a single-wave CTA-pair GEMM spends its time: per-CTA globaltimer
stamps (build with NVFLAGS_EXTRA=-DDH_GEMM_TRACE). usage: gemm_trace.py m n k"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_15871_b200 import device as dh
m, n, k = (int(x) for x in sys.argv[1:4])
kw = dict(tile_n=512)  # the 256 x 256 CTA-pair kernel
a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
b = torch.randn(n, k, device="cuda", dtype=torch.bfloat16)
d = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
flush = torch.empty(256 << 20, dtype=torch.int8, device="cuda")
for _ in range(3):
    dh.gemm(a, b, d, **kw)
torch.cuda.synchronize()
torch.cuda.synchronize()
flush.zero_()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
dh.gemm(a, b, d, **kw)
e.record()
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (512 * 8))()
dh.lib().dh_gemm_trace_read(buf, 512 * 8)
tiles = -(-m // 256) * -(-n // 256)
ctas = 2 * min(torch.cuda.get_device_properties(0).multi_processor_count // 2, tiles)
rows = [[buf[c * 8 + i] for i in range(6)] for c in range(ctas)]
t0 = min(r[0] for r in rows)
print(f"event time {s.elapsed_time(e) * 1e3:.1f} us; {ctas} CTAs; stamps relative to the first CTA entry (us)")
names = ["entry", "prologue", "first_mma", "last_acc", "stores_drained", "exit"]
for i, nm in enumerate(names):
    vals = sorted((r[i] - t0) / 1e3 for r in rows if r[i] >= t0)
    if vals:
        print(f"  {nm:15s} min {vals[0]:7.2f}  median {vals[len(vals) // 2]:7.2f}  max {vals[-1]:7.2f}")

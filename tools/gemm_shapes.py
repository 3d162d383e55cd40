"""CUDA-event TF/s of the layer GEMM shapes (TP=1 and TP=8 per-GPU), L2 flushed
between launches, for A/B builds."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_15871_b200 import device as dh
flush = torch.empty(256 << 20, dtype=torch.int8, device="cuda")


def timeit(fn, iters=15):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(iters):
        flush.zero_()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


shapes = [("tp1_gate", 4096, 14336, 4096, 0, 0, 0), ("tp1_down", 4096, 4096, 14336, 0, 0, 0),
          ("tp1_fc1_wgrad", 14336, 4096, 4096, 1, 1, 1), ("tp1_qkv", 4096, 6144, 4096, 0, 0, 0),
          ("tp8_gate", 4096, 1792, 4096, 0, 0, 0), ("tp8_qkv", 4096, 768, 4096, 0, 0, 0),
          ("tp8_attn_proj", 4096, 4096, 512, 0, 0, 0), ("tp8_fc1_wgrad", 1792, 4096, 4096, 1, 1, 1)]
for name, m, n, k, amn, bmn, f32 in shapes:
    a = torch.randn((k, m) if amn else (m, k), device="cuda", dtype=torch.bfloat16)
    b = torch.randn((k, n) if bmn else (n, k), device="cuda", dtype=torch.bfloat16)
    d = torch.zeros(m, n, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
    ms = timeit(lambda: dh.gemm(a, b, d, a_mn=bool(amn), b_mn=bool(bmn), m=m, n=n, k=k, accumulate=bool(f32)))
    print(json.dumps({"name": name, "us": round(ms * 1e3, 1), "tflops": round(2 * m * n * k / ms / 1e9, 1)}), flush=True)

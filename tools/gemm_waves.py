"""Does wave quantisation cost time on a power-capped B200? Time 256x256
CTA-pair GEMMs (K=4096) with exactly 2, 3, 4 waves of 74 pairs and with 3.46
waves (Llama-3-8B TP=1 attn_proj / mlp_down / dgrad shapes), warm back-to-back
launches (in-step-like power state) and L2-flushed; microseconds per tile."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_15871_b200 import device as dh
flush = torch.empty(256 << 20, dtype=torch.int8, device="cuda")


def timeit(fn, fl, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    if not fl:
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(iters):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / iters
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


for m, n in [(9472, 1024), (9472, 1536), (9472, 2048), (4096, 4096), (4096, 3840)]:
    k = 4096
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(n, k, device="cuda", dtype=torch.bfloat16)
    d = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    tiles = (m // 256) * (n // 256)
    for fl in (False, True):
        ms = timeit(lambda: dh.gemm(a, b, d, tile_n=512), fl)
        print(json.dumps({"m": m, "n": n, "tiles": tiles, "waves": round(tiles / 74, 2), "flush": fl,
                          "us": round(ms * 1e3, 1), "us_per_tile": round(ms * 1e3 / tiles, 3),
                          "tflops": round(2 * m * n * k / ms / 1e9, 1)}), flush=True)

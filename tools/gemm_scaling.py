"""Per-pair k-block time of the CTA-pair GEMM vs the number of active pairs
(max_ctas), with and without an L2 flush: is there a shared throughput limit?"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_15871_b200 import device as dh

flush = torch.empty(256 * 1024 * 1024, dtype=torch.int8, device="cuda")


def timeit(fn, do_flush, iters=15):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(iters):
        if do_flush:
            flush.zero_()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


for name, m, n, k in [("qkv", 4096, 768, 4096), ("gate", 4096, 1792, 4096), ("tp1_gate", 4096, 14336, 4096)]:
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(n, k, device="cuda", dtype=torch.bfloat16)
    d = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    tiles = -(-m // 256) * -(-n // 256)
    for cap in (148, 132, 96, 64, 32, 16):
        for fl in (True, False):
            ms = timeit(lambda: dh.gemm(a, b, d, tile_n=512, max_ctas=cap), fl)
            pairs = min(cap // 2, tiles)
            waves = -(-tiles // pairs)
            kb_per_pair = waves * (k // 64)
            print(json.dumps(dict(name=name, cap=cap, flush=fl, pairs=pairs, waves=waves, us=round(ms * 1e3, 1),
                                  tflops=round(2 * m * n * k / ms / 1e9, 1),
                                  ns_per_kblock=round(ms * 1e6 / kb_per_pair, 1))), flush=True)

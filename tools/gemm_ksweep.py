"""Graph-timed tile comparison for output-heavy GEMMs (large M x N, small K): the
chooser pick (t0) vs CTA-pair and one-CTA tiles at the GEMM SM caps 132 / 148."""
import os, sys, json
sys.path.insert(0, os.getcwd())
import torch
from paper_2411_15871_b200 import device as dh
def timeit(fn, iters=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    st = torch.cuda.Stream(); g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(iters): fn()
    g.replay(); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); g.replay(); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) / iters)
    ts.sort(); return ts[2]
for cap in [int(c) for c in os.environ.get("CAPS", "132,148").split(",")]:
  for (m, n, k) in [tuple(int(x) for x in s.split("x")) for s in os.environ.get("SHAPES", "4096x4096x512,4096x4096x1024,4096x4096x2048,4096x4096x768,4096x4096x1792,4096x5120x1280").split(",")]:
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16); b = torch.randn(n, k, device="cuda", dtype=torch.bfloat16)
    d = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    row = {"m": m, "n": n, "k": k, "cap": cap}
    for t in (0, 512, -192, 256, 192):
        try:
            row[f"t{t}"] = round(2 * m * n * k / timeit(lambda: dh.gemm(a, b, d, tile_n=t, max_ctas=cap)) / 1e9, 1)
        except Exception as ex:
            row[f"t{t}"] = str(ex)[:30]
    print(json.dumps(row), flush=True)

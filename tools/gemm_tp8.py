"""Time every GEMM of one TP=8 layer (Llama-3-8B shapes, seq 4096) the way the
model calls it (majors, fp32 accumulate / bf16 outputs), for each tile choice
and the overlap CTA cap. CUDA events over graph-replayed back-to-back launches
(GRAPH=0: eager single launches after an L2 flush)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_15871_b200 import device as dh  # noqa: E402

flush = torch.empty(256 * 1024 * 1024, dtype=torch.int8, device="cuda")


def timeit(fn, iters=15):
    """Device time per launch: `iters` launches captured in one CUDA graph (no host
    cost between them) and replayed; GRAPH=0 for eager single launches after an L2
    flush (host launch cost included)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    if os.environ.get("GRAPH", "1") != "0":
        st = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(iters):
                fn()
        g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            s, e = torch.cuda.Event(True), torch.cuda.Event(True)
            s.record()
            g.replay()
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e) / iters)
        ts.sort()
        return ts[1]
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


S, H, Q, A, F = 4096, 4096, 768, 512, 1792
# name, m, n, k, a_mn, b_mn, fp32 out (accumulate)
shapes = [("qkv", S, Q, H, 0, 0, 0), ("attn_proj", S, H, A, 0, 0, 0), ("mlp_gate", S, F, H, 0, 0, 0),
          ("mlp_down", S, H, F, 0, 0, 0), ("mlp_down_dgrad", S, F, H, 0, 1, 0),
          ("mlp_gate_dgrad", S, H, F, 0, 1, 0), ("attn_proj_dgrad", S, A, H, 0, 1, 0),
          ("qkv_dgrad", S, H, Q, 0, 1, 0), ("mlp_down_wgrad", H, F, S, 1, 1, 1),
          ("fc1_wgrad", F, H, S, 1, 1, 1), ("attn_proj_wgrad", H, A, S, 1, 1, 1),
          ("qkv_wgrad", Q, H, S, 1, 1, 1)]
caps = [int(c) for c in os.environ.get("CAPS", "132").split(",")]
tiles = [int(t) for t in os.environ.get("TILES", "0,128,192,256,512,-192,-128").split(",")]
out = []
for name, m, n, k, amn, bmn, f32 in shapes:
    a = torch.randn((k, m) if amn else (m, k), device="cuda", dtype=torch.bfloat16)
    b = torch.randn((k, n) if bmn else (n, k), device="cuda", dtype=torch.bfloat16)
    d = torch.zeros(m, n, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
    for cap in caps:
        row = dict(name=name, m=m, n=n, k=k, cap=cap)
        for tn in tiles:
            try:
                ms = timeit(lambda: dh.gemm(a, b, d, a_mn=bool(amn), b_mn=bool(bmn), m=m, n=n, k=k,
                                            accumulate=bool(f32), max_ctas=cap, tile_n=tn))
                row[f"t{tn}"] = round(2 * m * n * k / ms / 1e9, 1)
            except Exception as ex:  # noqa: BLE001
                row[f"t{tn}"] = str(ex)[:40]
        print(json.dumps(row), flush=True)
        out.append(row)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/gemm_tp8.json", "w"), indent=1)

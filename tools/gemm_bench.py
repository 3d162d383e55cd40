"""Time the tcgen05 GEMM on the layer's shapes (CUDA events, L2-flushed)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_15871_b200 import device as dh

flush = torch.empty(256 * 1024 * 1024, dtype=torch.int8, device="cuda")
def timeit(fn, iters=20):
    for _ in range(3): fn()
    ts = []
    for _ in range(iters):
        flush.zero_()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]

shapes = [("qkv_tp8", 4096, 768, 4096, 0, 0), ("attn_proj_tp8", 4096, 4096, 512, 0, 0),
          ("mlp_gate_tp8", 4096, 1792, 4096, 0, 0), ("mlp_down_tp8", 4096, 4096, 1792, 0, 0),
          ("dgrad_mlp_down", 4096, 1792, 4096, 0, 1), ("wgrad_fc1", 1792, 4096, 4096, 1, 1),
          ("square8k", 8192, 8192, 8192, 0, 0), ("mlp_gate_tp1", 4096, 14336, 4096, 0, 0),
          ("wgrad_tp1", 14336, 4096, 4096, 1, 1), ("wgrad_tp1_f32acc", 14336, 4096, 4096, 1, 1),
          ("wgrad_down_tp1_f32acc", 4096, 14336, 4096, 1, 1), ("wgrad_qkv_tp1_f32acc", 6144, 4096, 4096, 1, 1)]
out = []
for name, m, n, k, amn, bmn in shapes:
    a = torch.randn((k, m) if amn else (m, k), device="cuda", dtype=torch.bfloat16)
    b = torch.randn((k, n) if bmn else (n, k), device="cuda", dtype=torch.bfloat16)
    f32 = name.endswith("f32acc")  # the wgrad path: fp32 main-grad, TMA reduce-add
    d = torch.zeros(m, n, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
    for tn in ((0,) if f32 else (256, 512, 0)):
        ms = timeit(lambda: dh.gemm(a, b, d, a_mn=bool(amn), b_mn=bool(bmn), m=m, n=n, k=k, tile_n=tn,
                                    accumulate=f32))
        tf = 2 * m * n * k / ms / 1e9
        ref = None
        if amn == 0 and bmn == 0:
            ref = 2 * m * n * k / timeit(lambda: torch.matmul(a, b.t(), out=d)) / 1e9
        row = dict(name=name, m=m, n=n, k=k, tile_n=tn, ms=round(ms, 4), tflops=round(tf, 1),
                   cublas_tflops=None if ref is None else round(ref, 1))
        print(json.dumps(row), flush=True)
        out.append(row)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/gemm_bench.json", "w"), indent=1)

"""Time attention fwd/bwd at the layer's shapes (CUDA events)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_15871_b200 import device as dh

def timeit(fn, iters=10):
    for _ in range(2): fn()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters

out = []
for T, nq, nkv, d in [(4096, 4, 1, 128), (4096, 8, 2, 128), (4096, 16, 4, 128), (4096, 32, 8, 128), (2048, 10, 10, 128)]:
    qkv = (torch.randn(T, (nq + 2 * nkv) * d, device="cuda") * 0.5).to(torch.bfloat16)
    q, k, v = qkv[:, :nq * d], qkv[:, nq * d:(nq + nkv) * d], qkv[:, (nq + nkv) * d:]
    o = torch.empty(T, nq * d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(nq, T, device="cuda")
    do = torch.randn_like(o)
    dqkv = torch.empty_like(qkv)
    scratch = torch.empty(dh.attn_bwd_scratch_floats(T, nq, nkv, d), device="cuda")
    f = timeit(lambda: dh.attn_fwd(q, k, v, o, lse, nq, nkv, d, d ** -0.5))
    f_nosplit = timeit(lambda: dh.attn_fwd(q, k, v, o, lse, nq, nkv, d, d ** -0.5, split=False))
    b = timeit(lambda: dh.attn_bwd(q, k, v, o, lse, do, dqkv[:, :nq * d], dqkv[:, nq * d:(nq + nkv) * d],
                                   dqkv[:, (nq + nkv) * d:], nq, nkv, d, d ** -0.5, scratch=scratch))
    flops = 2 * T * T * nq * d  # causal fwd: 4*T^2/2*nq*d
    row = dict(T=T, nq=nq, nkv=nkv, d=d, fwd_ms=round(f, 4), fwd_ms_nosplit=round(f_nosplit, 4), bwd_ms=round(b, 4),
               fwd_tflops=round(flops / f / 1e9, 1), bwd_tflops=round(2.5 * flops / b / 1e9, 1))
    print(json.dumps(row), flush=True)
    out.append(row)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/attn_bench.json", "w"), indent=1)

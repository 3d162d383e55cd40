"""Device times of the HBM-bound layer kernels at the TP=8 (512-row SP shard)
and TP=1 (4096-row) Llama-3-8B shapes: each kernel captured 20x in a CUDA
graph (no host launch cost), replayed warm; microseconds per launch."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_15871_b200 import device as dh


def timeit(fn, n=20, reps=10):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        fn()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            for _ in range(n):
                fn()
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(reps):
        gr.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / (n * reps) * 1e3


H = 4096
for rows in (512, 4096):
    bf = dict(device="cuda", dtype=torch.bfloat16)
    x, dy, resid, xo = (torch.randn(rows, H, **bf) for _ in range(4))
    g = torch.ones(H, **bf)
    y, dx = torch.empty(rows, H, **bf), torch.empty(rows, H, **bf)
    rstd = torch.empty(rows, device="cuda")
    dg = torch.zeros(H, device="cuda")
    part = torch.empty(min(rows, 1184) * H, device="cuda")
    dh.rmsnorm_fwd(x, g, y, rstd)
    mb = rows * H * 2 / 1e6
    cur = lambda: torch.cuda.current_stream()  # noqa: E731
    res = {"rows": rows,
           "rmsnorm_fwd": timeit(lambda: dh.rmsnorm_fwd(x, g, y, rstd, stream=cur())),
           "add_rmsnorm_fwd": timeit(lambda: dh.add_rmsnorm_fwd(x, resid, xo, g, y, rstd, stream=cur())),
           "add": timeit(lambda: dh.add(x, resid, y, stream=cur())),
           "rmsnorm_bwd": timeit(lambda: dh.rmsnorm_bwd(x, g, rstd, dy, dx, dgamma_acc=dg, partial=part,
                                                        resid=resid, stream=cur()))}
    nbytes = {"rmsnorm_fwd": 2 * mb, "add_rmsnorm_fwd": 4 * mb, "add": 3 * mb, "rmsnorm_bwd": 4 * mb}
    out = {"rows": rows}
    for k, b in nbytes.items():
        out[k] = {"us": round(res[k], 2), "GBs": round(b * 1e3 / res[k])}
    print(json.dumps(out), flush=True)

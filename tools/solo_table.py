"""Per-node solo times (the G4 profiler's solo table) of one Llama-3-8B-shaped
layer at a given TP (emulated collectives for TP > 1), sorted, with each
GEMM/attention node's achieved TF/s: where a layer pair's time goes."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_15871_b200.runtime import LLAMA3_8B, Context, LlamaShape, Model  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tp", type=int, default=1)
ap.add_argument("--cap", type=int, default=0, help="GEMM SM cap while profiling (0 = all SMs)")
a = ap.parse_args()
shape = LlamaShape(**{**LLAMA3_8B.__dict__, "layers": 2, "micro_batches": 2})
ctx = Context.emulated(0, a.tp, 16, 770.0) if a.tp > 1 else Context.create(0)
m = Model(ctx, shape)
m.set_overlap_ctas(a.cap)
prof = json.loads(m.profile(iters=10))
S, H, F, D, tp = shape.seq_len, shape.hidden, shape.ffn // a.tp, shape.head_dim, a.tp
nq, nkv = shape.n_heads // tp, shape.n_kv_heads // tp
Q, A = (nq + 2 * nkv) * D, nq * D
g = lambda m_, n, k: 2.0 * m_ * n * k  # noqa: E731
attn = 2.0 * S * S * D * nq
flops = {"qkv": g(S, Q, H), "attn": attn, "attn_proj": g(S, H, A), "mlp_gate": g(S, F, H), "mlp_up": g(S, F, H),
         "mlp_down": g(S, H, F), "mlp_down_dgrad": g(S, F, H), "mlp_down_wgrad": g(H, F, S),
         "mlp_gate_dgrad": g(S, H, F), "mlp_up_dgrad": g(S, H, F), "mlp_fc1_wgrad": 2 * g(F, H, S),
         "attn_proj_dgrad": g(S, A, H), "attn_proj_wgrad": g(H, A, S), "attn_bwd": 2.5 * attn,
         "qkv_dgrad": g(S, H, Q), "qkv_wgrad": g(Q, H, S)}
rows = sorted(prof["solo"], key=lambda e: -e["t_us"])
tot = sum(e["t_us"] for e in rows)
out = []
for e in rows:
    f = flops.get(e["shape"])
    tf = f / e["t_us"] / 1e6 if f else None
    out.append({"node": e["shape"], "class": e["class"], "us": round(e["t_us"], 1),
                "tflops": None if tf is None else round(tf, 1)})
    print(f"{e['shape']:18s} {e['class']:18s} {e['t_us']:8.1f} us" + (f"  {tf:7.1f} TF/s" if tf else ""))
print(f"total {tot:.1f} us")
json.dump({"tp": a.tp, "cap": a.cap, "nodes": out, "total_us": round(tot, 1)},
          open(os.path.join("gpurun_out", f"solo_table_tp{a.tp}.json"), "w"), indent=1)

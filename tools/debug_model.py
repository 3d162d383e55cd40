import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_15871_b200.runtime import Context, Model, TINY, LlamaShape
from paper_2411_15871_b200 import planner
variant = sys.argv[1]
if variant == "torch_first":
    torch.zeros(1, device="cuda")
ctx = Context.create(0)
shape = LlamaShape(hidden=256, ffn=768, n_heads=4, n_kv_heads=2, head_dim=64, layers=4, seq_len=128, micro_batches=2, rope_theta=10000.0)
m = Model(ctx, shape)
if variant == "touch":
    t = m.tensor("w.wqkv", 0); t.copy_(torch.zeros_like(t)); torch.cuda.synchronize()
if variant == "plan":
    B200 = {"name": "b200_8", "gpus": 8, "per_node": 8, "peak_tflops": 2250.0, "local_bw_gbs": 900.0, "cross_bw_gbs": 50.0, "mem_gb": 180.0}
    r = planner.lib().search_si_plan(shape.planner_model(), {"tp": 1, "sp": False}, B200, {"archetype": "nvlink_h100"})
    print(r["plan_json"])
    m.set_plan(r["plan_json"], mode="si")
else:
    m.set_plan(None, mode="si")
m.zero_grads(); m.run_program(); m.sync()
print(variant, "loss", m.tensor("loss").cpu())

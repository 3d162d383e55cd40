"""Run a few training steps of the Llama-3-8B-shaped stack (for ncu launch lists)."""
import argparse, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_15871_b200 import planner
from paper_2411_15871_b200.runtime import LLAMA3_8B, Context, Model

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=2)
ap.add_argument("--mb", type=int, default=2)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--graph", type=int, default=0)
ap.add_argument("--mode", default="si")
ap.add_argument("--emulate-tp", type=int, default=0)
args = ap.parse_args()
shape = LLAMA3_8B
shape.layers, shape.micro_batches = args.layers, args.mb
ctx = Context.emulated(0, args.emulate_tp, 16, 770.0) if args.emulate_tp > 1 else Context.create(0)
tp = max(1, args.emulate_tp)
m = Model(ctx, shape)
cl = {"name": "b200_8", "gpus": 8, "per_node": 8, "peak_tflops": 2250.0, "local_bw_gbs": 900.0, "cross_bw_gbs": 50.0, "mem_gb": 180.0}
plan = planner.lib().search_si_plan(shape.planner_model(), {"tp": tp, "sp": tp > 1}, cl, {"archetype": "nvlink_h100"})["plan_json"]
m.set_plan(plan, mode=args.mode)
if tp > 1:
    m.set_overlap_ctas(148 - 16)
for _ in range(args.steps):
    m.step({"lr": 1e-5}, use_graph=bool(args.graph))
m.sync()
print("done", m.info()["program"]["ops"])

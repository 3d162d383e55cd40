"""Where a compute-only training step's time goes at TP=<tp> per-GPU shapes
(emulated collectives, left out of the program): the graph-replayed step time
against the sum of its kernels' durations and against the graph-replayed solo
table. Run plain for the step times; run under
  ncu --profile-from-start off --cache-control none --clock-control none \
      --metrics gpu__time_duration.sum --csv --log-file L python tools/step_kernels.py --ncu MODE
for the in-step per-kernel durations of one step of MODE (caches as the step
leaves them; ncu serialises the kernels, so their sum excludes concurrency).
Writes gpurun_out/step_kernels_tp<tp>.json."""
import argparse
import copy
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_15871_b200 import planner  # noqa: E402
from paper_2411_15871_b200.runtime import LLAMA3_8B, Context, Model  # noqa: E402
from tests.planner_corpus import B200_CLUSTER  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tp", type=int, default=8)
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--mb", type=int, default=4)
ap.add_argument("--ncu", default="", help="executor mode whose one step is captured (sequential | si_relaxed)")
a = ap.parse_args()

shape = copy.copy(LLAMA3_8B)
shape.layers, shape.micro_batches, shape.slots = a.layers, a.mb, a.layers + 2
ctx = Context.emulated(0, a.tp, 16, 770.0)
m = Model(ctx, shape)
m.set_overlap_ctas(132)
prof = json.loads(m.profile(iters=3))
plan = planner.lib().search_si_plan(shape.planner_model(), {"tp": a.tp, "sp": True}, B200_CLUSTER, prof,
                                    caps=bench.WIDE_CAPS, parallel=True)["plan_json"]
stream = torch.cuda.ExternalStream(ctx.stream_ptr(0))
step = lambda: m.step({"lr": 0.0}, use_graph=True)  # noqa: E731


def timed(n):
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(n):
        step()
    e.record(stream)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


out = {"tp": a.tp, "layers": a.layers, "micro_batches": a.mb,
       "solo_compute_us_per_layer_pair": round(sum(e["t_us"] for e in prof["solo"]
                                                   if e["class"] not in ("AllGather", "ReduceScatter")), 1)}
modes = [a.ncu] if a.ncu else ["sequential", "si_relaxed"]
for mode in modes:
    m.set_plan(plan, json.dumps(prof), mode=mode)
    m.set_overlap_ctas(0)
    m.set_skip_comm(True)
    for _ in range(3):
        step()
    if a.ncu:
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        step()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        continue
    ms = sorted(timed(5) for _ in range(3))[1]
    out[f"{mode}_compute_only_ms"] = round(ms, 3)
    out[f"{mode}_us_per_layer_pair"] = round(ms * 1e3 / (a.layers * a.mb), 1)
print(json.dumps(out))
if not a.ncu:
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", f"step_kernels_tp{a.tp}.json"), "w"), indent=1)

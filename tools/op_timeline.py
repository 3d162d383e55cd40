"""On-device timeline of one SI training step (eager issue, CUDA events around
every op: DH_OP_TIMES) at TP=<tp> per-GPU shapes with emulated collectives.
Also writes a Chrome trace (lanes as rows). Reports where the compute lane idles and which collectives are exposed
(collective running while the compute lane is idle), split by what the idle
compute op was waiting for. Writes gpurun_out/op_timeline_tp<tp>.json."""
import argparse
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2411_15871_b200 import planner  # noqa: E402
from paper_2411_15871_b200.runtime import LLAMA3_8B, Context, LlamaShape, Model, lower  # noqa: E402
from tests.planner_corpus import B200_CLUSTER  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tp", type=int, default=8)
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--mb", type=int, default=4)
ap.add_argument("--mode", default="si")
ap.add_argument("--wide", action="store_true", help="the bench's wide search caps (si_wide* variants)")
a = ap.parse_args()
shape = LlamaShape(**{**LLAMA3_8B.__dict__, "layers": a.layers, "micro_batches": a.mb, "slots": a.layers + 2})
ctx = Context.emulated(0, a.tp, 16, 770.0) if a.tp > 1 else Context.create(0)
m = Model(ctx, shape)
m.set_overlap_ctas(148 - 16)
prof = json.loads(m.profile(iters=5))
caps = ({"sequences": 64, "segments": 14, "candidates": 1000000} if a.wide
        else {"sequences": 16, "segments": 14, "candidates": 200000})
plan = planner.lib().search_si_plan(shape.planner_model(), {"tp": a.tp, "sp": a.tp > 1}, B200_CLUSTER, prof,
                                    caps=caps, parallel=True)["plan_json"]
m.set_plan(plan, json.dumps(prof), mode=a.mode)
m.set_overlap_ctas(148 - 16)
for _ in range(2):
    m.run_program(use_graph=False)
m.sync()
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
path = os.path.join(ROOT, "gpurun_out", "op_times.jsonl")
os.environ["DH_OP_TIMES"] = path
m.run_program(use_graph=False)
m.sync()
del os.environ["DH_OP_TIMES"]
ops = [json.loads(line) for line in open(path)]
prog = lower(shape, a.tp, plan, a.mode, profile_json=json.dumps(prof))["ops"]
assert len(prog) == len(ops)
names = {n["id"]: n["name"] for d in planner.lib().build_layer_dag(shape.planner_model(), {"tp": a.tp, "sp": a.tp > 1},
                                                                   B200_CLUSTER, profile=prof) for n in d["nodes"]}
names[100] = "adamw"


def busy(lane):
    iv = sorted((o["start_ms"], o["end_ms"]) for o in ops if o["lane"] == lane)
    merged = []
    for s, e in iv:
        if merged and s <= merged[-1][1]:
            merged[-1][1] = max(merged[-1][1], e)
        else:
            merged.append([s, e])
    return merged


def overlap(a_iv, b_iv):
    t, i, j = 0.0, 0, 0
    while i < len(a_iv) and j < len(b_iv):
        lo, hi = max(a_iv[i][0], b_iv[j][0]), min(a_iv[i][1], b_iv[j][1])
        t += max(0.0, hi - lo)
        if a_iv[i][1] < b_iv[j][1]:
            i += 1
        else:
            j += 1
    return t


end = max(o["end_ms"] for o in ops)
comp, comm = busy(0), busy(1)
comp_busy = sum(e - s for s, e in comp)
comm_busy = sum(e - s for s, e in comm)
hidden = overlap(comp, comm)
# compute-lane idle gaps, attributed to the op that ends each gap and what it waited on
gaps = collections.Counter()
gap_n = collections.Counter()
steady = collections.Counter()  # gaps before ops of the paired middle (not F_0 / B_last)


def at_end(o):
    fwd = o["node"] < 20
    return (fwd and o["strand"] == 0) or (not fwd and o["node"] != 100 and o["strand"] == a.mb - 1)


comp_ops = sorted((o for o in ops if o["lane"] == 0), key=lambda o: o["start_ms"])
prev_end = 0.0
for o in comp_ops:
    g = o["start_ms"] - prev_end
    if g > 0.002:
        w = prog[o["op"]]["waits"]
        why = "+".join(sorted({names.get(ops[x]["node"], str(ops[x]["node"])) for x in w})) or "launch/stream"
        key = f"{names.get(o['node'], o['node'])} <- {why}"
        gaps[key] += g
        gap_n[key] += 1
        if not at_end(o):
            steady[key] += g
    prev_end = max(prev_end, o["end_ms"])
res = {"tp": a.tp, "layers": a.layers, "micro_batches": a.mb, "mode": a.mode, "step_ms": round(end, 3),
       "compute_busy_ms": round(comp_busy, 3), "compute_idle_ms": round(end - comp_busy, 3),
       "comm_busy_ms": round(comm_busy, 3), "comm_hidden_ms": round(hidden, 3),
       "comm_exposed_ms": round(comm_busy - hidden, 3),
       "top_compute_gaps": [{"gap": k, "ms": round(v, 3), "count": gap_n[k]} for k, v in gaps.most_common(15)],
       "steady_gaps_ms": round(sum(steady.values()), 3),
       "top_steady_gaps": [{"gap": k, "ms": round(v, 3)} for k, v in steady.most_common(10)]}
print(json.dumps(res, indent=1))
json.dump({"summary": res, "ops": ops}, open(os.path.join(ROOT, "gpurun_out", f"op_timeline_tp{a.tp}.json"), "w"))
# Chrome trace (chrome://tracing, Perfetto): one row per lane, an event per op
lane_names = {0: "compute", 1: "local_comm", 2: "cross_comm"}
events = [{"name": "process_name", "ph": "M", "pid": 0, "args": {"name": f"SI step, TP={a.tp} ({a.mode})"}}]
events += [{"name": "thread_name", "ph": "M", "pid": 0, "tid": l, "args": {"name": n}} for l, n in lane_names.items()]
for o in ops:
    events.append({"name": names.get(o["node"], str(o["node"])), "ph": "X", "pid": 0, "tid": o["lane"],
                   "ts": o["start_ms"] * 1e3, "dur": max(0.0, (o["end_ms"] - o["start_ms"]) * 1e3),
                   "args": {"strand": o["strand"], "layer": o["layer"], "capped": o["capped"]}})
json.dump({"traceEvents": events}, open(os.path.join(ROOT, "gpurun_out", f"op_timeline_tp{a.tp}_{a.mode}.trace.json"),
                                        "w"))

"""GPU: the on-device overlap profiler emits a weft Profile the planner accepts;
with an emulated TP group the cross-lane class pairs are all measured and the
plan searched from the measured table runs through the SI executor."""
import json

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2411_15871_b200 import planner  # noqa: E402
from paper_2411_15871_b200.runtime import Context, Model  # noqa: E402
from tests.test_model_gpu import B200, _tiny  # noqa: E402


def test_profile_tp1_solo_table():
    ctx = Context.create(0)
    shape = _tiny(mb=2, layers=2)
    m = Model(ctx, shape)
    prof = json.loads(m.profile(iters=3))
    names = {e["shape"] for e in prof["solo"]}
    assert {"ln0", "qkv", "attn", "mlp_down", "attn_bwd", "qkv_wgrad", "ln0_bwd"} <= names
    assert all(e["t_us"] > 0 for e in prof["solo"])
    assert prof["oef"] == []  # tp=1: no communication lane, nothing co-runs
    assert prof["interference"] == {"launch_overhead_frac": 0.0, "slowdown_factor": 0.0}
    # the solo table is device time of graph-replayed launches, as the executor runs them
    assert prof["metadata"]["solo_timing"] == "graph"
    # the planner consumes it unchanged; durations now come from the measurement
    fwd, bwd = planner.lib().build_layer_dag(shape.planner_model(), {"tp": 1}, B200, profile=prof)
    measured = {e["shape"]: e["t_us"] for e in prof["solo"]}
    assert all(n["duration_us"] == measured[n["name"]] for n in fwd["nodes"] + bwd["nodes"])
    m.close()
    ctx.close()


def test_profile_emulated_tp_pairs_and_plan():
    ctx = Context.emulated(0, tp_size=4, comm_ctas=16, link_gbs=770.0)
    shape = _tiny(mb=2, layers=2, nkv=4)
    m = Model(ctx, shape)
    prof = json.loads(m.profile(iters=3))
    pairs = {frozenset((e["a"], e["b"])) for e in prof["oef"]}
    comp = {"GEMM", "FlashAttention", "FlashAttentionBwd", "FusedBDA", "LayerNorm", "WeightGrad"}
    for c in comp:
        for comm in ("AllGather", "ReduceScatter"):
            assert frozenset((c, comm)) in pairs, (c, comm)
    assert all(-0.05 <= e["value"] <= 1.05 for e in prof["oef"])
    r = planner.lib().search_si_plan(shape.planner_model(), {"tp": 4, "sp": True}, B200, prof)
    m.set_plan(r["plan_json"], json.dumps(prof), mode="si")
    m.zero_grads()
    m.step(None, use_graph=True)
    m.sync()
    assert m.info()["program"]["comm"] == "emulated"
    m.close()
    ctx.close()

"""GPU, BASELINE.json full sizes: size-independent properties on the real
layer shapes (the small-shape tests pin the numerics against the oracle).

  * config 2 layers (Llama-3-8B-shaped, seq 4096) at TP = 1: SI == sequential ==
    CUDA-graph replay, bit for bit, and the losses, output, input gradient and
    every weight gradient within the bf16 tolerance of the numpy oracle on the
    same weights and inputs;
  * config 2 at TP = 8 per-GPU shapes and config 4 (Phi-3.5-MoE, EP = 8) with
    emulated collectives: every executor mode gives bitwise the same losses and
    gradients (the emulated collectives are deterministic, not numerically
    collectives, so this checks the executor's ordering at full size).
"""
import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.layer_oracle import LlamaTPOracle, bf16_round  # noqa: E402
from paper_2411_15871_b200 import planner  # noqa: E402
from paper_2411_15871_b200.runtime import LLAMA3_8B, PHI35_MOE, Context, LlamaShape, Model  # noqa: E402
from tests.test_model_gpu import B200, _rel, _upload  # noqa: E402


def _grads_equal(a, b, names, layers):
    for l in range(layers):
        for n in names:
            assert torch.equal(a.tensor("grad." + n, l), b[(l, n)]), f"grad.{n} layer {l}"


def _run_modes(m, shape, plan, prof, modes, names):
    ref = None
    for mode, graph in modes:
        m.set_plan(plan, prof, mode=mode)
        m.zero_grads()
        m.run_program(use_graph=graph)
        m.sync()
        snap = {"loss": m.tensor("loss").clone(), "dx": m.tensor("dx").clone()}
        snap.update({(l, n): m.tensor("grad." + n, l).clone() for l in range(shape.layers) for n in names})
        if ref is None:
            ref = snap
            continue
        assert torch.equal(ref["loss"], snap["loss"]), (mode, ref["loss"], snap["loss"])
        assert torch.equal(ref["dx"], snap["dx"]), mode
        for k in ref:
            if isinstance(k, tuple):
                assert torch.equal(ref[k], snap[k]), (mode, k)
    return ref


def test_llama3_8b_tp1_full_size_si_equals_sequential_and_oracle():
    """Config-2 layer shapes at seq 4096 (TP = 1, 2 layers, 2 micro-batches):
    SI == sequential == relaxed SI bitwise, and against the numpy oracle on the
    same weights and inputs: both strands' losses, the last strand's output and
    input gradient, and every weight gradient of both layers (summed over the
    two strands, as the device accumulates them)."""
    shape = LlamaShape(**{**LLAMA3_8B.__dict__, "layers": 2, "micro_batches": 2})
    ctx = Context.create(0)
    m = Model(ctx, shape)
    orc = LlamaTPOracle(shape.hidden, shape.ffn, shape.n_heads, shape.n_kv_heads, shape.head_dim, shape.layers,
                        shape.seq_len, tp=1, theta=shape.rope_theta, bf16=True, seed=31, init_std=0.02)
    for l in range(shape.layers):
        for name, arr in orc.shard(l, 0).items():
            _upload(m.tensor("w." + name, l), arr)
    rng = np.random.default_rng(5)
    xs = [bf16_round(rng.standard_normal((shape.seq_len, shape.hidden)).astype(np.float32)) for _ in range(2)]
    rs = [bf16_round(rng.standard_normal((shape.seq_len, shape.hidden)).astype(np.float32)) for _ in range(2)]
    for s in range(2):
        _upload(m.tensor("x_in", strand=s), xs[s])
        _upload(m.tensor("dy", strand=s), rs[s])
    torch.cuda.synchronize()
    plan = planner.lib().search_si_plan(shape.planner_model(), {"tp": 1}, B200, {"archetype": "nvlink_h100"})["plan_json"]
    names = ("wqkv", "wo", "wg", "wu", "wd", "g0", "g1")
    ref = _run_modes(m, shape, plan, None, [("sequential", False), ("si_relaxed", True), ("si", True)], names)
    y_dev = m.tensor("y", strand=1).float().cpu().numpy().reshape(shape.seq_len, shape.hidden)
    m.close()
    ctx.close()
    # both strands through the oracle: same weights, same inputs, same gate/up order
    p = planner.parse_plan(plan)
    first_gate = p["bwd_seq"].index(24) < p["bwd_seq"].index(25)
    grads = orc.zero_grads()
    out = []
    for s in range(2):
        loss, y, dx, grads = orc.run(xs[s], rs[s], grads, dx_first_gate=first_gate)
        out.append((loss, y, dx))
    for s in range(2):
        tol = 2e-2 * float(np.sqrt(np.sum((out[s][1] * rs[s]) ** 2)))
        assert abs(float(ref["loss"][s]) - out[s][0]) < tol, (s, float(ref["loss"][s]), out[s][0], tol)
    # bf16 tolerances (relative Frobenius error): activations / gradients 3e-2
    assert _rel(y_dev, out[1][1]) < 3e-2
    assert _rel(ref["dx"].float().cpu().numpy().reshape(shape.seq_len, shape.hidden), out[1][2]) < 3e-2
    for l in range(shape.layers):
        g = grads[l]
        want = {"wqkv": np.concatenate([g["wq"], g["wk"], g["wv"]], 0), "wo": g["wo"], "wg": g["wg"],
                "wu": g["wu"], "wd": g["wd"], "g0": g["g0"], "g1": g["g1"]}
        for n, arr in want.items():
            err = _rel(ref[(l, n)].cpu().numpy(), np.ascontiguousarray(arr).reshape(-1))
            assert err < 3e-2, (l, n, err)


def _emulated_modes(shape, group, par, names):
    ctx = Context.emulated(0, group, 16, 770.0)
    m = Model(ctx, shape)
    m.set_overlap_ctas(148 - 16)
    prof = json.loads(m.profile(iters=2))
    plan = planner.lib().search_si_plan(shape.planner_model(), par, B200, prof)["plan_json"]
    _run_modes(m, shape, plan, json.dumps(prof),
               [("si", True), ("sequential", True), ("si_relaxed", True), ("si_deferred", True), ("si", False)],
               names)
    m.close()
    ctx.close()


def test_llama3_8b_tp8_shapes_all_modes_bitwise():
    shape = LlamaShape(**{**LLAMA3_8B.__dict__, "layers": 3, "micro_batches": 3, "slots": 5})
    _emulated_modes(shape, 8, {"tp": 8, "sp": True}, ("wqkv", "wo", "wg", "wu", "wd", "g0", "g1"))


def test_phi35_moe_ep8_shapes_all_modes_bitwise():
    shape = LlamaShape(**{**PHI35_MOE.__dict__, "layers": 2, "micro_batches": 3, "slots": 4})
    _emulated_modes(shape, 8, {"tp": 1, "ep": 8, "dp": 8}, ("wqkv", "wo", "wr", "w1g", "w1u", "w2", "g0", "g1"))

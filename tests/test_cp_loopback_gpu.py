"""GPU, single device: context parallelism (reference
cp_kv_exchange / cp_kv_exchange_bwd nodes, op_model.cpp:83,108, cost
:297-301). A CP group of `cp` ranks runs as host threads over the loopback
communicator; each rank holds seq/cp consecutive tokens, all-gathers the
layer's K/V (cp_kv_exchange) for causal attention at its global offset,
re-gathers them before attn_bwd (cp_kv_exchange_bwd) and reduce-scatters the
dK/dV partials back to their owners.

Checked against the numpy oracle on the FULL sequence (the CP ranks together
must reproduce the unpartitioned layer stack): per-rank loss shards sum to the
full loss, the concatenated input gradient and the CP-summed weight gradients
match within bf16 tolerance; SI == sequential bit for bit on every rank."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.layer_oracle import LlamaTPOracle, bf16_round  # noqa: E402
from paper_2411_15871_b200 import planner  # noqa: E402
from paper_2411_15871_b200.runtime import Context, LlamaShape, Model  # noqa: E402
from tests.test_model_gpu import _rel, _upload  # noqa: E402
from tests.test_tp_loopback_gpu import _run_ranks  # noqa: E402

NAMES = ("wqkv", "wo", "wg", "wu", "wd", "g0", "g1")


@pytest.mark.parametrize("cp,d", [(2, 128), (4, 64)])
def test_cp_loopback_vs_full_sequence_oracle(cp, d):
    heads = 512 // d
    shape = LlamaShape(hidden=512, ffn=1024, n_heads=heads, n_kv_heads=heads // 2, head_dim=d, layers=2,
                       seq_len=256 * cp, micro_batches=2, rope_theta=500000.0, slots=4, context_parallel=1)
    S, H, T = shape.seq_len, shape.hidden, shape.seq_len // cp
    orc = LlamaTPOracle(H, shape.ffn, shape.n_heads, shape.n_kv_heads, d, shape.layers, S, tp=1,
                        theta=shape.rope_theta, bf16=True, seed=17, init_std=0.05)
    rng = np.random.default_rng(9)
    xs = [bf16_round(rng.standard_normal((S, H)).astype(np.float32)) for _ in range(2)]
    rs = [bf16_round(rng.standard_normal((S, H)).astype(np.float32)) for _ in range(2)]
    cluster = {"name": "b200_8", "gpus": 8, "per_node": 8, "peak_tflops": 2250.0, "local_bw_gbs": 900.0,
               "cross_bw_gbs": 50.0, "mem_gb": 180.0}
    plan = planner.lib().search_si_plan(shape.planner_model(), {"tp": 1, "cp": cp, "dp": 8 // cp}, cluster,
                                        {"archetype": "pcie_a40"})["plan_json"]
    p = planner.parse_plan(plan)
    assert 3 in p["fwd_seq"] and 33 in p["bwd_seq"], "cp_kv_exchange nodes in the plan"
    ctxs = Context.loopback_group(0, cp)

    def rank_main(r):
        torch.cuda.set_device(0)
        m = Model(ctxs[r], shape)
        for l in range(shape.layers):
            sh = orc.shard(l, 0)
            for n in NAMES:
                _upload(m.tensor("w." + n, l), sh[n])
        for s in range(2):
            _upload(m.tensor("x_in", strand=s), xs[s][r * T:(r + 1) * T])
            _upload(m.tensor("dy", strand=s), rs[s][r * T:(r + 1) * T])
        torch.cuda.synchronize()
        res = {}
        for mode in ("si", "sequential"):
            m.set_plan(plan, mode=mode)
            m.zero_grads()
            m.run_program(use_graph=True)
            m.sync()
            snap = {"loss": m.tensor("loss").cpu().clone(), "dx": m.tensor("dx").float().cpu().clone()}
            for l in range(shape.layers):
                for n in NAMES:
                    snap[f"{l}.{n}"] = m.tensor("grad." + n, l).cpu().clone()
            res[mode] = snap
        m.close()
        return res

    outs = _run_ranks(rank_main, cp)
    for c in ctxs:
        c.close()
    for r in range(cp):
        for k in outs[r]["si"]:
            assert torch.equal(outs[r]["si"][k], outs[r]["sequential"][k]), (r, k)
    first_gate = p["bwd_seq"].index(24) < p["bwd_seq"].index(25)
    grads = orc.zero_grads()
    dx = None
    for s in range(2):
        loss, y, dx, grads = orc.run(xs[s], rs[s], grads, dx_first_gate=first_gate)
        got = sum(float(outs[r]["si"]["loss"][s]) for r in range(cp))
        tol = 2e-2 * float(np.sqrt(np.sum((y * rs[s]) ** 2)))
        assert abs(got - loss) < tol, (s, got, loss)
    dx_got = np.concatenate([outs[r]["si"]["dx"].numpy().reshape(T, H) for r in range(cp)], 0)
    assert _rel(dx_got, dx) < 3e-2
    for l in range(shape.layers):
        g = grads[l]
        want = {"wqkv": np.concatenate([g["wq"], g["wk"], g["wv"]], 0), "wo": g["wo"], "wg": g["wg"],
                "wu": g["wu"], "wd": g["wd"], "g0": g["g0"], "g1": g["g1"]}
        for n, arr in want.items():
            tot = sum(outs[r]["si"][f"{l}.{n}"].numpy() for r in range(cp))
            err = _rel(tot, np.ascontiguousarray(arr).reshape(-1))
            assert err < 3e-2, (l, n, err)

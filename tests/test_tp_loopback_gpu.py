"""GPU, single device: TP=2 and TP=4 Megatron TP+SP numerics and the SI
executor's collective ordering, with tp ranks as host threads over the
loopback communicator (dh_loopback_group_create). Every rank's shards of the
loss, input gradient and weight gradients are checked against the TP oracle,
and SI (collectives of one strand overlapping the other strand's compute on
the comm lane) must equal sequential bit for bit on every rank."""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.layer_oracle import bf16_round  # noqa: E402
from paper_2411_15871_b200 import planner  # noqa: E402
from paper_2411_15871_b200.runtime import Context, LlamaShape, Model  # noqa: E402
from tests.test_model_gpu import B200, _rel, _tiny, _upload  # noqa: E402
from oracle.layer_oracle import LlamaTPOracle  # noqa: E402


def _run_ranks(fn, tp):
    errs = [None] * tp
    out = [None] * tp

    def body(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            errs[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(tp)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for e in errs:
        if e is not None:
            raise e
    return out


def _tp8_shape():
    """TP=8 (the north-star degree): 16 q / 8 kv heads, so every rank holds one
    kv head and two q heads, head_dim 128 (the tcgen05 attention kernels), seq
    512 (64 tokens per sequence-parallel shard)."""
    return LlamaShape(hidden=1024, ffn=2048, n_heads=16, n_kv_heads=8, head_dim=128, layers=2,
                      seq_len=512, micro_batches=2, rope_theta=500000.0, slots=4)


@pytest.mark.parametrize("tp,merge", [(2, None), (4, None), (8, None), (2, "1")])
def test_tp_loopback_vs_oracle_and_si_equals_sequential(tp, merge, monkeypatch):
    # merge="1": the merged MLP GEMMs (SwiGLU pair, K-concatenated dgrads), off by
    # default at TP > 1, also under tensor parallelism
    if merge is not None:
        monkeypatch.setenv("DH_MLP_MERGE", merge)
    # one spare activation slot: mode 4 (deferred weight gradients) needs L + 2
    shape = _tp8_shape() if tp == 8 else LlamaShape(**{**_tiny(mb=2, layers=2, nkv=4).__dict__, "slots": 4})
    orc = LlamaTPOracle(shape.hidden, shape.ffn, shape.n_heads, shape.n_kv_heads, shape.head_dim,
                        shape.layers, shape.seq_len, tp=tp, theta=shape.rope_theta, bf16=True, seed=21,
                        init_std=0.05)
    rng = np.random.default_rng(4)
    xs = [bf16_round(rng.standard_normal((shape.seq_len, shape.hidden)).astype(np.float32)) for _ in range(2)]
    rs = [bf16_round(rng.standard_normal((shape.seq_len, shape.hidden)).astype(np.float32)) for _ in range(2)]
    plan = planner.lib().search_si_plan(shape.planner_model(), {"tp": tp, "sp": True}, B200,
                                        {"archetype": "pcie_a40"})["plan_json"]
    ctxs = Context.loopback_group(0, tp)
    T = shape.seq_len // tp

    def rank_main(r):
        torch.cuda.set_device(0)
        m = Model(ctxs[r], shape)
        for l in range(shape.layers):
            sh = orc.shard(l, r)
            for name in ("wqkv", "wo", "wg", "wu", "wd", "g0", "g1"):
                _upload(m.tensor("w." + name, l), sh[name])
        for s in range(2):
            _upload(m.tensor("x_in", strand=s), xs[s][r * T:(r + 1) * T])
            _upload(m.tensor("dy", strand=s), rs[s][r * T:(r + 1) * T])
        torch.cuda.synchronize()
        res = {}
        for mode in ("si", "sequential", "si_relaxed", "si_deferred"):
            m.set_plan(plan, mode=mode)
            m.zero_grads()
            m.run_program(use_graph=True)  # loopback is not capturable: runs eagerly
            m.sync()
            snap = {"loss": m.tensor("loss").cpu().clone(), "dx": m.tensor("dx").float().cpu().clone()}
            for l in range(shape.layers):
                for name in ("wqkv", "wo", "wg", "wu", "wd", "g0", "g1"):
                    snap[f"{l}.{name}"] = m.tensor("grad." + name, l).cpu().clone()
            res[mode] = snap
        info = m.info()
        m.close()
        return res, info

    outs = _run_ranks(rank_main, tp)
    for c in ctxs:
        c.close()
    for r in range(tp):
        si, seq, dfr = outs[r][0]["si"], outs[r][0]["sequential"], outs[r][0]["si_deferred"]
        for k in si:
            assert torch.equal(si[k], seq[k]), f"rank {r}: SI != sequential for {k}"
            assert torch.equal(si[k], dfr[k]), f"rank {r}: SI with deferred wgrads != SI for {k}"
            assert torch.equal(si[k], outs[r][0]["si_relaxed"][k]), f"rank {r}: relaxed SI != SI for {k}"
        assert outs[r][1]["program"]["comm"] == "loopback"

    p = planner.parse_plan(plan)
    first_gate = p["bwd_seq"].index(24) < p["bwd_seq"].index(25)
    grads = orc.zero_grads()
    losses, ys, dx = [], [], None
    for s in range(2):
        loss, y, dx, grads = orc.run(xs[s], rs[s], grads, dx_first_gate=first_gate)
        losses.append(loss)
        ys.append(y)
    for s in range(2):
        got = sum(float(outs[r][0]["si"]["loss"][s]) for r in range(tp))
        tol = 2e-2 * float(np.sqrt(np.sum((ys[s] * rs[s]) ** 2)))
        assert abs(got - losses[s]) < tol, (got, losses[s])
    dx_got = np.concatenate([outs[r][0]["si"]["dx"].numpy().reshape(T, -1) for r in range(tp)], 0)
    assert _rel(dx_got, dx) < 3e-2
    D, nq_l, nkv_l, F_l = shape.head_dim, shape.n_heads // tp, shape.n_kv_heads // tp, shape.ffn // tp
    for l in range(shape.layers):
        g = grads[l]
        for r in range(tp):
            q = g["wq"][r * nq_l * D:(r + 1) * nq_l * D]
            k = g["wk"][r * nkv_l * D:(r + 1) * nkv_l * D]
            v = g["wv"][r * nkv_l * D:(r + 1) * nkv_l * D]
            ref = {"wqkv": np.concatenate([q, k, v], 0),
                   "wo": g["wo"][:, r * nq_l * D:(r + 1) * nq_l * D],
                   "wg": g["wg"][r * F_l:(r + 1) * F_l], "wu": g["wu"][r * F_l:(r + 1) * F_l],
                   "wd": g["wd"][:, r * F_l:(r + 1) * F_l]}
            for name, arr in ref.items():
                err = _rel(outs[r][0]["si"][f"{l}.{name}"].numpy(), np.ascontiguousarray(arr).reshape(-1))
                assert err < 3e-2, (tp, r, l, name, err)
        for name in ("g0", "g1"):  # sequence-parallel: gamma grads are per-rank partial sums
            tot = sum(outs[r][0]["si"][f"{l}.{name}"].numpy() for r in range(tp))
            assert _rel(tot, g[name]) < 3e-2

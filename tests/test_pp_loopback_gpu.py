"""GPU, single device: the W-shaped pipeline (weft schedule_w_pipeline with
p = 2, U-folded layers, SI visits pairing the forward of micro-batch i with
the backward of micro-batch i - p) executed by two stage contexts as host
threads, their activation / gradient transfers staged through the loopback
stage group (dh_loopback_pp_group_create).

Every layer sees its micro-batches' backward in the same order as the
single-stage program, so the stages' losses, weight gradients and input
gradient must equal the single-stage stack bit for bit."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2411_15871_b200 import planner  # noqa: E402
from paper_2411_15871_b200.runtime import Context  # noqa: E402
from tests.test_model_gpu import B200, _build, _tiny  # noqa: E402
from tests.test_tp_loopback_gpu import _run_ranks  # noqa: E402

NAMES = ("wqkv", "wo", "wg", "wu", "wd", "g0", "g1")


def _fold(layers, p):
    """Global layer of each stage's local layer (weft fold_layers)."""
    c = layers // (2 * p)
    out = []
    for d in range(p):
        front = list(range(d * c, (d + 1) * c))
        back = list(range(layers - (d + 1) * c, layers - d * c))
        out.append(front + back)
    return out


@pytest.mark.parametrize("p,layers,mb", [(2, 4, 4), (2, 8, 3), (3, 6, 5)])
def test_w_pipeline_stages_equal_single_stage(p, layers, mb):
    from paper_2411_15871_b200.runtime import LlamaShape, Model
    shape = _tiny(mb=mb, layers=layers)
    plan = planner.lib().search_si_plan(shape.planner_model(), {"tp": 1}, B200, {"archetype": "nvlink_h100"})["plan_json"]
    # single-stage reference (the SI executor over the whole stack)
    ref_ctx = Context.create(0)
    _, ref, xs, rs = _build(shape, ref_ctx)
    ref.set_plan(plan, mode="sequential")
    ref.zero_grads()
    ref.run_program(use_graph=True)
    ref.sync()
    fold = _fold(layers, p)
    c = layers // (2 * p)
    ref_w = {(g, n): ref.tensor("w." + n, g).clone() for g in range(layers) for n in NAMES}
    ref_x = [ref.tensor("x_in", strand=s).clone() for s in range(mb)]
    ref_dy = [ref.tensor("dy", strand=s).clone() for s in range(mb)]
    want = {"loss": ref.tensor("loss").cpu().clone(), "dx": ref.tensor("dx").float().cpu().clone()}
    for g in range(layers):
        for n in NAMES:
            want[(g, n)] = ref.tensor("grad." + n, g).cpu().clone()
    ref.close()
    ref_ctx.close()

    ctxs = Context.loopback_pp_group(0, p)

    def stage_main(d):
        torch.cuda.set_device(0)
        st = LlamaShape(**{**shape.__dict__, "layers": 2 * c, "split_layer": c if d + 1 < p else 0,
                           "pp_rank": d, "pp_size": p, "slots": mb * 2 * c + 1})
        m = Model(ctxs[d], st)
        for local, g in enumerate(fold[d]):
            for n in NAMES:
                m.tensor("w." + n, local).copy_(ref_w[(g, n)])
        if d == 0:  # the global first and last layers live on stage 0
            for s in range(mb):
                m.tensor("x_in", strand=s).copy_(ref_x[s])
                m.tensor("dy", strand=s).copy_(ref_dy[s])
        torch.cuda.synchronize()
        m.set_plan(plan, mode="w_pipeline")
        m.zero_grads()
        m.run_program(use_graph=False)
        m.sync()
        got = {(g, n): m.tensor("grad." + n, local).cpu().clone() for local, g in enumerate(fold[d]) for n in NAMES}
        if d == 0:
            got["loss"] = m.tensor("loss").cpu().clone()
            got["dx"] = m.tensor("dx").float().cpu().clone()
        info = m.info()
        m.close()
        return got, info

    outs = _run_ranks(stage_main, p)
    seen = set()
    for got, _ in outs:
        for k, v in got.items():
            assert torch.equal(v, want[k]), k
            seen.add(k)
    assert seen == set(want)
    for ctx in ctxs:
        ctx.close()


# ---------------------------------------------------------------------------
# Helpers shared with the two-GPU NCCL stage test (tests/test_nccl_multi_gpu.py):
# the stage's weights and inputs are rebuilt from the same seeds in each
# process, so no tensors cross process boundaries.
LAYERS, MB, P = 4, 4, 2


def _pp_shape():
    return _tiny(mb=MB, layers=LAYERS)


def stage_plan():
    return planner.lib().search_si_plan(_pp_shape().planner_model(), {"tp": 1}, B200,
                                        {"archetype": "nvlink_h100"})["plan_json"]


def reference_single_stage(plan):
    """The whole stack on one device (sequential SI program): numpy results."""
    shape = _pp_shape()
    ctx = Context.create(0)
    _, ref, _, _ = _build(shape, ctx)
    ref.set_plan(plan, mode="sequential")
    ref.zero_grads()
    ref.run_program(use_graph=True)
    ref.sync()
    want = {"loss": ref.tensor("loss").cpu().numpy().copy(), "dx": ref.tensor("dx").float().cpu().numpy().copy()}
    for g in range(LAYERS):
        for n in NAMES:
            want[f"{g}.{n}"] = ref.tensor("grad." + n, g).cpu().numpy().copy()
    ref.close()
    ctx.close()
    return want


def run_stage(ctx, d, p, plan, layers):
    """Stage d of a p-stage W pipeline on `ctx` (weights of its U-fold layers,
    the inputs on stage 0); returns its gradients (and loss / dx on stage 0)."""
    import numpy as np

    from oracle.layer_oracle import LlamaTPOracle, bf16_round
    from paper_2411_15871_b200.runtime import LlamaShape, Model
    from tests.test_model_gpu import _upload
    shape = _pp_shape()
    orc = LlamaTPOracle(shape.hidden, shape.ffn, shape.n_heads, shape.n_kv_heads, shape.head_dim, shape.layers,
                        shape.seq_len, tp=1, theta=shape.rope_theta, bf16=True, seed=5, init_std=0.05)
    fold = _fold(layers, p)
    c = layers // (2 * p)
    st = LlamaShape(**{**shape.__dict__, "layers": 2 * c, "split_layer": c if d + 1 < p else 0,
                       "pp_rank": d, "pp_size": p, "slots": MB * 2 * c + 1})
    m = Model(ctx, st)
    for local, g in enumerate(fold[d]):
        sh = orc.shard(g, 0)
        for n in NAMES:
            _upload(m.tensor("w." + n, local), sh[n])
            _upload(m.tensor("master." + n, local), sh[n])
    rng = np.random.default_rng(11)  # tests.test_model_gpu._build's input stream
    for s in range(MB):
        x = bf16_round(rng.standard_normal((shape.seq_len, shape.hidden)).astype(np.float32))
        r = bf16_round(rng.standard_normal((shape.seq_len, shape.hidden)).astype(np.float32))
        if d == 0:
            _upload(m.tensor("x_in", strand=s), x)
            _upload(m.tensor("dy", strand=s), r)
    torch.cuda.synchronize()
    m.set_plan(plan, mode="w_pipeline")
    m.zero_grads()
    m.run_program(use_graph=False)
    m.sync()
    got = {f"{g}.{n}": m.tensor("grad." + n, local).cpu().numpy().copy() for local, g in enumerate(fold[d])
           for n in NAMES}
    if d == 0:
        got["loss"] = m.tensor("loss").cpu().numpy().copy()
        got["dx"] = m.tensor("dx").float().cpu().numpy().copy()
    m.close()
    return got


def test_w_pipeline_helpers_loopback():
    """run_stage over the loopback stage group equals the single-stage stack
    (the same helpers the two-GPU NCCL test runs one per process)."""
    import numpy as np
    plan = stage_plan()
    want = reference_single_stage(plan)
    ctxs = Context.loopback_pp_group(0, P)
    outs = _run_ranks(lambda d: (torch.cuda.set_device(0), run_stage(ctxs[d], d, P, plan, LAYERS))[1], P)
    got = {}
    for o in outs:
        got.update(o)
    assert set(got) == set(want)
    for k, v in want.items():
        assert np.array_equal(got[k], v), k
    for c in ctxs:
        c.close()

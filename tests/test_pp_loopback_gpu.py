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

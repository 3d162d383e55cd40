"""GPU: the MoE layer (moe_ep template, reference op_model.cpp:121-169) through
the dh C ABI against the CPU oracle (oracle/layer_oracle.py MoEOracle):
  * router + slot assignment kernels on the device's own ln1: expert ids and
    slot maps identical to the oracle's, probabilities / weights within fp32
    rounding;
  * EP = 1: per-strand losses, input gradient and every weight gradient
    (router, stacked experts, attention, gammas) within bf16 tolerance, with
    and without capacity drops; SI == sequential == graph replay, bit for bit;
  * EP = 2 over the loopback group (two ranks as host threads on one GPU, the
    all-to-alls as device copies): each rank's loss equals the oracle on its
    own micro-batches, each expert's gradient (held by its owner) equals the
    sum of both ranks' oracle gradients; SI == sequential on every rank.
"""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.layer_oracle import MoEOracle, bf16_round  # noqa: E402
from paper_2411_15871_b200 import planner  # noqa: E402
from paper_2411_15871_b200.runtime import Context, LlamaShape, Model  # noqa: E402
from tests.test_model_gpu import B200, _rel, _upload  # noqa: E402

MOE_W = ("wr", "w1g", "w1u", "w2")
DENSE_W = ("wqkv", "wo", "g0", "g1")


def _shape(mb=2, layers=2, capacity=0, experts=4):
    return LlamaShape(hidden=256, ffn=512, n_heads=4, n_kv_heads=2, head_dim=64, layers=layers, seq_len=128,
                      micro_batches=mb, rope_theta=10000.0, experts=experts, topk=2, capacity=capacity)


def _oracle(shape, seed=9):
    return MoEOracle(shape.hidden, shape.ffn, shape.n_heads, shape.n_kv_heads, shape.head_dim, shape.layers,
                     shape.seq_len, shape.experts, topk=shape.topk, capacity=shape.moe_capacity(),
                     theta=shape.rope_theta, bf16=True, seed=seed, init_std=0.05)


def _device_routes(ctx, orc, shape, xs, rs):
    """The device's expert choice per (micro-batch, layer), from one-micro-batch
    runs (every layer then keeps its own activation slot). The oracle replays
    them (MoEOracle.forced) so that a near-tie the two sides break differently
    (bf16 rounding of ln1; top-2 / 3rd logit gaps reach ~1e-3 of their spread at
    these sizes) cannot masquerade as a numerics error; real disagreements raise."""
    one = LlamaShape(**{**shape.__dict__, "micro_batches": 1})
    routes = []
    for x, r in zip(xs, rs):
        m = Model(ctx, one)
        _load(m, orc, one, [x], [r])
        m.set_plan(None, mode="sequential")
        m.zero_grads()
        m.run_program()
        m.sync()
        for l in range(shape.layers):
            routes.append(m.tensor("act.ids", l, 0).cpu().view(torch.int32).numpy().reshape(-1, shape.topk).copy())
        m.close()
    return routes


def _params(orc, l, ep=1, rank=0):
    p = orc.params[l]
    el = orc.E // ep
    ex = slice(rank * el, (rank + 1) * el)
    return {"wqkv": np.concatenate([p["wq"], p["wk"], p["wv"]], 0), "wo": p["wo"], "g0": p["g0"],
            "g1": p["g1"], "wr": p["wr"], "w1g": p["w1g"][ex], "w1u": p["w1u"][ex], "w2": p["w2"][ex]}


def _grads(orc_grads, l, ep=1, rank=0, E=4):
    g = orc_grads[l]
    el = E // ep
    ex = slice(rank * el, (rank + 1) * el)
    return {"wqkv": np.concatenate([g["wq"], g["wk"], g["wv"]], 0), "wo": g["wo"], "g0": g["g0"],
            "g1": g["g1"], "wr": g["wr"], "w1g": g["w1g"][ex], "w1u": g["w1u"][ex], "w2": g["w2"][ex]}


def _load(m, orc, shape, xs, rs, ep=1, rank=0):
    for l in range(shape.layers):
        for name, arr in _params(orc, l, ep, rank).items():
            _upload(m.tensor("w." + name, l), arr)
            _upload(m.tensor("master." + name, l), arr)
    for s in range(shape.micro_batches):
        _upload(m.tensor("x_in", strand=s), xs[s])
        _upload(m.tensor("dy", strand=s), rs[s])
    torch.cuda.synchronize()


def _inputs(shape, n, seed=11):
    rng = np.random.default_rng(seed)
    mk = lambda: bf16_round(rng.standard_normal((shape.seq_len, shape.hidden)).astype(np.float32))  # noqa: E731
    return [mk() for _ in range(n)], [mk() for _ in range(n)]


def _plan(shape, ep, arch="nvlink_h100"):
    return planner.lib().search_si_plan(shape.planner_model(), {"tp": 1, "ep": ep, "dp": ep}, B200,
                                        {"archetype": arch})["plan_json"]


def _snapshot(m, shape):
    out = {"loss": m.tensor("loss").cpu().clone(), "dx": m.tensor("dx").float().cpu().clone()}
    for l in range(shape.layers):
        for name in DENSE_W + MOE_W:
            out[f"{l}.{name}"] = m.tensor("grad." + name, l).cpu().clone()
    return out


@pytest.fixture(scope="module")
def ctx():
    c = Context.create(0)
    yield c
    c.close()


def test_router_and_assignment_on_device_ln1(ctx):
    """Router top-k and capacity slots from the kernels == the oracle's route()
    applied to the same (device) ln1 rows; capacity 48 forces drops."""
    shape = _shape(mb=1, layers=1, capacity=48)
    orc = _oracle(shape)
    xs, rs = _inputs(shape, 1)
    m = Model(ctx, shape)
    _load(m, orc, shape, xs, rs)
    m.set_plan(None, mode="sequential")
    m.zero_grads()
    m.run_program()
    m.sync()
    T, E, K, C = shape.seq_len, shape.experts, shape.topk, 48
    ln1 = m.tensor("act.ln1_full", 0, 0).float().cpu().numpy().reshape(T, shape.hidden)
    probs, ids, wts, slot = orc.route(ln1, orc.params[0]["wr"])
    got_p = m.tensor("act.probs", 0, 0).cpu().numpy().reshape(T, E)
    got_ids = m.tensor("act.ids", 0, 0).cpu().view(torch.int32).numpy().reshape(T, K)
    got_w = m.tensor("act.wts", 0, 0).cpu().numpy().reshape(T, K)
    got_slot = m.tensor("act.mslot", 0, 0).cpu().view(torch.int32).numpy().reshape(T, K)
    got_src = m.tensor("act.slot_src", 0, 0).cpu().view(torch.int32).numpy()
    assert np.max(np.abs(got_p - probs)) < 1e-5
    # no near-ties at this seed: the selection must agree exactly
    srt = np.sort(probs, 1)[:, ::-1]
    assert np.min(srt[:, K - 1] - srt[:, K]) > 1e-5
    assert np.array_equal(got_ids, ids)
    assert np.max(np.abs(got_w - wts)) < 1e-5
    assert np.array_equal(got_slot, slot)
    assert (slot < 0).any(), "capacity 48 should drop assignments"
    ref_src = np.full(E * C, -1, np.int64)
    for t in range(T):
        for k in range(K):
            if slot[t, k] >= 0:
                ref_src[slot[t, k]] = t * K + k
    assert np.array_equal(got_src, ref_src)
    m.close()


@pytest.mark.parametrize("capacity", [0, 128, 48], ids=["default_capacity", "no_drops", "drops"])
def test_ep1_moe_vs_oracle_and_si_equals_sequential(ctx, capacity):
    shape = _shape(mb=2, capacity=capacity)
    orc = _oracle(shape)
    xs, rs = _inputs(shape, 2)
    m = Model(ctx, shape)
    _load(m, orc, shape, xs, rs)
    plan = _plan(shape, 1)
    runs = {}
    for mode, graph in (("si", False), ("sequential", False), ("si", True)):
        m.set_plan(plan, mode=mode)
        m.zero_grads()
        m.run_program(use_graph=graph)
        m.sync()
        runs[(mode, graph)] = _snapshot(m, shape)
    a = runs[("si", False)]
    for key in (("sequential", False), ("si", True)):
        for k in a:
            assert torch.equal(a[k], runs[key][k]), f"{key} != SI eager for {k}"

    orc.forced = _device_routes(ctx, orc, shape, xs, rs)
    grads = orc.zero_grads()
    dx = None
    for s in range(2):
        loss, y, dx, grads = orc.run(xs[s], rs[s], grads)
        tol = 2e-2 * float(np.sqrt(np.sum((y * rs[s]) ** 2)))
        assert abs(float(a["loss"][s]) - loss) < tol, (s, float(a["loss"][s]), loss, tol)
    assert _rel(a["dx"].numpy().reshape(dx.shape), dx) < 3e-2
    for l in range(shape.layers):
        for name, ref in _grads(grads, l, E=shape.experts).items():
            err = _rel(a[f"{l}.{name}"].numpy(), ref.reshape(-1))
            assert err < 3e-2, (l, name, err)
    info = m.info()
    assert info["slots"] == shape.layers + 1
    m.close()


def _run_ranks(fn, n):
    errs, out = [None] * n, [None] * n

    def body(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            errs[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(n)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for e in errs:
        if e is not None:
            raise e
    return out


def test_ep2_loopback_vs_oracle():
    ep = 2
    shape = _shape(mb=2)
    orc = _oracle(shape, seed=13)
    xs, rs = _inputs(shape, 2 * ep, seed=17)  # rank r strands: micro-batches 2r, 2r+1
    plan = _plan(shape, ep, arch="pcie_a40")
    ctxs = Context.loopback_group(0, ep)

    def rank_main(r):
        torch.cuda.set_device(0)
        m = Model(ctxs[r], shape)
        _load(m, orc, shape, xs[2 * r:2 * r + 2], rs[2 * r:2 * r + 2], ep, r)
        res = {}
        for mode in ("si", "sequential"):
            m.set_plan(plan, mode=mode)
            m.zero_grads()
            m.run_program(use_graph=True)  # loopback is not capturable: runs eagerly
            m.sync()
            res[mode] = _snapshot(m, shape)
        info = m.info()
        m.close()
        return res, info

    outs = _run_ranks(rank_main, ep)
    for c in ctxs:
        c.close()
    for r in range(ep):
        si, seq = outs[r][0]["si"], outs[r][0]["sequential"]
        for k in si:
            assert torch.equal(si[k], seq[k]), f"rank {r}: SI != sequential for {k}"
        assert outs[r][1]["program"]["comm"] == "loopback"

    # EP = 2 rank r == EP = 1 on rank r's micro-batches, bit for bit, for
    # everything that sees only rank r's tokens: the all-to-alls move rows
    # without touching them and every GEMM row is computed independently of
    # where its slot sits, so any layout error in the exchange shows up here.
    ctx1 = Context.create(0)
    for r in range(ep):
        m = Model(ctx1, shape)
        _load(m, orc, shape, xs[2 * r:2 * r + 2], rs[2 * r:2 * r + 2])
        m.set_plan(_plan(shape, 1), mode="si")
        m.zero_grads()
        m.run_program(use_graph=False)
        m.sync()
        one = _snapshot(m, shape)
        m.close()
        for k in ["loss", "dx"] + [f"{l}.{n}" for l in range(shape.layers) for n in DENSE_W + ("wr",)]:
            assert torch.equal(outs[r][0]["si"][k], one[k]), f"rank {r}: EP=2 != EP=1 for {k}"

    orc.forced = _device_routes(ctx1, orc, shape, xs, rs)  # micro-batch order 0..3 = rank-major
    ctx1.close()
    rank_grads = []
    for r in range(ep):
        g = orc.zero_grads()
        for s in range(2):
            loss, y, dx, g = orc.run(xs[2 * r + s], rs[2 * r + s], g)
            tol = 2e-2 * float(np.sqrt(np.sum((y * rs[2 * r + s]) ** 2)))
            got = float(outs[r][0]["si"]["loss"][s])
            assert abs(got - loss) < tol, (r, s, got, loss, tol)
        assert _rel(outs[r][0]["si"]["dx"].numpy().reshape(dx.shape), dx) < 3e-2
        rank_grads.append(g)
    for l in range(shape.layers):
        for r in range(ep):
            # replicated weights: this rank's own (pre-all-reduce) gradient;
            # experts: the owner sees every rank's tokens
            own = _grads(rank_grads[r], l, ep, r, shape.experts)
            for name in DENSE_W + ("wr",):
                err = _rel(outs[r][0]["si"][f"{l}.{name}"].numpy(), own[name].reshape(-1))
                assert err < 3e-2, (r, l, name, err)
            tot = [_grads(rank_grads[q], l, ep, r, shape.experts) for q in range(ep)]
            for name in ("w1g", "w1u", "w2"):
                ref = sum(t[name] for t in tot)
                err = _rel(outs[r][0]["si"][f"{l}.{name}"].numpy(), ref.reshape(-1))
                assert err < 3e-2, (r, l, name, err)



def test_ep2_optimizer_keeps_replicas_identical():
    """EP = 2 training step with AdamW: the replicated (attention, router, gamma)
    gradients are all-reduced over the EP group before the update, so both
    ranks' replicas stay bitwise identical while each rank's experts move."""
    ep = 2
    shape = _shape(mb=2)
    orc = _oracle(shape, seed=23)
    xs, rs = _inputs(shape, 2 * ep, seed=29)
    plan = _plan(shape, ep)
    ctxs = Context.loopback_group(0, ep)

    def rank_main(r):
        torch.cuda.set_device(0)
        m = Model(ctxs[r], shape)
        _load(m, orc, shape, xs[2 * r:2 * r + 2], rs[2 * r:2 * r + 2], ep, r)
        # fp32 master copies: a 1e-3 step on a ~1.0 gamma is below the bf16 ulp
        w0 = {n: m.tensor("master." + n, 0).cpu().clone() for n in DENSE_W + MOE_W}
        m.set_plan(plan, mode="si")
        m.zero_grads()
        m.step({"lr": 1e-3}, use_graph=True)
        m.sync()
        w1 = {n: m.tensor("master." + n, 0).cpu().clone() for n in DENSE_W + MOE_W}
        m.close()
        return w0, w1

    outs = _run_ranks(rank_main, ep)
    for c in ctxs:
        c.close()
    for n in DENSE_W + ("wr",):
        assert torch.equal(outs[0][1][n], outs[1][1][n]), f"replica {n} diverged across EP ranks"
    for r in range(ep):
        for n in DENSE_W + MOE_W:
            assert not torch.equal(outs[r][0][n], outs[r][1][n]), f"rank {r}: {n} not updated"


@pytest.mark.parametrize("T,E,K,C", [(200, 8, 1, 16), (96, 16, 3, 12), (130, 12, 2, 16)])
def test_moe_kernels_vs_oracle_edge_cases(T, E, K, C):
    """Kernel level, against the oracle's routing and numpy restatements: top-1 /
    top-3, expert counts that are not powers of two, token counts that are not
    multiples of anything, and capacities small enough to drop most assignments."""
    from paper_2411_15871_b200 import device as dh
    H = 256
    rng = np.random.default_rng(T + E + K)
    x = bf16_round(rng.standard_normal((T, H)).astype(np.float32))
    wr = bf16_round((rng.standard_normal((E, H)) * 0.05).astype(np.float32))
    orc = MoEOracle(H, 256, 4, 2, 64, 1, T, E, topk=K, capacity=C, bf16=True, seed=1)
    probs, ids, wts, slot = orc.route(x, wr)
    cuda = dict(device="cuda")
    xd = torch.from_numpy(x).to(torch.bfloat16).cuda()
    wrd = torch.from_numpy(wr).to(torch.bfloat16).cuda()
    pd = torch.empty(T, E, **cuda)
    idd = torch.empty(T, K, dtype=torch.int32, **cuda)
    wd = torch.empty(T, K, **cuda)
    dh.moe_router_fwd(xd, wrd, pd, idd, wd, K)
    srt = np.sort(probs, 1)[:, ::-1]
    decisive = (srt[:, K - 1] - srt[:, K]) > 1e-5 if K < E else np.ones(T, bool)
    assert np.array_equal(idd.cpu().numpy()[decisive], ids[decisive])
    assert np.max(np.abs(pd.cpu().numpy() - probs)) < 1e-5
    # slots from the device's own expert choice (near-ties aside, the same)
    ids_dev = idd.cpu().numpy().astype(np.int64)
    sl = torch.empty(T, K, dtype=torch.int32, **cuda)
    src = torch.empty(E * C, dtype=torch.int32, **cuda)
    dh.moe_assign(idd, E, C, sl, src)
    fill, ref_slot = np.zeros(E, np.int64), np.full((T, K), -1, np.int64)
    for t in range(T):
        for k in range(K):
            e = ids_dev[t, k]
            if fill[e] < C:
                ref_slot[t, k] = e * C + fill[e]
                fill[e] += 1
    assert np.array_equal(sl.cpu().numpy(), ref_slot)
    assert (ref_slot < 0).any()
    # permute / unpermute / their backwards against numpy on the same slots
    xp = torch.empty(E * C, H, dtype=torch.bfloat16, **cuda)
    dh.moe_permute(xd, src, xp, K)
    ref_xp = np.zeros((E * C, H), np.float32)
    for t in range(T):
        for k in range(K):
            if ref_slot[t, k] >= 0:
                ref_xp[ref_slot[t, k]] = x[t]
    assert np.array_equal(xp.float().cpu().numpy(), ref_xp)
    y = bf16_round(rng.standard_normal((E * C, H)).astype(np.float32))
    yd = torch.from_numpy(y).to(torch.bfloat16).cuda()
    out = torch.empty(T, H, dtype=torch.bfloat16, **cuda)
    dh.moe_unpermute(yd, sl, wd, out)
    w_dev = wd.cpu().numpy()
    ref_out = np.zeros((T, H), np.float32)
    for k in range(K):
        ok = ref_slot[:, k] >= 0
        ref_out[ok] += w_dev[ok, k:k + 1] * y[ref_slot[ok, k]]
    assert np.array_equal(out.float().cpu().numpy(), bf16_round(ref_out))
    dxp = torch.empty(T, H, dtype=torch.bfloat16, **cuda)
    dh.moe_permute_bwd(yd, sl, dxp)
    ref_dx = np.zeros((T, H), np.float32)
    for k in range(K):
        ok = ref_slot[:, k] >= 0
        ref_dx[ok] += y[ref_slot[ok, k]]
    assert np.array_equal(dxp.float().cpu().numpy(), bf16_round(ref_dx))

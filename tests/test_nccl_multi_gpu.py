"""GPU, >= 2 devices: the real NCCL path (NcclComm, csrc/runtime/context.cpp).

One process per GPU, as bench.py runs it. Each rank builds the Megatron TP+SP
layer stack over an NCCL communicator and runs the SI program. Checked:
  * every rank's loss, input-gradient and weight-gradient shards against the
    numpy TP oracle (oracle/layer_oracle.py), bf16 tolerance 3e-2;
  * SI == sequential == relaxed SI, bit for bit, on every rank;
  * pipeline stage transfers (NcclComm::send / recv, weft SendRecv): a
    2-stage W pipeline on two GPUs equals the single-stage stack.

NCCL's reduction order depends on the algorithm, protocol and channel count it
picks. The test pins them, so the bitwise SI == sequential claim rests on a
fixed order: NCCL_ALGO=Ring, NCCL_PROTO=Simple, NCCL_NVLS_ENABLE=0.

Skipped, with the reason, when fewer GPUs are visible than a case needs (the
driver's GPU box has one).
"""
import multiprocessing as mp
import os
import traceback

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

PINNED_NCCL_ENV = {"NCCL_ALGO": "Ring", "NCCL_PROTO": "Simple", "NCCL_NVLS_ENABLE": "0"}
SHAPE = dict(hidden=1024, ffn=2048, n_heads=16, n_kv_heads=8, head_dim=128, layers=2, seq_len=512,
             micro_batches=2, rope_theta=500000.0, slots=4)
NAMES = ("wqkv", "wo", "wg", "wu", "wd", "g0", "g1")


def _ngpus():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _inputs(shape):
    from oracle.layer_oracle import bf16_round
    rng = np.random.default_rng(4)
    xs = [bf16_round(rng.standard_normal((shape.seq_len, shape.hidden)).astype(np.float32)) for _ in range(2)]
    rs = [bf16_round(rng.standard_normal((shape.seq_len, shape.hidden)).astype(np.float32)) for _ in range(2)]
    return xs, rs


def _oracle(shape, tp):
    from oracle.layer_oracle import LlamaTPOracle
    return LlamaTPOracle(shape.hidden, shape.ffn, shape.n_heads, shape.n_kv_heads, shape.head_dim, shape.layers,
                         shape.seq_len, tp=tp, theta=shape.rope_theta, bf16=True, seed=21, init_std=0.05)


def _tp_worker(rank, tp, nid, plan, q):
    try:
        os.environ.update(PINNED_NCCL_ENV)
        import torch as th

        from paper_2411_15871_b200.runtime import Context, LlamaShape, Model
        from tests.test_model_gpu import _upload
        th.cuda.set_device(rank)
        shape = LlamaShape(**SHAPE)
        orc = _oracle(shape, tp)
        xs, rs = _inputs(shape)
        T = shape.seq_len // tp
        ctx = Context.create(rank, rank, tp, nid, 16)
        m = Model(ctx, shape)
        for l in range(shape.layers):
            sh = orc.shard(l, rank)
            for n in NAMES:
                _upload(m.tensor("w." + n, l), sh[n])
        for s in range(2):
            _upload(m.tensor("x_in", strand=s), xs[s][rank * T:(rank + 1) * T])
            _upload(m.tensor("dy", strand=s), rs[s][rank * T:(rank + 1) * T])
        th.cuda.synchronize()
        res = {}
        for mode in ("si", "sequential", "si_relaxed"):
            m.set_plan(plan, mode=mode)
            m.zero_grads()
            m.run_program(use_graph=True)  # NCCL is capturable: graph replay
            m.sync()
            snap = {"loss": m.tensor("loss").cpu().numpy().copy(),
                    "dx": m.tensor("dx").float().cpu().numpy().copy()}
            for l in range(shape.layers):
                for n in NAMES:
                    snap[f"{l}.{n}"] = m.tensor("grad." + n, l).cpu().numpy().copy()
            res[mode] = snap
        comm = m.info()["program"]["comm"]
        m.close()
        ctx.close()
        q.put((rank, res, comm, None))
    except BaseException:  # noqa: BLE001
        q.put((rank, None, None, traceback.format_exc()))


def _spawn(target, n, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=target, args=(r, n, *args, q)) for r in range(n)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(n):
        r, res, extra, err = q.get(timeout=900)
        assert err is None, f"rank {r}:\n{err}"
        out[r] = (res, extra)
    for p in procs:
        p.join(timeout=60)
    return out


@pytest.mark.parametrize("tp", [2, 8])
def test_nccl_tp_vs_oracle_and_si_equals_sequential(tp):
    if _ngpus() < tp:
        pytest.skip(f"needs {tp} GPUs, {_ngpus()} visible")
    from paper_2411_15871_b200 import planner
    from paper_2411_15871_b200.runtime import LlamaShape, nccl_unique_id
    from tests.test_model_gpu import B200, _rel
    shape = LlamaShape(**SHAPE)
    plan = planner.lib().search_si_plan(shape.planner_model(), {"tp": tp, "sp": True}, B200,
                                        {"archetype": "pcie_a40"})["plan_json"]
    outs = _spawn(_tp_worker, tp, nccl_unique_id(), plan)
    for r in range(tp):
        res, comm = outs[r]
        assert comm == "nccl"
        for k in res["si"]:
            assert np.array_equal(res["si"][k], res["sequential"][k]), f"rank {r}: SI != sequential for {k}"
            assert np.array_equal(res["si"][k], res["si_relaxed"][k]), f"rank {r}: relaxed SI != SI for {k}"
    orc = _oracle(shape, tp)
    xs, rs = _inputs(shape)
    p = planner.parse_plan(plan)
    first_gate = p["bwd_seq"].index(24) < p["bwd_seq"].index(25)
    grads = orc.zero_grads()
    T = shape.seq_len // tp
    for s in range(2):
        loss, y, dx, grads = orc.run(xs[s], rs[s], grads, dx_first_gate=first_gate)
        got = sum(float(outs[r][0]["si"]["loss"][s]) for r in range(tp))
        tol = 2e-2 * float(np.sqrt(np.sum((y * rs[s]) ** 2)))
        assert abs(got - loss) < tol, (s, got, loss)
    dx_got = np.concatenate([outs[r][0]["si"]["dx"].reshape(T, -1) for r in range(tp)], 0)
    assert _rel(dx_got, dx) < 3e-2
    D, nq_l, nkv_l, F_l = shape.head_dim, shape.n_heads // tp, shape.n_kv_heads // tp, shape.ffn // tp
    for l in range(shape.layers):
        g = grads[l]
        for r in range(tp):
            q = g["wq"][r * nq_l * D:(r + 1) * nq_l * D]
            k = g["wk"][r * nkv_l * D:(r + 1) * nkv_l * D]
            v = g["wv"][r * nkv_l * D:(r + 1) * nkv_l * D]
            ref = {"wqkv": np.concatenate([q, k, v], 0), "wo": g["wo"][:, r * nq_l * D:(r + 1) * nq_l * D],
                   "wg": g["wg"][r * F_l:(r + 1) * F_l], "wu": g["wu"][r * F_l:(r + 1) * F_l],
                   "wd": g["wd"][:, r * F_l:(r + 1) * F_l]}
            for n, arr in ref.items():
                err = _rel(outs[r][0]["si"][f"{l}.{n}"], np.ascontiguousarray(arr).reshape(-1))
                assert err < 3e-2, (tp, r, l, n, err)
        for n in ("g0", "g1"):
            tot = sum(outs[r][0]["si"][f"{l}.{n}"] for r in range(tp))
            assert _rel(tot, g[n]) < 3e-2


def _pp_worker(rank, p, nid, plan, layers, q):
    try:
        os.environ.update(PINNED_NCCL_ENV)
        import torch as th

        from paper_2411_15871_b200.runtime import Context
        from tests.test_pp_loopback_gpu import run_stage
        th.cuda.set_device(rank)
        ctx = Context.create_pp(rank, rank, p, nid)
        res = run_stage(ctx, rank, p, plan, layers)
        ctx.close()
        q.put((rank, res, None, None))
    except BaseException:  # noqa: BLE001
        q.put((rank, None, None, traceback.format_exc()))


def test_nccl_pipeline_two_stages_equal_single_stage():
    if _ngpus() < 2:
        pytest.skip(f"needs 2 GPUs, {_ngpus()} visible")
    from paper_2411_15871_b200.runtime import nccl_unique_id
    from tests.test_pp_loopback_gpu import LAYERS, reference_single_stage, stage_plan
    plan = stage_plan()
    ref = reference_single_stage(plan)
    outs = _spawn(_pp_worker, 2, nccl_unique_id(), plan, LAYERS)
    got = {}
    for r in range(2):
        got.update(outs[r][0])
    for k, v in ref.items():
        assert np.array_equal(got[k], v), k


# --------------------------------------------------------------------------- collectives alone (dh_comm_run)

def _coll_inputs(n, rank, count, seed=7):
    """bf16-exact inputs: small integers, so sums are exact in any order."""
    g = torch.Generator().manual_seed(seed + rank)
    return torch.randint(-8, 8, (n * count,), generator=g).to(torch.bfloat16)


def _check_collectives(ctx, rank, n, count):
    dev = torch.device("cuda", torch.cuda.current_device())
    send = [_coll_inputs(n, r, count) for r in range(n)]
    mine = send[rank].to(dev)
    # all-gather: every rank's first `count` elements, rank-major
    ag = torch.empty(n * count, dtype=torch.bfloat16, device=dev)
    ctx.collective("all_gather", mine[:count].contiguous(), ag, count)
    # reduce-scatter: this rank's chunk summed over ranks
    rs = torch.empty(count, dtype=torch.bfloat16, device=dev)
    ctx.collective("reduce_scatter", mine, rs, count)
    # fp32 all-reduce
    ar = mine.float().clone()
    ctx.collective("all_reduce_f32", ar, ar, n * count)
    torch.cuda.synchronize()
    want_ag = torch.cat([s[:count] for s in send])
    want_rs = sum(s[rank * count:(rank + 1) * count].float() for s in send).to(torch.bfloat16)
    want_ar = sum(s.float() for s in send)
    assert torch.equal(ag.cpu(), want_ag)
    assert torch.equal(rs.cpu(), want_rs)
    assert torch.equal(ar.cpu(), want_ar)


def test_nccl_one_rank_collectives():
    """The NCCL backend on one GPU: a one-rank communicator (dh_ctx_create with
    tp_size 1 and an id) runs every collective kind through ncclAllGather /
    ncclReduceScatter / ncclAllReduce, against their definitions."""
    if _ngpus() < 1:
        pytest.skip("no GPU")
    from paper_2411_15871_b200.runtime import Context, nccl_unique_id
    os.environ.update(PINNED_NCCL_ENV)
    ctx = Context.create(0, 0, 1, nccl_unique_id(), 16)
    _check_collectives(ctx, 0, 1, 4096 * 16)
    ctx.close()


def test_loopback_collectives_match_definitions():
    if _ngpus() < 1:
        pytest.skip("no GPU")
    import threading

    from paper_2411_15871_b200.runtime import Context
    n = 4
    ctxs = Context.loopback_group(0, n)
    errs = []

    def body(r):
        try:
            torch.cuda.set_device(0)
            _check_collectives(ctxs[r], r, n, 8192)
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(n)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    for c in ctxs:
        c.close()
    if errs:
        raise errs[0]


def _coll_worker(rank, n, nid, q):
    try:
        os.environ.update(PINNED_NCCL_ENV)
        import torch as th

        from paper_2411_15871_b200.runtime import Context
        th.cuda.set_device(rank)
        ctx = Context.create(rank, rank, n, nid, 16)
        _check_collectives(ctx, rank, n, 1 << 16)
        ctx.close()
        q.put((rank, True, None, None))
    except BaseException:  # noqa: BLE001
        q.put((rank, None, None, traceback.format_exc()))


@pytest.mark.parametrize("n", [2, 8])
def test_nccl_collectives_multi_gpu(n):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs, {_ngpus()} visible")
    from paper_2411_15871_b200.runtime import nccl_unique_id
    _spawn(_coll_worker, n, nccl_unique_id())

"""CPU: the MoE layer (moe_ep template, reference op_model.cpp:121-169) on the
host side — no GPU needed.

  * the executor lowers moe_ep plans with the same invariants as dense ones
    (acyclic waits, strand order = the plan's sequences, safe slot reuse,
    per-layer AdamW after every gradient writer) at EP = 1, 2 and 8;
  * the four all-to-all nodes sit on the local_comm lane, everything else
    on compute, and every EP rank lowers the identical all-to-all sequence
    (NCCL grouped send/recv must match across ranks), also across 2 gloo
    processes;
  * the device's default capacity equals the oracle's moe_capacity();
  * the oracle's forced-route replay accepts near-ties only.
"""
import hashlib
import json
import multiprocessing as mp
import os

import numpy as np
import pytest

from oracle.layer_oracle import MoEOracle, moe_capacity
from paper_2411_15871_b200 import planner
from paper_2411_15871_b200.runtime import PHI35_MOE, TINY_MOE, LlamaShape, lower
from tests.planner_corpus import B200_CLUSTER
from tests.test_executor_lowering import check_program

A2A = {11, 14, 22, 27}


def _plan(shape, ep, arch="nvlink_h100"):
    return planner.lib().search_si_plan(shape.planner_model(), {"tp": 1, "ep": ep, "dp": ep}, B200_CLUSTER,
                                        {"archetype": arch})["plan_json"]


@pytest.mark.parametrize("ep", [1, 2, 4])
@pytest.mark.parametrize("mb", [1, 2, 3])
def test_moe_programs(ep, mb):
    shape = LlamaShape(**{**TINY_MOE.__dict__, "micro_batches": mb})
    plan = _plan(shape, ep)
    p = json.loads(plan)
    # moe_ep template: a2a nodes exist exactly when ep > 1, tp_sp nodes never (tp = 1)
    assert (set(p["fwd_seq"]) & A2A) == ({11, 14} if ep > 1 else set())
    assert (set(p["bwd_seq"]) & A2A) == ({22, 27} if ep > 1 else set())
    assert not set(p["fwd_seq"]) & {1, 6} and not set(p["bwd_seq"]) & {32, 39}
    si = lower(shape, ep, plan, "si")
    seq = lower(shape, ep, plan, "sequential")
    used_si = check_program(si, shape, mb)
    used_seq = check_program(seq, shape, mb)
    assert len(used_seq) == shape.layers
    assert len(used_si) == (shape.layers + 1 if mb > 1 else shape.layers)
    for o in si["ops"]:
        if o["node"] == 100:
            assert o["lane"] == 2
        else:
            assert o["lane"] == (1 if o["node"] in A2A else 0), o
    # EP > 1: replicated weights need the DP all-reduce first, so AdamW runs after the program
    assert any(o["node"] == 100 for o in si["ops"]) == (ep == 1)


def test_phi35_moe_ep8_program():
    shape = LlamaShape(**{**PHI35_MOE.__dict__, "layers": 4, "micro_batches": 4})
    plan = _plan(shape, 8)
    prog = lower(shape, 8, plan, "si")
    check_program(prog, shape, 4)
    assert sum(o["node"] in A2A for o in prog["ops"]) == 4 * 4 * 4


def _a2a_signature(shape, ep, rank, plan):
    prog = lower(shape, ep, plan, "si", rank=rank)
    seq = [(o["strand"], o["layer"], o["node"]) for o in prog["ops"] if o["node"] in A2A]
    return hashlib.sha256(json.dumps(seq).encode()).hexdigest()


def test_ep_ranks_lower_identical_all_to_all_order():
    shape = LlamaShape(**{**TINY_MOE.__dict__, "micro_batches": 3})
    plan = _plan(shape, 4, "pcie_a40")
    assert len({_a2a_signature(shape, 4, r, plan) for r in range(4)}) == 1


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shape = LlamaShape(**{**TINY_MOE.__dict__, "micro_batches": 2})
    plan = _plan(shape, world)
    sig = _a2a_signature(shape, world, rank, plan)
    t = torch.tensor(list(bytes.fromhex(sig)), dtype=torch.int64)
    gathered = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(gathered, t)
    q.put((rank, all(torch.equal(g, gathered[0]) for g in gathered)))
    dist.destroy_process_group()


def test_gloo_two_ep_ranks_agree_on_all_to_all_order():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 500
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res)


@pytest.mark.parametrize("tokens,experts,topk", [(128, 4, 2), (3072, 16, 2), (4096, 8, 1), (100, 3, 2)])
def test_default_capacity_matches_oracle(tokens, experts, topk):
    shape = LlamaShape(hidden=256, ffn=512, n_heads=4, n_kv_heads=2, head_dim=64, layers=1, seq_len=tokens,
                       experts=experts, topk=topk)
    assert shape.moe_capacity() == moe_capacity(tokens, experts, topk)


def test_oracle_forced_routes_accept_only_near_ties():
    orc = MoEOracle(256, 512, 4, 2, 64, 1, 16, 4, topk=2, bf16=True, seed=3, init_std=0.05)
    rng = np.random.default_rng(0)
    ln1 = rng.standard_normal((16, 256)).astype(np.float32)
    wr = orc.params[0]["wr"]
    _, ids, _, _ = orc.route(ln1, wr)
    logits = ln1 @ wr.T
    # swap the 2nd choice of the token with the smallest 2nd/3rd logit gap: a near-tie
    srt = np.sort(logits, 1)[:, ::-1]
    t = int(np.argmin(srt[:, 1] - srt[:, 2]))
    third = int(np.argsort(-logits[t])[2])
    forced = ids.copy()
    forced[t, 1] = third
    orc.tie_tol = 10.0 * float(srt[t, 1] - srt[t, 2]) / float(np.std(logits))
    orc.forced = [forced]
    _, got, _, _ = orc.route(ln1, wr)
    assert np.array_equal(got, forced) and orc.flips == 1
    # a decisive disagreement (the last choice instead of the first) raises
    bad = ids.copy()
    t2 = int(np.argmax(srt[:, 0] - srt[:, -1]))
    bad[t2, 0] = int(np.argmin(logits[t2]))
    orc.tie_tol = 1e-2
    orc.forced = [bad]
    with pytest.raises(AssertionError):
        orc.route(ln1, wr)

"""CPU: invariants of the SI executor's lowering (csrc/runtime/executor.cpp),
through the host-only dh_lower_json entry point — no GPU needed.

  * every event wait refers to an earlier op (acyclic, deadlock-free issue);
  * each strand runs forward layers 0..L-1 in the plan's fwd_seq order and
    backward layers L-1..0 in bwd_seq order, whatever the interleaving;
  * activation-slot reuse is safe: when (strand, layer) instance B takes the
    slot instance A used, every op of A happens-before every op of B in the
    stream-order + event-wait graph;
  * SI uses L+1 slots (one more than sequential), and interleaves strands;
  * every TP rank lowers the identical collective sequence (NCCL requires it),
    also checked across 2 gloo processes;
  * the per-layer AdamW ops happen after every gradient writer of their layer.
"""
import hashlib
import json
import os

import pytest

from paper_2411_15871_b200 import planner
from paper_2411_15871_b200.runtime import LLAMA3_8B, TINY, LlamaShape, lower
from tests.planner_corpus import B200_CLUSTER

COMM_NODES = {1, 6, 9, 13, 21, 27, 30, 37}


def _plan(shape, tp, arch="nvlink_h100", caps=None):
    return planner.lib().search_si_plan(shape.planner_model(), {"tp": tp, "sp": tp > 1}, B200_CLUSTER,
                                        {"archetype": arch}, caps=caps)["plan_json"]


def _happens_before(ops):
    """preds[i] = direct predecessors (same-lane previous op + waits)."""
    last = {}
    preds = []
    for i, o in enumerate(ops):
        p = set(o["waits"])
        if o["lane"] in last:
            p.add(last[o["lane"]])
        last[o["lane"]] = i
        preds.append(p)
    return preds


def _reachable_from(preds, target_set, start):
    """Is every op in target_set an ancestor of `start`?"""
    seen, stack = set(), [start]
    while stack:
        i = stack.pop()
        for p in preds[i]:
            if p not in seen:
                seen.add(p)
                stack.append(p)
    return target_set <= seen


def check_program(prog, shape, mb, strict_order=True):
    """strict_order=False (mode 4, deferred weight gradients): each (strand,
    layer) still issues its ops in the plan's order, layers may interleave."""
    ops = prog["ops"]
    L = shape.layers
    for i, o in enumerate(ops):
        assert all(w < i for w in o["waits"]), "wait on a later op"
    for s in range(mb):
        # (not transfers; mlp_fc1_wgrad issued as two halves counts once, at its first half)
        mine = [(o["layer"], o["node"]) for o in ops if o["strand"] == s and o["node"] < 100 and o.get("part", -1) != 1]
        expect = [(l, n) for l in range(L) for n in prog["fwd_seq"]] + \
                 [(l, n) for l in reversed(range(L)) for n in prog["bwd_seq"]]
        # SI modes: the unpaired last backward strand re-places its weight gradients
        # under its own collectives (executor.cpp backward_layer_dag)
        lone = s == mb - 1 and prog.get("mode", 0) != 1
        if strict_order and not lone:
            assert mine == expect, f"strand {s} order"
        else:
            assert sorted(mine) == sorted(expect), f"strand {s} ops"
            # deferrable weight gradients (mlp_down_wgrad, attention; the lone last
            # backward strand also moves mlp_fc1_wgrad under rs0_bwd_ag)
            moved = {34, 38} if 40 in prog["bwd_seq"] else {23, 26, 32, 36}  # moe_ep ids: attention wgrads
            for l in range(L):
                fb = [n for (ll, n) in mine if ll == l and n not in moved]
                want = [n for n in list(prog["fwd_seq"]) + list(prog["bwd_seq"]) if n not in moved]
                assert fb == want, f"strand {s} layer {l} order"
    # slot reuse safety
    preds = _happens_before(ops)
    inst_ops = {}
    for i, o in enumerate(ops):
        inst_ops.setdefault((o["strand"], o["layer"]), []).append(i)
    by_slot = {}
    for key, idx in inst_ops.items():
        by_slot.setdefault(ops[idx[0]]["slot"], []).append((idx[0], key))
    for slot, users in by_slot.items():
        users.sort()
        for (_, a), (_, b) in zip(users, users[1:]):
            a_ops, b_first = set(inst_ops[a]), inst_ops[b][0]
            # b's first op must come after all of a's ops (a's last op on each lane suffices)
            assert _reachable_from(preds, a_ops - {b_first}, b_first) or not (a_ops - {b_first}), \
                f"slot {slot}: {b} may start before {a} finished"
    # the layer input of (s, l) lives in (s, l-1)'s slot and must stay live until (s, l) bwd finishes
    for (s, l), idx in inst_ops.items():
        if l == 0:
            continue
        prev_slot = ops[inst_ops[(s, l - 1)][0]]["slot"]
        assert all(ops[i]["prev_slot"] == prev_slot for i in idx)
    # the in-program AdamW of layer l (strand -1, node 100) runs after every
    # strand's backward of layer l, once per layer, on the cross lane
    opt = [i for i, o in enumerate(ops) if o["node"] == 100]
    if opt:
        assert sorted(ops[i]["layer"] for i in opt) == list(range(L))
        for i in opt:
            l = ops[i]["layer"]
            writers = {j for j, o in enumerate(ops) if o["strand"] >= 0 and o["layer"] == l
                       and o["node"] in prog["bwd_seq"]}
            assert _reachable_from(preds, writers, i), f"AdamW of layer {l} may run before its gradients"
    return {o["slot"] for o in ops if o["node"] != 100}


@pytest.mark.parametrize("tp", [1, 2, 4, 8])
@pytest.mark.parametrize("mb", [1, 2, 3])
def test_tiny_programs(tp, mb):
    shape = LlamaShape(**{**TINY.__dict__, "micro_batches": mb, "n_kv_heads": 4 if tp > 2 else 2})
    if tp == 8:
        shape = LlamaShape(**{**shape.__dict__, "n_heads": 8, "n_kv_heads": 8, "head_dim": 64, "hidden": 512,
                              "ffn": 1024})
    plan = _plan(shape, tp)
    si = lower(shape, tp, plan, "si")
    seq = lower(shape, tp, plan, "sequential")
    rel = lower(shape, tp, plan, "si_relaxed")
    used_si = check_program(si, shape, mb)
    used_seq = check_program(seq, shape, mb)
    # relaxed steps: the same launches in the same order, a subset of the waits
    assert check_program(rel, shape, mb) == used_si
    assert [(o["strand"], o["layer"], o["node"], o["lane"], o["slot"]) for o in rel["ops"]] == \
           [(o["strand"], o["layer"], o["node"], o["lane"], o["slot"]) for o in si["ops"]]
    # ... and every ordering it imposes is one SI also imposes (its graph is a relaxation)
    si_preds = _happens_before(si["ops"])
    for i, o in enumerate(rel["ops"]):
        extra = set(o["waits"]) - set(si["ops"][i]["waits"])
        assert not extra or _reachable_from(si_preds, extra, i)
    assert sum(len(o["waits"]) for o in rel["ops"]) <= sum(len(o["waits"]) for o in si["ops"])
    assert len(used_seq) == shape.layers
    assert len(used_si) == (shape.layers + 1 if mb > 1 else shape.layers)
    if mb > 1:  # SI interleaves the two strands inside each SI block
        strands = [o["strand"] for o in si["ops"]]
        switches = sum(1 for a, b in zip(strands, strands[1:]) if a != b)
        assert switches > 2 * shape.layers
    if tp > 1:
        comm = [o for o in si["ops"] if o["node"] in COMM_NODES]
        assert comm and all(o["lane"] == 1 for o in comm)
        assert all(o["lane"] == 0 for o in si["ops"] if o["node"] not in COMM_NODES and o["node"] != 100)
        assert all(o["lane"] == 2 for o in si["ops"] if o["node"] == 100)


def test_llama3_8b_tp8_h100_plan_program():
    shape = LlamaShape(**{**LLAMA3_8B.__dict__, "layers": 4, "micro_batches": 2})
    plan = _plan(shape, 8)
    p = json.loads(plan)
    assert p["fwd_cuts"] == [1] and p["bwd_cuts"] == [4]
    prog = lower(shape, 8, plan, "si")
    check_program(prog, shape, 2)
    # first_dx follows the plan's order of mlp_gate_dgrad / mlp_up_dgrad
    first = p["bwd_seq"].index(24) < p["bwd_seq"].index(25)
    for o in prog["ops"]:
        if o["node"] == 24:
            assert o["first_dx"] == first
        if o["node"] == 25:
            assert o["first_dx"] == (not first)


def _comm_signature(shape, tp, rank, plan):
    prog = lower(shape, tp, plan, "si", rank=rank)
    seq = [(o["strand"], o["layer"], o["node"]) for o in prog["ops"] if o["node"] in COMM_NODES]
    return hashlib.sha256(json.dumps(seq).encode()).hexdigest()


def test_ranks_lower_identical_collective_order():
    shape = LlamaShape(**{**TINY.__dict__, "n_kv_heads": 4, "micro_batches": 3})
    plan = _plan(shape, 4, "pcie_a40")
    sigs = {_comm_signature(shape, 4, r, plan) for r in range(4)}
    assert len(sigs) == 1


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shape = LlamaShape(**{**TINY.__dict__, "n_kv_heads": 2, "micro_batches": 2})
        # rank 0 plans and broadcasts (as bench.py broadcasts the NCCL unique id)
        obj = [_plan(shape, world) if rank == 0 else None, b"\x01" * 128 if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        plan, uid = obj
        mine = _comm_signature(shape, world, rank, plan)
        allsig = [None] * world
        dist.all_gather_object(allsig, mine)
        q.put((rank, len(set(allsig)) == 1 and uid == b"\x01" * 128))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_agree_on_program():
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    res = dict(q.get(timeout=10) for _ in range(2))
    assert res == {0: True, 1: True}
    assert all(p.exitcode == 0 for p in procs)


def _stage_shape(shape, layers, p, d, mb, slots=None):
    c = layers // (2 * p)
    return LlamaShape(**{**shape.__dict__, "layers": 2 * c, "split_layer": c if d + 1 < p else 0,
                         "pp_rank": d, "pp_size": p, "micro_batches": mb, "slots": slots or mb * 2 * c + 1})


@pytest.mark.parametrize("p,layers,mb", [(2, 4, 4), (2, 8, 8), (4, 16, 6)])
def test_w_pipeline_stage_programs(p, layers, mb):
    """Mode 3 (W pipeline stage): every stage runs each of its micro-batches'
    forward / backward over its U-fold layers in plan order, every transfer has
    exactly one matching transfer on the peer (same tag: kind and micro-batch),
    and the per-layer AdamW follows the last micro-batch's backward."""
    plan = _plan(TINY, 1)
    progs = [lower(_stage_shape(TINY, layers, p, d, mb), 1, plan, "w_pipeline") for d in range(p)]
    sends, recvs = {}, {}
    for d, prog in enumerate(progs):
        shape = _stage_shape(TINY, layers, p, d, mb)
        check_program(prog, shape, mb)
        for o in prog["ops"]:
            kind = {101: "act", 102: "act", 103: "grad", 104: "grad"}.get(o["node"])
            if kind:
                key = (d, o["peer"], kind, o["strand"]) if o["node"] in (101, 103) else (o["peer"], d, kind, o["strand"])
                book = sends if o["node"] in (101, 103) else recvs
                assert key not in book
                book[key] = o
    assert set(sends) == set(recvs) and sends
    # each micro-batch crosses every stage boundary twice per pass (down and back up)
    assert len(sends) == 2 * 2 * (p - 1) * mb


def test_w_pipeline_slots_vs_reference_memory_replay():
    """Activation slots the stage program holds at once against the reference
    memory replay of the same W schedule (simulate_memory, one byte per layer
    activation): the replay frees and allocates at the same block end, the
    executor's SI visits need one extra slot (the forward strand takes its
    slot before the backward strand returns one)."""
    layers, p, mb = 80, 2, 8  # config 5's layer count on PP = 2
    plan = _plan(TINY, 1)
    sched = {"discipline": "w_shape", "m": mb, "p": p}
    replay = planner.lib().memory({"act_bytes_per_layer": 1, "state_bytes_per_layer": 0, "layers": layers,
                                   "capacity_bytes": 1 << 40}, schedule=sched)
    dev = json.loads(replay["peaks_json"])["devices"]
    for d in range(p):
        prog = lower(_stage_shape(TINY, layers, p, d, mb, slots=8 * layers), 1, plan, "w_pipeline")
        assert dev[d]["peak_bytes"] <= prog["peak_slots"] <= dev[d]["peak_bytes"] + 1, (d, prog["peak_slots"], dev[d])


# ---------------------------------------------------------------------------
# Transient-buffer hazards. The bwd transient set, the fwd transient set and
# the running-gradient ping-pong are shared by every (strand, layer); each
# node's reads / writes below restate csrc/runtime/model.cpp launch_node and
# csrc/runtime/moe.cpp. Every two accesses to one buffer where either writes
# must be ordered (program order) in the stream + event happens-before graph:
# RAW, WAR and WAW across lanes, strands and layers, in every executor mode.

def _dense_access(node, tp, L, l, s):
    """(reads, writes) of shared buffers for one dense op (activation slots excluded)."""
    t1 = tp == 1
    dy = f"mb_dy{s}" if l == L - 1 else f"grad{(L - 2 - l) & 1}"
    dx = f"grad{(L - 1 - l) & 1}"
    x_in = f"mb_in{s}" if l == 0 else None
    part = "fs.rs_out" if t1 else "fs.part"
    dpart = "bs.rs_out" if t1 else "bs.dx_part"
    R, W = set(), set()
    if node == 0:
        R |= {x_in}; W |= set() if t1 else {"fs.ln_loc"}
    elif node in (1, 9):
        R |= {"fs.ln_loc"}
    elif node == 4:
        R |= {"bs.attn_scratch"}; W |= {"bs.attn_scratch"}
    elif node in (5, 12):
        W |= {part}
    elif node in (6, 13):
        R |= {"fs.part"}; W |= {"fs.rs_out"}
    elif node == 7:
        R |= {x_in, "fs.rs_out"}
    elif node == 8:
        W |= set() if t1 else {"fs.ln_loc"}
    elif node == 14:
        R |= {"fs.rs_out"} | ({f"mb_dy{s}", "loss"} if l == L - 1 else set())
        W |= {"loss"} if l == L - 1 else set()
    elif node == 21:
        R |= {dy}; W |= {f"bs.dy_full{l & 1}"}
    elif node in (22, 23):
        R |= {dy if t1 else f"bs.dy_full{l & 1}"}; W |= {"bs.d_gate", "bs.d_up"} if node == 22 else set()
    elif node in (24, 25):
        R |= {"bs.d_gate", "bs.d_up", dpart}; W |= {dpart}
    elif node == 26:
        R |= {"bs.d_gate", "bs.d_up"}
    elif node in (27, 37):
        R |= {"bs.dx_part"}; W |= {"bs.rs_out"}
    elif node == 28:
        R |= {"bs.rs_out", dy}; W |= {"bs.d_x1", "bs.ln_partial"}
    elif node == 30:
        R |= {"bs.d_x1"}; W |= {"bs.dx1_full"}
    elif node in (31, 32):
        R |= {"bs.d_x1" if t1 else "bs.dx1_full"}; W |= {"bs.d_o"} if node == 31 else set()
    elif node == 34:
        R |= {"bs.d_o", "bs.attn_scratch"}; W |= {"bs.dqkv", "bs.attn_scratch"}
    elif node == 35:
        R |= {"bs.dqkv"}; W |= {dpart}
    elif node == 36:
        R |= {"bs.dqkv"}
    elif node == 38:
        R |= {x_in, "bs.rs_out", "bs.d_x1"}; W |= {dx, "bs.ln_partial"}
    return R - {None}, W


MOE_DENSE = {0: 0, 2: 2, 4: 4, 5: 5, 7: 7, 8: 8, 16: 14, 20: 20, 30: 28, 31: 29, 33: 31, 34: 32, 36: 34, 37: 35,
             38: 36, 40: 38}


def _moe_access(node, ep, L, l, s):
    if node in MOE_DENSE:
        return _dense_access(MOE_DENSE[node], 1, L, l, s)
    a2a = ep > 1
    dy = f"mb_dy{s}" if l == L - 1 else f"grad{(L - 2 - l) & 1}"
    R, W = set(), set()
    if node == 10:
        W |= {"fs.xp"} if a2a else set()
    elif node == 11:
        R |= {"fs.xp"}
    elif node == 13:
        W |= {"fs.ye"} if a2a else set()
    elif node == 14:
        R |= {"fs.ye"}
    elif node == 15:
        W |= {"fs.rs_out"}
    elif node == 21:
        R |= {dy}; W |= {"bs.dys" if a2a else "bs.dys_e", "bs.dw"}
    elif node == 22:
        R |= {"bs.dys"}; W |= {"bs.dys_e"}
    elif node in (23, 24):
        R |= {"bs.dys_e"}; W |= {"bs.d_gate", "bs.d_up"} if node == 23 else set()
    elif node == 25:
        R |= {"bs.d_gate", "bs.d_up"}; W |= {"bs.dxe"}
    elif node == 26:
        R |= {"bs.d_gate", "bs.d_up"}
    elif node == 27:
        R |= {"bs.dxe"}; W |= {"bs.dxp"}
    elif node == 28:
        R |= {"bs.dxp" if a2a else "bs.dxe"}; W |= {"bs.rs_out"}
    elif node == 29:
        R |= {"bs.dw", "bs.rs_out"}; W |= {"bs.rs_out", "bs.router_scratch"}
    return R, W


def observed_writers(prog, L, access):
    """{(strand, layer, node, buffer): (strand, layer, node) of the write it reads}:
    what each read sees when the program runs in its (hazard-checked) order."""
    last, seen = {}, {}
    for o in prog["ops"]:
        if o["strand"] < 0 or o["node"] >= 100:
            continue
        R, W = access(o["node"], L, o["layer"], o["strand"])
        me = (o["strand"], o["layer"], o["node"])
        for b in R:
            seen[me + (b,)] = last.get(b)
        for b in W:
            last[b] = me
    return seen


def check_buffer_hazards(prog, L, access):
    ops = prog["ops"]
    preds = _happens_before(ops)
    anc = []
    for i, p in enumerate(preds):
        a = 0
        for j in p:
            a |= anc[j] | (1 << j)
        anc.append(a)
    last_w, reads_since = {}, {}
    for j, o in enumerate(ops):
        if o["strand"] < 0 or o["node"] >= 100:
            continue
        R, W = access(o["node"], L, o["layer"], o["strand"])
        for b in R | W:
            w = last_w.get(b)
            if w is not None:
                assert anc[j] >> w & 1, f"{b}: op {j} {o} not ordered after writer {w} {ops[w]}"
        for b in W:
            for r in reads_since.get(b, ()):
                assert anc[j] >> r & 1, f"{b}: writer {j} {o} not ordered after reader {r} {ops[r]}"
        for b in R:
            reads_since.setdefault(b, []).append(j)
        for b in W:
            last_w[b] = j
            reads_since[b] = []


@pytest.mark.parametrize("tp", [1, 2, 4])
@pytest.mark.parametrize("mode", ["si", "si_relaxed", "sequential"])
def test_transient_buffer_hazards_dense(tp, mode):
    shape = LlamaShape(**{**TINY.__dict__, "micro_batches": 3, "n_kv_heads": 4})
    for arch in ("nvlink_h100", "pcie_a40"):
        prog = lower(shape, tp, _plan(shape, tp, arch), mode)
        check_buffer_hazards(prog, shape.layers, lambda n, L, l, s: _dense_access(n, tp, L, l, s))


@pytest.mark.parametrize("ep", [1, 2, 4])
@pytest.mark.parametrize("mode", ["si", "si_relaxed", "sequential"])
def test_transient_buffer_hazards_moe(ep, mode):
    from paper_2411_15871_b200.runtime import TINY_MOE
    shape = LlamaShape(**{**TINY_MOE.__dict__, "micro_batches": 3})
    for arch in ("nvlink_h100", "pcie_a40"):
        plan = planner.lib().search_si_plan(shape.planner_model(), {"tp": 1, "ep": ep, "dp": ep}, B200_CLUSTER,
                                            {"archetype": arch})["plan_json"]
        prog = lower(shape, ep, plan, mode)
        check_buffer_hazards(prog, shape.layers, lambda n, L, l, s: _moe_access(n, ep, L, l, s))


@pytest.mark.parametrize("tp", [2, 4, 8])
@pytest.mark.parametrize("mb", [2, 3])
def test_deferred_wgrad_programs(tp, mb):
    """Mode 4: relaxed SI steps with the attention weight gradients deferred
    into the next layer pair; one extra activation slot; hazard-free."""
    base = {**TINY.__dict__, "micro_batches": mb, "n_kv_heads": 4 if tp > 2 else 2}
    if tp == 8:
        base.update(n_heads=8, n_kv_heads=8, head_dim=64, hidden=512, ffn=1024)
    shape = LlamaShape(**{**base, "slots": TINY.layers + 2})
    for arch in ("nvlink_h100", "pcie_a40"):
        plan = _plan(shape, tp, arch)
        prog = lower(shape, tp, plan, "si_deferred")
        check_program(prog, shape, mb, strict_order=False)
        acc = lambda n, L, l, s: _dense_access(n, tp, L, l, s)  # noqa: E731
        check_buffer_hazards(prog, shape.layers, acc)
        rel = lower(shape, tp, plan, "si_relaxed")
        # every read sees the same write as in the undeferred program
        assert observed_writers(prog, shape.layers, acc) == observed_writers(rel, shape.layers, acc)
        # (the lone strand's mlp_fc1_wgrad runs as two halves: counted at its first)
        assert sorted((o["strand"], o["layer"], o["node"], o["part"]) for o in prog["ops"]) == \
            sorted((o["strand"], o["layer"], o["node"], o["part"]) for o in rel["ops"])
    # with only L + 1 slots the deferral cannot release the slot in time
    with pytest.raises(Exception):
        lower(LlamaShape(**base), tp, _plan(LlamaShape(**base), tp), "si_deferred")


def test_deferred_wgrads_with_measured_tp8_profile():
    """With the measured B200 TP=8 profile the wide-caps plan ends the backward
    layer with ag0_bwd_rs, attn_proj_wgrad, qkv_wgrad, ln0_bwd: mode 4 issues
    qkv_wgrad right before the forward strand's bda1 (waiting for rs1) and
    attn_proj_wgrad after the next layer's leading collective."""
    prof = json.load(open(os.path.join(os.path.dirname(os.path.dirname(__file__)), "profiles",
                                       "r01_b200_profile_tp8_emulated.json")))
    shape = LlamaShape(**{**LLAMA3_8B.__dict__, "layers": 4, "micro_batches": 3, "slots": 6})
    caps = {"sequences": 16, "segments": 14, "candidates": 200000}
    plan = planner.lib().search_si_plan(shape.planner_model(), {"tp": 8, "sp": True}, B200_CLUSTER, prof,
                                        caps=caps, parallel=True)["plan_json"]
    prog = lower(shape, 8, plan, "si_deferred", profile_json=json.dumps(prof))
    check_program(prog, shape, 3, strict_order=False)
    acc = lambda n, L, l, s: _dense_access(n, 8, L, l, s)  # noqa: E731
    check_buffer_hazards(prog, shape.layers, acc)
    rel = lower(shape, 8, plan, "si_relaxed", profile_json=json.dumps(prof))
    assert observed_writers(prog, shape.layers, acc) == observed_writers(rel, shape.layers, acc)
    pos = {(o["strand"], o["layer"], o["node"]): i for i, o in enumerate(prog["ops"])}
    late = [k for k in pos if k[2] in (32, 36) and (k[0], k[1] - 1, 21) in pos and
            pos[k] > pos[(k[0], k[1] - 1, 21)]]
    # attn_proj_wgrad crosses into the next pair (2 SI blocks, all but each block's
    # last pair); qkv_wgrad stays in its pair, right before the forward strand's bda1
    assert len([k for k in late if k[2] == 32]) >= 2 * (shape.layers - 1)
    fwd_bda1 = [i for i, o in enumerate(prog["ops"]) if o["node"] == 14]
    assert any(prog["ops"][i - 1]["node"] == 36 for i in fwd_bda1)


def test_deferred_wgrads_single_step_plan():
    """A one-step plan (the whole layer pair in one step): the deferred
    gradients must still be issued before the next layer overwrites dqkv /
    dx1_full (the case the first GPU run of mode 4 caught)."""
    from tests.test_model_gpu import B200, _tiny
    shape = LlamaShape(**{**_tiny(mb=2, layers=2, nkv=4).__dict__, "slots": 4})
    plan = planner.lib().search_si_plan(shape.planner_model(), {"tp": 2, "sp": True}, B200,
                                        {"archetype": "pcie_a40"})["plan_json"]
    acc = lambda n, L, l, s: _dense_access(n, 2, L, l, s)  # noqa: E731
    prog, rel = lower(shape, 2, plan, "si_deferred"), lower(shape, 2, plan, "si_relaxed")
    check_buffer_hazards(prog, shape.layers, acc)
    assert observed_writers(prog, shape.layers, acc) == observed_writers(rel, shape.layers, acc)


def test_deferred_wgrads_issue_each_node_once():
    """Mode 4 with split deferral: a plan whose backward strand has trailing
    backward-only steps and places qkv_wgrad (36) after ag0_bwd_rs (37).
    qkv_wgrad is issued early, before the forward strand's bda1. A later step
    must not issue it again (qkv_wgrad accumulates, so a second issue would
    double dWqkv silently). Every (strand, layer, node) appears exactly once."""
    from collections import Counter
    shape = LlamaShape(**{**TINY.__dict__, "micro_batches": 2, "n_kv_heads": 2, "slots": TINY.layers + 2})
    plan = json.loads(_plan(shape, 2))
    plan.update(bwd_seq=[20, 21, 22, 26, 24, 25, 27, 23, 28, 29, 30, 31, 34, 35, 37, 32, 36, 38],
                fwd_cuts=[], bwd_cuts=[15],
                steps=[{"fwd_seg": 1, "bwd_seg": 1}, {"fwd_seg": None, "bwd_seg": 2}])
    plan_json = json.dumps(plan)
    prog = lower(shape, 2, plan_json, "si_deferred")
    rel = lower(shape, 2, plan_json, "si_relaxed")
    cnt = Counter((o["strand"], o["layer"], o["node"], o["part"]) for o in prog["ops"] if o["node"] != 100)
    assert max(cnt.values()) == 1, [k for k, v in cnt.items() if v > 1]
    # mlp_fc1_wgrad of the lone last strand runs as its gate half and its up half
    halves = Counter((k[0], k[1]) for k in cnt if k[2] == 26 and k[3] >= 0)
    assert all(v == 2 for v in halves.values())
    assert sorted(cnt) == sorted((o["strand"], o["layer"], o["node"], o["part"]) for o in rel["ops"]
                                 if o["node"] != 100)
    check_program(prog, shape, 2, strict_order=False)
    acc = lambda n, L, l, s: _dense_access(n, 2, L, l, s)  # noqa: E731
    check_buffer_hazards(prog, shape.layers, acc)
    assert observed_writers(prog, shape.layers, acc) == observed_writers(rel, shape.layers, acc)


@pytest.mark.parametrize("ep", [1, 2, 4])
def test_moe_deferred_lone_strand(ep):
    """Mode 4 with moe_ep: the lone last backward strand issues each layer's
    attention weight gradients (attn_proj_wgrad 34, qkv_wgrad 38) under the
    next layer's a2a_combine_bwd (EP > 1); hazard-free, every read sees the
    write it sees in the relaxed program, the same ops."""
    from paper_2411_15871_b200.runtime import TINY_MOE
    mb = 3
    shape = LlamaShape(**{**TINY_MOE.__dict__, "micro_batches": mb, "slots": TINY_MOE.layers + 2})
    acc = lambda n, L, l, s: _moe_access(n, ep, L, l, s)  # noqa: E731
    for arch in ("nvlink_h100", "pcie_a40"):
        plan = planner.lib().search_si_plan(shape.planner_model(), {"tp": 1, "ep": ep, "dp": ep}, B200_CLUSTER,
                                            {"archetype": arch})["plan_json"]
        prog, rel = lower(shape, ep, plan, "si_deferred"), lower(shape, ep, plan, "si_relaxed")
        check_buffer_hazards(prog, shape.layers, acc)
        assert observed_writers(prog, shape.layers, acc) == observed_writers(rel, shape.layers, acc)
        key = lambda o: (o["strand"], o["layer"], o["node"])  # noqa: E731
        assert sorted(map(key, prog["ops"])) == sorted(map(key, rel["ops"]))
        pos = {key(o): i for i, o in enumerate(prog["ops"])}
        s = mb - 1
        for l in range(1, shape.layers):
            after = pos[(s, l, 34)] > pos[(s, l - 1, 22)] if ep > 1 else pos[(s, l, 34)] < pos[(s, l - 1, 20)]
            assert after, (l, ep)

"""CPU: the numpy layer oracle (oracle/layer_oracle.py) against torch autograd
on the same fp32 math, so the hand-written backward of the oracle is itself
checked. Also checks the bf16 rounding helper and TP-partition invariance."""
import numpy as np
import pytest
import torch

from oracle.layer_oracle import LlamaTPOracle, bf16_round, from_bf16_bits, to_bf16_bits


def test_bf16_round_matches_torch():
    x = np.random.default_rng(0).standard_normal(10000).astype(np.float32) * 3
    x[:5] = [0.0, -0.0, 1e-40, 65504.0, -3.4e38]
    ours = bf16_round(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    assert np.array_equal(ours, ref)
    assert np.array_equal(from_bf16_bits(to_bf16_bits(x)), ref)


def _torch_model(o: LlamaTPOracle, x, r):
    """Straight fp32 torch autograd of the same layer stack (no TP, no rounding)."""
    S, D = o.S, o.D
    P = [{k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in p.items()}
         for p in o.params]
    cos = torch.tensor(o.cos, dtype=torch.float64)[:, None, :]
    sin = torch.tensor(o.sin, dtype=torch.float64)[:, None, :]

    def rope(t):
        a, b = t[..., :D // 2], t[..., D // 2:]
        return torch.cat([a * cos - b * sin, b * cos + a * sin], -1)

    def rms(t, g):
        return t * torch.rsqrt(t.pow(2).mean(-1, keepdim=True) + o.eps) * g

    h = torch.tensor(x, dtype=torch.float64, requires_grad=True)
    x0 = h
    mask = torch.ones(S, S, dtype=torch.bool).triu(1)
    for p in P:
        ln0 = rms(h, p["g0"])
        q = rope((ln0 @ p["wq"].T).view(S, o.nq, D))
        k = rope((ln0 @ p["wk"].T).view(S, o.nkv, D))
        v = (ln0 @ p["wv"].T).view(S, o.nkv, D)
        grp = o.nq // o.nkv
        k, v = k.repeat_interleave(grp, 1), v.repeat_interleave(grp, 1)
        s = torch.einsum("qhd,khd->hqk", q, k) * float(o.scale)
        s = s.masked_fill(mask, float("-inf"))
        att = torch.einsum("hqk,khd->qhd", torch.softmax(s, -1), v).reshape(S, -1)
        x1 = h + att @ p["wo"].T
        ln1 = rms(x1, p["g1"])
        mlp = (torch.nn.functional.silu(ln1 @ p["wg"].T) * (ln1 @ p["wu"].T)) @ p["wd"].T
        h = x1 + mlp
    loss = (h * torch.tensor(r, dtype=torch.float64)).sum()
    loss.backward()
    return loss.item(), x0.grad.numpy(), [{k: v.grad.numpy() for k, v in p.items()} for p in P]


@pytest.mark.parametrize("nq,nkv", [(4, 2), (4, 4)])
def test_oracle_backward_matches_autograd(nq, nkv):
    o = LlamaTPOracle(hidden=64, ffn=96, n_heads=nq, n_kv_heads=nkv, head_dim=16, layers=2, seq=24,
                      bf16=False, seed=3, init_std=0.2)
    rng = np.random.default_rng(1)
    x = rng.standard_normal((24, 64)).astype(np.float32)
    r = rng.standard_normal((24, 64)).astype(np.float32)
    loss, _, dx, grads = o.run(x, r)
    tl, tdx, tg = _torch_model(o, x, r)
    assert abs(loss - tl) < 1e-3 * max(1.0, abs(tl))
    assert np.abs(dx - tdx).max() < 1e-3 * np.abs(tdx).max()
    for l in range(2):
        for k in tg[l]:
            err = np.abs(grads[l][k] - tg[l][k]).max() / max(1e-12, np.abs(tg[l][k]).max())
            assert err < 2e-3, (l, k, err)


@pytest.mark.parametrize("tp", [2, 4])
def test_tp_partition_invariance(tp):
    """Without rounding, TP partitioning must not change the math."""
    kw = dict(hidden=64, ffn=128, n_heads=4, n_kv_heads=4, head_dim=16, layers=2, seq=16, bf16=False,
              seed=9, init_std=0.2)
    a, b = LlamaTPOracle(tp=1, **kw), LlamaTPOracle(tp=tp, **kw)
    rng = np.random.default_rng(2)
    x = rng.standard_normal((16, 64)).astype(np.float32)
    r = rng.standard_normal((16, 64)).astype(np.float32)
    la, ya, dxa, ga = a.run(x, r)
    lb, yb, dxb, gb = b.run(x, r)
    assert np.allclose(ya, yb, atol=1e-4) and np.allclose(dxa, dxb, atol=1e-4)
    for k in ga[0]:
        assert np.allclose(ga[0][k], gb[0][k], atol=1e-3)
    sh = b.shard(0, 1)
    assert sh["wqkv"].shape == ((4 // tp + 2 * 4 // tp) * 16, 64)


def _torch_moe(o, x, r):
    """fp64 torch autograd of the MoE layer stack with the oracle's routing
    decisions (top-k ids and capacity slots) held fixed, as they are
    non-differentiable; weights flow through softmax and the renormalisation."""
    from oracle.layer_oracle import MoEOracle  # noqa: F401
    S, D = o.S, o.D
    P = [{k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in p.items()} for p in o.params]
    cos = torch.tensor(o.cos, dtype=torch.float64)[:, None, :]
    sin = torch.tensor(o.sin, dtype=torch.float64)[:, None, :]

    def rope(t):
        a, b = t[..., :D // 2], t[..., D // 2:]
        return torch.cat([a * cos - b * sin, b * cos + a * sin], -1)

    def rms(t, g):
        return t * torch.rsqrt(t.pow(2).mean(-1, keepdim=True) + o.eps) * g

    h = torch.tensor(x, dtype=torch.float64, requires_grad=True)
    x0 = h
    mask = torch.ones(S, S, dtype=torch.bool).triu(1)
    for p in P:
        ln0 = rms(h, p["g0"])
        q = rope((ln0 @ p["wq"].T).view(S, o.nq, D))
        k = rope((ln0 @ p["wk"].T).view(S, o.nkv, D))
        v = (ln0 @ p["wv"].T).view(S, o.nkv, D)
        grp = o.nq // o.nkv
        k, v = k.repeat_interleave(grp, 1), v.repeat_interleave(grp, 1)
        s = torch.einsum("qhd,khd->hqk", q, k) * float(o.scale)
        s = s.masked_fill(mask, float("-inf"))
        att = torch.einsum("hqk,khd->qhd", torch.softmax(s, -1), v).reshape(S, -1)
        x1 = h + att @ p["wo"].T
        ln1 = rms(x1, p["g1"])
        probs = torch.softmax(ln1 @ p["wr"].T, -1)
        _, ids, _, slot = o.route(ln1.detach().numpy().astype(np.float32), p["wr"].detach().numpy())
        ids_t = torch.tensor(ids)
        top = probs.gather(1, ids_t)
        w = top / top.sum(1, keepdim=True)
        moe = torch.zeros_like(ln1)
        for t in range(S):
            for kk in range(o.K):
                if slot[t, kk] < 0:
                    continue
                e = int(ids[t, kk])
                xe = ln1[t]
                y = (torch.nn.functional.silu(p["w1g"][e] @ xe) * (p["w1u"][e] @ xe)) @ p["w2"][e].T
                moe = moe.index_add(0, torch.tensor([t]), (w[t, kk] * y)[None])
        h = x1 + moe
    loss = (h * torch.tensor(r, dtype=torch.float64)).sum()
    loss.backward()
    return loss.item(), x0.grad.numpy(), [{k: v.grad.numpy() for k, v in p.items()} for p in P]


@pytest.mark.parametrize("capacity", [16, 6])  # 6: some assignments dropped
def test_moe_oracle_backward_matches_autograd(capacity):
    from oracle.layer_oracle import MoEOracle
    o = MoEOracle(hidden=64, ffn=48, n_heads=4, n_kv_heads=2, head_dim=16, layers=1, seq=16, experts=4,
                  topk=2, capacity=capacity, bf16=False, seed=2, init_std=0.3)
    rng = np.random.default_rng(5)
    x = rng.standard_normal((16, 64)).astype(np.float32)
    r = rng.standard_normal((16, 64)).astype(np.float32)
    loss, _, dx, grads = o.run(x, r)
    _, cache = o.layer_fwd(0, x)
    assert (cache["slot"] < 0).any() == (capacity == 6)  # the small capacity drops assignments
    tl, tdx, tg = _torch_moe(o, x, r)
    assert abs(loss - tl) < 1e-3 * max(1.0, abs(tl))
    assert np.abs(dx - tdx).max() < 1e-3 * np.abs(tdx).max()
    for k in tg[0]:
        err = np.abs(grads[0][k] - tg[0][k]).max() / max(1e-12, np.abs(tg[0][k]).max())
        assert err < 2e-3, (k, err)


# --------------------------------------------------------------------------- pinned to transformers' Llama

def _hf_golden():
    import importlib.util
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("make_hf_llama_golden",
                                                  os.path.join(root, "tests", "golden", "make_hf_llama_golden.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod, np.load(os.path.join(root, "tests", "golden", "hf_llama_layers.npz"))


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


@pytest.mark.parametrize("case", ["tiny_d64", "gqa_d128"])
def test_oracle_matches_transformers_llama_golden(case):
    """The layer oracle (fp32, bf16 rounding off) against golden vectors from
    HuggingFace transformers' LlamaDecoderLayer in fp64 (committed fixture,
    tests/golden/make_hf_llama_golden.py): output, input gradient, and every
    weight gradient's norm and 64 random projections. Tolerance 2e-5 relative
    (fp32 vs fp64 arithmetic)."""
    gen, gold = _hf_golden()
    c = gen.CASES[case]
    orc = gen.oracle_for(c)
    x, r = gen.inputs_for(c)
    _, y, dx, grads = orc.run(x, r)
    flat = {f"{l}.{k}": g for l, gl in enumerate(grads) for k, g in gl.items()}
    mine = gen.summarise(y, dx, flat, c["seed"])
    assert _rel(mine["y"], gold[f"{case}/y"]) < 2e-5
    assert _rel(mine["dx"], gold[f"{case}/dx"]) < 2e-5
    for k in flat:
        assert _rel(mine[f"g.{k}.norm"], gold[f"{case}/g.{k}.norm"]) < 2e-5, k
        assert _rel(mine[f"g.{k}.proj"], gold[f"{case}/g.{k}.proj"]) < 2e-5, k


def test_transformers_llama_live_matches_fixture():
    """Regenerate the HF vectors live (when transformers is importable) and
    compare them to the committed fixture: the fixture is what the script makes."""
    pytest.importorskip("transformers")
    gen, gold = _hf_golden()
    c = gen.CASES["tiny_d64"]
    y, dx, grads = gen.hf_run(c)
    live = gen.summarise(y, dx, grads, c["seed"])
    for k, v in live.items():
        assert _rel(v, gold[f"tiny_d64/{k}"]) < 1e-6, k

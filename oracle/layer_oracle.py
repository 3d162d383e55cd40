"""CPU numerics oracle for the Llama TP+SP layer (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module; the product path never does.

The reference (weft) has no layer math at all ("Oracle for layer
numerics: None in the reference ... parity unpinned"), and the paper's math
lived in Megatron-LM, which is not in /root/reference. This file is therefore
OUR restatement of standard Llama semantics — RMSNorm, half-split RoPE, causal
GQA softmax attention, SwiGLU MLP, residuals — under the Megatron TP+SP
partitioning implied by the reference's layer DAG (node order, names and
granularity: reference proj/src/op_model.cpp:79-119):

  forward  ln0 -> ag0 -> qkv -> attn -> attn_proj -> rs0 -> bda0 -> ln1 -> ag1
           -> {mlp_gate, mlp_up} -> mlp_down -> rs1 -> bda1
  backward the 18-node mirror (bda1_bwd ... ln0_bwd)

The reference holds no golden vectors for this math, so the oracle is pinned
to a third-party Llama implementation instead: golden vectors from
HuggingFace transformers 5.5.0 LlamaDecoderLayer (fp64, eager attention;
tests/golden/make_hf_llama_golden.py -> tests/golden/hf_llama_layers.npz) for
the output, the input gradient and every weight gradient of 2-layer stacks at
head_dim 64 and 128 agree with this file within 2e-5 (fp32 vs fp64); its
hand-written backward is also checked against torch autograd
(tests/test_layer_oracle.py).

Arithmetic is numpy float32 (float64 where asked). With `bf16=True` every
value the GPU stores in bf16 is rounded to bf16 here at the same point
(round-to-nearest-even), row-parallel partial sums are rounded per TP rank and
summed in rank order (the ReduceScatter), so GPU-vs-oracle differences reduce
to fp32 summation order.
"""
from __future__ import annotations

import numpy as np

# --------------------------------------------------------------------------- bf16


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bfloat16 (ties to even), as float32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    out = r.astype(np.uint32).view(np.float32)
    return np.where(np.isnan(x), x, out).astype(np.float32)


def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """float32 -> uint16 bf16 bit patterns (after rounding)."""
    return (bf16_round(x).view(np.uint32) >> 16).astype(np.uint16)


def from_bf16_bits(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)


class Numerics:
    def __init__(self, bf16: bool = True, dtype=np.float32):
        self.bf16 = bf16
        self.dt = dtype

    def rb(self, x):
        return bf16_round(x) if self.bf16 else x.astype(self.dt)


# --------------------------------------------------------------------------- ops


def rmsnorm_fwd(x, g, eps, nm: Numerics):
    rstd = 1.0 / np.sqrt((x.astype(np.float64) ** 2).mean(-1) + eps)
    rstd = rstd.astype(np.float32)
    y = nm.rb(x * rstd[:, None] * g[None, :])
    return y, rstd


def rmsnorm_bwd(x, g, rstd, dy):
    xh = x * rstd[:, None]
    dxh = dy * g[None, :]
    dot = (dxh * xh).mean(-1, keepdims=True)
    dx = rstd[:, None] * (dxh - xh * dot)
    dg = (dy * xh).sum(0)
    return dx.astype(np.float32), dg.astype(np.float32)


def rope_tables(seq, head_dim, theta):
    i = np.arange(head_dim // 2, dtype=np.float64)
    inv = np.exp(-np.log(theta) * (2.0 * i) / head_dim)
    ang = np.arange(seq, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


def rope(x, cos, sin, inverse=False):
    """x: [S, heads, D]; half-split rotation (pair i with i + D/2)."""
    half = x.shape[-1] // 2
    a, b = x[..., :half], x[..., half:]
    s = -sin if inverse else sin
    c = cos[:, None, :]
    s = s[:, None, :]
    return np.concatenate([a * c - b * s, b * c + a * s], axis=-1).astype(np.float32)


def attention_fwd(q, k, v, scale, nm: Numerics):
    """q [S, nq, D], k/v [S, nkv, D]; causal GQA. Returns o [S, nq, D], lse [nq, S]."""
    S, nq, D = q.shape
    nkv = k.shape[1]
    grp = nq // nkv
    o = np.empty_like(q)
    lse = np.empty((nq, S), np.float32)
    mask = np.triu(np.ones((S, S), bool), 1)
    for h in range(nq):
        kh, vh = k[:, h // grp], v[:, h // grp]
        s = (q[:, h] @ kh.T) * scale
        s[mask] = -np.inf
        m = s.max(-1, keepdims=True)
        p = np.exp(s - m)
        l = p.sum(-1, keepdims=True)
        lse[h] = (m + np.log(l))[:, 0]
        o[:, h] = (p / l) @ vh
    return nm.rb(o), lse


def attention_bwd(q, k, v, o, lse, do, scale):
    S, nq, D = q.shape
    nkv = k.shape[1]
    grp = nq // nkv
    dq = np.zeros_like(q)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    mask = np.triu(np.ones((S, S), bool), 1)
    for h in range(nq):
        kh, vh = k[:, h // grp], v[:, h // grp]
        s = (q[:, h] @ kh.T) * scale
        p = np.exp(s - lse[h][:, None])
        p[mask] = 0.0
        dvec = (do[:, h] * o[:, h]).sum(-1, keepdims=True)
        dp = do[:, h] @ vh.T
        ds = p * (dp - dvec)
        dq[:, h] = scale * (ds @ kh)
        dk[:, h // grp] += scale * (ds.T @ q[:, h])
        dv[:, h // grp] += p.T @ do[:, h]
    return dq, dk, dv


def silu(x):
    return x / (1.0 + np.exp(-x))


# --------------------------------------------------------------------------- layer


class LlamaTPOracle:
    """One Llama layer stack with explicit Megatron TP+SP partitioning.

    Full (unsharded) parameters per layer: wq [nq*D, H], wk, wv [nkv*D, H],
    wo [H, nq*D], wg, wu [F, H], wd [H, F], g0, g1 [H]. `shard(layer, r)`
    returns rank r's packed qkv shard and its wo/wg/wu/wd slices exactly as
    the GPU model stores them.
    """

    def __init__(self, hidden, ffn, n_heads, n_kv_heads, head_dim, layers, seq, tp=1,
                 theta=10000.0, eps=1e-5, bf16=True, seed=0, init_std=0.02):
        self.H, self.F, self.nq, self.nkv, self.D = hidden, ffn, n_heads, n_kv_heads, head_dim
        self.L, self.S, self.tp, self.theta, self.eps = layers, seq, tp, theta, eps
        self.nm = Numerics(bf16)
        self.scale = np.float32(1.0 / np.sqrt(head_dim))
        self.cos, self.sin = rope_tables(seq, head_dim, theta)
        rng = np.random.default_rng(seed)
        H, F, D = hidden, ffn, head_dim

        def w(*shape):
            return bf16_round(rng.standard_normal(shape, dtype=np.float32) * init_std)

        self.params = []
        for _ in range(layers):
            self.params.append({
                "wq": w(n_heads * D, H), "wk": w(n_kv_heads * D, H), "wv": w(n_kv_heads * D, H),
                "wo": w(H, n_heads * D), "wg": w(F, H), "wu": w(F, H), "wd": w(H, F),
                "g0": bf16_round(1.0 + 0.1 * rng.standard_normal(H, dtype=np.float32)),
                "g1": bf16_round(1.0 + 0.1 * rng.standard_normal(H, dtype=np.float32)),
            })

    # ---- TP shards as stored by the GPU model (csrc/runtime/model.cpp)
    def shard(self, layer, r):
        p, tp, D = self.params[layer], self.tp, self.D
        nq_l, nkv_l, F_l = self.nq // tp, self.nkv // tp, self.F // tp
        q = p["wq"][r * nq_l * D:(r + 1) * nq_l * D]
        k = p["wk"][r * nkv_l * D:(r + 1) * nkv_l * D]
        v = p["wv"][r * nkv_l * D:(r + 1) * nkv_l * D]
        return {
            "wqkv": np.concatenate([q, k, v], 0),
            "wo": np.ascontiguousarray(p["wo"][:, r * nq_l * D:(r + 1) * nq_l * D]),
            "wg": p["wg"][r * F_l:(r + 1) * F_l], "wu": p["wu"][r * F_l:(r + 1) * F_l],
            "wd": np.ascontiguousarray(p["wd"][:, r * F_l:(r + 1) * F_l]),
            "g0": p["g0"], "g1": p["g1"],
        }

    def _row_parallel(self, pieces):
        """Sum of per-rank bf16 partials in rank order (the ReduceScatter)."""
        acc = np.zeros_like(pieces[0], dtype=np.float32)
        for part in pieces:
            acc = acc + self.nm.rb(part)
        return self.nm.rb(acc)

    def layer_fwd(self, l, x):
        nm, p, tp, D = self.nm, self.params[l], self.tp, self.D
        S = self.S
        nq_l = self.nq // tp
        ln0, rstd0 = rmsnorm_fwd(x, p["g0"], self.eps, nm)                     # ln0 (+ ag0)
        q = nm.rb(ln0 @ p["wq"].T).reshape(S, self.nq, D)                      # qkv
        k = nm.rb(ln0 @ p["wk"].T).reshape(S, self.nkv, D)
        v = nm.rb(ln0 @ p["wv"].T).reshape(S, self.nkv, D)
        q = nm.rb(rope(q, self.cos, self.sin))
        k = nm.rb(rope(k, self.cos, self.sin))
        o, lse = attention_fwd(q, k, v, self.scale, nm)                        # attn
        of = o.reshape(S, -1)
        attn = self._row_parallel([of[:, r * nq_l * D:(r + 1) * nq_l * D]
                                   @ p["wo"][:, r * nq_l * D:(r + 1) * nq_l * D].T
                                   for r in range(tp)])                       # attn_proj + rs0
        x1 = nm.rb(x + attn)                                                   # bda0
        ln1, rstd1 = rmsnorm_fwd(x1, p["g1"], self.eps, nm)                   # ln1 (+ ag1)
        cache = dict(x=x, ln0=ln0, rstd0=rstd0, q=q, k=k, v=v, o=o, lse=lse, x1=x1, ln1=ln1,
                     rstd1=rstd1)
        y = nm.rb(x1 + self._mlp_fwd(l, ln1, cache))                           # bda1
        return y, cache

    def _mlp_fwd(self, l, ln1, cache):
        """Dense SwiGLU MLP of layer l (mlp_gate, mlp_up, mlp_down + rs1)."""
        nm, p, tp = self.nm, self.params[l], self.tp
        F_l = self.F // tp
        gate = nm.rb(ln1 @ p["wg"].T)                                          # mlp_gate
        up = nm.rb(ln1 @ p["wu"].T)                                            # mlp_up
        act = nm.rb(silu(gate) * up)                                           # mlp_down
        cache.update(gate=gate, up=up, act=act)
        return self._row_parallel([act[:, r * F_l:(r + 1) * F_l] @ p["wd"][:, r * F_l:(r + 1) * F_l].T
                                   for r in range(tp)])                       # + rs1

    def layer_bwd(self, l, c, dy, grads, dx_first_gate=True):
        nm, p, tp, D, S = self.nm, self.params[l], self.tp, self.D, self.S
        nq_l, nkv_l = self.nq // tp, self.nkv // tp
        g = grads[l]
        d_x1 = dy.copy()                                                       # bda1_bwd
        dln1 = self._mlp_bwd(l, c, dy, g, dx_first_gate)
        dxn, dg1 = rmsnorm_bwd(c["x1"], p["g1"], c["rstd1"], dln1)             # ln1_bwd
        d_x1 = nm.rb(dxn + d_x1)
        g["g1"] += dg1
        d_x = d_x1.copy()                                                      # bda0_bwd
        d_o = nm.rb(d_x1 @ p["wo"]).reshape(S, self.nq, D)                     # attn_proj_dgrad
        g["wo"] += d_x1.T @ c["o"].reshape(S, -1)                              # attn_proj_wgrad
        dq, dk, dv = attention_bwd(c["q"], c["k"], c["v"], c["o"], c["lse"], d_o, self.scale)
        dq = nm.rb(rope(nm.rb(dq), self.cos, self.sin, inverse=True))         # attn_bwd
        dk = nm.rb(rope(nm.rb(dk), self.cos, self.sin, inverse=True))
        dv = nm.rb(dv)
        dqf, dkf, dvf = dq.reshape(S, -1), dk.reshape(S, -1), dv.reshape(S, -1)
        parts = []
        for r in range(tp):                                                    # qkv_dgrad
            qs, ks = slice(r * nq_l * D, (r + 1) * nq_l * D), slice(r * nkv_l * D, (r + 1) * nkv_l * D)
            parts.append(dqf[:, qs] @ p["wq"][qs] + dkf[:, ks] @ p["wk"][ks] + dvf[:, ks] @ p["wv"][ks])
        g["wq"] += dqf.T @ c["ln0"]                                            # qkv_wgrad
        g["wk"] += dkf.T @ c["ln0"]
        g["wv"] += dvf.T @ c["ln0"]
        dln0 = self._row_parallel(parts)                                       # ag0_bwd_rs
        dxn, dg0 = rmsnorm_bwd(c["x"], p["g0"], c["rstd0"], dln0)              # ln0_bwd
        g["g0"] += dg0
        return nm.rb(dxn + d_x)

    def _mlp_bwd(self, l, c, dy, g, dx_first_gate=True):
        """Dense MLP backward of layer l: dL/d(ln1 output) after ag1_bwd_rs."""
        nm, p, tp = self.nm, self.params[l], self.tp
        F_l = self.F // tp
        d_act = nm.rb(dy @ p["wd"])                                            # mlp_down_dgrad
        sg = 1.0 / (1.0 + np.exp(-c["gate"]))
        d_up = nm.rb(d_act * c["gate"] * sg)
        d_gate = nm.rb(d_act * c["up"] * sg * (1.0 + c["gate"] * (1.0 - sg)))
        g["wd"] += dy.T @ c["act"]                                             # mlp_down_wgrad
        parts = []
        for r in range(tp):                                                    # gate/up dgrad
            sl = slice(r * F_l, (r + 1) * F_l)
            a = d_gate[:, sl] @ p["wg"][sl]
            b = d_up[:, sl] @ p["wu"][sl]
            first, second = (a, b) if dx_first_gate else (b, a)
            # the GPU accumulates the second partial with a bf16 TMA reduce-add
            parts.append(nm.rb(nm.rb(first) + nm.rb(second)))
        g["wg"] += d_gate.T @ c["ln1"]                                         # mlp_fc1_wgrad
        g["wu"] += d_up.T @ c["ln1"]
        return self._row_parallel(parts)                                       # ag1_bwd_rs

    def zero_grads(self):
        return [{k: np.zeros_like(v, dtype=np.float32) for k, v in p.items()} for p in self.params]

    def run(self, x, r_grad, grads=None, dx_first_gate=True):
        """Forward + backward of one micro-batch. loss = sum(y * r_grad).
        Returns (loss, y, dx, grads)."""
        grads = self.zero_grads() if grads is None else grads
        caches, h = [], x
        for l in range(self.L):
            h, cch = self.layer_fwd(l, h)
            caches.append(cch)
        y = h
        loss = float((y.astype(np.float64) * r_grad).sum())
        d = r_grad
        for l in reversed(range(self.L)):
            d = self.layer_bwd(l, caches[l], d, grads, dx_first_gate)
        return loss, y, d, grads


# --------------------------------------------------------------------------- MoE layer


class MoEOracle(LlamaTPOracle):
    """The reference's moe_ep layer (proj/src/op_model.cpp:121-169: router ->
    permute -> [a2a_dispatch] -> expert_fc1 -> expert_fc2 -> [a2a_combine] ->
    unpermute -> bda1) at TP = EP = 1, restated as the B200 model computes it
    (csrc/runtime/moe.cpp). The reference has no MoE math either; this is OUR
    definition (unpinned, cross-checked against torch autograd):

      router   logits = ln1 @ wr^T (fp32), p = softmax(logits), top-k experts by
               p (ties: lower expert id), weights w = p_top / sum(p_top)
      permute  each expert owns `capacity` slots, filled by its (token, k)
               assignments in (token, k) order; assignments beyond capacity
               are dropped (they contribute nothing)
      experts  SwiGLU FFN per expert: act = silu(xp w1g^T) * (xp w1u^T),
               y = act w2^T (empty slots are zero rows)
      unpermute moe[t] = sum_k w[t,k] y[slot(t,k)]  (k ascending, fp32, one rounding)
    """

    def __init__(self, hidden, ffn, n_heads, n_kv_heads, head_dim, layers, seq, experts, topk=2,
                 capacity=None, theta=10000.0, eps=1e-5, bf16=True, seed=0, init_std=0.02):
        super().__init__(hidden, ffn, n_heads, n_kv_heads, head_dim, layers, seq, tp=1, theta=theta,
                         eps=eps, bf16=bf16, seed=seed, init_std=init_std)
        self.E, self.K = experts, topk
        self.C = capacity if capacity is not None else moe_capacity(seq, experts, topk)
        self.forced, self.flips, self.tie_tol = [], 0, 1e-2
        rng = np.random.default_rng(seed + 7919)
        H, F = hidden, ffn

        def w(*shape):
            return bf16_round(rng.standard_normal(shape, dtype=np.float32) * init_std)

        for p in self.params:
            for k in ("wg", "wu", "wd"):
                del p[k]
            p["wr"] = w(experts, H)
            p["w1g"] = w(experts, F, H)
            p["w1u"] = w(experts, F, H)
            p["w2"] = w(experts, H, F)

    def route(self, ln1, wr):
        """-> (probs [S,E] f32, ids [S,K], weights [S,K] f32, slot [S,K] (-1 dropped)).

        `self.forced` (a queue of [S,K] id arrays, one per route() call) replaces
        the top-k choice by the device's, for tokens where the two differ only
        by a near-tie (logit gap below `tie_tol` of the logits' spread): the
        device's ln1 differs from ours by bf16 rounding, which can flip such a
        token. Any other disagreement raises."""
        logits = ln1.astype(np.float32) @ wr.T.astype(np.float32)
        z = logits - logits.max(1, keepdims=True)
        e = np.exp(z)
        probs = (e / e.sum(1, keepdims=True)).astype(np.float32)
        ids = np.argsort(-probs, axis=1, kind="stable")[:, :self.K]
        if self.forced:
            fid = np.asarray(self.forced.pop(0), np.int64).reshape(ids.shape)
            spread = float(np.std(logits)) or 1.0
            for t in np.nonzero((np.sort(fid, 1) != np.sort(ids, 1)).any(1))[0]:
                kth = np.sort(logits[t])[::-1][self.K - 1]
                worst = min(logits[t, fid[t]])
                if kth - worst > self.tie_tol * spread:
                    raise AssertionError(f"token {t}: device routes to {fid[t]}, oracle to {ids[t]} "
                                         f"(logit gap {kth - worst:.3g} is not a near-tie)")
                self.flips += 1
            ids = fid
        top = np.take_along_axis(probs, ids, 1)
        wts = (top / top.sum(1, keepdims=True)).astype(np.float32)
        slot = np.full(ids.shape, -1, np.int64)
        fill = np.zeros(self.E, np.int64)
        for t in range(ids.shape[0]):
            for k in range(self.K):
                ex = ids[t, k]
                if fill[ex] < self.C:
                    slot[t, k] = ex * self.C + fill[ex]
                    fill[ex] += 1
        return probs, ids, wts, slot

    def _mlp_fwd(self, l, ln1, cache):
        nm, p, E, C, F = self.nm, self.params[l], self.E, self.C, self.F
        probs, ids, wts, slot = self.route(ln1, p["wr"])                         # router
        xp = np.zeros((E * C, self.H), np.float32)                              # permute
        for t, k in zip(*np.nonzero(slot >= 0)):
            xp[slot[t, k]] = ln1[t]
        gate = np.zeros((E * C, F), np.float32)
        up = np.zeros((E * C, F), np.float32)
        y = np.zeros((E * C, self.H), np.float32)
        for e in range(E):                                                      # expert_fc1
            rows = slice(e * C, (e + 1) * C)
            gate[rows] = nm.rb(xp[rows] @ p["w1g"][e].T)
            up[rows] = nm.rb(xp[rows] @ p["w1u"][e].T)
        act = nm.rb(silu(gate) * up)
        for e in range(E):                                                      # expert_fc2
            rows = slice(e * C, (e + 1) * C)
            y[rows] = nm.rb(act[rows] @ p["w2"][e].T)
        moe = np.zeros_like(ln1, dtype=np.float32)                              # unpermute
        for k in range(self.K):
            sk = slot[:, k]
            ok = sk >= 0
            moe[ok] += wts[ok, k:k + 1] * y[sk[ok]]
        cache.update(probs=probs, ids=ids, wts=wts, slot=slot, xp=xp, gate=gate, up=up, act=act, y=y)
        return nm.rb(moe)

    def _mlp_bwd(self, l, c, dy, g, dx_first_gate=True):
        nm, p, E, C, K = self.nm, self.params[l], self.E, self.C, self.K
        slot, wts, ids, probs = c["slot"], c["wts"], c["ids"], c["probs"]
        dys = np.zeros_like(c["y"])                                             # unpermute_bwd
        dw = np.zeros(wts.shape, np.float32)
        for t, k in zip(*np.nonzero(slot >= 0)):
            s_ = slot[t, k]
            dys[s_] = wts[t, k] * dy[t]
            dw[t, k] = float(np.dot(c["y"][s_].astype(np.float64), dy[t].astype(np.float64)))
        dys = nm.rb(dys)
        d_act = np.zeros_like(c["act"])
        for e in range(E):                                                      # expert_fc2_dgrad
            rows = slice(e * C, (e + 1) * C)
            d_act[rows] = nm.rb(dys[rows] @ p["w2"][e])
            g["w2"][e] += dys[rows].T @ c["act"][rows]                          # expert_fc2_wgrad
        sg = 1.0 / (1.0 + np.exp(-c["gate"]))
        d_up = nm.rb(d_act * c["gate"] * sg)
        d_gate = nm.rb(d_act * c["up"] * sg * (1.0 + c["gate"] * (1.0 - sg)))
        dxp = np.zeros_like(c["xp"])
        for e in range(E):                                                      # expert_fc1_dgrad
            rows = slice(e * C, (e + 1) * C)
            dxp[rows] = nm.rb(nm.rb(d_gate[rows] @ p["w1g"][e]) + nm.rb(d_up[rows] @ p["w1u"][e]))
            g["w1g"][e] += d_gate[rows].T @ c["xp"][rows]                       # expert_fc1_wgrad
            g["w1u"][e] += d_up[rows].T @ c["xp"][rows]
        dln1 = np.zeros((slot.shape[0], self.H), np.float32)                    # permute_bwd
        for k in range(K):
            sk = slot[:, k]
            ok = sk >= 0
            dln1[ok] += dxp[sk[ok]]
        dln1 = nm.rb(dln1)
        # router_bwd: through the top-k renormalisation and the softmax
        top = np.take_along_axis(probs, ids, 1)
        ssum = top.sum(1, keepdims=True)
        dtop = dw / ssum - (dw * top).sum(1, keepdims=True) / ssum ** 2
        dp = np.zeros_like(probs)
        np.put_along_axis(dp, ids, dtop.astype(np.float32), 1)
        dlogits = (probs * (dp - (probs * dp).sum(1, keepdims=True))).astype(np.float32)
        g["wr"] += dlogits.T @ c["ln1"]
        return nm.rb(dln1 + dlogits @ p["wr"])


def moe_capacity(tokens, experts, topk, factor=1.25, multiple=32):
    """Slots per expert: ceil(tokens * topk / experts * factor), rounded up to a multiple of `multiple`."""
    c = int(np.ceil(tokens * topk / experts * factor))
    return (c + multiple - 1) // multiple * multiple

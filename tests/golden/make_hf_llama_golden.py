"""Generate tests/golden/hf_llama_layers.npz: golden vectors for the layer
numerics oracle from a THIRD-PARTY Llama implementation (HuggingFace
transformers' LlamaDecoderLayer + LlamaRotaryEmbedding, eager attention, fp64).

The reference (weft) has no layer math; the paper's math lived in Megatron-LM,
which is not available here. transformers' Llama is the public definition the
oracle's semantics follow (RMSNorm, half-split RoPE, causal GQA softmax
attention, SwiGLU MLP, pre-norm residuals), so these vectors pin
oracle/layer_oracle.py to it: tests/test_layer_oracle.py checks the oracle
(bf16=False) against them, and, when transformers is importable, re-runs this
comparison live.

Cases (seeded; weights come from LlamaTPOracle(seed) so the test rebuilds them
without the fixture holding weights): the tiny config-1 shape (h256, 4/2 heads,
head_dim 64, theta 1e4) and a head_dim-128 GQA shape (h512, 8/2 heads, theta
5e5). Stored: the 2-layer output y, dL/dx for loss = sum(y * r), and per
weight gradient its norm plus 64 seeded random projections.

    python tests/golden/make_hf_llama_golden.py      (run from the repo root)
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.layer_oracle import LlamaTPOracle  # noqa: E402

CASES = {
    "tiny_d64": dict(hidden=256, ffn=768, n_heads=4, n_kv_heads=2, head_dim=64, layers=2, seq=128, theta=10000.0,
                     seed=11),
    "gqa_d128": dict(hidden=512, ffn=1024, n_heads=8, n_kv_heads=2, head_dim=128, layers=2, seq=96,
                     theta=500000.0, seed=12),
}
NPROBE = 64
HF_NAMES = {"wq": "self_attn.q_proj.weight", "wk": "self_attn.k_proj.weight", "wv": "self_attn.v_proj.weight",
            "wo": "self_attn.o_proj.weight", "wg": "mlp.gate_proj.weight", "wu": "mlp.up_proj.weight",
            "wd": "mlp.down_proj.weight", "g0": "input_layernorm.weight", "g1": "post_attention_layernorm.weight"}


def oracle_for(c):
    return LlamaTPOracle(c["hidden"], c["ffn"], c["n_heads"], c["n_kv_heads"], c["head_dim"], c["layers"], c["seq"],
                         tp=1, theta=c["theta"], bf16=False, seed=c["seed"], init_std=0.05)


def inputs_for(c):
    rng = np.random.default_rng(c["seed"] + 100)
    x = rng.standard_normal((c["seq"], c["hidden"])).astype(np.float32)
    r = rng.standard_normal((c["seq"], c["hidden"])).astype(np.float32)
    return x, r


def probes(shape, seed):
    return np.random.default_rng(seed).standard_normal((NPROBE, int(np.prod(shape))))


def hf_run(c):
    """2 LlamaDecoderLayers in fp64: (y, dx, {layer.name: grad})."""
    from transformers import LlamaConfig
    from transformers.models.llama import modeling_llama as ml
    cfg = LlamaConfig(hidden_size=c["hidden"], intermediate_size=c["ffn"], num_attention_heads=c["n_heads"],
                      num_key_value_heads=c["n_kv_heads"], head_dim=c["head_dim"], num_hidden_layers=c["layers"],
                      rope_theta=c["theta"], rms_norm_eps=1e-5, max_position_embeddings=c["seq"],
                      attention_bias=False, mlp_bias=False, hidden_act="silu")
    cfg._attn_implementation = "eager"
    orc = oracle_for(c)
    layers = []
    for l in range(c["layers"]):
        layer = ml.LlamaDecoderLayer(cfg, l).double()
        sd = {HF_NAMES[k]: torch.tensor(v, dtype=torch.float64) for k, v in orc.params[l].items()}
        layer.load_state_dict(sd)
        layers.append(layer)
    rot = ml.LlamaRotaryEmbedding(cfg)
    x, r = inputs_for(c)
    S = c["seq"]
    h = torch.tensor(x, dtype=torch.float64)[None].requires_grad_(True)
    pos = torch.arange(S)[None]
    cos, sin = rot(h, pos)
    mask = torch.full((S, S), float("-inf"), dtype=torch.float64).triu(1)[None, None]
    out = h
    for layer in layers:
        out = layer(out, attention_mask=mask, position_ids=pos, position_embeddings=(cos, sin))
        out = out[0] if isinstance(out, tuple) else out
    loss = (out[0] * torch.tensor(r, dtype=torch.float64)).sum()
    loss.backward()
    grads = {}
    for l, layer in enumerate(layers):
        for k, name in HF_NAMES.items():
            grads[f"{l}.{k}"] = dict(layer.named_parameters())[name].grad.numpy()
    return out[0].detach().numpy(), h.grad[0].numpy(), grads


def summarise(y, dx, grads, case_seed):
    d = {"y": y.astype(np.float32), "dx": dx.astype(np.float32)}
    for i, (k, g) in enumerate(sorted(grads.items())):
        d[f"g.{k}.norm"] = np.array(np.linalg.norm(g))
        d[f"g.{k}.proj"] = probes(g.shape, case_seed * 1000 + i) @ g.reshape(-1).astype(np.float64)
    return d


def main():
    out = {}
    for name, c in CASES.items():
        y, dx, grads = hf_run(c)
        for k, v in summarise(y, dx, grads, c["seed"]).items():
            out[f"{name}/{k}"] = v
    path = os.path.join(ROOT, "tests", "golden", "hf_llama_layers.npz")
    np.savez_compressed(path, **out)
    import transformers
    print(f"wrote {path} ({os.path.getsize(path)} bytes), transformers {transformers.__version__}")


if __name__ == "__main__":
    main()

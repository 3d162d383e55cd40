"""Planner parity corpus: the five BASELINE.json configs x the three synthetic
archetypes, cap variations, and seeded random measured-style tables (solo
entries keyed by node name, as the B200 profiler emits them)."""
from __future__ import annotations

import random

B200_CLUSTER = {"name": "b200_8", "gpus": 8, "per_node": 8, "peak_tflops": 2250.0,
                "local_bw_gbs": 900.0, "cross_bw_gbs": 50.0, "mem_gb": 180.0}

CONFIGS = {
    "c1_tiny_tp2": ({"name": "tiny", "family": "llama", "hidden": 256, "intermediate": 768,
                     "layers": 4, "seq_len": 128}, {"tp": 2, "dp": 4, "sp": True}),
    "c2_llama3_8b_tp8": ({"name": "llama3-8b", "family": "llama", "hidden": 4096,
                          "intermediate": 14336, "layers": 32, "seq_len": 4096},
                         {"tp": 8, "sp": True}),
    "c3_gpt3_13b_tp4": ({"name": "gpt3-13b", "family": "gpt", "hidden": 5120, "intermediate": 20480,
                         "layers": 40, "seq_len": 2048}, {"tp": 4, "dp": 2, "sp": True}),
    "c4_phi_moe_ep8": ({"name": "phi-3.5-moe", "family": "phi_moe", "hidden": 4096,
                        "intermediate": 6400, "layers": 32, "seq_len": 4096, "experts": 16,
                        "topk": 2}, {"tp": 1, "dp": 8, "ep": 8}),
    "c5_llama2_70b_tp4": ({"name": "llama2-70b", "family": "llama", "hidden": 8192,
                           "intermediate": 28672, "layers": 80, "seq_len": 8192},
                          {"tp": 4, "pp": 2, "sp": True}),
}

CLASSES = ["GEMM", "FlashAttention", "FlashAttentionBwd", "GroupGEMM", "FusedBDA", "LayerNorm",
           "Router", "Permute", "WeightGrad", "AllGather", "ReduceScatter", "AllToAll", "SendRecv"]

DENSE_NODES = [
    ("ln0", "LayerNorm"), ("ag0", "AllGather"), ("qkv", "GEMM"), ("attn", "FlashAttention"),
    ("attn_proj", "GEMM"), ("rs0", "ReduceScatter"), ("bda0", "FusedBDA"), ("ln1", "LayerNorm"),
    ("ag1", "AllGather"), ("mlp_gate", "GEMM"), ("mlp_up", "GEMM"), ("mlp_down", "GEMM"),
    ("rs1", "ReduceScatter"), ("bda1", "FusedBDA"), ("bda1_bwd", "FusedBDA"),
    ("rs1_bwd_ag", "AllGather"), ("mlp_down_dgrad", "GEMM"), ("mlp_down_wgrad", "WeightGrad"),
    ("mlp_gate_dgrad", "GEMM"), ("mlp_up_dgrad", "GEMM"), ("mlp_fc1_wgrad", "WeightGrad"),
    ("ag1_bwd_rs", "ReduceScatter"), ("ln1_bwd", "LayerNorm"), ("bda0_bwd", "FusedBDA"),
    ("rs0_bwd_ag", "AllGather"), ("attn_proj_dgrad", "GEMM"), ("attn_proj_wgrad", "WeightGrad"),
    ("attn_bwd", "FlashAttentionBwd"), ("qkv_dgrad", "GEMM"), ("qkv_wgrad", "WeightGrad"),
    ("ag0_bwd_rs", "ReduceScatter"), ("ln0_bwd", "LayerNorm"),
]


def random_profile(rng: random.Random, with_solo: bool = True, full_oef: bool = True) -> dict:
    oef = []
    for i, a in enumerate(CLASSES):
        for b in CLASSES[i:]:
            if full_oef or ((a in CLASSES[9:]) != (b in CLASSES[9:])):
                # quantised values make exact ties (and the tie-breaks) likely
                oef.append({"a": a, "b": b, "value": rng.choice([-0.05, 0.0, 0.25, 0.5, 0.8, 1.0,
                                                                  round(rng.uniform(-0.05, 1.05), 6)])})
    solo = []
    if with_solo:
        for name, cls in DENSE_NODES:
            t = rng.choice([5.0, 10.0, 20.0, round(rng.uniform(1.0, 200.0), 4)])
            solo.append({"class": cls, "shape": name, "t_us": t})
    return {"solo": solo, "oef": oef,
            "interference": {"slowdown_factor": rng.choice([0.0, 0.1, round(rng.uniform(0, 0.5), 4)]),
                             "launch_overhead_frac": rng.choice([0.0, 0.05, round(rng.uniform(0, 0.3), 4)])},
            "metadata": {"source": "random", "seed": str(rng.random())}}


def corpus_requests():
    for cname, (model, par) in CONFIGS.items():
        for arch in ("nvlink_h100", "nvlink_a800", "pcie_a40"):
            yield f"{cname}/{arch}", {"model": model, "parallelism": par, "cluster": B200_CLUSTER,
                                      "profile": {"archetype": arch},
                                      "metadata": {"config": cname, "archetype": arch}}
    model, par = CONFIGS["c2_llama3_8b_tp8"]
    for caps in ({"sequences": 64, "segments": 8, "candidates": 65536},
                 {"sequences": 4, "segments": 3, "candidates": 64},
                 {"sequences": 1, "segments": 1, "candidates": 1},
                 {"sequences": 16, "segments": 12, "candidates": 20000}):
        yield f"c2/caps{caps['sequences']}_{caps['segments']}_{caps['candidates']}", {
            "model": model, "parallelism": par, "cluster": B200_CLUSTER,
            "profile": {"archetype": "nvlink_h100"}, "caps": caps}
    yield "c2/barrier2.5", {"model": model, "parallelism": par, "cluster": B200_CLUSTER,
                            "profile": {"archetype": "nvlink_h100"}, "barrier_cost_us": 2.5}
    for tp in (1, 2, 4):
        yield f"llama3_8b_tp{tp}/h100", {"model": model, "parallelism": {"tp": tp, "sp": tp > 1},
                                        "cluster": B200_CLUSTER, "profile": {"archetype": "nvlink_h100"}}
    rng = random.Random(2411_15871)
    for k in range(24):
        cname = ["c1_tiny_tp2", "c2_llama3_8b_tp8", "c3_gpt3_13b_tp4", "c5_llama2_70b_tp4"][k % 4]
        m, p = CONFIGS[cname]
        prof = random_profile(rng, with_solo=k % 3 != 2, full_oef=k % 5 != 4)
        yield f"random{k}/{cname}", {"model": m, "parallelism": p, "cluster": B200_CLUSTER,
                                     "profile": prof, "barrier_cost_us": [0.0, 0.5, 3.0][k % 3]}

"""Parity of the L5/L6 planner modules (W-pipeline schedules, memory replay,
iteration-time estimate) with the reference.

  1. golden corpus (tests/golden/pipeline_corpus.json, generated from the
     reference by tests/golden/make_pipeline_golden.py): every output must be
     identical — trace JSON and CSV text byte for byte, doubles bit for bit;
  2. seeded random requests run live against oracle/_ref/libweft_ref.so;
  3. the reference's own Catch suites for these modules run against our library
     (test_planner_parity.py::test_reference_catch_suites_against_our_library).
"""
from __future__ import annotations

import json
import os
import random

import pytest

from paper_2411_15871_b200.planner import ConfigError, InfeasibleError, PlannerLib, lib
from tests.planner_corpus import B200_CLUSTER, CONFIGS, random_profile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libweft_ref.so")
with open(os.path.join(ROOT, "tests", "golden", "pipeline_corpus.json")) as f:
    GOLDEN = json.load(f)["cases"]


@pytest.fixture(scope="module")
def ref():
    if not os.path.exists(REF_LIB):
        pytest.skip("oracle/_ref not built (needs /root/reference + `make -C oracle`)")
    return PlannerLib(REF_LIB, "weft_ref_")


@pytest.mark.parametrize("case", GOLDEN, ids=[c["name"] for c in GOLDEN])
def test_golden(case):
    assert lib().call(case["fn"], case["request"]) == case["result"]


def test_w_schedule_p1_is_the_executor_block_order():
    """p = 1: F_1 | SI(F_2, B_1) | ... | SI(F_m, B_{m-1}) | B_m back to back —
    the block sequence the B200 executor lowers (executor.cpp)."""
    r = lib().pipeline("w_shape", 8, 1, f_us=1.0, b_us=2.0, si_us=3.0)
    rows = [line.split(",") for line in r["csv"].strip().splitlines()[1:]]
    kinds = [(k, f, b) for _, k, f, b, *_ in rows]
    assert kinds == [("F", "1", "")] + [("SI", str(i + 1), str(i)) for i in range(1, 8)] + [("B", "", "8")]
    assert r["violations"] == [] and r["bubble_ratio"] == 0.0
    assert r["makespan_us"] == 2 * 1.0 + 7 * 2 * 3.0 + 2 * 2.0  # p = 1: each visit spans two half-stages


def test_random_schedules_vs_reference_live(ref):
    rng = random.Random(5)
    for _ in range(60):
        disc = rng.choice(["w_shape", "one_f_one_b", "bidirectional"])
        m, p = rng.randint(1, 12), rng.randint(1, 6)
        durs = {k: rng.choice([1.0, 2.0, round(rng.uniform(0.1, 5.0), 5)]) for k in ("f_us", "b_us", "si_us")}
        req = {"schedule": dict(discipline=disc, m=m, p=p, **durs)}
        assert lib().call("pipeline_json", req) == ref.call("pipeline_json", req)
        mem = {"act_bytes_per_layer": rng.randint(0, 1 << 30), "state_bytes_per_layer": rng.randint(0, 1 << 30),
               "capacity_bytes": 1 << 40, "layers": 2 * p * rng.randint(1, 4)}
        mreq = dict(req, memory=mem)
        assert lib().call("memory_json", mreq) == ref.call("memory_json", mreq)


def test_random_estimates_vs_reference_live(ref):
    rng = random.Random(11)
    names = [n for n in CONFIGS if not n.startswith("c4")]
    for k in range(12):
        model, par = CONFIGS[names[k % len(names)]]
        req = {"model": model, "parallelism": par, "cluster": B200_CLUSTER, "profile": random_profile(rng),
               "source": ["megatron_baseline", "intra_batch", "wavelet_rr", "dhelix"][k % 4],
               "microbatches": rng.randint(1, 16), "caps": {"sequences": 6, "segments": 4, "candidates": 600}}
        assert lib().call("estimate_json", req) == ref.call("estimate_json", req)


def test_error_mapping_l5_l6():
    with pytest.raises(InfeasibleError):
        lib().pipeline("w_shape", 4, 3, fold_layers=16)  # 16 % (2*3) != 0
    with pytest.raises(ConfigError):
        lib().pipeline("zigzag", 4, 2)
    model, par = CONFIGS["c2_llama3_8b_tp8"]
    with pytest.raises(ConfigError):
        lib().estimate(model, par, B200_CLUSTER, {"archetype": "nvlink_h100"}, source="nope")

"""Planner parity: our drop-in weft planner vs the reference planner.

Three layers of evidence:
  1. golden corpus (tests/golden/planner_corpus.json, produced by the reference
     via oracle/_ref) — plan_to_json bytes, FNV-1a64, candidates_evaluated and
     the DAG tables must match exactly; runs anywhere;
  2. live differential tests against oracle/_ref/libweft_ref.so (segment
     costs, DP vs brute force, topological orders) on seeded random inputs;
  3. the reference's own Catch test suites compiled unmodified against our
     library (oracle/_ref/ours_suite) and against the reference itself.
Appendix A hashes of SURVEY.md are pinned explicitly.
"""
import json
import os
import random
import subprocess

import pytest

from paper_2411_15871_b200.planner import (ConfigError, MissingProfileEntry, PlannerLib, lib,
                                            parse_plan)
from tests.planner_corpus import B200_CLUSTER, CLASSES, CONFIGS, random_profile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden", "planner_corpus.json")
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libweft_ref.so")


def fnv1a64(s: str) -> str:
    h = 0xCBF29CE484222325
    for ch in s.encode():
        h = ((h ^ ch) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return "%016x" % h


with open(GOLDEN) as _f:
    CORPUS = json.load(_f)["cases"]


@pytest.fixture(scope="module")
def ref():
    if not os.path.exists(REF_LIB):
        pytest.skip("oracle/_ref not built (needs /root/reference + `make -C oracle`)")
    return PlannerLib(REF_LIB, "weft_ref_")


@pytest.mark.parametrize("case", CORPUS, ids=[c["name"] for c in CORPUS])
def test_golden_plan_bytes(case):
    r = lib().call("search_json", case["request"])
    assert r["plan_json"] == case["plan_json"]
    assert fnv1a64(r["plan_json"]) == case["fnv1a64"]
    assert r["candidates_evaluated"] == case["candidates_evaluated"]
    assert r["fwd"] == case["fwd"] and r["bwd"] == case["bwd"]


def test_golden_parallel_equals_serial():
    for case in CORPUS[:12]:
        req = dict(case["request"], parallel=True, threads=4)
        assert lib().call("search_json", req)["plan_json"] == case["plan_json"]


# hashes captured from the reference with nlohmann 3.11.3.
APPENDIX_A = {
    "c1_tiny_tp2/nvlink_h100": ("53d2893ee7a02ed3", 0.6835805298),
    "c1_tiny_tp2/nvlink_a800": ("081c2cebc32d5516", 0.6440496515),
    "c1_tiny_tp2/pcie_a40": ("86349098aac976a5", 0.6110691692),
    "c2_llama3_8b_tp8/nvlink_h100": ("2e9b59e92f903481", 791.8541166),
    "c2_llama3_8b_tp8/nvlink_a800": ("8510ef75d868fb78", 723.3928636),
    "c2_llama3_8b_tp8/pcie_a40": ("3d6c95af071216cf", 666.2758644),
}


@pytest.mark.parametrize("name", sorted(APPENDIX_A))
def test_appendix_a_hashes(name):
    case = next(c for c in CORPUS if c["name"] == name)
    req = dict(case["request"])
    req.pop("metadata", None)  # Appendix A plans carry empty metadata
    r = lib().call("search_json", req)
    h, total = APPENDIX_A[name]
    assert fnv1a64(r["plan_json"]) == h
    assert abs(r["total_us"] - total) < 1e-6 * max(1.0, total)


def test_config2_candidate_budget_quirk():
    # 128 + 15*128 + 128 + 15*121 = 3991 evaluated candidates.
    case = next(c for c in CORPUS if c["name"] == "c2_llama3_8b_tp8/nvlink_h100")
    assert case["candidates_evaluated"] == 3991
    plan = parse_plan(case["plan_json"])
    assert plan["bwd_seq"] == [20, 21, 22, 26, 24, 25, 27, 23, 28, 29, 30, 31, 34, 35, 37, 36, 32, 38]


def test_plan_parser_round_trip():
    for case in CORPUS:
        p = parse_plan(case["plan_json"])
        assert sum(len(s) for s in p["fwd_segments"]) == len(p["fwd_seq"])
    bad = json.loads(CORPUS[0]["plan_json"])
    bad["steps"] = bad["steps"][:-1]
    with pytest.raises(ConfigError):
        parse_plan(json.dumps(bad))


def _random_seg(rng, max_len):
    pool = ["GEMM", "FlashAttention", "WeightGrad", "LayerNorm", "AllGather", "ReduceScatter",
            "AllToAll", "SendRecv"]
    return [{"id": i, "class": rng.choice(pool), "name": f"t{i}",
             "duration_us": rng.choice([1.0, 2.0, round(rng.uniform(0.5, 10.0), 6)])}
            for i in range(rng.randint(0, max_len))]


def test_segment_pair_cost_vs_reference(ref):
    rng = random.Random(17)
    for trial in range(300):
        prof = random_profile(rng, with_solo=False)
        prof["solo"] = [{"class": "GEMM", "shape": "t1", "t_us": 3.5}] if trial % 4 == 0 else []
        a, b = _random_seg(rng, 7), _random_seg(rng, 9)
        assert lib().segment_pair_cost(a, b, prof) == ref.segment_pair_cost(a, b, prof)


def test_single_op_alone_is_its_solo_time():
    # reference test_overlap_profile.cpp:181-189 (empty side == solo sum) via the C ABI
    prof = random_profile(random.Random(0), with_solo=False)
    r = lib().segment_pair_cost([{"class": "GEMM", "duration_us": 10.0, "name": "x"}], [],
                                prof)
    assert r["p_us"] == 10.0


def test_dp_align_vs_brute_force_and_reference(ref):
    rng = random.Random(41)
    for trial in range(200):
        nf, nb = rng.randint(0, 7), rng.randint(0, 7)
        cost = [[0.0 if (i == 0 and j == 0) else rng.choice([1.0, 2.0, 3.0, round(rng.uniform(0.1, 9), 3)])
                 for j in range(nb + 1)] for i in range(nf + 1)]
        barrier = 2.5 if trial % 3 == 0 else 0.0
        ours = lib().dp_align(cost, barrier, brute_force=True)
        theirs = ref.dp_align(cost, barrier, brute_force=True)
        assert ours == theirs
        assert ours["dp"]["total_us"] == ours["brute_force"]["total_us"]


def test_topological_orders_vs_reference(ref):
    rng = random.Random(7)
    for trial in range(40):
        n = rng.randint(1, 8)
        edges = [[i, j] for i in range(n) for j in range(i + 1, n) if rng.random() < 0.3]
        dag = {"nodes": list(range(n)), "edges": edges}
        cap = rng.choice([1, 5, 64, 10000])
        assert lib().enumerate_topological_orders(dag, cap) == ref.enumerate_topological_orders(dag, cap)
    m, p = CONFIGS["c2_llama3_8b_tp8"]
    kw = dict(model=m, parallelism=p, cluster=B200_CLUSTER, profile={"archetype": "nvlink_h100"},
              **{"pass": "backward"})
    ours = lib().enumerate_topological_orders(cap=20000, **kw)
    assert len(ours) == 12544
    assert ours == ref.enumerate_topological_orders(cap=20000, **kw)


def test_random_tables_vs_reference_live(ref):
    rng = random.Random(99)
    for k in range(10):
        cname = list(CONFIGS)[k % 5]
        if cname.startswith("c4"):
            continue
        m, p = CONFIGS[cname]
        req = {"model": m, "parallelism": p, "cluster": B200_CLUSTER,
               "profile": random_profile(rng), "caps": {"sequences": 8, "segments": 5, "candidates": 1500}}
        assert lib().call("search_json", req)["plan_json"] == ref.call("search_json", req)["plan_json"]


def test_error_mapping():
    m, p = CONFIGS["c2_llama3_8b_tp8"]
    prof = {"solo": [], "oef": [{"a": "GEMM", "b": "GEMM", "value": 0.1}],
            "interference": {"slowdown_factor": 0.0, "launch_overhead_frac": 0.0}}
    with pytest.raises(MissingProfileEntry, match="no OEF entry for pair"):
        lib().search_si_plan(m, p, B200_CLUSTER, prof)
    with pytest.raises(ConfigError):
        lib().search_si_plan(m, {"tp": 1, "sp": True}, B200_CLUSTER, {"archetype": "nvlink_h100"})


def test_reference_catch_suites_against_our_library():
    """The reference's own tests (proj/tests/test_{op_model,overlap_profile,
    pairing_search,folding_pipeline,memory_sim,runner}.cpp), compiled
    unmodified against our planner: all 88 cases, as against the reference."""
    exe = os.path.join(ROOT, "oracle", "_ref", "ours_suite")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/ours_suite not built")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "cases=88 passed=88 failed=0" in out.stdout


def test_reference_catch_suites_against_reference():
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_suite")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/ref_suite not built")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert "cases=88 passed=88 failed=0" in out.stdout, out.stdout + out.stderr


def test_shipped_template_file_matches_builtin():
    with open(os.path.join(ROOT, "data", "dag_templates.json")) as f:
        assert json.loads(f.read()) == json.loads(lib().builtin_template_json())


SCENARIOS = [
    {"name": "llama25b-a40", "model": "llama-25B", "cluster": "a40_64",
     "parallelism": {"dp": 4, "tp": 8, "pp": 2, "sp": True}, "microbatches": 8,
     "profile": {"archetype": "pcie_a40"}, "caps": {"sequences": 8, "segments": 5, "candidates": 512}, "seed": 7},
    {"name": "c2-b200", "model": {"name": "llama3-8b", "family": "llama", "hidden": 4096, "intermediate": 14336,
                                  "layers": 32, "seq_len": 4096},
     "cluster": B200_CLUSTER, "parallelism": {"tp": 8, "sp": True}, "microbatches": 8,
     "profile": {"archetype": "nvlink_h100"}, "barrier_cost_us": 2.5, "parallel_search": True,
     "memory": {"capacity_bytes": 180 * 2 ** 30}},
    {"name": "c5-pp2", "model": {"name": "llama2-70b", "family": "llama", "hidden": 8192, "intermediate": 28672,
                                 "layers": 80, "seq_len": 8192},
     "cluster": B200_CLUSTER, "parallelism": {"tp": 4, "pp": 2, "sp": True}, "microbatches": 6,
     "profile": {"archetype": "nvlink_a800"}, "caps": {"sequences": 4, "segments": 4, "candidates": 256}},
    {"name": "phi-ep", "model": "phi-42B", "cluster": "a40_64", "parallelism": {"dp": 16, "pp": 4, "ep": 8},
     "microbatches": 8, "profile": {"archetype": "nvlink_h100"}, "caps": {"sequences": 4, "segments": 4, "candidates": 128}},
]


@pytest.mark.parametrize("sc", SCENARIOS, ids=[s["name"] for s in SCENARIOS])
def test_compare_report_byte_identical_to_reference(sc, ref):
    """compare_report (reference report.cpp:179-223): JSON and CSV reports and
    the config hash are byte-identical to the reference's on the same scenario."""
    a, b = lib().compare(sc), ref.compare(sc)
    assert a["config_hash"] == b["config_hash"]
    assert a["report_json"] == b["report_json"]
    assert a["report_csv"] == b["report_csv"]
    assert [r["plan_source"] for r in a["report"]["rows"]] == ["megatron_baseline", "intra_batch", "wavelet_rr",
                                                               "dhelix"]


def test_compare_report_schema_errors():
    with pytest.raises(ConfigError, match="typo_field"):
        lib().compare({**SCENARIOS[0], "typo_field": 1})


@pytest.mark.parametrize("par", [{"tp": 8, "sp": True}, {"tp": 4, "dp": 2, "sp": True}, {"tp": 2, "cp": 2, "dp": 2},
                                 {"dp": 8}, {"tp": 1, "ep": 8, "dp": 8}])
def test_comm_volume_equals_reference(par, ref):
    model = {"name": "phi", "family": "phi_moe", "hidden": 4096, "intermediate": 6400, "layers": 32,
             "seq_len": 3072, "experts": 16, "topk": 2} if par.get("ep", 1) > 1 else CONFIGS["c2_llama3_8b_tp8"][0]
    a = lib().comm_volume(model, par, B200_CLUSTER, 4096, 8)
    b = ref.comm_volume(model, par, B200_CLUSTER, 4096, 8)
    assert a == b

"""Generate tests/golden/pipeline_corpus.json from the REFERENCE planner: the
L5/L6 entry points (folding_pipeline.hpp, memory_sim.hpp, estimate.hpp).

Build container only (needs oracle/_ref/libweft_ref.so compiled from
/root/reference by oracle/Makefile). tests/test_pipeline_parity.py replays the
stored reference outputs against our planner anywhere, and additionally runs
seeded random requests live against oracle/_ref when it is present.

    python tests/golden/make_pipeline_golden.py
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2411_15871_b200.planner import PlannerLib  # noqa: E402
from tests.planner_corpus import B200_CLUSTER, CONFIGS  # noqa: E402


def pipeline_requests():
    for disc in ("w_shape", "one_f_one_b", "bidirectional"):
        for m, p in ((1, 1), (2, 1), (8, 1), (4, 2), (8, 2), (12, 4), (5, 3), (16, 8)):
            yield f"{disc}_m{m}_p{p}", {"schedule": {"discipline": disc, "m": m, "p": p, "f_us": 1.0,
                                                     "b_us": 2.0, "si_us": 2.6},
                                        "fold_layers": 16 * p}
    yield "w_uneven", {"schedule": {"discipline": "w_shape", "m": 7, "p": 3, "f_us": 0.37, "b_us": 0.91,
                                    "si_us": 1.13}}


def memory_requests():
    for disc in ("w_shape", "one_f_one_b", "bidirectional"):
        yield f"mem_{disc}", {"memory": {"act_bytes_per_layer": 1 << 20, "state_bytes_per_layer": 3 << 20,
                                         "capacity_bytes": 1 << 33, "layers": 16},
                              "schedule": {"discipline": disc, "m": 8, "p": 2, "f_us": 1.0, "b_us": 2.0,
                                           "si_us": 3.0}}
    for name in ("c2_llama3_8b_tp8", "c3_gpt3_13b_tp4", "c5_llama2_70b_tp4", "c4_phi_moe_ep8"):
        model, par = CONFIGS[name]
        par = dict(par, pp=par.get("pp", 1))
        for disc in ("w_shape", "one_f_one_b"):
            yield f"max_{name}_{disc}", {"memory": {"defaults": True, "capacity_bytes": 180 << 30},
                                         "model": model, "parallelism": par,
                                         "max_model": {"discipline": disc, "m": 8}}


def estimate_requests():
    for name, (model, par) in CONFIGS.items():
        for arch in ("nvlink_h100", "pcie_a40"):
            for src in ("megatron_baseline", "intra_batch", "wavelet_rr", "dhelix"):
                yield f"est_{name}_{arch}_{src}", {"model": model, "parallelism": par, "cluster": B200_CLUSTER,
                                                   "profile": {"archetype": arch}, "source": src,
                                                   "microbatches": 8}


def main() -> None:
    ref = PlannerLib(os.path.join(ROOT, "oracle", "_ref", "libweft_ref.so"), "weft_ref_")
    cases = []
    for fn, reqs in (("pipeline_json", pipeline_requests()), ("memory_json", memory_requests()),
                     ("estimate_json", estimate_requests())):
        for name, req in reqs:
            cases.append({"name": name, "fn": fn, "request": req, "result": ref.call(fn, req)})
    out = os.path.join(ROOT, "tests", "golden", "pipeline_corpus.json")
    with open(out, "w") as f:
        json.dump({"generator": "tests/golden/make_pipeline_golden.py",
                   "oracle": "reference weft planner (/root/reference/proj/src) via oracle/_ref",
                   "cases": cases}, f, indent=1, sort_keys=True)
    print(f"wrote {len(cases)} cases to {out}")


if __name__ == "__main__":
    main()

"""Generate tests/golden/planner_corpus.json from the REFERENCE planner.

Runs in the build container only (needs oracle/_ref/libweft_ref.so, i.e. the
reference sources compiled by oracle/Makefile from /root/reference). For every
request of the corpus it stores the reference's exact outputs: the plan_to_json
text (byte-for-byte), its FNV-1a64 hash, candidates_evaluated, and the DAG
node tables. tests/test_planner_parity.py replays the corpus against our planner
on any machine (including the GPU box, where /root/reference is absent).

    python tests/golden/make_planner_golden.py
"""
from __future__ import annotations

import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2411_15871_b200.planner import PlannerLib  # noqa: E402
from tests.planner_corpus import corpus_requests  # noqa: E402


def fnv1a64(s: str) -> str:
    h = 0xCBF29CE484222325
    for ch in s.encode():
        h = ((h ^ ch) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return "%016x" % h


def main() -> None:
    ref = PlannerLib(os.path.join(ROOT, "oracle", "_ref", "libweft_ref.so"), "weft_ref_")
    cases = []
    for name, req in corpus_requests():
        r = ref.call("search_json", req)
        cases.append({
            "name": name,
            "request": req,
            "plan_json": r["plan_json"],
            "fnv1a64": fnv1a64(r["plan_json"]),
            "candidates_evaluated": r["candidates_evaluated"],
            "fwd": r["fwd"],
            "bwd": r["bwd"],
        })
    out = os.path.join(ROOT, "tests", "golden", "planner_corpus.json")
    with open(out, "w") as f:
        json.dump({"generator": "tests/golden/make_planner_golden.py",
                   "oracle": "reference weft planner (/root/reference/proj/src) via oracle/_ref",
                   "cases": cases}, f, indent=1, sort_keys=True)
    print(f"wrote {len(cases)} cases to {out}")


if __name__ == "__main__":
    random.seed(0)
    main()

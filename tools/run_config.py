"""Run one emulated experiment of bench.py (emulated_tp_experiment) in its own
process: a BASELINE.json config slice (`c3`, `c4`, `c5`) or the Llama-3-8B
stack at a TP size (`llama3 --group 8`). Prints one JSON object as the last
line. bench.py runs each emulated experiment this way, under a timeout, so a
failure there cannot take the headline measurement with it."""
import argparse
import json
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=["c3", "c4", "c5", "llama3"])
    ap.add_argument("--group", type=int, default=0, help="TP / EP group size (default: the config's)")
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--micro-batches", type=int, default=4)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--nccl-ctas", type=int, default=16)
    ap.add_argument("--full", action="store_true")
    ap.add_argument("--overlap-ctas", type=int, default=None, help="GEMM SM cap under SI (0 = none)")
    ap.add_argument("--wide-caps", default=None, help="JSON caps for the wide plan search (default: bench.WIDE_CAPS)")
    a = ap.parse_args()
    import torch

    from paper_2411_15871_b200.runtime import GPT3_13B, LLAMA2_70B, LLAMA3_8B, PHI35_MOE
    base, group = {"c3": (GPT3_13B, 4), "c4": (PHI35_MOE, 8), "c5": (LLAMA2_70B, 4),
                   "llama3": (LLAMA3_8B, 8)}[a.config]
    group = a.group or group

    def timed(n, fn, st):
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(st)
        for _ in range(n):
            fn()
        e.record(st)
        torch.cuda.synchronize()
        return s.elapsed_time(e) / n

    if a.wide_caps:
        bench.WIDE_CAPS = json.loads(a.wide_caps)
    args = types.SimpleNamespace(nccl_ctas=a.nccl_ctas, steps=a.steps, layers=a.layers,
                                 micro_batches=a.micro_batches, overlap_ctas=a.overlap_ctas)
    r = bench.emulated_tp_experiment(args, group, timed, full=a.full, base_shape=base, layers=a.layers,
                                     micro_batches=a.micro_batches)
    print(json.dumps(r))


if __name__ == "__main__":
    main()

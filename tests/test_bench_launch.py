"""CPU: bench.py's launch contract. `--gpus N` without a torchrun
environment starts N ranks itself (torch.distributed.run on 127.0.0.1) that
form ONE group; checked with the gloo dry run (no GPU), as the driver's
N > 1 launch would form it over NCCL."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=300, env=env, cwd=ROOT)
    lines = [x for x in p.stdout.splitlines() if x.startswith("{")]
    return p.returncode, (json.loads(lines[-1]) if lines else None), p.stderr


def test_gpus_2_spawns_two_ranks_in_one_group():
    rc, line, err = _run(["--gpus", "2", "--dry-run"])
    assert rc == 0, err[-2000:]
    assert line == {"dry_run": True, "n_gpus": 2, "rank_sum": 1, "nccl_debug": "INFO"}


def test_gpus_1_runs_in_process():
    rc, line, err = _run(["--gpus", "1", "--dry-run"])
    assert rc == 0, err[-2000:]
    assert line["n_gpus"] == 1 and line["rank_sum"] == 0


def test_world_size_mismatch_is_an_error():
    env = {"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"}
    rc, line, err = _run(["--gpus", "4", "--steps", "1"], env)
    assert rc == 2 and line is None and "WORLD_SIZE=1" in err

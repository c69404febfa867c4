"""bench.py's launch contract on a box without enough GPUs (runs anywhere):
--gpus N outside torchrun re-launches N ranks, one per GPU, and refuses to
oversubscribe instead of silently timing one rank."""

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_refuses_more_gpus_than_visible():
    import torch
    n = torch.cuda.device_count() + 2  # >= 2: the spawn path
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("EBC_BENCH_SHARE_GPU", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--steps", "1"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 2, r.stdout + r.stderr
    assert f"--gpus {n} needs {n} GPUs" in r.stderr
    assert r.stdout.strip() == ""

"""bench.py --gpus N launcher (CPU, gloo): with no torchrun environment the
script re-launches itself under torch.distributed.run with N ranks, and the
line rank 0 prints carries the world the ranks actually formed."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*argv):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *argv], capture_output=True, text=True,
                       timeout=300, env=env, cwd=ROOT)
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    return p.returncode, [json.loads(ln) for ln in lines], p.stderr


@pytest.mark.parametrize("n", [1, 2])
def test_launcher_forms_n_ranks(n):
    rc, lines, err = _run("--gpus", str(n), "--launch-selftest")
    assert rc == 0, err[-2000:]
    assert len(lines) == 1, lines  # rank 0 alone prints
    ln = lines[0]
    assert ln["n_gpus"] == n and ln["ranks_seen"] == n and ln["gpus_requested"] == n
    if n > 1:
        assert ln["nccl_debug"] == "INFO"  # communicator init lines requested from NCCL


def test_launcher_refuses_missing_gpus():
    # no GPU in this container: --gpus 2 must fail loudly, not run one rank
    import torch

    if torch.cuda.device_count() >= 2:
        pytest.skip("this host has >= 2 GPUs")
    rc, lines, err = _run("--gpus", "2", "--steps", "1", "--warmup", "0")
    assert rc != 0
    assert lines and "error" in lines[0]

"""bench.py --gpus N without torchrun spawns N ranks itself (RANK / LOCAL_RANK /
WORLD_SIZE / MASTER_* like torchrun) and rank 0 prints ONE JSON line whose
n_gpus is the world size; the timing is the max over ranks.  The CPU self-test
target drives the same spawn_ranks() path with gloo instead of NCCL."""

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(extra):
    env = dict(os.environ)
    for k in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--selftest-spawn",
                          "--steps", "3", "--warmup", "3", *extra], env=env, cwd=REPO,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_self_spawn_world2_prints_one_line_with_n_gpus_2():
    d = _run(["--gpus", "2"])
    assert d["n_gpus"] == 2 and d["steps"] == 3 and d["value"] > 0


def test_single_process_default():
    d = _run([])
    assert d["n_gpus"] == 1

"""bench.py's multi-rank path on the CPU (no GPU): `python bench.py --gpus N --dry-run`
re-executes itself as N torchrun ranks (gloo), each rank takes its shard of the batched
configs and the shards are all-gathered with the same gather_batches the GPU run uses over
NCCL; rank 0 prints one JSON line.  A launch whose WORLD_SIZE differs from --gpus fails."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=300, env=e, cwd=ROOT)


@pytest.mark.parametrize("n", [2, 3])
def test_dry_run_multi_rank(n):
    p = _run(["--gpus", str(n), "--dry-run"])
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # only rank 0 prints
    res = json.loads(lines[0])
    assert res["n_gpus"] == n and res["dry_run"] and res["backend"] == "gloo"
    for key in ("batched", "batched_f32_n512"):
        sh = res[key]["shards"]
        assert len(sh) == n and sh[0][0] == 0 and sh[-1][1] == res[key]["total"]
        assert res[key]["gather"]["order_ok"]
        assert "gather" in res[key] and res[key]["gather"]["bytes"] > 0


def test_world_size_mismatch_fails_loudly():
    p = _run(["--gpus", "2", "--dry-run"], env={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert p.returncode != 0
    assert "WORLD_SIZE=1" in (p.stderr + p.stdout)

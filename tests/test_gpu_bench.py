"""bench.py's N-rank path on the box's one GPU: `--gpus 2 --oversubscribe`
re-launches itself under torchrun with two ranks (the driver's N > 1 form
without WORLD_SIZE), each rank runs the library's pipeline on its shard of
the C5 stream (batch t -> rank t % 2, no data-path collective), rank 0
checks its last step against the reference cursor and prints ONE line with
n_gpus = 2.  Device times are summed over ranks sharing a GPU
("oversubscribed")."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_self_spawn(torch_cuda):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--oversubscribe", "--steps",
                        "3", "--warmup", "3", "--e2e-steps", "0", "--no-configs", "--sharded-steps", "1",
                        "--probe-steps", "2"], capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    assert "oversubscribed" in d
    assert d["check"]["ok"] is True, d["check"]
    assert d["gpu_launches"] > 0
    assert "launching" in r.stderr and "rank 1/2" in r.stderr

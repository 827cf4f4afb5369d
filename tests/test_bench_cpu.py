"""bench.py's multi-rank launcher on CPU: `--gpus 2` outside torchrun must
re-execute itself as two ranks (torch.distributed.run, 127.0.0.1), time with
the max over ranks, and print exactly one JSON line from rank 0 that reports
the world size it ran at."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("n", [1, 2])
def test_bench_self_launches_n_ranks(n):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", str(n), "--steps", "3",
                        "--selftest-dist"], capture_output=True, text=True, timeout=240,
                       cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 only
    out = json.loads(lines[0])
    assert out["n_gpus"] == n and out["ranks_seen"] == n
    assert out["value"] > 0

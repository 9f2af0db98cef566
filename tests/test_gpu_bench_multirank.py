"""GPU: `bench.py --gpus 2` with no launcher spawns two ranks itself.

Only one GPU is available here, so both ranks share cuda:0 (MQ_DIST_BACKEND=gloo
for the host plumbing); the data path is the same peer-memory exchange inside
the step graphs that one-GPU-per-rank runs use.  The printed line must carry
n_gpus = 2, the exchange actually used, and whole-job seed accounting
(every rank's batches, round-robin dealt)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("staleness", [0, 1])
def test_bench_spawns_ranks(staleness):
    env = dict(os.environ, MQ_DIST_BACKEND="gloo")
    cmd = [sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--shape", "cfg1",
           "--steps", "12", "--warmup", "3", "--no-cpu-baseline", "--profile-steps", "2",
           "--e2e-steps", "6", "--staleness", str(staleness)]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = lines[0]
    assert line["n_gpus"] == 2 and line["steps"] == 12
    assert line["config"]["exchange"].startswith("peer memory")
    assert line["config"]["parallelism"].startswith("dp2")
    assert line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["windows_per_epoch"] >= 1

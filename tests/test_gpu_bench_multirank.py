"""GPU: the N > 1 bench path end to end -- `bench.py --gpus 2` self-launches
two ranks (torch.distributed.run), each builds only its slices
(distbuild.build_partitioned) and the sweep runs over the fused exchange.
Here both ranks share the one GPU (FLYCOO_PG_BACKEND=gloo, host barriers):
a functional check of the path the 8-GPU run takes, not a measurement."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("cfg,nnz,world", [(2, 4_000_000, 2), (3, 2_000_000, 3)])
def test_bench_self_launched_ranks(cfg, nnz, world):
    env = dict(os.environ, FLYCOO_PG_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", str(world), "--config",
                        str(cfg), "--nnz", str(nnz), "--steps", "3", "--warmup", "3", "--no-e2e"],
                       capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = lines[0]
    assert d["n_gpus"] == world and d["value"] > 0
    assert d["config"]["build"].startswith("partitioned")
    assert "fused peer exchange unavailable" not in d["config"]["parallelism"]

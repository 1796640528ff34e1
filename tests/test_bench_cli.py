"""bench.py plumbing on the CPU: the --gpus N self-launcher (torch.distributed
.run on 127.0.0.1, no torchrun needed) and the reference arm's JSON line,
which carries the same config keys as our arm's; plus the chunk-size rule a
partitioned sweep shares with the single-GPU plan."""
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def test_self_launch_reference_arm_two_ranks():
    env = dict(os.environ, FLYCOO_PG_BACKEND="gloo", CUDA_VISIBLE_DEVICES="")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--config", "1", "--nnz", "20000", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["config"]["nnz"] == 20000 and line["config"]["sample_nnz"] == 20000
    for k in ("workload", "config_index", "dims", "rank"):
        assert k in line["config"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["value"] > 0


def test_gpus_mismatch_fails():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--config", "1", "--nnz", "1000"], capture_output=True, text=True,
                       timeout=300, env=env, cwd=ROOT)
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr


def test_partitioned_chunk_size_follows_global_plan(monkeypatch):
    """dist.py used default_chunk_elems(nnz) without the
    super-shard average, so c5-like plans (32k chunks) got 8k chunks on the
    NCCL path.  plan_chunk_elems mirrors make_mode_work for both cases."""
    from paper_2309_09131_b200 import layout
    from paper_2309_09131_b200.layout import make_mode_work, plan_chunk_elems, plan_from_counts
    from paper_2309_09131_b200.params import device_params
    dims = (46, 3000, 3000)
    nnz = 40_000_000  # > 148 * 4 * 32768: the chunk cap decides
    params = device_params(dims, nnz, 32, g=4096, m=[32, 32, 32])
    rng = np.random.default_rng(3)
    counts = []
    for n in range(3):
        c = rng.multinomial(nnz, np.full(params.k[n], 1.0 / params.k[n]))
        counts.append(c.astype(np.int64))
    plan = plan_from_counts(params, counts)
    for thresh, want_big in ((10**9, False), (1_000, True)):
        monkeypatch.setattr(layout, "BIG_SS_AVG", thresh)
        C = plan_chunk_elems(plan, 0, 32)
        w = make_mode_work(plan, 0, 32, "cpu")
        assert C == w.chunk_elems
        assert C == (32768 if want_big else 8192)

import os
import sys
from pathlib import Path

# the full-size tests (c4: 1.74B nonzeros) need the allocator to reuse freed
# build scratch without fragmentation, as bench.py does
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def golden_layout_names():
    return sorted(p.stem[len("layout_"):] for p in GOLDEN.glob("layout_*.npz"))


def load_layout(name):
    return dict(np.load(GOLDEN / f"layout_{name}.npz"))


def rel_close(got, want, rtol, atol=0.0):
    got, want = np.asarray(got, dtype=np.float64), np.asarray(want, dtype=np.float64)
    bad = np.abs(got - want) > atol + rtol * np.maximum(np.abs(got), np.abs(want))
    return not bad.any(), int(bad.sum())

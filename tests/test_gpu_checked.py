"""GPU: every K1 family (packed, WIDE, tile, general, direct chunks, heavy
super-shards with K2, peer stores) run through the checked build
(libflycoo_checked.so: FC_DEVICE_CHECKS, every shared-tile / output-row index
tested in the kernels) on tools/sanitize_case.py -- the bounds evidence in
place of compute-sanitizer, which is closed on this GPU pool.  Results are
checked against the oracle inside the script."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def test_checked_build_all_kernel_families():
    lib = ROOT / "paper_2309_09131_b200" / "libflycoo_checked.so"
    assert lib.exists(), "build with __graft_entry__.build() (make CHECKED=1)"
    env = dict(os.environ, FLYCOO_LIB="libflycoo_checked.so")
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "sanitize_case.py")], env=env,
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "sanitize_case: all ok" in r.stdout

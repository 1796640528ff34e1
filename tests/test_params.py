"""Host planning restated from the reference, pinned to its outputs."""
import json

import pytest

from conftest import GOLDEN
from paper_2309_09131_b200.params import (InfeasibleParamsError, PartitionParams,
                                          device_params, select_params)

CASES = json.loads((GOLDEN / "select_params.json").read_text())


@pytest.mark.parametrize("case", CASES, ids=[f"{c['shape']}-{i}" for i, c in enumerate(CASES)])
def test_select_params_matches_reference(case):
    kw = dict(case["kw"])
    if "g_range" in kw:
        kw["g_range"] = tuple(kw["g_range"])
    if "infeasible" in case:
        with pytest.raises(InfeasibleParamsError):
            select_params(case["dims"], case["nnz"], **kw)
        return
    p = select_params(case["dims"], case["nnz"], **kw)
    want = case["params"]
    assert list(p.m) == want["m"] and list(p.k) == want["k"] and p.g == want["g"]
    assert p.beta == want["beta"] and list(p.eq2_exact) == want["eq2_exact"]


def test_params_validation():
    with pytest.raises(ValueError):
        PartitionParams((10, 10), 5, (2, 2), (4, 5), 4, 1, 1 << 20, 0.5, 8, 8, 56, 8)
    with pytest.raises(ValueError):
        PartitionParams((10, 10), 5, (2, 2), (5, 5), 4, 1, 1 << 20, 1.5, 8, 8, 56, 8)


def test_device_params_cover_dims():
    # explicit tile: m = bytes / 4R rows in every mode
    p = device_params((12092, 9184, 28818), 76_900_000, 32, acc_tile_bytes=8192)
    assert p.m == (64, 64, 64)
    assert all(m * k >= d for m, k, d in zip(p.m, p.k, p.dims))
    q = device_params((46, 239172, 239172), 10, 16, acc_tile_bytes=8192)
    assert q.m[0] == 46 and q.k[0] == 1
    # 3-mode tensors: 4 KB tiles (c2, c4); 4-mode: per mode, 4 KB tiles for large or very
    # sparse (c3 modes 1-3) super-shards, 8 KB otherwise (c3 mode 0); always covering the dims
    assert device_params((12092, 9184, 28818), 76_900_000, 32).m == (32, 32, 32)
    assert device_params((4821207, 1774269, 1805187), 1_740_000_000, 32).m == (32, 32, 32)
    c3 = device_params((532924, 17262471, 2480308, 1443), 140_000_000, 32)
    assert c3.m == (64, 32, 32, 32)
    assert all(m * k >= d for m, k, d in zip(c3.m, c3.k, c3.dims))

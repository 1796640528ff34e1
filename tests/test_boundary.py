"""Reference-facing call shapes on the host, pinned to the
reference's own outputs (tests/golden/boundary.npz, make_golden.py
golden_boundary): FactorSet.random's Philox stream, CooTensor validation and
duplicate rejection, the device duplicate check (run here on CPU tensors)."""
import json

import numpy as np
import pytest
import torch

from paper_2309_09131_b200 import CooTensor, FactorSet, device_has_duplicates
from paper_2309_09131_b200.coo import coords_key, has_duplicates
from conftest import GOLDEN

Z = np.load(GOLDEN / "boundary.npz")


@pytest.mark.parametrize("i", [0, 1, 2])
def test_factorset_random_reproduces_reference_stream(i):
    dims = tuple(int(d) for d in Z[f"rand{i}_dims"])
    fs = FactorSet.random(dims, int(Z[f"rand{i}_rank"]), int(Z[f"rand{i}_seed"]), device="cpu")
    for n in range(len(dims)):
        want = Z[f"rand{i}_f{n}"].astype(np.float32)
        assert np.array_equal(fs.factors[n].numpy(), want), n


def test_cootensor_errors_match_reference():
    cases = {
        "one_mode": ((5,), [[1]], [1.0]),
        "zero_dim": ((5, 0), [[1, 0]], [1.0]),
        "empty": ((5, 4), np.zeros((0, 2), np.int64), np.zeros(0)),
        "misaligned": ((5, 4), [[1, 1], [2, 2]], [1.0]),
        "nonfinite": ((5, 4), [[1, 1]], [np.inf]),
        "negative": ((5, 4), [[-1, 1]], [1.0]),
        "out_of_range": ((5, 4), [[5, 1]], [1.0]),
        "duplicate": ((5, 4), [[1, 1], [2, 2], [1, 1]], [1.0, 2.0, 3.0]),
    }
    want = json.loads(str(Z["coo_errors"]))
    for name, (dims, subs, vals) in cases.items():
        with pytest.raises(ValueError) as e:
            CooTensor(dims, subs, vals)
        assert str(e.value) == want[name], name


def test_cootensor_same_nonzeros_and_views():
    t = CooTensor((60, 50, 40), Z["seq_subs"], Z["seq_vals"])
    assert t.nnz == len(Z["seq_vals"]) and t.num_modes == 3
    p = np.random.default_rng(1).permutation(t.nnz)
    assert t.same_nonzeros(CooTensor(t.dims, t.subs[p], t.vals[p]))
    v = t.vals.copy()
    v[5] += 1e-9
    assert not t.same_nonzeros(CooTensor(t.dims, t.subs, v))
    assert t.same_nonzeros(CooTensor(t.dims, t.subs, v), rtol=1e-6)
    e = t.element(3)
    assert e.indices == tuple(int(x) for x in t.subs[3]) and e.value == float(t.vals[3])
    assert t.norm() == pytest.approx(float(np.linalg.norm(t.vals)))


@pytest.mark.parametrize("dims", [(50, 40, 30), (4821207, 1774269, 1805187),
                                  (1 << 30, 1 << 30, 1 << 30, 1 << 20)])
def test_duplicate_checks_host_and_device(dims):
    rng = np.random.default_rng(7)
    subs = np.stack([rng.integers(0, d, 30_000) for d in dims], 1)
    uniq = np.unique(subs, axis=0)
    rng.shuffle(uniq)
    dup = np.concatenate([uniq, uniq[11:12]])
    rng.shuffle(dup)
    assert (coords_key(uniq, dims) is None) == (np.prod(np.asarray(dims, dtype=object)) >= 1 << 63)
    for arr, want in ((uniq, False), (dup, True)):
        assert has_duplicates(arr, dims) == want
        for b in (None, 1, 4):
            assert device_has_duplicates(torch.as_tensor(arr), dims, buckets=b) == want


def test_device_duplicate_check_hash_collisions():
    """Equal hashes without equal rows must not count as duplicates: force
    every row into one hash group by checking the exact-compare branch on a
    tiny tensor whose dims overflow 63 bits."""
    dims = (1 << 40, 1 << 40)
    rows = np.array([[1, 2], [2, 1], [3, 4]], dtype=np.int64)
    assert not device_has_duplicates(torch.as_tensor(rows), dims)
    assert device_has_duplicates(torch.as_tensor(np.concatenate([rows, rows[:1]])), dims)


def test_device_duplicate_check_bucket_count(monkeypatch):
    """The automatic bucket count is a power of two for any size (1.74B
    nonzeros asked for 7 buckets before and raised)."""
    import paper_2309_09131_b200.layout as L
    rows = torch.as_tensor(np.stack([np.arange(1000), np.arange(1000)], 1))
    monkeypatch.setattr(L, "_BUCKET_KEYS", 300)  # tiny buckets: 4 for 1000 keys
    assert not L.device_has_duplicates(rows, (1000, 1000))
    assert L.device_has_duplicates(torch.cat([rows, rows[:1]]), (1000, 1000))

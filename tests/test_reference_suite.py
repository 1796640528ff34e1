"""The reference's own test intents (/root/reference/pkg/tests/test_coo.py)
replayed against this package's reference-shaped entry points: FROSTT
parsing / writing (coalescing, comments, error lines, dims override),
CooTensor validation, the seeded generator, rank checks and MCFD factor
dumps.  The oracle-level restatements are pinned to the reference's outputs
in test_oracle_golden.py / test_host.py; this file checks the API surface a
reference user calls."""
import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2309_09131_b200 as mc
from paper_2309_09131_b200 import (CooTensor, FactorSet, FrosttParseError, load_factor_set,
                                   parse_frostt, save_factor_set, synth_tensor, write_frostt)


def random_coo(seed: int) -> CooTensor:
    rng = np.random.Generator(np.random.PCG64(seed))
    dims = tuple(int(x) for x in rng.integers(1, 7, size=int(rng.integers(2, 5))))
    space = int(np.prod(dims))
    nnz = int(rng.integers(1, min(space, 40) + 1))
    flat = rng.choice(space, size=nnz, replace=False)
    subs = np.stack(np.unravel_index(flat, dims), axis=1)
    return CooTensor(dims, subs, rng.uniform(-3, 3, size=nnz))


def test_parse_basic_line():
    t = parse_frostt("1 2 3 4.5\n")
    assert t.dims == (1, 2, 3)
    assert t.element(0).indices == (0, 1, 2) and t.element(0).value == 4.5


def test_parse_coalesces_duplicates():
    t = parse_frostt("1 1 1 2.0\n1 1 1 3.0\n")
    assert t.nnz == 1 and t.element(0).indices == (0, 0, 0) and t.element(0).value == 5.0


def test_parse_comments_and_blank_lines():
    t = parse_frostt("# header comment\n\n2 1 1 1.5\n# mid comment\n1 2 2 2.5\n")
    assert t.nnz == 2 and t.dims == (2, 2, 2)


@pytest.mark.parametrize("text,msg", [
    ("# comment\n", "no nonzero"),
    ("1 1 1 1.0\n2 2 2 2.0\n3 3 3\n", "line 3"),
    ("1 1 1 1.0\n1 2 x 2.0\n", "line 2"),
    ("0 1 1 1.0\n", "1-based"),
    ("1.5 1 1 1.0\n", "non-integer"),
])
def test_parse_errors(text, msg):
    with pytest.raises(FrosttParseError, match=msg):
        parse_frostt(text)


def test_dims_override():
    assert parse_frostt("1 1 1 1.0\n", dims=(4, 5, 6)).dims == (4, 5, 6)
    with pytest.raises(FrosttParseError, match="smaller"):
        parse_frostt("3 1 1 1.0\n", dims=(2, 2, 2))


def test_write_single_element():
    t = CooTensor((1, 2, 3), np.array([[0, 1, 2]]), np.array([4.5]))
    assert write_frostt(t) == "1 2 3 4.5\n"


def test_empty_tensor_rejected():
    with pytest.raises(ValueError, match="no nonzeros"):
        CooTensor((2, 2), np.empty((0, 2), dtype=np.int64), np.empty(0))


@settings(max_examples=60, deadline=None)
@given(st.integers(0, 10_000))
def test_roundtrip_identity(seed):
    t = random_coo(seed)
    assert t.same_nonzeros(parse_frostt(write_frostt(t), dims=t.dims))


def test_roundtrip_through_file(tmp_path):
    t = random_coo(3)
    path = tmp_path / "t.tns"
    write_frostt(t, path)
    assert t.same_nonzeros(mc.read_frostt(path, dims=t.dims))


def test_synth_full_space_is_dense():
    t = synth_tensor([4, 4, 4], 64, seed=11)
    assert t.nnz == 64
    assert sorted(map(tuple, t.subs.tolist())) == sorted(
        (i, j, k) for i in range(4) for j in range(4) for k in range(4))
    assert np.all((t.vals > 0) & (t.vals <= 1))


def test_synth_deterministic():
    a = synth_tensor([50, 60, 70], 900, seed=123, skew=0.7)
    b = synth_tensor([50, 60, 70], 900, seed=123, skew=0.7)
    assert np.array_equal(a.subs, b.subs) and np.array_equal(a.vals, b.vals)
    assert not np.array_equal(a.subs, synth_tensor([50, 60, 70], 900, seed=124, skew=0.7).subs)


def test_synth_rejects_oversized_request():
    with pytest.raises(ValueError, match="exceeds"):
        synth_tensor([3, 3], 10, seed=0)


def test_factor_rank_mismatch_rejected():
    t = random_coo(5)
    mats = [np.ones((d, 3)) for d in t.dims]
    mats[1] = np.ones((t.dims[1], 4))
    with pytest.raises(ValueError, match="rank"):
        FactorSet(tuple(mats), np.ones(3), device="cpu")


def test_factor_dump_roundtrip(tmp_path):
    fs = FactorSet.random((5, 7, 3), 4, seed=2, device="cpu")
    fs = FactorSet(fs.factors, np.array([1.0, 2.0, 0.5, 3.0]), device="cpu")
    path = tmp_path / "f.bin"
    save_factor_set(fs, path)
    back = load_factor_set(path, device="cpu")
    assert back.rank == 4
    assert all(np.array_equal(a.numpy(), b.numpy()) for a, b in zip(back.factors, fs.factors))
    assert np.array_equal(back.lambdas, fs.lambdas)


def test_factor_dump_bad_magic():
    with pytest.raises(ValueError, match="magic"):
        load_factor_set(b"XXXX" + b"\0" * 32, device="cpu")

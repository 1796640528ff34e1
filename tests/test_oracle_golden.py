"""Pin the CPU oracle to the reference: every fixture under tests/golden/ was
produced by the reference package itself (tests/golden/make_golden.py)."""
import json

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, golden_layout_names, load_layout

LAYOUTS = golden_layout_names()


def test_morton_matches_reference():
    z = np.load(GOLDEN / "morton.npz")
    ncase = len([k for k in z.files if k.endswith("_coords")])
    assert ncase >= 5
    for c in range(ncase):
        hi, lo = oracle.morton_interleave(z[f"m{c}_coords"], z[f"m{c}_counts"])
        assert np.array_equal(hi, z[f"m{c}_hi"]), c
        assert np.array_equal(lo, z[f"m{c}_lo"]), c


def test_morton_rejects_wide_keys():
    with pytest.raises(ValueError):
        oracle.morton_interleave(np.zeros((1, 5), np.int64), [1 << 30] * 5)


def _layout(z):
    N = len(z["dims"])
    return oracle.canonical_build(z["subs"], z["vals"], z["dims"], z["m"], z["k"], int(z["g"])), N


@pytest.mark.parametrize("name", LAYOUTS)
def test_canonical_build_matches_reference(name):
    z = load_layout(name)
    L, N = _layout(z)
    for n in range(N):
        for key in ("ss_counts", "ss_elem_offsets", "ss_shard_counts", "ss_first_shard",
                    "shard_offsets"):
            assert np.array_equal(getattr(L, key)[n], z[f"{key}{n}"]), (key, n)
        assert np.array_equal(L.slot_maps[n], z[f"slot_map{n}"]), n
    t = oracle.OracleTensor(L, "reference")
    s, i, v = t.active_arrays()
    assert np.array_equal(s, z["sids0"]) and np.array_equal(i, z["idxs0"])
    assert np.array_equal(v, z["vals0"])


@pytest.mark.parametrize("name", LAYOUTS)
def test_reference_mttkrp_bitwise(name):
    z = load_layout(name)
    N = len(z["dims"])
    fs = [z[f"factor{n}"] for n in range(N)]
    for n in range(N):
        got = oracle.reference_mttkrp(z["subs"], z["vals"], fs, n)
        assert np.array_equal(got, z[f"ref_mttkrp{n}"]), n


@pytest.mark.parametrize("name", LAYOUTS)
@pytest.mark.parametrize("workers", [1, 3])
def test_engine_modes_and_remap_bitwise(name, workers):
    z = load_layout(name)
    L, N = _layout(z)
    fs = [z[f"factor{n}"] for n in range(N)]
    t = oracle.OracleTensor(L, "reference", nu=workers)
    for n in range(N):
        out = t.mttkrp_mode(fs, n)
        assert np.array_equal(out, z[f"engine_mttkrp{n}"]), n
        s, i, v = t.active_arrays()
        assert np.array_equal(s, z[f"after{n}_sids"]), n
        assert np.array_equal(i, z[f"after{n}_idxs"]), n
        assert np.array_equal(v, z[f"after{n}_vals"]), n


@pytest.mark.parametrize("name", LAYOUTS)
def test_sweep_bitwise(name):
    z = load_layout(name)
    L, N = _layout(z)
    fs = [z[f"factor{n}"] for n in range(N)]
    res = oracle.OracleTensor(L, "reference", nu=2).sweep_all_modes(fs)
    for n in range(N):
        assert np.array_equal(res[n], z[f"sweep{n}"]), n


@pytest.mark.parametrize("name", LAYOUTS)
def test_device_order_keeps_reference_shards(name):
    """The B200 order permutes only inside shards: per-shard multisets and
    shard offsets equal the reference's after every remap."""
    z = load_layout(name)
    L, N = _layout(z)
    fs = [z[f"factor{n}"] for n in range(N)]
    t = oracle.OracleTensor(L, "device", nu=2)
    for n in range(N):
        out = t.mttkrp_mode(fs, n)
        np.testing.assert_allclose(out, z[f"engine_mttkrp{n}"], rtol=1e-12, atol=0)
        nxt = (n + 1) % N
        _, i, v = t.active_arrays()
        a = oracle.shard_multiset_keys(i, v.view(np.uint64), L.shard_offsets[nxt])
        b = oracle.shard_multiset_keys(z[f"after{n}_idxs"], z[f"after{n}_vals"].view(np.uint64),
                                       z[f"shard_offsets{nxt}"])
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]), n


def test_lpt_schedule_matches_reference():
    for case in json.loads((GOLDEN / "schedule.json").read_text()):
        assert oracle.lpt_schedule(case["counts"], case["nu"]) == case["assign"]


@pytest.mark.parametrize("name", golden_layout_names())
def test_streaming_shard_hashes_match_canonical_build(name):
    """The C streaming restatement of the canonical shard assignment
    (oracle.shard_hashes, used for c3-c5) against canonical_build's shard
    ids on the reference-generated layouts, every mode."""
    z = load_layout(name)
    N = len(z["dims"])
    L = oracle.canonical_build(z["subs"], z["vals"], z["dims"], z["m"], z["k"], int(z["g"]))
    rec = np.zeros((L.nnz, N + 1), dtype=np.int32)
    rec[:, :N] = z["subs"]
    vb = z["vals"].astype(np.float32).view(np.uint32)
    rec[:, N] = vb.view(np.int32)
    for n in range(N):
        nsh = int(L.ss_first_shard[n][-1])
        want_h, want_c = oracle.shard_digests_from_ids(z["subs"], vb, L.sids_all[:, n], nsh)
        for threads in (1, 3):
            ss, h, c = oracle.shard_hashes(rec, N, n, z["m"], z["k"], int(z["g"]), threads=threads)
            assert np.array_equal(ss, L.ss_counts[n])
            assert np.array_equal(c, want_c) and np.array_equal(h, want_h), (name, n, threads)

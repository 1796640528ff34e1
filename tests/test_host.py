"""CPU-only checks: generators pinned to the reference, host planning,
the C-ABI library loads and exports every symbol of include/flycoo.h."""
import hashlib
import json
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT
from paper_2309_09131_b200 import _lib
from paper_2309_09131_b200.layout import make_mode_work, plan_from_counts
from paper_2309_09131_b200.params import device_params, select_params
from paper_2309_09131_b200.schedule import _lpt
from paper_2309_09131_b200.synth import synth_tensor, zipf_cdf


def test_synth_small_matches_reference():
    z = np.load(GOLDEN / "synth_small.npz")
    subs, vals = synth_tensor((50, 40, 30), 3000, seed=5, skew=0.0)
    assert np.array_equal(subs, z["subs"]) and np.array_equal(vals, z["vals"])


@pytest.mark.slow
def test_synth_c1_matches_reference_digest():
    d = json.loads((GOLDEN / "synth_c1.json").read_text())
    subs, vals = synth_tensor((1000, 800, 600), 1_000_000, seed=1, skew=0.0)
    assert subs[:8].tolist() == d["head_subs"]
    assert hashlib.sha256(np.ascontiguousarray(subs, dtype="<i8").tobytes()).hexdigest() == d["subs_sha256"]
    assert hashlib.sha256(np.ascontiguousarray(vals, dtype="<f8").tobytes()).hexdigest() == d["vals_sha256"]


def test_zipf_cdf():
    c = zipf_cdf(10, 1.1)
    assert c[-1] == 1.0 and np.all(np.diff(c) > 0)
    p = np.diff(np.concatenate(([0], c)))
    assert abs(p[0] / p[1] - 2 ** 1.1) < 1e-9


def test_schedule_lpt_matches_reference():
    for case in json.loads((GOLDEN / "schedule.json").read_text()):
        assert _lpt(case["counts"], case["nu"]) == case["assign"]


def test_header_symbols_exported():
    """Every entry point declared in include/flycoo.h is bound and exported."""
    hdr = (ROOT / "include" / "flycoo.h").read_text()
    declared = set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(fc_[a-z_0-9]+)\(", hdr, re.M))
    assert declared, "no declarations parsed"
    assert declared == set(_lib.exported_symbols())
    L = _lib.load()
    for name in declared:
        assert getattr(L, name) is not None
    assert L.fc_version() == 1
    assert L.fc_crd_words(3) == 4 and L.fc_value_embedded(3) == 1
    assert L.fc_crd_words(4) == 4 and L.fc_value_embedded(4) == 0
    assert L.fc_crd_words(6) == 8 and L.fc_value_embedded(6) == 1
    assert L.fc_tile_elems() == 2048
    assert L.fc_smem_acc_rows_max(32) == 512


def test_plan_from_counts_matches_reference_layout():
    z = dict(np.load(GOLDEN / "layout_n3_skew.npz"))
    N = len(z["dims"])
    params = select_params(tuple(z["dims"]), len(z["vals"]), 4, 32 << 20, int(z["rank"]),
                           g_range=(64, 1024))
    plan = plan_from_counts(params, [z[f"ss_counts{n}"] for n in range(N)])
    for n in range(N):
        assert np.array_equal(plan.shard_offsets[n], z[f"shard_offsets{n}"])
        assert np.array_equal(plan.ss_first_shard[n], z[f"ss_first_shard{n}"])


def test_mode_work_partitions_elements():
    rng = np.random.default_rng(0)
    params = device_params((1000, 300, 50), 200_000, 32)
    counts = [np.bincount(np.minimum(rng.zipf(1.5, 200_000) - 1, d - 1) // params.m[n],
                          minlength=params.k[n]) for n, d in enumerate(params.dims)]
    plan = plan_from_counts(params, counts)
    for n in range(3):
        w = make_mode_work(plan, n, 32, "cpu", chunk_elems=2048, merge=False)
        cs = w.chunk_start.numpy()
        assert cs[0] == 0 and cs[-1] == plan.nnz and np.all(np.diff(cs) > 0)
        ss = w.chunk_ss.numpy()
        offs = plan.ss_elem_offsets[n]
        # every chunk lies inside its super-shard
        assert np.all(cs[:-1] >= offs[ss]) and np.all(cs[1:] <= offs[ss + 1])
        part = w.chunk_part.numpy()
        nch = np.bincount(ss, minlength=params.k[n])
        assert np.all((part >= 0) == (nch[ss] >= 2))
        r1 = w.red1.numpy()
        r2 = w.red2.numpy()
        red = sorted(set(r1[:, 0].tolist()))
        assert red == sorted(np.nonzero((nch == 0) | (nch >= 2))[0].tolist())
        # every partial of a multi-chunk super-shard is summed exactly once
        for s_ in red:
            t1 = r1[r1[:, 0] == s_]
            covered = sorted(q for a_, b_ in t1[:, 1:3] for q in range(a_, b_))
            assert covered == sorted(part[ss == s_].tolist()) if nch[s_] >= 2 else covered == []
            if (t1[:, 3] >= 0).any():
                assert (t1[:, 3] >= 0).all()
                t2 = r2[r2[:, 0] == s_]
                assert len(t2) == 1 and list(range(t2[0, 1], t2[0, 2])) == sorted(t1[:, 3].tolist())


def test_mode_work_merges_small_super_shards():
    """Sparse modes: chunks partition the elements, every output row has
    exactly one writer (a chunk or a reduce task), direct chunks hold whole
    super-shards, at most one tile of nonzeros and <= fc_chunk_rows_max rows."""
    from paper_2309_09131_b200.layout import PART_DIRECT
    rng = np.random.default_rng(1)
    dims = (200000, 300, 50)
    params = device_params(dims, 100_000, 32)
    counts = [np.bincount(np.minimum(rng.zipf(1.3, 100_000) - 1, d - 1) // params.m[n],
                          minlength=params.k[n]) for n, d in enumerate(dims)]
    plan = plan_from_counts(params, counts)
    L = _lib.load()
    tile = L.fc_tile_elems()
    for n in range(3):
        w = make_mode_work(plan, n, 32, "cpu", chunk_elems=4096)
        m = params.m[n]
        cs = w.chunk_start.numpy()
        assert cs[0] == 0 and cs[-1] == plan.nnz and np.all(np.diff(cs) >= 0)
        ss = w.chunk_ss.numpy().astype(np.int64)
        part = w.chunk_part.numpy()
        offs = plan.ss_elem_offsets[n]
        owner = np.zeros(dims[n], dtype=np.int64)
        rows = (np.minimum(m, dims[n] - ss * m) if w.chunk_rows is None
                else w.chunk_rows.numpy().astype(np.int64))
        for c in range(w.nchunks):
            nss = -(-rows[c] // m)
            assert cs[c] >= offs[ss[c]] and cs[c + 1] <= offs[ss[c] + nss]
            if part[c] == PART_DIRECT:
                assert cs[c + 1] - cs[c] <= tile and rows[c] <= L.fc_chunk_rows_max(3, 32, m)
                assert cs[c] == offs[ss[c]] and cs[c + 1] == offs[ss[c] + nss]  # whole super-shards
            if part[c] < 0:
                owner[ss[c] * m: ss[c] * m + rows[c]] += 1
        for s_, p0, p1, dst in w.red1.numpy():
            if dst < 0:
                owner[s_ * m: min((s_ + 1) * m, dims[n])] += 1
        for s_, q0, q1 in w.red2.numpy():
            owner[s_ * m: min((s_ + 1) * m, dims[n])] += 1
        assert np.all(owner == 1), n
    w0 = make_mode_work(plan, 0, 32, "cpu", chunk_elems=4096)
    assert (w0.chunk_part.numpy() == PART_DIRECT).any() and w0.hist_rows > params.m[0]


def test_mcfd_dump_byte_compatible_with_reference():
    """Our MCFD writer reproduces the reference's bytes; the reader round-trips."""
    import struct as _s
    from paper_2309_09131_b200 import io as fio
    blob = (GOLDEN / "mcfd_small.bin").read_bytes()
    _, _, nm = _s.unpack_from("<4sII", blob, 0)
    rows = _s.unpack_from(f"<{nm}Q", blob, 12)
    rank = _s.unpack_from("<I", blob, 12 + 8 * nm)[0]
    off = 12 + 8 * nm + 5
    lam = np.frombuffer(blob, "<f8", rank, off)
    off += 8 * rank
    mats = []
    for r in rows:
        mats.append(np.frombuffer(blob, "<f8", r * rank, off).reshape(r, rank))
        off += 8 * r * rank

    class FS:
        factors = mats
        lambdas = lam
    assert fio.save_factor_set(FS()) == blob
    with pytest.raises(ValueError, match="magic"):
        fio.load_factor_set(b"XXXX" + b"\0" * 32, device="cpu")


def test_frostt_parse_and_write_match_reference():
    from paper_2309_09131_b200 import io as fio
    z = np.load(GOLDEN / "frostt_parse.npz")
    subs, vals, dims = fio.parse_frostt("# comment\n1 1 1 1.5\n2 3 1 2.0\n1 1 1 0.25\n\n3 2 2 -1\n")
    assert np.array_equal(subs, z["subs"]) and np.array_equal(vals, z["vals"])
    assert tuple(dims) == tuple(z["dims"])
    ref_text = (GOLDEN / "frostt_small.tns").read_text()
    assert fio.write_frostt(z["synth_subs"], z["synth_vals"]) == ref_text
    s2, v2, _ = fio.parse_frostt(ref_text)
    o = np.lexsort(z["synth_subs"].T[::-1])
    assert np.array_equal(s2, z["synth_subs"][o]) and np.array_equal(v2, z["synth_vals"][o])
    for bad, line in (("1 1 1.5 2\n", 1), ("1 1 1\n0 1 2\n", 2), ("1 2 3\n1 2\n", 2)):
        with pytest.raises(fio.FrosttParseError) as e:
            fio.parse_frostt(bad)
        assert e.value.lineno == line


def test_lean_build_rejects_unsupported_layouts():
    """build_device_sharded_lean validates before touching the device: 16-B
    records of a 2/3-mode tensor, the declared nonzero count, <= 32-bit Morton keys."""
    import pytest
    import torch
    from paper_2309_09131_b200 import device_params
    from paper_2309_09131_b200.layout import build_device_sharded_lean
    rec = torch.zeros((10, 4), dtype=torch.int32)
    with pytest.raises(ValueError, match="16-B records"):
        build_device_sharded_lean(torch.zeros((10, 8), dtype=torch.int32),
                                  device_params((5, 5, 5, 5), 10, 8), device="cpu")
    with pytest.raises(ValueError, match="different nonzero count"):
        build_device_sharded_lean(rec, device_params((50, 50, 50), 11, 8), device="cpu")
    with pytest.raises(ValueError, match="Morton key"):
        build_device_sharded_lean(rec, device_params((1 << 20, 1 << 20, 1 << 20), 10, 8, m=[1, 1, 1]),
                                  device="cpu")


def _header_params(name: str) -> list:
    """Parameter types of a declaration in include/flycoo.h (comments stripped)."""
    hdr = (ROOT / "include" / "flycoo.h").read_text()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    m = re.search(rf"\b{name}\((.*?)\);", hdr, re.S)
    assert m, name
    return [p.strip() for p in m.group(1).split(",")]


def test_reference_binding_matches_header():
    """INTEGRATION.md section 2's ctypes binding (tests/reference_binding.py)
    declares one ctypes type per C parameter of fc_mode_worker, with the
    integer widths of the header."""
    import ctypes
    import reference_binding as rb
    params = _header_params("fc_mode_worker")
    assert len(params) == len(rb.MODE_WORKER_ARGTYPES)
    for p, t in zip(params, rb.MODE_WORKER_ARGTYPES):
        if "*" in p:
            assert t is ctypes.c_void_p, p
        elif p.startswith("int64_t"):
            assert t is ctypes.c_int64, p
        else:
            assert p.startswith("int ") and t is ctypes.c_int, p
    assert rb.lib().fc_version() == 1

"""GPU parity: the sm_100a path (through libflycoo's C ABI) against the CPU
oracle and the reference's golden fixtures.

Bars (north_star): remapped shards bit-exact as per-shard multisets with
identical shard offsets (this build is stricter: the whole buffer equals the
oracle's restatement of the B200 order); MTTKRP within rel 1e-4 per entry in
fp32 against float64 (empty rows exactly 0).
"""
import numpy as np
import pytest
import torch

import oracle
from conftest import golden_layout_names, load_layout
from gpu_helpers import (RTOL, assert_rel, factors_f32, host_records, oracle_records, params_of)
from paper_2309_09131_b200 import (BufferOrderError, DeviceFactorSet, ShardOverflowError,
                                   TrafficCounters, build_device_sharded, device_params,
                                   mttkrp_mode, schedule_super_shards, select_params,
                                   sweep_all_modes)
from paper_2309_09131_b200.synth import synth_tensor, zipf_tensor

pytestmark = pytest.mark.gpu

LAYOUTS = golden_layout_names()


def _golden(name):
    z = load_layout(name)
    N = len(z["dims"])
    params = params_of(z["dims"], len(z["vals"]), z["m"], z["k"], int(z["g"]), int(z["rank"]),
                       int(z["nu"]))
    return z, N, params


@pytest.mark.parametrize("name", LAYOUTS)
def test_build_matches_reference_plan_and_oracle_order(name):
    z, N, params = _golden(name)
    st = build_device_sharded(z["subs"], z["vals"], params)
    for n in range(N):
        for key in ("ss_counts", "ss_elem_offsets", "ss_shard_counts", "ss_first_shard",
                    "shard_offsets"):
            assert np.array_equal(getattr(st.plan, key)[n], z[f"{key}{n}"]), (key, n)
    L = oracle.canonical_build(z["subs"], z["vals"], z["dims"], z["m"], z["k"], int(z["g"]))
    d = oracle.device_order(L)
    for n in range(N):
        got = st.slot_maps[n].cpu().numpy().view(np.uint32).astype(np.int64)
        assert np.array_equal(got, d.slot_maps[n]), n
    c, vb = host_records(st)
    assert np.array_equal(c, z["subs"][d.orders[0]])
    assert np.array_equal(vb, z["vals"][d.orders[0]].astype(np.float32).view(np.uint32))
    # reference-dtype view: shard ids of every mode match the reference build
    sids, idxs, vals = st.active_arrays()
    ref = oracle.shard_multiset_keys(z["idxs0"], z["vals0"].view(np.uint64), z["shard_offsets0"])
    got = oracle.shard_multiset_keys(idxs, vals.view(np.uint64), st.plan.shard_offsets[0])
    assert np.array_equal(ref[0], got[0]) and np.array_equal(ref[1], got[1])
    assert np.array_equal(np.sort(sids, axis=0), np.sort(z["sids0"], axis=0))


@pytest.mark.parametrize("name", LAYOUTS)
def test_mode_passes_match_reference(name):
    z, N, params = _golden(name)
    st = build_device_sharded(z["subs"], z["vals"], params)
    smap = schedule_super_shards(st.plan, 2)
    fs = DeviceFactorSet.from_host([z[f"factor{n}"] for n in range(N)])
    L = oracle.canonical_build(z["subs"], z["vals"], z["dims"], z["m"], z["k"], int(z["g"]))
    ot = oracle.OracleTensor(L, "device")
    counters = TrafficCounters()
    for n in range(N):
        out = mttkrp_mode(st, fs, n, smap, counters=counters)
        assert_rel(out.double().cpu().numpy(), z[f"engine_mttkrp{n}"], what=f"mode {n}")
        ot.mttkrp_mode([z[f"factor{w}"] for w in range(N)], n)
        c, vb = host_records(st)
        oc, ovb = oracle_records(ot)
        assert np.array_equal(c, oc) and np.array_equal(vb, ovb), f"remap after mode {n}"
        nxt = (n + 1) % N
        a = oracle.shard_multiset_keys(c, vb.astype(np.uint64), st.plan.shard_offsets[nxt])
        b = oracle.shard_multiset_keys(z[f"after{n}_idxs"],
                                       z[f"after{n}_vals"].astype(np.float32).view(np.uint32).astype(np.uint64),
                                       z[f"shard_offsets{nxt}"])
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]), f"shards after mode {n}"
    eb = st.element_nbytes
    assert counters.tensor_bytes_read == N * st.nnz * eb
    assert counters.remap_bytes_written == N * st.nnz * eb
    assert counters.factor_bytes_read == N * st.nnz * (N - 1) * int(z["rank"]) * 8


@pytest.mark.parametrize("name", LAYOUTS)
def test_sweep_matches_oracle_chain(name):
    """Updated-factor sweep; mode n's oracle gets the GPU's own inputs
    (upcast), so errors do not compound."""
    z, N, params = _golden(name)
    st = build_device_sharded(z["subs"], z["vals"], params)
    smap = schedule_super_shards(st.plan, 1)
    f0 = [z[f"factor{n}"] for n in range(N)]
    secs = []
    res = sweep_all_modes(st, DeviceFactorSet.from_host(f0), smap, mode_seconds=secs)
    assert len(secs) == N and all(s > 0 for s in secs)
    working = [np.asarray(f, dtype=np.float64) for f in f0]
    got = res.to_numpy()
    for n in range(N):
        want = oracle.reference_mttkrp(z["subs"], z["vals"], working, n)
        assert_rel(got[n], want, what=f"sweep mode {n}")
        working[n] = got[n]
    # a full cycle returns the buffer to the mode-0 arrangement
    st2 = build_device_sharded(z["subs"], z["vals"], params)
    assert st.active_mode == 0
    assert np.array_equal(host_records(st)[0], host_records(st2)[0])


def test_sweep_bitwise_deterministic():
    z, N, params = _golden("n3_skew")
    smap = None
    outs = []
    for _ in range(2):
        st = build_device_sharded(z["subs"], z["vals"], params)
        smap = schedule_super_shards(st.plan, 4)
        res = sweep_all_modes(st, DeviceFactorSet.from_host([z[f"factor{n}"] for n in range(N)]), smap)
        outs.append([f.cpu().numpy().tobytes() for f in res.factors])
    assert outs[0] == outs[1]


@pytest.mark.parametrize("rank", [1, 3, 8, 16, 32, 40, 64, 200])
def test_ranks(rank):
    subs, vals = synth_tensor((300, 200, 100), 40_000, seed=3, skew=0.7)
    vals = vals.astype(np.float32).astype(np.float64)
    params = device_params((300, 200, 100), len(vals), rank, g=1024)
    st = build_device_sharded(subs, vals, params)
    smap = schedule_super_shards(st.plan, 1)
    fs = factors_f32(params.dims, rank, 7)
    dfs = DeviceFactorSet.from_host(fs)
    for n in range(3):
        out = mttkrp_mode(st, dfs, n, smap)
        want = oracle.reference_mttkrp(subs, vals, fs, n)
        assert_rel(out.double().cpu().numpy(), want, what=f"R={rank} mode {n}")


@pytest.mark.parametrize("nm", [2, 4, 5, 6, 8])
def test_mode_counts(nm):
    dims = [37, 23, 11, 9, 7, 6, 5, 4][:nm]
    rng = np.random.default_rng(nm)
    draws = np.stack([rng.integers(0, d, 30_000) for d in dims], axis=1)
    _, first = np.unique(draws, axis=0, return_index=True)
    subs = draws[np.sort(first)][:20_000]
    vals = rng.uniform(0.5, 1.5, len(subs)).astype(np.float32).astype(np.float64)
    for rank in (16, 32, 7):
        params = device_params(dims, len(vals), rank, g=512, m=[5] * nm)
        st = build_device_sharded(subs, vals, params)
        smap = schedule_super_shards(st.plan, 1)
        fs = factors_f32(dims, rank, nm)
        L = oracle.canonical_build(subs, vals, dims, params.m, params.k, params.g)
        ot = oracle.OracleTensor(L, "device")
        for n in range(nm):
            out = mttkrp_mode(st, DeviceFactorSet.from_host(fs), n, smap)
            assert_rel(out.double().cpu().numpy(), oracle.reference_mttkrp(subs, vals, fs, n),
                       what=f"N={nm} R={rank} mode {n}")
            ot.mttkrp_mode(fs, n)
            assert np.array_equal(host_records(st)[0], oracle_records(ot)[0])
            assert np.array_equal(host_records(st)[1], oracle_records(ot)[1])


def test_global_accumulator_path():
    """Reference CPU params (m = whole mode at nu=1): rows accumulate in
    global memory, one chunk per super-shard."""
    subs, vals = synth_tensor((1000, 800, 600), 60_000, seed=9, skew=0.3)
    vals = vals.astype(np.float32).astype(np.float64)
    params = select_params((1000, 800, 600), len(vals), 1, 32 << 20, 32)
    assert params.m == (1000, 800, 600)
    st = build_device_sharded(subs, vals, params)
    smap = schedule_super_shards(st.plan, 1)
    fs = factors_f32(params.dims, 32, 2)
    for n in range(3):
        out = mttkrp_mode(st, DeviceFactorSet.from_host(fs), n, smap)
        assert_rel(out.double().cpu().numpy(), oracle.reference_mttkrp(subs, vals, fs, n),
                   what=f"global mode {n}")


def test_heavy_rows_split_and_reduced():
    """One output row with ~300k nonzeros (many chunks -> K2 reduce) and a
    Zipf tail; fp32 stays within 1e-4."""
    rng = np.random.default_rng(5)
    n_heavy = 300_000
    a = np.column_stack([np.zeros(n_heavy, np.int64), rng.integers(0, 3000, n_heavy),
                         rng.integers(0, 3000, n_heavy)])
    b = np.column_stack([rng.integers(1, 5000, 200_000), rng.integers(0, 3000, 200_000),
                         rng.integers(0, 3000, 200_000)])
    draws = np.concatenate([a, b])
    _, first = np.unique(draws, axis=0, return_index=True)
    subs = draws[np.sort(first)]
    vals = rng.uniform(0, 1, len(subs)).astype(np.float32).astype(np.float64)
    dims = (5000, 3000, 3000)
    params = device_params(dims, len(vals), 32)
    st = build_device_sharded(subs, vals, params)
    smap = schedule_super_shards(st.plan, 1)
    w = st.mode_work(0, 32)
    assert w.nparts > 10  # the heavy super-shard is split over many chunks
    fs = factors_f32(dims, 32, 4)
    for n in range(3):
        out = mttkrp_mode(st, DeviceFactorSet.from_host(fs), n, smap)
        assert_rel(out.double().cpu().numpy(), oracle.reference_mttkrp(subs, vals, fs, n),
                   what=f"heavy mode {n}")


def test_cursor_strategy_shards_and_values():
    z, N, params = _golden("n3_small")
    st = build_device_sharded(z["subs"], z["vals"], params)
    smap = schedule_super_shards(st.plan, 2)
    fs = DeviceFactorSet.from_host([z[f"factor{n}"] for n in range(N)])
    for n in range(N):
        out = mttkrp_mode(st, fs, n, smap, remap="cursor")
        assert_rel(out.double().cpu().numpy(), z[f"engine_mttkrp{n}"], what=f"cursor mode {n}")
        nxt = (n + 1) % N
        c, vb = host_records(st)
        a = oracle.shard_multiset_keys(c, vb.astype(np.uint64), st.plan.shard_offsets[nxt])
        b = oracle.shard_multiset_keys(z[f"after{n}_idxs"],
                                       z[f"after{n}_vals"].astype(np.float32).view(np.uint32).astype(np.uint64),
                                       z[f"shard_offsets{nxt}"])
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert not st.canonical
    with pytest.raises(BufferOrderError):
        mttkrp_mode(st, fs, 0, smap, remap="slot")


def test_split_remap_matches_fused():
    z, N, params = _golden("n4_small")
    fs = DeviceFactorSet.from_host([z[f"factor{n}"] for n in range(N)])
    st1 = build_device_sharded(z["subs"], z["vals"], params)
    st2 = build_device_sharded(z["subs"], z["vals"], params)
    smap = schedule_super_shards(st1.plan, 1)
    for n in range(N):
        a = mttkrp_mode(st1, fs, n, smap)
        b = mttkrp_mode(st2, fs, n, smap, split_remap=True)
        assert torch.equal(a, b)
        assert torch.equal(st1.crd[st1.active], st2.crd[st2.active])


def test_precondition_errors():
    z, N, params = _golden("n3_small")
    st = build_device_sharded(z["subs"], z["vals"], params)
    smap = schedule_super_shards(st.plan, 2)
    fs = DeviceFactorSet.from_host([z[f"factor{n}"] for n in range(N)])
    with pytest.raises(BufferOrderError):
        mttkrp_mode(st, fs, 1, smap)
    with pytest.raises(ValueError):
        mttkrp_mode(st, fs, 5, smap)
    with pytest.raises(ValueError):
        mttkrp_mode(st, fs, 0, smap, remap="bogus")
    with pytest.raises(ValueError):
        mttkrp_mode(st, fs, 0, smap, workers=0)
    other = schedule_super_shards(build_device_sharded(z["subs"][:-1], z["vals"][:-1], params_of(
        z["dims"], len(z["vals"]) - 1, z["m"], z["k"], int(z["g"]), 8)).plan, 2)
    with pytest.raises(ValueError):
        mttkrp_mode(st, fs, 0, other)
    bad = DeviceFactorSet.from_host([z[f"factor{n}"][:-1] for n in range(N)])
    with pytest.raises(ValueError):
        mttkrp_mode(st, bad, 0, smap)


def test_injected_faults_raise():
    """Fault injection (bench.py:279-289 analogue): a corrupted slot overflows,
    a record moved to the wrong super-shard is an order error."""
    z, N, params = _golden("n3_small")
    fs = DeviceFactorSet.from_host([z[f"factor{n}"] for n in range(N)])
    st = build_device_sharded(z["subs"], z["vals"], params)
    smap = schedule_super_shards(st.plan, 2)
    st.slot_maps[0][3] = st.nnz + 5
    with pytest.raises(ShardOverflowError):
        mttkrp_mode(st, fs, 0, smap)
    st = build_device_sharded(z["subs"], z["vals"], params)
    # an output coordinate outside every super-shard row range of the chunk
    st.crd[0][0, 0] = int(z["dims"][0]) + 3
    with pytest.raises(BufferOrderError):
        mttkrp_mode(st, fs, 0, smap)


def test_c1_full_fixed_factors():
    """Config 1 at full size against the oracle engine (fixed factors)."""
    subs, vals = synth_tensor((1000, 800, 600), 1_000_000, seed=1, skew=0.0)
    vals = vals.astype(np.float32).astype(np.float64)
    params = device_params((1000, 800, 600), len(vals), 16)
    st = build_device_sharded(subs, vals, params)
    smap = schedule_super_shards(st.plan, 1)
    fs = factors_f32(params.dims, 16, 1001)
    dfs = DeviceFactorSet.from_host(fs)
    L = oracle.canonical_build(subs, vals, params.dims, params.m, params.k, params.g)
    ot = oracle.OracleTensor(L, "device", nu=8)
    for n in range(3):
        out = mttkrp_mode(st, dfs, n, smap)
        want = ot.mttkrp_mode(fs, n)
        assert_rel(out.double().cpu().numpy(), want, what=f"c1 mode {n}")
        assert np.array_equal(host_records(st)[0], oracle_records(ot)[0])


def test_c2_sample_vs_oracle_and_full_cycle():
    """Config-2 law at 3M nonzeros: parity against the oracle; then the
    size-independent properties (cycle returns the buffer bit-exactly,
    multiset conserved) at the same size."""
    coords, vals = zipf_tensor((12092, 9184, 28818), 3_000_000, seed=2, exponents=(1.1, 1.1, 1.1))
    subs = coords.cpu().numpy().astype(np.int64)
    v64 = vals.cpu().numpy().astype(np.float64)
    assert len(np.unique(subs, axis=0)) == len(subs)
    params = device_params((12092, 9184, 28818), len(v64), 32)
    st = build_device_sharded(coords, vals, params)
    smap = schedule_super_shards(st.plan, 1)
    fs = factors_f32(params.dims, 32, 1002)
    dfs = DeviceFactorSet.from_host(fs)
    start = host_records(st)
    for n in range(3):
        out = mttkrp_mode(st, dfs, n, smap)
        assert_rel(out.double().cpu().numpy(), oracle.reference_mttkrp(subs, v64, fs, n),
                   what=f"c2 sample mode {n}")
    end = host_records(st)
    assert np.array_equal(start[0], end[0]) and np.array_equal(start[1], end[1])


def test_sparse_mode_direct_chunks():
    """A mode with far more rows than nonzeros per super-shard: consecutive
    super-shards are packed into direct chunks (rows stored straight to
    `out`, empty rows zeroed); parity with the oracle, including empty rows."""
    from paper_2309_09131_b200.layout import PART_DIRECT
    rng = np.random.default_rng(8)
    dims = (300000, 400, 60)
    draws = np.column_stack([np.minimum(rng.zipf(1.2, 300_000) - 1, dims[0] - 1),
                             rng.integers(0, dims[1], 300_000), rng.integers(0, dims[2], 300_000)])
    _, first = np.unique(draws, axis=0, return_index=True)
    subs = draws[np.sort(first)][:200_000]
    vals = rng.uniform(0.1, 1.0, len(subs)).astype(np.float32).astype(np.float64)
    for rank in (16, 32):
        params = device_params(dims, len(vals), rank)
        st = build_device_sharded(subs, vals, params)
        smap = schedule_super_shards(st.plan, 1)
        w = st.mode_work(0, rank)
        assert (w.chunk_part.cpu().numpy() == PART_DIRECT).any()
        fs = factors_f32(dims, rank, 5)
        for n in range(3):
            out = mttkrp_mode(st, DeviceFactorSet.from_host(fs), n, smap)
            assert_rel(out.double().cpu().numpy(), oracle.reference_mttkrp(subs, vals, fs, n),
                       what=f"direct R={rank} mode {n}")


@pytest.mark.parametrize("cfg", [2, 3])
def test_gpu_generator_matches_host_twin(cfg):
    """K6 (GPU Philox + bounded-Zipf + first-occurrence dedup) equals its
    numpy twin: 64-bit keys (config 2 shape) and 128-bit keys (config 3)."""
    from paper_2309_09131_b200.synth import CONFIGS, zipf_tensor_host
    c = CONFIGS[cfg]
    coords, vals = zipf_tensor(c["dims"], 200_000, seed=cfg, exponents=c["law"])
    subs, hv = zipf_tensor_host(c["dims"], 200_000, seed=cfg, exponents=c["law"])
    assert np.array_equal(coords.cpu().numpy().astype(np.int64), subs)
    assert np.array_equal(vals.cpu().numpy(), hv)


def test_packed_and_unpacked_modes_in_one_sweep():
    """Modes 0/1 fit 8-byte packed records (17 + 7 coordinate bits), mode 2
    does not (17 + 17 > 32) and runs the 16-byte tile kernel; the chained
    sweep must match the oracle through both."""
    dims = (1 << 17, 1 << 17, 100)
    coords, vals = zipf_tensor(dims, 400_000, seed=12, exponents=(0.8, 0.8, 1.0))
    subs = coords.cpu().numpy().astype(np.int64)
    v64 = vals.cpu().numpy().astype(np.float64)
    assert subs[:, 0].max() >= 1 << 16 and subs[:, 1].max() >= 1 << 16
    params = device_params(dims, len(v64), 32)
    st = build_device_sharded(coords, vals, params)
    smap = schedule_super_shards(st.plan, 1)
    f0 = factors_f32(dims, 32, 9)
    res = sweep_all_modes(st, DeviceFactorSet.from_host(f0), smap).to_numpy()
    working = [f.astype(np.float64) for f in f0]
    for n in range(3):
        want = oracle.reference_mttkrp(subs, v64, working, n)
        assert_rel(res[n], want, what=f"mixed mode {n}")
        working[n] = res[n]


def test_remap_store_single_element_mirror():
    """remap_store / RemapCursors (engine.py:94-135): first store lands at the
    shard base, a full shard raises ShardOverflowError."""
    from paper_2309_09131_b200 import RemapCursors, remap_store
    z, N, params = _golden("n3_small")
    st = build_device_sharded(z["subs"], z["vals"], params)
    cur = RemapCursors.for_mode(st, 1)
    sids = st.shard_ids()
    shard = int(sids[0, 1])
    slot = remap_store(0, 1, cur, st)
    assert slot == int(st.plan.shard_offsets[1][shard])
    rec = st.crd[1 - st.active][slot].cpu()
    assert torch.equal(rec, st.crd[st.active][0].cpu())
    fill = cur.planned_fill(shard)
    cur.fills[shard] = fill
    with pytest.raises(ShardOverflowError):
        remap_store(0, 1, cur, st)
    assert not cur.complete()


@pytest.mark.parametrize("m", [(32, 32, 32), (64, 64, 64)])
def test_wide_coordinates_packed_kernel(m):
    """Modes whose two input coordinates need more than 32 bits together
    (here mode 2: 17 + 17 bits, like c4 / c5 mode 0) run the packed kernel's
    WIDE variant ({c_w1, c_w2} words + value array): outputs within 1e-4 of
    the oracle and remapped buffers bit-exact with its B200 order."""
    rng = np.random.default_rng(17)
    dims = (70_000, 70_001, 300)
    n = 250_000
    # a Zipf-ish head so that rows span pieces and super-shards split over chunks
    c0 = np.minimum((rng.pareto(1.2, n) * 50).astype(np.int64), dims[0] - 1)
    c1 = np.minimum((rng.pareto(1.2, n) * 50).astype(np.int64), dims[1] - 1)
    c2 = rng.integers(0, dims[2], n)
    draws = np.column_stack([c0, c1, c2])
    _, first = np.unique(draws, axis=0, return_index=True)
    subs = draws[np.sort(first)]
    vals = rng.uniform(0, 1, len(subs)).astype(np.float32).astype(np.float64)
    params = device_params(dims, len(vals), 32, g=4096, m=m)
    st = build_device_sharded(subs, vals, params)
    smap = schedule_super_shards(st.plan, 1)
    L = oracle.canonical_build(subs, vals, dims, params.m, params.k, params.g)
    ot = oracle.OracleTensor(L, "device")
    fs = factors_f32(dims, 32, 9)
    for mode in range(3):
        out = mttkrp_mode(st, DeviceFactorSet.from_host(fs), mode, smap)
        assert_rel(out.double().cpu().numpy(), oracle.reference_mttkrp(subs, vals, fs, mode),
                   what=f"wide mode {mode}")
        ot.mttkrp_mode(fs, mode)
        c, vb = host_records(st)
        oc, ovb = oracle_records(ot)
        assert np.array_equal(c, oc) and np.array_equal(vb, ovb), f"remap after mode {mode}"


def test_config5_law_every_row():
    """Config 5's law and dims (46 x 239172 x 239172; mode 0 uniform over 46
    rows, modes 1-2 Zipf 1.0) at 4M nonzeros, every output row of every mode
    against the oracle: 46 rows of ~87k nonzeros each (super-shards split over
    many chunks, two-level K2), mode 0's 18 + 18-bit inputs on the WIDE
    packed kernel, and the bucketed generator's records as the input."""
    from paper_2309_09131_b200.synth import CONFIGS, zipf_records_bucketed
    c = CONFIGS[5]
    dims = tuple(c["dims"])
    rec = zipf_records_bucketed(dims, 4_000_000, seed=5, exponents=c["law"],
                                bucket_draws=1 << 20, scan=1 << 22)
    subs = rec[:, :3].cpu().numpy().astype(np.int64)
    v64 = rec[:, 3].view(torch.float32).cpu().numpy().astype(np.float64)
    params = device_params(dims, len(v64), 32)
    st = build_device_sharded(rec[:, :3].contiguous(), rec[:, 3].view(torch.float32).contiguous(),
                              params)
    assert st.mode_work(0, 32).nparts > 100
    smap = schedule_super_shards(st.plan, 1)
    fs = factors_f32(dims, 32, 1005)
    dfs = DeviceFactorSet.from_host(fs)
    start = host_records(st)
    for n in range(3):
        out = mttkrp_mode(st, dfs, n, smap)
        assert_rel(out.double().cpu().numpy(), oracle.reference_mttkrp(subs, v64, fs, n),
                   what=f"c5 law mode {n}")
    end = host_records(st)
    assert np.array_equal(start[0], end[0]) and np.array_equal(start[1], end[1])


@pytest.mark.parametrize("cfg,nnz", [(3, 2_000_000), (4, 3_000_000)])
def test_config_law_every_row(cfg, nnz):
    """Configs 3 (4 modes, 17M-row sparse mode: direct chunks) and 4 (every
    mode on the WIDE packed kernel: 21-23-bit coordinates) with their dims and
    laws at a few million nonzeros: every output row of every mode against the
    oracle, and the cycle identity."""
    from paper_2309_09131_b200.synth import CONFIGS
    c = CONFIGS[cfg]
    dims = tuple(c["dims"])
    coords, vals = zipf_tensor(dims, nnz, seed=cfg, exponents=c["law"])
    subs = coords.cpu().numpy().astype(np.int64)
    v64 = vals.cpu().numpy().astype(np.float64)
    params = device_params(dims, nnz, 32)
    st = build_device_sharded(coords, vals, params)
    smap = schedule_super_shards(st.plan, 1)
    fs = factors_f32(dims, 32, 1000 + cfg)
    dfs = DeviceFactorSet.from_host(fs)
    start = host_records(st)
    for n in range(len(dims)):
        out = mttkrp_mode(st, dfs, n, smap)
        assert_rel(out.double().cpu().numpy(), oracle.reference_mttkrp(subs, v64, fs, n),
                   what=f"c{cfg} law mode {n}")
    end = host_records(st)
    assert np.array_equal(start[0], end[0]) and np.array_equal(start[1], end[1])

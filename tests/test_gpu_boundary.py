"""GPU: the reference-facing call shapes end to end, and the
layout build with Morton keys wider than 64 bits (morton.py:20-44 `hi` word,
layout.py:477).

* the reference's own call sequence with this package standing in for
  ``modecycle`` -- select_params -> build_sharded(CooTensor, params) ->
  schedule_super_shards -> sweep_all_modes(st, FactorSet.random(dims, R,
  seed), smap) (ref bench.py:119-134) -- against the reference's outputs
  (tests/golden/boundary.npz) and against the oracle;
* validate_plan's check list equals the reference's on the same tensor;
* back_arrays / to_coo views; duplicate coordinates rejected on the device;
* >64-bit Morton keys: the golden 105-bit keys through fc_build_morton, and
  full builds + sweeps of 4- and 5-mode tensors whose keys need 68 / 70 bits
  against the oracle, bit-exactly.
"""
import json

import numpy as np
import pytest
import torch

import oracle
from conftest import GOLDEN
from gpu_helpers import assert_rel, factors_f32, host_records, params_of
import paper_2309_09131_b200 as mc
from paper_2309_09131_b200 import _lib

pytestmark = pytest.mark.gpu

Z = np.load(GOLDEN / "boundary.npz")


def _seq_tensor():
    return mc.CooTensor((60, 50, 40), Z["seq_subs"], Z["seq_vals"])


def _fp32(t):
    """The device holds fp32 values: the source at that precision."""
    return mc.CooTensor(t.dims, t.subs, t.vals.astype(np.float32).astype(np.float64))


def test_reference_call_sequence():
    t = _seq_tensor()
    params = mc.select_params(t.dims, t.nnz, 4, 1 << 16, 16, g_range=(64, 1024))
    assert tuple(params.m) == tuple(int(x) for x in Z["seq_m"]) and params.g == int(Z["seq_g"])
    st = mc.build_sharded(t, params)
    smap = mc.schedule_super_shards(st.plan, 4)
    fs = mc.FactorSet.random(t.dims, 16, 77)
    res = mc.sweep_all_modes(st, fs, smap, remap="slot")
    got = res.to_numpy()
    # against the reference's own sweep (float64 factors; ours are their fp32 rounding)
    for n in range(3):
        assert_rel(got[n], Z[f"seq_out{n}"], what=f"reference sweep mode {n}")
    # against the oracle fed the GPU's own upcast inputs, mode by mode
    working = [f.double().cpu().numpy() for f in fs.factors]
    for n in range(3):
        want = oracle.reference_mttkrp(t.subs, t.vals, working, n)
        assert_rel(got[n], want, what=f"oracle mode {n}")
        working[n] = got[n]
    # the tensor is back in mode-0 order and still holds the source nonzeros
    assert st.active_mode == 0
    assert st.to_coo().same_nonzeros(_fp32(t))


def test_validate_plan_matches_reference_checks():
    t = _seq_tensor()
    params = mc.select_params(t.dims, t.nnz, 4, 1 << 16, 16, g_range=(64, 1024))
    st = mc.build_sharded(t, params)
    rep = mc.validate_plan(st, t)
    assert [c.name for c in rep.checks] == json.loads(str(Z["validate_names"]))
    assert [c.passed for c in rep.checks] == list(Z["validate_passed"])
    assert rep.passed, rep.format()
    # a record moved between super-shards fails interval containment
    st.crd[0][0, 0] = (int(st.crd[0][0, 0]) + params.m[0]) % t.dims[0]
    rep = mc.validate_plan(st)
    assert not rep.passed
    assert rep.first_failure().name.startswith("mode0-interval") or \
        rep.first_failure().name == "active-order"


def test_back_arrays_and_to_coo():
    t = _seq_tensor()
    params = mc.select_params(t.dims, t.nnz, 4, 1 << 16, 16, g_range=(64, 1024))
    st = mc.build_sharded(t, params)
    s, i, v = st.back_arrays()
    assert not s.any() and not i.any() and not v.any()  # fresh back buffer: zeros
    before = st.active_arrays()
    smap = mc.schedule_super_shards(st.plan, 1)
    mc.mttkrp_mode(st, mc.FactorSet.random(t.dims, 16, 3), 0, smap)
    after_back = st.back_arrays()
    for a, b in zip(before, after_back):
        assert np.array_equal(a, b)
    coo = st.to_coo()
    assert isinstance(coo, mc.CooTensor) and coo.same_nonzeros(_fp32(t))


def test_device_build_rejects_duplicates():
    t = _seq_tensor()
    subs = np.concatenate([t.subs, t.subs[5:6]])
    vals = np.concatenate([t.vals, [1.0]])
    params = mc.device_params(t.dims, len(vals), 16, g=256)
    with pytest.raises(ValueError, match="duplicate"):
        mc.build_device_sharded(subs, vals, params)
    with pytest.raises(ValueError, match="duplicate"):
        mc.CooTensor(t.dims, subs, vals)
    # out-of-range coordinates are reported too
    bad = t.subs.copy()
    bad[0, 1] = t.dims[1]
    with pytest.raises(ValueError):
        mc.build_device_sharded(bad, t.vals, mc.device_params(t.dims, t.nnz, 16, g=256))


@pytest.mark.parametrize("case", range(5))
def test_golden_morton_keys_on_device(case):
    """fc_build_morton against the reference's morton.interleave keys,
    including the 105-bit case (hi word set)."""
    z = np.load(GOLDEN / "morton.npz")
    coords = torch.as_tensor(z[f"m{case}_coords"].astype(np.int32), device="cuda").contiguous()
    counts = [int(k) for k in z[f"m{case}_counts"]]
    n, N = coords.shape
    W = sum((k - 1).bit_length() for k in counts)
    lo = torch.empty(n, dtype=torch.int64, device="cuda")
    hi = torch.zeros(n, dtype=torch.int64, device="cuda") if W > 64 else None
    _lib.call("fc_build_morton", coords.data_ptr(), n, N, _lib.i64_array([1] * N),
              _lib.i64_array(counts), hi.data_ptr() if hi is not None else None, lo.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    assert np.array_equal(lo.cpu().numpy().view(np.uint64), z[f"m{case}_lo"])
    want_hi = z[f"m{case}_hi"]
    if hi is None:
        assert not want_hi.any()
    else:
        assert np.array_equal(hi.cpu().numpy().view(np.uint64), want_hi)


@pytest.mark.parametrize("dims,m", [((1 << 17,) * 4, (1, 1, 1, 1)),
                                    ((1 << 14,) * 5, (1, 1, 1, 1, 1)),
                                    ((3 << 20, 1 << 22, 5 << 19), (1, 1, 1))])
def test_build_and_sweep_wide_morton_keys(dims, m):
    N = len(dims)
    rng = np.random.default_rng(N)
    nnz = 60_000
    subs = np.stack([rng.integers(0, d, nnz * 2) for d in dims], 1)
    _, first = np.unique(subs, axis=0, return_index=True)
    subs = subs[np.sort(first)[:nnz]]
    vals = rng.random(len(subs)).astype(np.float32).astype(np.float64)
    k = [-(-d // mm) for d, mm in zip(dims, m)]
    assert sum((x - 1).bit_length() for x in k) > 64
    R = 8
    params = params_of(dims, len(vals), m, k, 4096, R)
    st = mc.build_device_sharded(subs, vals, params)
    L = oracle.canonical_build(subs, vals, dims, m, k, 4096)
    d = oracle.device_order(L)
    for n in range(N):
        assert np.array_equal(st.plan.shard_offsets[n], L.shard_offsets[n]), n
        got = st.slot_maps[n].cpu().numpy().view(np.uint32).astype(np.int64)
        assert np.array_equal(got, d.slot_maps[n]), n
    c, vb = host_records(st)
    assert np.array_equal(c, subs[d.orders[0]])
    fs = factors_f32(dims, R, 5)
    smap = mc.schedule_super_shards(st.plan, 1)
    ot = oracle.OracleTensor(L, "device", nu=4)
    dfs = mc.DeviceFactorSet.from_host(fs)
    for n in range(N):
        out = mc.mttkrp_mode(st, dfs, n, smap)
        assert_rel(out.double().cpu().numpy(), ot.mttkrp_mode(fs, n), what=f"mode {n}")
        assert np.array_equal(host_records(st)[0], ot.active_arrays()[1])

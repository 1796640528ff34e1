"""Tile plans (engine.build_tile_plans, fc_tile_plan_emit / fc_mode_worker_planned):
the static per-tile sort precomputed once.  Planned sweeps must equal the
in-kernel ranking bitwise (outputs and remapped buffers), on packed, WIDE,
direct-chunk and heavy-super-shard plans, and against the oracle."""
import numpy as np
import pytest
import torch

import oracle
from gpu_helpers import assert_rel

pytestmark = pytest.mark.gpu


def _build(dims, nnz, law, **kw):
    from paper_2309_09131_b200 import build_device_sharded, device_params, schedule_super_shards
    from paper_2309_09131_b200.synth import zipf_tensor
    coords, vals = zipf_tensor(dims, nnz, seed=11, exponents=law)
    params = device_params(dims, nnz, 32, **kw)
    st = build_device_sharded(coords, vals, params)
    return coords, vals, params, st, schedule_super_shards(st.plan, 1)


CASES = {
    # packed kernel (input coordinates fit 32 bits), Zipf head split over many chunks (K2)
    "packed": dict(dims=(3000, 2000, 2500), nnz=600_000, law=(1.1, 1.1, 1.1), kw=dict(g=4096)),
    # WIDE packed kernel (two input coordinates need more than 32 bits together)
    "wide": dict(dims=(70_000, 90_000, 80_000), nnz=500_000, law=(1.1, 1.1, 1.1), kw=dict(g=4096)),
    # a sparse mode (direct chunks: many small super-shards per tile) next to dense ones
    "direct": dict(dims=(400_000, 300, 200), nnz=400_000, law=(1.0, 1.1, 1.1), kw=dict(g=2048)),
    # 46 rows in mode 0: two super-shards holding everything (heavy rows)
    "heavy": dict(dims=(46, 20_000, 20_000), nnz=700_000, law=(None, 1.0, 1.0), kw=dict(g=8192)),
    # 4 modes (tile kernel, separate value array), one of them sparse (direct chunks)
    "four": dict(dims=(5000, 300_000, 4000, 90), nnz=500_000, law=(1.2, 1.2, 1.2, 1.2), kw=dict(g=4096)),
}


@pytest.mark.parametrize("name", list(CASES))
def test_planned_sweeps_equal_ranked_sweeps(name, monkeypatch):
    from paper_2309_09131_b200 import DeviceFactorSet, build_device_sharded, sweep_all_modes
    from paper_2309_09131_b200.engine import build_tile_plans
    c = CASES[name]
    coords, vals, params, st, smap = _build(c["dims"], c["nnz"], c["law"], **c["kw"])
    monkeypatch.setenv("FLYCOO_TILE_PLAN", "0")
    ref = build_device_sharded(coords, vals, params)
    fs = DeviceFactorSet.random_device(c["dims"], 32, seed=3)
    want = sweep_all_modes(ref, fs, smap)
    assert all(w.tile_perm is None for w in ref._work.values())
    monkeypatch.setenv("FLYCOO_TILE_PLAN", "1")
    before = st.crd[st.active].clone()
    assert build_tile_plans(st, 32)
    assert st.active_mode == 0 and st.canonical
    assert torch.equal(st.crd[st.active], before)  # the emission walk returns to mode 0
    assert all(st.mode_work(n, 32).tile_perm is not None for n in range(len(c["dims"])))
    for rep in range(2):  # both buffer parities
        got = sweep_all_modes(st, fs, smap)
        if rep:
            want = sweep_all_modes(ref, fs, smap)
        for n, (a, b) in enumerate(zip(got.factors, want.factors)):
            assert torch.equal(a, b), (name, rep, n)
        assert torch.equal(st.crd[st.active], ref.crd[ref.active]), (name, rep)


def test_planned_rank16_equals_ranked(monkeypatch):
    from paper_2309_09131_b200 import (DeviceFactorSet, build_device_sharded, device_params,
                                       schedule_super_shards, sweep_all_modes)
    from paper_2309_09131_b200.synth import zipf_tensor
    dims = (1000, 800, 600)
    coords, vals = zipf_tensor(dims, 300_000, seed=6, exponents=(None, None, None))
    params = device_params(dims, 300_000, 16)
    monkeypatch.setenv("FLYCOO_TILE_PLAN", "0")
    ref = build_device_sharded(coords, vals, params)
    smap = schedule_super_shards(ref.plan, 1)
    fs = DeviceFactorSet.random_device(dims, 16, seed=3)
    want = sweep_all_modes(ref, fs, smap)
    monkeypatch.setenv("FLYCOO_TILE_PLAN", "1")
    st = build_device_sharded(coords, vals, params)
    got = sweep_all_modes(st, fs, smap)  # planned on its first mode-0 pass
    assert all(st.mode_work(n, 16).tile_perm is not None for n in range(3))
    for a, b in zip(got.factors, want.factors):
        assert torch.equal(a, b)
    assert torch.equal(st.crd[st.active], ref.crd[ref.active])


def test_planned_mode_passes_match_the_oracle():
    from paper_2309_09131_b200 import DeviceFactorSet, mttkrp_mode
    c = CASES["packed"]
    coords, vals, params, st, smap = _build(c["dims"], c["nnz"], c["law"], **c["kw"])
    fs = DeviceFactorSet.random_device(c["dims"], 32, seed=4)
    subs = coords.cpu().numpy().astype(np.int64)
    v64 = vals.cpu().numpy().astype(np.float64)
    f64 = [f.cpu().numpy().astype(np.float64) for f in fs.factors]
    for n in range(3):
        out = mttkrp_mode(st, fs, n, smap)
        assert st.mode_work(n, 32).tile_perm is not None  # planned on the first mode-0 pass
        assert_rel(out.cpu().numpy(), oracle.reference_mttkrp(subs, v64, f64, n), what=f"mode {n}")


def test_plan_is_skipped_where_it_does_not_apply(monkeypatch):
    """Ranks other than 16 / 32 keep the in-kernel ranking; a cursor-remapped
    (non-canonical) buffer does not use a plan emitted for the canonical order."""
    from paper_2309_09131_b200 import (DeviceFactorSet, build_device_sharded, device_params,
                                       mttkrp_mode, schedule_super_shards, sweep_all_modes)
    from paper_2309_09131_b200.engine import build_tile_plans
    from paper_2309_09131_b200.synth import zipf_tensor
    monkeypatch.setenv("FLYCOO_TILE_PLAN", "1")
    dims = (3000, 2000, 2500)
    coords, vals = zipf_tensor(dims, 200_000, seed=5, exponents=(1.1,) * 3)
    st8 = build_device_sharded(coords, vals, device_params(dims, 200_000, 8, g=4096))
    assert not build_tile_plans(st8, 8)
    smap8 = schedule_super_shards(st8.plan, 1)
    sweep_all_modes(st8, DeviceFactorSet.random_device(dims, 8, seed=1), smap8)
    assert all(w.tile_perm is None for w in st8._work.values())

    params = device_params(dims, 200_000, 32, g=4096)
    st = build_device_sharded(coords, vals, params)
    ref = build_device_sharded(coords, vals, params)
    smap = schedule_super_shards(st.plan, 1)
    fs = DeviceFactorSet.random_device(dims, 32, seed=2)
    assert build_tile_plans(st, 32)
    subs = coords.cpu().numpy().astype(np.int64)
    v64 = vals.cpu().numpy().astype(np.float64)
    f64 = [f.cpu().numpy().astype(np.float64) for f in fs.factors]
    out0 = mttkrp_mode(st, fs, 0, smap, remap="cursor")  # planned compute, cursor remap
    assert not st.canonical
    assert_rel(out0.cpu().numpy(), oracle.reference_mttkrp(subs, v64, f64, 0), what="mode 0")
    out1 = mttkrp_mode(st, fs, 1, smap, remap="cursor")  # non-canonical order: ranked in the kernel
    assert_rel(out1.cpu().numpy(), oracle.reference_mttkrp(subs, v64, f64, 1), what="mode 1")
    del ref

"""Parity at BASELINE.json's full sizes (SURVEY §8c "where the oracle does
not fit"), through the public API on one B200:

* c2 (76.9M nonzeros): every output row of every mode against the oracle's
  sequential ``reference_mttkrp`` (coo.py:406-426 restated in C), fixed
  factors;
* c3 (140M, 4 modes), c4 (1.74B) and c5 (3.6B, bucketed generator + lean
  build): a sample of output rows per mode --
  uniform rows plus moderately heavy ones that span several chunks (K2) --
  recomputed in float64 on the host from the nonzeros that carry them;
* all three: after every pass every element sits in the super-shard of its
  active mode (BufferOrderError territory, layout.py:474-497), and after N
  remaps the buffer equals the initial one bit-exactly (position-dependent
  checksum), the size-independent cycle identity.
"""
import numpy as np
import pytest
import torch

import oracle
from gpu_helpers import assert_rel

pytestmark = pytest.mark.gpu


def _checksum(crd: torch.Tensor, chunk: int = 1 << 26) -> int:
    """Position-dependent 64-bit checksum of a record buffer (wrapping int64)."""
    total = torch.zeros((), dtype=torch.int64, device=crd.device)
    cw = crd.shape[1]
    mult = torch.tensor([0x9E3779B1, 0x85EBCA77, 0xC2B2AE3D, 0x27D4EB2F, 0x165667B1, 0xD3A2646C,
                         0xFD7046C5, 0xB55A4F09][:cw], dtype=torch.int64, device=crd.device)
    for a in range(0, crd.shape[0], chunk):
        c = crd[a:a + chunk].to(torch.int64)
        pos = torch.arange(a, a + c.shape[0], dtype=torch.int64, device=crd.device)
        h = (c * mult).sum(1) ^ (pos * 0x2545F4914F6CDD1D)
        total += (h * (h | 1)).sum()
    return int(total)


def _assert_in_super_shards(st, mode: int, chunk: int = 1 << 26):
    """Every element of the active buffer lies inside its super-shard's range."""
    m = int(st.plan.params.m[mode])
    offs = torch.as_tensor(np.asarray(st.plan.ss_elem_offsets[mode]), dtype=torch.int64,
                           device=st.device)
    crd = st.crd[st.active]
    for a in range(0, crd.shape[0], chunk):
        iv = crd[a:a + chunk, mode].to(torch.int64) // m
        pos = torch.arange(a, a + iv.shape[0], dtype=torch.int64, device=st.device)
        ok = (pos >= offs[iv]) & (pos < offs[iv + 1])
        assert bool(ok.all()), f"mode {mode}: element outside its super-shard near {a}"


def _sample_rows(st, mode: int, rows: np.ndarray, factors64):
    """float64 MTTKRP of `rows` from the nonzeros of the active buffer."""
    N = st.num_modes
    dim = st.plan.params.dims[mode]
    lut = torch.zeros(dim, dtype=torch.bool, device=st.device)
    lut[torch.as_tensor(rows, device=st.device)] = True
    crd = st.crd[st.active]
    sel_c, sel_v = [], []
    for a in range(0, crd.shape[0], 1 << 26):
        c = crd[a:a + (1 << 26)]
        keep = lut[c[:, mode].to(torch.int64)]
        cs = c[keep]
        sel_c.append(cs[:, :N].cpu())
        if st.val[st.active] is None:
            sel_v.append(cs[:, 3].view(torch.float32).cpu())
        else:
            sel_v.append(st.val[st.active][a:a + (1 << 26)][keep].cpu())
    subs = torch.cat(sel_c).numpy().astype(np.int64)
    vals = torch.cat(sel_v).numpy().astype(np.float64)
    R = factors64[0].shape[1]
    out = torch.zeros((dim, R), dtype=torch.float64)
    for a in range(0, len(vals), 1 << 22):
        s = subs[a:a + (1 << 22)]
        t = vals[a:a + (1 << 22), None]
        for w in range(N):
            if w != mode:
                t = t * factors64[w][s[:, w]]
        out.index_add_(0, torch.from_numpy(s[:, mode]), torch.from_numpy(t))
    return out.numpy()[rows], len(vals)


def _run(cfg: int, full_oracle: bool):
    from paper_2309_09131_b200 import (DeviceFactorSet, build_device_sharded, device_params,
                                       mttkrp_mode, schedule_super_shards)
    from paper_2309_09131_b200.synth import CONFIGS, config_tensor
    torch.cuda.empty_cache()
    c = CONFIGS[cfg]
    dims, R = tuple(c["dims"]), 32
    if cfg == 5:  # 3.6B nonzeros: bucketed generator + lean build (158 GB resident)
        from paper_2309_09131_b200.layout import build_device_sharded_lean
        from paper_2309_09131_b200.synth import zipf_records_bucketed
        rec = zipf_records_bucketed(dims, c["nnz"], seed=cfg, exponents=c["law"])
        params = device_params(dims, c["nnz"], R)
        st = build_device_sharded_lean(rec, params)
        del rec
    else:
        coords, vals = config_tensor(cfg)
        params = device_params(dims, int(vals.shape[0]), R)
        if full_oracle:
            subs = coords.cpu().numpy().astype(np.int64)
            v64 = vals.cpu().numpy().astype(np.float64)
        st = build_device_sharded(coords, vals, params)
        del coords, vals
    torch.cuda.empty_cache()
    smap = schedule_super_shards(st.plan, 1)
    fs = DeviceFactorSet.random_device(dims, R, seed=2000 + cfg)
    f64 = [f.double().cpu().numpy() for f in fs.factors]
    start = _checksum(st.crd[st.active])
    rng = np.random.default_rng(cfg)
    N = len(dims)
    for n in range(N):
        _assert_in_super_shards(st, n)
        if full_oracle:
            want = oracle.reference_mttkrp(subs, v64, f64, n)
            got = mttkrp_mode(st, fs, n, smap)
            assert_rel(got.double().cpu().numpy(), want, what=f"c{cfg} mode {n}")
        else:
            rows = np.unique(np.concatenate([
                rng.integers(0, dims[n], 48),
                [r for r in (100, 1000, 20000) if r < dims[n]],
                [dims[n] - 1]]))
            if cfg == 5 and n == 0:  # 46 rows of 78M nonzeros each: two of them
                rows = np.array([3, dims[0] - 1])
            want, cnt = _sample_rows(st, n, rows, f64)
            got = mttkrp_mode(st, fs, n, smap)
            assert cnt > 0
            assert_rel(got[torch.as_tensor(rows, device=got.device)].double().cpu().numpy(), want,
                       what=f"c{cfg} mode {n} sampled rows")
    _assert_in_super_shards(st, 0)
    assert _checksum(st.crd[st.active]) == start, f"c{cfg}: cycle identity broken"


def test_c2_full_every_row():
    _run(2, full_oracle=True)


def test_c3_full_sampled_rows():
    _run(3, full_oracle=False)


def test_c4_full_sampled_rows():
    _run(4, full_oracle=False)


def test_c5_full_sampled_rows():
    """3.6B nonzeros, 46 mode-0 rows of ~78M nonzeros each (heavy rows split
    over ~9.5k chunks each, two-level K2)."""
    _run(5, full_oracle=False)

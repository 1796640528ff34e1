"""Shared helpers of the GPU parity tests (oracle = checker only)."""
import numpy as np
import torch

import oracle
from paper_2309_09131_b200 import (DeviceFactorSet, PartitionParams, build_device_sharded,
                                   default_element_bytes, schedule_super_shards)

RTOL = 1e-4  # north_star: MTTKRP rows within rel. 1e-4 in fp32


def params_of(dims, nnz, m, k, g, rank, nu=1):
    N = len(dims)
    return PartitionParams(dims=tuple(int(d) for d in dims), nnz=int(nnz),
                           m=tuple(int(x) for x in m), k=tuple(int(x) for x in k), g=int(g),
                           nu=int(nu), gamma=1 << 20, theta=0.5, rank=int(rank), alpha=8,
                           beta=default_element_bytes(N), sigma=8)


def host_records(st, which=None):
    """(coords int64 (nnz, N), value bits uint32) of a device buffer."""
    b = st.active if which is None else which
    N = st.num_modes
    crd = st.crd[b].cpu()
    c = crd[:, :N].to(torch.int64).numpy()
    if st.val[b] is None:
        vb = crd[:, -1].numpy().view(np.uint32)
    else:
        vb = st.val[b].cpu().numpy().view(np.uint32)
    return c, vb


def oracle_records(t):
    s, i, v = t.active_arrays()
    return i, v.astype(np.float32).view(np.uint32)


def assert_rel(got, want, rtol=RTOL, what=""):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape, (got.shape, want.shape)
    scale = np.maximum(np.abs(got), np.abs(want))
    bad = np.abs(got - want) > rtol * scale
    assert not bad.any(), f"{what}: {bad.sum()} of {bad.size} entries off; worst rel " \
        f"{float((np.abs(got - want) / np.where(scale > 0, scale, 1)).max()):.3e}"
    # empty rows must be exactly zero
    zero_rows = np.all(want == 0, axis=1)
    assert np.all(got[zero_rows] == 0), f"{what}: empty rows not exactly zero"


def factors_f32(dims, rank, seed):
    rng = np.random.Generator(np.random.Philox(seed))
    return [rng.random((int(d), rank)).astype(np.float32) for d in dims]


# --------------------------------------------------------- shard digests (GPU)

def _s64(x: int) -> int:
    return ((x + (1 << 63)) % (1 << 64)) - (1 << 63)


_M1 = _s64(0xBF58476D1CE4E5B9)
_M2 = _s64(0x94D049BB133111EB)
_H0 = _s64(0x9E3779B97F4A7C15)


def _mix64_t(x: torch.Tensor) -> torch.Tensor:
    """orc_mix64 on int64 tensors (uint64 arithmetic in two's complement;
    logical right shifts through masks)."""
    x = x ^ ((x >> 30) & ((1 << 34) - 1))
    x = x * _M1
    x = x ^ ((x >> 27) & ((1 << 37) - 1))
    x = x * _M2
    return x ^ ((x >> 31) & ((1 << 33) - 1))


def elem_hash_t(coords: torch.Tensor, vbits: torch.Tensor) -> torch.Tensor:
    """oracle.elem_hash on the device: coords (n, N) int32, vbits (n,) int32."""
    h = torch.full((coords.shape[0],), _H0, dtype=torch.int64, device=coords.device)
    for w in range(coords.shape[1]):
        h = _mix64_t(h ^ (coords[:, w].to(torch.int64) & 0xFFFFFFFF))
    v = vbits.to(torch.int64) & 0xFFFFFFFF
    return _mix64_t(h ^ ((v << 32) | 0x5BD1E995))


def device_shard_digests(st, mode: int, chunk: int = 1 << 27):
    """Per-shard (hash uint64, count) of the active buffer, which must be in
    `mode` order: shard s = positions [shard_offsets[s], shard_offsets[s+1])."""
    assert st.active_mode == mode
    N = st.num_modes
    offs = torch.as_tensor(st.plan.shard_offsets[mode], device=st.device)
    nsh = int(offs.shape[0]) - 1
    acc = torch.zeros(nsh, dtype=torch.int64, device=st.device)
    crd, val = st.crd[st.active], st.val[st.active]
    for lo in range(0, st.nnz, chunk):
        hi = min(st.nnz, lo + chunk)
        c = crd[lo:hi, :N]
        vb = crd[lo:hi, -1] if val is None else val[lo:hi].view(torch.int32)
        pos = torch.arange(lo, hi, device=st.device, dtype=torch.int64)
        sid = torch.searchsorted(offs, pos, right=True) - 1
        acc.index_add_(0, sid, elem_hash_t(c, vb))
    cnt = (offs[1:] - offs[:-1]).cpu().numpy()
    return acc.cpu().numpy().view(np.uint64), cnt

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

"""The per-rank (partitioned) FLYCOO build on CPU ranks over gloo, world 2
and 3: each rank starts from a contiguous block of the input COO and must
end with exactly the slices of the single-GPU layout -- mode-0 records and
every mode's global slot-map slice -- that the fused exchange would cut from
it (oracle.device_order restates that layout, pinned to the reference), and
the same plan.  No rank holds the global layout."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from test_dist import _global_records


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(N, nnz=40_000):
    from paper_2309_09131_b200.params import device_params
    from paper_2309_09131_b200.synth import zipf_tensor_host
    if N == "c5":  # c5's shape of skew: mode 0 has 46 rows -> two super-shards
        dims = (46, 3000, 3000)
        subs, vals = zipf_tensor_host(dims, nnz, seed=12, exponents=(None, 1.0, 1.0))
        return dims, subs, vals, device_params(dims, len(vals), 8, g=1024, m=[32, 16, 16])
    dims = {3: (900, 700, 800), 4: (120, 150, 90, 60)}[N]
    subs, vals = zipf_tensor_host(dims, nnz, seed=11, exponents=(1.1,) * N)
    params = device_params(dims, len(vals), 8, g=1024, m=[16] * N)
    return dims, subs, vals, params


def _worker(rank, world, port, N, result):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2309_09131_b200.distbuild import build_partitioned
        from paper_2309_09131_b200.peer import PeerShardedTensor, slice_bounds
        dims, subs, vals, params = _case(N)
        nnz = len(vals)
        N = len(dims)
        # uneven input blocks
        cuts = np.linspace(0, nnz, world + 1).astype(np.int64)
        cuts[1:-1] += np.arange(1, world) * 37
        lo, hi = int(cuts[rank]), int(cuts[rank + 1])
        loc = build_partitioned(torch.from_numpy(subs[lo:hi]), torch.from_numpy(vals[lo:hi]), lo,
                                params, R=8, device="cpu")
        L = oracle.canonical_build(subs, vals.astype(np.float64), dims, params.m, params.k,
                                   params.g)
        d = oracle.device_order(L)
        for n in range(N):
            assert np.array_equal(loc.plan.shard_offsets[n], L.shard_offsets[n]), n
            assert np.array_equal(loc.plan.ss_counts[n], L.ss_counts[n]), n
        bounds = slice_bounds(loc.plan, world, 8, "cpu")
        assert bounds == loc.bounds
        for n in range(N):
            a, b = bounds[n][rank], bounds[n][rank + 1]
            got = loc.slots[n].numpy().view(np.uint32).astype(np.int64)
            assert np.array_equal(got, d.slot_maps[n][a:b]), (rank, n)
        rec, val = _global_records(subs, vals, d.orders[0], N)
        a, b = bounds[0][rank], bounds[0][rank + 1]
        assert np.array_equal(loc.crd0.numpy(), rec[a:b]), rank
        if val is not None:
            assert np.array_equal(loc.val0.numpy(), val[a:b]), rank
        # the sample sort spreads heavy super-shards: no rank sorts much more
        # than its share (c5 shape: 2 super-shards in mode 0, 3 ranks)
        assert max(loc.received) <= 1.25 * nnz / world + 2048, loc.received
        # the fused exchange takes it like a sliced global tensor
        pt = PeerShardedTensor(loc, world, rank, ipc=False, R=8)
        for n in range(N):
            p = pt.plans[n]
            assert np.array_equal(p.global_slots.numpy().view(np.uint32).astype(np.int64),
                                  d.slot_maps[n][p.e_lo:p.e_hi])
        result[rank] = 1
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,N", [(2, 3), (3, 3), (2, 4), (3, "c5")])
def test_partitioned_build_equals_global_slices(world, N):
    ctx = mp.get_context("spawn")
    result = ctx.Manager().dict()
    mp.start_processes(_worker, args=(world, _free_port(), N, result), nprocs=world, join=True,
                       start_method="spawn")
    assert sorted(result.keys()) == list(range(world))


def test_morton_key_matches_oracle():
    from paper_2309_09131_b200.distbuild import morton_key
    rng = np.random.default_rng(2)
    k = (700, 33, 5000, 2)
    iv = np.stack([rng.integers(0, x, 5000) for x in k], 1)
    hi, lo = oracle.morton_interleave(iv, k)
    assert not hi.any()
    got = morton_key(torch.from_numpy(iv), k).numpy().view(np.uint64)
    assert np.array_equal(got, lo)


def test_sample_index_stays_in_range():
    """Sample positions for the splitters at the bench's block sizes (c2 at
    2 ranks: 38.45M elements per rank; c5 at 8: 450M): float linspace would
    round the last index to n."""
    from paper_2309_09131_b200.distbuild import _sample_index
    for n in (1, 2, 1023, 1024, 38_450_000, 450_000_000, 3_600_000_000):
        idx = _sample_index(n, 1024, "cpu")
        assert int(idx.min()) == 0 and int(idx.max()) == n - 1
        assert bool((idx[1:] >= idx[:-1]).all())

"""Host logic of the fused remap + exchange (peer.py) on CPU: virtual ranks
in one process, the device store emulated with torch exactly as
``remap_store`` resolves it (owner q from the peer bounds, local position
d - E'_q).  Every rank's slice after every mode must equal the single-GPU
layout, and the pulled factors must equal the single-process sweep (oracle
reference_mttkrp).  The CUDA path is tests/test_gpu_peer.py."""
import types

import numpy as np
import pytest
import torch

import oracle
from paper_2309_09131_b200.peer import PeerShardedTensor, peer_plans
from test_dist import _case, _global_records


def _emulated_pass(ranks, r, factors, mode, contrib):
    """K1 of virtual rank r: its chunks' contributions to the output rows
    (into `contrib`, full size) + peer stores of every record."""
    dt = ranks[r]
    p = dt.plans[mode]
    a, b = dt.active, 1 - dt.active
    recs = dt.crd[a][:p.count]
    N = dt.num_modes
    v = recs[:, 3].view(torch.float32).double() if dt.val[a] is None else dt.val[a][:p.count].double()
    t = v[:, None].clone()
    for w in range(N):
        if w != mode:
            t = t * factors[w][recs[:, w].long()]
    contrib.index_add_(0, recs[:, mode].long(), t.to(contrib.dtype))
    d = p.global_slots.long() & 0xFFFFFFFF
    base = torch.tensor(p.peer_base)
    q = torch.searchsorted(base, d, right=True) - 1
    assert bool(((q >= 0) & (q < dt.world)).all())
    for qq in range(dt.world):
        sel = q == qq
        l = d[sel] - base[qq]
        ranks[qq].crd[b][l] = recs[sel]
        if dt.val[b] is not None:
            ranks[qq].val[b][l] = dt.val[a][:p.count][sel]


@pytest.mark.parametrize("world,N", [(2, 3), (3, 3), (2, 4), (4, 3)])
def test_peer_sweep_virtual_ranks_cpu(world, N):
    dims, subs, vals, params, L, d, plan = _case(N)
    rec0, val0 = _global_records(subs, vals, d.orders[0], N)
    st = types.SimpleNamespace(
        plan=plan, device=torch.device("cpu"), num_modes=N, active=0,
        slot_maps=[torch.from_numpy(s.astype(np.int64)) for s in d.slot_maps],
        crd=[torch.from_numpy(rec0), None],
        val=[None if val0 is None else torch.from_numpy(val0), None])
    ranks = [PeerShardedTensor(st, world, r, ipc=False, R=8) for r in range(world)]
    rng = np.random.default_rng(9)
    f0 = [torch.from_numpy(rng.random((dd, 8))) for dd in dims]
    working = [list(f0) for _ in range(world)]
    for n in range(N):
        contrib = [torch.zeros((dims[n], 8), dtype=torch.float64) for _ in range(world)]
        for r in range(world):
            _emulated_pass(ranks, r, working[r], n, contrib[r])
        total = sum(contrib)  # owners reduce split super-shards; the gather spreads rows
        rb = ranks[0].plans[n].row_bounds
        assert rb[0] == 0 and rb[-1] == dims[n] and all(x <= y for x, y in zip(rb, rb[1:]))
        for r, dt in enumerate(ranks):
            dt.swap()
            working[r][n] = total.clone()
        nxt = (n + 1) % N
        want, wval = _global_records(subs, vals, d.orders[nxt], N)
        for r, dt in enumerate(ranks):
            p = dt.plans[nxt]
            got, gval = dt.local_records()
            assert np.array_equal(got.numpy(), want[p.e_lo:p.e_hi]), (r, n)
            if wval is not None:
                assert np.array_equal(gval.numpy(), wval[p.e_lo:p.e_hi]), (r, n)
    ref = [f.numpy() for f in f0]
    v64 = vals.astype(np.float32).astype(np.float64)
    for n in range(N):
        ref[n] = oracle.reference_mttkrp(subs, v64, ref, n)
        for r in range(world):
            np.testing.assert_allclose(working[r][n].numpy(), ref[n], rtol=1e-9, atol=0)


def test_peer_plans_cover_every_slot_once():
    dims, subs, vals, params, L, d, plan = _case(3)
    slot_maps = [torch.from_numpy(s.astype(np.int64)) for s in d.slot_maps]
    for world in (1, 2, 5, 8):
        per_rank = [peer_plans(plan, slot_maps, world, r, 8, "cpu")[0] for r in range(world)]
        for n in range(3):
            base = per_rank[0][n].peer_base
            assert len(base) == world + 1 and base[0] == 0 and base[-1] == len(vals)
            allslots = torch.cat([pr[n].global_slots.long() for pr in per_rank])
            assert torch.equal(torch.sort(allslots).values, torch.arange(len(vals)))
            # every rank's bounds are the same static table
            assert all(pr[n].peer_base == base for pr in per_rank)
            # chunk ranges tile the chunk list; each super-shard has one owner
            assert per_rank[0][n].c_lo == 0
            for a, b in zip(per_rank, per_rank[1:]):
                assert a[n].c_hi == b[n].c_lo and a[n].ss_hi == b[n].ss_lo
            assert per_rank[-1][n].ss_hi == params.k[n]


def test_peer_world_limit():
    dims, subs, vals, params, L, d, plan = _case(3)
    st = types.SimpleNamespace(plan=plan, device=torch.device("cpu"), num_modes=3, active=0,
                               slot_maps=[torch.zeros(1)] * 3, crd=[None, None], val=[None, None])
    with pytest.raises(ValueError, match="at most 8"):
        PeerShardedTensor(st, 9, 0, ipc=False)


def test_chunk_partition_balances_a_heavy_super_shard():
    """A super-shard holding most nonzeros is split across GPUs at chunk
    granularity; its rows (and K2 tasks) stay with the GPU of its first chunk."""
    from paper_2309_09131_b200.layout import make_mode_work, plan_from_counts
    from paper_2309_09131_b200.params import device_params
    from paper_2309_09131_b200.peer import partition_chunks, super_shard_owners
    dims = (640, 50, 50)
    rng = np.random.default_rng(3)
    n0, n1 = 30_000, 20_000  # ~60% of the nonzeros in super-shard 0 (rows < 64)
    c0 = np.stack([rng.integers(0, 64, n0), rng.integers(0, 50, n0), rng.integers(0, 50, n0)], 1)
    c1 = np.stack([rng.integers(64, 640, n1), rng.integers(0, 50, n1), rng.integers(0, 50, n1)], 1)
    subs = np.unique(np.concatenate([c0, c1]), axis=0)
    params = device_params(dims, len(subs), 8, g=1024, m=[64, 16, 16])
    counts = [np.bincount(subs[:, w] // params.m[w], minlength=params.k[w]) for w in range(3)]
    plan = plan_from_counts(params, counts)
    w = make_mode_work(plan, 0, 8, "cpu", chunk_elems=2048)
    cs = w.chunk_start.numpy()
    for world in (2, 4, 8):
        # pure nonzero balance (chunk_weight 0): within one chunk of the ideal
        loads = np.diff(cs[partition_chunks(cs, world, chunk_weight=0)])
        assert loads.max() <= len(subs) / world + 2048, (world, loads)
        # default: nonzeros + a fixed cost per chunk, balanced within one chunk's cost
        cb = partition_chunks(cs, world)
        nch = len(cs) - 1
        kw = 2048
        costs = np.diff(cs[cb]) + kw * np.diff(cb)
        assert costs.max() <= (len(subs) + kw * nch) / world + 2048 + kw, (world, costs)
        gpu = np.repeat(np.arange(world), np.diff(cb))
        owner = super_shard_owners(w, params.k[0], 64, gpu, world)
        assert owner[0] == 0 and np.all(np.diff(owner) >= 0)
        # the heavy super-shard's chunks run on several GPUs once it holds more
        # than one GPU's share of the cost (at world 2 the cut may land on its end)
        if world >= 4:
            assert len(set(gpu[w.chunk_ss.numpy() == 0])) > 1

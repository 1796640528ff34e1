"""Multi-rank logic of the distributed sweep (dist.py) on CPU with gloo,
world size 2 and 3: every rank's slice after every remap equals the
single-GPU layout's slice bit-exactly, and the all-gathered updated factors
equal the single-process sweep.  Local kernels are emulated with torch here
(the CUDA kernels are covered by the GPU parity tests); the plan, the
exchange (all_to_all_single) and the factor all-gather are the product code."""
import os
import socket
import types

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2309_09131_b200.dist import (DistShardedTensor, dist_sweep_all_modes,
                                        partition_super_shards)
from paper_2309_09131_b200.layout import plan_from_counts
from paper_2309_09131_b200.params import device_params
from paper_2309_09131_b200.synth import zipf_tensor_host


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(N=3):
    dims = (300, 200, 250) if N == 3 else (60, 70, 50, 40)
    law = (1.1,) * N
    subs, vals = zipf_tensor_host(dims, 30_000, seed=4, exponents=law)
    params = device_params(dims, len(vals), 8, g=512, m=[7] * N)
    L = oracle.canonical_build(subs, vals.astype(np.float64), dims, params.m, params.k, params.g)
    d = oracle.device_order(L)
    plan = plan_from_counts(params, L.ss_counts)
    return dims, subs, vals, params, L, d, plan


def _global_records(subs, vals, order, N):
    cw = 4
    rec = np.zeros((len(order), cw), dtype=np.int32)
    rec[:, :N] = subs[order]
    emb = N < cw
    if emb:
        rec[:, cw - 1] = vals[order].astype(np.float32).view(np.int32)
        return rec, None
    return rec, vals[order].astype(np.float32)


class TorchOps:
    """CPU emulation of the two local kernels (K1 compute+remap, unpack)."""

    def mode_pass(self, dt, factors, mode, out):
        p = dt.plans[mode]
        a, b = dt.active, 1 - dt.active
        recs = dt.crd[a][:p.count]
        N = dt.num_modes
        if dt.val[a] is None:
            v = recs[:, 3].view(torch.float32).double()
        else:
            v = dt.val[a][:p.count].double()
        t = v[:, None].clone()
        for w in range(N):
            if w != mode:
                t = t * factors[w][recs[:, w].long()]
        out.index_add_(0, recs[:, mode].long(), t.to(out.dtype))
        slots = p.local_slots.long() & 0xFFFFFFFF
        dt.crd[b][slots] = recs
        if dt.val[b] is not None:
            dt.val[b][slots] = dt.val[a][:p.count]

    def scatter(self, dt, mode):
        p = dt.plans[mode]
        b = 1 - dt.active
        m = p.recv_map.long()
        dt.crd[b][m] = dt.recv_crd[:p.recv_total]
        if dt.val[b] is not None:
            dt.val[b][m] = dt.recv_val[:p.recv_total]


def _worker(rank, world, port, N, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dims, subs, vals, params, L, d, plan = _case(N)
        rec0, val0 = _global_records(subs, vals, d.orders[0], N)
        st = types.SimpleNamespace(
            plan=plan, device=torch.device("cpu"), num_modes=N, active=0,
            slot_maps=[torch.from_numpy(s.astype(np.int64)) for s in d.slot_maps],
            crd=[torch.from_numpy(rec0), None],
            val=[None if val0 is None else torch.from_numpy(val0), None])
        dt = DistShardedTensor(st, world, rank)
        rng = np.random.default_rng(9)
        f0 = [torch.from_numpy(rng.random((dd, 8))) for dd in dims]
        # the distributed sweep, checking each rank's slice after every mode
        working = list(f0)
        for n in range(N):
            from paper_2309_09131_b200.dist import allgather_rows, dist_mttkrp_mode
            out = dist_mttkrp_mode(dt, working, n, TorchOps())
            working[n] = allgather_rows(dt, n, out)
            nxt = (n + 1) % N
            want, wval = _global_records(subs, vals, d.orders[nxt], N)
            p = dt.plans[nxt]
            got, gval = dt.local_records()
            assert np.array_equal(got.numpy(), want[p.e_lo:p.e_hi]), (rank, n)
            if wval is not None:
                assert np.array_equal(gval.numpy(), wval[p.e_lo:p.e_hi])
        # single-process chain (oracle reference_mttkrp, fp64)
        ref = [f.numpy() for f in f0]
        v64 = vals.astype(np.float32).astype(np.float64)
        for n in range(N):
            ref[n] = oracle.reference_mttkrp(subs, v64, ref, n)
            np.testing.assert_allclose(working[n].double().numpy(), ref[n], rtol=1e-5, atol=0)  # fp32 out
        result[rank] = 1
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,N", [(2, 3), (3, 3), (2, 4)])
def test_dist_sweep_gloo(world, N):
    ctx = mp.get_context("spawn")
    result = ctx.Manager().dict()
    mp.start_processes(_worker, args=(world, _free_port(), N, result), nprocs=world, join=True,
                       start_method="spawn")
    assert sorted(result.keys()) == list(range(world))


def test_partition_never_splits_super_shards():
    counts = np.array([50, 0, 3, 7, 100, 1, 1, 1, 20, 0, 0, 9])
    for world in (1, 2, 3, 5, 12, 20):
        sb, eb = partition_super_shards(counts, world)
        assert sb[0] == 0 and sb[-1] == len(counts) and np.all(np.diff(sb) >= 0)
        cum = np.concatenate(([0], np.cumsum(counts)))
        assert np.array_equal(eb, cum[sb])

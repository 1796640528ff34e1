"""GPU: the per-rank partitioned build (distbuild.build_partitioned) feeding
the fused exchange, two processes sharing the GPU (gloo for the host-side
exchanges, host barriers): each rank's slices equal the global build's
bit-exactly, and chained sweeps over the fused exchange equal the
single-GPU sweep bit-exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, result):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), FLYCOO_PEER_SYNC="host")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2309_09131_b200 import (DeviceFactorSet, build_device_sharded, device_params,
                                           mttkrp_mode, schedule_super_shards)
        from paper_2309_09131_b200.distbuild import build_partitioned
        from paper_2309_09131_b200.peer import PeerShardedTensor, peer_sweep_all_modes
        from paper_2309_09131_b200.synth import zipf_tensor
        for N, dims in ((3, (3000, 2000, 2500)), (4, (300, 400, 250, 90))):
            nnz = 300_000
            coords, vals = zipf_tensor(dims, nnz, seed=6, exponents=(1.1,) * N)
            params = device_params(dims, nnz, 32, g=4096, m=[16] * N)
            lo, hi = nnz * rank // world, nnz * (rank + 1) // world
            loc = build_partitioned(coords[lo:hi], vals[lo:hi], lo, params, R=32)
            ref = build_device_sharded(coords, vals, params)
            for n in range(N):
                b = loc.bounds[n]
                assert torch.equal(loc.slots[n], ref.slot_maps[n][b[rank]:b[rank + 1]]), (N, n)
            b = loc.bounds[0]
            assert torch.equal(loc.crd0, ref.crd[0][b[rank]:b[rank + 1]]), N
            if loc.val0 is not None:
                assert torch.equal(loc.val0, ref.val[0][b[rank]:b[rank + 1]]), N
            dt = PeerShardedTensor(loc, world, rank)
            dt.connect()
            f0 = DeviceFactorSet.random_device(dims, 32, seed=3)
            got, working = list(f0.factors), list(f0.factors)
            smap = schedule_super_shards(ref.plan, 1)
            for _ in range(2):
                got = [g.clone() for g in peer_sweep_all_modes(dt, got)]
                for n in range(N):
                    working[n] = mttkrp_mode(ref, DeviceFactorSet(working, None, validate=False),
                                             n, smap)
                for n in range(N):
                    assert torch.equal(got[n], working[n]), (rank, N, n)
            dt.barrier()
            dt.close()
            dist.barrier()
        result[rank] = 1
    finally:
        dist.destroy_process_group()


def test_partitioned_build_feeds_fused_exchange():
    world = 2
    ctx = mp.get_context("spawn")
    result = ctx.Manager().dict()
    mp.start_processes(_worker, args=(world, _free_port(), result), nprocs=world, join=True,
                       start_method="spawn")
    assert sorted(result.keys()) == list(range(world))

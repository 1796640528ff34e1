"""The distributed sweep's CUDA kernels (K1 writing local slots + the send
region, the receiver scatter) on one GPU with two ranks.  The ranks' kernels
never wait on each other; only the exchange is staged through host memory
with gloo (NCCL needs one GPU per rank).  Each rank's slice must equal the
single-GPU layout after every mode and the outputs must equal the
single-GPU sweep bitwise."""
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
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2309_09131_b200 import (DeviceFactorSet, build_device_sharded, device_params,
                                           schedule_super_shards, sweep_all_modes)
        from paper_2309_09131_b200.dist import (CudaOps, DistShardedTensor, dist_mttkrp_mode)
        from paper_2309_09131_b200.synth import zipf_tensor

        class StagedOps(CudaOps):
            def exchange(self, dt, mode):
                p = dt.plans[mode]
                b = 1 - dt.active
                send = dt.crd[b][dt.cap:dt.cap + p.send_total].cpu()
                recv = torch.empty((p.recv_total, send.shape[1]), dtype=send.dtype)
                dist.all_to_all_single(recv, send, p.recv_counts, p.send_counts)
                dt.recv_crd[:p.recv_total] = recv.cuda()
                if dt.val[b] is not None:
                    sv = dt.val[b][dt.cap:dt.cap + p.send_total].cpu()
                    rv = torch.empty(p.recv_total, dtype=sv.dtype)
                    dist.all_to_all_single(rv, sv, p.recv_counts, p.send_counts)
                    dt.recv_val[:p.recv_total] = rv.cuda()

            def allgather(self, dt, mode, out):
                parts = [torch.empty_like(out.cpu()) for _ in range(dt.world)]
                dist.all_gather(parts, out.cpu())
                full = torch.empty_like(out)
                for r in range(dt.world):
                    lo = min(int(dt.bounds[mode][0][r]) * dt.plan.params.m[mode], out.shape[0])
                    hi = min(int(dt.bounds[mode][0][r + 1]) * dt.plan.params.m[mode], out.shape[0])
                    full[lo:hi] = parts[r][lo:hi].cuda()
                return full

        torch.cuda.set_device(0)
        for N, dims in ((3, (3000, 2000, 2500)), (4, (300, 400, 250, 90))):
            coords, vals = zipf_tensor(dims, 400_000, seed=6, exponents=(1.1,) * N)
            params = device_params(dims, 400_000, 32, g=4096, m=[16] * N)
            st = build_device_sharded(coords, vals, params)
            ref_st = build_device_sharded(coords, vals, params)
            dt = DistShardedTensor(st, world, rank)
            f0 = DeviceFactorSet.random_device(dims, 32, seed=3)
            ops = StagedOps()
            working = list(f0.factors)
            ref_working = list(f0.factors)
            smap = schedule_super_shards(ref_st.plan, 1)
            from paper_2309_09131_b200 import mttkrp_mode
            for n in range(N):
                out = dist_mttkrp_mode(dt, working, n, ops)
                working[n] = ops.allgather(dt, n, out)
                ref_out = mttkrp_mode(ref_st, DeviceFactorSet(ref_working, None, validate=False), n, smap)
                ref_working[n] = ref_out
                p = dt.plans[(n + 1) % N]
                got, gval = dt.local_records()
                assert torch.equal(got, ref_st.crd[ref_st.active][p.e_lo:p.e_hi]), (rank, N, n)
                # merged-chunk grouping may differ at rank boundaries: fp32 reassociation only
                assert torch.allclose(working[n], ref_out, rtol=1e-5, atol=0), (rank, N, n)
            ops.check(dt)
        result[rank] = 1
    finally:
        dist.destroy_process_group()


def test_dist_cuda_kernels_two_ranks_one_gpu():
    ctx = mp.get_context("spawn")
    result = ctx.Manager().dict()
    mp.start_processes(_worker, args=(2, _free_port(), result), nprocs=2, join=True,
                       start_method="spawn")
    assert sorted(result.keys()) == [0, 1]

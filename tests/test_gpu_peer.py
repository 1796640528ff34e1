"""Fused remap + exchange over peer memory (peer.py, fc_mode_worker_peers).

1. Virtual ranks in one process on one GPU: every rank's pass stores its
   records straight into the owners' back buffers through the peer table
   (ordinary device allocations here) and the partial tiles of split
   super-shards into their owners' workspaces; after every mode each rank's
   slice equals the single-GPU layout and the gathered factor equals the
   single-GPU sweep's, both bit-exactly.
2. Two processes sharing the GPU through CUDA IPC (gloo for the host-side
   handle exchange and the barrier): the real mapping path.  The ranks'
   kernels never wait on each other -- the barrier is on the host.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _case(N, nnz=400_000, m=16):
    from paper_2309_09131_b200 import build_device_sharded, device_params
    from paper_2309_09131_b200.synth import zipf_tensor
    dims = {3: (3000, 2000, 2500), 4: (300, 400, 250, 90), 5: (60, 50, 40, 30, 20)}[N]
    coords, vals = zipf_tensor(dims, nnz, seed=6, exponents=(1.1,) * N)
    params = device_params(dims, nnz, 32, g=4096, m=[m] * N)
    return dims, coords, vals, params, build_device_sharded


def _virtual_sweep(N, world, sweeps=2, m=16):
    from paper_2309_09131_b200 import DeviceFactorSet, mttkrp_mode, schedule_super_shards
    from paper_2309_09131_b200.peer import PeerShardedTensor
    dims, coords, vals, params, build = _case(N, m=m)
    st = build(coords, vals, params)
    ref = build(coords, vals, params)
    ranks = [PeerShardedTensor(st, world, r, ipc=False) for r in range(world)]
    PeerShardedTensor.connect_local(ranks)
    # the Zipf head super-shard is split: some GPU runs chunks another owns
    # (shared-memory accumulator tiles; global accumulation never splits)
    assert not ranks[0].works[0].acc_in_smem or any(bool((dt.plans[n].chunk_owner != dt.rank).any())
               for dt in ranks for n in range(N)), "no split super-shard in this case"
    f0 = DeviceFactorSet.random_device(dims, 32, seed=3)
    working = [list(f0.factors) for _ in range(world)]
    ref_working = list(f0.factors)
    smap = schedule_super_shards(ref.plan, 1)
    for _ in range(sweeps):
        for n in range(N):
            outs = [dt.output(n, 32)[0] for dt in ranks]
            # one stream orders the virtual GPUs: all K1, all K2, all gathers
            for r, dt in enumerate(ranks):
                dt.mode_pass(working[r], n, outs[r])
            for r, dt in enumerate(ranks):
                dt.reduce(n, outs[r])
            ptrs = [o.data_ptr() for o in outs]
            for r, dt in enumerate(ranks):
                dt.pull_rows(n, outs[r], ptrs)
                dt.swap()
                working[r][n] = outs[r]
            torch.cuda.synchronize()
            ref_out = mttkrp_mode(ref, DeviceFactorSet(ref_working, None, validate=False), n, smap)
            ref_working[n] = ref_out
            nxt = (n + 1) % N
            for r, dt in enumerate(ranks):
                p = dt.plans[nxt]
                got, gval = dt.local_records()
                assert torch.equal(got, ref.crd[ref.active][p.e_lo:p.e_hi]), (world, N, n, r)
                if gval is not None:
                    assert torch.equal(gval, ref.val[ref.active][p.e_lo:p.e_hi]), (world, N, n, r)
                # same chunks, partial tiles and reduce order as one GPU: bitwise
                assert torch.equal(working[r][n], ref_out), (world, N, n, r)
    for dt in ranks:
        dt.check()
    # the 3- and 4-mode shared-memory plans ran on tile plans emitted per slice
    # (PeerShardedTensor._tile_plan): still bitwise the single-GPU results
    if N in (3, 4) and ranks[0].works[0].acc_in_smem and os.environ.get("FLYCOO_TILE_PLAN") != "0":
        assert all(dt._tile_plans.get(n) is not None for dt in ranks for n in range(N)
                   if dt.plans[n].count > 0)


@pytest.mark.parametrize("world", [2, 3])
def test_peer_store_virtual_ranks_global_accumulator(world):
    """m = 600 rows at R = 32 (75 KB tiles): the general kernel accumulates
    in `out`, which PeerShardedTensor reuses across sweeps -- the owned rows
    must be re-zeroed every pass (second sweep bit-exact)."""
    torch.cuda.set_device(0)
    _virtual_sweep(3, world, sweeps=2, m=600)


def test_stream_wait_flush_query_and_graph_capture():
    """The flush capability is a per-device attribute query (no failing
    wait probes); a signal + wait pair on the same stream captures into a
    CUDA graph and replays."""
    from paper_2309_09131_b200 import _lib
    torch.cuda.set_device(0)
    L = _lib.load()
    assert L.fc_stream_wait_flush_supported() in (0, 1)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            _lib.call("fc_stream_signal", flag.data_ptr(), 1, s.cuda_stream)
            _lib.call("fc_stream_wait", flag.data_ptr(), 1, s.cuda_stream)
            _lib.call("fc_stream_signal", flag.data_ptr(), 0, s.cuda_stream)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert int(flag.item()) == 0


@pytest.mark.parametrize("N", [3, 4, 5])
@pytest.mark.parametrize("world", [2, 3])
def test_peer_store_virtual_ranks(N, world):
    torch.cuda.set_device(0)
    _virtual_sweep(N, world)


def test_peer_store_slot_out_of_range_flags():
    """A global slot past the last owner's range raises the slot-range flag."""
    from paper_2309_09131_b200 import DeviceFactorSet
    from paper_2309_09131_b200.peer import PeerShardedTensor
    dims, coords, vals, params, build = _case(3, 50_000)
    st = build(coords, vals, params)
    ranks = [PeerShardedTensor(st, 2, r, ipc=False) for r in range(2)]
    PeerShardedTensor.connect_local(ranks)
    ranks[0].plans[0].global_slots[5] = -2  # 0xFFFFFFFE
    f = list(DeviceFactorSet.random_device(dims, 32, seed=1).factors)
    out = ranks[0].output(0, 32)[0]
    ranks[0].mode_pass(f, 0, out)
    with pytest.raises(RuntimeError, match="flags 0x1"):
        ranks[0].check()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ipc_worker(rank, world, port, result, sync, distinct=False):
    os.environ["FLYCOO_PEER_SYNC"] = sync
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # distinct: one GPU per rank, the records and rows cross NVLink
        torch.cuda.set_device(rank if distinct else 0)
        from paper_2309_09131_b200 import DeviceFactorSet, mttkrp_mode, schedule_super_shards
        from paper_2309_09131_b200.peer import PeerShardedTensor, peer_sweep_all_modes
        for N in (3, 4):
            dims, coords, vals, params, build = _case(N)
            st = build(coords, vals, params)
            ref = build(coords, vals, params)
            dt = PeerShardedTensor(st, world, rank)
            dt.connect()
            assert dt.device_sync == (sync == "device")
            f0 = DeviceFactorSet.random_device(dims, 32, seed=3)
            ref_working = list(f0.factors)
            got = list(f0.factors)
            smap = schedule_super_shards(ref.plan, 1)
            for sweep in range(3):  # chained sweeps: outputs feed the next sweep
                got = [g.clone() for g in peer_sweep_all_modes(dt, got)]
                for n in range(N):
                    ref_working[n] = mttkrp_mode(
                        ref, DeviceFactorSet(ref_working, None, validate=False), n, smap)
                for n in range(N):
                    assert torch.equal(got[n], ref_working[n]), (rank, N, n)
            p = dt.plans[0]
            c, v = dt.local_records()
            assert torch.equal(c, ref.crd[ref.active][p.e_lo:p.e_hi]), (rank, N)
            if sync == "device":  # the whole sweep as a CUDA graph, chained replays
                from paper_2309_09131_b200.peer import PeerSweepGraph
                g = PeerSweepGraph(dt, got)
                for _ in range(1 if N % 2 == 0 else 2):  # the graph's warm-up sweeps
                    for n in range(N):
                        ref_working[n] = mttkrp_mode(
                            ref, DeviceFactorSet(ref_working, None, validate=False), n, smap)
                got = [t.clone() for t in ref_working]
                for rep in range(3):
                    got = [t.clone() for t in g.run(got)]
                    for n in range(N):
                        ref_working[n] = mttkrp_mode(
                            ref, DeviceFactorSet(ref_working, None, validate=False), n, smap)
                    for n in range(N):
                        assert torch.equal(got[n], ref_working[n]), ("graph", rank, N, rep, n)
                p = dt.plans[0]
                c, v = dt.local_records()
                assert torch.equal(c, ref.crd[ref.active][p.e_lo:p.e_hi]), ("graph", rank, N)
            dt.barrier()
            dt.close()
            dist.barrier()
        result[rank] = 1
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,sync", [(2, "device"), (2, "host"), (3, "device")])
def test_peer_exchange_processes_ipc(world, sync):
    ctx = mp.get_context("spawn")
    result = ctx.Manager().dict()
    mp.start_processes(_ipc_worker, args=(world, _free_port(), result, sync), nprocs=world,
                       join=True, start_method="spawn")
    assert sorted(result.keys()) == list(range(world))


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs (one per rank)")
@pytest.mark.parametrize("sync", ["device", "host"])
def test_peer_exchange_multi_gpu_nvlink(sync):
    """One process per GPU (up to 4): the fused exchange over real NVLink
    peer mappings; slices and factors bit-exact against the single-GPU sweep
    after every chained sweep and graph replay."""
    world = min(torch.cuda.device_count(), 4)
    ctx = mp.get_context("spawn")
    result = ctx.Manager().dict()
    mp.start_processes(_ipc_worker, args=(world, _free_port(), result, sync, True), nprocs=world,
                       join=True, start_method="spawn")
    assert sorted(result.keys()) == list(range(world))

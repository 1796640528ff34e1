"""Multi-GPU sweep with the remap fused into the exchange.

Same partition as :mod:`dist` -- per mode, GPU p owns a contiguous
super-shard range and the matching contiguous slice [E_p, E_{p+1}) of the
single-GPU mode-n buffer -- but no send region, all-to-all or unpack pass:

* every GPU's record buffers (and its per-mode output rows) are cudaMalloc
  allocations shared with all peers through CUDA IPC, mapped over NVLink;
* the mode pass (``fc_mode_worker_peers``) reads the element's GLOBAL
  mode-(n+1) slot d from the single-GPU slot map and stores the record
  straight into the back buffer of the owner q of d (E'_q <= d < E'_{q+1})
  at d - E'_q: the NVLink transfer overlaps the compute tile by tile, and a
  remote record crosses the fabric exactly once;
* after a barrier, each GPU pulls the peers' owned rows of the updated
  factor from their output buffers (copy engines over NVLink) -- the
  all-gather of engine.sweep_all_modes' factor replacement (engine.py:292).

Between modes the GPUs order themselves on the device: each sets a
per-mode flag in every peer's memory with a stream write (fenced after its
pass), waits for all peers' flags with stream waits and resets them -- "all peers
finished writing my back buffer / reading their front buffer" -- without a
host round trip or any SM spinning (``FLYCOO_PEER_SYNC=host``: stream
synchronize + ``dist.barrier``).  After every mode each
GPU's slice equals the single-GPU buffer's slice bit-exactly
(tests/test_gpu_peer.py).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .dist import _local_plan, partition_super_shards
from .layout import DeviceShardedTensor, PartitionPlan, default_chunk_elems, make_mode_work

__all__ = ["PeerModePlan", "peer_plans", "IpcBuffer", "PeerShardedTensor", "peer_mttkrp_mode",
           "peer_sweep_all_modes", "PeerSweepGraph"]


@dataclass
class PeerModePlan:
    ss_lo: int
    ss_hi: int
    e_lo: int
    e_hi: int
    global_slots: torch.Tensor  # int32 (uint32 bits): global mode-(n+1) positions
    peer_base: list             # world + 1 element bounds of mode n+1

    @property
    def count(self) -> int:
        return self.e_hi - self.e_lo


def peer_plans(plan: PartitionPlan, slot_maps, world: int, rank: int):
    """Per-mode plan of `rank`: its element slice, the slot-map slice (global
    destinations) and the next mode's ownership bounds.  Returns
    (plans, bounds, cap) like dist.build_rank_plans."""
    N = plan.num_modes
    bounds = [partition_super_shards(plan.ss_counts[n], world) for n in range(N)]
    cap = max(int(bounds[n][1][p + 1] - bounds[n][1][p]) for n in range(N) for p in range(world))
    plans = []
    for n in range(N):
        sb, eb = bounds[n]
        lo, hi = int(eb[rank]), int(eb[rank + 1])
        base = [int(x) for x in bounds[(n + 1) % N][1]]
        plans.append(PeerModePlan(int(sb[rank]), int(sb[rank + 1]), lo, hi,
                                  slot_maps[n][lo:hi].to(torch.int32).clone(), base))
    return plans, bounds, max(cap, 1)


class IpcBuffer:
    """A cudaMalloc allocation that peers can map (fc_ipc_*), viewed as a
    torch tensor through __cuda_array_interface__."""

    _TYPESTR = {torch.int32: "<i4", torch.float32: "<f4", torch.int64: "<i8"}

    def __init__(self, shape, dtype, device):
        self.shape = tuple(int(s) for s in shape)
        self.dtype = dtype
        nbytes = int(np.prod(self.shape)) * torch.empty(0, dtype=dtype).element_size()
        self.nbytes = max(nbytes, 16)
        ptr = ctypes.c_void_p()
        with torch.cuda.device(device):
            _lib.call("fc_ipc_alloc", self.nbytes, ctypes.addressof(ptr))
        self.ptr = int(ptr.value)
        self.device = device
        self.__cuda_array_interface__ = {"shape": self.shape, "typestr": self._TYPESTR[dtype],
                                         "data": (self.ptr, False), "version": 3, "strides": None}
        self.tensor = torch.as_tensor(self, device=device)

    def handle(self) -> bytes:
        n = _lib.load().fc_ipc_handle_bytes()
        buf = ctypes.create_string_buffer(n)
        _lib.call("fc_ipc_handle", self.ptr, ctypes.addressof(buf))
        return buf.raw

    def __del__(self):
        try:
            if self.ptr:
                _lib.call("fc_ipc_free", self.ptr)
                self.ptr = 0
        except Exception:
            pass


def _open_handle(h: bytes) -> int:
    ptr = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(h, len(h))
    _lib.call("fc_ipc_open", ctypes.addressof(buf), ctypes.addressof(ptr))
    return int(ptr.value)


class PeerShardedTensor:
    """Rank-local slice for the fused exchange.  ``ipc=True`` (one process
    per GPU): buffers are IPC allocations and :meth:`connect` maps the peers'
    through torch.distributed; ``ipc=False``: ordinary device tensors, peers
    wired by :meth:`connect_local` (several virtual ranks in one process --
    the single-GPU parity test of the peer-store kernel path)."""

    def __init__(self, st: DeviceShardedTensor, world: int, rank: int, group=None,
                 ipc: bool = True):
        if world > 8:
            raise ValueError("the fused exchange maps at most 8 peers")
        self.plan = st.plan
        self.world, self.rank, self.group, self.ipc = world, rank, group, ipc
        self.device = st.device
        self.num_modes = st.num_modes
        self.plans, self.bounds, self.cap = peer_plans(st.plan, st.slot_maps, world, rank)
        cw = st.crd[0].shape[1]
        self.cw = cw
        emb = st.val[0] is None
        self._bufs = []
        self.crd = [self._alloc((self.cap, cw), torch.int32) for _ in range(2)]
        self.val = [None, None] if emb else [self._alloc((self.cap,), torch.float32)
                                            for _ in range(2)]
        p0 = self.plans[0]
        self.crd[0][:p0.count] = st.crd[st.active][p0.e_lo:p0.e_hi]
        if not emb:
            self.val[0][:p0.count] = st.val[st.active][p0.e_lo:p0.e_hi]
        self.active = 0
        self.active_mode = 0
        self.peer_crd = None     # [buffer k][rank q] -> device pointer
        self.peer_val = None
        self.outs = {}           # (mode, R) -> (tensor, [peer pointers])
        self._work = {}
        self._stat = torch.zeros(2, dtype=torch.int64, device=self.device)
        self._expected = 0
        self._opened = []
        # cross-GPU ordering between passes (stream memory operations, no host
        # round trip): flags[n][q] = 1 once GPU q finished its mode-n pass;
        # reset to 0 by this GPU after its wait.  Constant values make the
        # protocol replayable in a CUDA graph; a peer's next signal on the same
        # slot always follows this GPU's reset (it first waits on a later
        # mode's signal of ours).  FLYCOO_PEER_SYNC=host: stream synchronize +
        # dist.barrier instead.
        self.flags = self._alloc((self.num_modes, world), torch.int32)
        self.peer_flags = None
        self.device_sync = ipc and os.environ.get("FLYCOO_PEER_SYNC", "device") != "host"

    # -- buffers and peer wiring
    def _alloc(self, shape, dtype):
        if not self.ipc:
            return torch.zeros(shape, dtype=dtype, device=self.device)
        b = IpcBuffer(shape, dtype, self.device)
        self._bufs.append(b)
        b.tensor.zero_()
        return b.tensor

    def _shared(self):
        ts = list(self.crd) + ([] if self.val[0] is None else list(self.val))
        return ts

    def _exchange_ptrs(self, tensors):
        """Collective: device pointers of every rank's `tensors` (own ones as
        is, peers' through IPC mappings).  Returns [tensor i][rank q]."""
        bufs = {b.tensor.data_ptr(): b for b in self._bufs}
        mine = [bufs[t.data_ptr()].handle() for t in tensors]
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=self.group)
        out = [[0] * self.world for _ in tensors]
        for q in range(self.world):
            for i, t in enumerate(tensors):
                if q == self.rank:
                    out[i][q] = t.data_ptr()
                else:
                    ptr = _open_handle(allh[q][i])
                    self._opened.append(ptr)
                    out[i][q] = ptr
        return out

    def connect(self):
        """Collective over the group: map every peer's record buffers and
        barrier flags."""
        ptrs = self._exchange_ptrs(self._shared() + [self.flags])
        self.peer_crd = [ptrs[0], ptrs[1]]
        self.peer_val = None if self.val[0] is None else [ptrs[2], ptrs[3]]
        self.peer_flags = ptrs[-1]

    @staticmethod
    def connect_local(ranks):
        """Wire virtual ranks living in one process (ipc=False)."""
        for dt in ranks:
            dt.peer_crd = [[r.crd[k].data_ptr() for r in ranks] for k in range(2)]
            dt.peer_val = None if dt.val[0] is None else [[r.val[k].data_ptr() for r in ranks]
                                                          for k in range(2)]
            dt._local_ranks = ranks

    def output(self, mode: int, R: int):
        """Persistent, peer-visible output rows of `mode` (every row is
        rewritten by each pass: owned rows by the pass, the rest by the
        pull)."""
        key = (mode, R)
        if key not in self.outs:
            t = self._alloc((self.plan.params.dims[mode], R), torch.float32)
            if self.ipc:
                ptrs = self._exchange_ptrs([t])[0]
            else:
                ptrs = None  # filled by the virtual-rank driver
            self.outs[key] = [t, ptrs]
        return self.outs[key]

    # -- static work plans
    def local_records(self):
        p = self.plans[self.active_mode]
        c = self.crd[self.active][:p.count]
        v = None if self.val[self.active] is None else self.val[self.active][:p.count]
        return c, v

    def mode_work(self, mode: int, R: int):
        key = (mode, R)
        if key not in self._work:
            lp = _local_plan(self.plan, mode, self.plans[mode])
            p = self.plans[mode]
            self._work[key] = make_mode_work(lp, mode, R, self.device,
                                             chunk_elems=default_chunk_elems(self.plan.nnz),
                                             ss_range=(p.ss_lo, p.ss_hi))
        return self._work[key]

    def owned_rows(self, mode: int):
        p = self.plans[mode]
        m = self.plan.params.m[mode]
        dim = self.plan.params.dims[mode]
        return min(p.ss_lo * m, dim), min(p.ss_hi * m, dim)

    def row_ranges(self, mode: int):
        m = self.plan.params.m[mode]
        dim = self.plan.params.dims[mode]
        sb = self.bounds[mode][0]
        return [(min(int(sb[q]) * m, dim), min(int(sb[q + 1]) * m, dim)) for q in range(self.world)]

    # -- passes
    def mode_pass(self, factors, mode: int, out: torch.Tensor, stream=None):
        """Fused K1 (+K2) of this rank: compute owned rows into `out`, store
        every record into its owner's back buffer."""
        if self.peer_crd is None:
            raise RuntimeError("peers not connected (connect / connect_local)")
        p = self.plans[mode]
        R = int(out.shape[1])
        w = self.mode_work(mode, R)
        a, b = self.active, 1 - self.active
        vp = lambda t: t.data_ptr() if t is not None else None
        params = self.plan.params
        stat = self._stat.data_ptr()
        pv = None if self.peer_val is None else _lib.ptr_array(self.peer_val[b])
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _lib.call("fc_mode_worker_peers", self.crd[a].data_ptr(), vp(self.val[a]),
                  _lib.ptr_array([f.data_ptr() for f in factors]), _lib.i64_array(params.dims),
                  out.data_ptr(), self.num_modes, mode, R, params.dims[mode], params.m[mode],
                  w.chunk_start.data_ptr(), w.chunk_ss.data_ptr(), w.chunk_part.data_ptr(),
                  vp(w.chunk_rows), w.tile_rows, w.hist_rows, w.nchunks, w.red1.data_ptr(),
                  w.nred1, w.red2.data_ptr(), w.nred2, vp(w.part_ws), vp(w.part_ws2),
                  p.global_slots.data_ptr(), p.count, 1, int(w.acc_in_smem), stat + 8, stat,
                  self.world, _lib.ptr_array(self.peer_crd[b]), pv, _lib.i64_array(p.peer_base),
                  st)
        self._expected += p.count

    def pull_rows(self, mode: int, out: torch.Tensor, peer_out_ptrs, stream=None):
        """Copy the peers' owned rows of `mode` into `out` (NVLink copy
        engines); `out` then holds the whole updated factor."""
        R = int(out.shape[1])
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        ranges = self.row_ranges(mode)
        bounds = [lo for lo, _ in ranges] + [ranges[-1][1]]
        if R % 4 == 0:  # one launch, NVLink loads
            _lib.call("fc_gather_peer_rows", out.data_ptr(), _lib.ptr_array(peer_out_ptrs),
                      _lib.i64_array(bounds), self.world, self.rank, R, st)
            return
        row_bytes = R * 4
        for q, (lo, hi) in enumerate(ranges):
            if q == self.rank or hi <= lo:
                continue
            off = lo * row_bytes
            _lib.call("fc_copy_async", out.data_ptr() + off, peer_out_ptrs[q] + off,
                      (hi - lo) * row_bytes, st)

    def swap(self):
        self.active = 1 - self.active
        self.active_mode = (self.active_mode + 1) % self.num_modes

    def check(self):
        stat = self._stat.cpu()
        flags = int(stat[1]) & 0xFFFFFFFF
        processed, expected = int(stat[0]), self._expected
        self._stat.zero_()
        self._expected = 0
        if processed != expected or flags:
            raise RuntimeError(f"fused-exchange pass failed: processed {processed} of {expected}, "
                               f"flags {flags:#x}")

    def barrier(self):
        """Host barrier: every GPU's queued work done (stream synchronize),
        then dist.barrier."""
        torch.cuda.current_stream().synchronize()
        if self.ipc:
            dist.barrier(group=self.group)

    def sync(self, mode: int = 0):
        """Order the GPUs after the mode-`mode` pass: afterwards every peer's
        pass (records stored into this GPU, owned output rows) is complete
        and visible, and no peer still reads this GPU's front buffer."""
        if not self.device_sync:
            self.barrier()
            return
        st = torch.cuda.current_stream().cuda_stream
        slot = 4 * mode * self.world
        for q in range(self.world):
            if q != self.rank:
                _lib.call("fc_stream_signal", self.peer_flags[q] + slot + 4 * self.rank, 1, st)
        base = self.flags.data_ptr() + slot
        for q in range(self.world):
            if q != self.rank:
                _lib.call("fc_stream_wait", base + 4 * q, 1, st)
                _lib.call("fc_stream_signal", base + 4 * q, 0, st)

    def close(self):
        """Unmap the peers' buffers (each GPU's own allocations are freed
        when their IpcBuffer objects go; call after a barrier so no peer is
        still using them)."""
        for ptr in self._opened:
            try:
                _lib.call("fc_ipc_close", ptr)
            except Exception:
                pass
        self._opened = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def peer_mttkrp_mode(dt: PeerShardedTensor, factors, mode: int) -> torch.Tensor:
    """One fused mode pass across the group; returns this rank's persistent
    output of `mode` with every row valid (owned rows computed here, the
    rest pulled from the peers)."""
    if dt.active_mode != mode:
        raise ValueError(f"active mode is {dt.active_mode}, not {mode}")
    R = int(factors[0].shape[1])
    out, ptrs = dt.output(mode, R)
    dt.mode_pass(factors, mode, out)
    dt.sync(mode)
    dt.pull_rows(mode, out, ptrs)
    dt.swap()
    return out


def peer_sweep_all_modes(dt: PeerShardedTensor, factors, mode_seconds=None):
    """engine.sweep_all_modes across GPUs with the fused exchange.  The
    returned factors are the persistent output buffers (valid until the
    next sweep on `dt` rewrites them)."""
    working = list(factors)
    events = []
    for n in range(dt.num_modes):
        if mode_seconds is not None:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record()
        working[n] = peer_mttkrp_mode(dt, working, n)
        if mode_seconds is not None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record()
            events.append((e0, e1))
    dt.check()  # synchronizes this GPU's stream
    if mode_seconds is not None:
        mode_seconds.extend(a.elapsed_time(b) / 1e3 for a, b in events)
    return working


class PeerSweepGraph:
    """CUDA-graph replay of :func:`peer_sweep_all_modes` on this GPU: the
    mode passes, the device-side barriers (stream memory operations with
    constant flag values, hence replayable) and the row gathers of a whole
    sweep in one launch -- no host work between modes.  Every GPU of the
    group builds and runs its own graph; outputs are the persistent
    per-mode buffers (valid until the next run)."""

    def __init__(self, dt: PeerShardedTensor, factors):
        if not dt.device_sync:
            raise ValueError("graph replay needs the device-side barrier (FLYCOO_PEER_SYNC=device)")
        if dt.active_mode != 0:
            raise ValueError(f"a sweep starts at mode 0, the tensor is at mode {dt.active_mode}")
        self.dt = dt
        self.N = dt.num_modes
        self.inputs = [f.clone() for f in factors]
        self.R = int(self.inputs[0].shape[1])
        self.pool = torch.cuda.graph_pool_handle()
        self.graphs = {}
        # eager sweeps: cache work plans, create and map the output buffers
        # (collective), configure the kernels -- both buffer parities
        for _ in range(1 if self.N % 2 == 0 else 2):
            peer_sweep_all_modes(dt, list(self.inputs))
        torch.cuda.synchronize()

    def _capture(self):
        dt = self.dt
        saved = (dt.active, dt.active_mode, dt._expected)
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(device=dt.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, pool=self.pool, stream=side):
                dt._stat.zero_()
                working = list(self.inputs)
                for n in range(self.N):
                    out, ptrs = dt.output(n, self.R)
                    dt.mode_pass(working, n, out)
                    dt.sync(n)
                    dt.pull_rows(n, out, ptrs)
                    dt.swap()
                    working[n] = out
        torch.cuda.current_stream().wait_stream(side)
        expected = dt._expected - saved[2]
        dt.active, dt.active_mode, dt._expected = saved
        self.graphs[saved[0]] = (g, working, expected)

    def run(self, factors=None):
        dt = self.dt
        if factors is not None:
            for dst, src in zip(self.inputs, factors):
                if src.data_ptr() != dst.data_ptr():
                    dst.copy_(src, non_blocking=True)
        if dt.active not in self.graphs:
            self._capture()
        g, outs, expected = self.graphs[dt.active]
        g.replay()
        dt.active ^= self.N % 2
        dt._expected = expected
        dt.check()
        return outs

"""Multi-GPU sweep with the remap fused into the exchange.

Partition.  GPUs take contiguous ranges of the single-GPU chunk list of each
mode (the same CTA chunks, partial-tile ids and K2 reduce plan as one GPU),
balanced by nonzeros -- so a Zipf head super-shard (c2: ~40% of a mode) is
split across GPUs instead of capping the speed-up.  Every super-shard's
rows stay owned by ONE GPU (the one running its first chunk), so each GPU
still owns a contiguous output-row range per mode (north_star); chunks of a
split super-shard write their partial tiles into the owner's workspace and
the owner reduces them in the single-GPU order -- outputs are bitwise
identical to the single-GPU sweep.

Exchange.  Every GPU's record buffers, partial workspace and per-mode output
rows are cudaMalloc allocations shared through CUDA IPC and mapped over
NVLink.  The mode pass (``fc_mode_worker_peers``) reads the element's
GLOBAL mode-(n+1) slot d from the single-GPU slot map and stores the record
straight into the back buffer of the owner q of d (E'_q <= d < E'_{q+1}) at
d - E'_q: the NVLink transfer overlaps the compute tile by tile and a remote
record crosses the fabric once -- no send region, all-to-all or unpack pass.

Ordering.  Per mode: K1 -> barrier (peers' partials are in) -> K2 of the
owned super-shards -> barrier (owned rows final) -> one kernel gathers the
peers' owned rows over NVLink (the factor all-gather of engine.py:292).  The
barriers run on the device: each GPU sets a flag in every peer's memory with
a fenced stream write and waits for its own flags with stream waits (no host
round trip, no SM spinning; ``FLYCOO_PEER_SYNC=host``: stream synchronize +
``dist.barrier``).  The flag values are constants, so a whole sweep is
captured as one CUDA graph per GPU (:class:`PeerSweepGraph`).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .layout import DeviceShardedTensor, PartitionPlan, make_mode_work

__all__ = ["PeerModePlan", "partition_chunks", "super_shard_owners", "peer_plans", "slice_bounds",
           "IpcBuffer",
           "PeerShardedTensor", "peer_mttkrp_mode", "peer_sweep_all_modes", "PeerSweepGraph"]


@dataclass
class PeerModePlan:
    """One GPU's share of one mode pass.  GPUs take contiguous ranges of the
    single-GPU chunk list (balanced by nonzeros + a per-chunk cost), so a heavy super-shard's
    chunks may run on several GPUs; its rows stay owned by ONE GPU (the one
    running its first chunk), which reduces all its partial tiles."""
    c_lo: int                   # chunk range [c_lo, c_hi) of the global plan
    c_hi: int
    e_lo: int                   # element range = chunk_start[c_lo], chunk_start[c_hi]
    e_hi: int
    ss_lo: int                  # owned super-shards [ss_lo, ss_hi)
    ss_hi: int
    global_slots: torch.Tensor  # int32 (uint32 bits): global mode-(n+1) positions
    peer_base: list             # world + 1 element bounds of mode n+1 (owner of a slot)
    row_bounds: list            # world + 1 owned-row bounds of mode n
    chunk_owner: torch.Tensor   # int32 per chunk of [c_lo, c_hi): GPU owning its super-shard
    red1: torch.Tensor          # K2 tasks of the owned super-shards
    red2: torch.Tensor

    @property
    def count(self) -> int:
        return self.e_hi - self.e_lo


# Cost of one chunk beyond its nonzeros, in nonzero equivalents: a chunk pays
# its tile passes' fixed work (barriers, histogram scan, boundary fold) and its
# accumulator tile however few nonzeros it holds, so a GPU whose range is the
# Zipf tail (many small super-shards) is slower than its nonzero share says.
CHUNK_WEIGHT = int(os.environ.get("FLYCOO_CHUNK_WEIGHT", "2048"))


def partition_chunks(chunk_start: np.ndarray, world: int, chunk_weight: int | None = None) -> np.ndarray:
    """world + 1 chunk bounds splitting the chunk list into contiguous ranges
    of ~equal cost = nonzeros + chunk_weight per chunk."""
    nch = chunk_start.shape[0] - 1
    kw = CHUNK_WEIGHT if chunk_weight is None else int(chunk_weight)
    # cost before chunk c (c = 0..nch)
    cost = (chunk_start - chunk_start[0]).astype(np.float64) + kw * np.arange(nch + 1, dtype=np.float64)
    total = cost[-1]
    cb = [0]
    for p in range(1, world):
        c = int(np.searchsorted(cost[:nch], p * total / world, side="left"))
        cb.append(min(max(c, cb[-1]), nch))
    cb.append(nch)
    return np.asarray(cb, dtype=np.int64)


def super_shard_owners(work, k: int, m: int, chunk_gpu: np.ndarray, world: int) -> np.ndarray:
    """Owner GPU of every super-shard: the GPU running the first chunk that
    covers it (a direct chunk covers several); super-shards without chunks
    (empty, zeroed by K2) go to the owner of the next covered one."""
    cs = work.chunk_ss.cpu().numpy().astype(np.int64)
    cp = work.chunk_part.cpu().numpy()
    if work.chunk_rows is not None:
        cr = work.chunk_rows.cpu().numpy().astype(np.int64)
        nss = np.where(cp == -2, -(-cr // m), 1)
    else:
        nss = np.ones_like(cs)
    ss_cov = np.repeat(cs, nss) + (np.arange(int(nss.sum())) -
                                   np.repeat(np.concatenate(([0], np.cumsum(nss)))[:-1], nss))
    gpu_cov = np.repeat(chunk_gpu, nss)
    owner = np.full(k, -1, dtype=np.int64)
    if ss_cov.size:
        idx = np.searchsorted(ss_cov, np.arange(k), side="left")
        ok = idx < ss_cov.size
        ok[ok] = ss_cov[idx[ok]] == np.arange(k)[ok]
        owner[ok] = gpu_cov[idx[ok]]
    nxt = world - 1  # backward fill of uncovered super-shards
    for s in range(k - 1, -1, -1):
        if owner[s] < 0:
            owner[s] = nxt
        else:
            nxt = owner[s]
    assert np.all(np.diff(owner) >= 0), "super-shard owners must be monotone"
    return owner


def _chunk_partition(plan: PartitionPlan, world: int, R: int, device):
    """The global work plan of every mode and its chunk / element bounds per GPU."""
    N = plan.num_modes
    works, cbs = [], []
    for n in range(N):
        w = make_mode_work(plan, n, R, device)
        works.append(w)
        cbs.append(partition_chunks(w.chunk_start.cpu().numpy(), world))
    starts = [w.chunk_start.cpu().numpy() for w in works]
    ebs = [starts[n][cbs[n]] for n in range(N)]
    return works, cbs, ebs


def slice_bounds(plan: PartitionPlan, world: int, R: int, device) -> list:
    """Per mode, the world + 1 element bounds of the GPUs' slices (a pure
    function of the plan: the partitioned build routes slot-map entries and
    records with it, distbuild.build_partitioned)."""
    return [[int(x) for x in eb] for eb in _chunk_partition(plan, world, R, device)[2]]


def _slot_slice(src, n: int, lo: int, hi: int) -> torch.Tensor:
    """[lo, hi) of mode n's global slot map from a DeviceShardedTensor, a
    LocalLayout (its own slice) or a plain list of slot maps."""
    if hasattr(src, "slot_slice"):
        return src.slot_slice(n, lo, hi)
    maps = src if isinstance(src, (list, tuple)) else src.slot_maps
    return maps[n][lo:hi]


def peer_plans(plan: PartitionPlan, src, world: int, rank: int, R: int, device):
    """Per-mode plans of `rank` on the global single-GPU work plans (one per
    mode, rank R); `src` provides the global slot maps (a DeviceShardedTensor)
    or this rank's slices of them (distbuild.LocalLayout).  Returns (plans,
    works, cap): cap = the largest element slice of any GPU in any mode
    (record buffer rows)."""
    N = plan.num_modes
    works, cbs, ebs = _chunk_partition(plan, world, R, device)
    cap = max(int(eb[p + 1] - eb[p]) for eb in ebs for p in range(world))
    plans = []
    for n in range(N):
        w, cb, eb = works[n], cbs[n], ebs[n]
        m, k, dim = int(plan.params.m[n]), int(plan.params.k[n]), int(plan.params.dims[n])
        chunk_gpu = np.repeat(np.arange(world), np.diff(cb))
        owner = super_shard_owners(w, k, m, chunk_gpu, world)
        lo_ss = [int(np.searchsorted(owner, p, side="left")) for p in range(world)] + [k]
        rows = [min(x * m, dim) for x in lo_ss]
        cs = w.chunk_ss.cpu().numpy().astype(np.int64)
        c_lo, c_hi = int(cb[rank]), int(cb[rank + 1])
        r1 = w.red1.cpu().numpy().reshape(-1, 4)
        r2 = w.red2.cpu().numpy().reshape(-1, 3)
        r1 = r1[owner[r1[:, 0]] == rank] if r1.size else r1
        r2 = r2[owner[r2[:, 0]] == rank] if r2.size else r2
        e_lo, e_hi = int(eb[rank]), int(eb[rank + 1])
        t = lambda a, dt=torch.int64: torch.from_numpy(np.ascontiguousarray(a)).to(dt).to(device)
        plans.append(PeerModePlan(
            c_lo, c_hi, e_lo, e_hi, lo_ss[rank], lo_ss[rank + 1],
            _slot_slice(src, n, e_lo, e_hi).to(torch.int32).clone().to(device),
            [int(x) for x in ebs[(n + 1) % N]], rows,
            t(owner[cs[c_lo:c_hi]], torch.int32), t(r1), t(r2)))
    return plans, works, max(cap, 1)


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
    the single-GPU parity test of the peer-store kernel path).  `R` is the
    factor rank the work plans are built for (default: the params' rank)."""

    def __init__(self, st, world: int, rank: int, group=None,
                 ipc: bool = True, R: int | None = None):
        """`st`: the global DeviceShardedTensor (sliced here), or this rank's
        distbuild.LocalLayout (the partitioned build: no rank holds the
        whole layout)."""
        if world > 8:
            raise ValueError("the fused exchange maps at most 8 peers")
        self.plan = st.plan
        self.world, self.rank, self.group, self.ipc = world, rank, group, ipc
        self.device = st.device
        self.num_modes = st.num_modes
        self.R = int(R if R is not None else st.plan.params.rank)
        self.plans, self.works, self.cap = peer_plans(st.plan, st, world, rank, self.R, st.device)
        p0 = self.plans[0]
        if hasattr(st, "records_slice"):
            crd0, val0 = st.records_slice(p0.e_lo, p0.e_hi)
        else:
            crd0 = st.crd[st.active][p0.e_lo:p0.e_hi]
            val0 = None if st.val[st.active] is None else st.val[st.active][p0.e_lo:p0.e_hi]
        cw = crd0.shape[1]
        self.cw = cw
        emb = val0 is None
        self._bufs = []
        self.crd = [self._alloc((self.cap, cw), torch.int32) for _ in range(2)]
        self.val = [None, None] if emb else [self._alloc((self.cap,), torch.float32)
                                            for _ in range(2)]
        self.crd[0][:p0.count] = crd0
        if not emb:
            self.val[0][:p0.count] = val0
        # partial tiles, indexed by the global partial id: peers write the
        # partials of super-shards this GPU owns into it (one buffer for all
        # modes: a mode's partials are reduced before any GPU starts the next)
        ws = max([w.part_ws.numel() for w in self.works if w.part_ws is not None] + [1])
        self.part_ws = self._alloc((ws,), torch.float32)
        for w in self.works:
            w.part_ws = None
        self.active = 0
        self.active_mode = 0
        self._tile_plans = {}    # mode -> (perm, bins, shifted pointers) or None (_tile_plan)
        self.peer_crd = None     # [buffer k][rank q] -> device pointer
        self.peer_val = None
        self.peer_part_ws = None
        self.outs = {}           # (mode, R) -> (tensor, [peer pointers])
        self._stat = torch.zeros(2, dtype=torch.int64, device=self.device)
        self._expected = 0
        self._opened = []
        # cross-GPU ordering (stream memory operations, no host round trip):
        # two barriers per mode (after K1: peers' partial tiles are in; after
        # K2: owned rows are final).  flags[b][q] = 1 once GPU q reached
        # barrier b, reset to 0 by this GPU after its wait; constant values
        # make the protocol replayable in a CUDA graph, and a peer's next set
        # of the same slot always follows this GPU's reset (it first waits on
        # a later barrier of ours).  FLYCOO_PEER_SYNC=host: stream synchronize
        # + dist.barrier instead.
        self.flags = self._alloc((2 * self.num_modes, world), torch.int32)
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
        # a local failure still joins the collective (with None), so every
        # rank raises together instead of leaving the others in the gather
        try:
            mine = [bufs[t.data_ptr()].handle() for t in tensors]
            err = None
        except Exception as e:  # noqa: BLE001
            mine, err = None, e
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=self.group)
        if err is not None:
            raise err
        missing = [q for q in range(self.world) if allh[q] is None]
        if missing:
            raise RuntimeError(f"ranks {missing} could not export their IPC handles")
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
        """Collective over the group: map every peer's record buffers,
        partial-tile workspace and barrier flags."""
        ptrs = self._exchange_ptrs(self._shared() + [self.part_ws, self.flags])
        self.peer_crd = [ptrs[0], ptrs[1]]
        self.peer_val = None if self.val[0] is None else [ptrs[2], ptrs[3]]
        self.peer_part_ws = ptrs[-2]
        self.peer_flags = ptrs[-1]

    @staticmethod
    def connect_local(ranks):
        """Wire virtual ranks living in one process (ipc=False)."""
        for dt in ranks:
            dt.peer_crd = [[r.crd[k].data_ptr() for r in ranks] for k in range(2)]
            dt.peer_val = None if dt.val[0] is None else [[r.val[k].data_ptr() for r in ranks]
                                                          for k in range(2)]
            dt.peer_part_ws = [r.part_ws.data_ptr() for r in ranks]
            dt._local_ranks = ranks

    def output(self, mode: int, R: int):
        """Persistent, peer-visible output rows of `mode` (owned rows are
        rewritten by every pass, the rest by the row gather)."""
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

    def mode_work(self, mode: int, R: int | None = None):
        """The global single-GPU work plan of `mode` (this GPU runs a chunk
        range of it)."""
        return self.works[mode]

    def owned_rows(self, mode: int):
        rb = self.plans[mode].row_bounds
        return rb[self.rank], rb[self.rank + 1]

    def row_ranges(self, mode: int):
        rb = self.plans[mode].row_bounds
        return [(rb[q], rb[q + 1]) for q in range(self.world)]

    # -- passes
    def mode_pass(self, factors, mode: int, out: torch.Tensor, stream=None):
        """K1 over this GPU's chunk range: rows of owned super-shards that
        need no reduce into `out`, partial tiles into their owners'
        workspaces, every record into its owner's back buffer."""
        if self.peer_crd is None:
            raise RuntimeError("peers not connected (connect / connect_local)")
        p = self.plans[mode]
        R = int(out.shape[1])
        if R != self.R:
            raise ValueError(f"work plans were built for rank {self.R}, factors have {R}")
        w = self.works[mode]
        a, b = self.active, 1 - self.active
        params = self.plan.params
        stat = self._stat.data_ptr()
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        c0 = p.c_lo
        # global element / chunk indices address this GPU's slices directly
        src = self.crd[a].data_ptr() - p.e_lo * self.cw * 4
        srcv = None if self.val[a] is None else self.val[a].data_ptr() - p.e_lo * 4
        slots = p.global_slots.data_ptr() - p.e_lo * 4 if p.count else None
        pv = None if self.peer_val is None else _lib.ptr_array(self.peer_val[b])
        plan = self._tile_plan(mode, w, p, src, srcv, factors, R, stat, st)
        if not w.acc_in_smem:
            # the general kernel accumulates straight into `out` (one chunk
            # per super-shard, owned by this GPU): the owned rows start at 0
            # on every pass, also when `out` is reused across sweeps
            lo, hi = self.owned_rows(mode)
            if hi > lo:
                with torch.cuda.stream(torch.cuda.ExternalStream(st, device=self.device)):
                    out[lo:hi].zero_()
        _lib.call("fc_mode_worker_peers_planned", src, srcv,
                  _lib.ptr_array([f.data_ptr() for f in factors]), _lib.i64_array(params.dims),
                  out.data_ptr(), self.num_modes, mode, R, params.dims[mode], params.m[mode],
                  w.chunk_start.data_ptr() + 8 * c0, w.chunk_ss.data_ptr() + 4 * c0,
                  w.chunk_part.data_ptr() + 4 * c0,
                  None if w.chunk_rows is None else w.chunk_rows.data_ptr() + 4 * c0,
                  w.tile_rows, w.hist_rows, p.c_hi - c0, None, 0, None, 0,
                  self.part_ws.data_ptr(), None, slots, p.count, 1, int(w.acc_in_smem),
                  stat + 8, stat, self.world, _lib.ptr_array(self.peer_crd[b]), pv,
                  _lib.i64_array(p.peer_base), _lib.ptr_array(self.peer_part_ws),
                  p.chunk_owner.data_ptr() if p.chunk_owner.numel() else None,
                  plan[2] if plan else None, plan[3] if plan else None, st)
        self._expected += p.count

    def _tile_plan(self, mode, w, p, src, srcv, factors, R, stat, st):
        """This GPU's tile plan of `mode` (engine.build_tile_plans for a slice):
        emitted on the first pass over the mode -- the slice is in its
        canonical order then and in every later sweep -- with the same
        shifted pointers and chunk range the mode pass uses.  Returns the
        tensors and their key-shifted pointers, or None (no plan: the kernel
        ranks)."""
        if mode in self._tile_plans:
            return self._tile_plans[mode]
        self._tile_plans[mode] = None
        env = os.environ.get("FLYCOO_TILE_PLAN")
        N = self.num_modes
        if (env == "0" or not w.acc_in_smem or p.count == 0
                or not ((N == 3 and R in (16, 32)) or (N == 4 and R == 32))):
            return None
        L = _lib.load()
        tile = int(L.fc_tile_elems())
        nch = p.c_hi - p.c_lo
        k0 = p.e_lo // tile  # first tile key of the slice (keys: global t0 // tile + local chunk)
        keys = (p.e_hi - 1) // tile - k0 + nch + 2
        if env is None:
            free, _ = torch.cuda.mem_get_info(self.device)
            free += torch.cuda.memory_reserved(self.device) - torch.cuda.memory_allocated(self.device)
            if 3 * keys * (tile + w.hist_rows) * 2 * N > free:
                return None
        perm = torch.empty(keys * tile, dtype=torch.int16, device=self.device)
        bins = torch.zeros(keys * w.hist_rows, dtype=torch.int16, device=self.device)
        perm_p = perm.data_ptr() - k0 * tile * 2
        bins_p = bins.data_ptr() - k0 * w.hist_rows * 2
        params = self.plan.params
        c0 = p.c_lo
        with torch.cuda.stream(torch.cuda.ExternalStream(st, device=self.device)):
            rc = L.fc_tile_plan_emit(
                src, srcv, _lib.ptr_array([f.data_ptr() for f in factors]),
                _lib.i64_array(params.dims), N, mode, R, params.dims[mode], params.m[mode],
                w.chunk_start.data_ptr() + 8 * c0, w.chunk_ss.data_ptr() + 4 * c0,
                w.chunk_part.data_ptr() + 4 * c0,
                None if w.chunk_rows is None else w.chunk_rows.data_ptr() + 4 * c0,
                w.tile_rows, w.hist_rows, nch, p.count, stat + 8, stat, perm_p, bins_p, st)
        if rc == _lib.ERR_UNSUPPORTED:
            return None
        if rc != 0:
            raise _lib.FlycooError(
                f"fc_tile_plan_emit failed ({rc}): {L.fc_last_error().decode(errors='replace')}")
        self._tile_plans[mode] = (perm, bins, perm_p, bins_p)
        return self._tile_plans[mode]

    def reduce(self, mode: int, out: torch.Tensor, stream=None):
        """K2 of the owned super-shards (after the post-K1 barrier)."""
        p = self.plans[mode]
        w = self.works[mode]
        n1, n2 = int(p.red1.shape[0]), int(p.red2.shape[0])
        if n1 == 0 and n2 == 0:
            return
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        params = self.plan.params
        _lib.call("fc_reduce_partials", p.red1.data_ptr() if n1 else None, n1,
                  p.red2.data_ptr() if n2 else None, n2, self.part_ws.data_ptr(),
                  None if w.part_ws2 is None else w.part_ws2.data_ptr(), out.data_ptr(),
                  params.dims[mode], params.m[mode], int(out.shape[1]), st)

    def pull_rows(self, mode: int, out: torch.Tensor, peer_out_ptrs, stream=None):
        """Gather the peers' owned rows of `mode` into `out` (one kernel,
        NVLink loads); `out` then holds the whole updated factor."""
        R = int(out.shape[1])
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        ranges = self.row_ranges(mode)
        bounds = [lo for lo, _ in ranges] + [ranges[-1][1]]
        if R % 4 == 0:
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

    def sync(self, slot: int = 0):
        """Device barrier `slot` (2n: after mode n's K1, 2n + 1: after its
        K2): afterwards every peer's work before its own barrier `slot` is
        complete and visible to this GPU."""
        if not self.device_sync:
            self.barrier()
            return
        st = torch.cuda.current_stream().cuda_stream
        off = 4 * slot * self.world
        for q in range(self.world):
            if q != self.rank:
                _lib.call("fc_stream_signal", self.peer_flags[q] + off + 4 * self.rank, 1, st)
        base = self.flags.data_ptr() + off
        for q in range(self.world):
            if q != self.rank:
                _lib.call("fc_stream_wait", base + 4 * q, 1, st)
                _lib.call("fc_stream_signal", base + 4 * q, 0, st)

    def full_pass(self, factors, mode: int, out: torch.Tensor, peer_out_ptrs):
        """K1, barrier, K2 (owned super-shards), barrier, row gather, swap."""
        self.mode_pass(factors, mode, out)
        self.sync(2 * mode)
        self.reduce(mode, out)
        self.sync(2 * mode + 1)
        self.pull_rows(mode, out, peer_out_ptrs)
        self.swap()

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
    rest gathered from the peers)."""
    if dt.active_mode != mode:
        raise ValueError(f"active mode is {dt.active_mode}, not {mode}")
    R = int(factors[0].shape[1])
    out, ptrs = dt.output(mode, R)
    dt.full_pass(factors, mode, out, ptrs)
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
                    dt.full_pass(working, n, out, ptrs)
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

"""The FLYCOO layout in HBM: plan, double-buffered element records, slot maps.

Mirrors the reference's data model (/root/reference/pkg/src/modecycle/
layout.py:344-531) with a B200 memory layout:

* records: int32 coordinates + fp32 value, 16 B per element for N <= 3
  (value in word 3), 20 B for N = 4 (value array beside the 16-B coordinate
  rows) -- see include/flycoo.h; two buffers (ping-pong) of nnz records;
* slot maps: one uint32 per element per mode, ``slot[n][i]`` = position in
  the mode-(n+1) buffer of the element at mode-n position i
  (layout.py:516-519);
* plan arrays (super-shard fills, shard offsets) on the host, identical to
  the reference's.

Element order: the reference's canonical order fixes shard membership and
shard offsets (layout.py:484-497) and this build keeps both bit-exactly.
Inside each shard the order is free (the reference checks shards only at
shard granularity, layout.py:615-625); this build orders a shard's elements
by (previous-mode shard id, Morton key, input position), so every remap
writes each (source shard -> destination shard) group as one contiguous run
(DESIGN.md "Layout").

:func:`build_device_sharded` runs the build on the GPU through the K5
entry points of libflycoo (radix sorts, histograms, scatters).
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .params import PartitionParams

__all__ = ["PartitionPlan", "DeviceShardedTensor", "build_sharded", "build_device_sharded",
           "plan_from_counts", "record_bytes", "ModeWork", "device_has_duplicates"]


def record_bytes(nmodes: int) -> int:
    """Logical bytes of one element record (int32 coords + fp32 value)."""
    return 4 * nmodes + 4


def _cdiv(a, b):
    return -(-a // b)


@dataclass(frozen=True, eq=False)
class PartitionPlan:
    """Per-mode geometry (layout.py:344-381): super-shard fills and prefix
    sums, shard counts, and every shard's element offset."""

    params: PartitionParams
    ss_counts: tuple
    ss_elem_offsets: tuple
    ss_shard_counts: tuple
    ss_first_shard: tuple
    shard_offsets: tuple

    @property
    def num_modes(self) -> int:
        return self.params.num_modes

    @property
    def nnz(self) -> int:
        return self.params.nnz

    def total_shards(self, mode: int) -> int:
        return int(self.ss_first_shard[mode][-1])

    def shard_fills(self, mode: int) -> np.ndarray:
        return np.diff(self.shard_offsets[mode])

    def ss_of_shard(self, mode: int) -> np.ndarray:
        return np.repeat(np.arange(self.params.k[mode], dtype=np.int64), self.ss_shard_counts[mode])

    def signature(self) -> tuple:
        return (self.params.dims, self.params.nnz, self.params.m, self.params.g)

    def pointer_entries(self) -> int:
        return sum(self.total_shards(n) for n in range(self.num_modes))


def plan_from_counts(params: PartitionParams, counts_per_mode) -> PartitionPlan:
    """Shard geometry from super-shard fills (layout.py:487-497)."""
    g, nnz = params.g, params.nnz
    cols = {k: [] for k in ("c", "o", "s", "f", "so")}
    for n, counts in enumerate(counts_per_mode):
        counts = np.asarray(counts, dtype=np.int64)
        offs = np.concatenate(([0], np.cumsum(counts))).astype(np.int64)
        shards = -(-counts // g)
        first = np.concatenate(([0], np.cumsum(shards))).astype(np.int64)
        ss_of = np.repeat(np.arange(params.k[n], dtype=np.int64), shards)
        q = np.arange(int(first[-1]), dtype=np.int64) - first[ss_of]
        soffs = np.concatenate((offs[ss_of] + q * g, [nnz])).astype(np.int64)
        for key, arr in zip(("c", "o", "s", "f", "so"), (counts, offs, shards, first, soffs)):
            cols[key].append(arr)
    return PartitionPlan(params, tuple(cols["c"]), tuple(cols["o"]), tuple(cols["s"]),
                         tuple(cols["f"]), tuple(cols["so"]))


@dataclass
class ModeWork:
    """Static CTA work plan of one mode (see fc_mode_worker in flycoo.h)."""
    acc_in_smem: bool
    nchunks: int
    chunk_start: torch.Tensor   # int64 (nchunks + 1)
    chunk_ss: torch.Tensor      # int32
    chunk_part: torch.Tensor    # int32
    chunk_rows: torch.Tensor | None  # int32 rows per chunk when small super-shards are merged
    tile_rows: int              # accumulator tile height (m)
    hist_rows: int              # max rows of any chunk (direct chunks: <= 256)
    red1: torch.Tensor          # int64 (nred1, 4): ss, p0, p1, dst
    nred1: int
    red2: torch.Tensor          # int64 (nred2, 3): ss, q0, q1
    nred2: int
    nparts: int
    part_ws: torch.Tensor | None
    part_ws2: torch.Tensor | None
    chunk_elems: int
    # tile plan (engine.build_tile_plans): every element's position in its
    # row-sorted 2048-element tile and every tile's bin starts, uint16 bits
    tile_perm: torch.Tensor | None = None
    tile_bins: torch.Tensor | None = None

    @property
    def launches(self) -> int:
        """Kernels one mode pass launches (K1, plus the K2 levels)."""
        return 1 + (1 if self.nred1 else 0) + (1 if self.nred2 else 0)


REDUCE_FAN = 64  # partials summed per level-1 reduce task


def reduce_plan(nch: np.ndarray, part_base: np.ndarray, fan: int = REDUCE_FAN):
    """Two-level deterministic reduce tasks (fc_mode_worker K2) for the
    super-shards with 0 or >= 2 chunks."""
    red1, red2 = [], []
    slot = 0
    for ss in np.nonzero((nch == 0) | (nch >= 2))[0]:
        P = int(nch[ss]) if nch[ss] >= 2 else 0
        p0 = int(part_base[ss])
        if P <= fan:
            red1.append((ss, p0, p0 + P, -1))
            continue
        groups = -(-P // fan)
        for g in range(groups):
            red1.append((ss, p0 + g * fan, p0 + min(P, (g + 1) * fan), slot + g))
        red2.append((ss, slot, slot + groups))
        slot += groups
    r1 = np.asarray(red1, dtype=np.int64).reshape(-1, 4)
    r2 = np.asarray(red2, dtype=np.int64).reshape(-1, 3)
    return r1, r2, slot


BIG_SS_AVG = 400_000  # super-shards averaging this many nonzeros get 32k-element chunks


def default_chunk_elems(nnz: int, tile: int = 2048, avg_ss: float = 0.0) -> int:
    """Chunk size: 8192 elements, smaller for small tensors so that every
    SM gets work (multiples of the 2048-element tile); 32768 for modes whose
    super-shards average >= 400k nonzeros (c5: a quarter of the partial tiles
    to write and reduce, 45.8 -> 44.9 ms at 1B nonzeros; c2 and c4 are
    neutral or slower with larger chunks and stay below the threshold)."""
    env = os.environ.get("FLYCOO_CHUNK")
    cap = int(env) if env else (32768 if avg_ss >= BIG_SS_AVG else 8192)
    want = _cdiv(max(int(nnz), 1), 148 * 4)
    return int(min(cap, max(tile, _cdiv(want, tile) * tile)))


PART_DIRECT = -2  # chunk_part of a direct chunk (see fc_mode_worker)


def direct_groups(counts: np.ndarray, tile: int, group: int):
    """Greedy packing of consecutive super-shards into direct chunks: at most
    `group` super-shards and at most one tile of nonzeros each (empty
    super-shards included).  Super-shards larger than a tile are left alone
    (n_ss = 0 marks them).  Returns (first_ss, n_ss) per chunk group."""
    first, nss = [], []
    k = counts.shape[0]
    i = 0
    while i < k:
        if int(counts[i]) > tile:
            first.append(i)
            nss.append(0)
            i += 1
            continue
        j, tot = i, 0
        while j < k and j - i < group and tot + int(counts[j]) <= tile:
            tot += int(counts[j])
            j += 1
        first.append(i)
        nss.append(j - i)
        i = j
    return np.asarray(first, dtype=np.int64), np.asarray(nss, dtype=np.int64)


def plan_chunk_elems(plan: PartitionPlan, mode: int, rank: int, merge: bool = True) -> int:
    """The chunk size :func:`make_mode_work` picks for the whole-tensor plan
    of `mode` -- what a partitioned sweep passes for its slices so that its
    chunks, partial tiles and sums are the single-GPU ones."""
    L = _lib.load()
    m = int(plan.params.m[mode])
    k = int(np.asarray(plan.ss_counts[mode]).shape[0])
    nnz = plan.nnz
    tile = int(L.fc_tile_elems())
    smem = m <= int(L.fc_smem_acc_rows_max(int(rank)))
    sparse = nnz < tile * max(k, 1)
    rows_cap = int(L.fc_chunk_rows_max(plan.num_modes, int(rank), m)) if smem else m
    if smem and merge and sparse and rows_cap // m > 1:
        return default_chunk_elems(nnz, tile)
    # (3-mode tensors only: c3's 4-mode tile kernel was slower with 32k chunks)
    return default_chunk_elems(nnz, tile, avg_ss=nnz / max(k, 1) if plan.num_modes == 3 else 0.0)


def make_mode_work(plan: PartitionPlan, mode: int, rank: int, device, chunk_elems: int | None = None,
                   merge: bool = True, ss_range: tuple | None = None) -> ModeWork:
    """Split every super-shard of `mode` into CTA chunks.  Shared-memory
    accumulation (m rows fit): chunks of `chunk_elems`, super-shards with
    several chunks get one partial tile per chunk, summed in chunk order by
    K2; on the fast path consecutive small super-shards are merged into one
    chunk (rows <= fc_chunk_rows_max).  Otherwise one chunk per super-shard
    accumulating in `out`.  `ss_range` = (lo, hi) restricts the work to those
    super-shards (a GPU's owned range in the multi-GPU sweep): no chunks or
    zeroing tasks for the rows other GPUs own."""
    L = _lib.load()
    params = plan.params
    m = int(params.m[mode])
    counts = np.asarray(plan.ss_counts[mode], dtype=np.int64)
    offs = np.asarray(plan.ss_elem_offsets[mode], dtype=np.int64)
    lo, hi = (0, counts.shape[0]) if ss_range is None else (int(ss_range[0]), int(ss_range[1]))
    counts, offs = counts[lo:hi], offs[lo:hi + 1]
    k = counts.shape[0]
    nnz = int(offs[-1]) if ss_range is not None else plan.nnz  # end of the last chunk
    tile = int(L.fc_tile_elems())
    smem = m <= int(L.fc_smem_acc_rows_max(int(rank)))
    dev = torch.device(device)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    # Sparse modes (super-shards average less than one tile of nonzeros):
    # consecutive small super-shards become "direct" chunks -- whole rows in
    # one tile, stored straight to `out` -- instead of one tiny chunk each.
    sparse = nnz < tile * max(k, 1)
    rows_cap = int(L.fc_chunk_rows_max(params.num_modes, int(rank), m)) if smem else m
    group = rows_cap // m if (merge and sparse) else 1
    if smem and group > 1:
        C = int(chunk_elems or default_chunk_elems(nnz, tile))
        first, nss = direct_groups(counts, tile, group)
        big = nss == 0
        pieces = np.where(big, -(-counts[first] // C), 1)
        total = int(pieces.sum())
        grp_of = np.repeat(np.arange(first.shape[0], dtype=np.int64), pieces)
        j = np.arange(total, dtype=np.int64) - np.concatenate(([0], np.cumsum(pieces)))[:-1][grp_of]
        ss_of = first[grp_of]
        starts = offs[ss_of] + j * C
        chunk_start = np.concatenate((starts, [nnz])).astype(np.int64)
        rows = np.minimum(np.where(big[grp_of], 1, nss[grp_of]) * m,
                          params.dims[mode] - (ss_of + lo) * m).astype(np.int32)
        nch_ss = np.ones(k, dtype=np.int64)
        nch_ss[first[big]] = pieces[big]
        multi = nch_ss >= 2
        part_base = np.concatenate(([0], np.cumsum(np.where(multi, nch_ss, 0))))
        part = np.where(big[grp_of],
                        np.where(multi[ss_of], part_base[:-1][ss_of] + j, -1),
                        PART_DIRECT).astype(np.int32)
        nparts = int(part_base[-1])
        r1, r2, nslots = reduce_plan(nch_ss, part_base)
        r1[:, 0] += lo
        r2[:, 0] += lo
        ws = (torch.empty(max(nparts * m * rank, 1), dtype=torch.float32, device=dev)
              if nparts or r1.shape[0] else None)
        ws2 = torch.empty(nslots * m * rank, dtype=torch.float32, device=dev) if nslots else None
        return ModeWork(True, total, t(chunk_start), t((ss_of + lo).astype(np.int32)), t(part), t(rows),
                        m, int(rows.max()) if rows.size else m, t(r1), int(r1.shape[0]), t(r2),
                        int(r2.shape[0]), nparts, ws, ws2, C)
    if smem:
        if chunk_elems is None:
            # (3-mode tensors only: c3's 4-mode tile kernel was slower with 32k chunks)
            chunk_elems = default_chunk_elems(
                nnz, tile, avg_ss=nnz / max(k, 1) if params.num_modes == 3 else 0.0)
        C = int(chunk_elems)
        nch = -(-counts // C)
    else:
        C = 0
        nch = (counts > 0).astype(np.int64)
    total = int(nch.sum())
    ss_of = np.repeat(np.arange(k, dtype=np.int64), nch)
    first_chunk = np.concatenate(([0], np.cumsum(nch)))[:-1]
    j = np.arange(total, dtype=np.int64) - first_chunk[ss_of]
    starts = offs[ss_of] + (j * C if smem else 0)
    chunk_start = np.concatenate((starts, [nnz])).astype(np.int64)
    if smem:
        multi = nch >= 2
        part_base = np.concatenate(([0], np.cumsum(np.where(multi, nch, 0))))
        part = np.where(multi[ss_of], part_base[:-1][ss_of] + j, -1).astype(np.int32)
        nparts = int(part_base[-1])
        r1, r2, nslots = reduce_plan(nch, part_base)
        r1[:, 0] += lo
        r2[:, 0] += lo
    else:
        part = np.full(total, -1, dtype=np.int32)
        nparts, nslots = 0, 0
        r1 = np.zeros((0, 4), dtype=np.int64)
        r2 = np.zeros((0, 3), dtype=np.int64)
    # K2 also zeroes the rows of empty super-shards (tasks with no partials),
    # so a plan can have reduce tasks but no partial tiles: 1-float workspace
    ws = (torch.empty(max(nparts * m * rank, 1), dtype=torch.float32, device=dev)
          if nparts or r1.shape[0] else None)
    ws2 = torch.empty(nslots * m * rank, dtype=torch.float32, device=dev) if nslots else None
    return ModeWork(smem, total, t(chunk_start), t((ss_of + lo).astype(np.int32)), t(part), None, m, m,
                    t(r1), int(r1.shape[0]), t(r2), int(r2.shape[0]), nparts, ws, ws2, C)


class DeviceShardedTensor:
    """Double-buffered FLYCOO tensor resident in HBM (the reference's
    ShardedTensor, layout.py:384-459, with device buffers)."""

    def __init__(self, plan: PartitionPlan, crd, val, slot_maps, device):
        self.plan = plan
        self.crd = crd              # [2] int32 (nnz, CW)
        self.val = val              # [2] float32 (nnz,) or [None, None]
        self.slot_maps = slot_maps  # per mode int32 (uint32 bits) (nnz,)
        self.device = torch.device(device)
        self.active = 0
        self.active_mode = 0
        self.canonical = True
        self._work = {}
        self._tile_plans_tried = {}  # rank -> tile plans were considered (engine.build_tile_plans)
        # [processed elements, error flags] for the deferred end-of-pass checks
        self._stat = torch.zeros(2, dtype=torch.int64, device=self.device)
        self._expected = 0
        self._sids = None           # per-element shard ids, only for the cursor strategy
        self._back_mode = None      # mode whose order the back buffer holds (None: unwritten)
        self.build_stages = {}      # build stage -> seconds (CUDA events), set by the builders

    # --------------------------------------------------------------- props
    @property
    def params(self) -> PartitionParams:
        return self.plan.params

    @property
    def nnz(self) -> int:
        return self.plan.nnz

    @property
    def num_modes(self) -> int:
        return self.plan.num_modes

    @property
    def element_nbytes(self) -> int:
        return record_bytes(self.num_modes)

    def swap(self, new_mode: int, still_canonical: bool) -> None:
        self._back_mode = self.active_mode
        self.active = 1 - self.active
        self.active_mode = new_mode
        self.canonical = self.canonical and still_canonical

    def mode_work(self, mode: int, rank: int) -> ModeWork:
        key = (mode, rank)
        if key not in self._work:
            self._work[key] = make_mode_work(self.plan, mode, rank, self.device)
        return self._work[key]

    # ----------------------------------------------------- host-side views
    def device_arrays(self, which: int | None = None):
        b = self.active if which is None else which
        return self.crd[b], self.val[b]

    def _host_coords_vals(self, which: int):
        crd, val = self.crd[which], self.val[which]
        N = self.num_modes
        c = crd[:, :N].to(torch.int64).cpu().numpy()
        if val is None:
            v = crd[:, -1].view(torch.float32).cpu().numpy().astype(np.float64)
        else:
            v = val.cpu().numpy().astype(np.float64)
        return c, v

    def positions_in_mode(self, mode: int, from_mode: int | None = None) -> torch.Tensor:
        """Mode-`mode` buffer position of every element of a buffer ordered
        for `from_mode` (default: the active buffer) -- composition of slot
        maps; needs the canonical arrangement."""
        if not self.canonical:
            raise ValueError("positions are only defined for the canonical arrangement")
        N = self.num_modes
        pos = torch.arange(self.nnz, device=self.device, dtype=torch.int64)
        n = self.active_mode if from_mode is None else from_mode
        while n != mode:
            pos = (self.slot_maps[n].to(torch.int64) & 0xFFFFFFFF)[pos]
            n = (n + 1) % N
        return pos

    def shard_ids(self, which: int | None = None) -> np.ndarray:
        """(nnz, N) int64 shard id per mode of a buffer's elements (default:
        the active buffer; zeros for a back buffer no pass has written yet,
        like the reference's freshly built back buffer, layout.py:526-528)."""
        b = self.active if which is None else which
        if self._sids is not None:
            return self._sids[b].to(torch.int64).cpu().numpy()
        from_mode = self.active_mode if b == self.active else self._back_mode
        out = np.zeros((self.nnz, self.num_modes), dtype=np.int64)
        if from_mode is None:
            return out
        for w in range(self.num_modes):
            pos = self.positions_in_mode(w, from_mode).cpu().numpy()
            out[:, w] = np.searchsorted(self.plan.shard_offsets[w], pos, side="right") - 1
        return out

    def active_arrays(self):
        """(sids, idxs, vals) of the active buffer as host numpy arrays in the
        reference's dtypes (int64, int64, float64) -- a validation view, not
        the hot path (layout.py:419-421)."""
        c, v = self._host_coords_vals(self.active)
        return self.shard_ids(), c, v

    def back_arrays(self):
        """(sids, idxs, vals) of the back buffer (layout.py:423-425): the
        previous mode's arrangement after a pass, zeros before the first."""
        b = 1 - self.active
        if self._back_mode is None and self._sids is None:
            z = np.zeros((self.nnz, self.num_modes), dtype=np.int64)
            return z, z.copy(), np.zeros(self.nnz)
        c, v = self._host_coords_vals(b)
        return self.shard_ids(b), c, v

    def to_coo(self, dims=None):
        """The active buffer as a validated :class:`~.coo.CooTensor`
        (layout.py:432-434)."""
        from .coo import CooTensor
        c, v = self._host_coords_vals(self.active)
        return CooTensor(tuple(dims or self.params.dims), c, v)

    def accounting(self) -> dict:
        plan_aux = sum(a.size for g in (self.plan.ss_counts, self.plan.ss_elem_offsets,
                                        self.plan.ss_shard_counts, self.plan.ss_first_shard)
                       for a in g)
        buf = sum(t.numel() * t.element_size() for t in self.crd)
        buf += sum(t.numel() * t.element_size() for t in self.val if t is not None)
        return {
            "buffer_elements": 2 * self.nnz,
            "element_bytes": self.element_nbytes,
            "buffer_bytes": buf,
            "remap_pointer_entries": self.plan.pointer_entries(),
            "slot_rank_entries": sum(s.numel() for s in self.slot_maps),
            "plan_aux_entries": plan_aux,
        }

    # ------------------------------------------------------ deferred checks
    def reset_checks(self):
        self._stat.zero_()
        self._expected = 0

    def stat_ptrs(self):
        base = self._stat.data_ptr()
        return base + 8, base  # (flags int32*, processed u64*)


# ------------------------------------------------------------------- build

def _stream_ptr():
    return torch.cuda.current_stream().cuda_stream


def _bitlen(x: int) -> int:
    return int(x).bit_length()


_MIX1 = -7046029254386353131   # 0x9E3779B97F4A7C15 as int64 (splitmix64 constants)
_MIX2 = -4658895280553007687   # 0xBF58476D1CE4E5B9
_MIX3 = -7723592293110705685   # 0x94D049BB133111EB


def _mix64(x: torch.Tensor) -> torch.Tensor:
    """splitmix64 finaliser on int64 tensors (two's-complement wrap-around;
    logical shifts emulated with masks)."""
    x = x * _MIX2
    x = x ^ ((x >> 30) & ((1 << 34) - 1))
    x = x * _MIX3
    return x ^ ((x >> 31) & ((1 << 33) - 1))


_BUCKET_KEYS = 1 << 28  # keys per sort bucket of the duplicate check


def device_has_duplicates(coords: torch.Tensor, dims, buckets: int | None = None) -> bool:
    """True iff two rows of the (nnz, N) integer coordinate tensor are equal
    -- the reference's "duplicate coordinates" check (coo.py:88-89), run
    where the coordinates live.  Rows are keyed by their row-major flattened
    index when prod(dims) fits 63 bits (exact), else by a 64-bit hash whose
    equal-hash groups are compared coordinate by coordinate; the keys are
    sorted in hash buckets so the sort scratch stays ~nnz/buckets * 24 B."""
    nnz, N = int(coords.shape[0]), int(coords.shape[1])
    if nnz < 2:
        return False
    dims = [int(d) for d in dims]
    exact = int(np.prod(np.asarray(dims, dtype=object))) < (1 << 63)
    key = torch.zeros(nnz, dtype=torch.int64, device=coords.device)
    for n in range(N):
        c = coords[:, n].to(torch.int64)
        if exact:
            key.mul_(dims[n]).add_(c)
        else:
            salt = (((n + 1) * _MIX1 + (1 << 63)) % (1 << 64)) - (1 << 63)  # wrapped to int64
            key = _mix64(key ^ _mix64(c + salt))
    if buckets is None:  # a power of two, <= _BUCKET_KEYS keys per bucket on average, <= 16
        buckets = 1
        while buckets < 16 and nnz > buckets * _BUCKET_KEYS:
            buckets *= 2
    bsel = _mix64(key) & (buckets - 1) if buckets > 1 and (buckets & (buckets - 1)) == 0 else None
    if buckets > 1 and bsel is None:
        raise ValueError("buckets must be a power of two")
    for b in range(buckets):
        idx = torch.arange(nnz, device=key.device) if bsel is None else torch.nonzero(bsel == b).squeeze(1)
        if idx.numel() < 2:
            continue
        kv, perm = torch.sort(key[idx])
        eq = kv[1:] == kv[:-1]
        if not bool(eq.any()):
            continue
        if exact:
            return True
        # hash collisions or true duplicates: compare the rows of every
        # equal-hash group exactly (on the host; groups are tiny)
        at = torch.nonzero(eq).squeeze(1)
        members = torch.unique(torch.cat([at, at + 1]))
        rows = idx[perm[members]]
        sub = coords[rows].to(torch.int64).cpu().numpy()
        hk = kv[members].cpu().numpy()
        for h in np.unique(hk):
            grp = sub[hk == h]
            if len(np.unique(grp, axis=0)) != len(grp):
                return True
    return False


class _StageClock:
    """CUDA-event timestamps between build stages (PAPER.md:762 reports the
    super-shard generation, Morton ordering and shard generation stages)."""

    def __init__(self):
        self.marks = [("start", torch.cuda.Event(enable_timing=True))]
        self.marks[0][1].record()

    def mark(self, name: str):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.marks.append((name, e))

    def seconds(self) -> dict:
        self.marks[-1][1].synchronize()
        out = {}
        for (_, a), (name, b) in zip(self.marks, self.marks[1:]):
            out[name] = out.get(name, 0.0) + a.elapsed_time(b) / 1e3
        return out


def build_sharded(tensor, params: PartitionParams, device="cuda") -> DeviceShardedTensor:
    """The reference's ``build_sharded(tensor, params)`` (layout.py:462-531):
    `tensor` is a :class:`~.coo.CooTensor` -- this package's or the
    reference's, anything with ``dims``, ``subs`` and ``vals`` -- already
    validated on construction (no duplicates), so the device build skips its
    own duplicate check."""
    dims = tuple(int(d) for d in tensor.dims)
    if tuple(params.dims) != dims:
        raise ValueError("params were selected for different dims")
    nnz = int(np.asarray(tensor.vals).shape[0])
    if params.nnz != nnz:
        raise ValueError("params were selected for a different nonzero count")
    return build_device_sharded(tensor.subs, tensor.vals, params, device=device,
                                check_duplicates=False)


def build_device_sharded(subs, vals, params: PartitionParams, device="cuda",
                         check_duplicates: bool = True) -> DeviceShardedTensor:
    """Device build of the FLYCOO layout (layout.py:462-531 + the B200
    intra-shard order).  `subs` (nnz, N) and `vals` (nnz,) in input order,
    as numpy arrays or torch tensors (any device).  Raises ValueError on
    duplicate coordinates (coo.py:88-89) unless `check_duplicates` is False
    (inputs that are duplicate-free by construction).  The stage times land
    in ``st.build_stages`` (seconds, CUDA events)."""
    L = _lib.load()
    dev = torch.device(device)
    subs_t = torch.as_tensor(subs)
    vals_t = torch.as_tensor(vals)
    nnz, N = int(subs_t.shape[0]), int(subs_t.shape[1])
    if tuple(params.dims) != tuple(int(d) for d in params.dims) or len(params.dims) != N:
        raise ValueError("params were selected for different dims")
    if params.nnz != nnz:
        raise ValueError("params were selected for a different nonzero count")
    if nnz >= 1 << 32:
        raise ValueError("nnz must fit uint32 positions")
    if max(params.dims) >= 1 << 31:
        raise ValueError("dims must fit int32 coordinates")
    clock = _StageClock()
    coords = subs_t.to(device=dev, dtype=torch.int32).contiguous()
    fvals = vals_t.to(device=dev, dtype=torch.float32).contiguous()
    clock.mark("upload")
    if check_duplicates:
        if nnz and (int(coords.min()) < 0 or bool((coords.max(0).values.cpu()
                                                   >= torch.as_tensor(params.dims)).any())):
            raise ValueError("coordinates outside the declared dims")
        if device_has_duplicates(coords, params.dims):
            raise ValueError("duplicate coordinates (coalesce first)")
        clock.mark("duplicate_check")
    st = _stream_ptr()
    P = lambda t: t.data_ptr() if t is not None else None
    m_arr = _lib.i64_array(params.m)
    k_arr = _lib.i64_array(params.k)

    # Memory-lean sequence (peak ~ coords + 2 sort key arrays + a few u32
    # arrays; the billion-nonzero configs need it):
    #   1. Morton keys, then ONE stable sort of element ids by (hi, lo):
    #      the mode-independent "Morton order" (ties by input position);
    #   2. per mode, canonical order = stable sort of the Morton order by
    #      iv_n (= lexsort(seq, lo, hi, iv_n), layout.py:484); its histogram
    #      gives the plan, and it is reduced to shard ids at once;
    #   3. per mode, B200 order = stable sort of the Morton order by
    #      (sid_n, sid_{n-1}); only its inverse (positions) is kept;
    #   4. slot maps and the mode-0 records by scatter from positions.
    widths = [_bitlen(k - 1) for k in params.k]
    W = sum(widths)
    lo = torch.empty(nnz, dtype=torch.int64, device=dev)
    hi = torch.empty(nnz, dtype=torch.int64, device=dev) if W > 64 else None
    _lib.call("fc_build_morton", P(coords), nnz, N, m_arr, k_arr, P(hi), P(lo), st)

    temp_bytes = int(L.fc_build_sort_temp_bytes(max(nnz, 1)))
    temp = torch.empty(max(temp_bytes, 1), dtype=torch.uint8, device=dev)
    keys_a = torch.empty(nnz, dtype=torch.int64, device=dev)
    keys_b = torch.empty(nnz, dtype=torch.int64, device=dev)

    def sort_by(ids, what, end_bit, mode=0, m=1, shift=0):
        """stable sort of `ids` by key f(id) on bits [0, end_bit)"""
        if end_bit <= 0:
            return ids
        _lib.call("fc_build_gather_key", P(ids), nnz, what, P(hi), P(lo), P(coords), N, mode, m,
                  shift, P(keys_a), st)
        out = torch.empty_like(ids)
        _lib.call("fc_build_sort_pairs", P(keys_a), P(keys_b), P(ids), P(out), nnz, min(end_bit, 64),
                  P(temp), temp_bytes, st)
        return out

    ids = torch.arange(nnz, dtype=torch.int32, device=dev)
    morton = sort_by(ids, 0, min(W, 64))
    if W > 64:
        morton = sort_by(morton, 1, W - 64)
    del ids, hi, lo
    hi = lo = None
    clock.mark("morton_order")

    counts_all, sids = [], []
    hist = torch.empty(max(params.k), dtype=torch.int64, device=dev)
    for n in range(N):
        order = sort_by(morton, 2, _bitlen(params.k[n] - 1), n, params.m[n])
        _lib.call("fc_build_ss_hist", P(coords), nnz, N, n, params.m[n], params.k[n], P(hist), st)
        counts = hist[: params.k[n]].cpu().numpy().astype(np.int64)
        if int(counts.sum()) != nnz:
            raise ValueError("coordinates outside the declared dims")
        counts_all.append(counts)
        # this mode's super-shard offsets and first shard ids (layout.py:487-490)
        offs = torch.from_numpy(np.concatenate(([0], np.cumsum(counts))).astype(np.int64)).to(dev)
        first = torch.from_numpy(np.concatenate(([0], np.cumsum(-(-counts // params.g))))
                                 .astype(np.int64)).to(dev)
        sid = torch.empty(nnz, dtype=torch.int32, device=dev)
        _lib.call("fc_build_shard_ids", P(order), nnz, P(coords), N, n, params.m[n], P(offs),
                  P(first), params.g, P(sid), st)
        sids.append(sid)
        del order
    plan = plan_from_counts(params, counts_all)
    clock.mark("super_shards")

    gpos = []
    for n in range(N):
        prev = (n - 1) % N
        end_bit = 32 + _bitlen(plan.total_shards(n) - 1)
        _lib.call("fc_build_device_key", P(morton), nnz, P(sids[n]), P(sids[prev]), P(keys_a), st)
        g_ord = torch.empty_like(morton)
        _lib.call("fc_build_sort_pairs", P(keys_a), P(keys_b), P(morton), P(g_ord), nnz,
                  min(end_bit, 64), P(temp), temp_bytes, st)
        pos = torch.empty(nnz, dtype=torch.int32, device=dev)
        _lib.call("fc_build_invert", P(g_ord), nnz, P(pos), st)
        gpos.append(pos)
        del g_ord
    del sids, morton, keys_a, keys_b, temp
    slot_maps = []
    for n in range(N):
        slot = torch.empty(nnz, dtype=torch.int32, device=dev)
        _lib.call("fc_build_slots_scatter", P(gpos[n]), P(gpos[(n + 1) % N]), nnz, P(slot), st)
        slot_maps.append(slot)
    cw = int(L.fc_crd_words(N))
    emb = bool(L.fc_value_embedded(N))
    crd = [torch.empty((nnz, cw), dtype=torch.int32, device=dev),
           torch.empty((nnz, cw), dtype=torch.int32, device=dev)]
    val = [None, None] if emb else [torch.empty(nnz, dtype=torch.float32, device=dev),
                                    torch.empty(nnz, dtype=torch.float32, device=dev)]
    _lib.call("fc_build_records_scatter", P(gpos[0]), nnz, N, P(coords), P(fvals), P(crd[0]),
              P(val[0]), st)
    del gpos
    clock.mark("shards_slots_records")
    out = DeviceShardedTensor(plan, crd, val, tuple(slot_maps), dev)
    out.build_stages = clock.seconds()
    return out


def build_device_sharded_lean(records, params: PartitionParams, device="cuda",
                              batch: int = 1 << 27) -> DeviceShardedTensor:
    """:func:`build_device_sharded` for a tensor whose layout fills most of
    HBM (config 5: 3.6B nonzeros, 158 GB of records + slot maps): the same
    plan, orders, slot maps and records (bit-identical), built inside the
    memory of the final buffers.

    `records` is the input COO as 16-B records (nnz, 4) int32
    ``{c0, c1, c2, bits(v)}`` (N <= 3, value embedded) in input order; a
    device `records` tensor is consumed (overwritten: it becomes the back
    buffer).  Sort keys are 32 bits (Morton keys of <= 32 bits, iv_n, shard
    ids; the (sid_n, sid_{n-1}) key as two stable passes), the scratch lives
    in the second record buffer and the not-yet-written slot maps, and the
    input records wait in host memory while their device copy is reused for
    the positions.  Peak device memory = the final layout + sort temp."""
    L = _lib.load()
    dev = torch.device(device)
    nnz, cw = int(records.shape[0]), int(records.shape[1])
    N = len(params.dims)
    if not (N <= 3 and cw == 4 and int(L.fc_crd_words(N)) == 4 and L.fc_value_embedded(N)):
        raise ValueError("the lean build takes 16-B records of a 2- or 3-mode tensor")
    if params.nnz != nnz:
        raise ValueError("params were selected for a different nonzero count")
    if nnz >= 1 << 32:
        raise ValueError("nnz must fit uint32 positions")
    widths = [_bitlen(k - 1) for k in params.k]
    if sum(widths) > 32:
        raise ValueError("the lean build needs a Morton key of <= 32 bits")
    st = _stream_ptr()
    P = lambda t: t.data_ptr()
    m_arr = _lib.i64_array(params.m)
    k_arr = _lib.i64_array(params.k)
    clock = _StageClock()
    crd = records.to(dev).contiguous()
    clock.mark("upload")

    other = torch.empty((nnz, 4), dtype=torch.int32, device=dev)
    A, B, C, D = (other.view(-1)[i * nnz:(i + 1) * nnz] for i in range(4))
    S = [torch.empty(nnz, dtype=torch.int32, device=dev) for _ in range(N)]
    temp_bytes = int(L.fc_build_sort32_temp_bytes(max(nnz, 1)))
    temp = torch.empty(max(temp_bytes, 1), dtype=torch.uint8, device=dev)

    def sort32(keys, ids_in, ids_out, bits):
        if bits <= 0:
            ids_out.copy_(ids_in)
            return
        _lib.call("fc_build_sort_pairs32", P(keys), P(B), P(ids_in), P(ids_out), nnz, min(bits, 32),
                  P(temp), temp_bytes, st)

    # Morton order (ties by input position): D
    _lib.call("fc_build_morton32", P(crd), nnz, N, 4, m_arr, k_arr, P(A), st)
    _lib.call("fc_build_iota", P(C), nnz, st)
    sort32(A, C, D, sum(widths))
    clock.mark("morton_order")
    # canonical orders -> plan and shard ids (S[n])
    counts_all = []
    hist = torch.empty(max(params.k), dtype=torch.int64, device=dev)
    for n in range(N):
        _lib.call("fc_build_iv_key32", P(D), nnz, P(crd), 4, n, params.m[n], P(A), st)
        sort32(A, D, C, _bitlen(params.k[n] - 1))
        _lib.call("fc_build_ss_hist", P(crd), nnz, 4, n, params.m[n], params.k[n], P(hist), st)
        counts = hist[: params.k[n]].cpu().numpy().astype(np.int64)
        if int(counts.sum()) != nnz:
            raise ValueError("coordinates outside the declared dims")
        counts_all.append(counts)
        offs = torch.from_numpy(np.concatenate(([0], np.cumsum(counts))).astype(np.int64)).to(dev)
        first = torch.from_numpy(np.concatenate(([0], np.cumsum(-(-counts // params.g))))
                                 .astype(np.int64)).to(dev)
        _lib.call("fc_build_shard_ids", P(C), nnz, P(crd), 4, n, params.m[n], P(offs), P(first),
                  params.g, P(S[n]), st)
    plan = plan_from_counts(params, counts_all)
    clock.mark("super_shards")

    # the input records wait on the host; their device memory holds positions
    # (the caller's tensor is overwritten: it becomes the back buffer)
    host = torch.empty((nnz, 4), dtype=torch.int32, pin_memory=False)
    for a in range(0, nnz, batch):
        host[a:a + batch].copy_(crd[a:a + batch])
    back, crd = crd, None
    E = back.view(-1)[:nnz]
    pos = [back.view(-1)[(i + 1) * nnz:(i + 2) * nnz] for i in range(N)]
    for n in range(N):
        prev = (n - 1) % N
        # B200 order: stable sort of the Morton order by (sid_n, sid_prev)
        _lib.call("fc_build_gather_u32", P(D), nnz, P(S[prev]), P(A), st)
        sort32(A, D, C, _bitlen(plan.total_shards(prev) - 1))
        _lib.call("fc_build_gather_u32", P(C), nnz, P(S[n]), P(A), st)
        sort32(A, C, E, _bitlen(plan.total_shards(n) - 1))
        _lib.call("fc_build_invert", P(E), nnz, P(pos[n]), st)
    for n in range(N):
        _lib.call("fc_build_slots_scatter", P(pos[n]), P(pos[(n + 1) % N]), nnz, P(S[n]), st)
    del temp
    # mode-0 records: scatter the input batches to their positions
    for a in range(0, nnz, batch):
        b = min(nnz, a + batch)
        stage = host[a:b].to(dev, non_blocking=False)
        _lib.call("fc_build_scatter_rec16", P(pos[0][a:b]), b - a, P(stage), P(other), st)
        del stage
    del host
    clock.mark("shards_slots_records")
    out = DeviceShardedTensor(plan, [other, back], [None, None], tuple(S), dev)
    out.build_stages = clock.seconds()
    return out


# -------------------------------------------------------------- validation

@dataclass(frozen=True)
class CheckResult:
    """One structural check of :func:`validate_plan` (layout.py:537-548)."""
    name: str
    passed: bool
    detail: str = ""

    def line(self) -> str:
        mark = "pass" if self.passed else "FAIL"
        suffix = f" ({self.detail})" if self.detail and not self.passed else ""
        return f"[{mark}] {self.name}{suffix}"


@dataclass(frozen=True)
class PlanReport:
    checks: tuple

    @property
    def passed(self) -> bool:
        return all(c.passed for c in self.checks)

    def first_failure(self):
        return next((c for c in self.checks if not c.passed), None)

    def format(self) -> str:
        return "\n".join(c.line() for c in self.checks)


def validate_plan(st: DeviceShardedTensor, source=None) -> PlanReport:
    """The reference's structural gate (layout.py:565-640) over the device
    tensor's host views: per mode, super-shard conservation, strictly rising
    shard offsets 0..nnz, every non-final shard holding exactly g elements,
    shard ids in range and each element inside its super-shard's interval;
    the active buffer in the active mode's shard order; the double buffer's
    byte count; and, given the source CooTensor, conservation of the
    nonzero multiset (values compared at the device's fp32 precision)."""
    plan, params = st.plan, st.params
    N, nnz = st.num_modes, st.nnz
    checks = []
    sids, idxs, vals = st.active_arrays()
    for n in range(N):
        total = int(plan.ss_counts[n].sum())
        checks.append(CheckResult(f"mode{n}-ss-conservation", total == nnz,
                                  f"super-shard fills sum to {total}, expected {nnz}"))
    for n in range(N):
        offs = plan.shard_offsets[n]
        ok = bool(np.all(np.diff(offs) > 0)) and int(offs[0]) == 0 and int(offs[-1]) == nnz
        checks.append(CheckResult(f"mode{n}-offsets", ok,
                                  "shard offsets must rise strictly from 0 to nnz"))
        fills = plan.shard_fills(n)
        last = plan.ss_first_shard[n][1:] - 1
        interior = np.ones(plan.total_shards(n), dtype=bool)
        interior[last[plan.ss_shard_counts[n] > 0]] = False
        bad = np.nonzero(fills[interior] != params.g)[0]
        checks.append(CheckResult(f"mode{n}-shard-fill", bad.size == 0,
                                  f"{bad.size} non-final shards not holding exactly g={params.g}"))
    for n in range(N):
        nshards = plan.total_shards(n)
        inrange = (sids[:, n] >= 0) & (sids[:, n] < nshards)
        if not inrange.all():
            e = int(np.argmin(inrange))
            checks.append(CheckResult(f"mode{n}-sid-range", False,
                                      f"element {e}: shard id {int(sids[e, n])} outside [0, {nshards})"))
            continue
        want = idxs[:, n] // params.m[n]
        got = plan.ss_of_shard(n)[sids[:, n]]
        ok = bool(np.array_equal(want, got))
        detail = ""
        if not ok:
            e = int(np.argmax(want != got))
            detail = (f"element {e}: index {int(idxs[e, n])} lies in interval {int(want[e])} but "
                      f"shard id {int(sids[e, n])} belongs to super-shard {int(got[e])}")
        checks.append(CheckResult(f"mode{n}-interval-containment", ok, detail))
    am = st.active_mode
    expected = np.repeat(np.arange(plan.total_shards(am), dtype=np.int64), plan.shard_fills(am))
    ok = bool(np.array_equal(sids[:, am], expected))
    detail = ""
    if not ok:
        e = int(np.argmax(sids[:, am] != expected))
        detail = f"position {e}: shard id {int(sids[e, am])}, plan assigns {int(expected[e])}"
    checks.append(CheckResult("active-order", ok, detail))
    acc = st.accounting()
    # stored bytes per record: the logical int32 coordinates + fp32 value,
    # padded to 32 B rows for N >= 5 (include/flycoo.h)
    L = _lib.load()
    stored = 4 * int(L.fc_crd_words(N)) + (0 if L.fc_value_embedded(N) else 4)
    want_bytes = 2 * nnz * stored
    checks.append(CheckResult("double-buffer-bytes", acc["buffer_bytes"] == want_bytes,
                              f"buffers hold {acc['buffer_bytes']} bytes, expected {want_bytes}"))
    if source is not None:
        # the device holds fp32 values: the source's values rounded to fp32
        from .coo import CooTensor
        sv = np.asarray(source.vals, dtype=np.float64).astype(np.float32).astype(np.float64)
        ok = CooTensor(tuple(source.dims), np.asarray(source.subs), sv) \
            .same_nonzeros(CooTensor(tuple(source.dims), idxs, vals))
        checks.append(CheckResult("conservation", ok,
                                  "active buffer nonzero multiset differs from the source tensor"))
    return PlanReport(tuple(checks))

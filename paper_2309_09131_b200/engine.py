"""Drop-in engine: mttkrp_mode / sweep_all_modes / remap_store on the B200.

Same signatures, preconditions, exceptions and counters as the reference
engine (/root/reference/pkg/src/modecycle/engine.py:28-293).  The per-thread
numba kernel and its thread fan-out (engine.py:214-245, _kernels.py:38-88)
become one stream-ordered call of ``fc_mode_worker`` (libflycoo, sm_100a),
whose CTAs own super-shard chunks.  There is no CPU path: the CUDA library
must be present.

Differences a caller can see, each forced by the device:
* ``st`` is a :class:`~.layout.DeviceShardedTensor`, ``factors`` a
  :class:`~.factors.DeviceFactorSet` (host FactorSet-likes are converted),
  outputs are fp32 CUDA tensors of shape (I_mode, R);
* ``workers`` is validated but the GPU decomposition ignores it, and the
  ScheduleMap is validated (engine.py:186-189) but its assignment unused;
* ``sweep_all_modes`` runs every mode back to back on the stream and checks
  the processed counts and device error flags once at the end (one host
  sync per sweep instead of one per mode); ``mode_seconds`` gets per-mode
  CUDA-event times.
"""

from __future__ import annotations

from dataclasses import dataclass

import os

import numpy as np
import torch

from . import _lib
from .factors import DeviceFactorSet
from .layout import DeviceShardedTensor

__all__ = ["TrafficCounters", "RemapCursors", "ShardOverflowError", "BufferOrderError",
           "mttkrp_mode", "sweep_all_modes", "remap_store", "REMAP_STRATEGIES"]

REMAP_STRATEGIES = ("slot", "cursor")

FLAG_SLOT_RANGE = 1
FLAG_ROW_OUTSIDE_SS = 2
FLAG_SHARD_OVERFLOW = 4
FLAG_INDEX_CHECK = 8  # checked build only (FC_DEVICE_CHECKS)


class ShardOverflowError(RuntimeError):
    """A destination shard received more elements than the plan assigns it."""


class BufferOrderError(ValueError):
    """The active buffer is not ordered for the requested mode/strategy."""


@dataclass
class TrafficCounters:
    """Model data-volume counters per mode, closed forms of engine.py:49-91
    (tensor read + rewritten once, N-1 rank-R factor rows gathered and one
    output row updated per element; factor entries counted at 8 bytes as in
    the reference model)."""

    tensor_bytes_read: int = 0
    factor_bytes_read: int = 0
    output_bytes_written: int = 0
    remap_bytes_written: int = 0

    def add_mode(self, nnz: int, num_modes: int, rank: int, element_bytes: int,
                 compute: bool = True, remap: bool = True) -> None:
        if compute:
            self.tensor_bytes_read += nnz * element_bytes
            self.factor_bytes_read += nnz * (num_modes - 1) * rank * 8
            self.output_bytes_written += nnz * rank * 8
        if remap:
            if not compute:
                self.tensor_bytes_read += nnz * element_bytes
            self.remap_bytes_written += nnz * element_bytes

    def total_bytes(self) -> int:
        return (self.tensor_bytes_read + self.factor_bytes_read + self.output_bytes_written
                + self.remap_bytes_written)

    def remap_ratio(self) -> float:
        other = self.tensor_bytes_read + self.factor_bytes_read + self.output_bytes_written
        return self.remap_bytes_written / other if other else 0.0

    def as_dict(self) -> dict:
        return {"tensor_bytes_read": self.tensor_bytes_read,
                "factor_bytes_read": self.factor_bytes_read,
                "output_bytes_written": self.output_bytes_written,
                "remap_bytes_written": self.remap_bytes_written,
                "remap_ratio": self.remap_ratio()}


@dataclass
class RemapCursors:
    """Fill records of the upcoming mode's shards (engine.py:94-121)."""

    base: np.ndarray
    fills: np.ndarray

    @classmethod
    def for_mode(cls, st, mode: int) -> "RemapCursors":
        base = st.plan.shard_offsets[mode]
        return cls(base=base, fills=np.zeros(base.shape[0] - 1, dtype=np.int64))

    def planned_fill(self, shard: int) -> int:
        return int(self.base[shard + 1] - self.base[shard])

    def reserve(self, shard: int) -> int:
        if self.fills[shard] >= self.planned_fill(shard):
            raise ShardOverflowError(
                f"shard {shard} already holds its planned {self.planned_fill(shard)} elements")
        slot = int(self.base[shard] + self.fills[shard])
        self.fills[shard] += 1
        return slot

    def complete(self) -> bool:
        return bool(np.array_equal(self.fills, np.diff(self.base)))


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ensure_sids(st: DeviceShardedTensor) -> None:
    """Materialise per-element shard ids (the reference's `sids`) for the
    cursor strategy; afterwards they travel with the elements."""
    if st._sids is None:
        sids = torch.from_numpy(st.shard_ids().astype(np.int32)).to(st.device)
        st._sids = [None, None]
        st._sids[st.active] = sids.contiguous()
        st._sids[1 - st.active] = torch.empty_like(sids)


def remap_store(element_row: int, next_mode: int, cursors: RemapCursors,
                st: DeviceShardedTensor) -> int:
    """Store one active element into its next-mode shard slot; returns the
    slot (engine.py:124-135, single-element mirror of the kernel remap)."""
    _ensure_sids(st)
    a, b = st.active, 1 - st.active
    shard = int(st._sids[a][element_row, next_mode])
    slot = cursors.reserve(shard)
    st.crd[b][slot] = st.crd[a][element_row]
    if st.val[a] is not None:
        st.val[b][slot] = st.val[a][element_row]
    st._sids[b][slot] = st._sids[a][element_row]
    return slot


def _coerce_factors(factors, device) -> DeviceFactorSet:
    if isinstance(factors, DeviceFactorSet):
        return factors
    # a reference FactorSet (numpy float64) or any object with .factors
    fs = getattr(factors, "factors", factors)
    lam = getattr(factors, "lambdas", None)
    return DeviceFactorSet(tuple(np.asarray(f, dtype=np.float32) if isinstance(f, np.ndarray) else f
                                 for f in fs), lam, device)


def check_errors(st: DeviceShardedTensor, next_mode: int | None = None) -> None:
    """Host check of the deferred device counters (engine.py:247-263)."""
    stat = st._stat.cpu()
    processed = int(stat[0])
    flags = int(stat[1]) & 0xFFFFFFFF
    expected = st._expected
    st.reset_checks()
    if flags & FLAG_INDEX_CHECK:
        raise RuntimeError("a kernel index check failed (checked build, FC_DEVICE_CHECKS)")
    if flags & FLAG_ROW_OUTSIDE_SS:
        raise BufferOrderError("an element's output row lies outside its super-shard: the active "
                               "buffer is not ordered for this mode")
    if flags & (FLAG_SLOT_RANGE | FLAG_SHARD_OVERFLOW):
        where = f" of mode {next_mode}" if next_mode is not None else ""
        raise ShardOverflowError(f"a destination shard{where} overflowed its planned fill")
    if processed != expected:
        raise RuntimeError(f"workers processed {processed} of {expected} elements")


def tile_plans_wanted(st: DeviceShardedTensor, rank: int) -> bool:
    """Tile plans cost 2 bytes per nonzero and mode; FLYCOO_TILE_PLAN=0/1
    forces them off/on, default: on when they fit in a third of the free
    device memory (config 5's 3.6B nonzeros keep the in-kernel ranking)."""
    env = os.environ.get("FLYCOO_TILE_PLAN")
    if env is not None:
        return env != "0"
    if not ((st.num_modes == 3 and rank in (16, 32)) or (st.num_modes == 4 and rank == 32)):
        return False
    # ~3 B per nonzero and mode with partial tiles; memory the caching
    # allocator holds but does not use counts as free
    free, _ = torch.cuda.mem_get_info(st.device)
    free += torch.cuda.memory_reserved(st.device) - torch.cuda.memory_allocated(st.device)
    return 3 * (3 * st.nnz * st.num_modes) < free


def build_tile_plans(st: DeviceShardedTensor, rank: int) -> bool:
    """Emit the tile plan of every mode (fc_tile_plan_emit) by walking the
    tensor once through its modes with remap-only passes (the layout and the
    chunk plan are static, so the per-tile sort the mode pass would redo in
    every sweep is done once here).  Needs the canonical mode-0 arrangement;
    returns False (and leaves no plan) when the kernels for this tensor do
    not take one.  The tensor ends as it started."""
    if st.active_mode != 0 or not st.canonical:
        raise BufferOrderError("tile plans are emitted from the canonical mode-0 arrangement")
    L = _lib.load()
    nmodes, params, dims = st.num_modes, st.params, st.params.dims
    works = [st.mode_work(n, rank) for n in range(nmodes)]
    if any(w.tile_perm is not None for w in works):
        return all(w.tile_perm is not None for w in works)
    if not all(w.acc_in_smem for w in works):
        return False
    check_errors(st)
    flags_p, proc_p = st.stat_ptrs()
    strm = _stream()
    val_p = lambda t: t.data_ptr() if t is not None else None
    plans = []
    ok = True
    failure = None
    for n in range(nmodes):
        w = works[n]
        a, b = st.active, 1 - st.active
        if ok:
            keys = int(L.fc_tile_plan_keys(st.nnz, w.nchunks))
            perm = torch.empty(keys * int(L.fc_tile_elems()), dtype=torch.int16, device=st.device)
            bins = torch.zeros(keys * w.hist_rows, dtype=torch.int16, device=st.device)
            dummy = _lib.ptr_array([st.crd[a].data_ptr()] * nmodes)  # factor rows are not read
            rc = L.fc_tile_plan_emit(
                st.crd[a].data_ptr(), val_p(st.val[a]), dummy, _lib.i64_array(dims), nmodes, n, rank,
                dims[n], params.m[n], w.chunk_start.data_ptr(), w.chunk_ss.data_ptr(),
                w.chunk_part.data_ptr(),
                w.chunk_rows.data_ptr() if w.chunk_rows is not None else None,
                w.tile_rows, w.hist_rows, w.nchunks, st.nnz, flags_p, proc_p, perm.data_ptr(),
                bins.data_ptr(), strm)
            if rc == _lib.ERR_UNSUPPORTED:
                ok = False
            elif rc != 0:  # raised after the walk has brought the tensor back to mode 0
                ok = False
                failure = _lib.FlycooError(
                    f"fc_tile_plan_emit failed ({rc}): {L.fc_last_error().decode(errors='replace')}")
            else:
                plans.append((perm, bins))
        # on to the next mode's arrangement: remap only
        _lib.call("fc_mode_worker", st.crd[a].data_ptr(), val_p(st.val[a]), st.crd[b].data_ptr(),
                  val_p(st.val[b]), None, None, None, nmodes, n, rank, dims[n], params.m[n],
                  None, None, None, None, 0, 0, 0, None, 0, None, 0, None, None,
                  st.slot_maps[n].data_ptr(), st.nnz, 0, 1, 1, flags_p, proc_p, strm)
        st._expected += st.nnz
        st.swap((n + 1) % nmodes, still_canonical=True)
    check_errors(st)
    if failure is not None:
        raise failure
    if ok:
        for w, (perm, bins) in zip(works, plans):
            w.tile_perm, w.tile_bins = perm, bins
    return ok


def mttkrp_mode(st: DeviceShardedTensor, factors, mode: int, smap, workers: int | None = None,
                remap: str = "slot", counters: TrafficCounters | None = None,
                split_remap: bool = False, alloc_log: dict | None = None, *,
                check: bool = True) -> torch.Tensor:
    """Output factor for `mode`; leaves the tensor ordered for mode
    (mode + 1) % N (engine.py:163-266).  For a fixed active order the result
    is bitwise reproducible (fixed-order sums, no data atomics)."""
    plan, params = st.plan, st.params
    nmodes = st.num_modes
    if not 0 <= mode < nmodes:
        raise ValueError(f"mode {mode} out of range")
    if st.active_mode != mode:
        raise BufferOrderError(f"active buffer is ordered for mode {st.active_mode}, not {mode}")
    if smap.plan_signature != plan.signature():
        raise ValueError("schedule was built for a different plan")
    if smap.num_modes != nmodes:
        raise ValueError("schedule does not cover this tensor's modes")
    if remap not in REMAP_STRATEGIES:
        raise ValueError(f"unknown remap strategy {remap!r}")
    if remap == "slot" and not st.canonical:
        raise BufferOrderError(
            "deterministic-slot remap needs the canonical build order; this tensor was last "
            "remapped with the cursor strategy")
    factors = _coerce_factors(factors, st.device)
    factors.require_match(params.dims)
    rank = factors.rank
    next_mode = (mode + 1) % nmodes
    workers = smap.nu if workers is None else int(workers)
    if workers < 1:
        raise ValueError("need at least one worker")

    L = _lib.load()
    work = st.mode_work(mode, rank)
    if (work.tile_perm is None and mode == 0 and st.canonical and not st._tile_plans_tried.get(rank)
            and remap == "slot"):
        # first pass over a fresh tensor: the static per-tile sort is planned once
        st._tile_plans_tried[rank] = True
        if tile_plans_wanted(st, rank):
            build_tile_plans(st, rank)
    dims = params.dims
    out = (torch.empty if work.acc_in_smem else torch.zeros)(
        (dims[mode], rank), dtype=torch.float32, device=st.device)
    if alloc_log is not None:
        alloc_log.clear()
        alloc_log.update({
            "output_factor": out.numel() * 4,
            "partial_tiles": 0 if work.part_ws is None else work.part_ws.numel() * 4,
            "chunk_plan": int(work.chunk_start.numel() * 8 + work.chunk_ss.numel() * 4
                              + work.chunk_part.numel() * 4),
        })
    a, b = st.active, 1 - st.active
    fptrs = _lib.ptr_array([f.data_ptr() for f in factors.factors])
    flags_p, proc_p = st.stat_ptrs()
    strm = _stream()
    use_cursor = remap == "cursor"
    if use_cursor:
        _ensure_sids(st)
    ref_passes = [(True, True)] if not split_remap else [(True, False), (False, True)]
    if counters is not None:
        for c, r in ref_passes:
            counters.add_mode(st.nnz, nmodes, rank, st.element_nbytes, compute=c, remap=r)
    # the cursor strategy remaps in its own kernel after the compute pass
    passes = [(True, False)] if use_cursor else ref_passes
    val_p = lambda t: t.data_ptr() if t is not None else None
    for do_compute, do_remap in passes:
        if do_compute and work.tile_perm is not None and st.canonical:
            # the planned pass: sorted positions and bin starts come from the tile plan
            _lib.call("fc_mode_worker_planned", st.crd[a].data_ptr(), val_p(st.val[a]),
                      st.crd[b].data_ptr(), val_p(st.val[b]), fptrs, _lib.i64_array(params.dims),
                      out.data_ptr(), nmodes, mode, rank, dims[mode], params.m[mode],
                      work.chunk_start.data_ptr(), work.chunk_ss.data_ptr(),
                      work.chunk_part.data_ptr(),
                      work.chunk_rows.data_ptr() if work.chunk_rows is not None else None,
                      work.tile_rows, work.hist_rows, work.nchunks, work.red1.data_ptr(),
                      work.nred1, work.red2.data_ptr(), work.nred2,
                      work.part_ws.data_ptr() if work.part_ws is not None else None,
                      work.part_ws2.data_ptr() if work.part_ws2 is not None else None,
                      st.slot_maps[mode].data_ptr(), st.nnz, int(do_remap), flags_p, proc_p,
                      work.tile_perm.data_ptr(), work.tile_bins.data_ptr(), strm)
            st._expected += st.nnz
            continue
        _lib.call("fc_mode_worker", st.crd[a].data_ptr(), val_p(st.val[a]), st.crd[b].data_ptr(),
                  val_p(st.val[b]), fptrs, _lib.i64_array(params.dims), out.data_ptr(), nmodes, mode, rank, dims[mode],
                  params.m[mode], work.chunk_start.data_ptr(), work.chunk_ss.data_ptr(),
                  work.chunk_part.data_ptr(),
                  work.chunk_rows.data_ptr() if work.chunk_rows is not None else None,
                  work.tile_rows, work.hist_rows, work.nchunks, work.red1.data_ptr(), work.nred1,
                  work.red2.data_ptr(), work.nred2,
                  work.part_ws.data_ptr() if work.part_ws is not None else None,
                  work.part_ws2.data_ptr() if work.part_ws2 is not None else None,
                  st.slot_maps[mode].data_ptr(), st.nnz, int(do_compute), int(do_remap),
                  int(work.acc_in_smem), flags_p, proc_p, strm)
        st._expected += st.nnz
    if use_cursor:
        base = torch.from_numpy(plan.shard_offsets[next_mode]).to(st.device)
        cursors = torch.zeros(plan.total_shards(next_mode), dtype=torch.int64, device=st.device)
        _lib.call("fc_remap_cursor", st.crd[a].data_ptr(), val_p(st.val[a]), st.crd[b].data_ptr(),
                  val_p(st.val[b]), st._sids[a].data_ptr(), st._sids[b].data_ptr(), nmodes,
                  next_mode, st.nnz, base.data_ptr(), cursors.data_ptr(), flags_p, strm)
        if check:
            check_errors(st, next_mode)
            want = torch.diff(base)
            if not torch.equal(cursors, want):
                bad = int(torch.nonzero(cursors != want)[0, 0])
                raise ShardOverflowError(
                    f"destination shard {bad} of mode {next_mode} ended at fill "
                    f"{int(cursors[bad])}, planned {int(want[bad])}")
    elif check:
        check_errors(st, next_mode)
    st.swap(next_mode, still_canonical=not use_cursor)
    return out


def sweep_all_modes(st: DeviceShardedTensor, factors, smap, workers: int | None = None,
                    remap: str = "slot", counters: TrafficCounters | None = None,
                    mode_seconds: list | None = None, split_remap: bool = False) -> DeviceFactorSet:
    """One pass over every mode, each factor overwritten by its raw MTTKRP
    output right after its mode (engine.py:269-293)."""
    factors = _coerce_factors(factors, st.device)
    working = list(factors.factors)
    lambdas = factors.lambdas.copy()
    events = []
    for n in range(st.num_modes):
        current = DeviceFactorSet(tuple(working), lambdas, st.device, validate=False)
        if mode_seconds is not None:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record()
        # cursor passes verify cursor fills per mode (needs a sync); slot
        # passes defer their device checks to the end of the sweep
        working[n] = mttkrp_mode(st, current, n, smap, workers=workers, remap=remap,
                                 counters=counters, split_remap=split_remap,
                                 check=(remap == "cursor"))
        if mode_seconds is not None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record()
            events.append((e0, e1))
    if remap != "cursor":
        check_errors(st)
    if mode_seconds is not None:
        torch.cuda.current_stream().synchronize()
        mode_seconds.extend(e0.elapsed_time(e1) / 1e3 for e0, e1 in events)
    return DeviceFactorSet(tuple(working), lambdas, st.device, validate=False)

"""CPU oracle for the FLYCOO all-mode spMTTKRP + dynamic-remap sweep.

TEST INFRASTRUCTURE ONLY.  Importable from ``tests/``, ``__graft_entry__.smoke``
and ``bench.py`` (cpu_baseline leg and ``--impl reference``) -- and there only
as the checker or the timed CPU baseline.  The product package
``paper_2309_09131_b200`` never imports this module.

It restates the reference (``/root/reference/pkg/src/modecycle``) in numpy +
the C kernel in ``flycoo_oracle.c``:

* :func:`morton_interleave`   -- morton.py:15-44 (C)
* :func:`canonical_build`     -- layout.py:462-531 (numpy + a C stable
  radix sort for the lexsort orders when the composite key fits 64 bits;
  super-shard / shard geometry, shard ids, slot maps, mode-0 active buffer)
* :func:`device_order`        -- the B200 layout's intra-shard order (this
  repo's design): same shard membership and offsets as the
  reference, elements inside a shard ordered by (previous-mode shard id,
  Morton hi, lo, input position).  Restated here so the GPU build is checked
  bit-exactly.
* :func:`shard_hashes`        -- layout.py:474-497 streamed (C): per-shard
  (hash, count) digests of the canonical shard assignment for tensors whose
  full canonical_build does not fit the host (c3-c5), with :func:`elem_hash`
* :func:`lpt_schedule`        -- schedule.py:57-66 (greedy LPT)
* :class:`OracleTensor`       -- engine.py:163-293 (mttkrp_mode /
  sweep_all_modes over the reference's int64/float64 double buffer, workers
  as pthreads inside the C kernel).
* :func:`reference_mttkrp`    -- coo.py:406-426 (C, sequential).

Parity pinning: ``tests/test_oracle_golden.py`` checks every function above
against the fixtures in ``tests/golden/`` produced by
``tests/golden/make_golden.py`` from the reference itself (bit-exact for
integers and float64 results).
"""

from __future__ import annotations

import ctypes
import heapq
import os
import subprocess
import threading
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "liboracle.so"
_lib = None
_lock = threading.Lock()

_i64p = ctypes.POINTER(ctypes.c_int64)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_f64p = ctypes.POINTER(ctypes.c_double)


def build() -> Path:
    """Compile liboracle.so (gcc, see Makefile)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            src = _HERE / "flycoo_oracle.c"
            if (not _LIB_PATH.exists()) or (src.exists() and
                                             src.stat().st_mtime > _LIB_PATH.stat().st_mtime):
                build()
            L = ctypes.CDLL(str(_LIB_PATH))
            L.orc_morton.restype = ctypes.c_int
            L.orc_morton.argtypes = [_i64p, ctypes.c_int64, ctypes.c_int, _i64p, _u64p, _u64p]
            L.orc_mode_pass.restype = ctypes.c_int64
            L.orc_mode_pass.argtypes = [
                _i64p, _i64p, _f64p, _i64p, _i64p, _f64p, _f64p, _i64p, ctypes.c_int64,
                _f64p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64p, _i64p, _i64p,
                ctypes.c_int, _i64p, _i64p, _i64p, ctypes.c_int, ctypes.c_int,
                ctypes.c_int, _i64p]
            L.orc_stable_sort_u64.restype = ctypes.c_int
            L.orc_stable_sort_u64.argtypes = [_u64p, ctypes.c_int64, ctypes.c_int, _i64p]
            L.orc_shard_hashes.restype = ctypes.c_int
            L.orc_shard_hashes.argtypes = [
                ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                ctypes.c_int, ctypes.c_int, _i64p, _i64p, ctypes.c_int64, ctypes.c_int, _i64p,
                _u64p, _i64p]
            L.orc_reference_mttkrp.restype = None
            L.orc_reference_mttkrp.argtypes = [
                _i64p, _f64p, ctypes.c_int64, ctypes.c_int, ctypes.POINTER(_f64p),
                ctypes.c_int64, ctypes.c_int, _f64p]
            _lib = L
    return _lib


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


# --------------------------------------------------------------------- morton

def morton_interleave(coords: np.ndarray, counts) -> tuple[np.ndarray, np.ndarray]:
    """morton.py:20-44 -> (hi, lo) uint64."""
    coords = np.ascontiguousarray(coords, dtype=np.int64)
    counts = np.ascontiguousarray(np.asarray(counts, dtype=np.int64))
    n, N = coords.shape
    hi = np.zeros(n, dtype=np.uint64)
    lo = np.zeros(n, dtype=np.uint64)
    rc = lib().orc_morton(_p(coords, _i64p), n, N, _p(counts, _i64p), _p(hi, _u64p), _p(lo, _u64p))
    if rc == -1:
        raise ValueError("morton key would need more than 128 bits")
    if rc != 0:
        raise ValueError(f"orc_morton failed ({rc})")
    return hi, lo


# --------------------------------------------------------------------- layout

@dataclass
class CanonicalLayout:
    """Everything build_sharded (layout.py:462-531) derives from (COO, m, k, g)."""
    dims: tuple
    m: tuple
    k: tuple
    g: int
    subs: np.ndarray          # (nnz, N) int64, input order
    vals: np.ndarray          # (nnz,) float64
    iv: np.ndarray            # (nnz, N) interval coordinates
    hi: np.ndarray
    lo: np.ndarray
    orders: list = field(default_factory=list)        # per mode canonical order
    positions: list = field(default_factory=list)     # per mode inverse
    ss_counts: list = field(default_factory=list)
    ss_elem_offsets: list = field(default_factory=list)
    ss_shard_counts: list = field(default_factory=list)
    ss_first_shard: list = field(default_factory=list)
    shard_offsets: list = field(default_factory=list)
    sids_all: np.ndarray | None = None                # (nnz, N) shard id per mode
    slot_maps: list = field(default_factory=list)

    @property
    def nnz(self) -> int:
        return int(self.subs.shape[0])

    @property
    def num_modes(self) -> int:
        return int(self.subs.shape[1])


def stable_order(key: np.ndarray, bits: int) -> np.ndarray:
    """order = np.lexsort((seq, key)) for a uint64 key on bits [0, bits)
    (C radix sort)."""
    key = np.ascontiguousarray(key, dtype=np.uint64)
    order = np.empty(key.shape[0], dtype=np.int64)
    if lib().orc_stable_sort_u64(_p(key, _u64p), key.shape[0], int(bits), _p(order, _i64p)) != 0:
        raise MemoryError("orc_stable_sort_u64")
    return order


def _lex_order(major: list, hi: np.ndarray, lo: np.ndarray, W: int) -> np.ndarray:
    """np.lexsort((seq, lo, hi, *reversed(major))) -- `major` keys most
    significant first, each given as (values, bit width) -- through one
    composite-key radix sort when everything fits 64 bits."""
    total = W + sum(b for _, b in major)
    if total <= 64 and not (W > 64):
        key = lo.astype(np.uint64, copy=True)
        shift = W
        for vals, b in reversed(major):
            key |= np.asarray(vals, dtype=np.uint64) << np.uint64(shift)
            shift += b
        return stable_order(key, total)
    seq = np.arange(lo.shape[0], dtype=np.int64)
    return np.lexsort((seq, lo, hi) + tuple(v for v, _ in reversed(major)))


def canonical_build(subs, vals, dims, m, k, g) -> CanonicalLayout:
    """layout.py:474-519 restated: iv = c // m; Morton (hi, lo) over all
    modes' interval coordinates; per mode lexsort by (iv_n, hi, lo, seq);
    super-shard fills, g-shards, shard ids, shard offsets, slot maps."""
    subs = np.ascontiguousarray(subs, dtype=np.int64)
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    nnz, N = subs.shape
    m = tuple(int(x) for x in m)
    k = tuple(int(x) for x in k)
    g = int(g)
    iv = np.empty_like(subs)
    for n in range(N):
        iv[:, n] = subs[:, n] // m[n]
    hi, lo = morton_interleave(iv, k)
    seq = np.arange(nnz, dtype=np.int64)
    L = CanonicalLayout(tuple(int(d) for d in dims), m, k, g, subs, vals, iv, hi, lo)
    L.sids_all = np.empty((nnz, N), dtype=np.int64)
    W = sum(int(x - 1).bit_length() for x in k)
    for n in range(N):
        order = _lex_order([(iv[:, n], int(k[n] - 1).bit_length())], hi, lo, W)
        pos = np.empty(nnz, dtype=np.int64)
        pos[order] = seq
        counts = np.bincount(iv[:, n], minlength=k[n]).astype(np.int64)
        offs = np.concatenate(([0], np.cumsum(counts))).astype(np.int64)
        shards = -(-counts // g)
        first = np.concatenate(([0], np.cumsum(shards))).astype(np.int64)
        L.sids_all[:, n] = first[iv[:, n]] + (pos - offs[iv[:, n]]) // g
        total = int(first[-1])
        ss_of = np.repeat(np.arange(k[n], dtype=np.int64), shards)
        q = np.arange(total, dtype=np.int64) - first[ss_of]
        soffs = np.concatenate((offs[ss_of] + q * g, [nnz])).astype(np.int64)
        L.orders.append(order)
        L.positions.append(pos)
        L.ss_counts.append(counts)
        L.ss_elem_offsets.append(offs)
        L.ss_shard_counts.append(shards)
        L.ss_first_shard.append(first)
        L.shard_offsets.append(soffs)
    L.slot_maps = [np.ascontiguousarray(L.positions[(n + 1) % N][L.orders[n]])
                   for n in range(N)]
    return L


@dataclass
class DeviceOrder:
    """Per mode: element order, inverse positions and slot maps of the B200
    layout (same shards as the reference, different order inside them)."""
    orders: list
    positions: list
    slot_maps: list


def device_order(L: CanonicalLayout) -> DeviceOrder:
    nnz, N = L.nnz, L.num_modes
    seq = np.arange(nnz, dtype=np.int64)
    orders, positions = [], []
    W = sum(int(x - 1).bit_length() for x in L.k)
    nsh = [int(L.ss_first_shard[n][-1]) for n in range(N)]
    for n in range(N):
        prev = (n - 1) % N
        order = _lex_order([(L.sids_all[:, n], max(nsh[n] - 1, 0).bit_length()),
                            (L.sids_all[:, prev], max(nsh[prev] - 1, 0).bit_length())],
                           L.hi, L.lo, W)
        pos = np.empty(nnz, dtype=np.int64)
        pos[order] = seq
        orders.append(order)
        positions.append(pos)
    slots = [np.ascontiguousarray(positions[(n + 1) % N][orders[n]]) for n in range(N)]
    return DeviceOrder(orders, positions, slots)


def shard_multiset_keys(coords: np.ndarray, vals_bits: np.ndarray, shard_offsets: np.ndarray):
    """Canonical per-shard multiset form: inside each shard, rows sorted by
    (coords..., value bits).  Two buffers hold identical per-shard multisets
    iff these arrays are equal."""
    nnz, N = coords.shape
    sid = np.repeat(np.arange(len(shard_offsets) - 1), np.diff(shard_offsets))
    keys = [vals_bits] + [coords[:, w] for w in range(N - 1, -1, -1)] + [sid]
    o = np.lexsort(keys)
    return coords[o], vals_bits[o]


# ------------------------------------------------------------- shard digests

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix64(x: np.ndarray) -> np.ndarray:
    x = x ^ (x >> np.uint64(30))
    x = x * _M1
    x = x ^ (x >> np.uint64(27))
    x = x * _M2
    return x ^ (x >> np.uint64(31))


def elem_hash(coords: np.ndarray, vbits: np.ndarray) -> np.ndarray:
    """Per-element digest of (int32 coordinates, fp32 value bits), the same
    function as orc_elem_hash (flycoo_oracle.c)."""
    coords = np.asarray(coords)
    h = np.full(coords.shape[0], 0x9E3779B97F4A7C15, dtype=np.uint64)
    with np.errstate(over="ignore"):
        for w in range(coords.shape[1]):
            h = _mix64(h ^ coords[:, w].astype(np.uint32).astype(np.uint64))
        v = np.asarray(vbits).astype(np.uint32).astype(np.uint64)
        return _mix64(h ^ ((v << np.uint64(32)) | np.uint64(0x5BD1E995)))


def shard_digests_from_ids(coords, vbits, shard_ids, nshards: int):
    """(hash, count) per shard from explicit shard ids (wrapping sums)."""
    h = elem_hash(coords, vbits)
    out = np.zeros(nshards, dtype=np.uint64)
    with np.errstate(over="ignore"):
        np.add.at(out, np.asarray(shard_ids, dtype=np.int64), h)
    cnt = np.bincount(np.asarray(shard_ids, dtype=np.int64), minlength=nshards).astype(np.int64)
    return out, cnt


def shard_hashes(records: np.ndarray, nmodes: int, mode: int, m, k, g: int,
                 vbits: np.ndarray | None = None, threads: int | None = None):
    """Streaming restatement of the reference's canonical shard assignment
    (layout.py:474-497) for `mode`, reduced to per-shard (hash, count)
    digests -- for tensors whose canonical_build does not fit the host
    (c3-c5).  `records` is (nnz, cs) int32 in input order: coordinates in
    columns 0..N-1, and the fp32 value bits in column `cs-1` unless `vbits`
    is given.  Returns (ss_counts, hash uint64 per shard, count per shard)."""
    records = np.ascontiguousarray(records, dtype=np.int32)
    nnz, cs = records.shape
    if vbits is None:
        vptr, vs = records[:, cs - 1:].ctypes.data, cs
        keep = records
    else:
        keep = np.ascontiguousarray(vbits).view(np.uint32)
        vptr, vs = keep.ctypes.data, 1
    m = np.ascontiguousarray(np.asarray(m, dtype=np.int64))
    k = np.ascontiguousarray(np.asarray(k, dtype=np.int64))
    K = int(k[mode])
    ss_counts = np.zeros(K, dtype=np.int64)
    # shard count is only known after the counts: size for the worst case
    nsh_max = K + nnz // int(g) + 1
    hsh = np.zeros(nsh_max, dtype=np.uint64)
    cnt = np.zeros(nsh_max, dtype=np.int64)
    rc = lib().orc_shard_hashes(records.ctypes.data, cs, vptr, vs, nnz, int(nmodes), int(mode),
                                _p(m, _i64p), _p(k, _i64p), int(g),
                                int(threads or os.cpu_count() or 1), _p(ss_counts, _i64p),
                                _p(hsh, _u64p), _p(cnt, _i64p))
    del keep
    if rc != 0:
        raise RuntimeError(f"orc_shard_hashes failed ({rc})")
    nsh = int((-(-ss_counts // int(g))).sum())
    return ss_counts, hsh[:nsh], cnt[:nsh]


# ------------------------------------------------------------------ schedule

def lpt_schedule(counts, nu: int) -> list[list[int]]:
    """schedule.py:57-66: largest-first (ties: lower id) to the lightest
    thread (ties: lower thread id)."""
    order = sorted(range(len(counts)), key=lambda j: (-int(counts[j]), j))
    heap = [(0, t) for t in range(nu)]
    heapq.heapify(heap)
    out = [[] for _ in range(nu)]
    for j in order:
        load, t = heapq.heappop(heap)
        out[t].append(j)
        heapq.heappush(heap, (load + int(counts[j]), t))
    return out


# ------------------------------------------------------------------- engine

def reference_mttkrp(subs, vals, factors, mode: int) -> np.ndarray:
    """coo.py:406-426 (sequential, nonzero storage order)."""
    subs = np.ascontiguousarray(subs, dtype=np.int64)
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    fs = [np.ascontiguousarray(f, dtype=np.float64) for f in factors]
    nnz, N = subs.shape
    R = fs[0].shape[1]
    out = np.zeros((fs[mode].shape[0], R))
    arr = (_f64p * N)(*[_p(f, _f64p) for f in fs])
    lib().orc_reference_mttkrp(_p(subs, _i64p), _p(vals, _f64p), nnz, N, arr, R, mode,
                               _p(out, _f64p))
    return out


class OracleTensor:
    """The reference's ShardedTensor double buffer (layout.py:384-459) plus
    its engine (engine.py:163-293), driven through the C mode worker.

    ``order`` selects the element order: "reference" (layout.py canonical)
    or "device" (the B200 layout's order; same shards)."""

    def __init__(self, L: CanonicalLayout, order: str = "reference", nu: int = 1):
        self.L = L
        N, nnz = L.num_modes, L.nnz
        if order == "reference":
            self.orders, self.slot_maps = L.orders, L.slot_maps
        elif order == "device":
            d = device_order(L)
            self.orders, self.slot_maps = d.orders, d.slot_maps
        else:
            raise ValueError(order)
        o0 = self.orders[0]
        self.sids = [np.ascontiguousarray(L.sids_all[o0]), np.zeros((nnz, N), np.int64)]
        self.idxs = [np.ascontiguousarray(L.subs[o0]), np.zeros((nnz, N), np.int64)]
        self.vals = [np.ascontiguousarray(L.vals[o0]), np.zeros(nnz)]
        self.active = 0
        self.active_mode = 0
        self.set_workers(nu)

    def set_workers(self, nu: int):
        """Static LPT schedule per mode (schedule.py:69-86) turned into
        per-worker element ranges (engine.py:138-150)."""
        L = self.L
        self.nu = int(nu)
        self.ranges = []
        for n in range(L.num_modes):
            assign = lpt_schedule(L.ss_shard_counts[n], self.nu)
            offs, counts = L.ss_elem_offsets[n], L.ss_counts[n]
            starts, ends, roffs = [], [], [0]
            for lst in assign:
                ss = np.asarray(lst, dtype=np.int64)
                starts.append(offs[ss])
                ends.append(offs[ss] + counts[ss])
                roffs.append(roffs[-1] + len(lst))
            self.ranges.append((np.ascontiguousarray(np.concatenate(starts).astype(np.int64)),
                                np.ascontiguousarray(np.concatenate(ends).astype(np.int64)),
                                np.asarray(roffs, dtype=np.int64)))

    def active_arrays(self):
        a = self.active
        return self.sids[a], self.idxs[a], self.vals[a]

    def mttkrp_mode(self, factors, mode: int, do_remap: bool = True) -> np.ndarray:
        L = self.L
        N = L.num_modes
        if self.active_mode != mode:
            raise ValueError(f"active buffer is ordered for mode {self.active_mode}, not {mode}")
        nxt = (mode + 1) % N
        fs = [np.ascontiguousarray(f, dtype=np.float64) for f in factors]
        R = fs[0].shape[1]
        foffs = np.cumsum([0] + [f.shape[0] for f in fs[:-1]]).astype(np.int64)
        fstack = np.ascontiguousarray(np.concatenate(fs, axis=0))
        out = np.zeros((L.dims[mode], R))
        a, b = self.active, 1 - self.active
        starts, ends, roffs = self.ranges[mode]
        err = np.zeros(1, dtype=np.int64)
        dest_base = L.shard_offsets[nxt]
        slots = self.slot_maps[mode]
        dummy = np.zeros(1, dtype=np.int64)
        got = lib().orc_mode_pass(
            _p(self.sids[a], _i64p), _p(self.idxs[a], _i64p), _p(self.vals[a], _f64p),
            _p(self.sids[b], _i64p), _p(self.idxs[b], _i64p), _p(self.vals[b], _f64p),
            _p(fstack, _f64p), _p(foffs, _i64p), R, _p(out, _f64p), N, mode, nxt,
            _p(starts, _i64p), _p(ends, _i64p), _p(roffs, _i64p), self.nu,
            _p(dest_base, _i64p), _p(dummy, _i64p), _p(slots, _i64p), 0, 1,
            1 if do_remap else 0, _p(err, _i64p))
        if got != L.nnz:
            raise RuntimeError(f"workers processed {got} of {L.nnz} elements")
        if do_remap:
            self.active = b
            self.active_mode = nxt
        return out

    def sweep_all_modes(self, factors) -> list[np.ndarray]:
        """engine.py:269-293: factor n replaced by its raw output after mode n."""
        working = list(factors)
        for n in range(self.L.num_modes):
            working[n] = self.mttkrp_mode(working, n)
        return working

"""Seeded synthetic inputs for the benchmark configurations.

* :func:`synth_tensor` restates the reference generator
  (/root/reference/pkg/src/modecycle/coo.py:323-399) bit-exactly -- numpy
  Philox, power law ``floor(d * u**(1 + skew))``, first ``nnz`` distinct
  coordinates in draw order -- and is what config 1 (uniform, skew 0) uses.
* :func:`zipf_tensor` is the bounded-Zipf generator of configs 2-5 (the
  reference has no Zipf law): draw j of mode w is ``u = Philox4x32-10(seed,
  j, w)``, index = inverse CDF of P(i) ~ (i+1)^-s on [0, I) (or uniform);
  duplicates are dropped keeping the first occurrence in draw order, the
  first ``nnz`` distinct coordinates are kept, values are fp32 U(0, 1].
  It runs on the GPU (libflycoo K6 entry points + CUB radix sort).

These are measurement inputs, not the product path.
"""

from __future__ import annotations

import math
from typing import Sequence

import os

import numpy as np
import torch

from . import _lib

__all__ = ["synth_tensor", "zipf_tensor", "CONFIGS", "config_tensor"]


# ---------------------------------------------------------------- uniform

def _probabilities(d: int, skew: float) -> np.ndarray:
    edges = (np.arange(d + 1) / d) ** (1.0 / (1.0 + skew))
    return np.diff(edges)


def synth_tensor(dims: Sequence[int], nnz: int, seed: int, skew: float = 0.0):
    """(subs int64 (nnz, N), vals float64 (nnz,)) exactly as coo.synth_tensor."""
    dims = tuple(int(d) for d in dims)
    if any(d < 1 for d in dims):
        raise ValueError("dims must be positive")
    if skew < 0:
        raise ValueError("skew must be >= 0")
    space = math.prod(dims)
    if nnz < 1:
        raise ValueError("nnz must be positive")
    if nnz > space:
        raise ValueError(f"nnz={nnz} exceeds index space of size {space}")
    rng = np.random.Generator(np.random.Philox(int(seed)))
    if space <= (1 << 20) and nnz * 4 >= space:
        # weighted sampling without replacement over all cells (keys u^(1/w))
        cells = np.stack(np.unravel_index(np.arange(space), dims), axis=1).astype(np.int64)
        logw = np.zeros(space)
        for n, d in enumerate(dims):
            logw += np.log(_probabilities(d, skew))[cells[:, n]]
        w = np.exp(logw - logw.max())
        keys = rng.random(space) ** (1.0 / w)
        top = np.argpartition(keys, space - nnz)[space - nnz:]
        subs = cells[np.sort(top)]
    else:
        batches, distinct, total = [], 0, 0
        while True:
            batch = max(256, int(1.3 * (nnz - distinct)))
            u = rng.random((batch, len(dims)))
            rows = np.empty((batch, len(dims)), dtype=np.int64)
            for n, d in enumerate(dims):
                rows[:, n] = np.minimum((d * u[:, n] ** (1.0 + skew)).astype(np.int64), d - 1)
            batches.append(rows)
            total += batch
            allrows = np.concatenate(batches)
            uniq, first = np.unique(allrows, axis=0, return_index=True)
            distinct = uniq.shape[0]
            if distinct >= nnz:
                subs = allrows[np.sort(first)[:nnz]]
                break
            if total > 200 * nnz + 100_000:
                raise RuntimeError("rejection sampling is not converging")
    vals = 1.0 - rng.random(nnz)
    return subs, vals


# ------------------------------------------------------------------- Zipf

def zipf_cdf(d: int, s: float) -> np.ndarray:
    """CDF of the bounded Zipf law P(i) ~ (i+1)^-s, i in [0, d)."""
    p = np.arange(1, d + 1, dtype=np.float64) ** (-float(s))
    c = np.cumsum(p)
    c /= c[-1]
    c[-1] = 1.0
    return c


def zipf_tensor(dims: Sequence[int], nnz: int, seed: int, exponents: Sequence, device="cuda",
                draw_factor: float = 1.25):
    """GPU bounded-Zipf COO tensor: (coords int32 (nnz, N), vals fp32 (nnz,))
    on `device`, in draw order.  ``exponents[w] = None`` means uniform."""
    dims = tuple(int(d) for d in dims)
    N = len(dims)
    dev = torch.device(device)
    strm = torch.cuda.current_stream(dev).cuda_stream
    L = _lib.load()
    cdfs = [None if s is None else torch.from_numpy(zipf_cdf(d, s)).to(dev)
            for d, s in zip(dims, exponents)]
    cdf_ptrs = _lib.ptr_array([c.data_ptr() if c is not None else 0 for c in cdfs])
    cdf_len = _lib.i64_array([c.numel() if c is not None else 0 for c in cdfs])
    dims_arr = _lib.i64_array(dims)
    bits = (math.prod(dims) - 1).bit_length()  # mixed-radix key width
    ndraws = int(nnz * draw_factor) + 1024
    while True:
        if ndraws >= 1 << 32:
            raise RuntimeError("too many draws for uint32 draw ids")
        coords = torch.empty((ndraws, N), dtype=torch.int32, device=dev)
        _lib.call("fc_synth_draw", int(seed), ndraws, N, dims_arr, cdf_ptrs, cdf_len,
                  coords.data_ptr(), strm)
        hi = torch.empty(ndraws, dtype=torch.int64, device=dev)
        lo = torch.empty(ndraws, dtype=torch.int64, device=dev)
        _lib.call("fc_synth_keys", coords.data_ptr(), ndraws, N, dims_arr, hi.data_ptr(),
                  lo.data_ptr(), strm)
        if bits <= 64:
            del hi
            hi = None
        temp_bytes = int(L.fc_build_sort_temp_bytes(ndraws))
        temp = torch.empty(max(temp_bytes, 1), dtype=torch.uint8, device=dev)
        ids = torch.arange(ndraws, dtype=torch.int32, device=dev)
        ks = torch.empty_like(lo)
        ids2 = torch.empty_like(ids)
        _lib.call("fc_build_sort_pairs", lo.data_ptr(), ks.data_ptr(), ids.data_ptr(),
                  ids2.data_ptr(), ndraws, max(1, min(bits, 64)), temp.data_ptr(), temp_bytes, strm)
        ids, ids2 = ids2, ids
        if bits > 64:
            kh = torch.empty_like(hi)
            _lib.call("fc_build_gather_key", ids.data_ptr(), ndraws, 1, hi.data_ptr(), lo.data_ptr(),
                      None, N, 0, 1, 0, kh.data_ptr(), strm)
            _lib.call("fc_build_sort_pairs", kh.data_ptr(), ks.data_ptr(), ids.data_ptr(),
                      ids2.data_ptr(), ndraws, bits - 64, temp.data_ptr(), temp_bytes, strm)
            ids = ids2
            del kh
            hs = torch.empty_like(hi)
            _lib.call("fc_build_gather_key", ids.data_ptr(), ndraws, 1, hi.data_ptr(), lo.data_ptr(),
                      None, N, 0, 1, 0, hs.data_ptr(), strm)
            _lib.call("fc_build_gather_key", ids.data_ptr(), ndraws, 0, hi.data_ptr(), lo.data_ptr(),
                      None, N, 0, 1, 0, ks.data_ptr(), strm)
        else:
            hs = ks  # the sorted low words are the whole key
        del temp, lo
        keep = torch.zeros(ndraws, dtype=torch.uint8, device=dev)
        _lib.call("fc_synth_mark_first", hs.data_ptr(), ks.data_ptr(), ids.data_ptr(), ndraws,
                  keep.data_ptr(), strm)
        del hs, ks, ids, ids2, hi
        kept = torch.nonzero(keep).squeeze(1)
        del keep
        if kept.numel() >= nnz:
            sel = kept[:nnz]
            del kept
            coords = coords.index_select(0, sel).contiguous()
            break
        # deterministic restart with more draws: draw j never depends on ndraws
        ratio = nnz / max(kept.numel(), 1)
        del kept, coords
        ndraws = int(ndraws * max(1.2, min(4.0, ratio * 1.1))) + 1024
    vals = torch.empty(nnz, dtype=torch.float32, device=dev)
    _lib.call("fc_synth_uniform", int(seed), 77, nnz, vals.data_ptr(), 1, strm)
    return coords, vals


def zipf_records_bucketed(dims: Sequence[int], nnz: int, seed: int, exponents: Sequence,
                          device="cuda", draw_factor: float = 1.25, bucket_draws: int = 1 << 28,
                          scan: int = 1 << 28):
    """The nonzeros of :func:`zipf_tensor` (same draws, same first-occurrence
    dedup, same "first nnz distinct in draw order" cut), for tensors whose
    single dedup sort does not fit HBM (config 5: 3.6B nonzeros from ~4.5B
    draws).  Draws are split into buckets by ranges of the mode-0 coordinate
    (duplicates share it, so each bucket dedups alone, a few GB at a time);
    the cut is the draw index T with exactly nnz first occurrences below it.

    Returns 16-byte records (nnz, 4) int32 ``{c0, c1, c2, bits(v)}`` on
    `device` (the 3-mode record layout), ordered by bucket and by draw index
    inside a bucket -- the same SET of nonzeros as zipf_tensor, not the same
    input order; values are drawn per output position as in zipf_tensor."""
    dims = tuple(int(d) for d in dims)
    N = len(dims)
    if N != 3:
        raise ValueError("the bucketed generator writes 3-mode records")
    if math.prod(dims) >= 1 << 63:
        raise ValueError("coordinate space must fit a 63-bit key")
    dev = torch.device(device)
    strm = torch.cuda.current_stream(dev).cuda_stream
    cdfs = [None if s is None else torch.from_numpy(zipf_cdf(d, s)).to(dev)
            for d, s in zip(dims, exponents)]
    cdf_ptrs = _lib.ptr_array([c.data_ptr() if c is not None else 0 for c in cdfs])
    cdf_len = _lib.i64_array([c.numel() if c is not None else 0 for c in cdfs])
    dims_arr = _lib.i64_array(dims)
    if exponents[0] is None:
        p0 = np.full(dims[0], 1.0 / dims[0])
    else:
        p0 = np.diff(np.concatenate(([0.0], zipf_cdf(dims[0], exponents[0]))))

    def draw_at(js, lo, hi, out, cstride):
        _lib.call("fc_synth_draw_at", int(seed), js.data_ptr(), js.numel(), N, dims_arr, cdf_ptrs,
                  cdf_len, lo, hi, out.data_ptr(), cstride, strm)

    ndraws = int(nnz * draw_factor) + 1024
    while True:
        # mode-0 value ranges of <= bucket_draws expected draws (one hot value
        # may exceed it alone)
        groups, v = [], 0
        while v < dims[0]:
            w, acc = v, 0.0
            while w < dims[0] and (w == v or acc + p0[w] * ndraws <= bucket_draws):
                acc += p0[w] * ndraws
                w += 1
            groups.append((v, w))
            v = w
        firsts = []
        for v0, v1 in groups:
            sel = []
            for j0 in range(0, ndraws, scan):
                js = torch.arange(j0, min(j0 + scan, ndraws), dtype=torch.int64, device=dev)
                c0 = torch.empty(js.numel(), dtype=torch.int32, device=dev)
                draw_at(js, 0, 1, c0, 1)
                sel.append(js[(c0 >= v0) & (c0 < v1)])
                del js, c0
            jb = torch.cat(sel)
            del sel
            c = torch.empty((jb.numel(), N), dtype=torch.int32, device=dev)
            draw_at(jb, 0, N, c, N)
            c = c.to(torch.int64)
            key = (c[:, 0] * dims[1] + c[:, 1]) * dims[2] + c[:, 2]
            del c
            skey, perm = torch.sort(key, stable=True)  # draw order kept inside equal keys
            del key
            first = torch.ones(skey.numel(), dtype=torch.bool, device=dev)
            first[1:] = skey[1:] != skey[:-1]
            del skey
            firsts.append(torch.sort(jb[perm[first]]).values)
            del perm, first, jb
        total = sum(int(f.numel()) for f in firsts)
        if total >= nnz:
            break
        del firsts
        ratio = nnz / max(total, 1)
        ndraws = int(ndraws * max(1.2, min(4.0, ratio * 1.1))) + 1024
    # the cut: smallest T with exactly nnz first occurrences below it
    lo, hi = 0, ndraws
    while lo < hi:
        mid = (lo + hi) // 2
        t = torch.tensor([mid], dtype=torch.int64, device=dev)
        cnt = sum(int(torch.searchsorted(f, t)) for f in firsts)
        if cnt >= nnz:
            hi = mid
        else:
            lo = mid + 1
    cut = torch.tensor([lo], dtype=torch.int64, device=dev)
    rec = torch.empty((nnz, 4), dtype=torch.int32, device=dev)
    off = 0
    for i in range(len(firsts)):
        f = firsts[i]
        f = f[: int(torch.searchsorted(f, cut))]
        if f.numel():
            draw_at(f, 0, N, rec[off:], 4)
        off += f.numel()
        firsts[i] = None
        del f
    assert off == nnz, (off, nnz)
    vals = torch.empty(nnz, dtype=torch.float32, device=dev)
    _lib.call("fc_synth_uniform", int(seed), 77, nnz, vals.data_ptr(), 1, strm)
    rec[:, 3] = vals.view(torch.int32)
    del vals
    return rec


# ---------------------------------------------------- host twin (numpy)

_M0, _M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
_W0, _W1 = np.uint64(0x9E3779B9), np.uint64(0xBB67AE85)
_MASK = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, seed: int):
    """Vectorised Philox4x32-10, the same bits as csrc/common.cuh."""
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint64) & _MASK for x in (c0, c1, c2, c3))
    k0 = np.uint64(seed & 0xFFFFFFFF)
    k1 = np.uint64((seed >> 32) & 0xFFFFFFFF)
    for _ in range(10):
        p0 = _M0 * c0
        p1 = _M1 * c2
        c0, c1, c2, c3 = ((p1 >> np.uint64(32)) ^ c1 ^ k0, p1 & _MASK,
                          (p0 >> np.uint64(32)) ^ c3 ^ k1, p0 & _MASK)
        k0 = (k0 + _W0) & _MASK
        k1 = (k1 + _W1) & _MASK
    return c0, c1, c2, c3


def _parallel_chunks(n: int, fn, chunk: int = 1 << 22) -> None:
    """fn(lo, hi) over [0, n) in chunks on the host's cores (numpy releases
    the GIL inside its ufuncs)."""
    spans = [(lo, min(n, lo + chunk)) for lo in range(0, n, chunk)]
    if len(spans) <= 1:
        for lo, hi in spans:
            fn(lo, hi)
        return
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(spans), os.cpu_count() or 1)) as ex:
        list(ex.map(lambda sp: fn(*sp), spans))


def _first_occurrences(rows: np.ndarray, dims) -> np.ndarray:
    """Index of the first occurrence of every distinct row (any order): a
    stable sort of the row-major flattened key when prod(dims) fits 63 bits,
    else a stable lexsort of the columns -- np.unique(rows, axis=0) sorts a
    void view and took minutes at c2's 96M draws."""
    from .coo import coords_key
    key = coords_key(rows, dims)
    if key is not None:
        o = np.argsort(key, kind="stable")
        k = key[o]
    else:
        o = np.lexsort(rows.T[::-1])
        k = rows[o]
    new = np.ones(len(o), dtype=bool)
    if len(o) > 1:
        new[1:] = (k[1:] != k[:-1]) if k.ndim == 1 else np.any(k[1:] != k[:-1], axis=1)
    return o[new]


def zipf_tensor_host(dims: Sequence[int], nnz: int, seed: int, exponents: Sequence,
                     draw_factor: float = 1.25):
    """numpy twin of :func:`zipf_tensor` (identical output; for CPU-side
    samples such as the CPU baseline).  Returns (subs int64, vals float32)."""
    dims = tuple(int(d) for d in dims)
    N = len(dims)
    cdfs = [None if s is None else zipf_cdf(d, s) for d, s in zip(dims, exponents)]

    def draw(rows, lo, hi):
        j = np.arange(lo, hi, dtype=np.uint64)
        for w in range(N):
            x, y, _, _ = philox4x32_10(j, j >> np.uint64(32), np.uint64(w), np.uint64(0x5EED), seed)
            u = ((x >> np.uint64(5)) * np.uint64(67108864) + (y >> np.uint64(6))).astype(np.float64)
            u *= 1.0 / 9007199254740992.0
            if cdfs[w] is None:
                rows[lo:hi, w] = np.minimum((u * dims[w]).astype(np.int64), dims[w] - 1)
            else:
                rows[lo:hi, w] = np.searchsorted(cdfs[w], u, side="right")

    ndraws = int(nnz * draw_factor) + 1024
    rows = np.empty((0, N), dtype=np.int64)
    while True:
        done = rows.shape[0]  # draws are indexed by j: a retry only adds the new ones
        rows = np.concatenate([rows, np.empty((ndraws - done, N), dtype=np.int64)])
        _parallel_chunks(ndraws - done, lambda lo, hi: draw(rows, done + lo, done + hi))
        first = _first_occurrences(rows, dims)
        if first.size >= nnz:
            subs = rows[np.sort(first)[:nnz]]
            break
        ratio = nnz / max(first.size, 1)
        ndraws = int(ndraws * max(1.2, min(4.0, ratio * 1.1))) + 1024
    vals = np.empty(nnz, dtype=np.float32)

    def draw_vals(lo, hi):
        i = np.arange(lo, hi, dtype=np.uint64)
        x, _, _, _ = philox4x32_10(i, i >> np.uint64(32), np.uint64(77), np.uint64(0xF00D), seed)
        vals[lo:hi] = ((x >> np.uint64(8)).astype(np.float64) + 1.0) * (1.0 / 16777216.0)

    _parallel_chunks(nnz, draw_vals)
    return subs, vals


# ---------------------------------------------------------------- configs

# BASELINE.json configs (index 1..5); seeds per SURVEY §8d: tensor seed =
# config index, factor seed = 1000 + index.
CONFIGS = {
    1: dict(dims=(1000, 800, 600), nnz=1_000_000, law=None, rank=16, semantics="fixed"),
    2: dict(dims=(12092, 9184, 28818), nnz=76_900_000, law=(1.1, 1.1, 1.1), rank=32,
            semantics="updated"),
    3: dict(dims=(532924, 17262471, 2480308, 1443), nnz=140_000_000, law=(1.2, 1.2, 1.2, 1.2),
            rank=32, semantics="fixed"),
    4: dict(dims=(4821207, 1774269, 1805187), nnz=1_740_000_000, law=(1.1, 1.1, 1.1), rank=32,
            semantics="updated"),
    5: dict(dims=(46, 239172, 239172), nnz=3_600_000_000, law=(None, 1.0, 1.0), rank=32,
            semantics="updated"),
}


def config_tensor(index: int, device="cuda", nnz: int | None = None):
    """Device COO (coords int32, vals fp32) of BASELINE config `index`;
    `nnz` overrides the size (same law, first nnz distinct draws)."""
    cfg = CONFIGS[index]
    n = cfg["nnz"] if nnz is None else int(nnz)
    if cfg["law"] is None:
        subs, vals = synth_tensor(cfg["dims"], n, seed=index, skew=0.0)
        return (torch.from_numpy(subs.astype(np.int32)).to(device),
                torch.from_numpy(vals.astype(np.float32)).to(device))
    return zipf_tensor(cfg["dims"], n, seed=index, exponents=cfg["law"], device=device)

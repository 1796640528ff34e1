"""Partition parameters of the FLYCOO layout (host-side planning).

Restates the reference's parameter model and search so that a plan chosen
here is the plan the reference would choose
(/root/reference/pkg/src/modecycle/layout.py:56-337):

* :class:`PartitionParams` -- layout.py:56-128 (same fields, same checks);
* :func:`select_params`    -- layout.py:247-318 (Eq. 2 divisibility + Eq. 3
  cache bound; widest interval per mode, then the largest power-of-two g);
* :func:`device_params`    -- new: the B200 choice, intervals sized so one
  super-shard's rank-R accumulator tile sits in shared memory.

Pinned against the reference's own outputs by tests/test_params.py
(tests/golden/select_params.json).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

__all__ = ["InfeasibleParamsError", "PartitionParams", "select_params", "device_params",
           "default_element_bytes", "element_size_bits"]


class InfeasibleParamsError(ValueError):
    """No (m, g) pair satisfies the divisibility and cache constraints."""


def _cdiv(a: int, b: int) -> int:
    return -(-a // b)


def _clog2(x: int) -> int:
    if x < 1:
        raise ValueError("log2 of non-positive value")
    return (x - 1).bit_length()


@dataclass(frozen=True)
class PartitionParams:
    """Interval width ``m[n]`` (output rows per super-shard), super-shard count
    ``k[n]`` (m*k >= dims[n]), shard size ``g``; ``alpha/beta/sigma`` are the
    modelled byte sizes of a factor entry, a tensor element and a cursor;
    ``theta`` the cache fraction of ``gamma`` bytes (layout.py:56-95)."""

    dims: tuple
    nnz: int
    m: tuple
    k: tuple
    g: int
    nu: int
    gamma: int
    theta: float
    rank: int
    alpha: int
    beta: int
    sigma: int
    eq2_exact: tuple = ()

    def __post_init__(self):
        if not self.eq2_exact:
            object.__setattr__(self, "eq2_exact", tuple(
                _cdiv(d, mm) == kk for d, mm, kk in zip(self.dims, self.m, self.k)))
        for n, (d, mm, kk) in enumerate(zip(self.dims, self.m, self.k)):
            if mm < 1 or kk < 1:
                raise ValueError(f"mode {n}: m and k must be positive")
            if mm * kk < d:
                raise ValueError(f"mode {n}: intervals cover only {mm * kk} of {d} indices")
        if not 0.0 < self.theta < 1.0:
            raise ValueError("theta must lie in (0, 1)")

    @property
    def num_modes(self) -> int:
        return len(self.dims)

    @property
    def cache_budget(self) -> float:
        return self.theta * self.gamma

    def divisibility_ok(self, mode: int) -> bool:
        if self.dims[mode] < self.nu:
            return self.m[mode] == 1
        return self.k[mode] % self.nu == 0

    def worst_case_shards(self, mode: int, g: int | None = None) -> int:
        return _cdiv(self.nnz, self.g if g is None else g) + self.k[mode]

    def cache_lhs(self, mode: int, g: int | None = None, shard_sum: int | None = None) -> int:
        g = self.g if g is None else g
        if shard_sum is None:
            shard_sum = self.worst_case_shards(mode, g)
        return (self.alpha * self.m[mode] * self.rank + self.beta * g) * self.nu + self.sigma * shard_sum

    def cache_slack(self, mode: int, shard_sum: int | None = None) -> float:
        return self.cache_budget - self.cache_lhs(mode, shard_sum=shard_sum)

    def cache_ok(self, mode: int, shard_sum: int | None = None) -> bool:
        return self.cache_lhs(mode, shard_sum=shard_sum) <= self.cache_budget


def default_element_bytes(num_modes: int) -> int:
    """Reference in-memory element: shard id + index per mode (int64) and a
    float64 value (layout.py:131-134)."""
    return (2 * num_modes + 1) * 8


def element_size_bits(params: PartitionParams) -> int:
    """Packed element size in bits (layout.py:137-145)."""
    shard_bits = _clog2(_cdiv(params.nnz, params.g))
    return params.num_modes * shard_bits + sum(_clog2(d) for d in params.dims) + 64


# ------------------------------------------------------------------ search

class _Model:
    """Eq. 3 left-hand side for one tensor shape (layout.py:207-211)."""

    def __init__(self, nnz, nu, budget, rank, alpha, beta, sigma):
        self.nnz, self.nu, self.budget = nnz, nu, budget
        self.rank, self.alpha, self.beta, self.sigma = rank, alpha, beta, sigma

    def lhs(self, m: int, k: int, g: int) -> int:
        return ((self.alpha * m * self.rank + self.beta * g) * self.nu
                + self.sigma * (_cdiv(self.nnz, g) + k))

    def fits(self, m: int, k: int, gs) -> bool:
        return any(self.lhs(m, k, g) <= self.budget for g in gs)


def _pow2_between(lo: int, hi: int) -> list[int]:
    if lo < 1 or hi < lo:
        raise ValueError(f"bad shard size range {(lo, hi)}")
    gs = [1 << b for b in range(lo.bit_length() - 1, hi.bit_length() + 1) if lo <= (1 << b) <= hi]
    if not gs:
        raise ValueError(f"no power of two inside shard size range {(lo, hi)}")
    return gs


def _band(dim: int, k: int):
    """Inclusive m range with ceil(dim / m) == k (layout.py:163-173)."""
    if k > dim:
        return None
    if k == 1:
        return dim, dim
    lo, hi = _cdiv(dim, k), _cdiv(dim, k - 1) - 1
    return (lo, hi) if lo <= hi else None


def _exact_counts(dim: int, nu: int) -> list[int]:
    """Multiples of nu reachable as ceil(dim / m), ascending (layout.py:176-187)."""
    r = math.isqrt(dim)
    out = {k for k in range(nu, min(dim, r + nu) + 1, nu) if _band(dim, k)}
    for m in range(1, r + 2):
        k = _cdiv(dim, m)
        if k % nu == 0 and _band(dim, k):
            out.add(k)
    return sorted(out)


def _mode_choice(dim: int, model: _Model, gs, m_max):
    """Widest feasible interval for one mode (layout.py:190-244)."""
    nu = model.nu
    if dim < nu:
        return (1, dim) if model.fits(1, dim, gs) else None
    cap = dim if m_max is None else min(dim, m_max)
    for k in _exact_counts(dim, nu):
        lo, hi = _band(dim, k)
        hi = min(hi, cap)
        if lo > hi:
            continue
        if model.fits(hi, k, gs):
            return hi, k
        if not model.fits(lo, k, gs):
            continue
        while lo < hi:  # Eq. 3 is monotone in m
            mid = (lo + hi + 1) // 2
            if model.fits(mid, k, gs):
                lo = mid
            else:
                hi = mid - 1
        return lo, k
    q = 1
    while True:  # ragged tail: k a multiple of nu, trailing intervals empty
        k = q * nu
        m = max(min(_cdiv(dim, k), cap) if cap >= 1 else 1, 1)
        if m * k >= dim and model.fits(m, k, gs):
            return m, k
        if m == 1 and m * k >= dim:
            return None
        q += 1


def select_params(dims: Sequence[int], nnz: int, nu: int, gamma: int, rank: int,
                  alpha: int = 8, beta: int | None = None, sigma: int = 8,
                  theta: float = 0.5, g_range: tuple = (1024, 32768),
                  m_max: int | None = None) -> PartitionParams:
    """The reference's parameter choice (layout.py:247-318)."""
    dims = tuple(int(d) for d in dims)
    if nu < 1 or gamma <= 0 or rank < 1:
        raise ValueError("nu, gamma and rank must be positive")
    beta = default_element_bytes(len(dims)) if beta is None else beta
    gs = _pow2_between(int(g_range[0]), int(g_range[1]))
    model = _Model(int(nnz), int(nu), theta * gamma, int(rank), int(alpha), int(beta), int(sigma))

    def solve(cands):
        picks = []
        for d in dims:
            got = _mode_choice(d, model, cands, m_max)
            if got is None:
                return None
            picks.append(got)
        return picks

    chosen = solve(gs)
    g_final = None
    if chosen is not None:
        g_final = next((g for g in reversed(gs)
                        if all(model.lhs(m, k, g) <= model.budget for m, k in chosen)), None)
    if g_final is None:
        for g in reversed(gs):
            chosen = solve([g])
            if chosen is not None:
                g_final = g
                break
    if g_final is None:
        raise InfeasibleParamsError(_explain(dims, model, gs))
    return PartitionParams(dims=dims, nnz=int(nnz), m=tuple(m for m, _ in chosen),
                           k=tuple(k for _, k in chosen), g=g_final, nu=int(nu),
                           gamma=int(gamma), theta=float(theta), rank=int(rank),
                           alpha=int(alpha), beta=int(beta), sigma=int(sigma))


def _explain(dims, model: _Model, gs) -> str:
    g = min(gs)
    parts = []
    for n, d in enumerate(dims):
        k = d if d < model.nu else model.nu * _cdiv(d, model.nu)
        terms = {"factor-interval": model.alpha * model.rank * model.nu,
                 "shard-elements": model.beta * g * model.nu,
                 "remap-cursors": model.sigma * (_cdiv(model.nnz, g) + k)}
        worst = max(terms, key=terms.get)
        parts.append(f"mode {n}: even m=1, g={g} needs {sum(terms.values())} bytes "
                     f"(budget {model.budget:.0f}, binding term {worst}={terms[worst]})")
    return "no feasible (m, g): " + "; ".join(parts)


def _auto_rows(dim: int, nnz: int, rank: int) -> int:
    """Super-shard height of one mode (measured on c2-c4, profiles/round1/r1_kernel_experiments.md):
    a 4 KB accumulator tile when super-shards stay large (>= 64k nonzeros: fewer rows per
    2048-element tile -> fewer segments, fewer ballot rounds) or become so sparse that
    <= 4k nonzeros share an 8 KB tile's rows (direct chunks: rows complete inside one tile);
    8 KB otherwise (fewer, fuller chunks)."""
    small = max(1, 4096 // (4 * int(rank)))
    big = max(1, 8192 // (4 * int(rank)))
    a_small = nnz * small / max(dim, 1)
    a_big = nnz * big / max(dim, 1)
    return min(dim, small if (a_small >= 65536 or a_big <= 4096) else big)


def device_params(dims: Sequence[int], nnz: int, rank: int, acc_tile_bytes: int | None = None,
                  g: int = 32768, m: Sequence[int] | None = None) -> PartitionParams:
    """B200 partition: per mode m rows per super-shard (one fp32 accumulator
    tile of m x R in shared memory) -- acc_tile_bytes / (4 R) when given,
    else chosen per mode by :func:`_auto_rows` -- and k = ceil(I / m).
    gamma/theta/nu are recorded for the cache model only (nu = 1: CTAs,
    not threads, consume super-shards)."""
    dims = tuple(int(d) for d in dims)
    if m is None:
        if acc_tile_bytes is None and len(dims) == 3:
            # 3-mode tensors run the packed kernel, whose <= 32-row ranking
            # (row-owner lanes) wins everywhere measured: c2, c4 (109.5 vs
            # 115.8 ms at 8 KB), c5; and c1 (R = 16): 0.121 ms per sweep at 32
            # rows vs 0.131 at the 4 KB tile's 64 (tools/c1_sweep.sh)
            small = max(1, 4096 // (4 * int(rank)))
            m = tuple(min(d, small, 32) for d in dims)
        elif acc_tile_bytes is None:
            m = tuple(_auto_rows(d, nnz, rank) for d in dims)
        else:
            width = max(1, int(acc_tile_bytes) // (4 * int(rank)))
            m = tuple(min(d, width) for d in dims)
    m = tuple(int(x) for x in m)
    k = tuple(_cdiv(d, mm) for d, mm in zip(dims, m))
    rec = 4 * len(dims) + 4
    return PartitionParams(dims=dims, nnz=int(nnz), m=m, k=k, g=int(g), nu=1,
                           gamma=126 << 20, theta=0.5, rank=int(rank), alpha=4, beta=rec,
                           sigma=4)

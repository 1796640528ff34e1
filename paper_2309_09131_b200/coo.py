"""Host COO tensor with the reference's validation (coo.py:52-121).

``CooTensor`` is the input type of ``build_sharded(tensor, params)`` (the
reference call shape, layout.py:462) and the return type of
``DeviceShardedTensor.to_coo()`` (layout.py:432-434).  It holds int64
coordinates and float64 values on the host, like the reference, and
validates on construction: at least 2 modes, positive dims, no empty tensor,
aligned values, finite values, coordinates in range and no duplicate
coordinates ("coalesce first", coo.py:88-89).

The duplicate check is a 1-D sort of a mixed-radix int64 key when the
dims' product fits 63 bits (every BASELINE config except c4), else a lexsort
of the columns -- both O(nnz log nnz) without ``np.unique(axis=0)``'s
void-typed sort, which took minutes at c2's 76.9M nonzeros.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np

__all__ = ["CooTensor", "Element", "coords_key", "has_duplicates", "parse_frostt", "read_frostt",
           "write_frostt", "synth_tensor"]


@dataclass(frozen=True)
class Element:
    """A single nonzero: zero-based coordinates and its value (coo.py:44-49)."""

    indices: tuple
    value: float


def coords_key(subs: np.ndarray, dims: Sequence[int]) -> np.ndarray | None:
    """Row-major flattened index of every coordinate row as int64, or None
    when prod(dims) does not fit 63 bits."""
    dims = [int(d) for d in dims]
    if math.prod(dims) >= 1 << 63:
        return None
    key = np.zeros(subs.shape[0], dtype=np.int64)
    for n, d in enumerate(dims):
        key *= d
        key += subs[:, n]
    return key


def has_duplicates(subs: np.ndarray, dims: Sequence[int]) -> bool:
    """True iff two rows of `subs` are equal (coordinates assumed in range)."""
    n = subs.shape[0]
    if n < 2:
        return False
    key = coords_key(subs, dims)
    if key is not None:
        key = np.sort(key)
        return bool(np.any(key[1:] == key[:-1]))
    o = np.lexsort(subs.T[::-1])
    s = subs[o]
    return bool(np.any(np.all(s[1:] == s[:-1], axis=1)))


@dataclass(frozen=True, eq=False)
class CooTensor:
    """Sparse tensor in coordinate form, validated on construction and
    treated as immutable (coo.py:52-121)."""

    dims: tuple
    subs: np.ndarray  # (nnz, N) int64
    vals: np.ndarray  # (nnz,) float64

    def __post_init__(self):
        object.__setattr__(self, "dims", tuple(int(d) for d in self.dims))
        subs = np.ascontiguousarray(np.asarray(self.subs, dtype=np.int64))
        vals = np.ascontiguousarray(np.asarray(self.vals, dtype=np.float64))
        object.__setattr__(self, "subs", subs)
        object.__setattr__(self, "vals", vals)
        if len(self.dims) < 2:
            raise ValueError("a tensor needs at least 2 modes")
        if any(d < 1 for d in self.dims):
            raise ValueError("every mode dimension must be positive")
        if subs.ndim != 2 or subs.shape[1] != len(self.dims):
            raise ValueError("subs must be (nnz, num_modes)")
        if subs.shape[0] == 0:
            raise ValueError("tensor has no nonzeros")
        if vals.shape != (subs.shape[0],):
            raise ValueError("vals must align with subs rows")
        if not np.all(np.isfinite(vals)):
            raise ValueError("values must be finite")
        if subs.min() < 0:
            raise ValueError("negative index")
        if np.any(subs.max(axis=0) >= np.asarray(self.dims, dtype=np.int64)):
            raise ValueError("index out of range for declared dims")
        if has_duplicates(subs, self.dims):
            raise ValueError("duplicate coordinates (coalesce first)")

    @property
    def num_modes(self) -> int:
        return len(self.dims)

    @property
    def nnz(self) -> int:
        return self.subs.shape[0]

    @property
    def density(self) -> float:
        return self.nnz / math.prod(self.dims)

    def element(self, i: int) -> Element:
        return Element(tuple(int(c) for c in self.subs[i]), float(self.vals[i]))

    def norm(self) -> float:
        """Frobenius norm (sqrt of the sum of squared nonzero values)."""
        return float(np.linalg.norm(self.vals))

    def same_nonzeros(self, other, rtol: float = 0.0) -> bool:
        """Multiset equality of (coordinates, value) pairs, ignoring order
        (coo.py:110-121)."""
        if tuple(self.dims) != tuple(other.dims) or self.nnz != other.nnz:
            return False
        a = np.lexsort(self.subs.T[::-1])
        b = np.lexsort(np.asarray(other.subs).T[::-1])
        if not np.array_equal(self.subs[a], np.asarray(other.subs)[b]):
            return False
        va, vb = self.vals[a], np.asarray(other.vals, dtype=np.float64)[b]
        if rtol == 0.0:
            return bool(np.array_equal(va, vb))
        return bool(np.allclose(va, vb, rtol=rtol, atol=0.0))


# ------------------------------------------------ reference-shaped entry points
# The reference's coo module returns and takes CooTensor objects
# (coo.py:212-355); the array-level implementations live in io.py / synth.py.

def parse_frostt(source, dims=None) -> CooTensor:
    """FROSTT text (1-based, '#' comments, duplicates summed) -> CooTensor
    (coo.py:212-272; errors are io.FrosttParseError with the line number)."""
    from . import io as _io
    subs, vals, d = _io.parse_frostt(source, dims=dims)
    return CooTensor(d, subs, vals)


def read_frostt(path, dims=None) -> CooTensor:
    """coo.py:298-299."""
    from pathlib import Path
    return parse_frostt(Path(path), dims=dims)


def write_frostt(tensor: CooTensor, destination=None):
    """1-based indices, exact %.17g values; text when `destination` is None
    (coo.py:302-316)."""
    from . import io as _io
    return _io.write_frostt(tensor.subs, tensor.vals, destination)


def synth_tensor(dims, nnz: int, seed: int, skew: float = 0.0) -> CooTensor:
    """The reference's seeded generator (coo.py:323-355), bit-identical."""
    from . import synth as _synth
    subs, vals = _synth.synth_tensor(dims, nnz, seed, skew=skew)
    return CooTensor(tuple(int(d) for d in dims), subs, vals)

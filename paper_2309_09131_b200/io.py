"""On-disk formats around the device path.

* MCFD factor dumps -- byte-compatible restatement of the reference's
  ``save_factor_set`` / ``load_factor_set`` (coo.py:433-474): magic "MCFD",
  version 1, N, per-mode row counts (u64), rank (u32), lambda flag (u8),
  little-endian float64 lambdas and row-major factors.
* FROSTT ``.tns`` text -- ``read_frostt`` / ``write_frostt`` with the
  reference's conventions (coo.py:212-316): 1-based indices, ``#`` comments,
  duplicates coalesced by summation (sorted unique coordinates), dims default
  to the largest index per mode, ``%.17g`` values.
* FLYCOO image -- a binary dump of a built :class:`DeviceShardedTensor`
  (plan fills, active records, slot maps) so that the billion-nonzero
  configurations reload in seconds instead of rebuilding.
"""

from __future__ import annotations

import io as _io
import json
import struct
from pathlib import Path

import numpy as np
import torch

from .factors import DeviceFactorSet
from .layout import DeviceShardedTensor, plan_from_counts
from .params import PartitionParams

__all__ = ["FrosttParseError", "read_frostt", "parse_frostt", "write_frostt", "save_factor_set",
           "load_factor_set", "save_flycoo", "load_flycoo"]

MCFD_MAGIC = b"MCFD"
FLYCOO_MAGIC = b"FLYC"


# --------------------------------------------------------------------- MCFD

def save_factor_set(fs, destination=None):
    """Serialise factors (DeviceFactorSet or any object with .factors /
    .lambdas) in the reference's MCFD v1 layout; returns bytes when
    `destination` is None."""
    mats = [f.double().cpu().numpy() if isinstance(f, torch.Tensor) else np.asarray(f, np.float64)
            for f in fs.factors]
    lam = np.asarray(fs.lambdas, dtype=np.float64)
    head = struct.pack("<4sII", MCFD_MAGIC, 1, len(mats))
    head += struct.pack(f"<{len(mats)}Q", *(m.shape[0] for m in mats))
    head += struct.pack("<IB", mats[0].shape[1], 1)
    blob = head + lam.astype("<f8").tobytes() + b"".join(
        np.ascontiguousarray(m, dtype="<f8").tobytes() for m in mats)
    if destination is None:
        return blob
    Path(destination).write_bytes(blob)
    return None


def load_factor_set(source, device="cuda") -> DeviceFactorSet:
    blob = Path(source).read_bytes() if isinstance(source, (str, Path)) else bytes(source)
    magic, version, nmodes = struct.unpack_from("<4sII", blob, 0)
    if magic != MCFD_MAGIC:
        raise ValueError("not a factor dump (bad magic)")
    if version != 1:
        raise ValueError(f"unsupported dump version {version}")
    off = 12
    rows = struct.unpack_from(f"<{nmodes}Q", blob, off)
    off += 8 * nmodes
    rank, has_lambdas = struct.unpack_from("<IB", blob, off)
    off += 5
    if has_lambdas:
        lam = np.frombuffer(blob, dtype="<f8", count=rank, offset=off).copy()
        off += 8 * rank
    else:
        lam = np.ones(rank)
    mats = []
    for r in rows:
        n = int(r) * rank
        mats.append(np.frombuffer(blob, dtype="<f8", count=n, offset=off).reshape(int(r), rank))
        off += 8 * n
    return DeviceFactorSet(tuple(m.astype(np.float32) for m in mats), lam, device)


# ------------------------------------------------------------------- FROSTT

class FrosttParseError(ValueError):
    """Malformed FROSTT text; carries the 1-based line number when known."""

    def __init__(self, message: str, lineno: int | None = None):
        self.lineno = lineno
        super().__init__(f"line {lineno}: {message}" if lineno is not None else message)


def _text_of(source) -> str:
    if isinstance(source, Path):
        return source.read_text()
    if isinstance(source, str) and "\n" not in source and Path(source).exists():
        return Path(source).read_text()
    if isinstance(source, bytes):
        return source.decode("ascii")
    if isinstance(source, str):
        return source
    data = source.read()
    return data.decode("ascii") if isinstance(data, bytes) else data


def parse_frostt(source, dims=None):
    """FROSTT text -> (subs int64 (nnz, N) zero-based, vals float64, dims)."""
    lines, linenos = [], []
    for no, raw in enumerate(_text_of(source).splitlines(), start=1):
        t = raw.strip()
        if t and not t.startswith("#"):
            lines.append(t)
            linenos.append(no)
    if not lines:
        raise FrosttParseError("no nonzero entries in input")
    ncols = len(lines[0].split())
    if ncols < 3:
        raise FrosttParseError(f"expected at least 2 indices and a value, got {ncols} tokens",
                               linenos[0])
    try:
        table = np.loadtxt(_io.StringIO("\n".join(lines)), dtype=np.float64, ndmin=2)
        if table.shape[1] != ncols:
            raise ValueError
    except ValueError:
        for t, no in zip(lines, linenos):
            parts = t.split()
            if len(parts) != ncols:
                raise FrosttParseError(f"expected {ncols} tokens, got {len(parts)}", no) from None
            for tok in parts:
                try:
                    float(tok)
                except ValueError:
                    raise FrosttParseError(f"non-numeric token {tok!r}", no) from None
        raise FrosttParseError("unparseable input")
    N = ncols - 1
    raw = table[:, :N]
    vals = np.ascontiguousarray(table[:, N])
    frac = np.any(raw != np.floor(raw), axis=1)
    if frac.any():
        raise FrosttParseError("non-integer index", linenos[int(np.argmax(frac))])
    nonpos = np.any(raw <= 0, axis=1)
    if nonpos.any():
        raise FrosttParseError("indices are 1-based and must be positive",
                               linenos[int(np.argmax(nonpos))])
    subs = raw.astype(np.int64) - 1
    uniq, inverse = np.unique(subs, axis=0, return_inverse=True)
    sums = np.zeros(uniq.shape[0])
    np.add.at(sums, inverse.reshape(-1), vals)
    seen = uniq.max(axis=0) + 1
    if dims is None:
        dims = tuple(int(d) for d in seen)
    else:
        dims = tuple(int(d) for d in dims)
        if len(dims) != N:
            raise FrosttParseError(f"dims override has {len(dims)} modes, file has {N}")
        if np.any(seen > np.asarray(dims)):
            raise FrosttParseError("dims override smaller than an observed index")
    return uniq, sums, dims


def read_frostt(path, dims=None):
    return parse_frostt(Path(path), dims=dims)


def write_frostt(subs, vals, destination=None):
    """1-based indices, %.17g values (exact round trip)."""
    subs = np.asarray(subs) + 1
    text = "".join(" ".join(str(int(c)) for c in row) + f" {v:.17g}\n"
                   for row, v in zip(subs, np.asarray(vals, dtype=np.float64)))
    if destination is None:
        return text
    Path(destination).write_text(text)
    return None


# ------------------------------------------------------------ FLYCOO image

_CHUNK = 1 << 26  # elements per host staging chunk


def save_flycoo(st: DeviceShardedTensor, path) -> None:
    """Plan fills, the active record buffer and the slot maps (canonical
    arrangement only -- the slot maps are invalid after a cursor remap)."""
    if not st.canonical:
        raise ValueError("only canonical (slot-strategy) layouts can be saved")
    p = st.params
    header = {"dims": list(p.dims), "nnz": p.nnz, "m": list(p.m), "k": list(p.k), "g": p.g,
              "nu": p.nu, "gamma": p.gamma, "theta": p.theta, "rank": p.rank, "alpha": p.alpha,
              "beta": p.beta, "sigma": p.sigma, "active_mode": st.active_mode,
              "cw": int(st.crd[0].shape[1]), "separate_values": st.val[0] is not None}
    hj = json.dumps(header).encode()
    crd, val = st.device_arrays()
    with open(path, "wb") as f:
        f.write(struct.pack("<4sII", FLYCOO_MAGIC, 1, len(hj)))
        f.write(hj)
        for counts in st.plan.ss_counts:
            f.write(np.ascontiguousarray(counts, dtype="<i8").tobytes())
        for t in [crd] + ([val] if val is not None else []) + list(st.slot_maps):
            for a in range(0, t.shape[0], _CHUNK):
                f.write(t[a:a + _CHUNK].cpu().numpy().tobytes())


def load_flycoo(path, device="cuda") -> DeviceShardedTensor:
    dev = torch.device(device)
    with open(path, "rb") as f:
        magic, version, hlen = struct.unpack("<4sII", f.read(12))
        if magic != FLYCOO_MAGIC:
            raise ValueError("not a FLYCOO image (bad magic)")
        if version != 1:
            raise ValueError(f"unsupported FLYCOO image version {version}")
        h = json.loads(f.read(hlen))
        params = PartitionParams(dims=tuple(h["dims"]), nnz=h["nnz"], m=tuple(h["m"]),
                                 k=tuple(h["k"]), g=h["g"], nu=h["nu"], gamma=h["gamma"],
                                 theta=h["theta"], rank=h["rank"], alpha=h["alpha"],
                                 beta=h["beta"], sigma=h["sigma"])
        counts = [np.frombuffer(f.read(8 * k), dtype="<i8").copy() for k in params.k]
        plan = plan_from_counts(params, counts)
        nnz, cw, N = params.nnz, h["cw"], len(params.dims)

        def load(shape, dtype):
            t = torch.empty(shape, dtype=dtype, device=dev)
            per = int(np.prod(shape[1:])) if len(shape) > 1 else 1
            isz = torch.empty(0, dtype=dtype).element_size()
            for a in range(0, shape[0], _CHUNK):
                n = min(_CHUNK, shape[0] - a)
                buf = np.frombuffer(f.read(n * per * isz), dtype=np.uint8).copy()
                t[a:a + n] = torch.from_numpy(buf).view(dtype).reshape((n,) + tuple(shape[1:])).to(dev)
            return t

        crd0 = load((nnz, cw), torch.int32)
        val0 = load((nnz,), torch.float32) if h["separate_values"] else None
        slots = tuple(load((nnz,), torch.int32) for _ in range(N))
    crd = [crd0, torch.empty_like(crd0)]
    val = [None, None] if val0 is None else [val0, torch.empty_like(val0)]
    st = DeviceShardedTensor(plan, crd, val, slots, dev)
    st.active_mode = h["active_mode"]
    return st

"""Device factor matrices (the reference's FactorSet, coo.py:124-192, held as
fp32 CUDA tensors, one (I_w, R) row-major matrix per mode)."""

from __future__ import annotations

from typing import Sequence

import numpy as np
import torch

from . import _lib

__all__ = ["DeviceFactorSet"]


def _as_device_f32(f, device) -> torch.Tensor:
    t = torch.as_tensor(f)
    if t.dtype != torch.float32 or t.device != device or not t.is_contiguous():
        t = t.to(device=device, dtype=torch.float32).contiguous()
    return t


class DeviceFactorSet:
    """Factor matrices sharing one rank, plus per-column lambdas (host
    float64, like the reference).  ``validate=True`` repeats the reference's
    checks, including the finiteness scan (coo.py:133-152); the engine builds
    its per-mode sets with ``validate=False`` to keep the sweep free of host
    synchronisation."""

    def __init__(self, factors: Sequence, lambdas=None, device="cuda", validate: bool = True):
        dev = torch.device(device)
        if dev.type == "cuda" and dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        fs = tuple(_as_device_f32(f, dev) for f in factors)
        if not fs:
            raise ValueError("need at least one factor matrix")
        if any(f.dim() != 2 for f in fs):
            raise ValueError("factor matrices must be 2-D")
        ranks = {int(f.shape[1]) for f in fs}
        if len(ranks) != 1:
            raise ValueError(f"factor matrices disagree on rank: {sorted(ranks)}")
        rank = ranks.pop()
        lam = np.ones(rank) if lambdas is None else np.ascontiguousarray(
            np.asarray(lambdas, dtype=np.float64))
        if lam.shape != (rank,):
            raise ValueError("lambdas must have one entry per rank column")
        if validate:
            for f in fs:
                if not bool(torch.isfinite(f).all()):
                    raise ValueError("factor entries must be finite")
        self.factors = fs
        self.lambdas = lam
        self.device = dev

    @property
    def rank(self) -> int:
        return int(self.factors[0].shape[1])

    @property
    def num_modes(self) -> int:
        return len(self.factors)

    def shapes_match(self, dims) -> bool:
        return len(dims) == len(self.factors) and all(
            int(f.shape[0]) == int(d) for f, d in zip(self.factors, dims))

    def require_match(self, dims) -> None:
        if not self.shapes_match(dims):
            got = [int(f.shape[0]) for f in self.factors]
            raise ValueError(f"factor rows {got} do not match tensor dims {list(dims)}")

    def replace_factor(self, mode: int, matrix) -> "DeviceFactorSet":
        fs = list(self.factors)
        fs[mode] = matrix
        return DeviceFactorSet(tuple(fs), self.lambdas.copy(), self.device, validate=False)

    def to_numpy(self) -> list:
        """float64 host copies (reference dtype)."""
        return [f.double().cpu().numpy() for f in self.factors]

    @classmethod
    def from_host(cls, factors, lambdas=None, device="cuda") -> "DeviceFactorSet":
        return cls(tuple(np.asarray(f, dtype=np.float32) for f in factors), lambdas, device)

    @classmethod
    def ones(cls, dims, rank: int, device="cuda") -> "DeviceFactorSet":
        return cls(tuple(torch.ones((int(d), rank), device=device) for d in dims), None, device,
                   validate=False)

    @classmethod
    def random(cls, dims, rank: int, seed: int, device="cuda") -> "DeviceFactorSet":
        """The reference's ``FactorSet.random`` (coo.py:184-192): U[0,1)
        float64 entries from ``np.random.Generator(np.random.Philox(seed))``,
        drawn mode by mode in the same order, then held as fp32 on the device
        -- the fp32 rounding of the reference's factors for the same seed."""
        rng = np.random.Generator(np.random.Philox(seed))
        return cls(tuple(rng.random((int(d), rank)).astype(np.float32) for d in dims), None, device,
                   validate=False)

    @classmethod
    def random_device(cls, dims, rank: int, seed: int, device="cuda") -> "DeviceFactorSet":
        """U(0,1) fp32 entries from Philox4x32-10 (stream = mode) generated on
        the device (the billion-row factors of c3/c4 without a host round
        trip).  Not the reference's stream: use :meth:`random` for that."""
        dev = torch.device(device)
        fs = []
        for w, d in enumerate(dims):
            f = torch.empty((int(d), rank), dtype=torch.float32, device=dev)
            _lib.call("fc_synth_uniform", int(seed), 1000 + w, f.numel(), f.data_ptr(), 0,
                      torch.cuda.current_stream(dev).cuda_stream)
            fs.append(f)
        return cls(tuple(fs), None, dev, validate=False)

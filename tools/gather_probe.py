"""Gather-only bound for the c2 mode-0 access pattern (factor rows of modes 1
and 2, in the layout's element order and in a random order)."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2309_09131_b200 import DeviceFactorSet, build_device_sharded, device_params
from paper_2309_09131_b200.synth import config_tensor

dev = torch.device("cuda", 0)
coords, vals = config_tensor(2, device=dev)
dims = (12092, 9184, 28818)
params = device_params(dims, coords.shape[0], 32)
st = build_device_sharded(coords, vals, params, device=dev)
fs = DeviceFactorSet.random_device(dims, 32, seed=1, device=dev)
crd = st.crd[0]
idx = torch.stack([crd[:, 1], crd[:, 2]], dim=1).contiguous()
n = idx.shape[0]
L = ctypes.CDLL(str(Path(__file__).with_name("libgather_probe.so")))
L.gather_probe.restype = ctypes.c_float
L.gather_probe_tma.restype = ctypes.c_float
L.gather_probe_tma.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                               ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
L.gather_probe.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
sink = torch.zeros(1, device=dev)
for name, ix in (("layout order", idx), ("random order", idx[torch.randperm(n, device=dev)].contiguous())):
    for u in (1, 4, 8):
        for blocks in (148 * 3, 148 * 8, 148 * 32):
            ms = L.gather_probe(ix.data_ptr(), n, fs.factors[1].data_ptr(), fs.factors[2].data_ptr(),
                                sink.data_ptr(), u, blocks)
            print(f"{name:13s} U={u} blocks={blocks:5d}: {ms:.3f} ms  ({n * 256 / ms / 1e6:.0f} GB/s of rows)")

for u in (4, 8):
    for blocks in (148 * 2, 148 * 3, 148 * 8):
        ms = L.gather_probe_tma(idx.data_ptr(), n, fs.factors[1].data_ptr(), fs.factors[2].data_ptr(),
                                sink.data_ptr(), u, blocks)
        print(f"TMA layout    U={u} blocks={blocks:5d}: {ms:.3f} ms  ({n * 256 / ms / 1e6:.0f} GB/s of rows)")

L.gather_probe_tex.restype = ctypes.c_float
L.gather_probe_tex.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                               ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int,
                               ctypes.c_int, ctypes.c_int]
for both in (0, 1):
    for u in (4, 8):
        for blocks in (148 * 8, 148 * 32):
            ms = L.gather_probe_tex(idx.data_ptr(), n, fs.factors[1].data_ptr(), fs.factors[1].numel(),
                                    fs.factors[2].data_ptr(), fs.factors[2].numel(), sink.data_ptr(),
                                    u, blocks, both)
            what = "TEX both" if both else "LDG+TEX"
            print(f"{what:13s} U={u} blocks={blocks:5d}: {ms:.3f} ms  ({n * 256 / ms / 1e6:.0f} GB/s of rows)")

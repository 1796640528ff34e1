"""LDG.E.256 (4 lanes per factor row) against LDG.E.128 (8 lanes) for the c2
mode-0 gathers in layout order.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
-O3 -shared -Xcompiler -fPIC -o tools/libgather_probe256.so tools/gather_probe256.cu"""
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
st = build_device_sharded(coords, vals, params, device=dev, check_duplicates=False)
fs = DeviceFactorSet.random_device(dims, 32, seed=1, device=dev)
crd = st.crd[0]
idx = torch.stack([crd[:, 1], crd[:, 2]], dim=1).contiguous()
n = idx.shape[0]
L = ctypes.CDLL(str(Path(__file__).with_name("libgather_probe256.so")))
L.gather_probe_w.restype = ctypes.c_float
L.gather_probe_w.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                             ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int]
sink = torch.zeros(1, device=dev)
for width, us in ((128, (2, 3, 4, 8)), (256, (1, 2, 4))):
    for u in us:
        for blocks in (148 * 3, 148 * 4, 148 * 8):
            ms = L.gather_probe_w(idx.data_ptr(), n, fs.factors[1].data_ptr(), fs.factors[2].data_ptr(),
                                  sink.data_ptr(), width, u, blocks)
            print(f"LDG.{width} U={u} blocks={blocks:5d} ({blocks // 148 * 8} warps/SM): {ms:.3f} ms  "
                  f"({n * 256 / ms / 1e6:.0f} GB/s of rows)")

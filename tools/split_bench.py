"""Time one mode pass of config 2 split into its parts: fused (compute+remap),
compute only, remap only (K1 with do_remap=0 / do_compute=0)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2309_09131_b200 import (DeviceFactorSet, build_device_sharded, device_params, _lib)
from paper_2309_09131_b200.synth import config_tensor

dev = torch.device("cuda", 0)
coords, vals = config_tensor(2, device=dev)
dims, R = (12092, 9184, 28818), 32
params = device_params(dims, coords.shape[0], R)
st = build_device_sharded(coords, vals, params, device=dev)
fs = DeviceFactorSet.random_device(dims, R, seed=1002, device=dev)
fptrs = _lib.ptr_array([f.data_ptr() for f in fs.factors])
strm = torch.cuda.current_stream().cuda_stream


def run(mode, comp, remap, reps=10):
    w = st.mode_work(mode, R)
    out = torch.empty((dims[mode], R), device=dev)
    flags_p, proc_p = st.stat_ptrs()
    a, b = st.active, 1 - st.active
    vp = lambda t: t.data_ptr() if t is not None else None

    def once():
        _lib.call("fc_mode_worker", st.crd[a].data_ptr(), None, st.crd[b].data_ptr(), None, fptrs, _lib.i64_array(dims),
                  out.data_ptr(), 3, mode, R, dims[mode], params.m[mode], w.chunk_start.data_ptr(),
                  w.chunk_ss.data_ptr(), w.chunk_part.data_ptr(),
                  w.chunk_rows.data_ptr() if w.chunk_rows is not None else None, w.tile_rows, w.hist_rows, w.nchunks, w.red1.data_ptr(),
                  w.nred1, w.red2.data_ptr(), w.nred2, vp(w.part_ws), vp(w.part_ws2),
                  st.slot_maps[mode].data_ptr(), st.nnz, comp, remap, int(w.acc_in_smem), flags_p,
                  proc_p, strm)
    once()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        once()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for name, c, r in (("fused", 1, 1), ("compute", 1, 0), ("remap", 0, 1)):
    print(name, " ".join(f"{run(m, c, r):.3f}" for m in (0,)), "ms (mode 0)")
# stream copy reference: read+write the record buffer once
x = st.crd[0]
y = torch.empty_like(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    y.copy_(x)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"copy of records {x.numel()*4/1e9:.2f} GB: {ms:.3f} ms = {2*x.numel()*4/ms/1e6:.0f} GB/s")

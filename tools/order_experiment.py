"""Experiment: intra-shard order 'source' (this build: by previous-mode shard,
coalesced remap writes) vs 'row' (by output row then next coordinate:
pre-sorted for compute, scattered remap writes).  Times the remap-only and
fused passes on config 2 for both layouts."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2309_09131_b200 import (DeviceFactorSet, build_device_sharded, device_params, _lib)
from paper_2309_09131_b200.synth import config_tensor

dev = torch.device("cuda", 0)
coords, vals = config_tensor(2, device=dev)
dims, R, N = (12092, 9184, 28818), 32, 3
params = device_params(dims, coords.shape[0], R)
st = build_device_sharded(coords, vals, params, device=dev)
nnz = st.nnz
fs = DeviceFactorSet.random_device(dims, R, seed=1002, device=dev)
fptrs = _lib.ptr_array([f.data_ptr() for f in fs.factors])
strm = torch.cuda.current_stream().cuda_stream


def timed(layout, mode, comp, remap, reps=5):
    crd, slots = layout
    w = st.mode_work(mode, R)
    out = torch.empty((dims[mode], R), device=dev)
    dst = torch.empty_like(crd)
    flags_p, proc_p = st.stat_ptrs()
    vp = lambda t: t.data_ptr() if t is not None else None

    def once():
        _lib.call("fc_mode_worker", crd.data_ptr(), None, dst.data_ptr(), None, fptrs, _lib.i64_array(dims),
                  out.data_ptr(), N, mode, R, dims[mode], params.m[mode], w.chunk_start.data_ptr(),
                  w.chunk_ss.data_ptr(), w.chunk_part.data_ptr(),
                  w.chunk_rows.data_ptr() if w.chunk_rows is not None else None, w.tile_rows, w.hist_rows, w.nchunks, w.red1.data_ptr(),
                  w.nred1, w.red2.data_ptr(), w.nred2, vp(w.part_ws), vp(w.part_ws2),
                  slots.data_ptr(), nnz, comp, remap, int(w.acc_in_smem), flags_p, proc_p, strm)
    once()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        once()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


# positions of every element (indexed by its mode-0 position) in each mode
pos = [torch.arange(nnz, device=dev, dtype=torch.int64)]
for n in range(N - 1):
    pos.append((st.slot_maps[n].to(torch.int64) & 0xFFFFFFFF)[pos[-1]])
rec0 = st.crd[0]
c = rec0[:, :N].to(torch.int64)


def layout_for(order_kind):
    newpos = []
    for n in range(N):
        so = torch.as_tensor(st.plan.shard_offsets[n], device=dev)
        shard = torch.searchsorted(so, pos[n], right=True) - 1
        if order_kind == "source":
            key = pos[n]
        else:
            w1 = (n + 1) % N
            key = (shard << 32) | (c[:, n] << 16) | (c[:, w1] & 0xFFFF)
        o = torch.argsort(key, stable=True)
        p = torch.empty_like(o)
        p[o] = torch.arange(nnz, device=dev)
        newpos.append(p)
    # mode-0 buffer and slot map of mode 0 under this order
    crd = torch.empty_like(rec0)
    crd[newpos[0]] = rec0
    slot0 = torch.empty(nnz, dtype=torch.int64, device=dev)
    slot0[newpos[0]] = newpos[1]
    return crd, slot0.to(torch.int32)


for kind in ("source", "row"):
    lay = layout_for(kind)
    print(kind, "remap-only %.3f ms" % timed(lay, 0, 0, 1), " fused %.3f ms" % timed(lay, 0, 1, 1),
          " compute-only %.3f ms" % timed(lay, 0, 1, 0))

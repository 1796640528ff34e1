"""Experiment: launch order of the mode-pass chunks.

CTA b normally runs chunk b (super-shard order).  Here the chunks are
launched by their relative position inside their super-shard (j / chunks of
the super-shard), so the CTAs resident at any moment work on the same part
of the Morton range of many super-shards -- and gather the same region of
the input factors.  Outputs are unchanged (partial tiles are indexed by id).
Needs an experiment build exposing fc_exp_set_chunk_order (a launch-order
array read by the kernels as chunk = order[blockIdx.x]); it was measured
and removed (no gain, see profiles/round1/r1_kernel_experiments.md).

usage: FLYCOO_LIB=libflycoo_ord.so python tools/chunk_order_experiment.py [config]
"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2309_09131_b200 import (DeviceFactorSet, _lib, build_device_sharded, device_params,
                                   mttkrp_mode, schedule_super_shards)
from paper_2309_09131_b200.synth import CONFIGS, config_tensor


def order_by_relative_position(work):
    ss = work.chunk_ss.cpu().numpy().astype(np.int64)
    n = ss.shape[0]
    first = np.r_[0, np.flatnonzero(np.diff(ss)) + 1]
    counts = np.diff(np.r_[first, n])
    j = np.arange(n) - np.repeat(first, counts)
    frac = j / np.repeat(counts, counts)
    return np.lexsort((ss, np.round(frac * 64))).astype(np.int32)


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    dev = torch.device("cuda", 0)
    c = CONFIGS[cfg]
    dims, R = tuple(c["dims"]), 32
    coords, vals = config_tensor(cfg, device=dev)
    params = device_params(dims, int(vals.shape[0]), R)
    st = build_device_sharded(coords, vals, params, device=dev)
    del coords, vals
    smap = schedule_super_shards(st.plan, 1)
    fs = DeviceFactorSet.random_device(dims, R, seed=1, device=dev)
    N = len(dims)
    L = _lib.load()
    L.fc_exp_set_chunk_order.argtypes = [ctypes.c_void_p]
    orders = [torch.from_numpy(order_by_relative_position(st.mode_work(n, R))).to(dev)
              for n in range(N)]
    ref = [mttkrp_mode(st, fs, n, smap) for n in range(N)]
    for label, use in (("super-shard order", False), ("relative-position order", True),
                       ("super-shard order", False), ("relative-position order", True)):
        times = []
        for rep in range(6):
            outs = []
            for n in range(N):
                L.fc_exp_set_chunk_order(orders[n].data_ptr() if use else None)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                outs.append(mttkrp_mode(st, fs, n, smap))
                e1.record()
                e1.synchronize()
                times.append(e0.elapsed_time(e1))
            for a, b in zip(outs, ref):
                assert torch.equal(a, b)
        L.fc_exp_set_chunk_order(None)
        t = np.asarray(times).reshape(-1, N)[1:].mean(0)
        print(f"c{cfg} {label:24s} per mode ms {np.round(t, 3)}  sweep {t.sum():.3f}", flush=True)


if __name__ == "__main__":
    main()

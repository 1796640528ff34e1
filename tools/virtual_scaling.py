"""Per-GPU work of the multi-GPU sweep, measured on ONE B200 (no NVLink).

For P = 1, 2, 4, 8 virtual ranks of the fused exchange (peer.py, chunk
partition), every rank's K1 (its chunk range, records stored into the other
ranks' buffers -- local memory here) and K2 run alone on the whole GPU and
are timed with CUDA events; the slowest rank per mode bounds a real P-GPU
sweep from below (NVLink transfer and barriers not included).  The same is
reported for the super-shard partition (rows never split; dist.py), to show
what splitting the Zipf head super-shard buys.

usage: python tools/virtual_scaling.py [config [nnz]]   (default 2; nnz overrides the size --
the P ranks' own buffers sit next to the global layout, so the billion-nonzero configs run at a
reduced size of the same law)
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2309_09131_b200 import DeviceFactorSet, build_device_sharded, device_params
from paper_2309_09131_b200.dist import partition_super_shards
from paper_2309_09131_b200.peer import PeerShardedTensor
from paper_2309_09131_b200.synth import CONFIGS, config_tensor


def timed(fn, reps=5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    nnz = int(sys.argv[2]) if len(sys.argv) > 2 else None
    dev = torch.device("cuda", 0)
    c = CONFIGS[cfg]
    dims, R = tuple(c["dims"]), 32
    coords, vals = config_tensor(cfg, device=dev, nnz=nnz)
    params = device_params(dims, int(vals.shape[0]), R)
    st = build_device_sharded(coords, vals, params, device=dev)
    del coords, vals
    N = len(dims)
    fs = DeviceFactorSet.random_device(dims, R, seed=1, device=dev)
    result = {"config": cfg, "nnz": int(st.nnz), "modes": {}}
    base = None
    for P in (1, 2, 4, 8):
        ranks = [PeerShardedTensor(st, P, r, ipc=False) for r in range(P)]
        PeerShardedTensor.connect_local(ranks)
        per_mode = []
        for n in range(N):
            outs = [dt.output(n, R)[0] for dt in ranks]
            worst = 0.0
            for r, dt in enumerate(ranks):
                # K1 + K2 of rank r alone (repeatable: same buffers, same inputs)
                def one():
                    dt.mode_pass(list(fs.factors), n, outs[r])
                    dt.reduce(n, outs[r])
                    dt._expected = 0
                worst = max(worst, timed(one))
            per_mode.append(worst)
            for dt in ranks:
                dt.swap()
        for dt in ranks:
            dt._stat.zero_()
        # the super-shard partition: the largest element share of any rank
        ss_share = max(
            float(np.diff(partition_super_shards(st.plan.ss_counts[n], P)[1]).max()) / st.nnz
            for n in range(N))
        sweep = sum(per_mode)
        base = base or sweep
        result["modes"][P] = {"per_mode_ms": [round(x, 4) for x in per_mode],
                              "sweep_ms_lower_bound": round(sweep, 4),
                              "efficiency_bound": round(base / (P * sweep), 3),
                              "largest_rank_share_super_shard_partition": round(ss_share, 3),
                              "efficiency_cap_super_shard_partition": round(1 / (P * ss_share), 3)}
        print(P, result["modes"][P], flush=True)
        del ranks
        torch.cuda.empty_cache()
    tag = f"c{cfg}" if nnz is None else f"c{cfg}_nnz{nnz}"
    out = Path(__file__).resolve().parents[1] / "profiles" / f"r2_virtual_scaling_{tag}.json"
    out.write_text(json.dumps(result, indent=1))


if __name__ == "__main__":
    main()

"""How the fused exchange's remote record stores coalesce (no GPU needed).

In K1 a warp instruction stores the 16-B records of 32 consecutive source
elements (thread tid handles elements j * 256 + tid of a tile).  For the
records whose next-mode owner is another GPU, count the distinct 32-B
sectors and 128-B lines each warp instruction writes: 0.5 sectors / 0.125
lines per record means every remote write is a full line.  The B200
intra-shard order (previous-mode shard, Morton) is what makes the elements
one source shard sends to one destination shard a contiguous run.
c2 law, 8M nonzeros, the bench's parameters, GPUs take equal element ranges.

usage: python tools/peer_store_coalescing.py [nnz]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

import oracle
from paper_2309_09131_b200.params import device_params
from paper_2309_09131_b200.synth import zipf_tensor_host

nnz_req = int(sys.argv[1]) if len(sys.argv) > 1 else 8_000_000
dims = (12092, 9184, 28818)
subs, vals = zipf_tensor_host(dims, nnz_req, seed=2, exponents=(1.1, 1.1, 1.1))
p = device_params(dims, len(vals), 32)
L = oracle.canonical_build(subs, vals.astype(np.float64), dims, p.m, p.k, p.g)
d = oracle.device_order(L)
nnz = len(vals)
warp = np.arange(nnz) // 32
for P in (2, 4, 8):
    recs = secs = lines = 0
    for n in range(3):
        slots = d.slot_maps[n]
        src = np.minimum(np.arange(nnz) * P // nnz, P - 1)
        dst = np.minimum(slots * P // nnz, P - 1)
        rem = src != dst
        recs += int(rem.sum())
        secs += len(np.unique(np.stack([warp[rem], (slots[rem] * 16) // 32], 1), axis=0))
        lines += len(np.unique(np.stack([warp[rem], (slots[rem] * 16) // 128], 1), axis=0))
    print(f"P={P}: remote share {recs / (3 * nnz):.3f}, 32-B sectors per remote record "
          f"{secs / recs:.3f} (0.5 = full), 128-B lines per record {lines / recs:.3f} (0.125 = full)")

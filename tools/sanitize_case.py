"""Small sweeps that launch every K1 family once or twice, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck, one tool per
run -- B200_PROFILING.md).  Each case is checked against the oracle, so a
clean run without the sanitizer exits 0.

  packed 8-B kernel   3-mode, input coordinates fit 32 bits (c2-like law)
  WIDE packed kernel  3-mode, 17 + 17-bit input coordinates (c4-like)
  tile kernel         4-mode (c3-like) and R = 16 (c1-like)
  general kernel      m * R * 4 > 64 KB (global accumulator)
  direct chunks       sparse mode (super-shards below one tile)
  peer kernels        two virtual ranks through fc_mode_worker_peers
  K2 reduce           heavy super-shard split over several chunks

usage: python tools/sanitize_case.py
"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]

import oracle  # noqa: E402
from gpu_helpers import assert_rel  # noqa: E402
from paper_2309_09131_b200 import (DeviceFactorSet, build_device_sharded, device_params,  # noqa: E402
                                   schedule_super_shards, sweep_all_modes, mttkrp_mode)
from paper_2309_09131_b200.synth import zipf_tensor  # noqa: E402


def sweep_case(name, dims, nnz, law, R, m=None, g=4096, fixed=False):
    coords, vals = zipf_tensor(dims, nnz, seed=len(name), exponents=law)
    subs = coords.cpu().numpy().astype(np.int64)
    v64 = vals.cpu().numpy().astype(np.float64)
    params = device_params(dims, nnz, R, g=g, **({"m": m} if m else {}))
    st = build_device_sharded(coords, vals, params, check_duplicates=False)
    smap = schedule_super_shards(st.plan, 1)
    rng = np.random.default_rng(3)
    f0 = [rng.random((d, R)).astype(np.float32) for d in dims]
    N = len(dims)
    if fixed:
        for n in range(N):
            out = mttkrp_mode(st, DeviceFactorSet.from_host(f0), n, smap)
            assert_rel(out.double().cpu().numpy(),
                       oracle.reference_mttkrp(subs, v64, [f.astype(np.float64) for f in f0], n),
                       what=f"{name} mode {n}")
    else:
        res = sweep_all_modes(st, DeviceFactorSet.from_host(f0), smap).to_numpy()
        working = [f.astype(np.float64) for f in f0]
        for n in range(N):
            assert_rel(res[n], oracle.reference_mttkrp(subs, v64, working, n), what=f"{name} {n}")
            working[n] = res[n]
    print(f"{name}: ok", flush=True)


def peer_case():
    from paper_2309_09131_b200.peer import PeerShardedTensor
    dims = (3000, 2000, 2500)
    coords, vals = zipf_tensor(dims, 100_000, seed=6, exponents=(1.1,) * 3)
    params = device_params(dims, 100_000, 32, g=4096, m=[16] * 3)
    st = build_device_sharded(coords, vals, params, check_duplicates=False)
    ref = build_device_sharded(coords, vals, params, check_duplicates=False)
    world = 2
    ranks = [PeerShardedTensor(st, world, r, ipc=False) for r in range(world)]
    PeerShardedTensor.connect_local(ranks)
    f0 = DeviceFactorSet.random_device(dims, 32, seed=3)
    working = [list(f0.factors) for _ in range(world)]
    ref_w = list(f0.factors)
    smap = schedule_super_shards(ref.plan, 1)
    for n in range(3):
        outs = [dt.output(n, 32)[0] for dt in ranks]
        for r, dt in enumerate(ranks):
            dt.mode_pass(working[r], n, outs[r])
        for r, dt in enumerate(ranks):
            dt.reduce(n, outs[r])
        ptrs = [o.data_ptr() for o in outs]
        for r, dt in enumerate(ranks):
            dt.pull_rows(n, outs[r], ptrs)
            dt.swap()
            working[r][n] = outs[r]
        ref_w[n] = mttkrp_mode(ref, DeviceFactorSet(ref_w, None, validate=False), n, smap)
        torch.cuda.synchronize()
        for r in range(world):
            assert torch.equal(working[r][n], ref_w[n]), (n, r)
    for dt in ranks:
        dt.check()
    print("peer: ok", flush=True)


def main():
    torch.cuda.set_device(0)
    sweep_case("packed", (1200, 900, 2800), 150_000, (1.1, 1.1, 1.1), 32)
    sweep_case("wide", (1 << 17, 1 << 17, 3000), 150_000, (0.8, 0.8, 1.0), 32, m=[32, 32, 32])
    sweep_case("tile4", (500, 900, 300, 40), 120_000, (1.2,) * 4, 32, fixed=True)
    sweep_case("tileR16", (1000, 800, 600), 100_000, (None, None, None), 16, fixed=True)
    sweep_case("general", (3000, 2000, 1000), 60_000, (1.1, 1.1, 1.1), 32, m=[600, 600, 600])
    sweep_case("direct", (200, 200_000, 300), 80_000, (1.0, 0.5, 1.0), 32, fixed=True)
    sweep_case("heavy", (64, 5000, 5000), 150_000, (None, 1.0, 1.0), 32, g=2048)
    peer_case()
    print("sanitize_case: all ok")


if __name__ == "__main__":
    main()

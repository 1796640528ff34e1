#!/usr/bin/env python
"""Benchmark: all-mode spMTTKRP + dynamic-remap sweep (FLYCOO) on B200.

Default workload = BASELINE.json configs[1] ("c2"): 12092 x 9184 x 28818,
76.9M distinct Zipf(1.1) nonzeros, R = 32, updated-factor sweep
(sweep_all_modes semantics), seeded synthetic data generated on the GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

One JSON line on rank 0.  `value` = N_modes * nnz / t_sweep (nonzero-mode
updates per second, summed over ranks), inputs resident in HBM; `e2e` is
the same metric through the public API with the factors coming from and the
results going back to pinned host memory every step; `roofline` covers the
fused mode-pass kernel (compulsory bytes per SURVEY §8d); `cpu_baseline` is
the CPU port of the reference (oracle/) on a bounded prefix of the same
workload, on this host's cores.  `--impl reference` times that CPU port
alone (the reference arm).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
# the billion-nonzero configs build near the HBM limit: avoid fragmentation
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

METRIC = "all-mode spMTTKRP+remap sweep time & nnz/s at R=32; % HBM roofline; 1/2/4/8 GPU"
UNIT = "nnz/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--nnz", type=int, default=None, help="override nnz (same law)")
    ap.add_argument("--cpu-sample", type=int, default=None,
                    help="nonzeros in the CPU-baseline prefix sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (FileNotFoundError, OSError):
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        for line in Path(self.path).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v == "Active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


# -------------------------------------------------------------- workloads

def workload(cfg_index: int, nnz: int | None):
    from paper_2309_09131_b200.synth import CONFIGS
    cfg = dict(CONFIGS[cfg_index])
    if nnz is not None:
        cfg["nnz"] = int(nnz)
    return cfg


def describe(cfg_index: int, cfg: dict) -> str:
    dims = "x".join(str(d) for d in cfg["dims"])
    law = "uniform" if cfg["law"] is None else "Zipf " + "/".join(
        "u" if s is None else str(s) for s in cfg["law"])
    return (f"c{cfg_index}: {dims}, {cfg['nnz']:,} distinct nonzeros ({law}), R={cfg['rank']}, "
            f"{cfg['semantics']}-factor sweep, fp32 values/factors U(0,1)")


def kernel_name(N: int, dims, rank: int) -> str:
    """The K1 instance the library dispatches for this shape (dispatch.cuh)."""
    if os.environ.get("FLYCOO_KERNEL") in ("warp", "pipe"):
        return f"mode_pass_{os.environ['FLYCOO_KERNEL']}_kernel"
    if N == 3 and rank % 4 == 0 and rank <= 64 and os.environ.get("FLYCOO_PACK") != "0":
        w = [(d - 1).bit_length() for d in dims]
        if all(sum(w) - w[n] <= 32 for n in range(3)):
            return "mode_pass_pack_kernel (8-B sorted records)"
    return "mode_pass_fast_kernel"


def compulsory_bytes(nnz: int, dims, rank: int):
    """Per mode-pass algorithmic bytes: records read + written,
    one uint32 slot read per element, each factor read once, output written
    once: B_n = nnz*(2*(4N+4)+4) + 4R*sum(I_w)."""
    N = len(dims)
    b = nnz * (2 * (4 * N + 4) + 4) + 4 * rank * sum(dims)
    return [b] * N


def cpu_sample(cfg_index: int, cfg: dict, sample: int):
    """First `sample` distinct nonzeros of the workload (a prefix of it:
    the generator keeps the first distinct draws in draw order)."""
    import numpy as np
    from paper_2309_09131_b200.synth import synth_tensor, zipf_tensor_host
    if cfg["law"] is None:
        subs, vals = synth_tensor(cfg["dims"], sample, seed=cfg_index, skew=0.0)
        return subs, vals.astype(np.float32).astype(np.float64)
    subs, vals = zipf_tensor_host(cfg["dims"], sample, seed=cfg_index, exponents=cfg["law"])
    return subs, vals.astype(np.float64)


def cpu_baseline(cfg_index: int, cfg: dict, sample: int, steps: int, warmup: int) -> dict:
    """The reference algorithm's CPU port (oracle/: restated mode_worker with
    one pthread per core, LPT schedule, reference params) timed per sweep."""
    import numpy as np
    import oracle
    from paper_2309_09131_b200.params import select_params
    threads = os.cpu_count() or 1
    subs, vals = cpu_sample(cfg_index, cfg, sample)
    R = cfg["rank"]
    params = select_params(cfg["dims"], len(vals), threads, 32 << 20, R)
    L = oracle.canonical_build(subs, vals, cfg["dims"], params.m, params.k, params.g)
    t = oracle.OracleTensor(L, "reference", nu=threads)
    rng = np.random.Generator(np.random.Philox(1000 + cfg_index))
    f0 = [rng.random((d, R)).astype(np.float32).astype(np.float64) for d in cfg["dims"]]
    N = len(cfg["dims"])

    def sweep():
        if cfg["semantics"] == "updated":
            t.sweep_all_modes(f0)
        else:
            for n in range(N):
                t.mttkrp_mode(f0, n)

    for _ in range(warmup):
        sweep()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        sweep()
        times.append(time.perf_counter() - t0)
    med = statistics.median(times)
    return {"value": N * len(vals) / med, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": (f"first {len(vals):,} distinct nonzeros of the same workload (prefix), "
                       f"reference params select_params(nu={threads}, 32 MiB, R={R}) -> "
                       f"m={list(params.m)}, g={params.g}; median of {steps} sweeps"),
            "ms_per_sweep": med * 1e3}


# ---------------------------------------------------------------- our arm

def run_ours(args, rank, world, local):
    import numpy as np
    import torch
    from paper_2309_09131_b200 import (DeviceFactorSet, build_device_sharded, device_params,
                                       schedule_super_shards, sweep_all_modes)
    from paper_2309_09131_b200.synth import config_tensor

    # FLYCOO_PG_BACKEND=gloo: host-side process group for the p2p exchange
    # (it needs only barriers and handle exchange), which also lets several
    # ranks share one GPU for a functional smoke run -- never a measurement
    backend = os.environ.get("FLYCOO_PG_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1) if backend == "gloo" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        if backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def max_over_ranks(x: float) -> float:
        tt = torch.tensor([x], device="cpu" if backend == "gloo" else dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())
    cfg = workload(args.config, args.nnz)
    N, R, nnz, dims = len(cfg["dims"]), cfg["rank"], cfg["nnz"], cfg["dims"]

    # tensors whose regular generator + build need more than ~80% of HBM
    # (config 5 at 3.6B nonzeros): bucketed generator + lean build, which
    # stay inside the memory of the final layout
    lean = (N == 3 and cfg["law"] is not None
            and nnz * 64 > 0.8 * torch.cuda.get_device_properties(dev).total_memory)
    # FLYCOO_ACC_TILE_BYTES: one accumulator-tile size for every mode (experiments);
    # default: chosen per mode (params._auto_rows)
    tile_env = os.environ.get("FLYCOO_ACC_TILE_BYTES")
    # FLYCOO_SHARD_G: shard size g (experiments; default device_params' 32768)
    g_env = os.environ.get("FLYCOO_SHARD_G")
    params = device_params(dims, nnz, R, acc_tile_bytes=int(tile_env) if tile_env else None,
                           **({"g": int(g_env)} if g_env else {}))
    t0 = time.perf_counter()
    if lean:
        from paper_2309_09131_b200.layout import build_device_sharded_lean
        from paper_2309_09131_b200.synth import zipf_records_bucketed
        rec = zipf_records_bucketed(dims, nnz, seed=args.config, exponents=cfg["law"], device=dev)
    else:
        coords, vals = config_tensor(args.config, device=dev, nnz=nnz)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    if lean:
        st = build_device_sharded_lean(rec, params, device=dev)
        del rec
    else:
        st = build_device_sharded(coords, vals, params, device=dev)
        del coords, vals
    build_s = time.perf_counter() - t0
    smap = schedule_super_shards(st.plan, 1)
    factors = DeviceFactorSet.random(dims, R, seed=1000 + args.config, device=dev)
    updated = cfg["semantics"] == "updated"
    exchange = os.environ.get("FLYCOO_EXCHANGE", "p2p")
    dt = None
    fallback = None  # why the fused peer exchange was not used (N > 1)
    if world > 1:
        # partitioned sweep: every rank builds the same global layout, keeps
        # its slices + static exchange plan, and frees the rest
        # exchange: "p2p" (default) = remap fused with the exchange, records
        # stored into the owners' buffers over NVLink (peer.py); "nccl" =
        # send region + all_to_all_single + unpack (dist.py)
        from paper_2309_09131_b200.dist import (CudaOps, DistShardedTensor, dist_mttkrp_mode,
                                                dist_sweep_all_modes)
        from paper_2309_09131_b200.peer import (PeerShardedTensor, peer_mttkrp_mode,
                                                peer_sweep_all_modes)
        t0 = time.perf_counter()
        if exchange == "p2p":
            # the fused exchange maps every peer's buffers (CUDA IPC over
            # NVLink); if any rank cannot, every rank falls back to NCCL
            try:
                dt = PeerShardedTensor(st, world, rank)
                dt.connect()
                ok = 1
            except Exception as e:  # noqa: BLE001 -- reported, then the NCCL path
                dt, ok, fallback = None, 0, f"{type(e).__name__}: {e}"[:200]
            flag = torch.tensor([ok], device="cpu" if backend == "gloo" else dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if int(flag.item()) == 0:
                if dt is not None:
                    dt.close()
                fallback = fallback or "a peer could not map the IPC buffers"
                print(f"[bench] fused peer exchange unavailable ({fallback}); using NCCL",
                      file=sys.stderr)
                exchange = "nccl"
        if exchange != "p2p":
            dt = DistShardedTensor(st, world, rank)
        plan_s = time.perf_counter() - t0
        del st
        torch.cuda.empty_cache()
        ops = CudaOps()

    # single GPU: the sweep (updated or fixed factors) is replayed as a CUDA graph
    # (graph.py; FLYCOO_GRAPH=0 for eager launches).  Per-mode times come from
    # eager sweeps (the replay is one launch).
    graph = peer_graph = None
    use_graph = os.environ.get("FLYCOO_GRAPH", "1") != "0"
    if dt is None and use_graph:
        from paper_2309_09131_b200.graph import SweepGraph
        graph = SweepGraph(st, factors, smap, updated=updated)
    elif use_graph and updated and exchange == "p2p" and dt.device_sync:
        # multi-GPU: the sweep with its device-side barriers as one graph per GPU
        from paper_2309_09131_b200.peer import PeerSweepGraph
        peer_graph = PeerSweepGraph(dt, list(factors.factors))

    def step(fs, mode_secs=None, eager=False):
        flist = fs.factors if hasattr(fs, "factors") else fs
        if graph is not None and not eager:
            # the timed loop re-runs on the same resident factors (already in
            # the graph's static inputs); other factors are copied in first
            return graph.run(None if fs is factors else fs).factors
        if peer_graph is not None and not eager:
            return peer_graph.run(list(flist))
        if dt is not None and exchange == "p2p":
            if updated:
                return peer_sweep_all_modes(dt, list(flist), mode_seconds=mode_secs)
            outs = [peer_mttkrp_mode(dt, list(flist), n).clone() for n in range(N)]
            dt.check()
            return outs
        if dt is not None:
            if updated:
                return dist_sweep_all_modes(dt, list(flist), ops, mode_seconds=mode_secs)
            outs = [dist_mttkrp_mode(dt, list(flist), n, ops) for n in range(N)]
            ops.check(dt)
            return outs
        if updated:
            return sweep_all_modes(st, fs, smap, mode_seconds=mode_secs).factors
        from paper_2309_09131_b200 import mttkrp_mode
        outs = []
        for n in range(N):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            outs.append(mttkrp_mode(st, fs, n, smap))
            e1.record()
            if mode_secs is not None:
                e1.synchronize()
                mode_secs.append(e0.elapsed_time(e1) / 1e3)
        return outs

    for _ in range(max(args.warmup, 0)):
        step(factors)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    mode_secs = []
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    # inputs that fit in L2 (config 1): flush L2 before every step by writing a
    # buffer 2x its size, outside the per-step events
    resident_bytes = nnz * (4 * N + 4 + 4 * N)
    flush_l2 = resident_bytes < (256 << 20)
    torch.cuda.synchronize()
    if flush_l2:
        scrub = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        t_ms = 0.0
        for _ in range(args.steps):
            scrub.fill_(1)
            ev0.record()
            step(factors, mode_secs)
            ev1.record()
            ev1.synchronize()
            t_ms += ev0.elapsed_time(ev1)
        del scrub
    else:
        ev0.record()
        for _ in range(args.steps):
            step(factors, mode_secs)
        ev1.record()
        torch.cuda.synchronize()
        t_ms = ev0.elapsed_time(ev1)
    clk = clocks.stop()
    if world > 1:
        t_ms = max_over_ranks(t_ms)
    ms_per_step = t_ms / args.steps
    # strong scaling for world > 1: the ranks share one tensor
    value = N * nnz / (ms_per_step / 1e3)
    if graph is not None or peer_graph is not None:  # per-mode times from eager sweeps
        for _ in range(args.steps):
            step(factors, mode_secs, eager=True)

    # dominant kernel: the fused mode pass (K1, plus K2 when a mode reduces);
    # multi-GPU: a rank's share of the compulsory bytes over its mode time
    # (which then also contains the exchange and the all-gather)
    per_mode = compulsory_bytes(nnz, dims, R)
    kern_s = sum(mode_secs)
    basis = "CUDA events around each eager mode pass (K1 + K2)"
    if graph is not None or peer_graph is not None:
        # graph replay: the timed sweeps contain only the passes (K1 + K2), with
        # no host gaps between them -- the tighter live measurement
        kern_s = min(kern_s, t_ms / 1e3)
        basis = "CUDA events around the graph-replayed sweeps (K1 + K2 of every mode)"
    achieved = sum(per_mode) / world * args.steps / kern_s / 1e9
    peak, peak_src = peaks()
    src = dt if dt is not None else st
    # + the unpack (NCCL exchange) or the row gather (fused exchange) per mode
    launches_per_step = sum(src.mode_work(n, R).launches + (1 if dt is not None else 0)
                            for n in range(N))
    traffic = None
    tpath = ROOT / "profiles" / "traffic.json"
    if tpath.exists():
        tj = json.loads(tpath.read_text())
        if tj.get("config") == args.config and tj.get("nnz") == nnz:
            traffic = tj.get("dram_bytes_per_launch")

    # end to end through the public API: pinned host factors in, results out
    e2e = None
    if not args.no_e2e:
        host_in = [f.cpu().pin_memory() for f in factors.factors]
        host_out = [torch.empty(f.shape, dtype=torch.float32).pin_memory() for f in factors.factors]
        if graph is not None:
            # the copies are graph nodes: inputs of mode 0 in (factor 0 is
            # replaced before anything reads it), each updated factor out on a
            # side stream while the later modes run
            graph.bind_host(host_in, host_out)

            def e2e_step():
                graph.run_host()

            h2d, d2h = graph.host_bytes()
            path = ("SweepGraph(DeviceShardedTensor).run_host(): pinned host factors -> sweep -> "
                    "pinned host factors, copies inside the graph")
        else:
            dev_in = [torch.empty_like(f) for f in factors.factors]

            def e2e_step():
                for d_, h_ in zip(dev_in, host_in):
                    d_.copy_(h_, non_blocking=True)
                outs = step(DeviceFactorSet(dev_in, None, dev, validate=False))
                for h_, o_ in zip(host_out, outs):
                    h_.copy_(o_, non_blocking=True)

            h2d = sum(h.numel() * 4 for h in host_in)
            d2h = sum(h.numel() * 4 for h in host_out) if updated else sum(d * R * 4 for d in dims)
            path = ("PeerSweepGraph(PeerShardedTensor).run(factors<-pinned host) -> pinned host"
                    if peer_graph is not None else
                    "peer_sweep_all_modes(PeerShardedTensor, factors<-pinned host) -> pinned host"
                    if dt is not None and exchange == "p2p" else
                    "dist_sweep_all_modes(DistShardedTensor, factors<-pinned host) -> pinned host"
                    if dt is not None else
                    "sweep_all_modes(DeviceShardedTensor, factors<-pinned host) -> pinned host")
        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            e2e_step()
        e1.record()
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1) / args.steps
        if world > 1:
            e_ms = max_over_ranks(e_ms)
        e2e = {"value": N * nnz / (e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e_ms, "path": path}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sample = args.cpu_sample or min(nnz, 8_000_000)
        cpu = cpu_baseline(args.config, cfg, sample, steps=3, warmup=1)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak" if world == 1 else "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": describe(args.config, cfg), "config_index": args.config,
                       "nnz": nnz, "dims": list(dims), "rank": R, "params_m": list(params.m),
                       "params_g": params.g,
                       "l2": ("L2 flushed before every step (256 MB write outside the per-step "
                              f"events): records {nnz * (4 * N + 4) / 1e6:.1f} MB + slots "
                              f"{nnz * 4 * N / 1e6:.1f} MB fit in the 126 MB L2") if flush_l2 else
                             ("inputs larger than L2 (records "
                              f"{nnz * (4 * N + 4) / 1e9:.2f} GB + slots {nnz * 4 * N / 1e9:.2f} GB vs 126 MB L2)"),
                       "parallelism": "1 GPU" if world == 1 else
                       (f"dp{world}: per-mode super-shard row ranges; remap fused with the "
                        "exchange (records stored into the owner GPU's buffer over NVLink peer "
                        "memory, CUDA IPC) + peer pull of updated factor rows"
                        if exchange == "p2p" else
                        f"dp{world}: per-mode super-shard row ranges, NCCL all_to_all_single remap + "
                        "all_gather_into_tensor of updated factor rows"
                        + (f" (fused peer exchange unavailable: {fallback})" if fallback else "")),
                       "gen_s": round(gen_s, 3), "build_s": round(build_s, 3),
                       "build": "lean (bucketed generator, layout.build_device_sharded_lean)" if lean else "regular",
                       "peak_hbm_gb": round(torch.cuda.max_memory_allocated(dev) / 1e9, 2),
                       # median over the measured sweeps of each mode pass
                       "mode_ms": [round(1e3 * statistics.median(mode_secs[n::N]), 4)
                                   for n in range(N)] if mode_secs else []},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": kernel_name(N, dims, R) + " (+ reduce_level_kernel)",
                         "algorithmic_bytes_per_launch": per_mode[0], "peak_source": peak_src,
                         "timing_basis": basis},
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
            "gpu_launches": launches_per_step * args.steps,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------- reference arm

def run_reference(args, rank, world, local):
    """The reference's CPU implementation of the path (oracle/ port, all host
    threads) on a bounded prefix of this arm's workload; rank 0 only."""
    if rank != 0:
        return
    cfg = workload(args.config, args.nnz)
    # bounded sample: 8M nonzeros (~0.5 s per sweep on a 16-core host) up to
    # ~150 sweeps, shrinking beyond that so the reference arm stays ~1-2 min
    budget = int(8_000_000 * 150 / max(args.steps + args.warmup, 150))
    sample = args.cpu_sample or min(cfg["nnz"], max(200_000, budget))
    res = cpu_baseline(args.config, cfg, sample, steps=max(args.steps, 1), warmup=max(args.warmup, 0))
    N = len(cfg["dims"])
    line = {
        "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_sweep"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": describe(args.config, cfg), "config_index": args.config,
                   "sample_nnz": sample},
        "cpu_baseline": {"value": res["value"], "unit": UNIT, "cores": res["cores"],
                         "kind": "port", "sample": res["sample"]},
        "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world, local)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()

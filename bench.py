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

CPU_FULL_MAX = 80_000_000  # whole-workload CPU baseline up to c2's 76.9M nonzeros
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
    """SM clocks and throttle reasons sampled DURING the timed region: NVML
    polled every ~2 ms from a thread (a 20-step c2 run lasts ~75 ms, shorter
    than nvidia-smi's sampling period); nvidia-smi -lms 50 when NVML is not
    available."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = self.thread = self.path = None
        self.nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM)
            self.bits = (pynvml.nvmlClocksEventReasonHwSlowdown,
                         pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                         pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                         pynvml.nvmlClocksEventReasonSwPowerCap)
        except Exception:  # noqa: BLE001 -- fall back to nvidia-smi
            self.nvml = None

    def start(self):
        if self.nvml is not None:
            import threading
            self.stop_flag = threading.Event()

            def poll():
                p = self.nvml
                while not self.stop_flag.is_set():
                    try:
                        mhz = p.nvmlDeviceGetClockInfo(self.handle, p.NVML_CLOCK_SM)
                        r = p.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
                        self.rows.append((float(mhz), float(self.max_mhz),
                                          [("Active" if r & b else "Not Active") for b in self.bits]))
                    except Exception:  # noqa: BLE001
                        pass
                    time.sleep(0.002)
            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (FileNotFoundError, OSError):
            self.proc = None

    def stop(self) -> dict:
        source = "nvml"
        if self.thread is not None:
            self.stop_flag.set()
            self.thread.join()
        elif self.proc is not None:
            source = "nvidia-smi"
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            for line in Path(self.path).read_text().splitlines():
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    self.rows.append((float(parts[1]), float(parts[2]), parts[5:9]))
                except ValueError:
                    continue
            os.unlink(self.path)
        else:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock source"]}
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        reasons = sorted({self.NAMES[i] for _, _, r in rows for i, v in enumerate(r) if v == "Active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows), "source": source}


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


def kernel_names(params, works, rank: int) -> list:
    """The K1 instance the library dispatches for each mode (mode_pass.cu
    dispatch + dispatch.cuh): the general kernel when the accumulator tile is
    not in shared memory or the shape is off the fast path; for 3-mode
    tensors the packed kernel (8-B sorted records when the two input
    coordinates fit 32 bits, else the WIDE {c_w1, c_w2} + value variant);
    otherwise the tile kernel."""
    dims = params.dims
    N = len(dims)
    names = []
    for n in range(N):
        w = works[n]
        fast = (w.acc_in_smem and w.hist_rows <= 256 and 2 <= N <= 4 and rank % 4 == 0
                and rank <= 64)
        if not fast:
            names.append("mode_pass_kernel (general)")
        elif N == 3 and os.environ.get("FLYCOO_PACK") != "0":
            w1, w2 = (1, 2) if n == 0 else (0, 2) if n == 1 else (0, 1)
            b1, b2 = ((dims[w1] - 1).bit_length(), (dims[w2] - 1).bit_length())
            planned = ", tile plan: sorted positions and bin starts read, not ranked" \
                if getattr(w, "tile_perm", None) is not None else ""
            if b2 >= 1 and b1 + b2 <= 32:
                names.append(f"mode_pass_pack_kernel (8-B sorted records{planned})")
            elif os.environ.get("FLYCOO_PACK_WIDE") != "0":
                names.append(f"mode_pass_pack_kernel WIDE ({{c_w1, c_w2}} + value{planned})")
            else:
                names.append("mode_pass_fast_kernel")
        else:
            names.append("mode_pass_fast_kernel")
    return names


def kernel_sources_hash() -> str:
    """sha256 (16 hex) of the CUDA sources: stamps the ncu traffic record so
    a number captured on other kernels is never reported."""
    import hashlib
    h = hashlib.sha256()
    for f in sorted((ROOT / "paper_2309_09131_b200" / "csrc").glob("*.cu*")):
        h.update(f.name.encode())
        h.update(f.read_bytes())
    return h.hexdigest()[:16]


def measured_traffic(cfg_index: int, nnz: int, params) -> tuple:
    """DRAM bytes per mode-pass launch from profiles/traffic.json, only when
    it was captured on these kernel sources and this workload
    (tools/traffic_from_ncu.py writes it); else (None, why)."""
    tpath = ROOT / "profiles" / "traffic.json"
    if not tpath.exists():
        return None, "no profiles/traffic.json"
    tj = json.loads(tpath.read_text())
    want = {"config": cfg_index, "nnz": nnz, "params_m": list(params.m), "params_g": params.g,
            "kernel_sources": kernel_sources_hash()}
    bad = [k for k, v in want.items() if tj.get(k) != v]
    if bad:
        return None, f"profiles/traffic.json does not match this run ({', '.join(bad)})"
    return tj.get("dram_bytes_per_launch"), tj.get("source")


def compulsory_bytes(nnz: int, dims, rank: int):
    """Per mode-pass algorithmic bytes: records read + written,
    one uint32 slot read per element, each factor read once, output written
    once: B_n = nnz*(2*(4N+4)+4) + 4R*sum(I_w)."""
    N = len(dims)
    b = nnz * (2 * (4 * N + 4) + 4) + 4 * rank * sum(dims)
    return [b] * N


def host_tensor(cfg_index: int, cfg: dict, nnz: int):
    """The workload's first `nnz` distinct nonzeros on the host (int64 subs,
    fp32-valued float64 vals): generated on the GPU when there is one (the
    same generator as our arm, copied back), else by its numpy twin
    (synth.zipf_tensor_host / synth_tensor: identical output, tested)."""
    import numpy as np
    import torch
    from paper_2309_09131_b200.synth import config_tensor, synth_tensor, zipf_tensor_host
    if cfg["law"] is None:
        subs, vals = synth_tensor(cfg["dims"], nnz, seed=cfg_index, skew=0.0)
        return subs, vals.astype(np.float32).astype(np.float64)
    if torch.cuda.is_available() and len(cfg["dims"]) <= 4:
        coords, vals = config_tensor(cfg_index, device="cuda", nnz=nnz)
        subs = coords.cpu().numpy().astype(np.int64)
        v = vals.cpu().numpy().astype(np.float64)
        del coords, vals
        torch.cuda.empty_cache()
        return subs, v
    subs, vals = zipf_tensor_host(cfg["dims"], nnz, seed=cfg_index, exponents=cfg["law"])
    return subs, vals.astype(np.float64)


def cpu_baseline(cfg_index: int, cfg: dict, sample: int, steps: int, warmup: int,
                 tensor=None) -> dict:
    """The reference algorithm's CPU port (oracle/: restated mode_worker with
    one pthread per core, LPT schedule, reference params select_params(nu =
    cores, 32 MiB, R) as the reference's run_bench, bench.py:94-160) timed
    per sweep (the reference times the sweep only, bench.py:129-147)."""
    import numpy as np
    import oracle
    from paper_2309_09131_b200.params import select_params
    threads = os.cpu_count() or 1
    subs, vals = tensor if tensor is not None else host_tensor(cfg_index, cfg, sample)
    R = cfg["rank"]
    params = select_params(cfg["dims"], len(vals), threads, 32 << 20, R)
    t0 = time.perf_counter()
    L = oracle.canonical_build(subs, vals, cfg["dims"], params.m, params.k, params.g)
    t = oracle.OracleTensor(L, "reference", nu=threads)
    build_s = time.perf_counter() - t0
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
    whole = len(vals) == cfg["nnz"]
    what = ("the whole workload" if whole else
            f"first {len(vals):,} distinct nonzeros of the workload (prefix)")
    return {"value": N * len(vals) / med, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": (f"{what}; reference params select_params(nu={threads}, 32 MiB, R={R}) -> "
                       f"m={list(params.m)}, g={params.g}; {cfg['semantics']}-factor sweep, "
                       f"median of {steps} sweeps after {warmup} warm-up"),
            "ms_per_sweep": med * 1e3, "nnz": len(vals), "build_s": round(build_s, 2)}


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
    # the CPU baseline runs on the whole workload when it is small enough for
    # the host port (c1, c2: <= 80M nonzeros, ~20 GB of host arrays), else on a
    # bounded prefix of it
    cpu_sample_n = None
    host_copy = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_sample_n = args.cpu_sample or (nnz if nnz <= CPU_FULL_MAX else 8_000_000)
        if cpu_sample_n == nnz and not lean:
            host_copy = (coords.cpu().numpy().astype(np.int64), vals.cpu().numpy().astype(np.float64))
    exchange = os.environ.get("FLYCOO_EXCHANGE", "p2p")
    # N > 1 with the fused exchange: every rank builds only its slices from its
    # block of the input (distbuild.build_partitioned) -- no rank holds the
    # global layout; FLYCOO_GLOBAL_BUILD=1: global build, then sliced
    partitioned = world > 1 and exchange == "p2p" and os.environ.get("FLYCOO_GLOBAL_BUILD") != "1"
    t0 = time.perf_counter()
    st = loc = None
    if partitioned:
        from paper_2309_09131_b200.distbuild import build_partitioned
        lo, hi = nnz * rank // world, nnz * (rank + 1) // world
        if lean:
            bc = rec[lo:hi, :3].clone()
            bv = rec[lo:hi, 3].clone().view(torch.float32)
            del rec
        else:
            bc, bv = coords[lo:hi].clone(), vals[lo:hi].clone()
            del coords, vals
        torch.cuda.empty_cache()
        loc = build_partitioned(bc, bv, lo, params, R=R, device=dev)
        del bc, bv
        torch.cuda.synchronize()
        build_stages = {"partitioned_build": time.perf_counter() - t0}
        plan = loc.plan
    elif lean:
        st = build_device_sharded_lean(rec, params, device=dev)
        del rec
    else:
        # generator output is duplicate-free by construction (first occurrences)
        st = build_device_sharded(coords, vals, params, device=dev, check_duplicates=False)
        del coords, vals
    build_s = time.perf_counter() - t0
    if st is not None:
        build_stages = dict(st.build_stages)
        plan = st.plan
    smap = schedule_super_shards(plan, 1)
    factors = DeviceFactorSet.random_device(dims, R, seed=1000 + args.config, device=dev)
    updated = cfg["semantics"] == "updated"
    dt = None
    fallback = None  # why the fused peer exchange was not used (N > 1)
    if world > 1:
        # partitioned sweep: each rank holds its slices + the static exchange
        # plan (from the per-rank build above, or cut from a global layout)
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
            # NVLink); if any rank cannot, every rank falls back to NCCL.  Two
            # agreements keep the collectives matched: construction (local
            # allocations) first, then the collective connect.
            def agree(ok: int) -> bool:
                flag = torch.tensor([ok], device="cpu" if backend == "gloo" else dev)
                dist.all_reduce(flag, op=dist.ReduceOp.MIN)
                return int(flag.item()) == 1

            try:
                dt = PeerShardedTensor(loc if partitioned else st, world, rank)
            except Exception as e:  # noqa: BLE001 -- reported, then the NCCL path
                dt, fallback = None, f"{type(e).__name__}: {e}"[:200]
            connected = False
            if agree(1 if dt is not None else 0):
                try:
                    dt.connect()
                    connected = True
                except Exception as e:  # noqa: BLE001
                    fallback = f"{type(e).__name__}: {e}"[:200]
                if not agree(1 if connected else 0):
                    connected = False
            if not connected:
                if dt is not None:
                    dt.close()
                    dt = None
                fallback = fallback or "a peer could not map the IPC buffers"
                print(f"[bench] fused peer exchange unavailable ({fallback}); using NCCL",
                      file=sys.stderr)
                exchange = "nccl"
        if exchange != "p2p":
            if st is None:  # the fallback slices a global layout
                coords, vals = config_tensor(args.config, device=dev, nnz=nnz)
                st = build_device_sharded(coords, vals, params, device=dev, check_duplicates=False)
                del coords, vals
            dt = DistShardedTensor(st, world, rank)
        plan_s = time.perf_counter() - t0
        st = loc = None
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
        def timed(fn, n):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            out = fn(n)
            e1.record()
            if mode_secs is not None:
                e1.synchronize()
                mode_secs.append(e0.elapsed_time(e1) / 1e3)
            return out

        if dt is not None and exchange == "p2p":
            if updated:
                return peer_sweep_all_modes(dt, list(flist), mode_seconds=mode_secs)
            outs = [timed(lambda n: peer_mttkrp_mode(dt, list(flist), n).clone(), n)
                    for n in range(N)]
            dt.check()
            return outs
        if dt is not None:
            if updated:
                return dist_sweep_all_modes(dt, list(flist), ops, mode_seconds=mode_secs)
            outs = [timed(lambda n: dist_mttkrp_mode(dt, list(flist), n, ops), n) for n in range(N)]
            ops.check(dt)
            return outs
        if updated:
            return sweep_all_modes(st, fs, smap, mode_seconds=mode_secs).factors
        from paper_2309_09131_b200 import mttkrp_mode
        return [timed(lambda n: mttkrp_mode(st, fs, n, smap), n) for n in range(N)]

    for _ in range(max(args.warmup, 0)):
        step(factors)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    mode_secs = []
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    # inputs that fit in L2 (config 1): flush L2 before every step by writing a
    # buffer 2x its size, outside the per-step events
    resident_bytes = nnz * (4 * N + 4 + 4 * N)
    flush_l2 = resident_bytes < (256 << 20)
    torch.cuda.synchronize()
    clocks.start()  # sampled from here to the end of the timed steps
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
    kern_s = sum(mode_secs) or t_ms / 1e3
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
    traffic, traffic_src = measured_traffic(args.config, nnz, params)
    kernels = kernel_names(params, [src.mode_work(n, R) for n in range(N)], R)

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
    if cpu_sample_n is not None:
        del graph, peer_graph, st, factors
        torch.cuda.empty_cache()
        cpu = cpu_baseline(args.config, cfg, cpu_sample_n, steps=3, warmup=1, tensor=host_copy)
        del host_copy

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
                       # build stages (CUDA events; PAPER.md:762 reports super-shard
                       # generation, Morton ordering and shard generation)
                       "build_stages_s": {k: round(v, 4) for k, v in build_stages.items()},
                       "build": ("partitioned (per-rank slices, distbuild.build_partitioned)"
                                 if partitioned else
                                 "lean (bucketed generator, layout.build_device_sharded_lean)"
                                 if lean else "regular"),
                       "peak_hbm_gb": round(torch.cuda.max_memory_allocated(dev) / 1e9, 2),
                       # static per-tile sort emitted once (engine.build_tile_plans), bytes held
                       "tile_plan_bytes": sum(
                           (w.tile_perm.numel() + w.tile_bins.numel()) * 2
                           for w in (src.mode_work(n, R) for n in range(N))
                           if getattr(w, "tile_perm", None) is not None),
                       # SURVEY 8(d) also asks for nnz / t_sweep (value is N * nnz / t_sweep)
                       "nnz_per_s_sweep": nnz / (ms_per_step / 1e3),
                       # median over the measured sweeps of each mode pass
                       "mode_ms": [round(1e3 * statistics.median(mode_secs[n::N]), 4)
                                   for n in range(N)] if mode_secs else []},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "kernel": "; ".join(f"mode {n}: {k}" for n, k in enumerate(kernels))
                                   + " (+ reduce_level_kernel)",
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
    """The reference's CPU implementation of the path (oracle/ port of the
    numba mode_worker, all host threads, the reference's own parameter
    choice) on this arm's workload -- the whole tensor for c1/c2, a bounded
    prefix for the billion-nonzero configs; rank 0 only."""
    if rank != 0:
        return
    cfg = workload(args.config, args.nnz)
    nnz = cfg["nnz"]
    sample = args.cpu_sample or (nnz if nnz <= CPU_FULL_MAX else 8_000_000)
    res = cpu_baseline(args.config, cfg, sample, steps=max(args.steps, 1),
                       warmup=max(args.warmup, 0))
    N = len(cfg["dims"])
    line = {
        "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_sweep"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        # the same config keys as our arm's line (same workload, whole tensor)
        "config": {"workload": describe(args.config, cfg), "config_index": args.config,
                   "nnz": nnz, "dims": list(cfg["dims"]), "rank": cfg["rank"],
                   "sample_nnz": res["nnz"]},
        "cpu_baseline": {"value": res["value"], "unit": UNIT, "cores": res["cores"],
                         "kind": "port", "sample": res["sample"]},
        "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def self_launch(args) -> int:
    """`python bench.py --gpus N` without torchrun: start N ranks through
    torch.distributed.run on 127.0.0.1 (one process per GPU) and return its
    exit code.  With FLYCOO_PG_BACKEND=gloo and fewer GPUs than ranks, ranks
    share GPUs (functional runs only; host barriers, never a measurement)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    try:
        import torch
        ngpu = torch.cuda.device_count()
    except Exception:  # noqa: BLE001
        ngpu = 0
    if ngpu < args.gpus:
        if env.get("FLYCOO_PG_BACKEND") != "gloo":
            print(f"[bench] --gpus {args.gpus} but {ngpu} GPU(s) visible (set "
                  "FLYCOO_PG_BACKEND=gloo for a functional run with shared GPUs)", file=sys.stderr)
            return 2
        env.setdefault("FLYCOO_PEER_SYNC", "host")  # ranks on one GPU never wait on each other
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    rank, world, local = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(self_launch(args))
    if world != args.gpus:
        sys.exit(f"[bench] --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, rank, world, local)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()

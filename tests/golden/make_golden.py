"""Generate the golden fixtures that pin the oracle to the reference.

Run HERE (the container that has /root/reference); the GPU box never runs it.
It imports the reference package read-only and records, for small seeded
cases, everything the hot path is defined by:

* ``select_params`` outputs for the five BASELINE config shapes and a grid of
  (nu, gamma, rank, g_range) choices (layout.py:247-318);
* ``morton.interleave`` keys (morton.py:20-44);
* ``build_sharded`` layouts: plan arrays, the mode-0 active buffer, slot maps
  (layout.py:462-531);
* per-mode ``mttkrp_mode`` outputs under fixed factors and the remapped active
  buffer after every mode, for both remap strategies' deterministic one
  ("slot"; engine.py:163-266);
* ``sweep_all_modes`` results (engine.py:269-293);
* ``reference_mttkrp`` outputs (coo.py:406-426);
* a digest of ``synth_tensor`` for config 1 (coo.py:323-355), which the
  package's uniform generator restates;
* ``cp_als`` fit histories, factors and ``fit`` (cpals.py:102-188).

Usage:  NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_golden.py
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import modecycle as mc  # noqa: E402
from modecycle import morton  # noqa: E402

OUT = Path(__file__).resolve().parent


def small_coo(seed: int, dims, nnz: int):
    """Distinct coordinates, draw order kept (first occurrence), PCG64."""
    rng = np.random.Generator(np.random.PCG64(seed))
    draws = rng.integers(0, dims, size=(nnz * 4, len(dims)))
    _, first = np.unique(draws, axis=0, return_index=True)
    keep = np.sort(first)[:nnz]
    subs = draws[keep]
    vals = rng.uniform(0.25, 2.0, size=subs.shape[0])
    # fp32-representable values, the same numbers the GPU path holds
    vals = vals.astype(np.float32).astype(np.float64)
    return mc.CooTensor(tuple(dims), subs, vals)


def fp32_factors(dims, rank, seed):
    fs = mc.FactorSet.random(dims, rank, seed)
    return mc.FactorSet(tuple(f.astype(np.float32).astype(np.float64) for f in fs.factors),
                        fs.lambdas)


def params_dict(p) -> dict:
    return {"dims": list(p.dims), "nnz": p.nnz, "m": list(p.m), "k": list(p.k),
            "g": p.g, "nu": p.nu, "gamma": p.gamma, "theta": p.theta,
            "rank": p.rank, "alpha": p.alpha, "beta": p.beta, "sigma": p.sigma,
            "eq2_exact": list(p.eq2_exact)}


def golden_params():
    shapes = {
        "c1": ((1000, 800, 600), 1_000_000),
        "c2": ((12092, 9184, 28818), 76_900_000),
        "c3": ((532924, 17262471, 2480308, 1443), 140_000_000),
        "c4": ((4821207, 1774269, 1805187), 1_740_000_000),
        "c5": ((46, 239172, 239172), 3_600_000_000),
        "tiny": ((5, 7, 3), 40),
        "ragged": ((1000, 999, 17), 5000),
    }
    grid = [
        dict(nu=1, gamma=32 << 20, rank=16),
        dict(nu=2, gamma=32 << 20, rank=16),
        dict(nu=8, gamma=32 << 20, rank=32),
        dict(nu=8, gamma=300 << 20, rank=32),
        dict(nu=148, gamma=126 << 20, rank=32),
        dict(nu=7, gamma=1 << 30, rank=8, g_range=(4, 64)),
        dict(nu=3, gamma=4 << 20, rank=32, alpha=4, beta=16, sigma=4),
    ]
    out = []
    for name, (dims, nnz) in shapes.items():
        for kw in grid:
            rec = {"shape": name, "dims": list(dims), "nnz": nnz, "kw": {
                k: (list(v) if isinstance(v, tuple) else v) for k, v in kw.items()}}
            try:
                p = mc.select_params(dims, nnz, **kw)
                rec["params"] = params_dict(p)
            except mc.InfeasibleParamsError as exc:
                rec["infeasible"] = str(exc)
            out.append(rec)
    (OUT / "select_params.json").write_text(json.dumps(out, indent=1))


def golden_morton():
    rng = np.random.Generator(np.random.PCG64(11))
    cases = {}
    for ci, counts in enumerate([(5, 7, 3), (1, 1, 9), (1024, 3, 77, 2),
                                 (70000, 60000, 50000), (1 << 30, 1 << 30, 1 << 25, 1 << 20)]):
        coords = np.stack([rng.integers(0, c, size=500) for c in counts], axis=1)
        hi, lo = morton.interleave(coords, counts)
        cases[f"m{ci}_coords"] = coords.astype(np.int64)
        cases[f"m{ci}_counts"] = np.asarray(counts, dtype=np.int64)
        cases[f"m{ci}_hi"] = hi
        cases[f"m{ci}_lo"] = lo
    np.savez_compressed(OUT / "morton.npz", **cases)


LAYOUT_CASES = [
    # name, dims, nnz, seed, params kwargs (select_params), rank
    ("n3_small", (30, 40, 50), 2000, 1, dict(nu=4, gamma=1 << 20, g_range=(16, 256)), 8),
    ("n4_small", (9, 11, 7, 13), 1500, 2, dict(nu=3, gamma=1 << 20, g_range=(8, 128)), 5),
    ("n2_small", (60, 45), 900, 3, dict(nu=2, gamma=1 << 18, g_range=(16, 64)), 4),
    ("n3_ragged", (1000, 37, 5), 3000, 4, dict(nu=2, gamma=32 << 20, g_range=(64, 512)), 16),
    ("n3_skew", (200, 150, 100), 20000, 7, None, 8),
    ("n5_small", (6, 5, 7, 4, 6), 700, 5, dict(nu=2, gamma=1 << 20, g_range=(8, 64)), 3),
    ("n3_one", (5, 6, 7), 1, 6, dict(nu=1, gamma=1 << 20, g_range=(4, 8)), 4),
]


def golden_layouts():
    for name, dims, nnz, seed, kw, rank in LAYOUT_CASES:
        if name == "n3_skew":
            t = mc.synth_tensor(dims, nnz, seed=seed, skew=0.5)
            t = mc.CooTensor(t.dims, t.subs, t.vals.astype(np.float32).astype(np.float64))
            params = mc.select_params(t.dims, t.nnz, 4, 32 << 20, rank, g_range=(64, 1024))
        else:
            t = small_coo(seed, dims, nnz)
            params = mc.select_params(t.dims, t.nnz, rank=rank, **kw)
        st = mc.build_sharded(t, params)
        plan = st.plan
        N = t.num_modes
        rec = {
            "subs": t.subs, "vals": t.vals, "dims": np.asarray(t.dims),
            "m": np.asarray(params.m), "k": np.asarray(params.k),
            "g": np.asarray(params.g), "rank": np.asarray(rank),
            "nu": np.asarray(params.nu),
        }
        for n in range(N):
            rec[f"ss_counts{n}"] = plan.ss_counts[n]
            rec[f"ss_elem_offsets{n}"] = plan.ss_elem_offsets[n]
            rec[f"ss_shard_counts{n}"] = plan.ss_shard_counts[n]
            rec[f"ss_first_shard{n}"] = plan.ss_first_shard[n]
            rec[f"shard_offsets{n}"] = plan.shard_offsets[n]
            rec[f"slot_map{n}"] = st.slot_maps[n]
        s, i, v = st.active_arrays()
        rec["sids0"], rec["idxs0"], rec["vals0"] = s.copy(), i.copy(), v.copy()

        fs = fp32_factors(t.dims, rank, seed + 100)
        for n in range(N):
            rec[f"factor{n}"] = fs.factors[n]
            rec[f"ref_mttkrp{n}"] = mc.reference_mttkrp(t, fs, n)
        # fixed-factor mode loop: engine output + remapped buffers per mode
        smap = mc.schedule_super_shards(plan, params.nu)
        counters = mc.TrafficCounters()
        for n in range(N):
            out = mc.mttkrp_mode(st, fs, n, smap, remap="slot", counters=counters)
            rec[f"engine_mttkrp{n}"] = out
            s, i, v = st.active_arrays()
            rec[f"after{n}_sids"], rec[f"after{n}_idxs"], rec[f"after{n}_vals"] = (
                s.copy(), i.copy(), v.copy())
        rec["counters"] = np.asarray([counters.tensor_bytes_read, counters.factor_bytes_read,
                                      counters.output_bytes_written,
                                      counters.remap_bytes_written], dtype=np.int64)
        # updated-factor sweep (engine.py:269-293), fresh build
        st2 = mc.build_sharded(t, params)
        res = mc.sweep_all_modes(st2, fs, smap, remap="slot")
        for n in range(N):
            rec[f"sweep{n}"] = res.factors[n]
        np.savez_compressed(OUT / f"layout_{name}.npz", **rec)


def golden_synth():
    t = mc.synth_tensor((1000, 800, 600), 1_000_000, seed=1, skew=0.0)
    d = {
        "subs_sha256": hashlib.sha256(np.ascontiguousarray(t.subs, dtype="<i8").tobytes()).hexdigest(),
        "vals_sha256": hashlib.sha256(np.ascontiguousarray(t.vals, dtype="<f8").tobytes()).hexdigest(),
        "head_subs": t.subs[:8].tolist(),
        "head_vals": [float(x) for x in t.vals[:8]],
    }
    small = mc.synth_tensor((50, 40, 30), 3000, seed=5, skew=0.0)
    np.savez_compressed(OUT / "synth_small.npz", subs=small.subs, vals=small.vals)
    (OUT / "synth_c1.json").write_text(json.dumps(d, indent=1))


def golden_schedule():
    rng = np.random.Generator(np.random.PCG64(3))
    out = []
    for trial in range(6):
        k = int(rng.integers(1, 40))
        counts = [int(x) for x in rng.integers(0, 50, size=k)]
        for nu in (1, 2, 3, 8):
            out.append({"counts": counts, "nu": nu,
                        "assign": [list(x) for x in mc.schedule._greedy(counts, nu)]})
    (OUT / "schedule.json").write_text(json.dumps(out))




def golden_cpals():
    """cp_als (cpals.py:123-188) on two small tensors; fp32-representable
    values so the device run starts from the same numbers."""
    out = {}
    for name, dims, nnz, seed, rank, iters in (("a", (30, 40, 50), 3000, 21, 4, 8),
                                               ("b", (9, 11, 7, 13), 800, 22, 3, 6)):
        t = small_coo(seed, dims, nnz)
        cfg = mc.CpalsConfig(rank=rank, max_iters=iters, tol=1e-12, seed=seed, nu=2,
                             gamma=1 << 20, g_range=(16, 256))
        res = mc.cp_als(t, cfg)
        out[f"{name}_subs"] = t.subs
        out[f"{name}_vals"] = t.vals
        out[f"{name}_dims"] = np.asarray(dims)
        out[f"{name}_cfg"] = np.asarray([rank, iters, seed])
        out[f"{name}_fit"] = np.asarray(res.fit_history)
        out[f"{name}_lambdas"] = res.factors.lambdas
        for n, f in enumerate(res.factors.factors):
            out[f"{name}_factor{n}"] = f
        out[f"{name}_fit_fn"] = np.asarray([mc.fit(t, res.factors)])
    np.savez_compressed(OUT / "cpals.npz", **out)


def golden_io():
    """MCFD factor dump bytes (coo.py:433-447) and FROSTT parse/write
    (coo.py:212-316)."""
    fs = mc.FactorSet.random((5, 7, 3), 4, seed=2)
    fs = mc.FactorSet(fs.factors, np.array([1.0, 2.0, 0.5, 3.0]))
    (OUT / "mcfd_small.bin").write_bytes(mc.save_factor_set(fs, None))
    t = mc.synth_tensor((6, 5, 4), 40, seed=3, skew=0.4)
    (OUT / "frostt_small.tns").write_text(mc.write_frostt(t))
    t2 = mc.parse_frostt("# comment\n1 1 1 1.5\n2 3 1 2.0\n1 1 1 0.25\n\n3 2 2 -1\n")
    np.savez_compressed(OUT / "frostt_parse.npz", subs=t2.subs, vals=t2.vals,
                        dims=np.asarray(t2.dims), synth_subs=t.subs, synth_vals=t.vals)


def golden_boundary():
    """The reference-facing call shapes: FactorSet.random
    streams (coo.py:184-192); CooTensor validation errors (coo.py:65-89);
    validate_plan's check list on a fresh build (layout.py:565-640); and the
    reference's own call sequence select_params -> build_sharded(tensor,
    params) -> schedule_super_shards -> sweep_all_modes(st,
    FactorSet.random(dims, R, seed), smap) (bench.py:119-134)."""
    out = {}
    for i, (dims, rank, seed) in enumerate([((5, 7, 3), 4, 2), ((40, 30, 20, 10), 8, 11),
                                            ((1000, 800, 600), 16, 1001)]):
        fs = mc.FactorSet.random(dims, rank, seed)
        out[f"rand{i}_dims"] = np.asarray(dims)
        out[f"rand{i}_rank"] = np.asarray(rank)
        out[f"rand{i}_seed"] = np.asarray(seed)
        for n, f in enumerate(fs.factors):
            out[f"rand{i}_f{n}"] = f
    errors = {}
    for name, (dims, subs, vals) in {
        "one_mode": ((5,), [[1]], [1.0]),
        "zero_dim": ((5, 0), [[1, 0]], [1.0]),
        "empty": ((5, 4), np.zeros((0, 2), np.int64), np.zeros(0)),
        "misaligned": ((5, 4), [[1, 1], [2, 2]], [1.0]),
        "nonfinite": ((5, 4), [[1, 1]], [np.inf]),
        "negative": ((5, 4), [[-1, 1]], [1.0]),
        "out_of_range": ((5, 4), [[5, 1]], [1.0]),
        "duplicate": ((5, 4), [[1, 1], [2, 2], [1, 1]], [1.0, 2.0, 3.0]),
    }.items():
        try:
            mc.CooTensor(dims, subs, vals)
            errors[name] = ""
        except ValueError as e:
            errors[name] = str(e)
    out["coo_errors"] = np.asarray(json.dumps(errors))
    t = mc.synth_tensor((60, 50, 40), 20_000, seed=9, skew=0.5)
    params = mc.select_params(t.dims, t.nnz, 4, 1 << 16, 16, g_range=(64, 1024))
    st = mc.build_sharded(t, params)
    smap = mc.schedule_super_shards(st.plan, 4)
    report = mc.validate_plan(st, t)
    out["validate_names"] = np.asarray(json.dumps([c.name for c in report.checks]))
    out["validate_passed"] = np.asarray([c.passed for c in report.checks])
    fs = mc.FactorSet.random(t.dims, 16, 77)
    res = mc.sweep_all_modes(st, fs, smap, remap="slot")
    out["seq_subs"] = t.subs
    out["seq_vals"] = t.vals
    out["seq_m"] = np.asarray(params.m)
    out["seq_g"] = np.asarray(params.g)
    for n, f in enumerate(res.factors):
        out[f"seq_out{n}"] = f
    np.savez_compressed(OUT / "boundary.npz", **out)


if __name__ == "__main__":
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nc")
    only = os.environ.get("GOLDEN_ONLY")  # e.g. GOLDEN_ONLY=cpals regenerates one fixture
    if only:
        globals()[f"golden_{only}"]()
        sys.exit(0)
    golden_params()
    golden_morton()
    golden_layouts()
    golden_synth()
    golden_schedule()
    golden_cpals()
    golden_io()
    golden_boundary()
    print("golden fixtures written to", OUT)

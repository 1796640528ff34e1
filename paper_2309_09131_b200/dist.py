"""Multi-GPU FLYCOO sweep: one process per GPU, NCCL over NVLink.

Per mode n, rank p owns a contiguous range of super-shards [a_p, b_p) --
rows are never split across GPUs -- chosen by a prefix-sum split of the
super-shard fills (layout.py:487-488).  Because the super-shards of a mode
are contiguous in the mode-n order, rank p holds the contiguous slice
[E_p, E_{p+1}) of the single-GPU mode-n buffer, in the same order.

The remap is the only exchange.  Everything about it is static (the layout
and the slot maps are), so it is planned once:

* element i of p's slice goes to global mode-(n+1) position d = slot_n[i];
  its owner q and local position l = d - E'_q follow from the mode-(n+1)
  ranges;
* the local K1 pass writes local destinations straight into the back
  buffer and remote ones into a send region appended to it, grouped by
  destination rank and ordered by l -- so ``local_slots`` is just another
  slot map, into [0, cap + send_total);
* ``all_to_all_single`` (NCCL) moves the send region; the receiver places
  the k-th received record at ``recv_map[k]`` (fc_scatter_records);
* the updated factor rows (owned row range) are all-gathered
  (padded ``all_gather_into_tensor``).

After every mode each rank's slice equals the single-GPU buffer's slice
bit-exactly (tests/test_dist.py checks the plan and the exchange on CPU with
gloo against the single-process layout); outputs equal the 1-GPU outputs up
to fp32 reassociation where merged small-super-shard chunks are grouped
differently at rank boundaries.

Data movement is parameterised by an ``ops`` object: :class:`CudaOps`
(libflycoo kernels, the product path) or a torch emulation in the tests.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .layout import DeviceShardedTensor, PartitionPlan, make_mode_work, plan_chunk_elems

__all__ = ["partition_super_shards", "RankModePlan", "build_rank_plans", "DistShardedTensor",
           "CudaOps", "dist_sweep_all_modes"]


def partition_super_shards(ss_counts, world: int):
    """Split super-shards into `world` contiguous ranges of ~equal element
    count (never splitting a super-shard).  Returns (ss_bounds, elem_bounds),
    each of length world + 1."""
    counts = np.asarray(ss_counts, dtype=np.int64)
    cum = np.concatenate(([0], np.cumsum(counts)))
    total = int(cum[-1])
    k = counts.shape[0]
    sb = [0]
    for p in range(1, world):
        target = p * total / world
        s = int(np.searchsorted(cum, target, side="left"))
        s = min(max(s, 1), k)
        if s > 0 and abs(cum[s - 1] - target) <= abs(cum[s] - target):
            s -= 1
        sb.append(max(s, sb[-1]))
    sb.append(k)
    sb = np.asarray(sb, dtype=np.int64)
    return sb, cum[sb]


@dataclass
class RankModePlan:
    ss_lo: int
    ss_hi: int
    e_lo: int
    e_hi: int
    local_slots: torch.Tensor   # int32 (uint32 bits), into [0, cap + send_total)
    send_counts: list
    recv_counts: list
    recv_map: torch.Tensor      # int32, local mode-(n+1) positions of received records

    @property
    def count(self) -> int:
        return self.e_hi - self.e_lo

    @property
    def send_total(self) -> int:
        return int(sum(self.send_counts))

    @property
    def recv_total(self) -> int:
        return int(sum(self.recv_counts))


def build_rank_plans(plan: PartitionPlan, slot_maps, world: int, rank: int, cap: int | None = None):
    """Per-mode static exchange plan of `rank` (torch ops; CPU or CUDA
    tensors).  `slot_maps` are the single-GPU slot maps (uint32 bits in
    int32/int64 tensors).  Returns (plans, bounds, cap)."""
    N = plan.num_modes
    bounds = [partition_super_shards(plan.ss_counts[n], world) for n in range(N)]
    if cap is None:
        cap = max(int(bounds[n][1][p + 1] - bounds[n][1][p]) for n in range(N) for p in range(world))
    plans = []
    for n in range(N):
        nxt = (n + 1) % N
        sb, eb = bounds[n]
        ebn = torch.as_tensor(bounds[nxt][1], dtype=torch.int64, device=slot_maps[n].device)
        full = slot_maps[n].to(torch.int64) & 0xFFFFFFFF
        lo, hi = int(eb[rank]), int(eb[rank + 1])
        d = full[lo:hi]
        q = torch.searchsorted(ebn, d, right=True) - 1
        l = d - ebn[q]
        remote = q != rank
        key = torch.where(remote, q * (1 << 32) + l, torch.full_like(d, -1))
        order = torch.argsort(key, stable=True)
        nloc = int((~remote).sum())
        pos = torch.empty_like(d)
        pos[order] = torch.arange(d.numel(), device=d.device) - nloc  # remotes sort after locals
        local_slots = torch.where(remote, cap + pos, l).to(torch.int64)
        send_counts = torch.bincount(q[remote], minlength=world).cpu().tolist()
        # receiver side: records of every other rank's slice whose owner is me
        elo, ehi = int(ebn[rank]), int(ebn[rank + 1])
        mine = (full >= elo) & (full < ehi)
        gpos = torch.nonzero(mine).squeeze(1)
        ebt = torch.as_tensor(eb, dtype=torch.int64, device=d.device)
        src = torch.searchsorted(ebt, gpos, right=True) - 1
        lr = full[gpos] - elo
        keep = src != rank
        src, lr = src[keep], lr[keep]
        o = torch.argsort(src * (1 << 32) + lr, stable=True)
        recv_map = lr[o]
        recv_counts = torch.bincount(src, minlength=world).cpu().tolist()
        plans.append(RankModePlan(int(sb[rank]), int(sb[rank + 1]), lo, hi,
                                  local_slots.to(torch.int32), send_counts, recv_counts,
                                  recv_map.to(torch.int32)))
    return plans, bounds, cap


def _local_plan(plan: PartitionPlan, mode: int, p: RankModePlan) -> PartitionPlan:
    """View of the global plan restricted to rank-owned super-shards of one
    mode (element offsets rebased to the local slice)."""
    counts = list(plan.ss_counts)
    offs = list(plan.ss_elem_offsets)
    c = np.zeros_like(plan.ss_counts[mode])
    c[p.ss_lo:p.ss_hi] = plan.ss_counts[mode][p.ss_lo:p.ss_hi]
    counts[mode] = c
    offs[mode] = np.concatenate(([0], np.cumsum(c))).astype(np.int64)
    params = plan.params
    from .params import PartitionParams
    local_params = PartitionParams(dims=params.dims, nnz=p.count, m=params.m, k=params.k,
                                   g=params.g, nu=params.nu, gamma=params.gamma,
                                   theta=params.theta, rank=params.rank, alpha=params.alpha,
                                   beta=params.beta, sigma=params.sigma)
    return PartitionPlan(local_params, tuple(counts), tuple(offs), plan.ss_shard_counts,
                         plan.ss_first_shard, plan.shard_offsets)


class DistShardedTensor:
    """Rank-local slice of a FLYCOO tensor plus its static exchange plan."""

    def __init__(self, st: DeviceShardedTensor, world: int, rank: int, group=None):
        self.plan = st.plan
        self.world, self.rank, self.group = world, rank, group
        self.device = st.device
        self.num_modes = st.num_modes
        self.plans, self.bounds, self.cap = build_rank_plans(st.plan, st.slot_maps, world, rank)
        send_cap = max(max(p.send_total for p in self.plans), 1)
        recv_cap = max(max(p.recv_total for p in self.plans), 1)
        cw = st.crd[0].shape[1]
        emb = st.val[0] is None
        total = self.cap + send_cap
        self.crd = [torch.zeros((total, cw), dtype=torch.int32, device=self.device) for _ in range(2)]
        self.val = [None, None] if emb else [torch.zeros(total, dtype=torch.float32, device=self.device)
                                            for _ in range(2)]
        self.recv_crd = torch.zeros((recv_cap, cw), dtype=torch.int32, device=self.device)
        self.recv_val = None if emb else torch.zeros(recv_cap, dtype=torch.float32, device=self.device)
        p0 = self.plans[0]
        self.crd[0][:p0.count] = st.crd[st.active][p0.e_lo:p0.e_hi]
        if not emb:
            self.val[0][:p0.count] = st.val[st.active][p0.e_lo:p0.e_hi]
        self.active = 0
        self.active_mode = 0
        self._work = {}
        self._stat = torch.zeros(2, dtype=torch.int64, device=self.device)
        self._expected = 0

    def local_records(self):
        p = self.plans[self.active_mode]
        c = self.crd[self.active][:p.count]
        v = None if self.val[self.active] is None else self.val[self.active][:p.count]
        return c, v

    def mode_work(self, mode: int, rank_r: int):
        key = (mode, rank_r)
        if key not in self._work:
            lp = _local_plan(self.plan, mode, self.plans[mode])
            # same chunking as the single-GPU plan -> bitwise-identical sums
            p = self.plans[mode]
            self._work[key] = make_mode_work(lp, mode, rank_r, self.device,
                                             chunk_elems=plan_chunk_elems(self.plan, mode, rank_r),
                                             ss_range=(p.ss_lo, p.ss_hi))
        return self._work[key]

    def owned_rows(self, mode: int):
        p = self.plans[mode]
        m = self.plan.params.m[mode]
        dim = self.plan.params.dims[mode]
        return min(p.ss_lo * m, dim), min(p.ss_hi * m, dim)

    def stat_ptrs(self):
        base = self._stat.data_ptr()
        return base + 8, base


class CudaOps:
    """Local data movement through libflycoo (the product path)."""

    def mode_pass(self, dt: DistShardedTensor, factors, mode: int, out: torch.Tensor):
        p = dt.plans[mode]
        R = int(out.shape[1])
        w = dt.mode_work(mode, R)
        a, b = dt.active, 1 - dt.active
        fptrs = _lib.ptr_array([f.data_ptr() for f in factors])
        flags_p, proc_p = dt.stat_ptrs()
        vp = lambda t: t.data_ptr() if t is not None else None
        params = dt.plan.params
        _lib.call("fc_mode_worker", dt.crd[a].data_ptr(), vp(dt.val[a]), dt.crd[b].data_ptr(),
                  vp(dt.val[b]), fptrs, _lib.i64_array(params.dims), out.data_ptr(), dt.num_modes, mode, R, params.dims[mode],
                  params.m[mode], w.chunk_start.data_ptr(), w.chunk_ss.data_ptr(),
                  w.chunk_part.data_ptr(),
                  w.chunk_rows.data_ptr() if w.chunk_rows is not None else None, w.tile_rows, w.hist_rows, w.nchunks, w.red1.data_ptr(), w.nred1, w.red2.data_ptr(),
                  w.nred2, vp(w.part_ws), vp(w.part_ws2), p.local_slots.data_ptr(),
                  dt.cap + p.send_total, 1, 1, int(w.acc_in_smem), flags_p, proc_p,
                  torch.cuda.current_stream().cuda_stream)
        dt._expected += p.count

    def scatter(self, dt: DistShardedTensor, mode: int):
        p = dt.plans[mode]
        b = 1 - dt.active
        flags_p, proc_p = dt.stat_ptrs()
        vp = lambda t: t.data_ptr() if t is not None else None
        _lib.call("fc_scatter_records", dt.recv_crd.data_ptr(), vp(dt.recv_val), p.recv_total,
                  dt.crd[b].data_ptr(), vp(dt.val[b]), dt.cap, p.recv_map.data_ptr(),
                  dt.num_modes, flags_p, proc_p, torch.cuda.current_stream().cuda_stream)
        dt._expected += p.recv_total

    def exchange(self, dt: DistShardedTensor, mode: int):
        exchange(dt, mode)

    def allgather(self, dt: DistShardedTensor, mode: int, out: torch.Tensor) -> torch.Tensor:
        return allgather_rows(dt, mode, out)

    def check(self, dt: DistShardedTensor):
        stat = dt._stat.cpu()
        flags = int(stat[1]) & 0xFFFFFFFF
        processed, expected = int(stat[0]), dt._expected
        dt._stat.zero_()
        dt._expected = 0
        if processed != expected or flags:
            raise RuntimeError(f"distributed mode pass failed: processed {processed} of "
                               f"{expected}, flags {flags:#x}")


def exchange(dt: DistShardedTensor, mode: int):
    """all_to_all_single of the send region into the receive buffer."""
    p = dt.plans[mode]
    b = 1 - dt.active
    send = dt.crd[b][dt.cap:dt.cap + p.send_total]
    recv = dt.recv_crd[:p.recv_total]
    dist.all_to_all_single(recv, send, p.recv_counts, p.send_counts, group=dt.group)
    if dt.val[b] is not None:
        dist.all_to_all_single(dt.recv_val[:p.recv_total], dt.val[b][dt.cap:dt.cap + p.send_total],
                               p.recv_counts, p.send_counts, group=dt.group)


def allgather_rows(dt: DistShardedTensor, mode: int, out: torch.Tensor) -> torch.Tensor:
    """Assemble the full updated factor from every rank's owned row range."""
    ranges = [(min(int(dt.bounds[mode][0][r]) * dt.plan.params.m[mode], out.shape[0]),
               min(int(dt.bounds[mode][0][r + 1]) * dt.plan.params.m[mode], out.shape[0]))
              for r in range(dt.world)]
    width = max(max(h - l for l, h in ranges), 1)
    lo, hi = ranges[dt.rank]
    block = torch.zeros((width, out.shape[1]), dtype=out.dtype, device=out.device)
    block[:hi - lo] = out[lo:hi]
    gathered = torch.empty((dt.world * width, out.shape[1]), dtype=out.dtype, device=out.device)
    dist.all_gather_into_tensor(gathered, block, group=dt.group)
    full = torch.empty_like(out)
    for r, (l, h) in enumerate(ranges):
        full[l:h] = gathered[r * width:r * width + (h - l)]
    return full


def dist_mttkrp_mode(dt: DistShardedTensor, factors, mode: int, ops=None) -> torch.Tensor:
    """One distributed mode pass: local K1 (+ remote records to the send
    region), exchange, scatter, swap.  Returns the rank's output with only
    its owned rows valid."""
    ops = ops or CudaOps()
    if dt.active_mode != mode:
        raise ValueError(f"active mode is {dt.active_mode}, not {mode}")
    R = int(factors[0].shape[1])
    out = torch.zeros((dt.plan.params.dims[mode], R), dtype=torch.float32, device=dt.device)
    ops.mode_pass(dt, factors, mode, out)
    (ops.exchange if hasattr(ops, "exchange") else exchange)(dt, mode)
    ops.scatter(dt, mode)
    dt.active = 1 - dt.active
    dt.active_mode = (mode + 1) % dt.num_modes
    return out


def dist_sweep_all_modes(dt: DistShardedTensor, factors, ops=None, mode_seconds=None):
    """engine.sweep_all_modes across ranks: factor n is replaced (on every
    rank) by the all-gathered output of mode n."""
    ops = ops or CudaOps()
    working = list(factors)
    events = []
    for n in range(dt.num_modes):
        if mode_seconds is not None and dt.device.type == "cuda":
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record()
        out = dist_mttkrp_mode(dt, working, n, ops)
        working[n] = (ops.allgather if hasattr(ops, "allgather") else allgather_rows)(dt, n, out)
        if mode_seconds is not None and dt.device.type == "cuda":
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record()
            events.append((e0, e1))
    if hasattr(ops, "check"):
        ops.check(dt)
    if events:
        torch.cuda.current_stream().synchronize()
        mode_seconds.extend(a.elapsed_time(b) / 1e3 for a, b in events)
    return working

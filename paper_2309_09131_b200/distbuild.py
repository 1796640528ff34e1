"""Per-rank FLYCOO build for the multi-GPU sweep: every rank
holds a contiguous block of the input COO and ends with exactly what its GPU
runs -- the records of its mode-0 slice and the global slot maps of its slice
of every mode -- without any rank ever holding the whole layout (c5: 158 GB
on one GPU).  The result is bit-identical to slicing the single-GPU build
(layout.build_device_sharded: the reference's shard assignment,
layout.py:474-497, with the B200 intra-shard order); tests/test_distbuild.py
checks it against the oracle's restatement on CPU ranks (gloo).

Steps (P ranks, element e with global input position gid(e)):

1. plan: per-mode super-shard histograms, all-reduced (layout.py:487-497);
   every rank derives the same PartitionPlan and the same per-mode slice
   bounds of the fused exchange (peer.slice_bounds).
2. canonical shard ids, per mode n: a sample sort of the elements on the
   canonical order (iv_n, Morton, gid) -- lexsort(seq, lo, hi, iv_n),
   layout.py:484: elements travel to the rank owning their range of a
   monotone route key (iv_n, leading Morton bits; splitters from an
   all-gathered sample, so a Zipf-heavy super-shard -- c5 mode 0 has two --
   is spread over ranks), which orders them with three stable sorts (they
   arrive in gid order); position = the rank's global offset (exclusive scan
   of the received counts) + local rank; g-shards cut as layout.py:491-492;
   sid_n(e) goes back to e's home rank.
3. global positions, per mode n: the same sample sort on the B200 order
   (sid_n, sid_{n-1}, Morton, gid) of build_device_sharded gives pos_n(e);
   back home.
4. slices: (pos_n(e), pos_{n+1}(e)) goes to the rank whose mode-n slice holds
   pos_n(e) (its slot map entry), and e's record to the owner of pos_0(e).

Every exchange is one all_to_all_single per array (NCCL on GPUs; gloo moves
CUDA tensors through the host).  Memory per rank is O(input block + slice).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .layout import PartitionPlan, plan_from_counts
from .params import PartitionParams

__all__ = ["morton_key", "build_partitioned", "LocalLayout"]


def morton_key(iv: torch.Tensor, k) -> torch.Tensor:
    """morton.interleave (morton.py:20-44) of the interval coordinates as one
    int64 key (keys of <= 63 bits, every BASELINE config: c4 50 bits)."""
    widths = [int(x - 1).bit_length() if x > 1 else 0 for x in k]
    if sum(widths) > 63:
        raise ValueError(f"the partitioned build needs a Morton key of <= 63 bits ({sum(widths)})")
    key = torch.zeros(iv.shape[0], dtype=torch.int64, device=iv.device)
    pos = 0
    for b in range(max(widths, default=0)):
        for w, wd in enumerate(widths):
            if b < wd:
                key |= ((iv[:, w] >> b) & 1) << pos
                pos += 1
    return key


class _Exchange:
    """Rows of per-element arrays sent to per-element destination ranks with
    all_to_all_single; remembers the permutation to send answers back."""

    def __init__(self, dest: torch.Tensor, world: int, group, host: bool):
        self.world, self.group, self.host = world, group, host
        self.order = torch.argsort(dest, stable=True)
        self.send = torch.bincount(dest, minlength=world).to(torch.int64)
        recv = torch.empty_like(self.send)
        self._a2a(recv, self.send, [1] * world, [1] * world)
        self.recv = recv
        self.send_l = [int(x) for x in self.send.cpu()]
        self.recv_l = [int(x) for x in self.recv.cpu()]

    def _a2a(self, out, inp, out_splits, in_splits):
        if self.host and inp.is_cuda:
            o = torch.empty(out.shape, dtype=out.dtype)
            dist.all_to_all_single(o, inp.cpu(), out_splits, in_splits, group=self.group)
            out.copy_(o)
        else:
            dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        """x (n, ...) in home order -> rows received by this rank."""
        xs = x[self.order].contiguous()
        out = torch.empty((sum(self.recv_l),) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        self._a2a(out, xs, self.recv_l, self.send_l)
        return out

    def backward(self, y: torch.Tensor) -> torch.Tensor:
        """y (received rows, ...) -> rows back at home, in home order."""
        back = torch.empty((sum(self.send_l),) + tuple(y.shape[1:]), dtype=y.dtype, device=y.device)
        self._a2a(back, y.contiguous(), self.send_l, self.recv_l)
        out = torch.empty_like(back)
        out[self.order] = back
        return out


def _sample_index(n: int, ns: int, device) -> torch.Tensor:
    """ns evenly spaced indices into [0, n), in exact integer arithmetic (a
    float linspace rounds past n - 1 once n exceeds 2^24)."""
    return (torch.arange(ns, dtype=torch.int64, device=device) * (n - 1)) // max(ns - 1, 1)


def _stable_sort_by(perm: torch.Tensor, key: torch.Tensor) -> torch.Tensor:
    """perm reordered stably by key[perm]."""
    return perm[torch.argsort(key[perm], stable=True)]


class LocalLayout:
    """One rank's part of the FLYCOO layout for the fused exchange: the
    global plan, this rank's mode-0 records and its slices of every mode's
    global slot map (what peer.PeerShardedTensor takes from a global
    DeviceShardedTensor)."""

    def __init__(self, plan: PartitionPlan, bounds, rank: int, crd, val, slots, device):
        self.plan = plan
        self.bounds = bounds          # per mode: world + 1 element bounds of the slices
        self.rank = rank
        self.crd0, self.val0 = crd, val
        self.slots = slots            # per mode: int32 (uint32 bits) global next-mode positions
        self.device = torch.device(device)
        self.num_modes = plan.num_modes
        self.received = []            # elements this rank sorted in each sample-sort step

    def records_slice(self, lo: int, hi: int):
        b = self.bounds[0]
        assert (lo, hi) == (int(b[self.rank]), int(b[self.rank + 1])), "not this rank's slice"
        return self.crd0, self.val0

    def slot_slice(self, n: int, lo: int, hi: int) -> torch.Tensor:
        b = self.bounds[n]
        assert (lo, hi) == (int(b[self.rank]), int(b[self.rank + 1])), "not this rank's slice"
        return self.slots[n]


def build_partitioned(subs: torch.Tensor, vals: torch.Tensor, gid0: int, params: PartitionParams,
                      R: int | None = None, group=None, device=None) -> LocalLayout:
    """This rank's LocalLayout from its input block `subs` (n_p, N), `vals`
    (n_p,) = input positions [gid0, gid0 + n_p) of the global COO (blocks in
    rank order, covering the tensor).  Collective over `group`.  `R` is the
    factor rank the slice bounds are planned for (default: params.rank)."""
    from .peer import slice_bounds
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if device is not None:
        dev = torch.device(device)
    elif isinstance(subs, torch.Tensor):
        dev = subs.device
    else:  # host arrays: the current GPU (CPU when there is none, e.g. gloo tests)
        dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() \
            else torch.device("cpu")
    host = dist.get_backend(group) == "gloo"
    N = len(params.dims)
    R = int(R if R is not None else params.rank)
    c = torch.as_tensor(subs, device=dev).to(torch.int64)
    v = torch.as_tensor(vals, device=dev).to(torch.float32)
    n_loc = c.shape[0]
    gid = torch.arange(gid0, gid0 + n_loc, dtype=torch.int64, device=dev)
    m = [int(x) for x in params.m]
    k = [int(x) for x in params.k]
    g = int(params.g)
    iv = torch.stack([c[:, w] // m[w] for w in range(N)], 1)
    mkey = morton_key(iv, k)

    def coll(t: torch.Tensor) -> torch.Tensor:
        """A tensor where this group's backend takes it: host for gloo, the
        device for NCCL."""
        return t.cpu() if host else t.to(dev)

    # 1. plan from all-reduced histograms (layout.py:487-497)
    counts = []
    for n in range(N):
        hh = coll(torch.bincount(iv[:, n], minlength=k[n]).to(torch.int64))
        dist.all_reduce(hh, group=group)
        counts.append(hh.cpu().numpy())
    if int(sum(x.sum() for x in counts)) != N * params.nnz:
        raise ValueError("the input blocks do not cover params.nnz nonzeros")
    plan = plan_from_counts(params, counts)
    bounds = slice_bounds(plan, world, R, dev)

    W = sum(int(x - 1).bit_length() if x > 1 else 0 for x in k)
    received = []
    nsh = [plan.total_shards(n) for n in range(N)]
    sbits = [max(x - 1, 1).bit_length() for x in nsh]

    def route_key(fields):
        """Monotone 63-bit summary of a lexicographic key given as (values,
        bits) fields, most significant first: the fields are packed from the
        top and the last one (the Morton key) is truncated to what is left --
        equal full keys give equal route keys, smaller full keys never give
        larger ones."""
        key = torch.zeros(n_loc, dtype=torch.int64, device=dev)
        left = 63
        for vals_, bits in fields:
            take = min(bits, left)
            if take <= 0:
                break
            key = (key << take) | (vals_ >> (bits - take))
            left -= take
        return key << left if left > 0 else key

    def sample_sort(rkey):
        """Exchange routing elements to the owner of their route-key range
        (splitters from an all-gathered sample of 1024 keys per rank) and the
        global position of the first element each rank receives."""
        ns = 1024
        if n_loc:
            smp = torch.sort(rkey)[0][_sample_index(n_loc, ns, dev)]
        else:
            smp = torch.full((ns,), (1 << 63) - 1, dtype=torch.int64, device=dev)
        smp = coll(smp)
        allsmp = [torch.empty_like(smp) for _ in range(world)]
        dist.all_gather(allsmp, smp, group=group)
        pool = torch.sort(torch.cat([t.to(dev) for t in allsmp]))[0]
        spl = pool[[(p * pool.numel()) // world for p in range(1, world)]]
        dest = torch.searchsorted(spl, rkey, right=True)
        E = _Exchange(dest, world, group, host)
        received.append(sum(E.recv_l))
        got = coll(torch.tensor(E.recv_l, dtype=torch.int64))
        counts_all = [torch.empty_like(got) for _ in range(world)]
        dist.all_gather(counts_all, got, group=group)
        per_rank = torch.stack([t.cpu() for t in counts_all]).sum(1)
        base = int(per_rank[:rank].sum())
        return E, base

    # 2. canonical shard ids (layout.py:484-492)
    sid = []
    for n in range(N):
        ivb = max(k[n] - 1, 1).bit_length()
        E, base = sample_sort(route_key([(iv[:, n], ivb), (mkey, max(W, 1))]))
        r_gid = E.forward(gid)
        r_key = E.forward(mkey)
        r_iv = E.forward(iv[:, n].contiguous())
        order = torch.argsort(r_gid, stable=True)          # (already in gid order)
        order = _stable_sort_by(order, r_key)
        order = _stable_sort_by(order, r_iv)
        offs = torch.as_tensor(plan.ss_elem_offsets[n], device=dev)
        first = torch.as_tensor(plan.ss_first_shard[n], device=dev)
        s_iv = r_iv[order]
        pos = base + torch.arange(order.shape[0], device=dev, dtype=torch.int64)
        sid_sorted = first[s_iv] + (pos - offs[s_iv]) // g
        r_sid = torch.empty_like(sid_sorted)
        r_sid[order] = sid_sorted
        sid.append(E.backward(r_sid))

    # 3. global positions in the B200 order (sid_n, sid_{n-1}, Morton, gid)
    gpos = []
    for n in range(N):
        prev = (n - 1) % N
        E, base = sample_sort(route_key([(sid[n], sbits[n]), (sid[prev], sbits[prev]),
                                         (mkey, max(W, 1))]))
        r_gid = E.forward(gid)
        r_key = E.forward(mkey)
        r_sn = E.forward(sid[n])
        r_sp = E.forward(sid[prev])
        order = torch.argsort(r_gid, stable=True)
        order = _stable_sort_by(order, r_key)
        order = _stable_sort_by(order, r_sp)
        order = _stable_sort_by(order, r_sn)
        r_pos = torch.empty(order.shape[0], dtype=torch.int64, device=dev)
        r_pos[order] = base + torch.arange(order.shape[0], device=dev, dtype=torch.int64)
        gpos.append(E.backward(r_pos))

    # 4. slot-map slices and the mode-0 records, to the slice owners
    slots = []
    for n in range(N):
        b = torch.as_tensor(bounds[n][1:-1], device=dev)
        dest = torch.searchsorted(b, gpos[n], right=True)
        E = _Exchange(dest, world, group, host)
        lo = int(bounds[n][rank])
        r_at = E.forward(gpos[n]) - lo
        r_to = E.forward(gpos[(n + 1) % N])
        s = torch.empty(int(bounds[n][rank + 1]) - lo, dtype=torch.int64, device=dev)
        s[r_at] = r_to
        slots.append(s.to(torch.int32) if s.numel() == 0 or int(s.max()) < (1 << 31)
                     else (s - (1 << 32) * (s >= (1 << 31))).to(torch.int32))
    L = _lib.load()
    cw = int(L.fc_crd_words(N))
    emb = bool(L.fc_value_embedded(N))
    rec = torch.zeros((n_loc, cw), dtype=torch.int32, device=dev)
    rec[:, :N] = c.to(torch.int32)
    if emb:
        rec[:, cw - 1] = v.view(torch.int32)
    b = torch.as_tensor(bounds[0][1:-1], device=dev)
    E = _Exchange(torch.searchsorted(b, gpos[0], right=True), world, group, host)
    lo = int(bounds[0][rank])
    r_at = E.forward(gpos[0]) - lo
    r_rec = E.forward(rec)
    n0 = int(bounds[0][rank + 1]) - lo
    crd = torch.empty((n0, cw), dtype=torch.int32, device=dev)
    crd[r_at] = r_rec
    val = None
    if not emb:
        r_val = E.forward(v)
        val = torch.empty(n0, dtype=torch.float32, device=dev)
        val[r_at] = r_val
    out = LocalLayout(plan, bounds, rank, crd, val, slots, dev)
    out.received = received
    return out

"""Super-shard schedule (host side).

The reference assigns super-shards to CPU threads with greedy LPT
(/root/reference/pkg/src/modecycle/schedule.py:33-86).  On the B200 the work
decomposition is per-CTA chunks (layout.make_mode_work), so the engine only
*validates* a ScheduleMap (engine.py:186-189) and ignores its assignment.
The type and the builder are kept so callers of the reference API run
unchanged.
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass

__all__ = ["ScheduleMap", "schedule_super_shards", "load_stats"]


@dataclass(frozen=True)
class ScheduleMap:
    """Per mode, per thread: super-shard lists and their shard-count loads,
    tied to a plan by ``plan_signature`` (schedule.py:33-54)."""

    nu: int
    assignments: tuple
    ss_loads: tuple
    plan_signature: tuple

    @property
    def num_modes(self) -> int:
        return len(self.assignments)

    def thread_loads(self, mode: int) -> list:
        loads = self.ss_loads[mode]
        return [sum(loads[s] for s in lst) for lst in self.assignments[mode]]

    def pointer_entries(self) -> int:
        return sum(len(lst) for mode in self.assignments for lst in mode)


def _lpt(loads, nu: int):
    """Largest load first (ties: lower id) onto the lightest thread (ties:
    lower thread id)."""
    heap = [(0, t) for t in range(nu)]
    heapq.heapify(heap)
    lists = [[] for _ in range(nu)]
    for j in sorted(range(len(loads)), key=lambda j: (-loads[j], j)):
        used, t = heapq.heappop(heap)
        lists[t].append(j)
        heapq.heappush(heap, (used + loads[j], t))
    return lists


def schedule_super_shards(plan, nu: int) -> ScheduleMap:
    if nu < 1:
        raise ValueError("need at least one thread")
    assigns, loads = [], []
    for n in range(plan.num_modes):
        counts = [int(c) for c in plan.ss_shard_counts[n]]
        assigns.append(tuple(tuple(x) for x in _lpt(counts, nu)))
        loads.append(tuple(counts))
    return ScheduleMap(nu=nu, assignments=tuple(assigns), ss_loads=tuple(loads),
                       plan_signature=plan.signature())


def load_stats(smap: ScheduleMap) -> dict:
    modes = []
    for n in range(smap.num_modes):
        loads = smap.thread_loads(n)
        mean = sum(loads) / len(loads)
        modes.append({"mode": n, "max_load": max(loads), "min_load": min(loads),
                      "mean_load": mean, "imbalance": max(loads) / mean if mean > 0 else 1.0})
    return {"nu": smap.nu, "modes": modes}

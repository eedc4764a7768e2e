"""The ILP memory bound of a concrete schedule.

``check_schedule`` restates pkg/src/remsched/oracle.py:287-327: it evaluates
every modeled peak state (forward steps, backward steps, active and settled
sweep positions) and returns ``(feasible, modeled_peak, violation_tags)``.
The executor's measured arena high-water mark is reported against
``modeled_peak`` (north_star: "measured peak HBM <= the ILP bound").
"""

from __future__ import annotations

from .costmodel import Catalog
from .graph import DependencySets, Graph
from .memmodel import MemModel

__all__ = ["check_schedule", "check_schedule_mm"]


def check_schedule_mm(mm: MemModel, schedule, budget: int):
    g, cat = mm.g, mm.catalog
    by_id = g.storable_by_id
    tags: list[str] = []
    peak = 0
    row0 = mm.mask_from_ids(schedule.forward_store)
    for i in range(1, g.n + 1):
        v = cat.fwd(i)[cat.fwd_index(i, schedule.forward_impls[i - 1])]
        m = mm.forward_mem(i, v, row0)
        peak = max(peak, m)
        if m > budget:
            tags.append(f"forward-mem[n{i}]")
    prev = row0
    for t, st in enumerate(schedule.stages, start=1):
        k = st.node
        l = cat.bwd_index(k, st.backward_impl)
        cur = mm.mask_from_ids(st.store)
        m = mm.backward_mem(t, l, cur)
        peak = max(peak, m)
        if m > budget:
            tags.append(f"backward-mem[t{t}]")
        rec = {u: impl for u, impl in st.recompute if not by_id[u].is_intermediate}
        for i in range(1, k + 1):
            if i in rec:
                v = cat.fwd(i)[cat.fwd_index(i, rec[i])]
                m = mm.recompute_mem_active(t, l, i, v, prev, cur)
                tag = f"recompute-mem[t{t},n{i}]"
            else:
                m = mm.recompute_mem_inactive(t, l, i, prev, cur)
                tag = f"settled-mem[t{t},n{i}]"
            peak = max(peak, m)
            if m > budget:
                tags.append(tag)
        prev = cur
    return (not tags, peak, tags)


def check_schedule(g: Graph, sets: DependencySets, catalog: Catalog, schedule, budget: int):
    """(feasible, modeled peak, violation tags) of ``schedule`` under ``budget``."""
    return check_schedule_mm(MemModel(g, sets, catalog), schedule, budget)

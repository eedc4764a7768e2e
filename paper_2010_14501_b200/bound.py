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


class FastBound:
    """Vectorised ``check_schedule`` for the "upper" bound (identical results).

    The modeled peak states are linear in the store rows, so per stage the
    sweep terms for all positions i are three matrix-vector products over
    fixed 0/1 matrices (strict-minus-local, inclusive, tail) instead of
    per-position bitmask sums.  Used by the planner to screen thousands of
    candidate schedules on ResNet-50-sized graphs (reference screening costs
    ~0.5 s per candidate there, SURVEY.md §7 hard part 5).
    """

    def __init__(self, g: Graph, sets: DependencySets, catalog: Catalog, mm: MemModel | None = None):
        import numpy as np

        if sets.bound_kind != "upper":
            raise ValueError("FastBound implements the 'upper' bound kind")
        self.np = np
        self.mm = mm or MemModel(g, sets, catalog)
        mm = self.mm
        self.g, self.sets, self.cat = g, sets, catalog
        n, nb = g.n, mm.n_storables

        def rows(masks):
            out = np.zeros((n + 1, nb), dtype=np.float64)
            for i in range(1, n + 1):
                m = masks[i]
                while m:
                    low = m & -m
                    out[i, low.bit_length() - 1] = 1.0
                    m ^= low
            return out

        local_mask = [0] * (n + 1)
        for i in range(1, n + 1):
            for j in sets.local_fwd[i]:
                local_mask[i] |= 1 << mm.bit_of_id[j]
        self.SL = rows([mm.sweep_mask_strict[i] & ~local_mask[i] if i else 0 for i in range(n + 1)])
        self.IN = rows(mm.sweep_mask_incl)
        self.TA = rows(mm.tail_mask)
        self.FE = rows(mm.forward_extra_mask)
        self.sizes = np.array(mm.sizes, dtype=np.float64)
        self.out_b = np.array([0] + [g.output_bytes(i) for i in range(1, n + 1)], dtype=np.float64)
        self.local_b = np.array([0] + [mm.local_bytes[i] for i in range(1, n + 1)], dtype=np.float64)

    def vec(self, ids):
        v = self.np.zeros(self.mm.n_storables, dtype=self.np.float64)
        for u in ids:
            v[self.mm.bit_of_id[u]] = 1.0
        return v

    def check(self, schedule, budget: int):
        np, mm, g, cat = self.np, self.mm, self.g, self.cat
        by_id = g.storable_by_id
        n = g.n
        tags: list[str] = []
        s0 = self.vec(schedule.forward_store) * self.sizes
        fws = np.array([0] + [cat.fwd(i)[cat.fwd_index(i, schedule.forward_impls[i - 1])].workspace_bytes
                              for i in range(1, n + 1)], dtype=np.float64)
        fwd = fws + self.out_b + g.params_bytes + self.local_b + self.FE @ s0
        fwd = fwd[1:].astype(np.int64)
        peak = int(fwd.max()) if n else 0
        tags.extend(f"forward-mem[n{i}]" for i in np.nonzero(fwd > budget)[0] + 1)
        prev = s0
        for t, st in enumerate(schedule.stages, start=1):
            k = st.node
            l = cat.bwd_index(k, st.backward_impl)
            curv = self.vec(st.store)
            cur = curv * self.sizes
            bm = mm.backward_mem(t, l, mm.mask_from_ids(st.store))
            peak = max(peak, bm)
            if bm > budget:
                tags.append(f"backward-mem[t{t}]")
            deps = cat.bwd(k)[l].deps
            sl = self.SL[1:k + 1] @ cur
            inc = self.IN[1:k + 1] @ cur
            tail = self.TA[1:k + 1] @ prev
            for d in deps:
                b = mm.bit_of_id[d]
                if cur[b]:
                    sl -= self.SL[1:k + 1, b] * cur[b]
                    inc -= self.IN[1:k + 1, b] * cur[b]
            glive = self.sets.grad_live_bytes[k] + g.params_bytes
            inact = np.array([mm.inactive_dep_bytes[(t, l, i)] for i in range(1, k + 1)], dtype=np.float64)
            vals = (glive + inact + inc + tail).astype(np.int64)
            active = np.zeros(k, dtype=bool)
            for u, impl in st.recompute:
                if by_id[u].is_intermediate:
                    continue
                i = u
                v = cat.fwd(i)[cat.fwd_index(i, impl)]
                vals[i - 1] = int(v.workspace_bytes + mm.active_base[(t, i)] + mm.active_dep_bytes[(t, l, i)]
                                  + sl[i - 1] + tail[i - 1])
                active[i - 1] = True
            peak = max(peak, int(vals.max()))
            for i in np.nonzero(vals > budget)[0]:
                tags.append(f"{'recompute' if active[i] else 'settled'}-mem[t{t},n{i + 1}]")
            prev = cur
        return (not tags, peak, tags)

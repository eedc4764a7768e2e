"""Exhaustive reference optimizer for small instances and the solver cross-check.

Public API of the reference module `remsched.oracle` (pkg/src/remsched/
oracle.py): `enumerate_schedules` (alias `enumerate`), `cross_check`,
`OracleResult`, `ORACLE_DEFAULTS`; `check_schedule` lives in bound.py.

The enumeration is the reference's optimum-preserving dynamic program
(oracle.py:3-31): it walks stages back to front over store rows as bitmasks,
forcing each stage's rematerialization set from (carried row, produced row,
backward variant) and its dependency closure, taking every forced rebuild's
cheapest byte-feasible implementation, and never using in-place rewrites.
Ties break as the reference does -- implementations by (cost, catalog order),
equal-cost table entries by the smaller (carried row, backward choice) -- so
the optimum, the schedule and `enumerated_count` are identical.
"""

from __future__ import annotations

import builtins
from dataclasses import dataclass
from fractions import Fraction

from .bound import check_schedule
from .costmodel import Catalog, catalog_to_doc
from .graph import Graph, compute_dependency_sets, graph_to_doc
from .memmodel import MemModel
from .schedule import Schedule, StagePlan, schedule_to_doc, simulate, validate
from .units import format_cost

__all__ = ["ORACLE_DEFAULTS", "OracleResult", "enumerate_schedules", "enumerate", "cross_check"]

_enum = builtins.enumerate  # the module exports its own `enumerate` (reference alias)

ORACLE_DEFAULTS = {"bound_kind": "upper", "node_cap": 6, "storable_cap": 12}


@dataclass(frozen=True)
class OracleResult:
    feasible: bool
    optimum: Fraction | None
    schedule: Schedule | None
    enumerated_count: int
    model_peak: int | None
    true_peak: int | None


def _submasks(mask: int):
    """All submasks of `mask`, largest first, ending with 0."""
    sub = mask
    while True:
        yield sub
        if sub == 0:
            return
        sub = (sub - 1) & mask


class _Tables:
    """Bit tables of one instance."""

    def __init__(self, g: Graph, catalog: Catalog, mm: MemModel):
        st = g.storables
        nb = mm.n_storables
        self.fwd_mask = sum(1 << b for b in range(nb) if not st[b].is_intermediate)
        self.dep_bits = [0] * nb
        self.creator_bit = [0] * nb
        for b, u in _enum(st):
            if u.is_intermediate:
                self.creator_bit[b] = mm.bit_of_id[u.creator]
            else:
                for j in g.deps(u.id):
                    self.dep_bits[b] |= 1 << mm.bit_of_id[j]
        self.avail = [0] * (g.n + 1)  # storables that exist by node i
        for b, u in _enum(st):
            for i in range(u.pos, g.n + 1):
                self.avail[i] |= 1 << b
        self.cheapest = {i: sorted(((l, v) for l, v in _enum(catalog.fwd(i))), key=lambda lv: (lv[1].cost, lv[0]))
                         for i in range(1, g.n + 1)}

    def closure(self, r: int, keep: int) -> int:
        """Rebuild set r plus everything its rebuilds need that `keep` lacks."""
        frontier = r
        while frontier:
            low = frontier & -frontier
            frontier &= frontier - 1
            b = low.bit_length() - 1
            need = (self.dep_bits[b] & ~keep & ~r) if low & self.fwd_mask else ((1 << self.creator_bit[b]) & ~r)
            r |= need
            frontier |= need
        return r


def enumerate_schedules(g: Graph, catalog: Catalog, budget: int, options: dict | None = None) -> OracleResult:
    """Exact optimum over the reduced schedule space (oracle.py:67-284)."""
    opts = {**ORACLE_DEFAULTS, **(options or {})}
    if g.n > opts["node_cap"]:
        raise ValueError(f"oracle caps out at {opts['node_cap']} nodes, got {g.n}")
    sets = compute_dependency_sets(g, opts["bound_kind"])
    mm = MemModel(g, sets, catalog)
    nb = mm.n_storables
    if nb > opts["storable_cap"]:
        raise ValueError(f"oracle caps out at {opts['storable_cap']} storables, got {nb}")
    tb = _Tables(g, catalog, mm)
    st = g.storables
    count = 0

    # forward: per row-0 mask, the cheapest feasible implementation of every node
    dp: dict[int, Fraction] = {}
    fwd_plan: dict[int, tuple[int, ...]] = {}
    for mask in range(1 << nb):
        count += 1
        impls, total = [], Fraction(0)
        for i in range(1, g.n + 1):
            pick = next((l for l, v in tb.cheapest[i] if mm.forward_mem(i, v, mask) <= budget), None)
            if pick is None:
                break
            impls.append(pick)
            total += catalog.fwd(i)[pick].cost
        else:
            dp[mask] = total
            fwd_plan[mask] = tuple(impls)

    T = mm.n_stages
    parents: list[dict[int, tuple]] = []
    for t in range(1, T + 1):
        k = mm.stage_node[t]
        nvar = len(catalog.bwd(k))
        produced = [0] if t == T else list(_submasks(tb.avail[k]))
        base = sets.grad_live_bytes[k] + g.params_bytes
        profiles: dict[tuple[int, int], tuple] = {}

        def profile(l: int, C: int):
            key = (l, C)
            if key not in profiles:
                settled = [0] * (k + 1)
                active = [0] * (k + 1)
                for i in range(1, k + 1):
                    settled[i] = (base + mm.inactive_dep_bytes[(t, l, i)]
                                  + mm.bytes_of(C & mm.inactive_alpha_mask[(t, l, i)]))
                    active[i] = (mm.active_base[(t, i)] + mm.active_dep_bytes[(t, l, i)]
                                 + mm.bytes_of(C & mm.active_alpha_mask[(t, l, i)]))
                profiles[key] = (mm.backward_mem(t, l, C), settled, active)
            return profiles[key]

        best: dict[int, tuple] = {}
        for P in sorted(dp):
            tail = [0] + [mm.bytes_of(P & mm.tail_mask[i]) for i in range(1, k + 1)]
            for C in produced:
                for l in range(nvar):
                    count += 1
                    peak_b, settled, active = profile(l, C)
                    if peak_b > budget:
                        continue
                    r = tb.closure((C & ~P) | (mm.d_mask[(t, l)] & ~C), C)
                    if r & ~tb.avail[k]:
                        continue
                    cost = catalog.bwd(k)[l].cost
                    impls = []
                    for i in range(1, k + 1):
                        if r >> mm.bit_of_id[i] & 1:
                            pick = next((li for li, v in tb.cheapest[i]
                                         if v.workspace_bytes + active[i] + tail[i] <= budget), None)
                            if pick is None:
                                break
                            impls.append((i, pick))
                            cost += catalog.fwd(i)[pick].cost
                        elif settled[i] + tail[i] > budget:
                            break
                    else:
                        total = dp[P] + cost
                        old = best.get(C)
                        if old is None or total < old[0] or (total == old[0] and (P, l) < old[1][:2]):
                            best[C] = (total, (P, l, r, tuple(impls)))
        parents.append({C: rec[1] for C, rec in best.items()})
        dp = {C: rec[0] for C, rec in best.items()}

    def finish(schedule: Schedule, optimum: Fraction) -> OracleResult:
        ok, model_peak, bad = check_schedule(g, sets, catalog, schedule, budget)
        if not ok:
            raise RuntimeError(f"oracle produced a schedule its own model rejects: {bad}")
        trace = simulate(schedule, g, catalog)
        if trace.total_cost != optimum:
            raise RuntimeError("oracle optimum does not match its schedule's simulated cost")
        return OracleResult(True, optimum, schedule, count, model_peak, trace.peak_memory)

    fwd_names = lambda mask: tuple(catalog.fwd(i)[l].name  # noqa: E731
                                   for i, l in zip(range(1, g.n + 1), fwd_plan[mask]))
    if T == 0:
        if not dp:
            return OracleResult(False, None, None, count, None, None)
        m0 = min(dp, key=lambda m: (dp[m], m))
        return finish(Schedule(fwd_names(m0), tuple(mm.ids_from_mask(m0)), (), dp[m0]), dp[m0])
    if 0 not in dp:
        return OracleResult(False, None, None, count, None, None)

    rows, info, cur = [0] * (T + 1), [None] * (T + 1), 0
    for t in range(T, 0, -1):  # walk parents back to the forward row
        P, l, r, impls = parents[t - 1][cur]
        rows[t], info[t] = cur, (l, r, dict(impls))
        cur = P
    rows[0] = cur
    stages = []
    for t in range(1, T + 1):
        k = mm.stage_node[t]
        l, r, impl_of = info[t]
        rec = tuple((u.id, None if u.is_intermediate else catalog.fwd(u.id)[impl_of[u.id]].name)
                    for b, u in _enum(st) if r >> b & 1)
        stages.append(StagePlan(node=k, recompute=rec, store=tuple(mm.ids_from_mask(rows[t])),
                                backward_impl=catalog.bwd(k)[l].name, inplace=()))
    return finish(Schedule(fwd_names(rows[0]), tuple(mm.ids_from_mask(rows[0])), tuple(stages), dp[0]), dp[0])


enumerate = enumerate_schedules  # noqa: A001  (reference alias, oracle.py:431)


def cross_check(g: Graph, catalog: Catalog, budgets, options: dict | None = None) -> dict:
    """Solve and enumerate the same instance per budget and compare (oracle.py:330-428)."""
    from .ilp import build_model
    from .schedule import decode
    from .solver import solve

    opts = {"bound_kind": "upper", "inplace": True, "solve": {}, "oracle": {}, **(options or {})}
    sets = compute_dependency_sets(g, opts["bound_kind"])
    cells, counterexamples = [], []
    for budget in budgets:
        model = build_model(g, sets, catalog, budget, {"inplace": opts["inplace"], "bound_kind": opts["bound_kind"]})
        res = solve(model, dict(opts["solve"]))
        orc = enumerate_schedules(g, catalog, budget, {"bound_kind": opts["bound_kind"], **opts["oracle"]})
        problems: list[str] = []
        solver_doc = None
        if res.status == "optimal":
            if not orc.feasible:
                problems.append("solver found an optimum where the oracle found no feasible schedule")
            elif res.objective != orc.optimum:
                problems.append(f"objective mismatch: solver {format_cost(res.objective)}"
                                f" vs oracle {format_cost(orc.optimum)}")
            if orc.feasible:
                sched = None
                try:
                    sched = decode(res, g, catalog)
                    solver_doc = schedule_to_doc(sched)
                except ValueError as exc:
                    problems.append(f"decode failed: {exc}")
                if sched is not None:
                    bad = validate(sched, g, sets, catalog)
                    if bad:
                        problems.append(f"solver schedule invalid: {bad}")
                    else:
                        ok, _, tags = check_schedule(g, sets, catalog, sched, budget)
                        if not ok:
                            problems.append(f"solver schedule over budget in the oracle's accounting: {tags}")
                        trace = simulate(sched, g, catalog)
                        if trace.total_cost != res.objective:
                            problems.append(f"simulated cost {format_cost(trace.total_cost)} "
                                            f"!= objective {format_cost(res.objective)}")
                        if trace.peak_memory > budget:
                            problems.append(f"simulated peak {trace.peak_memory} exceeds budget {budget}")
        elif res.status == "infeasible":
            if orc.feasible:
                problems.append("solver reported infeasible but the oracle found a schedule costing "
                                f"{format_cost(orc.optimum)}")
        else:
            problems.append(f"solver stopped early with status {res.status}")
        cells.append({
            "budget": budget, "solver_status": res.status,
            "solver_objective": None if res.objective is None else format_cost(res.objective),
            "solver_nodes": res.nodes, "oracle_feasible": orc.feasible,
            "oracle_objective": None if orc.optimum is None else format_cost(orc.optimum),
            "oracle_enumerated": orc.enumerated_count, "oracle_model_peak": orc.model_peak,
            "oracle_true_peak": orc.true_peak, "agree": not problems, "problems": problems,
        })
        if problems:
            counterexamples.append({
                "budget": budget, "problems": problems, "graph": graph_to_doc(g),
                "catalog": catalog_to_doc(catalog), "solver_schedule": solver_doc,
                "oracle_schedule": None if orc.schedule is None else schedule_to_doc(orc.schedule),
            })
    return {"pass": all(c["agree"] for c in cells), "bound_kind": opts["bound_kind"], "inplace": opts["inplace"],
            "cells": cells, "counterexamples": counterexamples}

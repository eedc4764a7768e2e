"""Host planner: budget-feasible schedules for large graphs.

The reference's exact 0-1 branch-and-bound does not find incumbents at
ResNet-50 scale (226k variables, SURVEY.md §7 hard part 5) and its warm-start
heuristic (schedule.py:634-667) both takes minutes there and emits schedules
its own simulator rejects (it rebuilds a creator that is still live to recover
an intermediate).  This planner builds schedules in the
same format from a *demand* construction that is valid by design:

* the forward pass keeps a checkpoint set S0 chosen by tensor family (conv
  outputs, BN outputs, ReLU outputs, residual sums, sign masks, pool
  indices) and optionally thinned per residual block;
* each backward stage picks the cheapest backward variant whose inputs can be
  made available — kept in the carried row, or rebuilt in-stage from what is
  available (never rebuilding a tensor that is still live);
* a stage's row keeps what the stage itself reads from the carried row plus
  what later stages read, optionally only within a window.

Every candidate is screened with the exact modeled bound
(bound.FastBound == check_schedule) and the simulator; the cheapest feasible
schedule under the catalog's costs wins.  The result can seed the
reference-exact ILP solver as its incumbent.
"""

from __future__ import annotations

from fractions import Fraction

from .bound import FastBound
from .costmodel import Catalog
from .graph import Graph, compute_dependency_sets
from .memmodel import schedule_cost
from .schedule import (Schedule, SimulationError, StagePlan, fastest_store_everything_schedule, simulate,
                       store_everything_schedule)

__all__ = ["plan_schedule", "demand_schedule", "FAMILIES"]


def _cheapest_fwd(cat: Catalog, i: int, ws_cap: int | None = None) -> int:
    vs = cat.fwd(i)
    ok = [l for l in range(len(vs)) if ws_cap is None or vs[l].workspace_bytes <= ws_cap]
    return min(ok or range(len(vs)), key=lambda l: (vs[l].cost, l))


def demand_schedule(g: Graph, cat: Catalog, store0: set, window: int | None = None,
                    prefer: str = "cost") -> Schedule | None:
    """Build a schedule that keeps ``store0`` from the forward pass.

    window: a tensor rebuilt in a stage is kept for later stages only if it is
    read again within ``window`` stages (None = until its last use).
    prefer: "cost" picks the cheapest backward variant; "lean" the one whose
    dependencies are already available, then the cheapest.
    """
    by_id = g.storable_by_id
    ints_of = g.intermediates_of
    fwd_impl = [cat.fwd(i)[_cheapest_fwd(cat, i)].name for i in range(1, g.n + 1)]
    stages = g.stage_nodes
    n_st = len(stages)
    store0 = set(store0)
    # the forward pass can only store what it produces: node outputs and the
    # intermediates of nodes (both always producible in forward)
    prev = set(store0)
    plans = []
    chosen_bwd: list = []
    # needs of later stages are only known after their variants are chosen; use
    # the default-variant needs of every variant as the future-need estimate
    future_need: list[dict] = [dict() for _ in range(n_st + 1)]
    for t in range(n_st - 1, -1, -1):
        fut = dict(future_need[t + 1])
        for v in cat.bwd(stages[t]):
            for d in v.deps:
                fut[d] = t  # stage index (0-based) of the soonest later reader
        future_need[t] = fut

    for t in range(1, n_st + 1):
        k = stages[t - 1]
        best = None
        for l, v in sorted(enumerate(cat.bwd(k)), key=lambda e: (e[1].cost, e[0])):
            rec: set = set()
            used_prev: set = set()
            ok = True

            def ensure(x, depth=0):
                nonlocal ok
                if not ok:
                    return
                if x in prev:
                    used_prev.add(x)
                    return
                if x in rec:
                    return
                u = by_id[x]
                if u.is_intermediate:
                    c = u.creator
                    if c in prev:  # creator live: rebuilding it would double-allocate
                        ok = False
                        return
                    ensure_node(c)
                    rec.add(x)
                else:
                    ensure_node(x)

            def ensure_node(i):
                nonlocal ok
                if i in prev:
                    used_prev.add(i)
                    return
                if i in rec:
                    return
                for j in g.deps(i):
                    ensure(j)
                rec.add(i)

            for d in v.deps:
                ensure(d)
            if not ok:
                continue
            if prefer == "lean":
                key = (len(rec), v.cost, l)
            else:
                key = (v.cost + sum(cat.fwd(i)[cat.fwd_index(i, fwd_impl[i - 1])].cost
                                    for i in rec if not by_id[i].is_intermediate), l)
            if best is None or key < best[0]:
                best = (key, l, rec, used_prev)
        if best is None:
            return None
        _, l, rec, used_prev = best
        v = cat.bwd(k)[l]
        if t == n_st:
            cur = set()
            if used_prev or rec - set(v.deps):
                # the final row must be empty: everything read must be rebuilt
                if used_prev:
                    return None
        else:
            later = future_need[t]  # readers in stages t+1.. (0-based index t)
            cur = set(used_prev)
            for x in (prev | rec):
                if x in later:
                    soon = later[x] - (t - 1)
                    if x in store0 or window is None or soon <= window:
                        cur.add(x)
            # intermediates rebuilt here must be kept or read by this backward
            for x in list(rec):
                if by_id[x].is_intermediate and x not in cur and x not in v.deps:
                    rec.discard(x)
        order = sorted(rec, key=lambda x: (by_id[x].pos, by_id[x].is_intermediate, x))
        entries = tuple((x, None if by_id[x].is_intermediate else fwd_impl[x - 1]) for x in order)
        # recompute in place (schedule.py:403-411) where the input dies with it: it is not kept,
        # not read by this backward, not read by a later recompute of the stage and was not
        # carried in as this node's output
        inplace = []
        nodes = [x for x in order if not by_id[x].is_intermediate]
        for pos, i in enumerate(nodes):
            deps = g.deps(i)
            if len(deps) != 1 or i in prev:
                continue
            fv = cat.fwd(i)[cat.fwd_index(i, fwd_impl[i - 1])]
            j = deps[0]
            if (fv.inplace_capable and g.output_bytes(i) == g.output_bytes(j) and j not in cur
                    and j not in v.deps and not any(j in g.deps(u) for u in nodes[pos + 1:])):
                inplace.append(i)
        plans.append(StagePlan(k, entries, tuple(u.id for u in g.storables if u.id in cur), v.name,
                               tuple(inplace)))
        chosen_bwd.append(l)
        prev = cur
    sched = Schedule(tuple(fwd_impl), tuple(u.id for u in g.storables if u.id in store0), tuple(plans), None)
    return Schedule(sched.forward_impls, sched.forward_store, sched.stages, schedule_cost(g, cat, sched))


def _fwd_cost(cat: Catalog, g: Graph, x: int):
    """Cheapest forward cost of a storable's creator (what keeping it saves per rebuild)."""
    u = g.storable_by_id[x]
    node = u.creator if u.is_intermediate else x
    return min(v.cost for v in cat.fwd(node))


def _families(g: Graph, kind_of) -> dict:
    """Named checkpoint sets by tensor family."""
    ids = [u.id for u in g.storables]
    fam = {}

    def pick(kinds):
        if "relu" in kinds:
            kinds = kinds | {"relu-join"}
        return {x for x in ids if kind_of(x) in kinds}

    base = {"input", "maxpool", "avgpool", "fc", "xent", "dropout", "wgrad"}  # wgrad anchors: 0 bytes
    fam["all"] = set(ids)
    fam["conv+relu+mask"] = pick(base | {"conv", "relu", "mask", "idx"})
    fam["conv+mask"] = pick(base | {"conv", "mask", "idx"})
    fam["bn+relu+mask"] = pick(base | {"bn", "relu", "mask", "idx"})
    fam["bn+mask"] = pick(base | {"bn", "mask", "idx"})
    fam["relu+mask"] = pick(base | {"relu", "mask", "idx"})
    fam["conv+add+mask"] = pick(base | {"conv", "add", "mask", "idx"})
    fam["add+mask"] = pick(base | {"add", "mask", "idx"})
    fam["join"] = pick(base | {"relu-join", "mask", "idx"})
    return fam


FAMILIES = ("all", "conv+relu+mask", "conv+mask", "bn+relu+mask", "bn+mask", "relu+mask",
            "conv+add+mask", "add+mask", "join")


EXACT_MAX_NODES = 64  # graphs up to this size also go through the exact ILP (VGG-16: 40 nodes)
LP_THRESHOLDS = (0.05, 0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9, 0.95)


def ilp_relaxation(g: Graph, cat: Catalog, budget: int, mip_time_s: float | None = None) -> dict | None:
    """The reference's 0-1 ILP (ilp.build_model: same variables, rows and objective as
    pkg/src/remsched/ilp.py:121) handed to HiGHS through scipy.optimize.milp.

    * LP relaxation (seconds at ResNet-50 scale, 58k variables / 113k rows): its optimum
      is a lower bound on the cost of every schedule at this budget, and its row-0 store
      values S[0, u] in [0, 1] say which tensors the forward pass should keep;
    * optionally the MIP itself for ``mip_time_s``: HiGHS's dual bound (tighter than the
      LP's) and its incumbent, decoded like the reference decodes its own (schedule.py:132).

    Returns {"lp_bound", "s0", "model"[, "mip_bound", "mip_schedule", "mip_status"]}, or
    None when scipy / HiGHS is unavailable.  Host-side planning only (no GPU)."""
    try:
        import numpy as np
        import scipy.sparse as sp
        from scipy.optimize import Bounds, LinearConstraint, milp
    except ImportError:
        return None
    from .ilp import build_model

    m = build_model(g, compute_dependency_sets(g), cat, budget)
    n = m.n_vars
    c = np.zeros(n)
    for j, cost in m.objective:
        c[j] += float(cost)
    ri, ci, va, lo, hi = [], [], [], [], []
    for r, row in enumerate(m.rows):
        for j, a in row.terms:
            ri.append(r)
            ci.append(j)
            va.append(float(a))
        lo.append(-np.inf if row.sense == "<=" else float(row.rhs))
        hi.append(float(row.rhs))
    A = sp.csr_matrix((va, (ri, ci)), shape=(len(m.rows), n))
    lb, ub = np.zeros(n), np.ones(n)
    for j, v in m.fixed.items():
        lb[j] = ub[j] = v
    cons, bnds = LinearConstraint(A, lo, hi), Bounds(lb, ub)
    lp = milp(c, constraints=cons, integrality=np.zeros(n), bounds=bnds)
    if lp.status != 0:
        return {"lp_bound": None, "s0": {}, "model": m, "lp_status": lp.message}
    s0 = {v.node: float(lp.x[j]) for j, v in enumerate(m.var_ids) if v.kind == "S" and v.row == 0}
    out = {"lp_bound": Fraction(lp.fun).limit_denominator(1 << 20), "s0": s0, "model": m}
    if mip_time_s:
        res = milp(c, constraints=cons, integrality=np.ones(n), bounds=bnds, options={"time_limit": mip_time_s})
        out["mip_status"] = res.message
        bound = getattr(res, "mip_dual_bound", None)
        out["mip_bound"] = None if bound is None else Fraction(bound).limit_denominator(1 << 20)
        if res.x is not None:
            from .ilp import evaluate_assignment
            from .schedule import decode

            x = [int(round(v)) for v in res.x]
            out["mip_s0"] = {v.node for j, v in enumerate(m.var_ids) if v.kind == "S" and v.row == 0 and x[j]}
            ev = evaluate_assignment(m, x)
            if ev["feasible"]:
                class _R:  # the fields decode() reads from a solver result
                    status, assignment, model, objective = "feasible-gap", x, m, ev["objective"]
                try:
                    out["mip_schedule"] = decode(_R, g, cat)
                except ValueError:
                    pass
    return out


def plan_schedule(g: Graph, cat: Catalog, budget: int, kinds: dict | None = None,
                  exact_time_s: float | None = None, exchange: bool = False, lp: bool = False,
                  mip_time_s: float | None = None):
    """Cheapest feasible schedule among the demand-construction candidates.

    ``kinds`` maps storable id -> family label; by default inferred from the
    graph structure is not possible, so the tracer's op kinds are expected via
    ``Network.storable_kinds()``; without it every storable counts as "all".
    ``exchange``: after the greedy additions, also try exchange moves (keep one more
    tensor, drop a cheaper one) -- offline planning (tools/make_schedules.py), seconds more.
    ``exact_time_s``: on graphs of at most EXACT_MAX_NODES nodes, also run the
    reference-exact 0-1 ILP (ilp.build_model + solver.solve) for that long,
    seeded with the best candidate as its incumbent; its schedule wins when it
    is cheaper or the only feasible one.
    ``lp``: solve the ILP's LP relaxation (ilp_relaxation, HiGHS) and add forward-store
    sets thresholded from its row-0 store values as demand-construction seeds; the LP
    optimum (or, with ``mip_time_s``, HiGHS's MIP dual bound) is reported as the lower
    bound and the chosen schedule's gap to it.
    Returns (schedule or None, info dict).
    """
    relax = ilp_relaxation(g, cat, budget, mip_time_s) if (lp or mip_time_s) else None
    seeds = []
    if relax and relax["s0"]:
        for thr in LP_THRESHOLDS:
            seeds.append((f"lp{thr:g}", {u for u, val in relax["s0"].items() if val >= thr}))
    if relax and relax.get("mip_s0"):  # the MIP incumbent's forward store set, rebuilt by demand
        seeds.append(("mip", relax["mip_s0"]))
    sch, info = _plan_heuristic(g, cat, budget, kinds, exchange, seeds)
    if relax is not None:
        mip = relax.get("mip_schedule")
        if mip is not None and (sch is None or mip.objective < sch.objective):
            ok, peak, _ = FastBound(g, compute_dependency_sets(g, "upper"), cat).check(mip, budget)
            try:  # an ILP-feasible decode the simulator rejects is not executable
                simulate(mip, g, cat)
            except SimulationError:
                ok = False
            if ok:
                se = info.get("se_cost")
                info = {"family": "ilp-highs/feasible", "candidates": info["candidates"], "modeled_peak": peak,
                        "objective": str(mip.objective), "se_cost": se,
                        "overhead_vs_store_everything": None if se is None else float(Fraction(mip.objective) / se - 1)}
                sch = mip
        bound = max(b for b in (relax.get("lp_bound"), relax.get("mip_bound")) if b is not None) \
            if relax.get("lp_bound") is not None else None
        info["ilp_lower_bound"] = None if bound is None else round(float(bound), 1)
        info["ilp_lower_bound_source"] = "highs-mip-dual" if relax.get("mip_bound") is not None else "highs-lp"
        if bound is not None and sch is not None:
            info["ilp_gap"] = float(1 - bound / Fraction(sch.objective))
    if exact_time_s and g.n <= EXACT_MAX_NODES:
        from .ilp import assignment_from_schedule, build_model
        from .schedule import decode
        from .solver import solve

        model = build_model(g, compute_dependency_sets(g), cat, budget)
        opts = {"time_limit_s": exact_time_s}
        if sch is not None:
            opts["incumbent"] = assignment_from_schedule(model, sch)
        res = solve(model, opts)
        if res.assignment is not None:
            ilp = decode(res, g, cat)
            if sch is None or ilp.objective < sch.objective:
                ok, peak, _ = FastBound(g, compute_dependency_sets(g, "upper"), cat).check(ilp, budget)
                simulate(ilp, g, cat)
                se = info.get("se_cost")
                info = {"family": f"exact-ilp/{res.status}", "candidates": info["candidates"], "modeled_peak": peak,
                        "objective": str(ilp.objective), "ilp_gap": None if res.gap is None else float(res.gap),
                        "overhead_vs_store_everything": None if se is None else float(Fraction(ilp.objective) / se - 1)}
                sch = ilp
    info.pop("se_cost", None)
    return sch, info


def _plan_heuristic(g: Graph, cat: Catalog, budget: int, kinds: dict | None = None, exchange: bool = False,
                    seeds=()):
    sets = compute_dependency_sets(g, "upper")
    fb = FastBound(g, sets, cat)
    kind_of = (lambda x: kinds.get(x, "other")) if kinds else (lambda x: "other")
    fams = _families(g, kind_of)
    # thinned variants: drop the family's tensors in every other "segment" of
    # the residual chain (nodes between consecutive joins)
    joins = sorted(x for x in fams["join"] if not g.storable_by_id[x].is_intermediate)
    cands = []
    try:
        cands.append(("store_everything", store_everything_schedule(g, cat)))
        cands.append(("store_everything/fastest", fastest_store_everything_schedule(g, cat)))
    except ValueError:
        pass
    for name in FAMILIES + tuple(n for n, _ in seeds):
        s0 = fams.get(name) if name in fams else dict(seeds).get(name)
        if not s0:
            continue
        variants = [(name, s0)]
        if name not in fams:  # LP-guided seeds are used as given (no residual thinning)
            for window in (None, 8, 2, 0):
                for prefer in ("cost", "lean"):
                    sch = demand_schedule(g, cat, s0, window=window, prefer=prefer)
                    if sch is not None:
                        cands.append((f"{name}/w{window}/{prefer}", sch, (s0, window, prefer)))
            continue
        for stride in (2, 3):
            for phase in range(stride):
                keep_segs = set()
                for si, (a, b) in enumerate(zip([0] + joins, joins + [g.n + 1])):
                    if si % stride == phase:
                        keep_segs.update(range(a + 1, b))
                thin = {x for x in s0 if g.storable_by_id[x].pos not in keep_segs or x in fams["join"]}
                variants.append((f"{name}/thin{stride}.{phase}", thin))
        for vname, s0v in variants:
            for window in (None, 8, 2, 0):
                for prefer in ("cost", "lean"):
                    sch = demand_schedule(g, cat, s0v, window=window, prefer=prefer)
                    if sch is not None:
                        cands.append((f"{vname}/w{window}/{prefer}", sch, (s0v, window, prefer)))
    best = None
    tried = 0
    feasible = []
    for name, sch, *rest in cands:
        tried += 1
        ok, peak, _ = fb.check(sch, budget)
        if not ok:
            continue
        try:
            simulate(sch, g, cat)
        except SimulationError:
            continue
        feasible.append((sch.objective, name, sch, peak, rest[0] if rest else None))
        if best is None or sch.objective < best[1].objective:
            best = (name, sch, peak)
    # greedy augmentation of the best few demand constructions: also keep one more
    # tensor from the forward pass (most expensive forward first) whenever the
    # schedule still fits and gets cheaper; repeat until no single addition helps
    feasible.sort(key=lambda e: e[0])
    order = sorted((u.id for u in g.storables), key=lambda x: -_fwd_cost(cat, g, x))
    for _, name, sch, peak, spec in feasible[:3]:
        if spec is None:
            continue
        s0v, window, prefer = spec
        cur_s0, cur, cur_peak, grown = set(s0v), sch, peak, 0
        improved = True
        while improved:
            improved = False
            for x in order:
                if x in cur_s0:
                    continue
                trial = demand_schedule(g, cat, cur_s0 | {x}, window=window, prefer=prefer)
                tried += 1
                if trial is None or trial.objective >= cur.objective:
                    continue
                ok, pk, _ = fb.check(trial, budget)
                if not ok:
                    continue
                try:
                    simulate(trial, g, cat)
                except SimulationError:
                    continue
                cur_s0, cur, cur_peak, grown = cur_s0 | {x}, trial, pk, grown + 1
                improved = True
        # exchange moves: keep an expensive-to-rebuild tensor in place of a cheap one
        swaps = 0
        improved = exchange
        while improved:
            improved = False
            adds = [x for x in order if x not in cur_s0][:24]
            drops = [y for y in reversed(order) if y in cur_s0 and y not in s0v][:32]
            for x in adds:
                for y in drops:
                    trial = demand_schedule(g, cat, (cur_s0 - {y}) | {x}, window=window, prefer=prefer)
                    tried += 1
                    if trial is None or trial.objective >= cur.objective:
                        continue
                    ok, pk, _ = fb.check(trial, budget)
                    if not ok:
                        continue
                    try:
                        simulate(trial, g, cat)
                    except SimulationError:
                        continue
                    cur_s0, cur, cur_peak, swaps = (cur_s0 - {y}) | {x}, trial, pk, swaps + 1
                    improved = True
                    break
                if improved:
                    break
        if (grown or swaps) and cur.objective < best[1].objective:
            best = (f"{name}/+{grown}~{swaps}", cur, cur_peak)
    se_cost = None
    try:
        se_cost = fastest_store_everything_schedule(g, cat).objective
    except ValueError:
        pass
    if best is None:
        return None, {"candidates": tried, "se_cost": se_cost}
    name, sch, peak = best
    info = {"family": name, "candidates": tried, "modeled_peak": peak,
            "objective": str(sch.objective), "se_cost": se_cost,
            "overhead_vs_store_everything": None if se_cost is None
            else float(Fraction(sch.objective) / se_cost - 1)}
    return sch, info

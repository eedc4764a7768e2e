"""Exact 0-1 branch-and-bound for the scheduling model (host, native core).

Same search as the reference solver (pkg/src/remsched/solver.py:441-650):
propagation, bound, branching order, dives, limits and statuses are
identical, so for a given model and options (deterministic `node_limit`,
same `incumbent`) the decisions are bit-exact.  The search loop runs in
C++ (csrc/bnb.cpp, `monet_bnb_*` in include/monet_b200.h) on integer-scaled
costs; this module packs the Model, translates options and rebuilds the
reference's SolveResult / telemetry records.
"""

from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from . import _native
from .ilp import Model, evaluate_assignment
from .units import cost_str

__all__ = ["BRANCH_ORDERS", "SolveResult", "solve", "propagate", "lower_bound"]

BRANCH_ORDERS = ("paper", "fixed", "most-tight")
# kinds tried at 1 first while diving; stores dive at 0 (solver.py:35-38)
_PREF1 = {"DeltaFwd", "DeltaBwd", "DeltaRe"}
_EVENTS = ("root", "warm-start", "incumbent", "tick", "final")
_STATUS = ("optimal", "feasible-gap", "infeasible", "timeout-no-incumbent")


@dataclass
class SolveResult:
    status: str  # optimal | feasible-gap | infeasible | timeout-no-incumbent
    objective: Fraction | None
    assignment: list[int] | None
    lower_bound: Fraction | None
    gap: Fraction | None
    nodes: int
    elapsed_s: float
    telemetry: list[dict]
    model: Model


def _i128(vals) -> np.ndarray:
    out = np.empty(2 * len(vals), dtype=np.int64)
    for i, v in enumerate(vals):
        v = int(v)
        hi, lo = v >> 64, v & ((1 << 64) - 1)
        out[2 * i] = hi
        out[2 * i + 1] = lo - (1 << 64) if lo >= 1 << 63 else lo
    return out


def _from128(arr, i) -> int:
    hi, lo = int(arr[2 * i]), int(arr[2 * i + 1])
    return (hi << 64) | (lo & ((1 << 64) - 1))


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class _Native:
    """A model packed for the native core (cached on the Model)."""

    def __init__(self, model: Model, surrogate: bool = True):
        lib = _native.lib().dll
        self.lib = lib
        self.scale = 1
        for _, c in model.objective:
            self.scale = self.scale * c.denominator // math.gcd(self.scale, c.denominator)
        self.integral = self.scale == 1
        S = self.scale
        rows = model.rows
        row_ptr = np.zeros(len(rows) + 1, dtype=np.int32)
        row_ptr[1:] = np.cumsum([len(r.terms) for r in rows])
        nnz = int(row_ptr[-1])
        row_var = np.fromiter((v for r in rows for v, _ in r.terms), dtype=np.int32, count=nnz)
        row_coef = np.fromiter((c for r in rows for _, c in r.terms), dtype=np.int64, count=nnz)
        rhs = np.array([r.rhs for r in rows], dtype=np.int64)
        is_eq = np.array([1 if r.sense == "=" else 0 for r in rows], dtype=np.int32)
        fix_var = np.array(list(model.fixed.keys()), dtype=np.int32)
        fix_val = np.array(list(model.fixed.values()), dtype=np.int32)
        obj_var = np.array([v for v, _ in model.objective], dtype=np.int32)
        obj_cost = _i128([c * S for _, c in model.objective])
        groups = list(model.fwd_groups) + list(model.bwd_groups) + [g for _, g in model.re_groups]
        grp_ptr = np.zeros(len(groups) + 1, dtype=np.int32)
        grp_ptr[1:] = np.cumsum([len(g) for g in groups])
        grp_var = np.array([v for g in groups for v, _ in g], dtype=np.int32)
        grp_cost = _i128([c * S for g in groups for _, c in g])
        re_rvar = np.array([r for r, _ in model.re_groups], dtype=np.int32)
        self._keep = (row_ptr, row_var, row_coef, rhs, is_eq, fix_var, fix_val, obj_var, obj_cost, grp_ptr,
                      grp_var, grp_cost, re_rvar)
        lib.monet_bnb_create.restype = C.c_void_p
        self.h = lib.monet_bnb_create(
            model.n_vars, len(rows), _p(row_ptr), _p(row_var), _p(row_coef), _p(rhs), _p(is_eq), len(fix_var),
            _p(fix_var), _p(fix_val), len(obj_var), _p(obj_var), _p(obj_cost), len(model.fwd_groups),
            len(model.bwd_groups), len(model.re_groups), _p(grp_ptr), _p(grp_var), _p(grp_cost), _p(re_rvar))
        if not self.h:
            raise MemoryError("native solver allocation failed")
        if surrogate:
            self._surrogate(model)

    def _surrogate(self, model: Model):
        """Capacity surrogate inputs (solver.py:226-249), storables in id order."""
        from .ilp import VarId
        g, sets, cat = model.g, model.sets, model.catalog
        st = sorted(g.storables, key=lambda u: u.id)
        idx = {u.id: i for i, u in enumerate(st)}
        T = len(g.stage_nodes)
        grad, var_ptr, var_db, var_ws, dep_ptr, dep_idx = [], [0], [], [], [0], []
        for t, k in zip(range(1, T + 1), g.stage_nodes):
            grad.append(sets.grad_live_bytes[k])
            for l, bv in enumerate(cat.bwd(k)):
                var_db.append(model.bwd_groups[t - 1][l][0])
                var_ws.append(bv.workspace_bytes)
                dep_idx += sorted(idx[d] for d in set(bv.deps))
                dep_ptr.append(len(dep_idx))
            var_ptr.append(len(var_db))
        size = [u.nbytes for u in st]
        recost = [0 if u.is_intermediate else int(min(v.cost for v in cat.fwd(u.id))) for u in st]
        rcol = [model.var_index[VarId("R", row=t, node=u.id)] for u in st for t in range(1, T + 1)]
        arrs = [np.array(a, dtype=d) for a, d in ((grad, np.int64), (var_ptr, np.int32), (var_db, np.int32),
                                                  (var_ws, np.int64), (dep_ptr, np.int32), (dep_idx, np.int32),
                                                  (size, np.int64), (recost, np.int64), (rcol, np.int32))]
        self._keep_s = arrs
        grad_a, vp, vdb, vws, dp, di, sz, rc, rcl = arrs
        self.lib.monet_bnb_set_surrogate(C.c_void_p(self.h), C.c_int64(model.budget - g.params_bytes), T,
                                         _p(grad_a), _p(vp), _p(vdb), _p(vws), _p(dp), _p(di), len(st), _p(sz),
                                         _p(rc), _p(rcl))

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.monet_bnb_destroy(C.c_void_p(self.h))
            self.h = None

    def partial(self, partial):
        items = list((partial or {}).items())
        pv = np.array([v for v, _ in items], dtype=np.int32)
        pb = np.array([b for _, b in items], dtype=np.int32)
        return len(items), pv, pb


def _native_of(model: Model, surrogate: bool = True) -> _Native:
    cache = model.__dict__.setdefault("_native_bnb", {})
    if surrogate not in cache:
        cache[surrogate] = _Native(model, surrogate)
    return cache[surrogate]


def _static_order(model: Model, mode: str) -> list[int]:
    """Branching order (solver.py:346-376)."""
    if mode == "fixed":
        return list(range(model.n_vars))
    by_cost = lambda grp: [v for v, _ in sorted(grp, key=lambda vc: (vc[1], vc[0]))]  # noqa: E731
    order = [v for grp in model.bwd_groups for v in by_cost(grp)]
    order += [v for grp in model.fwd_groups for v in by_cost(grp)]
    kinds: dict[str, list[int]] = {}
    for i, vid in enumerate(model.var_ids):
        kinds.setdefault(vid.kind, []).append(i)
    # recompute flags column-major: one tensor's column before the next
    order += sorted(kinds.get("R", []), key=lambda v: (model.var_ids[v].node, model.var_ids[v].row))
    order += [v for _, grp in model.re_groups for v in by_cost(grp)]
    for kind in ("S", "Q", "P", "Alpha"):
        order += kinds.get(kind, [])
    return order


def propagate(model: Model, partial: dict[int, int] | None = None):
    """Fixpoint propagation from the fixings plus `partial` (solver.py:406-422).

    Returns (consistent, {var: value} for every decided variable)."""
    nat = _native_of(model)
    n, pv, pb = nat.partial(partial)
    out = np.empty(model.n_vars, dtype=np.int8)
    if not nat.lib.monet_bnb_propagate(C.c_void_p(nat.h), n, _p(pv), _p(pb), _p(out)):
        return False, {}
    return True, {v: int(x) for v, x in enumerate(out) if x != -1}


def lower_bound(model: Model, partial: dict[int, int] | None = None) -> Fraction | None:
    """Admissible objective bound under `partial`; None if inconsistent (solver.py:425-438)."""
    nat = _native_of(model)
    n, pv, pb = nat.partial(partial)
    out = np.zeros(2, dtype=np.int64)
    if not nat.lib.monet_bnb_lower_bound(C.c_void_p(nat.h), n, _p(pv), _p(pb), C.c_int64(nat.scale), _p(out)):
        return None
    return Fraction(_from128(out, 0), nat.scale)


def solve(model: Model, options: dict | None = None) -> SolveResult:
    """Branch-and-bound with the reference's options (solver.py:441-456):
    time_limit_s, node_limit, gap_target, branch_order, dive, telemetry_every,
    bound ("surrogate" or anything else for the plain bound), incumbent."""
    options = dict(options or {})
    time_limit = options.get("time_limit_s")
    node_limit = options.get("node_limit")
    gap_target = options.get("gap_target")
    if gap_target is not None:
        gap_target = Fraction(gap_target)
    branch_order = options.get("branch_order", "paper")
    if branch_order not in BRANCH_ORDERS:
        raise ValueError(f"branch_order must be one of {BRANCH_ORDERS}")
    dive = options.get("dive", "bound")
    if dive not in ("bound", "static"):
        raise ValueError(f"dive must be 'bound' or 'static', got {dive!r}")
    telemetry_every = int(options.get("telemetry_every", 8192))
    surrogate = options.get("bound", "surrogate") == "surrogate"

    start = time.monotonic()
    nat = _native_of(model, surrogate)
    S = nat.scale

    order = np.array(_static_order(model, branch_order), dtype=np.int32)
    pref = np.array([1 if v.kind in _PREF1 else 0 for v in model.var_ids], dtype=np.int8)
    inc = options.get("incumbent")
    has_inc, inc_obj, inc_vals = 0, np.zeros(2, dtype=np.int64), np.zeros(1, dtype=np.int8)
    if inc is not None:
        seeded = evaluate_assignment(model, inc)
        if seeded["feasible"]:
            has_inc = 1
            inc_obj = _i128([seeded["objective"] * S])
            inc_vals = np.array([int(x) for x in inc], dtype=np.int8)
    opts = np.array([-1 if node_limit is None else int(node_limit), telemetry_every, 1 if dive == "bound" else 0,
                     1 if branch_order == "most-tight" else 0,
                     0 if gap_target is None else gap_target.numerator,
                     0 if gap_target is None else gap_target.denominator, S], dtype=np.int64)
    nodes = np.zeros(1, dtype=np.int64)
    res = np.zeros(10, dtype=np.int64)
    code = nat.lib.monet_bnb_solve(C.c_void_p(nat.h), _p(opts),
                                   C.c_double(-1.0 if time_limit is None else float(time_limit)), _p(order),
                                   len(order), _p(pref), has_inc, _p(inc_obj), _p(inc_vals), _p(nodes), _p(res))
    elapsed = time.monotonic() - start
    telemetry = []
    kinds = np.zeros(4, dtype=np.int32)
    counts = np.zeros(2, dtype=np.int64)
    vals = np.zeros(8, dtype=np.int64)
    for i in range(nat.lib.monet_bnb_n_events(C.c_void_p(nat.h))):
        nat.lib.monet_bnb_event(C.c_void_p(nat.h), i, _p(kinds), _p(counts), _p(vals))
        inc_v = Fraction(_from128(vals, 0), S) if kinds[1] else None
        bnd = Fraction(_from128(vals, 1), S) if kinds[2] else None
        gap = Fraction(_from128(vals, 2), _from128(vals, 3)) if kinds[3] else None
        telemetry.append({"event": _EVENTS[kinds[0]], "nodes": int(counts[0]), "elapsed_ms": int(counts[1]),
                          "incumbent": None if inc_v is None else cost_str(inc_v),
                          "bound": None if bnd is None else cost_str(bnd),
                          "gap": None if gap is None else cost_str(gap)})
    status = _STATUS[code]
    n_nodes = int(nodes[0])
    if status == "infeasible":
        return SolveResult(status, None, None, None, None, n_nodes, elapsed, telemetry, model)
    if status == "timeout-no-incumbent":
        lb = Fraction(_from128(res, 1), S) if res[8] else None
        return SolveResult(status, None, None, lb, None, n_nodes, elapsed, telemetry, model)
    best = np.empty(model.n_vars, dtype=np.int8)
    nat.lib.monet_bnb_best(C.c_void_p(nat.h), _p(best))
    obj = Fraction(_from128(res, 0), S)
    assignment = [int(x) for x in best]
    if status == "optimal":
        return SolveResult(status, obj, assignment, obj, Fraction(0), n_nodes, elapsed, telemetry, model)
    gap = Fraction(_from128(res, 2), _from128(res, 3)) if res[8] else None
    return SolveResult(status, obj, assignment, Fraction(_from128(res, 1), S), gap, n_nodes, elapsed, telemetry,
                       model)

"""The 0-1 program that jointly picks checkpointing and implementations.

Same model as the reference (pkg/src/remsched/ilp.py:1-604): identical
variables in identical registration order, identical rows (terms, senses,
right-hand sides, tags) in identical order, identical objective and
fixings.  That identity is what makes the branch-and-bound's decisions
bit-exact against the reference (tests/test_ilp_parity.py pins it with
fixtures the reference generated) and the LP export byte-identical.

Variable families (all binary), cf. ilp.py:3-12:
    DeltaFwd(i,l)  DeltaBwd(t,l)  S(row,u)  R(t,u)  DeltaRe(t,i,l)
    Q(t,i)  P(t,j)  Alpha(t,l,u) = DeltaBwd(t,l) * S(t,u) (linearized)

The build is organised as a list of row emitters, one per row family, each
a generator over (terms, sense, rhs, tag); memory coefficients are integer
bytes, objective coefficients exact Fractions.
"""

from __future__ import annotations

import io
from dataclasses import dataclass, field
from fractions import Fraction

from .costmodel import Catalog
from .graph import DependencySets, Graph
from .units import FormatError

__all__ = ["VAR_KINDS", "VarId", "Row", "Model", "build_model", "assignment_from_schedule",
           "evaluate_assignment", "export_lp", "export_lp_string"]

VAR_KINDS = ("DeltaFwd", "DeltaBwd", "S", "R", "DeltaRe", "Q", "P", "Alpha")

_NAME_FMT = {  # ilp.py:50-66
    "S": lambda v: f"s_{v.row}_{v.node}",
    "R": lambda v: f"r_{v.row}_{v.node}",
    "DeltaFwd": lambda v: f"df_{v.node}_{v.variant}",
    "DeltaRe": lambda v: f"dr_{v.row}_{v.node}_{v.variant}",
    "DeltaBwd": lambda v: f"db_{v.row}_{v.variant}",
    "Q": lambda v: f"q_{v.row}_{v.node}",
    "P": lambda v: f"p_{v.row}_{v.node}",
    "Alpha": lambda v: f"al_{v.row}_{v.variant}_{v.node}",
}


@dataclass(frozen=True)
class VarId:
    kind: str
    row: int = -1      # store row for S, stage for the other per-stage kinds
    node: int = -1     # node or storable id
    variant: int = -1  # implementation index

    def name(self) -> str:
        return _NAME_FMT[self.kind](self)


@dataclass(frozen=True)
class Row:
    terms: tuple[tuple[int, int], ...]  # (variable index, integer coefficient)
    sense: str                          # "<=" or "="
    rhs: int
    tag: str


@dataclass
class Model:
    g: Graph
    sets: DependencySets
    catalog: Catalog
    budget: int
    options: dict
    var_ids: list[VarId] = field(default_factory=list)
    var_index: dict[VarId, int] = field(default_factory=dict)
    rows: list[Row] = field(default_factory=list)
    objective: list[tuple[int, Fraction]] = field(default_factory=list)
    fixed: dict[int, int] = field(default_factory=dict)
    # one-hot groups the solver's bound uses: [(var, cost)] per forward node /
    # backward stage, and (R var, group) per (stage, node) rematerialization
    fwd_groups: list[list[tuple[int, Fraction]]] = field(default_factory=list)
    bwd_groups: list[list[tuple[int, Fraction]]] = field(default_factory=list)
    re_groups: list[tuple[int, list[tuple[int, Fraction]]]] = field(default_factory=list)

    @property
    def n_vars(self) -> int:
        return len(self.var_ids)

    def var(self, vid: VarId) -> int:
        return self.var_index[vid]

    def stats(self) -> dict:
        """Variable / row family counts (ilp.py:102-118)."""
        kinds = dict.fromkeys(VAR_KINDS, 0)
        for v in self.var_ids:
            kinds[v.kind] += 1
        fams: dict[str, int] = {}
        nnz = 0
        for r in self.rows:
            fam = r.tag.split("[", 1)[0]
            fams[fam] = fams.get(fam, 0) + 1
            nnz += len(r.terms)
        return {"budget": self.budget,
                "vars": {**{k: c for k, c in kinds.items() if c}, "total": self.n_vars},
                "fixed": len(self.fixed),
                "rows": {**dict(sorted(fams.items())), "total": len(self.rows)},
                "nonzeros": nnz}


class _Builder:
    """State shared by the row emitters of one build."""

    def __init__(self, m: Model, inplace: bool):
        g, cat = m.g, m.catalog
        self.m, self.g, self.cat, self.inplace = m, g, cat, inplace
        self.st = g.storables
        self.bit = {u.id: b for b, u in enumerate(self.st)}
        self.size = [u.nbytes for u in self.st]
        self.stages = list(g.stage_nodes)
        self.T = len(self.stages)
        self.S: dict[tuple[int, int], int] = {}
        self.R: dict[tuple[int, int], int] = {}
        self.DR: dict[tuple[int, int, int], int] = {}
        self.Q: dict[tuple[int, int], int] = {}
        self.P: dict[tuple[int, int], int] = {}
        self.AL: dict[tuple[int, int, int], int] = {}
        self.dmask: dict[tuple[int, int], int] = {}
        # an in-place rewrite reuses its first input's buffer (ilp.py:193-198)
        self.elig = [i for i in range(1, g.n + 1)
                     if any(v.inplace_capable for v in cat.fwd(i)) and g.deps(i)
                     and g.output_bytes(i) == g.output_bytes(g.deps(i)[0])]

    def new(self, vid: VarId, cost=None, fix=None) -> int:
        m = self.m
        idx = len(m.var_ids)
        m.var_ids.append(vid)
        m.var_index[vid] = idx
        if cost is not None:
            m.objective.append((idx, cost))
        if fix is not None:
            m.fixed[idx] = fix
        return idx

    def stage_iter(self):
        return zip(range(1, self.T + 1), self.stages)

    def db(self, t: int, l: int) -> int:
        return self.m.bwd_groups[t - 1][l][0]

    # ------------------------------------------------------------ variables
    def variables(self):
        g, cat, m = self.g, self.cat, self.m
        for i in range(1, g.n + 1):
            m.fwd_groups.append([(self.new(VarId("DeltaFwd", node=i, variant=l), v.cost), v.cost)
                                 for l, v in enumerate(cat.fwd(i))])
        for t, k in self.stage_iter():
            m.bwd_groups.append([(self.new(VarId("DeltaBwd", row=t, variant=l), v.cost), v.cost)
                                 for l, v in enumerate(cat.bwd(k))])
        for row in range(self.T + 1):
            last = row == self.T and self.T > 0  # the last store row is empty (ilp.py:165-169)
            for b, u in enumerate(self.st):
                self.S[(row, b)] = self.new(VarId("S", row=row, node=u.id), fix=0 if last else None)
        for t, k in self.stage_iter():
            for b, u in enumerate(self.st):
                self.R[(t, b)] = self.new(VarId("R", row=t, node=u.id), fix=0 if u.pos > k else None)
        for t, k in self.stage_iter():
            for i in range(1, g.n + 1):
                grp = []
                for l, v in enumerate(cat.fwd(i)):
                    idx = self.new(VarId("DeltaRe", row=t, node=i, variant=l), v.cost,
                                   fix=0 if i > k else None)
                    self.DR[(t, i, l)] = idx
                    grp.append((idx, v.cost))
                m.re_groups.append((self.R[(t, self.bit[i])], grp))
        if self.inplace:
            for t, k in self.stage_iter():
                live = [i for i in self.elig if i <= k]
                for i in live:
                    self.Q[(t, i)] = self.new(VarId("Q", row=t, node=i))
                for j in sorted({g.deps(i)[0] for i in live}):
                    self.P[(t, j)] = self.new(VarId("P", row=t, node=j))
        for t, k in self.stage_iter():
            for l, v in enumerate(cat.bwd(k)):
                dm = 0
                for d in v.deps:
                    dm |= 1 << self.bit[d]
                self.dmask[(t, l)] = dm
                for b, u in enumerate(self.st):
                    if not dm >> b & 1:
                        self.AL[(t, l, b)] = self.new(VarId("Alpha", row=t, variant=l, node=u.id))

    # ------------------------------------------------------------ row families
    def choose_rows(self):
        for i, grp in enumerate(self.m.fwd_groups, start=1):
            yield [(v, 1) for v, _ in grp], "=", 1, f"choose-forward[n{i}]"
        for t, grp in enumerate(self.m.bwd_groups, start=1):
            yield [(v, 1) for v, _ in grp], "=", 1, f"choose-backward[t{t}]"
        for t, _ in self.stage_iter():
            for i in range(1, self.g.n + 1):
                terms = [(self.DR[(t, i, l)], 1) for l in range(len(self.cat.fwd(i)))]
                yield terms + [(self.R[(t, self.bit[i])], -1)], "=", 0, f"recompute-impl[t{t},n{i}]"

    def carry_rows(self):
        for t, _ in self.stage_iter():
            for b, u in enumerate(self.st):
                yield ([(self.S[(t, b)], 1), (self.S[(t - 1, b)], -1), (self.R[(t, b)], -1)], "<=", 0,
                       f"store-carry[t{t},u{u.id}]")

    def _needs(self, t: int, b: int):
        """-DeltaBwd terms of the stage-t backward variants that read storable bit b."""
        return [(self.db(t, l), -1) for l in range(len(self.m.bwd_groups[t - 1]))
                if self.dmask[(t, l)] >> b & 1]

    def dependency_rows(self):
        g, R, S, bit = self.g, self.R, self.S, self.bit
        for t, k in self.stage_iter():
            for i in range(1, k + 1):
                for j in g.deps(i):
                    src = self.P.get((t, j), R[(t, bit[j])])
                    yield ([(R[(t, bit[i])], 1), (S[(t, bit[j])], -1), (src, -1)], "<=", 0,
                           f"recompute-deps[t{t},n{i},d{j}]")
            for u in self.st:
                if not u.is_intermediate or u.pos > k:
                    continue
                b = bit[u.id]
                yield ([(R[(t, b)], 1), (R[(t, bit[u.creator])], -1)], "<=", 0,
                       f"intermediate-with-creator[t{t},u{u.id}]")
                yield ([(R[(t, b)], 1), (S[(t, b)], -1)] + self._needs(t, b), "<=", 0,
                       f"intermediate-usefulness[t{t},u{u.id}]")

    def usefulness_rows(self):
        # a rebuilt node output must feed the row, the backward or another
        # rebuild of the same sweep (ilp.py:267-296)
        g, R, S, bit = self.g, self.R, self.S, self.bit
        consumers = {i: [] for i in range(1, g.n + 1)}
        for c in range(1, g.n + 1):
            for j in g.deps(c):
                consumers[j].append(c)
        ints = {i: [] for i in range(1, g.n + 1)}
        for u in self.st:
            if u.is_intermediate:
                ints[u.creator].append(u.id)
        for t, k in self.stage_iter():
            for u in self.st:
                if u.is_intermediate or u.pos > k:
                    continue
                b = bit[u.id]
                terms = [(R[(t, b)], 1), (S[(t, b)], -1)] + self._needs(t, b)
                terms += [(R[(t, bit[c])], -1) for c in consumers[u.id] if c <= k]
                terms += [(R[(t, bit[w])], -1) for w in ints[u.id]]
                yield terms, "<=", 0, f"recompute-usefulness[t{t},u{u.id}]"

    def backward_rows(self):
        R, S, bit = self.R, self.S, self.bit
        for t, k in self.stage_iter():
            for l, v in enumerate(self.cat.bwd(k)):
                for d in v.deps:
                    b = bit[d]
                    yield ([(self.db(t, l), 1), (S[(t, b)], -1), (R[(t, b)], -1)], "<=", 0,
                           f"backward-needs[t{t},l{l},u{d}]")
        # telescoped carry + needs: kept since the forward or rebuilt by stage t
        for t, k in self.stage_iter():
            for l, v in enumerate(self.cat.bwd(k)):
                for d in v.deps:
                    b = bit[d]
                    terms = [(self.db(t, l), 1), (S[(0, b)], -1)]
                    terms += [(R[(t2, b)], -1) for t2 in range(1, t + 1)]
                    yield terms, "<=", 0, f"reach[t{t},l{l},u{d}]"

    def inplace_rows(self):
        if not self.inplace:
            return
        g, R, S, bit = self.g, self.R, self.S, self.bit
        for t, k in self.stage_iter():
            for i in self.elig:
                if i > k:
                    continue
                q, j = self.Q[(t, i)], g.deps(i)[0]
                p = self.P[(t, j)]
                cap = [(self.DR[(t, i, l)], -1) for l, v in enumerate(self.cat.fwd(i)) if v.inplace_capable]
                yield [(q, 1)] + cap, "<=", 0, f"inplace-variant[t{t},n{i}]"
                yield [(q, 1), (R[(t, bit[i])], -1)], "<=", 0, f"inplace-needs-recompute[t{t},n{i}]"
                yield [(S[(t - 1, bit[i])], 1), (q, 2)], "<=", 2, f"inplace-fresh-output[t{t},n{i}]"
                yield ([(R[(t, bit[j])], 1), (p, -1), (q, -2)], "<=", 0,
                       f"inplace-release-lower[t{t},n{i},d{j}]")
                yield [(p, 1), (q, 2)], "<=", 2, f"inplace-release-upper[t{t},n{i},d{j}]"
            for j in sorted({g.deps(i)[0] for i in self.elig if i <= k}):
                yield [(self.P[(t, j)], 1), (R[(t, bit[j])], -1)], "<=", 0, f"inplace-release-cap[t{t},d{j}]"

    def linearization_rows(self):
        for (t, l, b), a in self.AL.items():
            db, s, uid = self.db(t, l), self.S[(t, b)], self.st[b].id
            yield [(db, 1), (s, 1), (a, -1)], "<=", 1, f"linearization-lb[t{t},l{l},u{uid}]"
            yield [(a, 1), (db, -1)], "<=", 0, f"linearization-impl[t{t},l{l},u{uid}]"
            yield [(a, 1), (s, -1)], "<=", 0, f"linearization-store[t{t},l{l},u{uid}]"

    def memory_rows(self):
        g, m, sets, cat = self.g, self.m, self.m.sets, self.cat
        st, S, size, bit = self.st, self.S, self.size, self.bit
        budget = m.budget
        # forward step i (Eq. 1): output + locals + params + stored row-0 bytes + workspace
        for i in range(1, g.n + 1):
            local = sets.local_fwd[i]
            terms = [(v, cat.fwd(i)[l].workspace_bytes) for l, (v, _) in enumerate(m.fwd_groups[i - 1])
                     if cat.fwd(i)[l].workspace_bytes]
            for b, u in enumerate(st):
                before = u.pos <= i if u.is_intermediate else (u.pos < i and u.id not in local)
                if before:
                    terms.append((S[(0, b)], u.nbytes))
            const = g.output_bytes(i) + g.params_bytes + sum(g.output_bytes(j) for j in local)
            yield terms, "<=", budget - const, f"forward-mem[n{i}]"
        # backward execution of stage t under each variant
        for t, k in self.stage_iter():
            rhs = budget - g.params_bytes - sets.grad_live_bytes[k]
            for l, v in enumerate(cat.bwd(k)):
                dm = self.dmask[(t, l)]
                dep_bytes = sum(size[b] for b in range(len(st)) if dm >> b & 1)
                terms = [(self.db(t, l), v.workspace_bytes + dep_bytes)]
                terms += [(self.AL[(t, l, b)], size[b]) for b in range(len(st)) if not dm >> b & 1]
                yield terms, "<=", rhs, f"backward-mem[t{t},l{l}]"
        # recompute sweep position i of stage t: active (i rebuilt) and settled
        nbwd = lambda k: len(cat.bwd(k))  # noqa: E731
        for t, k in self.stage_iter():
            rhs = budget - g.params_bytes - sets.grad_live_bytes[k]
            for i in range(1, k + 1):
                lb_ids = sets.local_bound[(i, k)]
                lb_bytes = sum(g.output_bytes(j) for j in lb_ids)
                strict = [b for b, u in enumerate(st) if (u.pos <= i if u.is_intermediate else u.pos < i)]
                incl = strict + [bit[i]]
                tail = [b for b, u in enumerate(st) if u.pos > i]

                terms = [(self.DR[(t, i, l)], v.workspace_bytes) for l, v in enumerate(cat.fwd(i))
                         if v.workspace_bytes]
                terms.append((self.R[(t, bit[i])], g.output_bytes(i) + lb_bytes))
                for l in range(nbwd(k)):
                    dm = self.dmask[(t, l)]
                    coef = sum(size[b] for b in strict if dm >> b & 1 and st[b].id not in lb_ids)
                    if coef:
                        terms.append((self.db(t, l), coef))
                    terms += [(self.AL[(t, l, b)], size[b]) for b in strict
                              if not dm >> b & 1 and st[b].id not in lb_ids]
                terms += [(S[(t - 1, b)], size[b]) for b in tail]
                yield terms, "<=", rhs, f"recompute-mem[t{t},n{i}]"

                terms = []
                for l in range(nbwd(k)):
                    dm = self.dmask[(t, l)]
                    coef = sum(size[b] for b in incl if dm >> b & 1)
                    if coef:
                        terms.append((self.db(t, l), coef))
                    terms += [(self.AL[(t, l, b)], size[b]) for b in incl if not dm >> b & 1]
                terms += [(S[(t - 1, b)], size[b]) for b in tail]
                yield terms, "<=", rhs, f"settled-mem[t{t},n{i}]"

    FAMILIES = ("choose_rows", "carry_rows", "dependency_rows", "usefulness_rows", "backward_rows",
                "inplace_rows", "linearization_rows", "memory_rows")


def build_model(g: Graph, sets: DependencySets, catalog: Catalog, budget: int,
                options: dict | None = None) -> Model:
    """Build the 0-1 program for one byte budget (ilp.py:121-421)."""
    options = dict(options or {})
    if "bound_kind" in options and options["bound_kind"] != sets.bound_kind:
        raise ValueError(f"options bound_kind {options['bound_kind']!r} does not match the "
                         f"dependency sets ({sets.bound_kind!r})")
    if budget < 0:
        raise ValueError(f"budget must be nonnegative, got {budget}")
    m = Model(g, sets, catalog, budget, options)
    b = _Builder(m, options.get("inplace", True))
    b.variables()
    for fam in _Builder.FAMILIES:
        for terms, sense, rhs, tag in getattr(b, fam)():
            m.rows.append(Row(tuple(terms), sense, rhs, tag))
    return m


def assignment_from_schedule(model: Model, schedule) -> list[int]:
    """The model's 0-1 vector for a schedule, taken at face value (ilp.py:424-484)."""
    g, cat, var = model.g, model.catalog, model.var_index
    vals = [0] * model.n_vars

    def fwd_index(i: int, name: str) -> int:
        for l, v in enumerate(cat.fwd(i)):
            if v.name == name:
                return l
        raise ValueError(f"node {i} has no forward implementation {name!r}")

    def on(vid):
        vals[var[vid]] = 1

    for i, name in enumerate(schedule.forward_impls, start=1):
        on(VarId("DeltaFwd", node=i, variant=fwd_index(i, name)))
    for uid in schedule.forward_store:
        on(VarId("S", row=0, node=uid))
    is_int = {u.id: u.is_intermediate for u in g.storables}
    for t, plan in enumerate(schedule.stages, start=1):
        for uid in plan.store:
            on(VarId("S", row=t, node=uid))
        for uid, impl in plan.recompute:
            on(VarId("R", row=t, node=uid))
            if is_int[uid]:
                continue
            if impl is None:
                raise ValueError(f"recompute of node {uid} at stage {t} carries no implementation choice")
            on(VarId("DeltaRe", row=t, node=uid, variant=fwd_index(uid, impl)))
        k = plan.node
        hits = [l for l, v in enumerate(cat.bwd(k)) if v.name == plan.backward_impl]
        if len(hits) != 1:
            raise ValueError(f"stage {t} has no backward implementation {plan.backward_impl!r}")
        on(VarId("DeltaBwd", row=t, variant=hits[0]))
        overwritten = set()
        for i in plan.inplace:
            key = VarId("Q", row=t, node=i)
            if key not in var:
                raise ValueError(f"schedule runs node {i} in place at stage {t} but the model has "
                                 f"no such variable")
            vals[var[key]] = 1
            overwritten.add(g.deps(i)[0])
        for vid, idx in var.items():
            if vid.kind == "P" and vid.row == t and vid.node not in overwritten:
                vals[idx] = vals[var[VarId("R", row=t, node=vid.node)]]
    for vid, idx in var.items():
        if vid.kind == "Alpha":
            vals[idx] = (vals[var[VarId("DeltaBwd", row=vid.row, variant=vid.variant)]]
                         & vals[var[VarId("S", row=vid.row, node=vid.node)]])
    return vals


def evaluate_assignment(model: Model, assignment) -> dict:
    """Check a full 0-1 vector against every row and fixing (ilp.py:487-510).

    Independent of the closed-form memory evaluators (memmodel.py)."""
    if len(assignment) != model.n_vars:
        raise ValueError(f"assignment has {len(assignment)} values, model has {model.n_vars} variables")
    bad = [f"not-binary[{model.var_ids[i].name()}]" for i, x in enumerate(assignment) if x not in (0, 1)]
    bad += [f"fixed-var[{model.var_ids[i].name()}]" for i, x in model.fixed.items() if assignment[i] != x]
    for r in model.rows:
        act = sum(c * assignment[v] for v, c in r.terms)
        if not (act == r.rhs if r.sense == "=" else act <= r.rhs):
            bad.append(r.tag)
    obj = sum((c * assignment[v] for v, c in model.objective), Fraction(0))
    return {"feasible": not bad, "violations": bad, "objective": obj}


# ---------------------------------------------------------------- LP export
def _decimal(c) -> str:
    """Exact decimal text of a rational with a terminating expansion."""
    f = Fraction(c)
    den, e2, e5 = f.denominator, 0, 0
    while den % 2 == 0:
        den, e2 = den // 2, e2 + 1
    while den % 5 == 0:
        den, e5 = den // 5, e5 + 1
    if den != 1:
        raise FormatError(f"coefficient {f} has no exact decimal form for the LP export")
    shift = max(e2, e5)
    scaled = f.numerator * 10 ** shift // f.denominator
    if shift == 0:
        return str(scaled)
    digits = str(abs(scaled)).rjust(shift + 1, "0")
    return ("-" if scaled < 0 else "") + digits[:-shift] + "." + digits[-shift:]


def _expr_lines(parts) -> list[str]:
    """'c name' pieces joined with signs, wrapped at 200 characters (ilp.py:536-554)."""
    pieces = []
    for n, (coef, name) in enumerate(parts):
        mag = abs(Fraction(coef))
        body = name if mag == 1 else f"{_decimal(mag)} {name}"
        sign = "-" if coef < 0 else ("+" if n else "")
        pieces.append(f"{sign} {body}" if sign else body)
    lines, cur = [], ""
    for piece in pieces:
        if cur and len(cur) + len(piece) + 1 > 200:
            lines.append(cur)
            cur = piece
        else:
            cur = f"{cur} {piece}" if cur else piece
    if cur:
        lines.append(cur)
    return lines


def _slug(tag: str) -> str:
    return "".join(ch if ch.isalnum() else "_" for ch in tag).strip("_")


def export_lp(model: Model, sink) -> None:
    """Write the model as LP text, byte-identical to the reference (ilp.py:561-598)."""
    close = isinstance(sink, (str, bytes)) or hasattr(sink, "__fspath__")
    fh = open(sink, "w", encoding="utf-8", newline="\n") if close else sink
    try:
        names = [v.name() for v in model.var_ids]
        out = ["\\ joint rematerialization and implementation schedule\n",
               f"\\ budget {model.budget} bytes, {model.n_vars} binaries, {len(model.rows)} rows\n",
               "Minimize\n"]
        obj = _expr_lines([(c, names[v]) for v, c in model.objective]) or ["0 " + names[0]]
        out += [(" obj: " if n == 0 else "      ") + line + "\n" for n, line in enumerate(obj)]
        out.append("Subject To\n")
        for ri, r in enumerate(model.rows):
            label = f" c{ri}_{_slug(r.tag)}: "
            lines = _expr_lines([(c, names[v]) for v, c in r.terms] or [(0, names[0])])
            lines[-1] += f" {'=' if r.sense == '=' else '<='} {r.rhs}"
            out += [(label if n == 0 else " " * len(label)) + line + "\n" for n, line in enumerate(lines)]
        out.append("Bounds\n")
        out += [f" {names[i]} = {model.fixed[i]}\n" for i in sorted(model.fixed)]
        out.append("Binary\n")
        out += [f" {nm}\n" for nm in names]
        out.append("End\n")
        fh.write("".join(out))
    finally:
        if close:
            fh.close()


def export_lp_string(model: Model) -> str:
    buf = io.StringIO()
    export_lp(model, buf)
    return buf.getvalue()

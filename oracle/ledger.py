"""Byte ledger of a schedule, restated from the reference simulator (test oracle).

Follows pkg/src/remsched/schedule.py:320-465 (Alg. 1-2 of PAPER.md:104-160)
but works directly on the JSON documents (graph, catalog, schedule) so it
shares no code with the product.  Returns the trace rows
(step, op, mem_before, mem_peak, mem_after, cost) and the peak; raises
LedgerError wherever the reference raises SimulationError.
"""
from fractions import Fraction


class LedgerError(RuntimeError):
    pass


def _cost(v):
    return Fraction(v) if not isinstance(v, str) else Fraction(v)


def replay(graph: dict, catalog: dict, schedule: dict):
    nodes = {nd["id"]: nd for nd in graph["nodes"]}
    n = len(nodes)
    deps = {i: sorted(nodes[i]["deps"]) for i in nodes}
    out_bytes = {i: nodes[i]["output_bytes"] for i in nodes}
    inter = {u["id"]: u for u in graph.get("intermediates", [])}
    size = dict(out_bytes)
    size.update({u: inter[u]["bytes"] for u in inter})
    pos = {i: i for i in nodes}
    pos.update({u: inter[u]["creator"] for u in inter})
    grad_bytes = {b["node"]: b["grad_bytes"] for b in graph.get("backward", [])}
    readers = {i: [] for i in nodes}
    for i in nodes:
        for j in deps[i]:
            readers[j].append(i)
    last_use = {i: max(readers[i]) if readers[i] else i for i in nodes}
    ints_by_creator = {}
    for u in sorted(inter):
        ints_by_creator.setdefault(inter[u]["creator"], []).append(u)

    fwd_var = {e["node"]: {v["name"]: v for v in e["variants"]} for e in catalog["forward"]}
    bwd_var = {e["node"]: {v["name"]: v for v in e["variants"]} for e in catalog["backward"]}

    mem = graph.get("params_bytes", 0)
    peak_all = mem
    rows = []
    act, grad = {}, {}

    def emit(label, before, peak, cost):
        nonlocal peak_all
        peak_all = max(peak_all, peak)
        rows.append((len(rows) + 1, label, before, peak, mem, _cost(cost)))

    row0 = set(schedule["forward_store"])
    for i in range(1, n + 1):
        name = schedule["forward_impls"][i - 1]
        var = fwd_var[i][name]
        if any(j not in act for j in deps[i]):
            raise LedgerError(f"forward {i} reads a dead input")
        keep = [u for u in ints_by_creator.get(i, []) if u in row0]
        before = mem
        grow = out_bytes[i] + sum(size[u] for u in keep)
        peak = mem + grow + var.get("workspace_bytes", 0)
        mem += grow
        act[i] = out_bytes[i]
        for u in keep:
            act[u] = size[u]
        for j in [j for j in act if j in nodes and j <= i]:
            if j not in row0 and last_use[j] <= i:
                mem -= act.pop(j)
        emit(f"forward {i} [{name}]", before, peak, var["cost"])
    if set(act) != row0:
        raise LedgerError("forward live set differs from row 0")

    carried = row0
    has_bwd = set(grad_bytes)
    for t, st in enumerate(schedule["stages"], start=1):
        k = st["node"]
        keep = set(st["store"])
        bvar = bwd_var[k][st["backward_impl"]]
        for u in sorted(carried - keep):
            if u in act:
                mem -= act.pop(u)
        fwd_entries = [(u, impl) for u, impl in st["recompute"] if u not in inter]
        planned = {}
        for u, _ in st["recompute"]:
            if u in inter:
                planned.setdefault(inter[u]["creator"], []).append(u)
        last = {}
        for e, (i, _) in enumerate(fwd_entries):
            for j in deps[i]:
                last[j] = e
            last[i] = e
            for u in planned.get(i, []):
                last[u] = e
        bslot = len(fwd_entries)
        for d in bvar["deps"]:
            last[d] = bslot

        def release(slot):
            nonlocal mem
            for u, s in last.items():
                if s == slot and u not in keep and u in act:
                    mem -= act.pop(u)

        inplace = set(st.get("inplace", []))
        for e, (i, impl) in enumerate(fwd_entries):
            if impl is None:
                raise LedgerError(f"stage {t}: recompute {i} without impl")
            var = fwd_var[i][impl]
            if any(j not in act for j in deps[i]):
                raise LedgerError(f"stage {t}: recompute {i} reads a dead input")
            ib = sum(size[u] for u in planned.get(i, []))
            before = mem
            if i in inplace:
                j = deps[i][0]
                if act.get(j) != out_bytes[i]:
                    raise LedgerError("in-place recompute without a same-size input")
                peak = mem + ib + var.get("workspace_bytes", 0)
                mem -= act.pop(j)
                label = f"recompute {i} [{impl}] inplace"
            else:
                peak = mem + out_bytes[i] + ib + var.get("workspace_bytes", 0)
                label = f"recompute {i} [{impl}]"
            act[i] = out_bytes[i]
            mem += out_bytes[i]
            for u in planned.get(i, []):
                act[u] = size[u]
                mem += size[u]
            release(e)
            emit(label, before, peak, var["cost"])

        if any(d not in act for d in bvar["deps"]):
            raise LedgerError(f"stage {t}: backward of {k} reads a dead tensor")
        before = mem
        if k not in grad:
            if t != 1:
                raise LedgerError(f"stage {t}: gradient of {k} never produced")
            grad[k] = grad_bytes[k]
            mem += grad[k]
        for j in deps[k]:
            if j in has_bwd and j not in grad:
                grad[j] = grad_bytes[j]
                mem += grad[j]
        peak = mem + bvar.get("workspace_bytes", 0)
        mem -= grad.pop(k)
        release(bslot)
        emit(f"backward {k} [{st['backward_impl']}]", before, peak, bvar["cost"])
        if set(act) != keep:
            raise LedgerError(f"stage {t}: live set differs from its row")
        carried = keep

    if schedule["stages"] and (act or grad or mem != graph.get("params_bytes", 0)):
        raise LedgerError("replay ended with live tensors or unaccounted bytes")
    return rows, peak_all


def trace_csv(rows, peak) -> str:
    def c(x):
        return str(x.numerator) if x.denominator == 1 else f"{x.numerator}/{x.denominator}"
    out = ["step,op,mem_before,mem_peak,mem_after,cost"]
    out += [f"{s},{op},{b},{p},{a},{c(cost)}" for s, op, b, p, a, cost in rows]
    out.append(f"total,,,{peak},,{c(sum((r[5] for r in rows), Fraction(0)))}")
    return "\n".join(out) + "\n"

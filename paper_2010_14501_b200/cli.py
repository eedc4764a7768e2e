"""Command line for the GPU path (`execute` / `train` reuse the reference's
exit-code table, pkg/src/remsched/cli.py:43-50).

    python -m paper_2010_14501_b200 trace    --arch resnet50 --batch 184 [--image 224] [--fuse] -o graph.json
    python -m paper_2010_14501_b200 profile  --arch resnet50 --batch 184 [--fuse] -o catalog.json   (GPU)
    python -m paper_2010_14501_b200 plan     --arch resnet50 --batch 184 --budget-gib 8 [--catalog c.json] -o s.json
    python -m paper_2010_14501_b200 execute  --arch resnet50 --batch 184 --schedule s.json [--budget-gib 8]  (GPU)
    python -m paper_2010_14501_b200 train    --arch resnet50 --batch 184 --budget-gib 8 --steps 10          (GPU)

Exit codes: 0 ok, 1 bad input, 2 feasible with a gap, 3 infeasible (no schedule fits),
4 no incumbent, 5 invalid schedule (the simulator rejects it), 6 over budget (the
planned physical footprint exceeds the budget), 7 mismatch.
"""
from __future__ import annotations

import argparse
import json
import sys

EXIT_OK = 0
EXIT_BAD_INPUT = 1
EXIT_FEASIBLE_GAP = 2
EXIT_INFEASIBLE = 3
EXIT_NO_INCUMBENT = 4
EXIT_INVALID_SCHEDULE = 5
EXIT_OVER_BUDGET = 6
EXIT_MISMATCH = 7


def _net(a):
    from .tracer import build_network, default_classes, parse_image

    return build_network(a.arch, a.batch, parse_image(a.image), num_classes=a.classes or default_classes(a.arch),
                         fuse=a.fuse)


def _docs(a, net):
    from . import load_catalog, load_graph

    gdoc = net.graph_doc()
    g = load_graph(gdoc)
    cdoc = json.loads(open(a.catalog).read()) if getattr(a, "catalog", None) else net.catalog_doc()
    if "catalog" in cdoc:  # a frozen profile (tools/profile_catalog.py) wraps the document
        cdoc = cdoc["catalog"]
    return g, load_catalog(cdoc, g)


def _write(obj, path):
    text = json.dumps(obj, indent=1, sort_keys=True) + "\n"
    if path in (None, "-"):
        sys.stdout.write(text)
    else:
        with open(path, "w") as f:
            f.write(text)


def cmd_trace(a) -> int:
    _write(_net(a).graph_doc(), a.output)
    return EXIT_OK


def cmd_profile(a) -> int:
    from .profiler import profile_network

    net = _net(a)
    _write(net.catalog_doc(profile_network(net)), a.output)
    return EXIT_OK


def _budget(a, g) -> int:
    return int(a.budget_gib * (1 << 30)) if a.budget_gib else g.params_bytes + (1 << 62)


def cmd_plan(a) -> int:
    from . import schedule_to_doc
    from .planner import plan_schedule

    net = _net(a)
    g, cat = _docs(a, net)
    sched, info = plan_schedule(g, cat, _budget(a, g), kinds=net.storable_kinds(), exact_time_s=a.exact)
    if sched is None:
        print(json.dumps({"status": "infeasible", **info}), file=sys.stderr)
        return EXIT_INFEASIBLE
    _write({"planner": info, "schedule": schedule_to_doc(sched)}, a.output)
    return EXIT_OK


def _run(a, net, g, cat, sched, steps) -> int:
    import torch

    from .engine import BudgetExceeded, Runtime
    from .schedule import SimulationError

    try:
        rt = Runtime(net, budget_bytes=_budget(a, g) if a.budget_gib else None)
        gen = torch.Generator().manual_seed(0)
        hw = net.ops[0].shape[1:3]
        x = torch.randn(a.batch, 3, *hw, generator=gen)
        y = torch.randint(0, net.num_classes, (net.label_count(),), generator=gen)
        rt.set_batch(x.to(rt.device), y.to(rt.device))
        plan = rt.plan(sched, g, cat)
    except SimulationError as e:
        print(f"invalid schedule: {e}", file=sys.stderr)
        return EXIT_INVALID_SCHEDULE
    except BudgetExceeded as e:
        print(f"over budget: {e}", file=sys.stderr)
        return EXIT_OVER_BUDGET
    losses = []
    for _ in range(steps):
        rt.run(plan)
        losses.append(rt.loss_value())
    _write({"losses": losses, "ledger_peak_bytes": plan.ledger_peak, "ilp_bound_bytes": plan.bound_peak,
            "physical_peak_bytes": g.params_bytes + plan.arena_bytes, "launches_per_step": plan.launches},
           a.output)
    return EXIT_OK


def cmd_execute(a) -> int:
    from . import schedule_from_doc

    net = _net(a)
    g, cat = _docs(a, net)
    doc = json.loads(open(a.schedule).read())
    try:
        sched = schedule_from_doc(doc.get("schedule", doc))
    except (ValueError, KeyError) as e:
        print(f"bad schedule document: {e}", file=sys.stderr)
        return EXIT_BAD_INPUT
    return _run(a, net, g, cat, sched, 1)


def cmd_train(a) -> int:
    from .planner import plan_schedule

    net = _net(a)
    g, cat = _docs(a, net)
    sched, _ = plan_schedule(g, cat, _budget(a, g), kinds=net.storable_kinds(), exact_time_s=a.exact)
    if sched is None:
        return EXIT_INFEASIBLE
    return _run(a, net, g, cat, sched, a.steps)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2010_14501_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name, fn in (("trace", cmd_trace), ("profile", cmd_profile), ("plan", cmd_plan), ("execute", cmd_execute),
                     ("train", cmd_train)):
        p = sub.add_parser(name)
        p.set_defaults(fn=fn)
        p.add_argument("--arch", required=True)
        p.add_argument("--batch", type=int, required=True)
        p.add_argument("--image", default="224")
        p.add_argument("--classes", type=int, default=None)
        p.add_argument("--fuse", action="store_true", help="fused BN+ReLU(6) / add+ReLU / BN+add+ReLU operators")
        p.add_argument("-o", "--output", default="-")
        if name in ("plan", "execute", "train"):
            p.add_argument("--budget-gib", type=float, default=None)
            p.add_argument("--catalog", default=None, help="catalog JSON (default: analytic costs)")
        if name in ("plan", "train"):
            p.add_argument("--exact", type=float, default=None, help="seconds of exact ILP on small graphs")
        if name == "execute":
            p.add_argument("--schedule", required=True)
        if name == "train":
            p.add_argument("--steps", type=int, default=1)
    a = ap.parse_args(argv)
    try:
        return a.fn(a)
    except (ValueError, OSError, json.JSONDecodeError, NotImplementedError, AttributeError, KeyError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_BAD_INPUT

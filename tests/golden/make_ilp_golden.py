"""Golden ILP fixtures from the REFERENCE (remsched): model stats, LP export
digest, branch-and-bound results and oracle optima for small instances.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_ilp_golden.py

The GPU box has no /root/reference, so tests/test_ilp_parity.py checks the
product's ilp / solver / enumerate modules against this committed file.
"""
import hashlib
import json
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
import remsched as R  # noqa: E402  (the reference)

HERE = Path(__file__).resolve().parent
SOLVE_OPTS = [{"node_limit": 3000}, {"node_limit": 1500, "branch_order": "fixed"},
              {"node_limit": 600, "dive": "static"}, {"node_limit": 800, "branch_order": "most-tight"},
              {"node_limit": 2000, "gap_target": "1/10", "telemetry_every": 64}]


def instances():
    yield "resnet_toy", R.resnet_toy(), (700, 1000, 1200)
    for kind, n, seed in (("chain", 4, 0), ("residual", 5, 1), ("inception-toy", 5, 2), ("unet-toy", 5, 0)):
        g, c = R.generate_synthetic(kind, n, seed, fwd_variants=2, bwd_variants=2, intermediate_every=2,
                                    inplace_marks=True)
        yield f"{kind}-{n}-{seed}", (g, c), (6, 12, 40)


def main():
    out = []
    for name, (g, c), budgets in instances():
        case = {"name": name, "graph": R.graph_to_doc(g), "catalog": R.catalog_to_doc(c), "cells": []}
        sets = R.compute_dependency_sets(g, "upper")
        for budget in budgets:
            m = R.build_model(g, sets, c, budget, {"inplace": True, "bound_kind": "upper"})
            cell = {"budget": budget, "stats": m.stats(),
                    "lp_sha256": hashlib.sha256(R.export_lp_string(m).encode()).hexdigest(), "solves": []}
            for opts in SOLVE_OPTS:
                r = R.solve(m, dict(opts))
                cell["solves"].append({
                    "options": opts, "status": r.status, "nodes": r.nodes,
                    "objective": None if r.objective is None else R.format_cost(r.objective),
                    "lower_bound": None if r.lower_bound is None else R.format_cost(r.lower_bound),
                    "gap": None if r.gap is None else R.format_cost(r.gap),
                    "schedule": None if r.assignment is None else R.schedule_to_doc(R.decode(r, g, c)),
                    "telemetry": [{k: v for k, v in e.items() if k != "elapsed_ms"} for e in r.telemetry]})
            if g.n <= 6 and len(g.storables) <= 12:
                o = R.enumerate_schedules(g, c, budget)
                cell["oracle"] = {"feasible": o.feasible, "enumerated": o.enumerated_count,
                                  "optimum": None if o.optimum is None else R.format_cost(o.optimum),
                                  "model_peak": o.model_peak, "true_peak": o.true_peak,
                                  "schedule": None if o.schedule is None else R.schedule_to_doc(o.schedule)}
            case["cells"].append(cell)
        out.append(case)
    (HERE / "ilp_parity.json").write_text(json.dumps(out, sort_keys=True, indent=1) + "\n")
    print("wrote", HERE / "ilp_parity.json")


if __name__ == "__main__":
    main()

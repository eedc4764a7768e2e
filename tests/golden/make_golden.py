"""Generate golden fixtures by running the REFERENCE planner (remsched) here.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

/root/reference exists only in the build container, so its outputs are
committed under tests/golden/*.json and the GPU box never needs it.  Each
fixture holds the inputs (graph, catalog docs), the reference's schedule for a
budget (solve with a deterministic node limit and the CLI's heuristic warm
start, cli.py:129-140, or checkpoint_heuristic for the larger traced graphs),
its simulate() trace CSV (schedule.py:320, 468), the modeled peak from
check_schedule (oracle.py:287) and validate() tags.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import remsched as R  # noqa: E402  (the reference)


def cj(obj):
    return json.dumps(obj, sort_keys=True, indent=1) + "\n"


def solve_case(gdoc, cdoc, budget, node_limit=4000, warm=True, heuristic_only=False):
    g = R.load_graph(gdoc)
    cat = R.load_catalog(cdoc, g)
    sets = R.compute_dependency_sets(g, "upper")
    out = {"budget": budget}
    if heuristic_only:
        sched = R.checkpoint_heuristic(g, sets, cat, budget)
        out["status"] = "heuristic" if sched is not None else "none"
    else:
        model = R.build_model(g, sets, cat, budget, {"inplace": True, "bound_kind": "upper"})
        opts = {"node_limit": node_limit, "branch_order": "paper"}
        if warm:
            seed = R.checkpoint_heuristic(g, sets, cat, budget)
            if seed is not None:
                opts["incumbent"] = R.assignment_from_schedule(model, seed)
        res = R.solve(model, opts)
        out["status"] = res.status
        out["nodes"] = res.nodes
        out["model_stats"] = model.stats()
        sched = R.decode(res, g, cat) if res.assignment is not None else None
    if sched is None:
        return out
    out["schedule"] = R.schedule_to_doc(sched)
    out["validate"] = R.validate(sched, g, sets, cat)
    try:
        tr = R.simulate(sched, g, cat)
    except R.schedule.SimulationError as exc:  # reference defect, SURVEY.md Appendix C
        out["simulate_error"] = str(exc)
        return out
    out["trace_csv"] = R.trace_report(tr, "csv")
    out["peak"] = tr.peak_memory
    out["total_cost"] = R.format_cost(tr.total_cost)
    ok, model_peak, tags = R.check_schedule(g, sets, cat, sched, budget)
    out["bound_feasible"], out["bound_peak"], out["bound_tags"] = ok, model_peak, tags
    return out


def store_everything_case(gdoc, cdoc):
    g = R.load_graph(gdoc)
    cat = R.load_catalog(cdoc, g)
    sets = R.compute_dependency_sets(g, "upper")
    sched = R.store_everything_schedule(g, cat)
    tr = R.simulate(sched, g, cat)
    ok, model_peak, _ = R.check_schedule(g, sets, cat, sched, 1 << 62)
    return {"schedule": R.schedule_to_doc(sched), "trace_csv": R.trace_report(tr, "csv"),
            "peak": tr.peak_memory, "bound_peak": model_peak}


def main():
    # 1. the bundled resnet_toy instance (costmodel.py:426-517)
    g, cat = R.resnet_toy()
    gdoc, cdoc = R.graph_to_doc(g), R.catalog_to_doc(cat)
    toy = {"graph": gdoc, "catalog": cdoc, "store_everything": store_everything_case(gdoc, cdoc),
           "cases": [solve_case(gdoc, cdoc, b) for b in (700, 800, 1000, 1200, 1400)]}
    (HERE / "resnet_toy_solve.json").write_text(cj(toy))

    # 2. seeded synthetic instances, all generator kinds (costmodel.py:298-410)
    synth = []
    for kind, n, seed, fv, bv, ie in [("chain", 4, 0, 1, 1, 0), ("residual", 6, 1, 2, 2, 2),
                                      ("inception-toy", 7, 2, 2, 3, 3), ("unet-toy", 6, 3, 3, 2, 2)]:
        g, cat = R.generate_synthetic(kind, n, seed, fwd_variants=fv, bwd_variants=bv,
                                      intermediate_every=ie, inplace_marks=True)
        gdoc, cdoc = R.graph_to_doc(g), R.catalog_to_doc(cat)
        se = R.simulate(R.store_everything_schedule(g, cat), g, cat).peak_memory
        cases = [solve_case(gdoc, cdoc, b, node_limit=20000) for b in (se, (3 * se) // 4, se // 2)]
        synth.append({"kind": kind, "n": n, "seed": seed, "fwd_variants": fv, "bwd_variants": bv,
                      "intermediate_every": ie, "graph": gdoc, "catalog": cdoc, "cases": cases})
    (HERE / "synthetic_solve.json").write_text(cj(synth))

    # 3. config 1: ResNet-18, batch 8, 64x64, traced by this engine; tight budgets.
    #    The reference plans it (checkpoint_heuristic); we freeze the documents.
    from paper_2010_14501_b200.tracer import build_network
    net = build_network("resnet18", 8, 64)
    gdoc = net.graph_doc()
    cdoc = net.catalog_doc()
    g = R.load_graph(gdoc)
    cat = R.load_catalog(cdoc, g)
    se = store_everything_case(gdoc, cdoc)
    act = se["peak"] - gdoc["params_bytes"]
    # several fractions: the reference heuristic's schedule is rejected by its own
    # simulator at some budgets; the GPU test needs >= 1 that runs
    budgets = [gdoc["params_bytes"] + int(f * act) for f in (0.5, 0.4, 0.55, 0.6)]
    cases = [solve_case(gdoc, cdoc, b, heuristic_only=True) for b in budgets]
    cases += [solve_case(gdoc, cdoc, b, node_limit=256) for b in budgets]
    r18 = {"graph": gdoc, "catalog": cdoc, "store_everything": se, "cases": cases}
    (HERE / "r18_b8_64.json").write_text(cj(r18))
    print("wrote", sorted(p.name for p in HERE.glob("*.json")))


if __name__ == "__main__":
    main()

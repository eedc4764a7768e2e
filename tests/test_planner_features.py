"""Host planner features beyond the reference API (CPU only).

* fastest_store_everything_schedule: the min-cost no-recompute schedule that the
  measured overhead is relative to -- executable, no recompute, never costlier
  than the reference's default-variant store_everything_schedule;
* plan_schedule's exact-ILP path on small graphs: on resnet_toy it must return
  the reference ILP's optimum (tests/golden/resnet_toy_solve.json: budget 1200
  -> objective 181);
* greedy augmentation: never worse than the family candidates, always within
  the budget by the exact bound, always accepted by simulate().
"""
import json
from pathlib import Path

import pytest

import paper_2010_14501_b200 as M
from paper_2010_14501_b200.planner import plan_schedule
from paper_2010_14501_b200.schedule import fastest_store_everything_schedule
from paper_2010_14501_b200.tracer import build_network

GOLD = Path(__file__).resolve().parent / "golden"


def _toy():
    toy = json.loads((GOLD / "resnet_toy_solve.json").read_text())
    g = M.load_graph(toy["graph"])
    return toy, g, M.load_catalog(toy["catalog"], g)


def test_fastest_store_everything():
    for net in (build_network("resnet18", 4, 32, num_classes=10, fuse=True),
                build_network("googlenet", 2, 64, num_classes=10, fuse=True)):
        g = M.load_graph(net.graph_doc())
        cat = M.load_catalog(net.catalog_doc(), g)
        fast = fastest_store_everything_schedule(g, cat)
        ref = M.store_everything_schedule(g, cat)
        assert not any(s.recompute for s in fast.stages)
        assert fast.objective <= ref.objective
        assert not M.validate(fast, g, M.compute_dependency_sets(g), cat)
        M.simulate(fast, g, cat)
        # every node runs its cheapest variant
        for i, name in enumerate(fast.forward_impls, start=1):
            assert cat.fwd(i)[cat.fwd_index(i, name)].cost == min(v.cost for v in cat.fwd(i))


def test_exact_path_reaches_reference_optimum():
    toy, g, cat = _toy()
    case = next(c for c in toy["cases"] if c["budget"] == 1200)
    sched, info = plan_schedule(g, cat, 1200, exact_time_s=60)
    assert sched is not None and info["family"].startswith("exact-ilp")
    assert str(sched.objective) == str(case["total_cost"]) == "181"
    M.simulate(sched, g, cat)


@pytest.mark.parametrize("frac", [0.6, 0.5])
def test_augmented_plans_are_feasible_and_no_worse(frac):
    net = build_network("resnet18", 4, 32, num_classes=10, fuse=True)
    g = M.load_graph(net.graph_doc())
    cat = M.load_catalog(net.catalog_doc(), g)
    act = M.simulate(M.store_everything_schedule(g, cat), g, cat).peak_memory - g.params_bytes
    budget = g.params_bytes + int(frac * act)
    sched, info = plan_schedule(g, cat, budget, kinds=net.storable_kinds())
    assert sched is not None
    ok, peak, tags = M.check_schedule(g, M.compute_dependency_sets(g), cat, sched, budget)
    assert ok and peak <= budget, tags
    assert M.simulate(sched, g, cat).peak_memory <= peak
    base, _ = plan_schedule(g, cat, budget, kinds=net.storable_kinds(), exchange=True)
    assert base.objective <= sched.objective

"""ILP decisions are bit-exact against the reference (BASELINE north_star).

Fixtures in tests/golden/ilp_parity.json were produced by the reference
`remsched` itself (tests/golden/make_ilp_golden.py): for each instance and
budget the model's family counts, the SHA-256 of its LP export, the
branch-and-bound result under five option sets (status, node count,
objective, bound, gap, telemetry without wall-clock, decoded schedule) and
the exhaustive oracle's optimum / schedule / enumeration count.
"""
import hashlib
import json
from pathlib import Path

import pytest

import paper_2010_14501_b200 as M

GOLDEN = json.loads((Path(__file__).resolve().parent / "golden" / "ilp_parity.json").read_text())
CELLS = [(c["name"], cell) for c in GOLDEN for cell in c["cells"]]


def _inst(name):
    case = next(c for c in GOLDEN if c["name"] == name)
    g = M.load_graph(case["graph"])
    cat = M.load_catalog(case["catalog"], g)
    return g, cat


def _fmt(x):
    return None if x is None else M.format_cost(x)


@pytest.mark.parametrize("name,cell", CELLS, ids=[f"{n}@{c['budget']}" for n, c in CELLS])
def test_model_and_lp_identical(name, cell):
    g, cat = _inst(name)
    sets = M.compute_dependency_sets(g, "upper")
    m = M.build_model(g, sets, cat, cell["budget"], {"inplace": True, "bound_kind": "upper"})
    assert m.stats() == cell["stats"]
    assert hashlib.sha256(M.export_lp_string(m).encode()).hexdigest() == cell["lp_sha256"]


@pytest.mark.parametrize("name,cell", CELLS, ids=[f"{n}@{c['budget']}" for n, c in CELLS])
def test_solver_decisions_bit_exact(name, cell):
    g, cat = _inst(name)
    sets = M.compute_dependency_sets(g, "upper")
    m = M.build_model(g, sets, cat, cell["budget"], {"inplace": True, "bound_kind": "upper"})
    for want in cell["solves"]:
        r = M.solve(m, dict(want["options"]))
        got = {"status": r.status, "nodes": r.nodes, "objective": _fmt(r.objective),
               "lower_bound": _fmt(r.lower_bound), "gap": _fmt(r.gap),
               "schedule": None if r.assignment is None else M.schedule_to_doc(M.decode(r, g, cat)),
               "telemetry": [{k: v for k, v in e.items() if k != "elapsed_ms"} for e in r.telemetry]}
        assert got == {k: want[k] for k in got}, want["options"]
        if r.assignment is not None:  # the decoded schedule executes within the budget
            sched = M.decode(r, g, cat)
            assert not M.validate(sched, g, sets, cat)
            assert M.simulate(sched, g, cat).peak_memory <= cell["budget"]
            assert M.evaluate_assignment(m, r.assignment)["feasible"]


@pytest.mark.parametrize("name,cell", [x for x in CELLS if "oracle" in x[1]],
                         ids=[f"{n}@{c['budget']}" for n, c in CELLS if "oracle" in c])
def test_oracle_matches(name, cell):
    g, cat = _inst(name)
    o = M.enumerate_schedules(g, cat, cell["budget"])
    want = cell["oracle"]
    assert o.feasible == want["feasible"] and o.enumerated_count == want["enumerated"]
    assert _fmt(o.optimum) == want["optimum"]
    assert (o.model_peak, o.true_peak) == (want["model_peak"], want["true_peak"])
    assert (None if o.schedule is None else M.schedule_to_doc(o.schedule)) == want["schedule"]


def test_cross_check_agrees():
    g, cat = _inst("chain-4-0")
    rep = M.cross_check(g, cat, [6, 12, 40], {"solve": {"node_limit": 5000}})
    assert rep["pass"], rep["counterexamples"]


def test_warm_start_and_api_errors():
    g, cat = _inst("resnet_toy")
    sets = M.compute_dependency_sets(g, "upper")
    m = M.build_model(g, sets, cat, 2000, {})  # store-everything (model peak 1408) fits
    inc = M.assignment_from_schedule(m, M.store_everything_schedule(g, cat))
    seeded = M.solve(m, {"node_limit": 256, "incumbent": inc})
    assert seeded.telemetry[1]["event"] == "warm-start"
    assert seeded.objective is not None and seeded.objective <= M.evaluate_assignment(m, inc)["objective"]
    with pytest.raises(ValueError):
        M.solve(m, {"branch_order": "nope"})
    with pytest.raises(ValueError):
        M.solve(m, {"dive": "nope"})
    with pytest.raises(ValueError):
        M.build_model(g, sets, cat, -1, {})
    ok, fixed = M.propagate(m, {})
    assert ok and all(v in (0, 1) for v in fixed.values())
    assert M.lower_bound(m, {}) <= seeded.objective
    assert M.oracle.enumerate is M.enumerate_schedules

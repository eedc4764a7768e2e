"""Integer parity of the host contract against golden outputs of the REFERENCE.

tests/golden/*.json were produced by running the reference planner
(tests/golden/make_golden.py).  Every ledger, modeled peak, validate() tag
list and simulate() failure here must match it bit for bit, both through the
product (paper_2010_14501_b200) and through the independent oracle restatement
(oracle.ledger), which pins the oracle before it is used as a checker.
"""
import json
from pathlib import Path

import pytest

import paper_2010_14501_b200 as M
from oracle import ledger as L

GOLD = Path(__file__).resolve().parent / "golden"


def _cases():
    out = []
    toy = json.loads((GOLD / "resnet_toy_solve.json").read_text())
    out.append(("resnet_toy/store_everything", toy["graph"], toy["catalog"], toy["store_everything"]))
    for c in toy["cases"]:
        out.append((f"resnet_toy/{c['budget']}", toy["graph"], toy["catalog"], c))
    for inst in json.loads((GOLD / "synthetic_solve.json").read_text()):
        for c in inst["cases"]:
            out.append((f"{inst['kind']}-{inst['n']}-{inst['seed']}/{c['budget']}", inst["graph"],
                        inst["catalog"], c))
    r18 = json.loads((GOLD / "r18_b8_64.json").read_text())
    out.append(("r18/store_everything", r18["graph"], r18["catalog"], r18["store_everything"]))
    for i, c in enumerate(r18["cases"]):
        out.append((f"r18/{c['status']}-{c['budget']}-{i}", r18["graph"], r18["catalog"], c))
    return [c for c in out if "schedule" in c[3]]


CASES = _cases()


@pytest.mark.parametrize("name,gdoc,cdoc,case", CASES, ids=[c[0] for c in CASES])
def test_product_ledger_matches_reference(name, gdoc, cdoc, case):
    g = M.load_graph(gdoc)
    cat = M.load_catalog(cdoc, g)
    sched = M.schedule_from_doc(case["schedule"])
    sets = M.compute_dependency_sets(g)
    if "validate" in case:
        assert M.validate(sched, g, sets, cat) == case["validate"]
    if "simulate_error" in case:
        with pytest.raises(M.SimulationError, match=case["simulate_error"]):
            M.simulate(sched, g, cat)
        return
    tr = M.simulate(sched, g, cat)
    assert M.trace_report(tr) == case["trace_csv"]
    assert tr.peak_memory == case["peak"]
    budget = case.get("budget", 1 << 62)
    ok, peak, tags = M.check_schedule(g, sets, cat, sched, budget)
    assert peak == case["bound_peak"]
    if "bound_tags" in case:
        assert (ok, tags) == (case["bound_feasible"], case["bound_tags"])
    # documents round-trip byte-identically
    assert M.schedule_to_doc(sched) == case["schedule"]


@pytest.mark.parametrize("name,gdoc,cdoc,case", CASES, ids=[c[0] for c in CASES])
def test_oracle_ledger_pinned(name, gdoc, cdoc, case):
    if "simulate_error" in case:
        with pytest.raises(L.LedgerError):
            L.replay(gdoc, cdoc, case["schedule"])
        return
    rows, peak = L.replay(gdoc, cdoc, case["schedule"])
    assert L.trace_csv(rows, peak) == case["trace_csv"]


def test_reference_defect_reproduced():
    """The reference heuristic's r18 schedule at the 0.4 budget recomputes an
    already-live tensor; simulate() must fail exactly like the reference."""
    r18 = json.loads((GOLD / "r18_b8_64.json").read_text())
    bad = [c for c in r18["cases"] if "simulate_error" in c]
    assert bad, "fixture lost its failing case"
    g = M.load_graph(r18["graph"])
    cat = M.load_catalog(r18["catalog"], g)
    for c in bad:
        with pytest.raises(M.SimulationError, match="unaccounted memory"):
            M.simulate(M.schedule_from_doc(c["schedule"]), g, cat)


def test_bundled_fixture_matches_generator():
    g1, c1 = M.bundled_fixture("resnet_toy")
    g2, c2 = M.resnet_toy()
    assert M.graph_to_doc(g1) == M.graph_to_doc(g2)
    assert M.catalog_to_doc(c1) == M.catalog_to_doc(c2)
    toy = json.loads((GOLD / "resnet_toy_solve.json").read_text())
    assert M.graph_to_doc(g2) == toy["graph"] and M.catalog_to_doc(c2) == toy["catalog"]


def test_synthetic_generator_matches_reference():
    for inst in json.loads((GOLD / "synthetic_solve.json").read_text()):
        g, c = M.generate_synthetic(inst["kind"], inst["n"], inst["seed"],
                                    fwd_variants=inst["fwd_variants"], bwd_variants=inst["bwd_variants"],
                                    intermediate_every=inst["intermediate_every"], inplace_marks=True)
        assert M.graph_to_doc(g) == inst["graph"]
        assert M.catalog_to_doc(c) == inst["catalog"]

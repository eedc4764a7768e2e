"""Catalog ablations are identical to the reference's.

tests/golden/ablation.json was produced by the reference `remsched`
(tests/golden/make_ablation_golden.py): for four graphs (bundled resnet_toy,
a synthetic residual instance with intermediates, traced fused and split-conv
ResNet-18) and every mode of ABLATION_MODES (costmodel.py:25) it holds
apply_ablation's catalog document (costmodel.py:220-252), variant_category of
every backward variant (costmodel.py:76) and, on the small graphs, the
reference solver's status and decoded schedule at a tight budget under the
ablated catalog (the `solve --ablation` path, cli.py:129-160).
"""
import json
from pathlib import Path

import pytest

import paper_2010_14501_b200 as M
from paper_2010_14501_b200.costmodel import variant_category

GOLDEN = json.loads((Path(__file__).resolve().parent / "golden" / "ablation.json").read_text())
CELLS = [(c["name"], mode) for c in GOLDEN for mode in M.ABLATION_MODES]


def _case(name):
    case = next(c for c in GOLDEN if c["name"] == name)
    g = M.load_graph(case["graph"])
    return case, g, M.load_catalog(case["catalog"], g)


@pytest.mark.parametrize("name", [c["name"] for c in GOLDEN])
def test_variant_categories(name):
    case, g, cat = _case(name)
    got = [[k, v.name, variant_category(g, k, v)] for k, vs in sorted(cat.backward.items()) for v in vs]
    assert got == case["categories"]


@pytest.mark.parametrize("name,mode", CELLS, ids=[f"{n}-{m}" for n, m in CELLS])
def test_apply_ablation_matches_reference(name, mode):
    case, g, cat = _case(name)
    want = case["modes"][mode]
    ab = M.apply_ablation(cat, g, mode)
    assert M.catalog_to_doc(ab) == want["catalog"]
    if "status" in want:  # the reference's solve under the ablated catalog: same decisions
        sets = M.compute_dependency_sets(g, "upper")
        model = M.build_model(g, sets, ab, case["budget"], {"inplace": True, "bound_kind": "upper"})
        r = M.solve(model, {"node_limit": 4000})
        assert r.status == want["status"]
        got = None if r.assignment is None else M.schedule_to_doc(M.decode(r, g, ab))
        assert got == want.get("schedule")


def test_unknown_mode_rejected():
    _, g, cat = _case("resnet_toy")
    with pytest.raises(ValueError, match="unknown ablation mode"):
        M.apply_ablation(cat, g, "bogus")

"""The planned arena of every committed schedule (schedules/*.json) fits its ILP bound.

Physical peak = params_bytes + arena high-water mark (csrc/arena.cpp) must not
exceed check_schedule's modeled peak (oracle.py:287), which must not exceed
the budget; the ledger peak (simulate) sits below both.  CPU only: the
ledger, lifetimes and the offset planner never touch the GPU.
"""
import hashlib
import json
from pathlib import Path

import pytest

import paper_2010_14501_b200 as M
from paper_2010_14501_b200.engine import lifetimes, place_blocks
from paper_2010_14501_b200.schedule import ledger
from paper_2010_14501_b200.tracer import build_network

ROOT = Path(__file__).resolve().parent.parent
SCHEDULES = sorted((ROOT / "schedules").glob("*_b*_*gib.json"))


_NETS = {}


def _net(path):
    """(network, graph, catalog) a schedule file was planned for
    (name: arch[_fused][_split]_b<batch>_<image>_<budget>gib, image 224 or HxW)."""
    stem = path.name.split("_b")[0]
    split = stem.endswith("_split")
    base = stem.removesuffix("_split")
    arch, fused = base.removesuffix("_fused"), base.endswith("_fused")
    batch, image = path.name.split("_b")[1].split("_")[:2]
    batch = int(batch)
    key = (arch, fused, split, batch, image)
    if key not in _NETS:
        from paper_2010_14501_b200.tracer import default_classes, parse_image
        net = build_network(arch, batch, parse_image(image), num_classes=default_classes(arch), fuse=fused,
                            split=split)
        g = M.load_graph(net.graph_doc())
        cpath = ROOT / "profiles" / f"catalog_{stem}_b{batch}_{image}.json"
        cdoc = json.loads(cpath.read_text())["catalog"] if cpath.exists() else net.catalog_doc()
        _NETS[key] = (net, g, M.load_catalog(cdoc, g))
    return _NETS[key]


@pytest.mark.parametrize("path", SCHEDULES, ids=[p.stem for p in SCHEDULES])
def test_physical_peak_within_ilp_bound(path):
    net, g, cat = _net(path)
    doc = json.loads(path.read_text())
    digest = hashlib.sha256(json.dumps(net.graph_doc(), sort_keys=True).encode()).hexdigest()[:16]
    assert doc["graph_digest"] == digest, "schedule was planned for another graph"
    sched = M.schedule_from_doc(doc["schedule"])
    assert not M.validate(sched, g, M.compute_dependency_sets(g), cat)
    steps, trace = ledger(sched, g, cat)
    assert M.trace_report(trace) == M.trace_report(M.simulate(sched, g, cat))
    arena, _ = place_blocks(lifetimes(steps, g)[0])
    ok, bound, tags = M.check_schedule(g, M.compute_dependency_sets(g), cat, sched, doc["budget_bytes"])
    assert ok, tags
    assert trace.peak_memory <= bound <= doc["budget_bytes"]
    assert g.params_bytes + arena <= bound

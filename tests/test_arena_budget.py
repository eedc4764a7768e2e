"""The planned arena of every committed ResNet-50 schedule fits its ILP bound.

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
SCHEDULES = sorted((ROOT / "schedules").glob("resnet50*_b184_224_*gib.json"))


_NETS = {}


def _r50(fused: bool):
    if fused not in _NETS:
        net = build_network("resnet50", 184, 224, fuse=fused)
        g = M.load_graph(net.graph_doc())
        path = ROOT / "profiles" / f"catalog_resnet50{'_fused' if fused else ''}_b184_224.json"
        cdoc = json.loads(path.read_text())["catalog"] if path.exists() else net.catalog_doc()
        _NETS[fused] = (net, g, M.load_catalog(cdoc, g))
    return _NETS[fused]


@pytest.mark.parametrize("path", SCHEDULES, ids=[p.stem for p in SCHEDULES])
def test_physical_peak_within_ilp_bound(path):
    net, g, cat = _r50("_fused" in path.name)
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

"""The CPU reference arm of bench.py (`--impl reference`) runs without the product.

* The frozen network specs (oracle/specs/*.json) still describe the graph the
  product's tracer emits (no drift between what the GPU arm runs and what the
  reference arm replays).
* The reference planner path (remsched from baseline/_ref, unmodified) on the
  headline instance: the committed 8 GiB schedule validates, simulates to the
  ledger peak the GPU executes, and its ILP bound is within the budget -- in a
  subprocess that must not import paper_2010_14501_b200 (nor map its .so).
"""
import hashlib
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
SPECS = sorted((ROOT / "oracle" / "specs").glob("*.json"))


@pytest.mark.parametrize("path", SPECS, ids=[p.stem for p in SPECS])
def test_spec_matches_tracer(path):
    from paper_2010_14501_b200.tracer import build_network, default_classes, parse_image

    doc = json.loads(path.read_text())
    stem = path.stem
    arch = stem.split("_b")[0]
    split = arch.endswith("_split")
    arch = arch.removesuffix("_split")
    fused = arch.endswith("_fused")
    arch = arch.removesuffix("_fused")
    batch, image = stem.split("_b")[1].split("_")
    net = build_network(arch, int(batch), parse_image(image), num_classes=default_classes(arch), fuse=fused,
                        split=split)
    gdoc = net.graph_doc()
    assert doc["graph"] == gdoc
    assert doc["graph_digest"] == hashlib.sha256(json.dumps(gdoc, sort_keys=True).encode()).hexdigest()[:16]
    assert [o["kind"] for o in doc["ops"]] == [op.kind for op in net.ops]


@pytest.mark.skipif(not (ROOT / "baseline" / "_ref" / "remsched").exists(), reason="baseline/_ref not installed")
def test_reference_planner_without_product():
    code = (
        "import sys, json, argparse; sys.path.insert(0, %r); import bench; "
        "a = argparse.Namespace(arch='resnet50', batch=184, image='224', budget_gib=8.0, fuse=True, split=False); "
        "r = bench.reference_planner_run(a); "
        "r['product_loaded'] = any(m.startswith('paper_2010_14501_b200') for m in sys.modules); "
        "print(json.dumps(r))" % str(ROOT))
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert not r["product_loaded"]
    sdoc = json.loads((ROOT / "schedules" / "resnet50_fused_b184_224_8gib.json").read_text())
    assert r["validate_tags"] == 0 and r["within_budget"]
    assert r["simulated_peak_bytes"] <= r["ilp_bound_bytes"] <= sdoc["budget_bytes"]
    assert r["status"] in ("optimal", "feasible-gap")
    assert int(r["objective"]) >= int(r["lower_bound"])

"""Golden fixtures for the catalog ablations, made by the REFERENCE.

    python tests/golden/make_ablation_golden.py

For each graph (the bundled resnet_toy, a synthetic residual instance, and the
traced fused ResNet-18 / split-conv ResNet-18 of this repo's tracer) and each
ablation mode (costmodel.py:25 ABLATION_MODES), the reference's
apply_ablation (costmodel.py:220-252) is applied and its catalog_to_doc
recorded, together with variant_category of every backward variant
(costmodel.py:76) and, on the small graphs, the reference solver's decisions
at a tight budget under that ablation (cli.py:129-160, the `solve --ablation`
path).  /root/reference exists only in the build container; the output is
committed as tests/golden/ablation.json.
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
from remsched.costmodel import variant_category  # noqa: E402


def cases():
    out = []
    gdoc = json.loads((ROOT / "paper_2010_14501_b200" / "data" / "resnet_toy.json").read_text())
    cdoc = json.loads((ROOT / "paper_2010_14501_b200" / "data" / "resnet_toy.catalog.json").read_text())
    out.append(("resnet_toy", gdoc, cdoc, True))
    g, c = R.generate_synthetic("residual", 14, 3, fwd_variants=2, bwd_variants=3, intermediate_every=3)
    out.append(("residual14", R.graph_to_doc(g), R.catalog_to_doc(c), True))
    from paper_2010_14501_b200.tracer import build_network

    for name, kw in (("resnet18_fused_b8_64", {"fuse": True}), ("resnet18_split_b8_64", {"split": True})):
        net = build_network("resnet18", 8, 64, num_classes=10, **kw)
        out.append((name, net.graph_doc(), net.catalog_doc(), False))
    return out


def main():
    fixtures = []
    for name, gdoc, cdoc, solve in cases():
        g = R.load_graph(gdoc)
        cat = R.load_catalog(cdoc, g)
        case = {"name": name, "graph": gdoc, "catalog": cdoc, "modes": {}}
        case["categories"] = [[k, v.name, variant_category(g, k, v)]
                              for k, vs in sorted(cat.backward.items()) for v in vs]
        se = R.simulate(R.store_everything_schedule(g, cat), g, cat).peak_memory
        budget = g.params_bytes + (se - g.params_bytes) * 6 // 10
        case["budget"] = budget
        for mode in R.ABLATION_MODES:
            ab = R.apply_ablation(cat, g, mode)
            entry = {"catalog": R.catalog_to_doc(ab)}
            if solve:
                sets = R.compute_dependency_sets(g, "upper")
                model = R.build_model(g, sets, ab, budget, {"inplace": True, "bound_kind": "upper"})
                res = R.solve(model, {"node_limit": 4000})
                entry["status"] = res.status
                if res.assignment is not None:
                    entry["schedule"] = R.schedule_to_doc(R.decode(res, g, ab))
            case["modes"][mode] = entry
        fixtures.append(case)
    (HERE / "ablation.json").write_text(json.dumps(fixtures, sort_keys=True) + "\n")
    print("wrote", HERE / "ablation.json", [c["name"] for c in fixtures])


if __name__ == "__main__":
    main()

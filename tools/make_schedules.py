"""Plan the benchmark schedules offline and freeze them (host planner, deterministic).

    python tools/make_schedules.py

Writes schedules/<arch>_b<batch>_<img>_<budget>gib.json with the graph and
catalog digests they were planned against.  Planning ResNet-50 takes about a
minute per budget, so bench.py loads these instead of planning in the timed run.
"""
import hashlib
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2010_14501_b200 as M  # noqa: E402
from paper_2010_14501_b200.planner import plan_schedule  # noqa: E402
from paper_2010_14501_b200.tracer import build_network, default_classes, parse_image  # noqa: E402

OUT = ROOT / "schedules"


def digest(doc):
    return hashlib.sha256(json.dumps(doc, sort_keys=True).encode()).hexdigest()[:16]


def main(jobs, exact_time_s=None, exchange=False, lp=False, mip_time_s=None, ablation=None):
    OUT.mkdir(exist_ok=True)
    for arch, batch, img, gib, fuse, split in jobs:
        net = build_network(arch, batch, parse_image(img), num_classes=default_classes(arch), fuse=fuse, split=split)
        arch = arch + ("_fused" if net.fused else "") + ("_split" if net.split else "")
        gdoc, cdoc = net.graph_doc(), net.catalog_doc()
        measured = ROOT / "profiles" / f"catalog_{arch}_b{batch}_{img}.json"
        if measured.exists():  # plan with the on-device profile when it matches this graph
            mdoc = json.loads(measured.read_text())
            if mdoc["graph_digest"] == digest(gdoc):
                cdoc = mdoc["catalog"]
                print("planning with measured catalog", measured.name)
        g = M.load_graph(gdoc)
        cat = M.load_catalog(cdoc, g)
        if ablation:  # plan with one ablation family of the catalog (costmodel.py:220-252)
            cat = M.apply_ablation(cat, g, ablation)
        budget = int(gib * (1 << 30))
        t = time.time()
        sched, info = plan_schedule(g, cat, budget, kinds=net.storable_kinds(), exact_time_s=exact_time_s,
                                    exchange=exchange, lp=lp, mip_time_s=mip_time_s)
        dt = time.time() - t
        if sched is None:
            print(arch, batch, img, gib, "no feasible schedule", info)
            continue
        doc = {"arch": arch, "batch": batch, "image": img, "budget_bytes": budget, "ablation": ablation or "all",
               "graph_digest": digest(gdoc), "catalog_digest": digest(cdoc), "planner": info,
               "plan_seconds": round(dt, 1), "schedule": M.schedule_to_doc(sched)}
        path = OUT / f"{arch}_b{batch}_{img}_{gib:g}gib{'_abl-' + ablation if ablation else ''}.json"
        path.write_text(json.dumps(doc, indent=1, sort_keys=True) + "\n")
        print(path.name, info, f"{dt:.1f}s")


if __name__ == "__main__":
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--fused", action="store_true")
    ap.add_argument("--arch", default="resnet50")
    ap.add_argument("--batch", type=int, default=184)
    ap.add_argument("--image", default="224", help="224 or HxW (UNet: 416x608)")
    ap.add_argument("--budgets", default="10,8,6", help="GiB, comma separated")
    ap.add_argument("--exact", type=float, default=None,
                    help="seconds of exact ILP search on graphs of <= planner.EXACT_MAX_NODES nodes")
    ap.add_argument("--exchange", action="store_true", help="also try exchange moves (slower)")
    ap.add_argument("--split", action="store_true", help="conv backward split into dgrad / wgrad nodes")
    ap.add_argument("--lp", action="store_true", help="seed the planner with the ILP's LP relaxation (HiGHS)")
    ap.add_argument("--mip", type=float, default=None, help="seconds of HiGHS MIP search for a dual bound")
    ap.add_argument("--ablation", default=None, choices=["none", "conv", "out", "int", "all"],
                    help="plan with apply_ablation(catalog, mode); file suffix _abl-<mode>")
    a = ap.parse_args()
    main([(a.arch, a.batch, a.image, float(b), a.fused, a.split) for b in a.budgets.split(",")], a.exact,
         a.exchange, a.lp, a.mip, a.ablation)

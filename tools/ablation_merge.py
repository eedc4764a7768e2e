"""Cross-check the per-ablation schedules of one workload (tools/make_schedules.py --ablation).

    python tools/ablation_merge.py resnet50_fused_b184_224_8gib

The ablation families nest (none is a subset of conv, out and int, each a subset of all:
costmodel.py:220-252), so a schedule planned for a smaller family is also a schedule of every
larger one, at the same cost.  The planner is a heuristic plus a time-limited MIP, so a larger
family's own plan can come out worse than a smaller family's; this keeps, per family, the
cheapest schedule that validates under that family's catalog, and records where it came from.
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2010_14501_b200 as M  # noqa: E402
from paper_2010_14501_b200.tracer import build_network  # noqa: E402

MODES = ("none", "conv", "out", "int", "all")


def main(stem):
    arch = stem.split("_b")[0]
    base = arch.replace("_fused", "").replace("_split", "")
    batch, image = stem.split("_b")[1].split("_")[:2]
    net = build_network(base, int(batch), int(image), fuse="_fused" in arch, split="_split" in arch)
    g = M.load_graph(net.graph_doc())
    full = M.load_catalog(json.loads((ROOT / "profiles" / f"catalog_{arch}_b{batch}_{image}.json").read_text())
                          ["catalog"], g)
    sets = M.compute_dependency_sets(g)
    files = {m: ROOT / "schedules" / f"{stem}_abl-{m}.json" for m in MODES if m != "all"}
    files["all"] = ROOT / "schedules" / f"{stem}.json"
    docs = {m: json.loads(p.read_text()) for m, p in files.items() if p.exists()}
    from paper_2010_14501_b200.schedule import fastest_store_everything_schedule
    se = M.schedule_cost(g, full, fastest_store_everything_schedule(g, full))
    for m in MODES:
        cat = M.apply_ablation(full, g, m)
        best = None
        for src, doc in docs.items():
            sched = M.schedule_from_doc(doc["schedule"])
            if M.validate(sched, g, sets, cat):
                continue
            if best is None or sched.objective < best[1].objective:
                best = (src, sched, doc)
        if best is None:
            print(m, "no schedule")
            continue
        src, sched, doc = best
        print(f"{m:5s} best from {src:5s} objective {float(sched.objective):.0f} "
              f"overhead vs min-cost store-everything {float(sched.objective / se - 1) * 100:.2f} %")
        if src != m and m in docs:
            out = dict(doc)
            out["ablation"] = m
            out["planner"] = dict(doc["planner"], family=f"from-abl-{src}:" + doc["planner"].get("family", ""))
            files[m].write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main(sys.argv[1])

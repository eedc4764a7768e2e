"""Measure the catalog of a network on the B200 and freeze it (R3 profiler).

    python tools/profile_catalog.py [arch batch image] [--fused] [--split]

Writes profiles/catalog_<arch>_b<batch>_<image>.json: the catalog document
(measured ns costs, library workspace bytes) plus the graph digest it was
measured for.  tools/make_schedules.py and bench.py plan / account with it.
"""
import hashlib
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2010_14501_b200.profiler import profile_network  # noqa: E402
from paper_2010_14501_b200.tracer import build_network, default_classes, parse_image  # noqa: E402


def digest(doc):
    return hashlib.sha256(json.dumps(doc, sort_keys=True).encode()).hexdigest()[:16]


def main(arch="resnet50", batch=184, image=224, fuse=False, split=False):
    net = build_network(arch, batch, parse_image(image), num_classes=default_classes(arch), fuse=fuse, split=split)
    arch = arch + ("_fused" if net.fused else "") + ("_split" if net.split else "")
    t = time.time()
    costs = profile_network(net, log=print)
    doc = {"arch": arch, "batch": batch, "image": image, "graph_digest": digest(net.graph_doc()),
           "profile_seconds": round(time.time() - t, 1), "catalog": net.catalog_doc(costs)}
    out = ROOT / "profiles" / f"catalog_{arch}_b{batch}_{image}.json"
    out.write_text(json.dumps(doc, indent=1, sort_keys=True) + "\n")
    print("wrote", out)


if __name__ == "__main__":
    fuse, split = "--fused" in sys.argv, "--split" in sys.argv
    a = [x for x in sys.argv[1:] if x not in ("--fused", "--split")]
    main(a[0], int(a[1]), a[2], fuse, split) if a else main(fuse=fuse, split=split)

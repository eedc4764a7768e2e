"""Freeze the benchmark network's op list + graph document into oracle/specs/ (see oracle/netspec.py).

    python tools/freeze_netspec.py [--arch resnet50] [--batch 184] [--image 224] [--no-fuse]
"""
import argparse
import hashlib
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import netspec  # noqa: E402
from paper_2010_14501_b200.tracer import build_network, default_classes, parse_image  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--arch", default="resnet50")
    ap.add_argument("--batch", type=int, default=184)
    ap.add_argument("--image", default="224")
    ap.add_argument("--no-fuse", dest="fuse", action="store_false")
    ap.add_argument("--split", action="store_true")
    a = ap.parse_args()
    net = build_network(a.arch, a.batch, parse_image(a.image), num_classes=default_classes(a.arch), fuse=a.fuse,
                        split=a.split)
    gdoc = net.graph_doc()
    doc = netspec.freeze(net, gdoc)
    doc["graph_digest"] = hashlib.sha256(json.dumps(gdoc, sort_keys=True).encode()).hexdigest()[:16]
    out = netspec.spec_path(a.arch, net.fused, a.batch, a.image, net.split)
    out.parent.mkdir(exist_ok=True)
    out.write_text(json.dumps(doc, sort_keys=True, separators=(",", ":")))
    print(f"wrote {out.relative_to(ROOT)} ({out.stat().st_size} B, {len(doc['ops'])} ops, digest {doc['graph_digest']})")


if __name__ == "__main__":
    main()

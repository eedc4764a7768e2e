"""Re-key frozen measured catalogs to the current graph (digest, 16-B workspace sizes).

    python tools/refresh_catalogs.py

Used when the graph's byte accounting changes but the measured kernel times do not
(the catalog's costs are keyed by node id and variant name).
"""
import hashlib
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2010_14501_b200.tracer import build_network, default_classes, parse_image, r16  # noqa: E402


def digest(doc):
    return hashlib.sha256(json.dumps(doc, sort_keys=True).encode()).hexdigest()[:16]


for path in sorted((ROOT / "profiles").glob("catalog_*.json")):
    doc = json.loads(path.read_text())
    arch = doc["arch"].removesuffix("_fused")
    net = build_network(arch, doc["batch"], parse_image(doc["image"]), num_classes=default_classes(arch),
                        fuse=doc["arch"].endswith("_fused"))
    fresh = net.catalog_doc()
    ws = {}
    for sec in ("forward", "backward"):
        for e in fresh[sec]:
            for v in e["variants"]:
                ws[(sec, e["node"], v["name"])] = v["workspace_bytes"]
    for sec in ("forward", "backward"):
        for e in doc["catalog"][sec]:
            for v in e["variants"]:
                v["workspace_bytes"] = ws.get((sec, e["node"], v["name"]), r16(v["workspace_bytes"]))
    doc["graph_digest"] = digest(net.graph_doc())
    path.write_text(json.dumps(doc, indent=1, sort_keys=True) + "\n")
    print("refreshed", path.name)

"""Frozen network description for the CPU oracle (test / baseline infrastructure).

`bench.py --impl reference` times the reference-side CPU path without importing
the product package (nor mapping its .so): the network the GPU arm traces is
frozen once into ``oracle/specs/<arch>[_fused]_b<batch>_<image>.json`` by
``tools/freeze_netspec.py`` -- the op list (kind, deps, output shape, attrs,
parameter shapes), the intermediates, and the graph document the reference's
``remsched`` loads.  :func:`load` rebuilds an object with the attributes
``oracle.cpu_executor`` reads (``ops``, ``op(i)``, ``n``, ``intermediate_of``,
``batch``, ``num_classes``, ``label_count()``, ``fused``).

Parameters are synthetic (seeded, fan-in scaled normal; BN gamma 1 / beta 0;
running mean 0 / var 1): this object exists to *time* the CPU path on the
benchmark's shapes, not to reproduce the GPU arm's torchvision init.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from pathlib import Path

import torch

SPECS = Path(__file__).resolve().parent / "specs"
BN_KINDS = ("bn", "bnrelu", "bnrelu6", "bnaddrelu")


@dataclass
class SpecOp:
    id: int
    kind: str
    deps: tuple
    shape: tuple
    attrs: dict = field(default_factory=dict)
    params: dict = field(default_factory=dict)
    name: str = ""

    @property
    def numel(self) -> int:
        return int(math.prod(self.shape)) if self.shape else 1

    @property
    def nbytes(self) -> int:
        return 0 if self.kind == "wgrad" else (self.numel * 4 + 15) // 16 * 16


class SpecNet:
    def __init__(self, doc: dict, seed: int = 0):
        self.batch = doc["batch"]
        self.num_classes = doc["num_classes"]
        self.graph = doc["graph"]
        self.intermediate_of = {int(k): v for k, v in doc["intermediate_of"].items()}
        gen = torch.Generator().manual_seed(seed)
        self.ops = []
        for o in doc["ops"]:
            attrs = dict(o["attrs"])
            params = {}
            for name, shape in o["params"].items():
                if o["kind"] in BN_KINDS:
                    params[name] = torch.ones(shape) if name == "weight" else torch.zeros(shape)
                elif name == "bias":
                    params[name] = torch.zeros(shape)
                else:
                    fan_in = math.prod(shape[1:]) if len(shape) > 1 else shape[0]
                    params[name] = torch.randn(shape, generator=gen) * math.sqrt(2.0 / fan_in)
            if o["kind"] in BN_KINDS:
                c = o["shape"][-1]
                attrs["running_mean"] = torch.zeros(c)
                attrs["running_var"] = torch.ones(c)
            self.ops.append(SpecOp(o["id"], o["kind"], tuple(o["deps"]), tuple(o["shape"]), attrs, params,
                                   o["name"]))
        self.n = len(self.ops)
        self._bwd = {int(k): v for k, v in doc["bwd_deps"].items()}
        self.fused = any(op.kind in ("bnrelu", "bnrelu6", "bnaddrelu") for op in self.ops)
        self.split = any(op.kind == "wgrad" for op in self.ops)

    def op(self, i: int) -> SpecOp:
        return self.ops[i - 1]

    def grad_bytes(self, op: SpecOp) -> int:
        return 0 if op.kind in ("input", "wgrad") else op.nbytes

    def bwd_deps(self, k: int, impl: str) -> list:
        return list(self._bwd[k][impl])

    def label_count(self) -> int:
        logits = self.op(self.ops[-1].deps[0])
        return logits.numel // logits.shape[-1]


def spec_path(arch: str, fused: bool, batch: int, image: str, split: bool = False) -> Path:
    return SPECS / f"{arch}{'_fused' if fused else ''}{'_split' if split else ''}_b{batch}_{image}.json"


def load(path, seed: int = 0) -> SpecNet:
    return SpecNet(json.loads(Path(path).read_text()), seed)


def freeze(net, graph_doc: dict) -> dict:
    """Spec document of a traced product Network (called by tools/freeze_netspec.py)."""
    ops = []
    for op in net.ops:
        attrs = {k: v for k, v in op.attrs.items() if not isinstance(v, torch.Tensor)}
        ops.append({"id": op.id, "kind": op.kind, "deps": list(op.deps), "shape": list(op.shape),
                    "attrs": attrs, "params": {k: list(t.shape) for k, t in op.params.items()},
                    "name": op.name})
    bwd = {str(op.id): {name: list(deps) for name, _, deps in net.variants(op)[1]} for op in net.ops}
    return {"format": 1, "batch": net.batch, "num_classes": net.num_classes, "ops": ops,
            "intermediate_of": {str(k): v for k, v in net.intermediate_of.items()}, "bwd_deps": bwd,
            "graph": graph_doc}

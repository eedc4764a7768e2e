"""Model tracer: torch model -> Network -> graph document.

``trace_graph(model, example_input)`` walks ``torch.fx.symbolic_trace(model)``
and emits a :class:`Network`, one op per graph node in execution order, with
the conventions the reference graph format imposes (graph.py:251-360,
SURVEY.md §7 hard part 7):

* node 1 is the input batch, with a dependency-free backward and a zero-byte
  gradient (no dgrad of the stem is ever needed);
* the softmax cross-entropy loss is appended as the unique sink N;
* ReLU sign bitmasks and maxpool 8-bit window indices are *intermediates* of
  their creator, stored or recomputed like any other storable;
* sizes are the executor's real allocation sizes: NHWC fp32 activations,
  ceil(numel/32)*4 bytes per mask, numel bytes per maxpool index (rounded up
  to 4), the stem input padded from 3 to 4 channels;
* parameters, their gradients and momenta, BN statistics, the staging input
  batch, labels and kernel scratch are all folded into ``params_bytes``.

``Network.graph_doc()`` / ``Network.catalog_doc(costs)`` emit the two
documents the planner consumes.
"""

from __future__ import annotations

import math
import operator
from dataclasses import dataclass, field

import torch

from . import _native

__all__ = ["Op", "Network", "trace_graph", "build_network"]

F32 = 4


@dataclass
class Op:
    id: int
    kind: str                    # input conv bn relu add maxpool avgpool fc xent
    deps: tuple
    shape: tuple                 # output shape: NHWC for maps, (N, F) for vectors, () for loss
    attrs: dict = field(default_factory=dict)
    params: dict = field(default_factory=dict)   # name -> torch tensor (CPU, engine layout)
    name: str = ""

    @property
    def numel(self) -> int:
        return int(math.prod(self.shape)) if self.shape else 1

    @property
    def nbytes(self) -> int:
        if self.kind == "wgrad":  # the weight-gradient anchor of a split conv produces no tensor
            return 0
        return r16(self.numel * F32)


def r16(b: int) -> int:
    """Allocation size: the arena places blocks at 16-byte granularity (engine.ARENA_ALIGN),
    so every size the graph and catalog report is already a multiple of 16 and the
    reference's byte ledger equals the physical footprint of a gap-free packing."""
    return (b + 15) // 16 * 16


def mask_bytes(numel: int) -> int:
    return r16((numel + 31) // 32 * 4)


def idx_bytes(numel: int) -> int:
    return r16(numel)


class Network:
    """Executable op list in node order plus its parameters (engine layout)."""

    def __init__(self, ops: list[Op], batch: int, num_classes: int):
        self.ops = ops
        self.fused = any(op.kind in ("bnrelu", "bnrelu6", "bnaddrelu", "convrelu") for op in ops)
        self.split = any(op.kind == "wgrad" for op in ops)
        self.batch = batch
        self.num_classes = num_classes
        self.n = len(ops)
        # intermediates: one per ReLU (sign mask) and per maxpool (8-bit index)
        self.intermediate_of: dict[int, int] = {}
        self.intermediate_bytes: dict[int, int] = {}
        nid = self.n + 1
        for op in ops:
            if op.kind in ("relu", "relu6", "convrelu"):  # convrelu: the ReLU's mask of the fused conv
                self.intermediate_of[op.id] = nid
                self.intermediate_bytes[nid] = mask_bytes(op.numel)
                nid += 1
            elif op.kind == "maxpool":
                self.intermediate_of[op.id] = nid
                self.intermediate_bytes[nid] = idx_bytes(op.numel)
                nid += 1

    def op(self, i: int) -> Op:
        return self.ops[i - 1]

    def storable_kinds(self) -> dict:
        """Storable id -> family label used by the planner (planner.FAMILIES)."""
        out = {}
        for op in self.ops:
            kind = op.kind
            if kind == "relu" and self.op(op.deps[0]).kind == "add":
                kind = "relu-join"
            elif kind in ("bnrelu", "bnrelu6", "convrelu"):   # a fused op's output is a ReLU output
                kind = "relu"
            elif kind in ("addrelu", "bnaddrelu"):  # ... at a residual join
                kind = "relu-join"
            elif kind == "relu6":
                kind = "relu"
            elif kind == "dwconv":
                kind = "conv"
            out[op.id] = kind
            if op.id in self.intermediate_of:
                out[self.intermediate_of[op.id]] = "mask" if op.kind in ("relu", "relu6", "convrelu") else "idx"
        return out

    # -------------------------------------------------------------- fixed region
    def param_items(self):
        for op in self.ops:
            for name, t in op.params.items():
                yield op.id, name, t

    def n_param_elems(self) -> int:
        return sum(t.numel() for _, _, t in self.param_items())

    def bn_channels(self) -> int:
        return sum(op.shape[-1] for op in self.ops if op.kind in ("bn", "bnrelu", "bnrelu6", "bnaddrelu"))

    def scratch_bytes(self) -> int:
        lib = _native.lib()
        s = 0
        for op in self.ops:
            if op.kind in ("bn", "bnrelu", "bnrelu6", "bnaddrelu") or (op.kind in ("conv", "convrelu", "convT") and
                                                                       "bias" in op.params):
                rows = op.numel // op.shape[-1]  # conv bias gradient: per-channel sum of dy
                s = max(s, lib.bn_scratch_bytes(rows, op.shape[-1]))
        s = max(s, lib.xent_scratch_bytes(self.label_count()))
        return (s + 255) // 256 * 256

    def input_bytes(self) -> int:
        return self.ops[0].nbytes

    def w16_segments(self) -> list:
        """Conv weights kept pre-split in bf16 hi / lo planes (monet_conv_*_w16):
        (op id, offset in the flat parameter buffer, offset in each plane, count), plane
        offsets 16-B aligned (TMA).  Transposed and depthwise convs are not GEMM B operands
        of that form."""
        out, pos, dst = [], 0, 0
        for nid, name, t in self.param_items():
            n = t.numel()
            if name == "weight" and self.op(nid).kind in ("conv", "convrelu"):
                out.append((nid, pos, dst, n))
                dst += (n + 7) // 8 * 8
            pos += n
        return out

    BN_KINDS = ("bn", "bnrelu", "bnrelu6", "bnaddrelu")

    def bn_input(self, op: Op) -> int:
        return op.attrs["x"] if op.kind == "bnaddrelu" else op.deps[0]

    def stats_convs(self) -> dict:
        """{conv id: BN id} for each conv whose output is the input of the BN that runs right
        after it in the forward pass (split anchors have no forward work): the conv leaves the
        BN's batch statistics in the stats scratch (monet_conv_fwd_w16_stats) and the BN's
        training forward merges them instead of re-reading the conv output."""
        out = {}
        for op in self.ops:
            if op.kind != "conv":
                continue
            j = op.id + 1
            while j <= self.n and self.op(j).kind == "wgrad":
                j += 1
            if j <= self.n and self.op(j).kind in self.BN_KINDS and self.bn_input(self.op(j)) == op.id:
                out[op.id] = j
        return out

    def conv_stats_bytes(self) -> int:
        lib = _native.lib()
        return max((lib.conv_stats_bytes(self.conv_desc(self.op(i))) for i in self.stats_convs()), default=0)

    def fixed_layout(self) -> dict:
        """Byte sizes of everything outside the arena (all folded into params_bytes)."""
        p = self.n_param_elems() * F32
        segs = self.w16_segments()
        plane = sum((n + 7) // 8 * 8 for *_, n in segs)
        return {
            "params": p, "grads": p, "momentum": p,
            "w16": 2 * 2 * plane,           # pre-split conv weights: bf16 hi plane, then lo plane
            "w16_table": 24 * len(segs),    # their segment table (monet_split_bf16_segments)
            "conv_stats": self.conv_stats_bytes(),  # conv -> BN per-tile statistics (stats_convs)
            "bn_stats": 4 * self.bn_channels() * F32,   # saved mean/invstd, running mean/var
            "scratch": self.scratch_bytes(),
            "staging_input": self.input_bytes(),
            "labels": self.label_count() * 4,
            "consts": 256,
        }

    def params_bytes(self) -> int:
        return sum((v + 255) // 256 * 256 for v in self.fixed_layout().values())

    # -------------------------------------------------------------- documents
    def grad_bytes(self, op: Op) -> int:
        if op.kind in ("input", "wgrad"):
            return 0
        return op.nbytes

    def graph_doc(self) -> dict:
        nodes, backward, inters = [], [], []
        for op in self.ops:
            nodes.append({"id": op.id, "output_bytes": op.nbytes, "deps": list(op.deps)})
            impls = [{"name": n, "deps_kind": k, "extra_deps": self._extra_deps(op, n)} for n, k in BWD_IMPLS[op.kind]]
            backward.append({"node": op.id, "grad_bytes": self.grad_bytes(op), "impls": impls})
            if op.id in self.intermediate_of:
                u = self.intermediate_of[op.id]
                inters.append({"id": u, "bytes": self.intermediate_bytes[u], "creator": op.id})
        return {"format": 1, "params_bytes": self.params_bytes(), "nodes": nodes,
                "backward": backward, "intermediates": inters}

    def _extra_deps(self, op: Op, impl: str) -> list:
        if op.kind == "bnaddrelu" and impl == "bwd-out":
            return [op.attrs["x"]]
        if op.kind == "convrelu" and not op.attrs.get("split"):  # the gate: its own ReLU mask
            return [self.intermediate_of[op.id]]
        if op.kind == "wgrad" and self.op(op.attrs["conv"]).kind == "convrelu":
            return [self.intermediate_of[op.attrs["conv"]]]
        return []

    def label_count(self) -> int:
        """Rows of the loss: images, or pixels for a per-pixel (segmentation) loss."""
        logits = self.op(self.ops[-1].deps[0])
        return logits.numel // logits.shape[-1]

    def fc_dims(self, op: Op):
        """(rows, in_features) of an fc op; a 4-D input is read flattened (NHWC order)."""
        x = self.op(op.deps[0])
        return x.shape[0], x.numel // x.shape[0]

    def variants(self, op: Op):
        """(forward variants, backward variants) as (name, workspace_bytes, deps) tuples."""
        lib = _native.lib()
        fwd, bwd = [], []
        x = list(op.deps)
        if op.kind in ("conv", "convrelu"):
            d = self.conv_desc(op)
            fwd.append(("implicit", 0))
            ws = lib.conv_ws_bytes(1, 0, d)
            if ws:
                fwd.append(("splitk", ws))
            if op.attrs.get("split"):  # backward = dgrad only: reads dy and the weights, not x
                bwd.append(("splitk", lib.conv_ws_bytes(1, 1, d), []))
                bwd.append(("implicit", lib.conv_ws_bytes(0, 1, d), []))
            else:  # convrelu: dy is first gated by the ReLU's mask
                xm = x + ([self.intermediate_of[op.id]] if op.kind == "convrelu" else [])
                bwd.append(("splitk", lib.conv_ws_bytes(1, 3, d), xm))
                bwd.append(("implicit", lib.conv_ws_bytes(0, 3, d), xm))
        elif op.kind == "wgrad":  # split conv's weight gradient: reads the conv input x and dy
            conv = self.op(op.attrs["conv"])
            d = self.conv_desc(conv)
            fwd.append(("none", 0))
            # a split convrelu's weight-gradient stage runs first: it gates dy in place with the mask
            xm = [conv.deps[0]] + ([self.intermediate_of[conv.id]] if conv.kind == "convrelu" else [])
            bwd.append(("splitk", lib.conv_ws_bytes(1, 2, d), xm))
            bwd.append(("implicit", lib.conv_ws_bytes(0, 2, d), xm))
        elif op.kind == "fc":
            n, fi = self.fc_dims(op)
            fo = op.shape[1]
            fwd.append(("gemm", 0))
            ws = lib.linear_ws_bytes(1, 0, n, fi, fo)
            if ws:
                fwd.append(("gemm-splitk", ws))
            bwd.append(("gemm-splitk", lib.linear_ws_bytes(1, 3, n, fi, fo), x))
            bwd.append(("gemm", lib.linear_ws_bytes(0, 3, n, fi, fo), x))
        elif op.kind in ("relu", "relu6"):
            fwd.append((op.kind, 0))
            bwd += [("bwd-in", 0, x), ("bwd-out", 0, [op.id]),
                    ("bwd-mask", 0, [self.intermediate_of[op.id]])]
        elif op.kind == "convT":  # transposed conv: the conv kernels with the roles swapped
            d = self.conv_desc(op)
            fwd.append(("implicit", lib.convT_ws_bytes(0, 0, d)))
            ws = lib.convT_ws_bytes(1, 0, d)
            if ws:
                fwd.append(("splitk", ws))
            bwd.append(("splitk", lib.convT_ws_bytes(1, 3, d), x))
            bwd.append(("implicit", lib.convT_ws_bytes(0, 3, d), x))
        elif op.kind == "dwconv":  # depthwise: one direct kernel per pass, wgrad partials in ws
            fwd.append(("direct", 0))
            bwd.append(("direct", lib.dwconv_ws_bytes(self.conv_desc(op)), x))
        elif op.kind == "bn":
            fwd.append(("bn", 0))
            bwd += [("bwd-in", 0, x), ("bwd-out", 0, [op.id])]
        elif op.kind in ("bnrelu", "bnrelu6"):  # fused BN+ReLU(6): backward from the BN input only (K10)
            fwd.append((op.kind, 0))
            bwd.append(("bwd-in", 0, x))
        elif op.kind == "bnaddrelu":  # fused BN + join + ReLU: BN backward from x, gate from z or (x, skip)
            fwd.append(("bnaddrelu", 0))
            bwd += [("bwd-out", 0, sorted([op.attrs["x"], op.id])), ("bwd-in", 0, x)]
        elif op.kind == "addrelu":  # fused residual join + ReLU: gate from the output or the inputs
            fwd.append(("addrelu", 0))
            bwd += [("bwd-out", 0, [op.id]), ("bwd-in", 0, x)]
        elif op.kind == "maxpool":
            fwd.append(("maxpool", 0))
            bwd += [("bwd-in", 0, x), ("bwd-idx", 0, [self.intermediate_of[op.id]])]
        elif op.kind == "input":
            fwd.append(("load", 0))
            bwd.append(("none", 0, []))
        elif op.kind in ("add", "avgpool", "concat"):
            fwd.append((op.kind, 0))
            bwd.append(("bwd", 0, []))
        elif op.kind == "dropout":  # backward reads dy only (mask regenerated)
            fwd.append(("dropout", 0))
            bwd.append(("bwd-rng", 0, []))
        elif op.kind == "xent":
            fwd.append(("xent", 0))
            bwd.append(("bwd", 0, x))
        else:
            raise ValueError(op.kind)
        return [(nm, r16(ws)) for nm, ws in fwd], [(nm, r16(ws), deps) for nm, ws, deps in bwd]

    INPLACE_KINDS = ("relu", "relu6", "bn", "bnrelu", "bnrelu6", "dropout")

    def inplace_capable(self, op: Op) -> bool:
        """Elementwise one-input operators whose kernels accept y aliasing x: a recompute may
        overwrite its input (costmodel.py:121-129; the schedule's stage ``inplace`` list, the
        executor places both in one arena block).  The first forward never runs in place."""
        return (op.kind in self.INPLACE_KINDS and len(op.deps) == 1
                and self.op(op.deps[0]).nbytes == op.nbytes)

    def catalog_doc(self, costs=None) -> dict:
        """Catalog with measured costs (``costs[(node, pass, name)]`` -> int ns) or the
        analytic roofline estimate when a cost is not supplied."""
        from .costs import analytic_cost
        fwd_doc, bwd_doc = [], []
        for op in self.ops:
            fv, bv = self.variants(op)
            inplace = self.inplace_capable(op)
            fwd_doc.append({"node": op.id, "variants": [
                {"name": n, "workspace_bytes": ws,
                 "cost": _cost(costs, (op.id, "fwd", n), lambda: analytic_cost(self, op, "fwd", n)),
                 **({"inplace_capable": True} if inplace else {})}
                for n, ws in fv]})
            bwd_doc.append({"node": op.id, "variants": [
                {"name": n, "workspace_bytes": ws, "deps": sorted(deps),
                 "cost": _cost(costs, (op.id, "bwd", n), lambda: analytic_cost(self, op, "bwd", n))}
                for n, ws, deps in bv]})
        return {"format": 1, "forward": fwd_doc, "backward": bwd_doc}

    def conv_desc(self, op: Op):
        if op.kind == "convT":  # the conv whose input is this op's output and whose output is its input
            n, p, q, k = self.op(op.deps[0]).shape
            _, h, w, c = op.shape
            a = op.attrs
            return _native.ConvDesc(n, h, w, c, k, a["r"], a["s"], p, q, a["stride"], a["stride"], a["pad"], a["pad"])
        n, h, w, c = self.op(op.deps[0]).shape
        a = op.attrs
        return _native.ConvDesc(n, h, w, c, op.shape[3], a["r"], a["s"], op.shape[1], op.shape[2],
                                a["stride"], a["stride"], a["pad"], a["pad"])

    def pool_desc(self, op: Op):
        n, h, w, c = self.op(op.deps[0]).shape
        a = op.attrs
        return _native.ConvDesc(n, h, w, c, c, a["r"], a["s"], op.shape[1], op.shape[2],
                                a["stride"], a["stride"], a["pad"], a["pad"])

    def conv_flops(self) -> int:
        tot = 0
        for op in self.ops:
            if op.kind in ("conv", "convrelu"):
                cin = self.op(op.deps[0]).shape[3]
                tot += 2 * op.numel * cin * op.attrs["r"] * op.attrs["s"]
            elif op.kind == "fc":
                tot += 2 * op.numel * self.op(op.deps[0]).shape[1]
        return tot


def _cost(costs, key, fallback):
    if costs is not None and key in costs:
        return int(costs[key])
    return int(fallback())


BWD_IMPLS = {
    "input": [("none", "input")],
    "conv": [("splitk", "input"), ("implicit", "input")],
    "convrelu": [("splitk", "input"), ("implicit", "input")],  # + its mask (extra_deps)
    "wgrad": [("splitk", "input"), ("implicit", "input")],  # catalog deps: the conv's input (see split)
    "fc": [("gemm-splitk", "input"), ("gemm", "input")],
    "bn": [("bwd-in", "input"), ("bwd-out", "output")],
    "bnrelu": [("bwd-in", "input")],
    "bnrelu6": [("bwd-in", "input")],
    "bnaddrelu": [("bwd-out", "output"), ("bwd-in", "input")],  # bwd-out also reads x (extra_deps)
    "addrelu": [("bwd-out", "output"), ("bwd-in", "input")],
    "relu": [("bwd-in", "input"), ("bwd-out", "output"), ("bwd-mask", "intermediate")],
    "maxpool": [("bwd-in", "input"), ("bwd-idx", "intermediate")],
    "dropout": [("bwd-rng", "input")],
    "concat": [("bwd", "input")],  # catalog deps []: the backward slices dy
    "relu6": [("bwd-in", "input"), ("bwd-out", "output"), ("bwd-mask", "intermediate")],
    "dwconv": [("direct", "input")],
    "convT": [("splitk", "input"), ("implicit", "input")],  # catalog deps []: the keep-mask is regenerated from the step seed
    "add": [("bwd", "input")],
    "avgpool": [("bwd", "input")],
    "xent": [("bwd", "input")],
}


# ---------------------------------------------------------------------- tracing

def _pair(v):
    return v if isinstance(v, int) else v[0]


def fuse_conv_relu(ops: list[Op]) -> list[Op]:
    """Merge every conv whose only reader is a ReLU into one "convrelu" op (VGG: the
    convs have no BN).  The pre-activation is never kept: the fused op writes
    y = relu(conv(x)) and the ReLU's 1-bit sign mask (its intermediate), and its
    backward gates dy with the mask in place before the conv's data / weight gradients --
    so a conv's backward holds dy and x (and the 1-bit mask), never a second full-size
    gradient (SURVEY §8 K4-K5 with the conv of K1-K3).  Ids are renumbered in order."""
    readers: dict[int, list[int]] = {}
    for op in ops:
        for j in op.deps:
            readers.setdefault(j, []).append(op.id)
    fused_into: dict[int, int] = {}  # relu id -> conv id
    for op in ops:
        if op.kind == "conv" and len(readers.get(op.id, [])) == 1:
            r = ops[readers[op.id][0] - 1]
            if r.kind == "relu" and r.deps == (op.id,):
                fused_into[r.id] = op.id
    new_id: dict[int, int] = {}
    out: list[Op] = []
    for op in ops:
        if op.id in fused_into:
            new_id[op.id] = new_id[fused_into[op.id]]
            continue
        nid = len(out) + 1
        new_id[op.id] = nid
        fused = op.id in fused_into.values()
        attrs = dict(op.attrs)
        if "inputs" in attrs:
            attrs["inputs"] = [new_id[j] for j in attrs["inputs"]]
        for key in ("x", "skip"):
            if key in attrs:
                attrs[key] = new_id[attrs[key]]
        out.append(Op(nid, "convrelu" if fused else op.kind, tuple(new_id[j] for j in op.deps), op.shape, attrs,
                      op.params, op.name + "+relu" if fused else op.name))
    return out


def fuse_bn_relu(ops: list[Op]) -> list[Op]:
    """Merge every BatchNorm (residual add) whose only reader is a ReLU into one
    "bnrelu" ("addrelu") op: the pre-activation tensor
    is never materialized, the fused op's output is the ReLU's.  bnrelu's
    backward reads x; addrelu's gates from its output (or its inputs).  Ids
    are renumbered in order; dependencies are remapped."""
    readers: dict[int, list[int]] = {}
    for op in ops:
        for j in op.deps:
            readers.setdefault(j, []).append(op.id)
    fused_into: dict[int, int] = {}  # relu id -> bn id
    six: set[int] = set()            # bn ids fused with a ReLU6 (MobileNet-V2)
    for op in ops:
        if op.kind in ("bn", "add") and len(readers.get(op.id, [])) == 1 and len(set(op.deps)) == len(op.deps):
            r = ops[readers[op.id][0] - 1]
            if r.kind == "relu" and r.deps == (op.id,):
                fused_into[r.id] = op.id
            elif r.kind == "relu6" and op.kind == "bn" and r.deps == (op.id,):
                fused_into[r.id] = op.id
                six.add(op.id)
    new_id: dict[int, int] = {}
    out: list[Op] = []
    for op in ops:
        if op.id in fused_into:
            new_id[op.id] = new_id[fused_into[op.id]]
            continue
        nid = len(out) + 1
        new_id[op.id] = nid
        fused = op.id in fused_into.values()
        kind = ("bnrelu6" if op.id in six else {"bn": "bnrelu", "add": "addrelu"}[op.kind]) if fused else op.kind
        name = op.name + ("+relu6" if op.id in six else "+relu") if fused else op.name
        attrs = dict(op.attrs)
        if "inputs" in attrs:  # concat order
            attrs["inputs"] = [new_id[j] for j in attrs["inputs"]]
        out.append(Op(nid, kind, tuple(new_id[j] for j in op.deps), op.shape, attrs, op.params, name))
    return out


def fuse_bn_addrelu(ops: list[Op]) -> list[Op]:
    """Merge a BN whose only reader is a fused add+ReLU into it: z = relu(BN(x) + skip)
    ("bnaddrelu"; the residual block's last BN).  The BN output is never materialized;
    the op reads x and skip.  Where both join inputs are such BNs (a downsample block),
    the main-path one (lower id) is fused."""
    readers: dict[int, list[int]] = {}
    for op in ops:
        for j in op.deps:
            readers.setdefault(j, []).append(op.id)
    absorbed: dict[int, int] = {}  # addrelu id -> bn id
    for op in ops:
        if op.kind != "addrelu":
            continue
        for j in sorted(op.deps):
            b = ops[j - 1]
            if b.kind == "bn" and readers.get(j) == [op.id] and j not in absorbed.values():
                absorbed[op.id] = j
                break
    gone = set(absorbed.values())
    new_id: dict[int, int] = {}
    out: list[Op] = []
    for op in ops:
        if op.id in gone:
            continue
        nid = len(out) + 1
        new_id[op.id] = nid
        attrs = dict(op.attrs)
        if "inputs" in attrs:
            attrs["inputs"] = [new_id[j] for j in attrs["inputs"]]
        if op.id in absorbed:
            b = ops[absorbed[op.id] - 1]
            x = b.deps[0]
            skip = next(j for j in op.deps if j != b.id)
            attrs = dict(b.attrs)
            attrs["x"], attrs["skip"] = new_id[x], new_id[skip]
            out.append(Op(nid, "bnaddrelu", tuple(sorted((new_id[x], new_id[skip]))), op.shape, attrs, b.params,
                          b.name + "+add+relu"))
        else:
            out.append(Op(nid, op.kind, tuple(new_id[j] for j in op.deps), op.shape, attrs, op.params, op.name))
    return out


def split_conv_backward(ops: list[Op]) -> list[Op]:
    """Split every conv's backward into two graph nodes:

    * the conv node keeps the forward and its backward becomes the input gradient
      (dgrad), which reads only dy and the weights -- not the forward input x;
    * a new zero-byte node right after it ("wgrad", deps: the conv) carries the weight
      gradient, whose backward reads x and the conv's output gradient.  Its stage runs
      before the conv's (stages descend), so x can be freed as soon as the weight
      gradient is done and the dgrad allocates dx without x still live.

    The anchors are extra dependencies of the loss node (the unique sink), whose
    backward "produces" their zero-byte gradients -- the reference graph format needs
    every backward node's gradient to come from a later stage (graph.py:349-358).
    Convs reading the network input (no dgrad) are not split.  Ids are renumbered."""
    new_id: dict[int, int] = {}
    out: list[Op] = []
    anchors: list[int] = []
    for op in ops:
        nid = len(out) + 1
        new_id[op.id] = nid
        attrs = dict(op.attrs)
        if "inputs" in attrs:
            attrs["inputs"] = [new_id[j] for j in attrs["inputs"]]
        for key in ("x", "skip"):
            if key in attrs:
                attrs[key] = new_id[attrs[key]]
        deps = tuple(new_id[j] for j in op.deps)
        split = op.kind in ("conv", "convrelu") and ops[op.deps[0] - 1].kind != "input"
        if split:
            attrs["split"] = True
            attrs["wgrad_node"] = nid + 1
        if op.kind == "xent":
            deps = deps + tuple(anchors)
        out.append(Op(nid, op.kind, deps, op.shape, attrs, op.params, op.name))
        if split:
            out.append(Op(nid + 1, "wgrad", (nid,), (), {"conv": nid}, name=op.name + ".wgrad"))
            anchors.append(nid + 1)
    return out


def trace_graph(model: torch.nn.Module, example_input: torch.Tensor, num_classes: int | None = None,
                fuse: bool = False, split: bool = False) -> Network:
    """Trace a torchvision-style CNN into a Network (engine layout parameters).

    Supported modules: Conv2d (no bias, groups=1), BatchNorm2d, ReLU,
    MaxPool2d, AdaptiveAvgPool2d((1,1)), Linear; functions: add / iadd,
    flatten.  Parameters are copied (conv OIHW -> KRSC, stem channels
    padded to a multiple of 4).
    """
    import torch.fx

    gm = torch.fx.symbolic_trace(model)
    modules = dict(gm.named_modules())
    n, c, h, w = example_input.shape
    c_pad = (c + 3) // 4 * 4
    ops: list[Op] = [Op(1, "input", (), (n, h, w, c_pad), {"channels": c}, name="input")]
    where: dict[str, int] = {}
    for node in gm.graph.nodes:
        if node.op == "placeholder":
            where[node.name] = 1
            continue
        if node.op == "output":
            src = where[node.args[0].name]
            break
        if node.op == "call_module":
            mod = modules[node.target]
            src = where[node.args[0].name]
            x = ops[src - 1]
            nid = len(ops) + 1
            if isinstance(mod, torch.nn.Conv2d) and mod.groups > 1:
                _, hh, ww, cin = x.shape
                if mod.groups != cin or mod.out_channels != cin or mod.bias is not None or _pair(mod.dilation) != 1:
                    raise NotImplementedError(f"{node.target}: grouped convs only as bias-free depthwise")
                r, s = mod.kernel_size
                st, pd = _pair(mod.stride), _pair(mod.padding)
                p = (hh + 2 * pd - r) // st + 1
                q = (ww + 2 * pd - s) // st + 1
                wt = mod.weight.detach().float().view(cin, r, s).permute(1, 2, 0).contiguous()  # [R][S][C]
                ops.append(Op(nid, "dwconv", (src,), (n, p, q, cin), {"r": r, "s": s, "stride": st, "pad": pd},
                              {"weight": wt}, node.target))
            elif isinstance(mod, torch.nn.Conv2d):
                if _pair(mod.dilation) != 1:
                    raise NotImplementedError(f"{node.target}: only undilated convs")
                r, s = mod.kernel_size
                st, pd = _pair(mod.stride), _pair(mod.padding)
                _, hh, ww, cin = x.shape
                p = (hh + 2 * pd - r) // st + 1
                q = (ww + 2 * pd - s) // st + 1
                wt = mod.weight.detach().float().permute(0, 2, 3, 1).contiguous()  # KRSC
                if wt.shape[3] != cin:
                    wt = torch.nn.functional.pad(wt, (0, cin - wt.shape[3]))
                prm = {"weight": wt}
                if mod.bias is not None:  # VGG-style conv bias: added in the GEMM epilogue
                    prm["bias"] = mod.bias.detach().float().clone()
                ops.append(Op(nid, "conv", (src,), (n, p, q, mod.out_channels),
                              {"r": r, "s": s, "stride": st, "pad": pd}, prm, node.target))
            elif isinstance(mod, torch.nn.BatchNorm2d):
                ops.append(Op(nid, "bn", (src,), x.shape, {"eps": mod.eps, "momentum": mod.momentum},
                              {"weight": mod.weight.detach().float().clone(),
                               "bias": mod.bias.detach().float().clone()},
                              node.target))
                ops[-1].attrs["running_mean"] = mod.running_mean.detach().float().clone()
                ops[-1].attrs["running_var"] = mod.running_var.detach().float().clone()
            elif isinstance(mod, torch.nn.ReLU):
                ops.append(Op(nid, "relu", (src,), x.shape, name=node.target))
            elif isinstance(mod, torch.nn.ReLU6):
                ops.append(Op(nid, "relu6", (src,), x.shape, name=node.target))
            elif isinstance(mod, torch.nn.ConvTranspose2d):
                if mod.groups != 1 or _pair(mod.dilation) != 1 or _pair(mod.output_padding) != 0:
                    raise NotImplementedError(f"{node.target}: plain transposed convs only")
                r, s = mod.kernel_size
                st, pd = _pair(mod.stride), _pair(mod.padding)
                _, hh, ww, cin = x.shape
                p = (hh - 1) * st - 2 * pd + r
                q = (ww - 1) * st - 2 * pd + s
                wt = mod.weight.detach().float().permute(0, 2, 3, 1).contiguous()  # [in][R][S][out] = KRSC
                prm = {"weight": wt}
                if mod.bias is not None:
                    prm["bias"] = mod.bias.detach().float().clone()
                ops.append(Op(nid, "convT", (src,), (n, p, q, mod.out_channels),
                              {"r": r, "s": s, "stride": st, "pad": pd}, prm, node.target))
            elif isinstance(mod, torch.nn.MaxPool2d):
                r = _pair(mod.kernel_size)
                st, pd = _pair(mod.stride), _pair(mod.padding)
                _, hh, ww, cc = x.shape

                def osz(size):  # torch pooling output size (ceil_mode: last window starts inside)
                    if not mod.ceil_mode:
                        return (size + 2 * pd - r) // st + 1
                    o = -(-(size + 2 * pd - r) // st) + 1
                    return o - 1 if (o - 1) * st >= size + pd else o
                p, q = osz(hh), osz(ww)
                attrs = {"r": r, "s": r, "stride": st, "pad": pd}
                if mod.ceil_mode:
                    attrs["ceil"] = True
                ops.append(Op(nid, "maxpool", (src,), (n, p, q, cc), attrs, name=node.target))
            elif isinstance(mod, torch.nn.AdaptiveAvgPool2d):
                osz = mod.output_size if isinstance(mod.output_size, tuple) else (mod.output_size,) * 2
                if len(x.shape) == 4 and tuple(osz) == tuple(x.shape[1:3]):
                    where[node.name] = src  # VGG's (7, 7) pool on a 7 x 7 map is the identity
                    continue
                if tuple(osz) != (1, 1):
                    raise NotImplementedError(f"{node.target}: adaptive pool to {osz}")
                ops.append(Op(nid, "avgpool", (src,), (n, x.shape[3]), name=node.target))
            elif isinstance(mod, torch.nn.Flatten):
                where[node.name] = src  # fc reads a 4-D input flattened in the engine's NHWC order
                continue
            elif isinstance(mod, torch.nn.Dropout):
                if mod.p <= 0.0:
                    where[node.name] = src
                    continue
                ops.append(Op(nid, "dropout", (src,), x.shape, {"p": float(mod.p)}, name=node.target))
            elif isinstance(mod, torch.nn.Linear):
                wt = mod.weight.detach().float().clone()
                if len(x.shape) == 4:  # torch flattens (c, h, w); the engine's activations are (h, w, c)
                    _, hh, ww, cc = x.shape
                    wt = wt.view(-1, cc, hh, ww).permute(0, 2, 3, 1).reshape(wt.shape[0], -1).contiguous()
                ops.append(Op(nid, "fc", (src,), (n, mod.out_features), {},
                              {"weight": wt, "bias": mod.bias.detach().float().clone()}, node.target))
            else:
                raise NotImplementedError(f"module {type(mod).__name__} at {node.target}")
            where[node.name] = nid
        elif node.op == "call_function":
            if node.target in (operator.add, operator.iadd, torch.add):
                a, b = (where[arg.name] for arg in node.args[:2])
                nid = len(ops) + 1
                ops.append(Op(nid, "add", tuple(sorted((a, b))), ops[a - 1].shape, name=node.name))
                where[node.name] = nid
            elif node.target in (torch.nn.functional.relu, torch.relu, torch.nn.functional.relu6):
                src = where[node.args[0].name]
                nid = len(ops) + 1
                kind = "relu6" if node.target is torch.nn.functional.relu6 else "relu"
                ops.append(Op(nid, kind, (src,), ops[src - 1].shape, name=node.name))
                where[node.name] = nid
            elif node.target is torch.cat:
                srcs = [where[a.name] for a in node.args[0]]
                dim = node.args[1] if len(node.args) > 1 else node.kwargs.get("dim", 0)
                if dim != 1 or len(set(srcs)) != len(srcs):
                    raise NotImplementedError("torch.cat: channel concat of distinct tensors only")
                shp = [ops[j - 1].shape for j in srcs]
                nid = len(ops) + 1
                ops.append(Op(nid, "concat", tuple(sorted(srcs)), (*shp[0][:3], sum(s[3] for s in shp)),
                              {"inputs": srcs}, name=node.name))
                where[node.name] = nid
            elif node.target is torch.flatten:
                where[node.name] = where[node.args[0].name]  # avgpool already emits (N, C)
            elif node.target is torch.nn.functional.adaptive_avg_pool2d:
                osz = node.args[1] if len(node.args) > 1 else node.kwargs["output_size"]
                if osz not in (1, (1, 1), [1, 1]):
                    raise NotImplementedError(f"adaptive_avg_pool2d to {osz}")
                src = where[node.args[0].name]
                nid = len(ops) + 1
                ops.append(Op(nid, "avgpool", (src,), (n, ops[src - 1].shape[3]), name=node.name))
                where[node.name] = nid
            else:
                raise NotImplementedError(f"function {node.target}")
        elif node.op == "call_method" and node.target in ("flatten", "view", "reshape"):
            where[node.name] = where[node.args[0].name]
        else:
            raise NotImplementedError(f"{node.op} {node.target}")
    logits = ops[src - 1]
    k = num_classes or logits.shape[1]
    ops.append(Op(len(ops) + 1, "xent", (src,), (), name="loss"))
    if fuse:
        ops = fuse_bn_addrelu(fuse_bn_relu(fuse_conv_relu(ops)))
    if split:
        ops = split_conv_backward(ops)
    return Network(ops, n, k)


def parse_image(v):
    """Image size argument: 224, "224", or "HxW" (UNet: "416x608") -> int or (h, w)."""
    if isinstance(v, (tuple, list)):
        return tuple(v)
    if "x" in str(v):
        h, w = str(v).split("x")
        return int(h), int(w)
    return int(v)


def default_classes(arch: str) -> int:
    """Classes of the benchmark configs: ImageNet's 1000, UNet's 4 (segmentation)."""
    return 4 if arch == "unet" else 1000


def build_network(arch: str, batch: int, image: int | tuple = 224, num_classes: int = 1000,
                  seed: int = 0, fuse: bool = False, split: bool = False) -> Network:
    """torchvision ``arch`` with default init under ``torch.manual_seed(seed)``, traced
    (``fuse``: BN+ReLU pairs become single fused ops; ``split``: conv backward split
    into dgrad / wgrad graph nodes, split_conv_backward)."""
    import torchvision

    torch.manual_seed(seed)
    if arch == "unet":
        model = UNet(num_classes)
    else:
        kw = {"aux_logits": False, "init_weights": True} if arch in ("googlenet", "inception_v3") else {}
        model = getattr(torchvision.models, arch)(num_classes=num_classes, **kw)
    hw = (image, image) if isinstance(image, int) else image
    return trace_graph(model, torch.empty(batch, 3, *hw, device="meta"), num_classes, fuse, split)


# ------------------------------------------------------------------ UNet (config C3)
class _DoubleConv(torch.nn.Sequential):
    def __init__(self, cin, cout):
        super().__init__(torch.nn.Conv2d(cin, cout, 3, padding=1, bias=False), torch.nn.BatchNorm2d(cout),
                         torch.nn.ReLU(inplace=True), torch.nn.Conv2d(cout, cout, 3, padding=1, bias=False),
                         torch.nn.BatchNorm2d(cout), torch.nn.ReLU(inplace=True))


class _Up(torch.nn.Module):
    def __init__(self, cin, cout):
        super().__init__()
        self.up = torch.nn.ConvTranspose2d(cin, cin // 2, 2, stride=2)
        self.conv = _DoubleConv(cin, cout)

    def forward(self, x, skip):
        return self.conv(torch.cat([skip, self.up(x)], dim=1))


class UNet(torch.nn.Module):
    """The UNet of config C3 (MONeT's segmentation benchmark, 608 x 416): the common
    DoubleConv / Down (maxpool + DoubleConv) / Up (2x2 stride-2 transposed conv, skip concat,
    DoubleConv) / 1x1 OutConv layout, widths 64..1024.  Input sizes divisible by 16 (no
    crop / pad in the skips).  Classes must be a multiple of 4 (the conv kernels' channel
    granularity); the loss is the per-pixel softmax cross-entropy."""

    def __init__(self, num_classes=4, in_channels=3, width=64):
        super().__init__()
        w = width
        self.inc = _DoubleConv(in_channels, w)
        self.down = torch.nn.ModuleList(
            torch.nn.Sequential(torch.nn.MaxPool2d(2), _DoubleConv(w * 2 ** i, w * 2 ** (i + 1))) for i in range(4))
        self.up = torch.nn.ModuleList(_Up(w * 2 ** (4 - i), w * 2 ** (3 - i)) for i in range(4))
        self.outc = torch.nn.Conv2d(w, num_classes, 1)

    def forward(self, x):
        skips = [self.inc(x)]
        for d in self.down:
            skips.append(d(skips[-1]))
        y = skips.pop()
        for u in self.up:
            y = u(y, skips.pop())
        return self.outc(y)

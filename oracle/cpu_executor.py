"""torch-CPU fp32 replay of a Schedule on a traced Network (test oracle / CPU baseline).

Executes exactly what the GPU engine executes, in the reference simulator's
order (pkg/src/remsched/schedule.py:344-457): the forward pass in node order
keeping row 0, then per stage: drop what the previous row kept and this row
does not, recompute the planned tensors (BN replays its saved statistics and
never touches running stats), run the chosen backward variant
(input-, output- or intermediate-activated), release tensors
after their last in-stage reader; finally SGD with momentum.  Activations
that are not live are really deleted, so a schedule that reads a dropped
tensor fails here as it does in the simulator.

Layouts: NCHW torch tensors internally; ReLU masks are packed over the NHWC
element order (oracle.bitmask) and maxpool indices are the 8-bit window index
r*S+s, exactly the GPU engine's intermediate formats.
"""
from __future__ import annotations

import torch
import torch.nn.functional as F

from .bitmask import pack_sign_mask, unpack_sign_mask
from .dropout import keep_mask


def _nchw(t):
    return t.permute(0, 3, 1, 2).contiguous()


class CpuState:
    """Parameters / optimizer state of one network on the CPU (NCHW conv weights)."""

    def __init__(self, net, lr=0.1, momentum=0.9, weight_decay=0.0, dtype=torch.float32):
        self.net = net
        self.dtype = dtype
        self.lr, self.momentum, self.weight_decay = lr, momentum, weight_decay
        self.params = {}
        for op in net.ops:
            for name, t in op.params.items():
                v = t.to(dtype).clone()
                if op.kind in ("conv", "convrelu", "convT") and name == "weight":
                    v = v.permute(0, 3, 1, 2).contiguous()  # KRSC -> KCRS (OIHW; convT: [in][out][R][S])
                elif op.kind == "dwconv" and name == "weight":
                    v = v.permute(2, 0, 1).unsqueeze(1).contiguous()  # [R][S][C] -> [C][1][R][S]
                self.params[(op.id, name)] = v
        self.mom = {k: torch.zeros_like(v) for k, v in self.params.items()}
        self.running = {op.id: [op.attrs["running_mean"].to(dtype).clone(),
                                op.attrs["running_var"].to(dtype).clone()]
                        for op in net.ops if op.kind in ("bn", "bnrelu", "bnrelu6", "bnaddrelu")}
        self.saved = {}
        self.grads = {}
        self.seed = 0  # dropout step seed: the engine's device counter, advanced once per step


def _mask_gate(mask, dy):
    """dy where the packed NHWC sign-mask bit is set, else 0 (relu_bwd_mask)."""
    bits = torch.from_numpy(unpack_sign_mask(mask, dy.numel()))
    keep = bits.view(dy.shape[0], dy.shape[2], dy.shape[3], dy.shape[1]).permute(0, 3, 1, 2)
    return torch.where(keep, dy, torch.zeros_like(dy))


def _bn_stats(x, eps):
    mean = x.mean(dim=(0, 2, 3))
    var = x.var(dim=(0, 2, 3), unbiased=False)
    return mean, 1.0 / torch.sqrt(var + eps), var


def _bn_apply(x, mean, invstd, g, b):
    v = lambda t: t.view(1, -1, 1, 1)
    return (x - v(mean)) * v(invstd) * v(g) + v(b)


def _bn_pre(x, mean, invstd, g, b):
    """The engine's BN affine value with its exact rounding (csrc/local_ops.cuh:bn_aff):
    t = fp32(fp32(x - mean) * invstd), then one fused multiply-add t * gamma + beta rounded
    once to fp32.  t * gamma is exact in fp64 (24 x 24 bits), so fp64 t*gamma + beta has the
    exact sum's sign; rounding it to fp32 matches the FMA except in the rare double-rounding
    case.  Recomputed ReLU gates use this so they agree with the GPU's bit for bit."""
    v = lambda t: t.view(1, -1, 1, 1)
    t = ((x.float() - v(mean.float())) * v(invstd.float())).double()
    return (t * v(g.double()) + v(b.double())).float()


def run_step(state: CpuState, schedule: dict, images: torch.Tensor, labels: torch.Tensor, record=None,
             forced=None, fwd_record=None, forced_stats=None):
    """One training step following ``schedule`` (a schedule document). Returns the loss.

    ``forced`` (node id -> NCHW tensor) substitutes the given forward outputs
    for the oracle's own (first forward and every recompute alike).  Parity
    tests use it to feed the GPU's activations so that ReLU/maxpool
    derivatives, which are discontinuous, are evaluated on the same inputs on
    both sides; ``record`` collects input gradients per stage;
    ``fwd_record`` collects the oracle's own forward outputs (computed from the
    possibly forced inputs) before any substitution; ``forced_stats`` (BN node id ->
    (mean, invstd)) substitutes the GPU's saved batch statistics for the oracle's own, so
    that recomputed ReLU gates (fused BN+ReLU backward from x) see the same values -- at
    batch 184 a 1e-7 difference in invstd flips hundreds of gates per step.
    """
    net = state.net
    dt = state.dtype
    P = state.params
    n_nodes = net.n
    ints = {u: op_id for op_id, u in net.intermediate_of.items()}
    readers = {i: [] for i in range(1, n_nodes + 1)}
    for op in net.ops:
        for j in op.deps:
            readers[j].append(op.id)
    last_use = {i: max(r) if r else i for i, r in readers.items()}
    act: dict[int, object] = {}
    grad: dict[int, torch.Tensor] = {}
    loss_val = None

    def x_of(i):
        if i not in act:
            raise RuntimeError(f"tensor {i} read while not live")
        return act[i]

    def fwd(op, mode, want_int):
        y, extra = _fwd(op, mode, want_int)
        if fwd_record is not None and mode == "forward":
            fwd_record[op.id] = y
        if forced is not None and op.id in forced and op.kind != "xent":
            y = forced[op.id].to(dt)
        return y, extra

    def _fwd(op, mode, want_int):
        nonlocal loss_val
        xs = [x_of(j) for j in op.deps]
        extra = None
        if op.kind == "wgrad":  # split conv's weight-gradient anchor: no forward tensor
            y = torch.zeros(0, dtype=dt)
        elif op.kind == "input":
            c_pad = op.shape[3]
            y = torch.zeros(images.shape[0], c_pad, images.shape[2], images.shape[3], dtype=dt)
            y[:, :images.shape[1]] = images.to(dt)
        elif op.kind in ("conv", "convrelu"):
            a = op.attrs
            y = F.conv2d(xs[0], P[(op.id, "weight")], P.get((op.id, "bias")), stride=a["stride"], padding=a["pad"])
            if op.kind == "convrelu":  # fused ReLU: the mask is the pre-activation's sign (relu_fwd in place)
                if want_int:
                    extra = pack_sign_mask(y.permute(0, 2, 3, 1).numpy())
                y = torch.where(y > 0, y, torch.zeros_like(y))
        elif op.kind == "dropout":
            y = xs[0] * _dropout_scale(op, xs[0], state.seed)
        elif op.kind == "concat":
            y = torch.cat([x_of(j) for j in op.attrs["inputs"]], dim=1)
        elif op.kind == "convT":
            a = op.attrs
            y = F.conv_transpose2d(xs[0], P[(op.id, "weight")], P.get((op.id, "bias")), stride=a["stride"],
                                   padding=a["pad"])
        elif op.kind == "dwconv":
            a = op.attrs
            y = F.conv2d(xs[0], P[(op.id, "weight")], stride=a["stride"], padding=a["pad"], groups=xs[0].shape[1])
        elif op.kind == "relu6":
            x = xs[0]
            y = torch.clamp(x, 0.0, 6.0)
            if want_int:
                gate = (x > 0) & (x < 6)
                extra = pack_sign_mask(torch.where(gate, 1.0, -1.0).permute(0, 2, 3, 1).numpy()
                                       if x.dim() == 4 else torch.where(gate, 1.0, -1.0).numpy())
        elif op.kind in ("bn", "bnrelu", "bnrelu6", "bnaddrelu"):
            g, b = P[(op.id, "weight")], P[(op.id, "bias")]
            xin = x_of(op.attrs["x"]) if op.kind == "bnaddrelu" else xs[0]
            if mode == "forward":
                mean, invstd, var = _bn_stats(xin, op.attrs["eps"])
                state.saved[op.id] = (mean, invstd)
                if forced_stats is not None and op.id in forced_stats:
                    state.saved[op.id] = tuple(t.to(dt) for t in forced_stats[op.id])
                m = op.attrs["momentum"]
                rows = xin.numel() // xin.shape[1]
                rm, rv = state.running[op.id]
                rm.mul_(1 - m).add_(m * mean)
                rv.mul_(1 - m).add_(m * var * rows / max(rows - 1, 1))
            mean, invstd = state.saved[op.id]
            y = _bn_apply(xin, mean, invstd, g, b)
            if op.kind == "bnaddrelu":  # fused: relu(BN(x) + skip); the BN output is never kept
                y = y + x_of(op.attrs["skip"])
                y = torch.where(y > 0, y, torch.zeros_like(y))
            elif op.kind == "bnrelu":  # fused: relu(BN(x)); the BN output is never kept
                y = torch.where(y > 0, y, torch.zeros_like(y))
            elif op.kind == "bnrelu6":  # fused: relu6(BN(x))
                y = torch.clamp(y, 0.0, 6.0)
        elif op.kind == "relu":
            x = xs[0]
            y = torch.where(x > 0, x, torch.zeros_like(x))
            if want_int:
                extra = pack_sign_mask((x.permute(0, 2, 3, 1) if x.dim() == 4 else x).numpy())
        elif op.kind == "add":
            y = xs[0] + xs[1]
        elif op.kind == "addrelu":
            y = xs[0] + xs[1]
            y = torch.where(y > 0, y, torch.zeros_like(y))
        elif op.kind == "maxpool":
            a = op.attrs
            y, flat = F.max_pool2d(xs[0], a["r"], a["stride"], a["pad"], ceil_mode=a.get("ceil", False),
                                   return_indices=True)
            if want_int:
                extra = _window_index(flat, xs[0].shape, y.shape, a)
        elif op.kind == "avgpool":
            y = xs[0].mean(dim=(2, 3))
        elif op.kind == "fc":
            y = F.linear(_flat_nhwc(xs[0]), P[(op.id, "weight")], P[(op.id, "bias")])
        elif op.kind == "xent":  # (N, K) logits, or per-pixel (N, K, H, W) with (N, H, W) labels
            y = F.cross_entropy(xs[0], labels.long())
            loss_val = float(y)
        else:
            raise ValueError(op.kind)
        return y, extra

    def put_grad(j, val, created):
        if net.grad_bytes(net.op(j)) == 0:
            return
        if j in created:
            grad[j] = val
        else:
            grad[j] = grad[j] + val

    def bwd(op, impl, created):
        if op.kind == "input":
            return
        if op.kind == "wgrad":  # split conv: dW from the conv input and the conv's output gradient
            conv = net.op(op.attrs["conv"])
            a = conv.attrs
            w = P[(conv.id, "weight")]
            if conv.kind == "convrelu":  # runs before the conv's stage: gates its dy in place with the mask
                grad[conv.id] = _mask_gate(x_of(net.intermediate_of[conv.id]), grad[conv.id])
            state.grads[(conv.id, "weight")] = torch.nn.grad.conv2d_weight(x_of(conv.deps[0]), w.shape, grad[conv.id],
                                                                          a["stride"], a["pad"])
            return
        dy = grad[op.id]
        if op.kind == "convrelu" and not op.attrs.get("split"):
            dy = _mask_gate(x_of(net.intermediate_of[op.id]), dy)
        if op.kind in ("conv", "convrelu"):
            a = op.attrs
            j = op.deps[0]
            w = P[(op.id, "weight")]
            if a.get("split"):  # dgrad only: reads dy and w, never x
                in_shape = net.op(j).shape
                shp = (in_shape[0], in_shape[3], in_shape[1], in_shape[2])
                if net.grad_bytes(net.op(j)) > 0:
                    put_grad(j, torch.nn.grad.conv2d_input(shp, w, dy, a["stride"], a["pad"]), created)
                if (op.id, "bias") in P:
                    state.grads[(op.id, "bias")] = dy.sum(dim=(0, 2, 3))
                return
            x = x_of(j)
            if net.grad_bytes(net.op(j)) > 0:
                put_grad(j, torch.nn.grad.conv2d_input(x.shape, w, dy, a["stride"], a["pad"]), created)
            state.grads[(op.id, "weight")] = torch.nn.grad.conv2d_weight(x, w.shape, dy, a["stride"], a["pad"])
            if (op.id, "bias") in P:
                state.grads[(op.id, "bias")] = dy.sum(dim=(0, 2, 3))
        elif op.kind == "dropout":
            put_grad(op.deps[0], dy * _dropout_scale(op, dy, state.seed), created)
        elif op.kind == "convT":
            a = op.attrs
            j = op.deps[0]
            x = x_of(j)
            w = P[(op.id, "weight")]
            if net.grad_bytes(net.op(j)) > 0:
                put_grad(j, F.conv2d(dy, w, stride=a["stride"], padding=a["pad"]), created)
            state.grads[(op.id, "weight")] = torch.nn.grad.conv2d_weight(dy, w.shape, x, a["stride"], a["pad"])
            if (op.id, "bias") in P:
                state.grads[(op.id, "bias")] = dy.sum(dim=(0, 2, 3))
        elif op.kind == "concat":
            off = 0
            for j in op.attrs["inputs"]:
                cj = net.op(j).shape[3]
                put_grad(j, dy[:, off:off + cj].contiguous(), created)
                off += cj
        elif op.kind == "dwconv":
            a = op.attrs
            j = op.deps[0]
            x = x_of(j)
            w = P[(op.id, "weight")]
            grp = x.shape[1]
            if net.grad_bytes(net.op(j)) > 0:
                put_grad(j, torch.nn.grad.conv2d_input(x.shape, w, dy, a["stride"], a["pad"], groups=grp), created)
            state.grads[(op.id, "weight")] = torch.nn.grad.conv2d_weight(x, w.shape, dy, a["stride"], a["pad"],
                                                                         groups=grp)
        elif op.kind == "relu6":
            j = op.deps[0]
            if impl == "bwd-mask":
                bits = torch.from_numpy(unpack_sign_mask(x_of(net.intermediate_of[op.id]), dy.numel()))
                if dy.dim() == 4:
                    keep = bits.view(dy.shape[0], dy.shape[2], dy.shape[3], dy.shape[1]).permute(0, 3, 1, 2)
                else:
                    keep = bits.view(dy.shape)
            else:
                s_ = x_of(op.id) if impl == "bwd-out" else x_of(j)
                keep = (s_ > 0) & (s_ < 6)
            put_grad(j, torch.where(keep, dy, torch.zeros_like(dy)), created)
        elif op.kind in ("bn", "bnrelu", "bnrelu6", "bnaddrelu"):
            j = op.attrs["x"] if op.kind == "bnaddrelu" else op.deps[0]
            g, b = P[(op.id, "weight")], P[(op.id, "bias")]
            mean, invstd = state.saved[op.id]
            v = lambda t: t.view(1, -1, 1, 1)
            if op.kind == "bnrelu":  # gate by the recomputed BN output's sign (PAPER App. D, K10)
                dy = torch.where(_bn_pre(x_of(j), mean, invstd, g, b) > 0, dy, torch.zeros_like(dy))
            elif op.kind == "bnrelu6":
                z = _bn_pre(x_of(j), mean, invstd, g, b)
                dy = torch.where((z > 0) & (z < 6), dy, torch.zeros_like(dy))
            elif op.kind == "bnaddrelu":  # gate from z (bwd-out) or recomputed from x and skip (bwd-in)
                if impl == "bwd-out":
                    gate = x_of(op.id) > 0
                else:
                    gate = (_bn_pre(x_of(j), mean, invstd, g, b) + x_of(op.attrs["skip"]).float()) > 0
                dy = torch.where(gate, dy, torch.zeros_like(dy))
                put_grad(op.attrs["skip"], dy.clone(), created)
            if impl == "bwd-in" or op.kind == "bnaddrelu":  # bnaddrelu's bwd-out names the gate source only
                xhat = (x_of(j) - v(mean)) * v(invstd)
            else:
                gc = torch.where(g.abs() < 1e-12, torch.full_like(g, 1e-12) * torch.where(g < 0, -1.0, 1.0), g)
                xhat = (x_of(op.id) - v(b)) / v(gc)
            m = dy.numel() // dy.shape[1]
            sdy = dy.sum(dim=(0, 2, 3))
            sdx = (dy * xhat).sum(dim=(0, 2, 3))
            state.grads[(op.id, "weight")] = sdx
            state.grads[(op.id, "bias")] = sdy
            put_grad(j, v(g * invstd) * (dy - v(sdy) / m - xhat * v(sdx) / m), created)
        elif op.kind == "relu":
            j = op.deps[0]
            if impl == "bwd-mask":
                bits = torch.from_numpy(unpack_sign_mask(x_of(net.intermediate_of[op.id]), dy.numel()))
                if dy.dim() == 4:
                    keep = bits.view(dy.shape[0], dy.shape[2], dy.shape[3], dy.shape[1]).permute(0, 3, 1, 2)
                else:
                    keep = bits.view(dy.shape)
            elif impl == "bwd-out":
                keep = x_of(op.id) > 0
            else:
                keep = x_of(j) > 0
            put_grad(j, torch.where(keep, dy, torch.zeros_like(dy)), created)
        elif op.kind == "add":
            for j in op.deps:
                put_grad(j, dy.clone(), created)
        elif op.kind == "addrelu":
            gate = x_of(op.id) > 0 if impl == "bwd-out" else (x_of(op.deps[0]) + x_of(op.deps[1])) > 0
            g = torch.where(gate, dy, torch.zeros_like(dy))
            for j in op.deps:
                put_grad(j, g.clone(), created)
        elif op.kind == "maxpool":
            a = op.attrs
            j = op.deps[0]
            in_shape = net.op(j).shape
            shp = (in_shape[0], in_shape[3], in_shape[1], in_shape[2])
            if impl == "bwd-idx":
                widx = x_of(net.intermediate_of[op.id])
                flat = _flat_index(widx, shp, dy.shape, a)
            else:
                _, flat = F.max_pool2d(x_of(j), a["r"], a["stride"], a["pad"], ceil_mode=a.get("ceil", False),
                                       return_indices=True)
            dx = torch.zeros(shp, dtype=dt).view(shp[0], shp[1], -1)
            dx.scatter_add_(2, flat.view(shp[0], shp[1], -1), dy.reshape(shp[0], shp[1], -1))
            put_grad(j, dx.view(shp), created)
        elif op.kind == "avgpool":
            j = op.deps[0]
            n, h, w, c = net.op(j).shape
            put_grad(j, (dy / (h * w)).view(n, c, 1, 1).expand(n, c, h, w).contiguous(), created)
        elif op.kind == "fc":
            j = op.deps[0]
            x = x_of(j)
            dx = dy @ P[(op.id, "weight")]
            if x.dim() == 4:  # back to NCHW from the NHWC flattening
                n, c, h, w = x.shape
                dx = dx.view(n, h, w, c).permute(0, 3, 1, 2).contiguous()
            put_grad(j, dx, created)
            state.grads[(op.id, "weight")] = dy.t() @ _flat_nhwc(x)
            state.grads[(op.id, "bias")] = dy.sum(dim=0)
        elif op.kind == "xent":
            j = op.deps[0]
            z = x_of(j)
            p = torch.softmax(z, dim=1)
            if z.dim() == 4:  # per-pixel loss: mean over N*H*W
                p = p - F.one_hot(labels.long(), z.shape[1]).permute(0, 3, 1, 2).to(p.dtype)
                put_grad(j, p * (dy / (z.numel() // z.shape[1])), created)
            else:
                p[torch.arange(z.shape[0]), labels.long()] -= 1.0
                put_grad(j, p * (dy / z.shape[0]), created)
        else:
            raise ValueError(op.kind)

    # ---------------------------------------------------------------- forward
    row0 = set(schedule["forward_store"])
    for op in net.ops:
        mid = net.intermediate_of.get(op.id)
        y, extra = fwd(op, "forward", mid in row0)
        act[op.id] = y
        if mid in row0:
            act[mid] = extra
        for j in list(act):
            if j <= op.id and j not in ints and j not in row0 and last_use[j] <= op.id:
                del act[j]

    # ---------------------------------------------------------------- stages
    carried = row0
    for t, st in enumerate(schedule["stages"], start=1):
        k = st["node"]
        keep = set(st["store"])
        impl_b = st["backward_impl"]
        bdeps = _bwd_deps(net, k, impl_b)
        for u in carried - keep:
            act.pop(u, None)
        entries = [(u, impl) for u, impl in st["recompute"] if u not in ints]
        planned = {ints[u] for u, _ in st["recompute"] if u in ints}
        last = {}
        for e, (i, _) in enumerate(entries):
            for j in net.op(i).deps:
                last[j] = e
            last[i] = e
            if i in planned:
                last[net.intermediate_of[i]] = e
        for d in bdeps:
            last[d] = len(entries)

        def release(slot):
            for u, s in list(last.items()):
                if s == slot and u not in keep and u in act:
                    del act[u]

        for e, (i, impl) in enumerate(entries):
            op = net.op(i)
            y, extra = fwd(op, "recompute", i in planned)
            act[i] = y
            if i in planned:
                act[net.intermediate_of[i]] = extra
            release(e)
        created = set()
        if t == 1:
            grad[k] = torch.ones((), dtype=dt)
        for j in net.op(k).deps:
            if j not in grad:
                created.add(j)
        bwd(net.op(k), impl_b, created)
        if record is not None:
            record[t] = {j: grad[j].clone() for j in net.op(k).deps if j in grad}
        grad.pop(k, None)
        release(len(entries))
        carried = keep

    state.seed += 1
    # ---------------------------------------------------------------- SGD
    for key, w in P.items():
        g = state.grads[key]
        d = g + state.weight_decay * w
        buf = state.mom[key]
        buf.mul_(state.momentum).add_(d)
        w.sub_(state.lr * buf)
    return loss_val


def _flat_nhwc(x):
    """fc input flattened in the engine's NHWC element order (2-D inputs unchanged)."""
    return x.permute(0, 2, 3, 1).reshape(x.shape[0], -1) if x.dim() == 4 else x


def _dropout_scale(op, like, seed):
    """keep / (1 - p) as a tensor shaped like ``like`` (mask drawn over NHWC order)."""
    import numpy as np

    p = float(np.float32(op.attrs["p"]))
    scale = np.float32(1.0 / (1.0 - p))
    keep = torch.from_numpy(keep_mask(like.numel(), p, seed, op.id))
    s = torch.where(keep, torch.tensor(scale, dtype=like.dtype), torch.tensor(0.0, dtype=like.dtype))
    if like.dim() == 4:
        n, c, h, w = like.shape
        return s.view(n, h, w, c).permute(0, 3, 1, 2)
    return s.view(like.shape)


def _bwd_deps(net, k, impl):
    if hasattr(net, "bwd_deps"):  # frozen network (oracle/netspec.py)
        return net.bwd_deps(k, impl)
    op = net.op(k)
    fv, bv = net.variants(op)
    for name, _, deps in bv:
        if name == impl:
            return list(deps)
    raise KeyError(impl)


def _window_index(flat, x_shape, y_shape, a):
    """torch flat input index -> 8-bit window index r*S+s (NHWC order numpy array)."""
    n, c, h, w = x_shape
    _, _, p, q = y_shape
    hh, ww = flat // w, flat % w
    pp = torch.arange(p).view(1, 1, -1, 1)
    qq = torch.arange(q).view(1, 1, 1, -1)
    r = hh - (pp * a["stride"] - a["pad"])
    s = ww - (qq * a["stride"] - a["pad"])
    idx = (r * a["s"] + s).to(torch.uint8)
    return idx.permute(0, 2, 3, 1).contiguous()


def _flat_index(widx, x_shape, y_shape, a):
    n, c, h, w = x_shape
    _, _, p, q = y_shape
    wi = widx.permute(0, 3, 1, 2).long()
    pp = torch.arange(p).view(1, 1, -1, 1)
    qq = torch.arange(q).view(1, 1, 1, -1)
    hh = pp * a["stride"] - a["pad"] + wi // a["s"]
    ww = qq * a["stride"] - a["pad"] + wi % a["s"]
    return hh * w + ww


def params_nhwc(state: CpuState):
    """Parameters in the engine layout (conv weights KRSC) for comparison with the GPU."""
    out = {}
    for (nid, name), v in state.params.items():
        if state.net.op(nid).kind in ("conv", "convrelu", "convT") and name == "weight":
            v = v.permute(0, 2, 3, 1).contiguous()
        elif state.net.op(nid).kind == "dwconv" and name == "weight":
            v = v.squeeze(1).permute(1, 2, 0).contiguous()
        out[(nid, name)] = v
    return out

"""The recompute executor (SURVEY.md §2.2 R1 + R2): replays a Schedule on a B200.

``execute(schedule, g, catalog, runtime=rt)`` is the GPU counterpart of the
reference ``simulate(schedule, g, catalog)`` (pkg/src/remsched/schedule.py:320):
the same plan goes in, the same ``Trace`` comes out, and in between every
ledger step launches the sm_100a kernel of the chosen catalog variant.

* Ledger.  Steps come from :func:`schedule.walk`, the one replay of Alg. 1-2
  shared with ``simulate``; the executed trace is therefore byte-identical to
  the simulator's (tests/test_engine_*.py check it against the reference).
* Memory.  Everything the graph folds into ``params_bytes`` (parameters,
  grads, momenta, BN statistics, kernel scratch, the staged input batch,
  labels) lives in one fixed region of exactly that size.  Every activation,
  intermediate, gradient and workspace instance of the ledger lives in one
  arena whose offsets are planned statically from the ledger's alloc/free
  points (csrc/arena.cpp); the arena is sized by the plan and capped by the
  budget, so the physical peak is params_bytes + arena high-water mark.
* Launch.  Each step is pre-bound to a ctypes call with resolved device
  pointers; ``Runtime.step`` just runs the list (and can be captured into a
  CUDA graph, ``Runtime.capture``).
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import torch

from . import _native
from .bound import check_schedule
from .costmodel import Catalog
from .graph import Graph, compute_dependency_sets
from .schedule import Schedule, SimulationError, Trace, ledger, validate

__all__ = ["Runtime", "Plan", "ExecResult", "BudgetExceeded", "execute", "lifetimes", "place_blocks"]

ALIGN = 256        # fixed region (params, grads, momentum, ...): cudaMalloc-like alignment
ARENA_ALIGN = 16   # arena blocks: TMA / float4 alignment; every graph size is a multiple of it
                   # (tracer.py), so a gap-free packing is exactly the ledger peak


class BudgetExceeded(RuntimeError):
    """The planned physical footprint exceeds the byte budget (CLI exit 6)."""


def _round(v: int) -> int:
    return (v + ALIGN - 1) // ALIGN * ALIGN


@dataclass
class Plan:
    schedule: Schedule
    trace: Trace
    calls: list
    arena_bytes: int
    ledger_peak: int
    bound_peak: int | None
    n_blocks: int
    launches: int
    step_kinds: dict = field(default_factory=dict)
    g: Graph | None = None
    catalog: Catalog | None = None
    graph: object = None  # captured torch.cuda.CUDAGraph (Runtime.capture)

    @property
    def within_bound(self) -> bool | None:
        """params_bytes + arena high-water mark <= check_schedule's ILP bound."""
        if self.bound_peak is None or self.g is None:
            return None
        return self.g.params_bytes + self.arena_bytes <= self.bound_peak


@dataclass
class ExecResult:
    trace: Trace
    loss: float
    ledger_peak: int           # simulate()'s peak (logical bytes, incl. params_bytes)
    physical_peak: int         # params_bytes + planned arena high-water mark
    bound_peak: int | None     # check_schedule() modeled peak (the ILP bound)
    arena_bytes: int
    params_bytes: int
    torch_peak_bytes: int      # torch.cuda.max_memory_allocated during the step
    launches: int


class Runtime:
    """Device state for one network on one GPU: the fixed region and the kernels."""

    def __init__(self, net, device="cuda:0", lr=0.1, momentum=0.9, weight_decay=0.0,
                 grad_scale=1.0, budget_bytes: int | None = None):
        self.net = net
        self.device = torch.device(device)
        self.lib = _native.lib()
        if self.lib.device_check() != 0:
            raise _native.NativeError("libmonet_b200 needs an sm_100 (B200) device")
        self.lr, self.momentum, self.weight_decay = lr, momentum, weight_decay
        self.grad_scale = grad_scale
        self.budget_bytes = budget_bytes
        self.params_bytes = net.params_bytes()
        self.fixed = torch.zeros(self.params_bytes, dtype=torch.uint8, device=self.device)
        self._carve()
        self.arena = None
        self._plans: dict[int, Plan] = {}
        self.graph = None
        self.comm = None  # set by dp.DataParallel for the gradient allreduce
        # batch prefetch (prefetch / train_step): copy stream and its two events
        self._copy_stream = None
        self._staging_free = torch.cuda.Event()
        self._staged = torch.cuda.Event()
        self._pending_labels = None

    # ------------------------------------------------------------ fixed region
    def _carve(self):
        lay = self.net.fixed_layout()
        base = 0
        self.region = {}
        for name, nbytes in lay.items():
            self.region[name] = (base, nbytes)
            base += _round(nbytes)
        assert base == self.params_bytes

        def f32(name, count=None):
            off, nb = self.region[name]
            n = nb // 4 if count is None else count
            return self.fixed[off:off + 4 * n].view(torch.float32)

        self.params = f32("params")
        self.grads = f32("grads")
        self.mom = f32("momentum")
        self.staging = f32("staging_input")
        off, nb = self.region["labels"]
        self.labels = self.fixed[off:off + nb].view(torch.int32)
        self.consts = f32("consts", 4)
        self.consts[0] = 1.0
        # dropout step seed (uint64 at consts + 8): read by the kernels at run time,
        # advanced on the device after every optimizer step
        off = self.region["consts"][0]
        self.seed = self.fixed[off + 8:off + 16].view(torch.int64)
        self.seed.zero_()
        self.seed_ptr = self.fixed.data_ptr() + off + 8
        self.scratch_ptr = self.fixed.data_ptr() + self.region["scratch"][0]
        self.pview, self.gview = {}, {}
        pos = 0
        for nid, name, t in self.net.param_items():
            n = t.numel()
            self.params[pos:pos + n].copy_(t.reshape(-1))
            self.pview[(nid, name)] = self.params[pos:pos + n]
            self.gview[(nid, name)] = self.grads[pos:pos + n]
            pos += n
        # pre-split conv weights (bf16 hi / lo planes, tracer.Network.w16_segments)
        segs = self.net.w16_segments()
        self.w16, self.w16_count = {}, len(segs)
        self.w16_max = max((n for _, _, _, n in segs), default=0)
        if segs:
            off, nb = self.region["w16_table"]
            table = self.fixed[off:off + 24 * len(segs)].view(torch.int64)
            table.copy_(torch.tensor([[src, dst, n] for _, src, dst, n in segs], dtype=torch.int64).reshape(-1))
            self.w16_table = self.fixed.data_ptr() + off
            off, nb = self.region["w16"]
            self.w16_hi = self.fixed.data_ptr() + off
            self.w16_lo = self.w16_hi + nb // 2
            for nid, _, dst, _ in segs:
                self.w16[nid] = (self.w16_hi + 2 * dst, self.w16_lo + 2 * dst)
        # MONET_NO_CONV_STATS=1 (measurement switch): BNs compute their own statistics
        self.stats_convs = {} if os.environ.get("MONET_NO_CONV_STATS") else self.net.stats_convs()
        self.stats_bns = {bn: conv for conv, bn in self.stats_convs.items()}
        self.conv_stats_ptr = self.fixed.data_ptr() + self.region["conv_stats"][0]
        stats = f32("bn_stats")
        self.bn = {}
        pos = 0
        for op in self.net.ops:
            if op.kind not in ("bn", "bnrelu", "bnrelu6", "bnaddrelu"):
                continue
            c = op.shape[-1]
            views = [stats[pos + j * c: pos + (j + 1) * c] for j in range(4)]
            pos += 4 * c
            views[2].copy_(op.attrs["running_mean"])
            views[3].copy_(op.attrs["running_var"])
            self.bn[op.id] = views  # saved_mean, saved_invstd, running_mean, running_var

    def set_batch(self, images: torch.Tensor, labels: torch.Tensor):
        """Stage one batch: images NCHW (any device), labels (N,) ints."""
        n, c, h, w = images.shape
        x = self.staging.view(n, h, w, -1)
        if x.shape[3] != c:
            x[..., c:].zero_()
        x[..., :c].copy_(images.permute(0, 2, 3, 1), non_blocking=True)
        self.labels.copy_(labels.to(torch.int32).reshape(-1), non_blocking=True)  # (N,) or per-pixel (N,H,W)

    def set_batch_nhwc(self, images_nhwc: torch.Tensor, labels: torch.Tensor):
        """Stage a batch already in the engine layout (N,H,W,Cpad) — one copy each."""
        self.staging.copy_(images_nhwc.reshape(-1), non_blocking=True)
        self.labels.copy_(labels.reshape(-1), non_blocking=True)

    def loss_value(self) -> float:
        return float(self.consts[1].item())

    def loss_tensor(self) -> torch.Tensor:
        """The last step's loss as a 1-element device tensor (no host sync)."""
        return self.consts[1:2]

    def prefetch(self, images: torch.Tensor, labels: torch.Tensor):
        """Start staging the NEXT step's batch (pinned host tensors, engine NHWC layout) on a
        copy stream.  The copy waits only until the running step has made its last read of
        the staging buffer (the input copies into the arena, captured as the first of the
        step's two graphs), so it overlaps that step's remaining work; the following
        train_step(plan) without images waits for it.  A data loader's double buffer, with
        no extra device memory."""
        if self._copy_stream is None:
            self._copy_stream = torch.cuda.Stream(self.device)
        self._copy_stream.wait_event(self._staging_free)
        with torch.cuda.stream(self._copy_stream):
            self.staging.copy_(images.reshape(-1), non_blocking=True)
        self._staged.record(self._copy_stream)
        self._pending_labels = labels

    def train_step(self, plan: "Plan", images: torch.Tensor | None = None,
                   labels: torch.Tensor | None = None) -> torch.Tensor:
        """Public per-step call: stage the batch (host or device, NCHW or engine NHWC
        layout) -- or take the one ``prefetch`` staged --, run the scheduled
        forward/backward/SGD, return the device loss."""
        if images is not None:
            if images.dim() == 4 and images.shape[1] in (1, 2, 3) and images.shape[-1] not in (1, 2, 3, 4):
                self.set_batch(images, labels)
            else:
                self.set_batch_nhwc(images, labels)
        elif self._pending_labels is not None:
            cur = torch.cuda.current_stream(self.device)
            cur.wait_event(self._staged)
            self.labels.copy_(self._pending_labels.reshape(-1), non_blocking=True)
            self._pending_labels = None
        if plan.calls is None:
            raise RuntimeError("this plan was invalidated when the runtime's arena was reallocated; "
                               "call Runtime.plan() again")
        if getattr(plan, "graph", None) is not None:
            plan.graph.replay()
        else:
            self.run(plan)
            self._staging_free.record()  # uncaptured: the staging buffer is free after the whole step
        return self.loss_tensor()

    def capture(self, plan: "Plan"):
        """Capture the whole training step into a CUDA graph (plan.graph); the
        kernels' device pointers are static because the arena is planned."""
        if self.comm is not None and not getattr(self.comm, "capturable", False):
            raise RuntimeError("CUDA-graph capture needs the native (stream-ordered) DataParallel backend; "
                               "the torch.distributed backend issues its all-reduces from Python")
        self.run(plan)  # first launches set kernel attributes outside capture
        torch.cuda.synchronize(self.device)
        # two graphs, cut after the step's last read of the staging buffer (the input's
        # forward copy, or its last recompute), so a prefetch of the next batch can start there
        sptr = self.staging.data_ptr()
        cut = 1 + max((i for i, grp in enumerate(plan.calls)
                       if any(c[0] == "copy" and c[2] == sptr for c in grp)), default=-1)
        cut = max(cut, 1)
        parts = []
        side = torch.cuda.Stream(self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        for groups in (plan.calls[:cut], plan.calls[cut:]):
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.stream(side):
                with torch.cuda.graph(graph, stream=side):
                    sp = C.c_void_p(side.cuda_stream)
                    for grp in groups:
                        self._run_group(grp, sp, _cudart())
            parts.append(graph)
        torch.cuda.current_stream(self.device).wait_stream(side)
        torch.cuda.synchronize(self.device)
        plan.graph = _StepGraph(parts[0], parts[1], self._staging_free)
        return plan.graph

    # ------------------------------------------------------------ planning
    def plan(self, schedule: Schedule, g: Graph, catalog: Catalog, check_bound: bool = True) -> Plan:
        key = (id(schedule), id(g), id(catalog))
        hit = self._plans.get(key)
        if hit is not None and hit.schedule is schedule and hit.g is g and hit.catalog is catalog:
            return hit
        self._check_graph(g)
        tags = validate(schedule, g, compute_dependency_sets(g), catalog)
        if tags:
            raise SimulationError(f"schedule is not executable: {tags}")
        steps, trace = ledger(schedule, g, catalog)
        blocks, step_blocks = lifetimes(steps, g)
        cap = 0 if self.budget_bytes is None else max(1, self.budget_bytes - self.params_bytes)
        arena_bytes, offsets = place_blocks(blocks, cap)
        fixed_peak = self.params_bytes + arena_bytes
        if self.budget_bytes is not None and fixed_peak > self.budget_bytes:
            raise BudgetExceeded(f"planned footprint {fixed_peak} B exceeds budget {self.budget_bytes} B "
                                 f"(ledger peak {trace.peak_memory} B)")
        if self.arena is None or self.arena.numel() < arena_bytes:
            # every cached plan (and its captured graph) holds absolute pointers into the
            # old arena: drop them before the buffer goes away
            for old in self._plans.values():
                old.graph = None
                old.calls = None
            self._plans.clear()
            self.arena = None
            torch.cuda.empty_cache()
            self.arena = torch.empty(max(arena_bytes, ALIGN), dtype=torch.uint8, device=self.device)
        bound = None
        if check_bound:
            ok, bound, _ = check_schedule(g, compute_dependency_sets(g), catalog, schedule,
                                          self.budget_bytes if self.budget_bytes else 1 << 62)
        base = self.arena.data_ptr()
        calls, step_ptrs = [], []
        for s, sb in zip(steps, step_blocks):
            ptrs = {k: base + offsets[b] for k, b in sb["blocks"].items()}
            calls.append(self._bind(s, sb, ptrs, catalog))
            step_ptrs.append(ptrs)
        if calls and self.w16_count:
            # refresh the weights' bf16 split before the step's first use (the conv forwards /
            # input gradients load it, monet_conv_*_w16): one launch over all conv weights
            calls[0].insert(0, ("k", self.lib.dll.monet_split_bf16_segments,
                                (self.params.data_ptr(), self.w16_hi, self.w16_lo, self.w16_table,
                                 self.w16_count, self.w16_max, None)))
        calls.append(self._bind_optimizer())
        plan = Plan(schedule, trace, calls, arena_bytes, trace.peak_memory, bound, len(blocks),
                    sum(1 for group in calls for c in group if c[0] == "k"))
        plan.steps, plan.step_ptrs = steps, step_ptrs
        plan.g, plan.catalog = g, catalog
        self._plans[key] = plan
        return plan

    def _check_graph(self, g: Graph):
        net = self.net
        if g.n != net.n or any(g.output_bytes(op.id) != op.nbytes for op in net.ops):
            raise ValueError("graph does not describe this runtime's network")
        if g.params_bytes != self.params_bytes:
            raise ValueError(f"graph params_bytes {g.params_bytes} != runtime fixed region "
                             f"{self.params_bytes}")

    # ------------------------------------------------------------ binding
    def _bind(self, s, sb, ptrs, catalog):
        """Kernel calls of one ledger step: list of ("k", fn, args) / ("py", callable)."""
        net, lib = self.net, self.lib.dll
        op = net.op(s.node)
        st = lambda: torch.cuda.current_stream(self.device).cuda_stream
        out = []
        P = lambda key: ptrs[key]
        if s.kind in ("forward", "recompute"):
            y = P(("a", op.id))
            xs = [P(("in", j)) for j in op.deps]
            ws = ptrs.get(("ws",))
            if op.kind == "input":
                nb = op.nbytes
                out.append(("copy", y, self.staging.data_ptr(), nb))
            elif op.kind == "wgrad":
                pass  # a split conv's weight-gradient anchor: no forward work, no tensor
            elif op.kind in ("conv", "convrelu"):
                d = net.conv_desc(op)
                v = _native.CONV_VARIANTS[s.impl]
                wt = self.pview[(op.id, "weight")].data_ptr()
                hi, lo = self.w16.get(op.id, (None, None))
                bias = self.pview[(op.id, "bias")].data_ptr() if "bias" in op.params else None
                if s.kind == "forward" and op.id in self.stats_convs:  # + the next BN's batch statistics
                    out.append(("k", lib.monet_conv_fwd_w16_stats, (v, C.byref(d), xs[0], wt, hi, lo, bias, y,
                                                                    self.conv_stats_ptr, ws, s.workspace, None), d))
                else:
                    out.append(("k", lib.monet_conv_fwd_w16, (v, C.byref(d), xs[0], wt, hi, lo, bias, y, ws,
                                                              s.workspace, None), d))
                if op.kind == "convrelu":  # the fused ReLU, in place on y (+ its sign mask when planned)
                    mid = net.intermediate_of[op.id]
                    mask = P(("a", mid)) if mid in s.planned_ints else None
                    out.append(("k", lib.monet_relu_fwd, (y, y, mask, op.numel, None)))
            elif op.kind == "convT":
                d = net.conv_desc(op)
                v = _native.CONV_VARIANTS[s.impl]
                b = self.pview[(op.id, "bias")].data_ptr() if "bias" in op.params else None
                out.append(("k", lib.monet_convT_fwd, (v, C.byref(d), xs[0], self.pview[(op.id, "weight")].data_ptr(),
                                                       b, y, ws, s.workspace, None), d))
            elif op.kind == "concat":
                pix, ct, off = op.numel // op.shape[3], op.shape[3], 0
                for j in op.attrs["inputs"]:
                    cj = net.op(j).shape[3]
                    out.append(("k", lib.monet_channel_copy, (P(("in", j)), cj, 0, y, ct, off, cj, pix, 0, None)))
                    off += cj
            elif op.kind == "dwconv":
                d = net.conv_desc(op)
                out.append(("k", lib.monet_dwconv_fwd, (C.byref(d), xs[0], self.pview[(op.id, "weight")].data_ptr(),
                                                        y, None), d))
            elif op.kind == "relu6":
                mid = net.intermediate_of[op.id]
                mask = P(("a", mid)) if mid in s.planned_ints else None
                out.append(("k", lib.monet_relu6_fwd, (xs[0], y, mask, op.numel, None)))
            elif op.kind == "dropout":
                out.append(("k", lib.monet_dropout_fwd, (xs[0], y, op.numel, C.c_float(op.attrs["p"]),
                                                         self.seed_ptr, op.id, None)))
            elif op.kind == "bn":
                c = op.shape[-1]
                rows = op.numel // c
                sm, si, rm, rv = (t.data_ptr() for t in self.bn[op.id])
                gma = self.pview[(op.id, "weight")].data_ptr()
                bta = self.pview[(op.id, "bias")].data_ptr()
                if s.kind == "forward" and op.id in self.stats_bns:  # statistics left by the conv
                    out.append(("k", lib.monet_bn_stats_finalize, (self.conv_stats_ptr, rows, c, C.c_float(op.attrs["eps"]), C.c_float(op.attrs["momentum"]), 1, sm, si, rm, rv, None)))
                    out.append(("k", lib.monet_bn_fwd_replay, (xs[0], y, gma, bta, sm, si, rows, c, None)))
                elif s.kind == "forward":
                    out.append(("k", lib.monet_bn_fwd_train,
                                (xs[0], y, gma, bta, sm, si, rm, rv, rows, c, C.c_float(op.attrs["eps"]),
                                 C.c_float(op.attrs["momentum"]), 1, self.scratch_ptr, None)))
                else:  # recompute: reuse saved statistics, running stats untouched
                    out.append(("k", lib.monet_bn_fwd_replay, (xs[0], y, gma, bta, sm, si, rows, c, None)))
            elif op.kind in ("bnrelu", "bnrelu6"):
                c = op.shape[-1]
                rows = op.numel // c
                sm, si, rm, rv = (t.data_ptr() for t in self.bn[op.id])
                gma = self.pview[(op.id, "weight")].data_ptr()
                bta = self.pview[(op.id, "bias")].data_ptr()
                six = op.kind == "bnrelu6"
                if s.kind == "forward" and op.id in self.stats_bns:  # statistics left by the conv
                    out.append(("k", lib.monet_bn_stats_finalize, (self.conv_stats_ptr, rows, c, C.c_float(op.attrs["eps"]), C.c_float(op.attrs["momentum"]), 1, sm, si, rm, rv, None)))
                    out.append(("k", lib.monet_bnrelu6_fwd_replay if six else lib.monet_bnrelu_fwd_replay,
                                (xs[0], y, gma, bta, sm, si, rows, c, None)))
                elif s.kind == "forward":
                    out.append(("k", lib.monet_bnrelu6_fwd_train if six else lib.monet_bnrelu_fwd_train,
                                (xs[0], y, gma, bta, sm, si, rm, rv, rows, c, C.c_float(op.attrs["eps"]),
                                 C.c_float(op.attrs["momentum"]), 1, self.scratch_ptr, None)))
                else:
                    out.append(("k", lib.monet_bnrelu6_fwd_replay if six else lib.monet_bnrelu_fwd_replay,
                                (xs[0], y, gma, bta, sm, si, rows, c, None)))
            elif op.kind == "relu":
                mid = net.intermediate_of[op.id]
                mask = P(("a", mid)) if mid in s.planned_ints else None
                out.append(("k", lib.monet_relu_fwd, (xs[0], y, mask, op.numel, None)))
            elif op.kind == "add":
                out.append(("k", lib.monet_add_fwd, (xs[0], xs[1], y, op.numel, None)))
            elif op.kind == "addrelu":
                out.append(("k", lib.monet_addrelu_fwd, (xs[0], xs[1], y, op.numel, None)))
            elif op.kind == "bnaddrelu":
                c = op.shape[-1]
                rows = op.numel // c
                sm, si, rm, rv = (t.data_ptr() for t in self.bn[op.id])
                gma = self.pview[(op.id, "weight")].data_ptr()
                bta = self.pview[(op.id, "bias")].data_ptr()
                xp, kp = P(("in", op.attrs["x"])), P(("in", op.attrs["skip"]))
                if s.kind == "forward" and op.id in self.stats_bns:  # statistics left by the conv
                    out.append(("k", lib.monet_bn_stats_finalize, (self.conv_stats_ptr, rows, c, C.c_float(op.attrs["eps"]), C.c_float(op.attrs["momentum"]), 1, sm, si, rm, rv, None)))
                    out.append(("k", lib.monet_bnaddrelu_fwd_replay, (xp, kp, y, gma, bta, sm, si, rows, c, None)))
                elif s.kind == "forward":
                    out.append(("k", lib.monet_bnaddrelu_fwd_train,
                                (xp, kp, y, gma, bta, sm, si, rm, rv, rows, c, C.c_float(op.attrs["eps"]),
                                 C.c_float(op.attrs["momentum"]), 1, self.scratch_ptr, None)))
                else:
                    out.append(("k", lib.monet_bnaddrelu_fwd_replay, (xp, kp, y, gma, bta, sm, si, rows, c, None)))
            elif op.kind == "maxpool":
                d = net.pool_desc(op)
                mid = net.intermediate_of[op.id]
                idx = P(("a", mid)) if mid in s.planned_ints else None
                out.append(("k", lib.monet_maxpool_fwd, (C.byref(d), xs[0], y, idx, None), d))
            elif op.kind == "avgpool":
                n, h, w, c = net.op(op.deps[0]).shape
                out.append(("k", lib.monet_avgpool_fwd, (xs[0], y, n, h * w, c, None)))
            elif op.kind == "fc":
                n, fi = net.fc_dims(op)
                fo = op.shape[1]
                v = 1 if s.impl == "gemm-splitk" else 0
                out.append(("k", lib.monet_linear_fwd,
                            (v, xs[0], self.pview[(op.id, "weight")].data_ptr(),
                             self.pview[(op.id, "bias")].data_ptr(), y, n, fi, fo, ws, s.workspace, None)))
            elif op.kind == "xent":
                out.append(("k", lib.monet_xent_fwd, (xs[0], self.labels.data_ptr(), y, net.label_count(),
                                                      net.num_classes, self.scratch_ptr, None)))
                out.append(("copy", self.consts.data_ptr() + 4, y, 4))
            else:
                raise ValueError(op.kind)
            return out

        # backward
        out = self._bind_backward(s, op, P, ptrs)
        if self.comm is not None and op.id in self.comm.ready_nodes():
            # this stage finalizes a gradient bucket: start its all-reduce now (async,
            # ordered after the kernels above) so it overlaps the remaining stages
            out += self.comm.bucket_calls(op.id)
        return out

    def _bind_backward(self, s, op, P, ptrs):
        net, lib = self.net, self.lib.dll
        out = []
        dy = P(("g", op.id))
        ws = ptrs.get(("ws",))
        written = set()

        def acc(j):
            # first write of a gradient this step overwrites, every later one (another
            # consumer, or the same input read twice as in add(x, x)) accumulates
            a = 0 if (j in s.new_grads and j not in written) else 1
            written.add(j)
            return a

        def needs(j):
            # inputs without a gradient buffer (the network input) get no dx kernel
            return net.grad_bytes(net.op(j)) > 0

        def must(j):
            if not needs(j):
                raise ValueError(f"{op.kind} node {op.id} reads node {j} directly, which has no gradient "
                                 "buffer; this operator's backward kernel always writes its input gradient")

        if op.kind in ("bn", "bnrelu", "bnrelu6", "bnaddrelu", "addrelu", "maxpool", "avgpool", "fc"):
            for j in op.deps:
                must(j)
        elif op.kind == "xent":
            must(op.deps[0])  # further deps: the zero-byte wgrad anchors of a split graph
        if op.id == net.n:
            out.append(("copy", dy, self.consts.data_ptr(), 4))  # seed dL/dL = 1
        if op.kind == "input":
            return out
        if op.kind in ("conv", "convrelu"):
            d = net.conv_desc(op)
            v = _native.CONV_VARIANTS[s.impl]
            j = op.deps[0]
            wt = self.pview[(op.id, "weight")].data_ptr()
            if op.kind == "convrelu" and not op.attrs.get("split"):  # gate dy with the ReLU mask, in place
                out.append(("k", lib.monet_relu_bwd_mask, (P(("in", net.intermediate_of[op.id])), dy, dy, op.numel,
                                                           0, None)))
            if net.grad_bytes(net.op(j)) > 0:
                hi, lo = self.w16.get(op.id, (None, None))
                out.append(("k", lib.monet_conv_dgrad_w16, (v, C.byref(d), dy, wt, hi, lo, P(("g", j)), acc(j), ws,
                                                            s.workspace, None), d))
            if not op.attrs.get("split"):  # split convs: the weight gradient is the wgrad node's stage
                out.append(("k", lib.monet_conv_wgrad, (v, C.byref(d), P(("in", j)), dy,
                                                        self.gview[(op.id, "weight")].data_ptr(), 0, ws,
                                                        s.workspace, None), d))
            if "bias" in op.params:
                out.append(("k", lib.monet_bias_grad, (dy, self.gview[(op.id, "bias")].data_ptr(),
                                                       op.numel // op.shape[-1], op.shape[-1], 0, self.scratch_ptr,
                                                       None)))
        elif op.kind == "wgrad":  # weight gradient of a split conv: reads x and the conv's dy
            conv = net.op(op.attrs["conv"])
            d = net.conv_desc(conv)
            v = _native.CONV_VARIANTS[s.impl]
            if conv.kind == "convrelu":  # this stage runs before the conv's: gate its dy in place first
                out.append(("k", lib.monet_relu_bwd_mask, (P(("in", net.intermediate_of[conv.id])), P(("g", conv.id)),
                                                           P(("g", conv.id)), conv.numel, 0, None)))
            out.append(("k", lib.monet_conv_wgrad, (v, C.byref(d), P(("in", conv.deps[0])), P(("g", conv.id)),
                                                    self.gview[(conv.id, "weight")].data_ptr(), 0, ws,
                                                    s.workspace, None), d))
        elif op.kind == "convT":
            d = net.conv_desc(op)
            v = _native.CONV_VARIANTS[s.impl]
            j = op.deps[0]
            dxp = P(("g", j)) if net.grad_bytes(net.op(j)) > 0 else None
            out.append(("k", lib.monet_convT_bwd, (v, C.byref(d), P(("in", j)), self.pview[(op.id, "weight")].data_ptr(),
                                                   dy, dxp, acc(j) if dxp else 0,
                                                   self.gview[(op.id, "weight")].data_ptr(), ws, s.workspace, None), d))
            if "bias" in op.params:
                out.append(("k", lib.monet_bias_grad, (dy, self.gview[(op.id, "bias")].data_ptr(),
                                                       op.numel // op.shape[-1], op.shape[-1], 0, self.scratch_ptr,
                                                       None)))
        elif op.kind == "concat":
            pix, ct, off = op.numel // op.shape[3], op.shape[3], 0
            for j in op.attrs["inputs"]:
                cj = net.op(j).shape[3]
                if net.grad_bytes(net.op(j)) > 0:
                    out.append(("k", lib.monet_channel_copy, (dy, ct, off, P(("g", j)), cj, 0, cj, pix, acc(j), None)))
                off += cj
        elif op.kind == "dwconv":
            d = net.conv_desc(op)
            j = op.deps[0]
            wt = self.pview[(op.id, "weight")].data_ptr()
            if net.grad_bytes(net.op(j)) > 0:
                out.append(("k", lib.monet_dwconv_dgrad, (C.byref(d), dy, wt, P(("g", j)), acc(j), None), d))
            out.append(("k", lib.monet_dwconv_wgrad, (C.byref(d), P(("in", j)), dy,
                                                      self.gview[(op.id, "weight")].data_ptr(), ws, s.workspace,
                                                      None), d))
        elif op.kind == "relu6":
            j = op.deps[0]
            if s.impl == "bwd-mask":
                src, fn = P(("in", net.intermediate_of[op.id])), lib.monet_relu_bwd_mask
            elif s.impl == "bwd-out":
                src, fn = P(("in", op.id)), lib.monet_relu6_bwd_out
            else:
                src, fn = P(("in", j)), lib.monet_relu6_bwd_in
            if needs(j):
                out.append(("k", fn, (src, dy, P(("g", j)), op.numel, acc(j), None)))
        elif op.kind == "dropout":
            j = op.deps[0]
            if needs(j):
                out.append(("k", lib.monet_dropout_bwd, (dy, P(("g", j)), op.numel, C.c_float(op.attrs["p"]),
                                                     self.seed_ptr, op.id, acc(j), None)))
        elif op.kind == "bn":
            c = op.shape[-1]
            rows = op.numel // c
            j = op.deps[0]
            sm, si, _, _ = (t.data_ptr() for t in self.bn[op.id])
            gma = self.pview[(op.id, "weight")].data_ptr()
            bta = self.pview[(op.id, "bias")].data_ptr()
            dg = self.gview[(op.id, "weight")].data_ptr()
            db = self.gview[(op.id, "bias")].data_ptr()
            if s.impl == "bwd-in":
                out.append(("k", lib.monet_bn_bwd_in, (P(("in", j)), dy, P(("g", j)), acc(j), gma, sm, si, dg, db,
                                                      rows, c, self.scratch_ptr, None)))
            else:
                out.append(("k", lib.monet_bn_bwd_out, (P(("in", op.id)), dy, P(("g", j)), acc(j), gma, bta, si,
                                                       dg, db, rows, c, self.scratch_ptr, None)))
        elif op.kind in ("bnrelu", "bnrelu6"):
            c = op.shape[-1]
            rows = op.numel // c
            j = op.deps[0]
            sm, si, _, _ = (t.data_ptr() for t in self.bn[op.id])
            out.append(("k", lib.monet_bnrelu6_bwd if op.kind == "bnrelu6" else lib.monet_bnrelu_bwd,
                        (P(("in", j)), dy, P(("g", j)), acc(j), self.pview[(op.id, "weight")].data_ptr(),
                         self.pview[(op.id, "bias")].data_ptr(), sm, si, self.gview[(op.id, "weight")].data_ptr(),
                         self.gview[(op.id, "bias")].data_ptr(), rows, c, self.scratch_ptr, None)))
        elif op.kind == "relu":
            j = op.deps[0]
            if s.impl == "bwd-mask":
                src, fn = P(("in", net.intermediate_of[op.id])), lib.monet_relu_bwd_mask
            elif s.impl == "bwd-out":
                src, fn = P(("in", op.id)), lib.monet_relu_bwd_out
            else:
                src, fn = P(("in", j)), lib.monet_relu_bwd_in
            if needs(j):
                out.append(("k", fn, (src, dy, P(("g", j)), op.numel, acc(j), None)))
        elif op.kind == "add":
            for j in op.deps:
                if not needs(j):
                    continue
                out.append(("k", lib.monet_grad_pass, (dy, P(("g", j)), op.numel, C.c_float(1.0), acc(j), None)))
        elif op.kind == "bnaddrelu":
            c = op.shape[-1]
            rows = op.numel // c
            jx, jk = op.attrs["x"], op.attrs["skip"]
            sm, si, _, _ = (t.data_ptr() for t in self.bn[op.id])
            from_out = s.impl == "bwd-out"
            gate = P(("in", op.id)) if from_out else P(("in", jk))
            out.append(("k", lib.monet_bnaddrelu_bwd,
                        (P(("in", jx)), gate, 1 if from_out else 0, dy, P(("g", jx)), acc(jx), P(("g", jk)), acc(jk),
                         self.pview[(op.id, "weight")].data_ptr(), self.pview[(op.id, "bias")].data_ptr(), sm, si,
                         self.gview[(op.id, "weight")].data_ptr(), self.gview[(op.id, "bias")].data_ptr(), rows, c,
                         self.scratch_ptr, None)))
        elif op.kind == "addrelu":
            j0, j1 = op.deps
            if s.impl == "bwd-out":
                out.append(("k", lib.monet_addrelu_bwd_out, (P(("in", op.id)), dy, P(("g", j0)), acc(j0),
                                                             P(("g", j1)), acc(j1), op.numel, None)))
            else:
                out.append(("k", lib.monet_addrelu_bwd_in, (P(("in", j0)), P(("in", j1)), dy, P(("g", j0)), acc(j0),
                                                            P(("g", j1)), acc(j1), op.numel, None)))
        elif op.kind == "maxpool":
            d = net.pool_desc(op)
            j = op.deps[0]
            if s.impl == "bwd-idx":
                args = (C.byref(d), P(("in", net.intermediate_of[op.id])), None, dy, P(("g", j)), acc(j), None)
            else:
                args = (C.byref(d), None, P(("in", j)), dy, P(("g", j)), acc(j), None)
            out.append(("k", lib.monet_maxpool_bwd, args, d))
        elif op.kind == "avgpool":
            j = op.deps[0]
            n, h, w, c = net.op(j).shape
            out.append(("k", lib.monet_avgpool_bwd, (dy, P(("g", j)), n, h * w, c, acc(j), None)))
        elif op.kind == "fc":
            j = op.deps[0]
            n, fi = net.fc_dims(op)
            fo = op.shape[1]
            v = 1 if s.impl == "gemm-splitk" else 0
            out.append(("k", lib.monet_linear_bwd,
                        (v, P(("in", j)), self.pview[(op.id, "weight")].data_ptr(), dy, P(("g", j)), acc(j),
                         self.gview[(op.id, "weight")].data_ptr(), self.gview[(op.id, "bias")].data_ptr(),
                         n, fi, fo, ws, s.workspace, None)))
        elif op.kind == "xent":
            j = op.deps[0]
            out.append(("k", lib.monet_xent_bwd, (P(("in", j)), self.labels.data_ptr(), dy, P(("g", j)),
                                                  net.label_count(), net.num_classes, acc(j), None)))
        else:
            raise ValueError(op.kind)
        return out

    def _bind_optimizer(self):
        calls = []
        if self.comm is not None:
            calls += self.comm.finish_calls()  # SGD waits for the bucket reductions
        calls.append(("k", self.lib.dll.monet_sgd_step,
                      (self.params.data_ptr(), self.grads.data_ptr(), self.mom.data_ptr(), self.params.numel(),
                       C.c_float(self.lr), C.c_float(self.momentum), C.c_float(self.weight_decay),
                       C.c_float(self.grad_scale), 0, None)))
        if any(op.kind == "dropout" for op in self.net.ops):
            calls.append(("k", self.lib.dll.monet_seed_advance, (self.seed_ptr, None)))
        return calls

    # ------------------------------------------------------------ running
    def run(self, plan: Plan, after_step=None):
        """Enqueue one training step (forward, scheduled backward, SGD) on the current stream.

        ``after_step(i)`` (debugging) is called after ledger step i is enqueued.
        """
        if plan.calls is None:
            raise RuntimeError("this plan was invalidated when the runtime's arena was reallocated; "
                               "call Runtime.plan() again")
        stream = torch.cuda.current_stream(self.device)
        sp = C.c_void_p(stream.cuda_stream)
        cudart = _cudart()
        for i, group in enumerate(plan.calls):
            self._run_group(group, sp, cudart)
            if after_step is not None and i < len(plan.calls) - 1:
                after_step(i)

    def _run_group(self, group, sp, cudart):
        for c in group:
            kind = c[0]
            if kind == "k":
                fn, args = c[1], c[2]
                rc = fn(*args[:-1], sp)
                if rc != 0:
                    raise _native.NativeError(f"{fn.__name__} failed with code {rc}")
            elif kind == "copy":
                rc = cudart.monet_copy_async(c[1], c[2], c[3], sp)
                if rc != 0:
                    raise _native.NativeError(f"monet_copy_async failed ({rc})")
            else:
                c[1]()


class _StepGraph:
    """A captured training step as two CUDA graphs: up to the last read of the staging
    buffer, then the rest; the event between them releases the staging buffer to a
    prefetch (Runtime.prefetch)."""

    def __init__(self, head, tail, staging_free):
        self.head, self.tail, self.staging_free = head, tail, staging_free

    def replay(self):
        self.head.replay()
        self.staging_free.record()
        self.tail.replay()


def lifetimes(steps, g: Graph):
    """Blocks [t_alloc, t_free) in half-step units and the blocks each step touches."""
    sizes_of = {u.id: u.nbytes for u in g.storables}
    live: dict[tuple, int] = {}
    blocks: list[list[int]] = []  # [size, t_alloc, t_free]
    per_step = []

    def new_block(size, t):
        blocks.append([size, t, None])
        return len(blocks) - 1

    def end(key, t):
        b = live.pop(key)
        blocks[b][2] = t

    for s_idx, s in enumerate(steps):
        t0, t1 = 2 * s_idx, 2 * s_idx + 1
        for key in s.drops:
            end(key, t0)
        touched = {}
        # inputs read by the step (resolved before allocations; in-place takes one over)
        if s.kind in ("forward", "recompute"):
            for j in g.deps(s.node):
                touched[("in", j)] = live[("a", j)]
        else:
            for d in s.variant.deps:
                touched[("in", d)] = live[("a", d)]
            for j in g.deps(s.node):
                if ("a", j) in live:
                    touched[("in", j)] = live[("a", j)]
            if s.node in g.backward_by_node and ("a", s.node) in live:
                touched[("in", s.node)] = live[("a", s.node)]
        for key in s.allocs:
            if key[0] == "a":
                if s.inplace_from is not None and key[1] == s.node:
                    b = live.pop(("a", s.inplace_from))
                    live[key] = b
                else:
                    live[key] = new_block(sizes_of[key[1]], t0)
            else:
                live[key] = new_block(g.grad_bytes(key[1]), t0)
            touched[key] = live[key]
        if s.kind == "backward":
            touched[("g", s.node)] = live[("g", s.node)]
            for j in g.deps(s.node):
                if ("g", j) in live:
                    touched[("g", j)] = live[("g", j)]
        if s.workspace:
            touched[("ws",)] = new_block(s.workspace, t0)
            blocks[touched[("ws",)]][2] = t1
        for key in s.frees:
            end(key, t1)
        per_step.append({"blocks": touched})
    for key in list(live):
        end(key, 2 * len(steps))
    return blocks, per_step

def place_blocks(blocks, capacity: int = 0):
    n = len(blocks)
    arr = lambda vals: (C.c_int64 * max(n, 1))(*vals)
    sizes = arr([b[0] for b in blocks])
    ta = arr([b[1] for b in blocks])
    tf = arr([b[2] for b in blocks])
    offs = (C.c_int64 * max(n, 1))()
    peak = C.c_int64(0)
    cap = capacity
    rc = _native.lib().dll.monet_arena_plan(n, C.cast(sizes, C.c_void_p), C.cast(ta, C.c_void_p),
                                       C.cast(tf, C.c_void_p), ARENA_ALIGN, cap, C.cast(offs, C.c_void_p),
                                       C.byref(peak))
    if rc == -12:
        raise BudgetExceeded(f"arena plan needs {peak.value} B, only {cap} B left under the budget")
    if rc:
        raise RuntimeError(f"arena planner failed ({rc})")
    return peak.value, list(offs)[:n]



def _cudart():
    """The copy entry point of the C ABI (monet_copy_async); kept as a callable
    object so ``_run_group`` does not look it up per launch."""
    return _native.lib().dll


def execute(schedule: Schedule, g: Graph, catalog: Catalog, *, runtime: Runtime,
            images: torch.Tensor | None = None, labels: torch.Tensor | None = None) -> ExecResult:
    """Run one scheduled training step on the GPU and return its ledger and measurements.

    Raises SimulationError for schedules the simulator rejects and
    BudgetExceeded when the planned footprint exceeds the runtime's budget.
    """
    if images is not None:
        runtime.set_batch(images, labels)
    plan = runtime.plan(schedule, g, catalog)
    torch.cuda.synchronize(runtime.device)
    torch.cuda.reset_peak_memory_stats(runtime.device)
    runtime.run(plan)
    torch.cuda.synchronize(runtime.device)
    return ExecResult(
        trace=plan.trace,
        loss=runtime.loss_value(),
        ledger_peak=plan.ledger_peak,
        physical_peak=runtime.params_bytes + plan.arena_bytes,
        bound_peak=plan.bound_peak,
        arena_bytes=plan.arena_bytes,
        params_bytes=runtime.params_bytes,
        torch_peak_bytes=torch.cuda.max_memory_allocated(runtime.device),
        launches=plan.launches,
    )

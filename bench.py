#!/usr/bin/env python
"""Benchmark: ResNet-50 (224x224, batch 184 per GPU) trained under a fixed
per-GPU memory budget with a MONeT schedule, on 1..8 B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--budget-gib 8]
    torchrun --nproc-per-node N bench.py --gpus N ...     (data parallel)
    python bench.py --impl reference ...                  (CPU oracle arm)

One JSON line (rank 0).  ``value``: training images/s over all ranks with the
batch resident in HBM; ``e2e``: the same through the public per-step call
(Runtime.train_step) with the batch copied from pinned host memory and the
loss read back every step.  ``roofline``: the dominant kernel (the tcgen05
implicit-GEMM convolution) timed live with CUDA events; ``cpu_baseline``: the
CPU oracle replay of the same kind of schedule on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "train imgs/s at fixed per-GPU memory budget"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--arch", default="resnet50")
    ap.add_argument("--batch", type=int, default=184)
    ap.add_argument("--image", default="224", help="224, or HxW (UNet: 416x608)")
    ap.add_argument("--budget-gib", type=float, default=8.0)
    ap.add_argument("--no-fuse", dest="fuse", action="store_false",
                    help="separate BN and ReLU operators (default: fused BN+ReLU ops, tracer fuse=True)")
    ap.add_argument("--ablation", default=None, choices=["none", "conv", "out", "int", "all"],
                    help="run the schedule planned with apply_ablation(catalog, mode) (schedules/*_abl-<mode>.json)")
    ap.add_argument("--split", action="store_true",
                    help="conv backward split into dgrad / wgrad graph nodes (tracer.split_conv_backward)")
    ap.add_argument("--no-graph", action="store_true", help="launch kernels from Python instead of a CUDA graph")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-overhead-run", action="store_true", help="skip timing the store-everything schedule")
    ap.add_argument("--cpu-sample", type=int, default=8, help="images per CPU baseline step")
    return ap.parse_args()


# --------------------------------------------------------------------------- helpers

def load_or_plan(net, g, cat, budget, arch, batch, image, gib, ablation=None):
    import hashlib

    import paper_2010_14501_b200 as M
    from paper_2010_14501_b200.planner import plan_schedule

    abl = f"_abl-{ablation}" if ablation else ""
    path = ROOT / "schedules" / f"{stem(arch, net)}_b{batch}_{image}_{gib:g}gib{abl}.json"
    digest = lambda d: hashlib.sha256(json.dumps(d, sort_keys=True).encode()).hexdigest()[:16]  # noqa: E731
    if path.exists():
        doc = json.loads(path.read_text())
        if doc["graph_digest"] == digest(net.graph_doc()):
            return M.schedule_from_doc(doc["schedule"]), doc.get("planner", {}), str(path.relative_to(ROOT))
    sched, info = plan_schedule(g, cat, budget, kinds=net.storable_kinds())
    if sched is None:
        raise SystemExit(f"no schedule fits {gib} GiB")
    return sched, info, "planned at startup"


def stem(arch, net=None, fused=None, split=None):
    """File-name stem of a workload: arch[_fused][_split] (schedules/, profiles/, oracle/specs/)."""
    fused = net.fused if net is not None else fused
    split = net.split if net is not None else split
    return f"{arch}{'_fused' if fused else ''}{'_split' if split else ''}"


def measured_catalog(net, args):
    """The frozen on-device profile (tools/profile_catalog.py) when it matches this graph."""
    import hashlib

    path = ROOT / "profiles" / f"catalog_{stem(args.arch, net)}_b{args.batch}_{args.image}.json"
    if not path.exists():
        return None
    doc = json.loads(path.read_text())
    dg = hashlib.sha256(json.dumps(net.graph_doc(), sort_keys=True).encode()).hexdigest()[:16]
    return doc["catalog"] if doc["graph_digest"] == dg else None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
        except OSError:
            rows = []
        rows = [[c.strip() for c in r] for r in rows if len(r) >= 7]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in rows for j in range(4) if r[3 + j].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())}


def conv_flops(net, op):
    x = net.op(op.deps[0])
    if op.kind == "convT":  # the adjoint conv's GEMM: input pixels x in-channels x out-channels x taps
        return 2.0 * x.numel * op.shape[3] * op.attrs["r"] * op.attrs["s"]
    return 2.0 * op.numel * x.shape[3] * op.attrs["r"] * op.attrs["s"]


def image_arg(v: str):
    from paper_2010_14501_b200.tracer import parse_image
    return parse_image(v)


def n_classes(arch: str) -> int:
    from paper_2010_14501_b200.tracer import default_classes
    return default_classes(arch)


LOCAL_BYTES = {  # minimal fp32 HBM bytes per element
    ("relu", "forward", True): 8.125, ("relu", "forward", False): 8.0, ("relu", "bwd-mask"): 8.125,
    ("relu", "bwd-in"): 12.0, ("relu", "bwd-out"): 12.0, ("bn", "train"): 12.0, ("bn", "replay"): 8.0,
    ("bn", "bwd"): 20.0, ("add", "forward"): 12.0, ("add", "bwd"): 16.0,
    ("bnrelu", "train"): 12.0, ("bnrelu", "replay"): 8.0, ("bnrelu", "bwd"): 20.0,
    ("bnrelu6", "train"): 12.0, ("bnrelu6", "replay"): 8.0, ("bnrelu6", "bwd"): 20.0,
    ("bnaddrelu", "train"): 16.0, ("bnaddrelu", "replay"): 12.0, ("bnaddrelu", "bwd"): 32.0,
    ("addrelu", "forward"): 12.0, ("addrelu", "bwd-out"): 16.0, ("addrelu", "bwd-in"): 20.0,
}


def kernel_roofline(rt, plan, net, peaks):
    """Time every ledger step's launches with CUDA events (one extra, untimed step)."""
    import ctypes as C

    import torch

    from paper_2010_14501_b200.engine import _cudart

    stream = torch.cuda.current_stream()
    sp = C.c_void_p(stream.cuda_stream)
    cudart = _cudart()
    evs = []
    for group in plan.calls:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        rt._run_group(group, sp, cudart)
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    conv_t = conv_f = 0.0
    local_t = local_b = 0.0
    total_t = 0.0
    n_conv = 0
    for (a, b), s in zip(evs, plan.steps):
        ms = a.elapsed_time(b)
        total_t += ms
        op = net.op(s.node)
        if op.kind in ("conv", "convrelu", "convT", "wgrad"):
            if op.kind == "wgrad":  # a split conv's weight gradient (no forward work)
                f = conv_flops(net, net.op(op.attrs["conv"])) if s.kind == "backward" else 0.0
            else:
                f = conv_flops(net, op)
            if s.kind == "backward" and op.kind != "wgrad":
                # dgrad (unless the input has no gradient) + wgrad, or dgrad alone when split
                dg = 0 if net.op(op.deps[0]).kind == "input" else 1
                f *= dg + (0 if op.attrs.get("split") else 1)
            conv_t += ms
            conv_f += f
            n_conv += 1
        elif op.kind in ("relu", "bn", "bnrelu", "bnrelu6", "bnaddrelu", "add", "addrelu"):
            if s.kind == "backward":
                key = (op.kind, s.impl) if op.kind in ("relu", "addrelu") else (op.kind, "bwd")
            elif op.kind in ("bn", "bnrelu", "bnrelu6", "bnaddrelu"):
                key = (op.kind, "train" if s.kind == "forward" else "replay")
            elif op.kind == "relu":
                key = ("relu", "forward", net.intermediate_of[op.id] in s.planned_ints)
            else:
                key = (op.kind, "forward")
            local_t += ms
            local_b += LOCAL_BYTES[key] * op.numel
    opt = evs[-1]
    total_t += opt[0].elapsed_time(opt[1])
    bf16_peak = peaks.get("bf16_tflops_sustained", 1400.0)
    achieved = conv_f / (conv_t * 1e-3) / 1e12
    roof = {"bound": "tensor", "kernel": "gemm_bf16x3_kernel (implicit-GEMM conv, bf16x3 split, A in TMEM, TMA)",
            "achieved": round(achieved, 1), "peak": round(bf16_peak, 1), "unit": "TFLOP/s",
            "frac": round(achieved / bf16_peak, 4),
            "peak_basis": "measured dense bf16 bf16_tflops_sustained (MEASURED_PEAKS.json)",
            "flops_per_step": conv_f, "conv_ms_per_step": round(conv_t, 3), "conv_share_of_step": round(conv_t / total_t, 3),
            "conv_launch_groups": n_conv,
            "note": "fp32 operands are split into bf16 hi+lo and each useful MMA issues 3 bf16 MMAs, so the ceiling "
                    "for algorithmic flops is peak/3; achieved counts algorithmic 2*N*K*P*Q*C*R*S flops (fwd, dgrad, "
                    "wgrad and recomputed forwards) only"}
    hbm = peaks.get("hbm_gbs", 6452.5)
    local = {"bound": "hbm", "achieved": round(local_b / (local_t * 1e-3) / 1e9, 1), "peak": hbm, "unit": "GB/s",
             "frac": round(local_b / (local_t * 1e-3) / 1e9 / hbm, 4), "ms_per_step": round(local_t, 3),
             "share_of_step": round(local_t / total_t, 3), "kernels": "relu/bn/add (SURVEY §8d algorithmic bytes)"}
    return roof, local, total_t


def _spec_and_schedule(args):
    """The frozen network (oracle/specs) and the committed schedule of this workload:
    plain JSON, so the CPU arms never import the product package or map its .so."""
    from oracle import netspec

    # architectures without BN+ReLU pairs (VGG-16) trace to the same graph with or without fusion
    fused = args.fuse and netspec.spec_path(args.arch, True, args.batch, args.image, args.split).exists()
    spec = netspec.spec_path(args.arch, fused, args.batch, args.image, args.split)
    name = stem(args.arch, fused=fused, split=args.split)
    sched = ROOT / "schedules" / f"{name}_b{args.batch}_{args.image}_{args.budget_gib:g}gib.json"
    cat = ROOT / "profiles" / f"catalog_{name}_b{args.batch}_{args.image}.json"
    missing = [str(p.relative_to(ROOT)) for p in (spec, sched, cat) if not p.exists()]
    if missing:
        raise FileNotFoundError(f"frozen inputs missing: {missing} (tools/freeze_netspec.py, tools/make_schedules.py)")
    sdoc = json.loads(sched.read_text())
    spec_doc = json.loads(spec.read_text())
    if sdoc["graph_digest"] != spec_doc["graph_digest"]:
        raise ValueError(f"{sched.name} was planned for another graph than {spec.name}")
    return spec, sdoc, json.loads(cat.read_text())["catalog"], sched


def cpu_baseline_run(args, steps=2, warmup=1):
    """The CPU oracle port (oracle/cpu_executor.py) replaying the committed schedule on the
    same workload (network, batch, budget) with all host threads; no product code."""
    import torch

    from oracle import netspec
    from oracle.cpu_executor import CpuState, run_step

    torch.set_num_threads(os.cpu_count() or 1)
    spec, sdoc, _, sched_path = _spec_and_schedule(args)
    net = netspec.load(spec)
    n = net.batch
    gen = torch.Generator().manual_seed(0)
    hw = _hw(args.image)
    x = torch.randn(n, 3, *hw, generator=gen)
    y = torch.randint(0, net.num_classes, (net.label_count(),), generator=gen)
    st = CpuState(net)
    for _ in range(warmup):
        run_step(st, sdoc["schedule"], x, y)
    t = time.perf_counter()
    for _ in range(steps):
        loss = run_step(st, sdoc["schedule"], x, y)
    dt = (time.perf_counter() - t) / steps
    return {"value": round(n / dt, 3), "unit": "img/s", "cores": torch.get_num_threads(), "kind": "port",
            "schedule": str(sched_path.relative_to(ROOT)),
            "sample": f"{args.arch} batch {n} at {hw[0]}x{hw[1]}: one training step replaying the committed "
                      f"{args.budget_gib:g} GiB schedule ({sched_path.relative_to(ROOT)}) with the torch-CPU fp32 "
                      f"oracle port, mean of {steps} step(s) after {warmup} warm-up; synthetic seeded weights "
                      f"(oracle/netspec.py)", "loss": round(float(loss), 4)}


def reference_planner_run(args, node_limit=1):
    """The reference's own CPU path for this workload, unmodified (remsched 0.1.0 from
    baseline/_ref): load the graph/catalog/schedule documents, build the 0-1 ILP at the
    budget (ilp.py:121), run its branch-and-bound with the committed schedule as the
    incumbent and a node limit (solver.py:441, cli.py:129), decode, validate, simulate
    (schedule.py:320) and compute the ILP bound (oracle.py:287).  Wall time per phase."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "remsched").exists():
        return {"unavailable": "baseline/_ref/remsched not installed"}
    sys.path.insert(0, str(ref))
    import remsched as R

    spec, sdoc, cat_doc, _ = _spec_and_schedule(args)
    graph_doc = json.loads(spec.read_text())["graph"]
    out = {"impl": f"remsched {getattr(R, '__version__', '0.1.0')} (baseline/_ref, unmodified)", "cores": 1}
    t0 = time.perf_counter()
    g = R.load_graph(graph_doc)
    cat = R.load_catalog(cat_doc, g)
    sched = R.schedule_from_doc(sdoc["schedule"])
    sets = R.compute_dependency_sets(g)
    t1 = time.perf_counter()
    model = R.build_model(g, sets, cat, sdoc["budget_bytes"], {"inplace": True})
    t2 = time.perf_counter()
    res = R.solve(model, {"node_limit": node_limit, "incumbent": R.assignment_from_schedule(model, sched)})
    t3 = time.perf_counter()
    dec = R.decode(res, g, cat) if res.assignment is not None else sched
    tags = R.validate(dec, g, sets, cat)
    tr = R.simulate(dec, g, cat)
    t4 = time.perf_counter()
    ok, bound, _ = R.check_schedule(g, sets, cat, dec, sdoc["budget_bytes"])
    t5 = time.perf_counter()
    out.update({"load_s": round(t1 - t0, 3), "build_model_s": round(t2 - t1, 3), "solve_s": round(t3 - t2, 3),
                "validate_simulate_s": round(t4 - t3, 3), "check_schedule_s": round(t5 - t4, 3),
                "total_s": round(t5 - t0, 3), "node_limit": node_limit, "status": res.status,
                "nodes": res.nodes, "objective": None if res.objective is None else str(res.objective),
                "lower_bound": None if res.lower_bound is None else str(res.lower_bound),
                "validate_tags": len(tags), "simulated_peak_bytes": tr.peak_memory, "ilp_bound_bytes": bound,
                "within_budget": bool(ok)})
    return out


def _hw(image):
    if "x" in str(image):
        h, w = str(image).split("x")
        return int(h), int(w)
    return int(image), int(image)


# --------------------------------------------------------------------------- arms

def reference_arm(args):
    """The reference-side CPU path on the same workload as ours_arm (no product code: the
    network, catalog and schedule are the committed JSON files).  ``value``: the oracle
    port replaying the committed schedule at the full batch on all host threads;
    ``reference_planner``: the reference's own remsched path for the same instance."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    steps = max(1, min(args.steps, 2))
    res = cpu_baseline_run(args, steps=steps, warmup=1)
    planner = reference_planner_run(args)
    hw = _hw(args.image)
    out = {"impl": "reference", "metric": METRIC, "value": res["value"], "unit": "img/s", "n_gpus": args.gpus,
           "steps": steps, "warmup": 1, "ms_per_step": round(1e3 * args.batch / res["value"], 1),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
           "data": "synthetic N(0,1) images, uniform labels; seeded synthetic weights",
           "config": {"workload": f"{args.arch} {hw[0]}x{hw[1]} batch {args.batch}/GPU, {args.budget_gib:g} GiB "
                                  f"per-GPU budget, MONeT schedule ({res['schedule']})"
                                  + (", fused BN+ReLU operators" if "_fused" in res["schedule"] else "")
                                  + (", conv backward split" if args.split else ""),
                      "model": args.arch, "global_batch": args.batch, "per_gpu_batch": args.batch,
                      "image": args.image, "budget_bytes": int(args.budget_gib * (1 << 30)),
                      "parallelism": "host cores"},
           "cpu_baseline": res, "reference_planner": planner,
           # this arm runs only oracle/ + the reference package: the product must not be loaded
           "product_loaded": "paper_2010_14501_b200" in sys.modules,
           "e2e": {"value": res["value"], "unit": "img/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def ours_arm(args):
    import torch
    import torch.distributed as dist

    import paper_2010_14501_b200 as M
    from paper_2010_14501_b200.engine import Runtime
    from paper_2010_14501_b200.tracer import build_network

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    peaks = {}
    pk = ROOT / "MEASURED_PEAKS.json"
    if pk.exists():
        peaks = json.loads(pk.read_text())

    gib = args.budget_gib
    budget = int(gib * (1 << 30))
    net = build_network(args.arch, args.batch, image_arg(args.image), num_classes=n_classes(args.arch), fuse=args.fuse,
                        split=args.split)
    gdoc = net.graph_doc()
    g = M.load_graph(gdoc)
    cat = M.load_catalog(measured_catalog(net, args) or net.catalog_doc(), g)
    from paper_2010_14501_b200.schedule import fastest_store_everything_schedule
    se = fastest_store_everything_schedule(g, cat)  # min-cost no-recompute
    cat_full = cat
    if args.ablation:  # the schedule is planned with one ablation family; the baseline stays the same
        cat = M.apply_ablation(cat, g, args.ablation)
    sched, pinfo, source = load_or_plan(net, g, cat, budget, args.arch, args.batch, args.image, gib, args.ablation)

    # SGD lr 0.1 (momentum 0.9) as in the paper's ResNet runs; VGG-16 has no BN and
    # diverges at 0.1 from torchvision's init (loss NaN within a few steps), so it
    # trains at torchvision's reference lr 0.01
    lr = 0.01 if args.arch.startswith("vgg") else 0.1
    rt = Runtime(net, device=dev, budget_bytes=budget, lr=lr)
    dp = None
    if world > 1:
        from paper_2010_14501_b200.dp import DataParallel
        dp = DataParallel(rt)
    plan = rt.plan(sched, g, cat)

    hw = image_arg(args.image)
    hw = hw if isinstance(hw, tuple) else (hw, hw)

    def batch():  # the synthetic batch (regenerated for the store-everything run, never kept)
        gen = torch.Generator(device=dev).manual_seed(1234 + rank)
        x = torch.randn(args.batch, 3, *hw, device=dev, generator=gen)
        y = torch.randint(0, n_classes(args.arch), (net.label_count(),), device=dev, generator=gen)
        return x, y

    x, y = batch()
    rt.set_batch(x, y)
    torch.cuda.synchronize()
    del x, y  # staged in the fixed region: nothing outside the runtime stays allocated
    torch.cuda.empty_cache()

    graph = None
    # N > 1: the native communicator's bucket all-reduces are stream operations, so the
    # data-parallel step is captured whole as well
    use_graph = not args.no_graph and (world == 1 or getattr(rt.comm, "capturable", False))
    if use_graph:
        graph = rt.capture(plan)

    def step():
        if graph is not None:
            graph.replay()
        else:
            rt.run(plan)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats(dev)
    free0, total0 = torch.cuda.mem_get_info(dev)
    # device memory the allocator holds for anything but the runtime (fixed region + arena)
    other0 = torch.cuda.memory_stats(dev).get("requested_bytes.all.current", 0) - rt.fixed.numel() - rt.arena.numel()

    sampler = ClockSampler(local)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with sampler:
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    mstats = torch.cuda.memory_stats(dev)  # before anything else is allocated
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = world * args.batch / (ms * 1e-3)
    loss = rt.loss_value()
    free1, _ = torch.cuda.mem_get_info(dev)
    device_mem = {
        # what the process asked the allocator for at its peak during the timed steps
        "torch_peak_requested_bytes": mstats.get("requested_bytes.all.peak"),
        "torch_peak_allocated_bytes": mstats.get("allocated_bytes.all.peak"),  # + 512-B allocator rounding
        "torch_reserved_bytes": mstats.get("reserved_bytes.all.current"),
        # allocations outside the runtime alive during the timed steps (bench bookkeeping)
        "other_allocated_bytes": other0,
        # the runtime's own peak: requested peak minus those
        "runtime_peak_bytes": (mstats.get("requested_bytes.all.peak") or 0) - other0,
        # CUDA context, NCCL buffers, cuBLAS/library workspaces: device memory in use that
        # torch's allocator does not hold
        "non_allocator_bytes": (total0 - min(free0, free1)) - mstats.get("reserved_bytes.all.current", 0),
    }

    # ---- end to end: pinned host batch in, loss out, through Runtime.train_step
    c_pad = net.ops[0].shape[3]
    host = torch.zeros(args.batch, hw[0], hw[1], c_pad, pin_memory=True)
    host[..., :3].normal_()
    host_y = torch.randint(0, n_classes(args.arch), (net.label_count(),), dtype=torch.int32).pin_memory()
    loss_host = torch.empty(1, pin_memory=True)
    for _ in range(2):
        rt.train_step(plan, host, host_y)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    # every step's batch is copied from pinned host memory inside the timed region; the copy of
    # batch i+1 is prefetched while step i runs (Runtime.prefetch: it starts once step i has
    # read the staging buffer), and step i's loss is read back before step i+1 is launched
    rt.prefetch(host, host_y)
    for i in range(args.steps):
        lt = rt.train_step(plan)
        if i + 1 < args.steps:
            rt.prefetch(host, host_y)
        loss_host.copy_(lt, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    b.record()
    torch.cuda.synchronize()
    e2e_ms = a.elapsed_time(b) / args.steps
    t = torch.tensor([e2e_ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item())

    # ---- roofline of the dominant kernel (one extra instrumented step)
    roof, local_roof, instr_ms = kernel_roofline(rt, plan, net, peaks)

    # ---- overhead vs the no-recompute schedule on the same kernels (analytic costs)
    overhead_model = float(plan.trace.total_cost / M.simulate(se, g, cat_full).total_cost - 1)

    # ---- measured overhead: the store-everything schedule (no budget, no
    # recompute, same kernels and variants' defaults) timed the same way
    se_ms = None
    if not args.no_overhead_run:
        del graph
        rt_se = Runtime(net, device=dev)
        plan_se = rt_se.plan(se, g, cat_full)
        xs, ys = batch()
        rt_se.set_batch(xs, ys)
        del xs, ys
        g_se = rt_se.capture(plan_se) if use_graph else None
        run_se = (lambda: g_se.replay()) if g_se is not None else (lambda: rt_se.run(plan_se))
        for _ in range(max(3, args.warmup)):
            run_se()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            run_se()
        b.record()
        torch.cuda.synchronize()
        se_ms = a.elapsed_time(b) / args.steps
        del g_se, rt_se, plan_se
        torch.cuda.empty_cache()

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline:
            try:
                cpu = cpu_baseline_run(args, steps=1, warmup=0)
            except Exception as exc:  # keep the GPU line even if the host run fails
                cpu = {"value": None, "error": str(exc)[:200]}
        n_rec = sum(sum(1 for u, impl in s.recompute if impl is not None) for s in sched.stages)
        out = {
            "metric": METRIC, "value": round(value, 2), "unit": "img/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": round(ms, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 (convs: bf16x3-split tensor-core MMAs, fp32 accumulate)",
            "data": "synthetic N(0,1) images, uniform labels; random-init torchvision weights (seed 0)",
            "config": {"workload": f"{args.arch} {hw[0]}x{hw[1]} batch {args.batch}/GPU, "
                                   f"{gib:g} GiB per-GPU budget, MONeT schedule ({source})"
                                   + (", fused BN+ReLU operators" if net.fused else "")
                                   + (", conv backward split" if net.split else ""),
                       "model": args.arch, "global_batch": world * args.batch, "per_gpu_batch": args.batch,
                       "image": args.image, "budget_bytes": budget, "parallelism": f"dp{world}",
                       "cuda_graph": use_graph, "ablation": args.ablation or "all",
                       "l2": "inputs larger than L2 (activations ~26 GB per step); no explicit flush"},
            "memory": {"ledger_peak_bytes": plan.ledger_peak, "ilp_bound_bytes": plan.bound_peak,
                       "physical_peak_bytes": g.params_bytes + plan.arena_bytes,
                       "params_bytes": g.params_bytes, "arena_bytes": plan.arena_bytes,
                       **device_mem,
                       "within_bound": g.params_bytes + plan.arena_bytes <= (plan.bound_peak or 0),
                       "device_within_bound": device_mem["runtime_peak_bytes"] <= (plan.bound_peak or 0),
                       "store_everything_ledger_peak_bytes": M.simulate(se, g, cat_full).peak_memory},
            "overhead": {"modeled_pct": round(100 * overhead_model, 2), "recomputes": n_rec,
                         "measured_pct": None if se_ms is None else round(100 * (ms / se_ms - 1), 2),
                         "unconstrained_ms_per_step": None if se_ms is None else round(se_ms, 3),
                         "unconstrained": "store-everything schedule with the cheapest variant per op (min-cost no-recompute), no budget, "
                                          "same kernels, same batch, timed like value",
                         "catalog": "measured (profiles/catalog_*.json)" if measured_catalog(net, args) else
                                    "analytic (costs.py)",
                         "planner": pinfo},
            "e2e": {"value": round(world * args.batch / (e2e_ms * 1e-3), 2), "unit": "img/s",
                    "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": host.numel() * 4 + args.batch * 4,
                    "d2h_bytes_per_step": 4, "api": "Runtime.prefetch(pinned host batch i+1) overlapping Runtime.train_step(plan) of batch i + loss D2H"},
            "gpu_launches": plan.launches * args.steps,
            "roofline": roof, "roofline_local_ops": local_roof,
            "cpu_baseline": cpu,
            "clocks": sampler.summary(), "loss": loss, "lr": lr,
            # a diverged run is not a valid measurement of a training step
            "loss_finite": math.isfinite(loss),
        }
        tr = ROOT / "profiles" / "traffic.json"
        if tr.exists():
            roof["traffic"] = json.loads(tr.read_text()).get("gemm_bytes_per_launch")
        else:
            roof["traffic"] = None
        print(json.dumps(out), flush=True)
        if not math.isfinite(loss):
            print(f"bench: loss is {loss} after {args.warmup + args.steps + 2} steps -- invalid run", file=sys.stderr)
    if world > 1:
        del graph
        dp.close()
        dist.destroy_process_group()
    if not math.isfinite(loss):
        sys.exit(3)


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
    else:
        ours_arm(args)


if __name__ == "__main__":
    main()

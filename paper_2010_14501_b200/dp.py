"""Batch-sharded data parallelism.

One process per GPU; every rank replays the SAME schedule on its own shard of
the global batch (per-GPU batch statistics, not SyncBN), under the same
per-GPU budget.  The only exchange is the gradient all-reduce: parameter
gradients live in one contiguous fp32 buffer of the fixed region, so the
all-reduce is issued over that buffer in a fixed number of buckets in
stage order (NCCL over NVLink/NVSwitch on the compute stream), and the
1/world averaging is folded into the SGD kernel's ``grad_scale``.

The buffers NCCL allocates internally live outside the budgeted arena and are
reported separately by the bench.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

__all__ = ["DataParallel", "bucket_ranges"]


def bucket_ranges(n_elems: int, n_buckets: int):
    step = (n_elems + n_buckets - 1) // n_buckets
    return [(s, min(n_elems, s + step)) for s in range(0, n_elems, step)]


class DataParallel:
    def __init__(self, runtime, group=None, buckets: int = 4):
        self.rt = runtime
        self.group = group
        self.world = dist.get_world_size(group)
        runtime.grad_scale = 1.0 / self.world
        runtime.comm = self
        # gradients are laid out in node order; stage order is descending, so the
        # last bucket (deepest layers) completes first
        self.ranges = bucket_ranges(runtime.grads.numel(), buckets)[::-1]

    def allreduce_grads(self):
        for a, b in self.ranges:
            dist.all_reduce(self.rt.grads[a:b], op=dist.ReduceOp.SUM, group=self.group)

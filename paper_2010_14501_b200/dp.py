"""Batch-sharded data parallelism.

One process per GPU; every rank replays the SAME schedule on its own shard of
the global batch (per-GPU batch statistics, not SyncBN) under the same
per-GPU budget.  The only exchange is the gradient all-reduce:

* parameter gradients live in one contiguous fp32 buffer of the fixed
  region, laid out in node order, so a bucket is a contiguous slice;
* a parameter gradient is final once its node's backward stage has run and
  stages run in descending node order, so the bucket holding the highest
  nodes is complete first.  `plan_buckets` cuts the buffer into ~`bucket_bytes`
  slices along node boundaries and records, per bucket, the node whose
  backward completes it;
* the executor calls `bucket_ready(node)` right after enqueuing that node's
  backward kernels: the slice's all-reduce is launched asynchronously (NCCL
  over NVLink / NVSwitch on its own stream, ordered after the producing
  kernels), so it overlaps the remaining backward stages;
* `finish()` (enqueued before SGD) waits for the outstanding reductions; the
  1/world average is folded into the SGD kernel's ``grad_scale``.

Two backends issue the bucket all-reduces:

* ``native`` (default on CUDA with an NCCL process group): the library's own
  communicator (include/monet_b200.h, csrc/comm.cu).  `monet_allreduce_bucket`
  forks the bucket's NCCL all-reduce onto a comm stream after the producing
  kernels and `monet_comm_join` joins it back before SGD -- plain stream
  operations in the plan's call list, so the whole data-parallel step is
  captured into one CUDA graph (no Python on the step's path);
* ``torch``: `torch.distributed.all_reduce(async_op=True)` from a Python call
  in the plan (any backend: gloo for the CPU and one-GPU multi-process tests);
  not graph-capturable.

NCCL's internal buffers live outside the budgeted arena and are reported
separately by the bench.
"""

from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist

__all__ = ["DataParallel", "plan_buckets", "bucket_ranges"]


def bucket_ranges(n_elems: int, n_buckets: int):
    """Equal contiguous slices (kept for callers that do not know the layout)."""
    step = (n_elems + n_buckets - 1) // n_buckets
    return [(s, min(n_elems, s + step)) for s in range(0, n_elems, step)]


def plan_buckets(net, bucket_bytes: int = 25 << 20):
    """[(start, end, ready_node)] over the flat gradient buffer, highest nodes first.

    Slices follow node boundaries; ready_node is the smallest node id in the
    slice (its backward is the last of the slice to run)."""
    spans = []  # (node, start, end) of every node with parameters, in buffer order
    pos = 0
    for nid, _, t in net.param_items():
        if spans and spans[-1][0] == nid:
            spans[-1][2] = pos + t.numel()
        else:
            spans.append([nid, pos, pos + t.numel()])
        pos += t.numel()
    buckets = []
    cur = None
    for nid, a, b in reversed(spans):
        if cur is None:
            cur = [a, b, nid]
        else:
            cur[0], cur[2] = a, nid
        if (cur[1] - cur[0]) * 4 >= bucket_bytes:
            buckets.append(tuple(cur))
            cur = None
    if cur is not None:
        buckets.append(tuple(cur))
    return buckets


class DataParallel:
    def __init__(self, runtime, group=None, bucket_bytes: int = 25 << 20, backend: str = "auto"):
        self.rt = runtime
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if backend == "auto":
            on_cuda = isinstance(getattr(runtime, "grads", None), torch.Tensor) and runtime.grads.is_cuda
            backend = "native" if on_cuda and dist.get_backend(group) == "nccl" else "torch"
        if backend not in ("native", "torch"):
            raise ValueError(f"unknown DataParallel backend {backend!r}")
        self.backend = backend
        runtime.grad_scale = 1.0 / self.world
        runtime.comm = self
        self.buckets = plan_buckets(runtime.net, bucket_bytes)
        self.by_node: dict[int, list[tuple[int, int]]] = {}
        for a, b, node in self.buckets:
            self.by_node.setdefault(node, []).append((a, b))
        self.works = []
        self.handle = None
        if backend == "native":
            self._init_native()

    # ------------------------------------------------------------ native communicator
    def _init_native(self):
        from . import _native

        lib = _native.lib().dll
        uid = (C.c_char * lib.monet_comm_unique_id_bytes())()
        if self.rank == 0:
            rc = lib.monet_comm_unique_id(uid)
            if rc:
                raise _native.NativeError(f"monet_comm_unique_id failed ({rc})")
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=dist.get_global_rank(self.group, 0) if self.group else 0,
                                   group=self.group)
        uid = (C.c_char * len(box[0])).from_buffer_copy(box[0])
        h = C.c_void_p()
        rc = lib.monet_comm_init(uid, self.rank, self.world, C.byref(h))
        if rc:
            raise _native.NativeError(f"monet_comm_init failed ({rc})")
        self.handle = h
        self._lib = lib

    def close(self):
        if self.handle is not None:
            self._lib.monet_comm_destroy(self.handle)
            self.handle = None

    @property
    def capturable(self) -> bool:
        """The step's calls are all stream operations (CUDA-graph capturable)."""
        return self.backend == "native"

    def bucket_calls(self, node: int) -> list:
        """Plan entries that start the all-reduce of every bucket `node`'s backward completes."""
        if self.backend == "native":
            g = self.rt.grads
            return [("k", self._lib.monet_allreduce_bucket,
                     (self.handle, g.data_ptr() + 4 * a, b - a, None)) for a, b in self.by_node.get(node, ())]
        return [("py", lambda node=node: self.bucket_ready(node))]

    def finish_calls(self) -> list:
        """Plan entries that order the optimizer after every outstanding reduction."""
        if self.backend == "native":
            return [("k", self._lib.monet_comm_join, (self.handle, None))]
        return [("py", self.finish)]

    def ready_nodes(self):
        return set(self.by_node)

    def bucket_ready(self, node: int):
        """Launch the all-reduce of every bucket that `node`'s backward completes."""
        for a, b in self.by_node.get(node, ()):
            self.works.append(dist.all_reduce(self.rt.grads[a:b], op=dist.ReduceOp.SUM, group=self.group,
                                              async_op=True))

    def finish(self):
        """Order the optimizer after every outstanding reduction."""
        for w in self.works:
            w.wait()
        self.works.clear()

    def allreduce_grads(self):
        """Blocking all-reduce of the whole buffer (no overlap; kept for tools)."""
        for a, b, _ in self.buckets:
            dist.all_reduce(self.rt.grads[a:b], op=dist.ReduceOp.SUM, group=self.group)

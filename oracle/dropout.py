"""CPU restatement of the dropout keep-mask (test infrastructure only).

Mirrors csrc/local_ops.cuh dropout_keep / include/monet_b200.h: the keep
decision of element i (index in the engine's NHWC order) is a splitmix64
finalizer of (seed, salt, i); keep <=> top 24 bits >= floor(p * 2^24).
PyTorch's dropout semantics (y = x * keep / (1 - p), torch.nn.Dropout in
training mode) with a counter-based generator in place of torch's Philox
stream, so that the GPU and this oracle draw the identical mask.
"""
from __future__ import annotations

import numpy as np

_M = np.uint64(0xFFFFFFFFFFFFFFFF)


def keep_mask(n: int, p: float, seed: int, salt: int) -> np.ndarray:
    """Boolean keep-mask of n elements (NHWC element order)."""
    thr = np.uint64(int(float(np.float32(p)) * 16777216.0))
    with np.errstate(over="ignore"):
        i = np.arange(n, dtype=np.uint64)
        z = (np.uint64(seed) * np.uint64(0x9E3779B97F4A7C15)
             + np.uint64(salt) * np.uint64(0xD1B54A32D192ED03) + i)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(40)) >= thr

"""Packed ReLU sign bitmask, numpy restatement (test oracle).

Layout fixed by the engine: bit b of uint32 word w is
(element 32*w + b of the tensor in physical NHWC order) > 0; NaN and -0.0 give
0; unused tail bits are 0.  Size = ceil(numel/32) * 4 bytes, the graph's
intermediate size (tracer.mask_bytes).
"""
import numpy as np


def pack_sign_mask(x) -> np.ndarray:
    flat = np.asarray(x, dtype=np.float32).reshape(-1)
    bits = (flat > 0).astype(np.uint64)
    pad = (-len(bits)) % 32
    if pad:
        bits = np.concatenate([bits, np.zeros(pad, np.uint64)])
    words = bits.reshape(-1, 32)
    weights = (np.uint64(1) << np.arange(32, dtype=np.uint64))
    return (words * weights).sum(axis=1).astype(np.uint32)


def unpack_sign_mask(words: np.ndarray, numel: int) -> np.ndarray:
    w = np.asarray(words, dtype=np.uint32).astype(np.uint64)
    bits = (w[:, None] >> np.arange(32, dtype=np.uint64)) & np.uint64(1)
    return bits.reshape(-1)[:numel].astype(bool)

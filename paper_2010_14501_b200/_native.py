"""ctypes binding of libmonet_b200.so (the C ABI in include/monet_b200.h).

The library is built in-tree (``build.py``).  There is no fallback: if the
shared object is missing or the device is not sm_100, every entry point raises
so a GPU run can never silently execute anything but the CUDA kernels.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libmonet_b200.so"

_vp, _i32, _i64, _f32, _sz = C.c_void_p, C.c_int, C.c_int64, C.c_float, C.c_size_t


class ConvDesc(C.Structure):
    _fields_ = [(name, C.c_int) for name in
                ("n", "h", "w", "c", "k", "r", "s", "p", "q", "stride_h", "stride_w", "pad_h", "pad_w")]


_PCONV = C.POINTER(ConvDesc)


class ProfDesc(C.Structure):
    """monet_prof_desc (include/monet_b200.h)."""
    _fields_ = [("op", C.c_int), ("pass_", C.c_int), ("conv", ConvDesc), ("conv_needs_dx", C.c_int),
                ("rows", C.c_int64), ("c", C.c_int), ("fused_stats", C.c_int)]


PROF_OP = {"conv": 0, "relu": 1, "bn": 2, "bnrelu": 3}
PROF_BWD = {"bwd-in": 0, "bwd-out": 1, "bwd-mask": 2}

# name -> (restype, argtypes)
SIGNATURES = {
    "monet_version": (C.c_char_p, []),
    "monet_device_check": (_i32, []),
    "monet_copy_async": (_i32, [_vp, _vp, _sz, _vp]),
    "monet_comm_unique_id_bytes": (_sz, []),
    "monet_comm_unique_id": (_i32, [_vp]),
    "monet_comm_init": (_i32, [_vp, _i32, _i32, C.POINTER(_vp)]),
    "monet_comm_destroy": (_i32, [_vp]),
    "monet_allreduce_bucket": (_i32, [_vp, _vp, _sz, _vp]),
    "monet_comm_join": (_i32, [_vp, _vp]),
    "monet_profile_variant": (_i32, [C.c_void_p, _i32, _i32, C.POINTER(_i64), C.POINTER(_sz), _vp]),
    "monet_conv_ws_bytes": (_sz, [_i32, _i32, _PCONV]),
    "monet_conv_fwd": (_i32, [_i32, _PCONV, _vp, _vp, _vp, _vp, _sz, _vp]),
    "monet_conv_dgrad": (_i32, [_i32, _PCONV, _vp, _vp, _vp, _i32, _vp, _sz, _vp]),
    "monet_conv_wgrad": (_i32, [_i32, _PCONV, _vp, _vp, _vp, _i32, _vp, _sz, _vp]),
    "monet_conv_fwd_bias": (_i32, [_i32, _PCONV, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "monet_bias_grad": (_i32, [_vp, _vp, _i64, _i32, _i32, _vp, _vp]),
    "monet_conv_fwd_w16": (_i32, [_i32, _PCONV, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "monet_conv_dgrad_w16": (_i32, [_i32, _PCONV, _vp, _vp, _vp, _vp, _vp, _i32, _vp, _sz, _vp]),
    "monet_split_bf16": (_i32, [_vp, _vp, _vp, _i64, _vp]),
    "monet_conv_stats_bytes": (_sz, [_PCONV]),
    "monet_conv_fwd_w16_stats": (_i32, [_i32, _PCONV, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "monet_bn_stats_finalize": (_i32, [_vp, _i64, _i32, _f32, _f32, _i32, _vp, _vp, _vp, _vp, _vp]),
    "monet_split_bf16_segments": (_i32, [_vp, _vp, _vp, _vp, _i32, _i64, _vp]),
    "monet_dropout_fwd": (_i32, [_vp, _vp, _i64, _f32, _vp, C.c_uint64, _vp]),
    "monet_dropout_bwd": (_i32, [_vp, _vp, _i64, _f32, _vp, C.c_uint64, _i32, _vp]),
    "monet_seed_advance": (_i32, [_vp, _vp]),
    "monet_convT_ws_bytes": (_sz, [_i32, _i32, _PCONV]),
    "monet_convT_fwd": (_i32, [_i32, _PCONV, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "monet_convT_bwd": (_i32, [_i32, _PCONV, _vp, _vp, _vp, _vp, _i32, _vp, _vp, _sz, _vp]),
    "monet_channel_copy": (_i32, [_vp, _i32, _i32, _vp, _i32, _i32, _i32, _i64, _i32, _vp]),
    "monet_dwconv_ws_bytes": (_sz, [_PCONV]),
    "monet_dwconv_fwd": (_i32, [_PCONV, _vp, _vp, _vp, _vp]),
    "monet_dwconv_dgrad": (_i32, [_PCONV, _vp, _vp, _vp, _i32, _vp]),
    "monet_dwconv_wgrad": (_i32, [_PCONV, _vp, _vp, _vp, _vp, _sz, _vp]),
    "monet_relu6_fwd": (_i32, [_vp, _vp, _vp, _i64, _vp]),
    "monet_relu6_bwd_out": (_i32, [_vp, _vp, _vp, _i64, _i32, _vp]),
    "monet_relu6_bwd_in": (_i32, [_vp, _vp, _vp, _i64, _i32, _vp]),
    "monet_linear_ws_bytes": (_sz, [_i32, _i32, _i32, _i32, _i32]),
    "monet_linear_fwd": (_i32, [_i32, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _vp, _sz, _vp]),
    "monet_linear_bwd": (_i32, [_i32, _vp, _vp, _vp, _vp, _i32, _vp, _vp, _i32, _i32, _i32, _vp, _sz, _vp]),
    "monet_relu_fwd": (_i32, [_vp, _vp, _vp, _i64, _vp]),
    "monet_relu_bwd_mask": (_i32, [_vp, _vp, _vp, _i64, _i32, _vp]),
    "monet_relu_bwd_out": (_i32, [_vp, _vp, _vp, _i64, _i32, _vp]),
    "monet_relu_bwd_in": (_i32, [_vp, _vp, _vp, _i64, _i32, _vp]),
    "monet_bn_scratch_bytes": (_sz, [_i64, _i32]),
    "monet_bn_fwd_train": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _f32, _f32, _i32, _vp,
                                  _vp]),
    "monet_bn_fwd_replay": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _vp]),
    "monet_bn_bwd_in": (_i32, [_vp, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _vp, _vp]),
    "monet_bn_bwd_out": (_i32, [_vp, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _vp, _vp]),
    "monet_bnrelu_fwd_train": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _f32, _f32, _i32, _vp,
                                      _vp]),
    "monet_bnrelu_fwd_replay": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _vp]),
    "monet_bnrelu_bwd": (_i32, [_vp, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _vp, _vp]),
    "monet_bnrelu6_fwd_train": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _f32, _f32, _i32, _vp,
                                       _vp]),
    "monet_bnrelu6_fwd_replay": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _vp]),
    "monet_bnrelu6_bwd": (_i32, [_vp, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _vp, _vp]),
    "monet_bnaddrelu_fwd_train": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _f32, _f32, _i32,
                                         _vp, _vp]),
    "monet_bnaddrelu_fwd_replay": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _vp]),
    "monet_bnaddrelu_bwd": (_i32, [_vp, _vp, _i32, _vp, _vp, _i32, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _i64,
                                   _i32, _vp, _vp]),
    "monet_add_fwd": (_i32, [_vp, _vp, _vp, _i64, _vp]),
    "monet_grad_pass": (_i32, [_vp, _vp, _i64, _f32, _i32, _vp]),
    "monet_addrelu_fwd": (_i32, [_vp, _vp, _vp, _i64, _vp]),
    "monet_addrelu_bwd_out": (_i32, [_vp, _vp, _vp, _i32, _vp, _i32, _i64, _vp]),
    "monet_addrelu_bwd_in": (_i32, [_vp, _vp, _vp, _vp, _i32, _vp, _i32, _i64, _vp]),
    "monet_maxpool_fwd": (_i32, [_PCONV, _vp, _vp, _vp, _vp]),
    "monet_maxpool_bwd": (_i32, [_PCONV, _vp, _vp, _vp, _vp, _i32, _vp]),
    "monet_avgpool_fwd": (_i32, [_vp, _vp, _i32, _i32, _i32, _vp]),
    "monet_avgpool_bwd": (_i32, [_vp, _vp, _i32, _i32, _i32, _i32, _vp]),
    "monet_xent_scratch_bytes": (_sz, [_i32]),
    "monet_xent_fwd": (_i32, [_vp, _vp, _vp, _i32, _i32, _vp, _vp]),
    "monet_xent_bwd": (_i32, [_vp, _vp, _vp, _vp, _i32, _i32, _i32, _vp]),
    "monet_sgd_step": (_i32, [_vp, _vp, _vp, _i64, _f32, _f32, _f32, _f32, _i32, _vp]),
    "monet_gemm": (_i32, [_i32, _vp, _i32, _i64, _vp, _i32, _i64, _vp, _i64, _i32, _i32, _i32, _i32, _vp, _sz,
                          _vp]),
    "monet_gemm_ws_bytes": (_sz, [_i32, _i32, _i32, _i32]),
    "monet_arena_plan": (_i32, [_i64, _vp, _vp, _vp, _i64, _i64, _vp, _vp]),
    # host ILP branch-and-bound (csrc/bnb.cpp)
    "monet_bnb_create": (_vp, [_i32, _i32] + [_vp] * 5 + [_i32, _vp, _vp, _i32, _vp, _vp, _i32, _i32, _i32] +
                         [_vp] * 4),
    "monet_bnb_set_surrogate": (_i32, [_vp, _i64, _i32] + [_vp] * 6 + [_i32] + [_vp] * 3),
    "monet_bnb_destroy": (None, [_vp]),
    "monet_bnb_propagate": (_i32, [_vp, _i32, _vp, _vp, _vp]),
    "monet_bnb_lower_bound": (_i32, [_vp, _i32, _vp, _vp, _i64, _vp]),
    "monet_bnb_solve": (_i32, [_vp, _vp, C.c_double, _vp, _i32, _vp, _i32, _vp, _vp, _vp, _vp]),
    "monet_bnb_best": (_i32, [_vp, _vp]),
    "monet_bnb_n_events": (_i32, [_vp]),
    "monet_bnb_event": (_i32, [_vp, _i32, _vp, _vp, _vp]),
}

CONV_VARIANTS = {"implicit": 0, "splitk": 1, "tf32": 2, "tf32x3": 3, "pair": 4}
PASS = {"fwd": 0, "dgrad": 1, "wgrad": 2, "bwd": 3}


class NativeError(RuntimeError):
    pass


class _Lib:
    def __init__(self, path: Path):
        if not path.exists():
            raise NativeError(f"{path.name} is not built; run `python -m paper_2010_14501_b200.build` "
                              f"(there is no CPU fallback)")
        self.path = path
        self.dll = C.CDLL(str(path))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(self.dll, name)
            fn.restype = res
            fn.argtypes = args

    def __getattr__(self, name):
        fn = getattr(self.dll, "monet_" + name)

        def call(*args):
            rc = fn(*args)
            if fn.restype is _i32 and rc != 0:
                raise NativeError(f"monet_{name} failed with code {rc}")
            return rc
        return call


_LIB: _Lib | None = None


def lib() -> _Lib:
    global _LIB
    if _LIB is None:
        _LIB = _Lib(LIB_PATH)
    return _LIB


_DBG: _Lib | None = None


def debug_lib() -> _Lib:
    """libmonet_b200_dbg.so (build.py --debug): the ABI plus the GEMM's operand-dump and
    wait-counter hooks, for tools/ only -- the product never loads it."""
    global _DBG
    if _DBG is None:
        from . import build
        _DBG = _Lib(build.build(debug=True))
        _DBG.dll.monet_debug_dump.restype = None
        _DBG.dll.monet_debug_dump.argtypes = [_vp, _vp]
        _DBG.dll.monet_debug_timers.restype = None
        _DBG.dll.monet_debug_timers.argtypes = [_vp]
    return _DBG


def conv_desc(n, h, w, c, k, r, s, stride=1, pad=0) -> ConvDesc:
    p = (h + 2 * pad - r) // stride + 1
    q = (w + 2 * pad - s) // stride + 1
    return ConvDesc(n, h, w, c, k, r, s, p, q, stride, stride, pad, pad)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()

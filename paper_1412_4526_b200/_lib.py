"""ctypes binding of libdenseprop_b200.so (the C ABI in include/denseprop_b200.h).

The library is the product's only compute path: if it cannot be loaded, or
no CUDA device is visible, calls raise -- there is no CPU fallback.  Status
codes map onto the reference's exception types: DP_ERR_ARG -> ValueError
(the reference wrappers raise ValueError on shape errors, forward.py:33-38,
backward.py:136-146), anything else -> RuntimeError.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
# DP_LIB_PATH: load another build of the library (A/B experiments on one box)
LIB_PATH = os.environ.get("DP_LIB_PATH") or os.path.join(PKG, "libdenseprop_b200.so")

DP_F32, DP_F64 = 0, 1
DP_IDENTITY, DP_TANH, DP_RELU, DP_TANH_FAST = 0, 1, 2, 3
DP_OK, DP_ERR_ARG, DP_ERR_CUDA, DP_ERR_UNSUPPORTED = 0, 1, 2, 3
NONLIN_CODE = {"identity": DP_IDENTITY, "tanh": DP_TANH, "relu": DP_RELU}
DP_POOL_MAX, DP_POOL_AVG = 0, 1  # enum dp_pool_kind
DP_FAST_INPUT_FP16_RANGE, DP_FAST_PACK_FWD = 1, 2  # enum dp_fast_flags
ABI_VERSION = 6

_vp, _i, _i64, _sz, _d = C.c_void_p, C.c_int, C.c_int64, C.c_size_t, C.c_double

# name -> (restype, argtypes); must match include/denseprop_b200.h
SIGNATURES = {
    "dp_last_error": (C.c_char_p, []),
    "dp_abi_version": (_i, []),
    "dp_device_count": (_i, []),
    "dp_host_conv_forward": (_i, [_i, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i]),
    "dp_host_conv_backward_data": (_i, [_i, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i]),
    "dp_host_conv_backward_kernel": (_i, [_i, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i]),
    "dp_host_maxpool_forward": (_i, [_i, _vp, _vp, _vp, _i, _i, _i, _i, _i]),
    "dp_host_maxpool_backward": (_i, [_i, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _i]),
    "dp_host_avgpool_forward": (_i, [_i, _vp, _vp, _i, _i, _i, _i, _i]),
    "dp_host_avgpool_backward": (_i, [_i, _vp, _vp, _i, _i, _i, _i, _i, _i, _i]),
    "dp_host_nonlin_forward": (_i, [_i, _vp, _vp, _i64, _i]),
    "dp_host_nonlin_backward": (_i, [_i, _vp, _vp, _vp, _i64, _i]),
    "dp_conv_forward": (_i, [_i, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _i, _i, _vp]),
    "dp_conv_backward_data": (_i, [_i, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _i, _vp, _i,
                                   _vp]),
    "dp_conv_fast_workspace": (_sz, [_i, _i, _i]),
    "dp_conv_forward_fast_workspace": (_sz, [_i] * 7),
    "dp_conv_backward_data_fast_workspace": (_sz, [_i] * 7),
    "dp_conv_fast_supported": (_i, [_i, _i, _i, _i]),
    "dp_conv_forward_fast": (_i, [_vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _i, _i, _vp, _sz,
                                  _vp]),
    "dp_conv_forward_fast_ex": (_i, [_vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _i, _i, _i,
                                     _vp, _sz, _vp]),
    "dp_conv_backward_data_fast": (_i, [_vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _i, _vp, _i,
                                        _vp, _sz, _vp]),
    "dp_debug_wgrad_trace": (_i, [_vp, _sz]),
    "dp_debug_conv_trace": (_i, [_vp, _sz]),
    "dp_debug_wgrad_plan": (_i, [_i] * 7 + [_vp, _i]),
    "dp_conv_backward_kernel_fast_supported": (_i, [_i, _i, _i, _i, _i, _i, _i]),
    "dp_conv_backward_kernel_fast_workspace": (_sz, [_i, _i, _i, _i, _i, _i, _i]),
    "dp_conv_backward_kernel_fast": (_i, [_vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _i, _vp,
                                          _sz, _vp]),
    "dp_conv_backward_kernel_fast_ex": (_i, [_vp, _sz, _vp, _i, _vp, _vp, _i, _i, _i, _i, _i,
                                             _i, _i, _vp, _sz, _vp]),
    "dp_maxpool_backward_pitched": (_i, [_i, _vp, _vp, _i, _vp, _i, _i, _i, _i, _i, _i, _i,
                                         _i, _i, _vp, _i, _vp]),
    "dp_conv_backward_kernel_fast_prepare": (_i, [_vp] + [_i] * 7 + [_vp, _sz, _vp]),
    "dp_conv_backward_kernel_fast_f16_workspace": (_sz, [_i] * 7),
    "dp_split_f16": (_i, [_vp, _vp, _vp, _vp, _vp, _i, _i64, _i, _i, _vp]),
    "dp_conv_backward_kernel_fast_f16_shift": (_i, [_i] * 7),
    "dp_maxpool_forward_split": (_i, [_vp, _vp, _vp] + [_i] * 7 + [_vp, _vp, _i, _vp]),
    "dp_conv_backward_kernel_fast_f16": (_i, [_vp, _sz, _vp, _vp, _vp, _vp, _sz, _i, _vp, _i,
                                              _vp, _vp] +
                                         [_i] * 7 + [_vp, _sz, _vp]),
    "dp_conv_backward_kernel_fast_staged": (_i, [_vp, _vp, _vp, _vp] + [_i] * 7 + [_vp, _sz, _vp]),
    "dp_conv_backward_kernel_workspace": (_sz, [_i, _i, _i, _i, _i, _i, _i, _i]),
    "dp_conv_backward_kernel": (_i, [_i, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _i, _vp,
                                     _sz, _vp]),
    "dp_maxpool_forward": (_i, [_i, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _i, _i, _vp]),
    "dp_maxpool_backward": (_i, [_i, _vp, _vp, _i, _vp, _i, _i, _i, _i, _i, _i, _i, _i, _vp,
                                 _i, _vp]),
    "dp_avgpool_forward": (_i, [_i, _vp, _vp, _i, _i, _i, _i, _i, _i, _i, _vp]),
    "dp_avgpool_backward": (_i, [_i, _vp, _vp, _i, _i, _i, _i, _i, _i, _i, _i, _vp, _i, _vp]),
    "dp_nonlin_forward": (_i, [_i, _vp, _vp, _i64, _i, _vp]),
    "dp_nonlin_backward": (_i, [_i, _vp, _vp, _vp, _i64, _i, _i, _vp]),
    "dp_mask_delta": (_i, [_i, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _vp]),
    "dp_pad": (_i, [_i, _vp, _vp, _i, _i, _i, _i, _i, _i, _i, _i, _vp]),
    "dp_crop": (_i, [_i, _vp, _vp, _i, _i, _i, _i, _i, _i, _i, _i, _vp]),
    "dp_patch_gather": (_i, [_i, _vp, _vp, _i, _i, _i, _i, _i, _i64, _i64, _vp]),
    "dp_softmax_xent_delta": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _vp]),
    "dp_sgd_update": (_i, [_i, _vp, _vp, _i64, _d, _vp]),
    "dp_pool_strided_forward": (_i, [_i, _i, _vp, _vp, _vp] + [_i] * 6 + [_vp]),
    "dp_pool_strided_backward": (_i, [_i, _i, _vp, _vp, _vp] + [_i] * 8 + [_vp]),
    "dp_subsample": (_i, [_i, _vp, _vp] + [_i] * 7 + [_vp]),
    "dp_zero_insert": (_i, [_i, _vp, _vp] + [_i] * 7 + [_vp]),
    "dp_patch_gather_pixels": (_i, [_i, _vp, _vp, _i, _i, _i, _i, _vp, _i64, _vp]),
}

_lock = threading.Lock()
_lib = None
_load_error: str | None = None


class KernelUnavailable(RuntimeError):
    """The CUDA library or a CUDA device is missing: the product refuses to run."""


def load():
    """Load and type the shared library (idempotent); raises KernelUnavailable."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            _load_error = (f"{LIB_PATH} is not built; run `python -m paper_1412_4526_b200.build`"
                           " (or __graft_entry__.build())")
            raise KernelUnavailable(_load_error)
        try:
            lib = C.CDLL(LIB_PATH)
        except OSError as exc:
            _load_error = f"cannot load {LIB_PATH}: {exc}"
            raise KernelUnavailable(_load_error) from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.dp_abi_version() != ABI_VERSION:
            raise KernelUnavailable("libdenseprop_b200.so ABI version mismatch; rebuild")
        _lib = lib
        return lib


def device_count() -> int:
    return load().dp_device_count()


def require_device():
    """Raise KernelUnavailable unless the library loads AND a CUDA device is visible."""
    n = device_count()
    if n < 1:
        raise KernelUnavailable("no CUDA device visible to libdenseprop_b200 "
                                "(the B200 path has no CPU fallback)")
    return load()


def last_error() -> str:
    msg = load().dp_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    if rc == DP_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == DP_ERR_ARG:
        raise ValueError(msg)
    raise RuntimeError(f"denseprop_b200 error {rc}: {msg}")


def dtype_code(dtype) -> int:
    import numpy as np
    dt = np.dtype(dtype)
    if dt == np.float32:
        return DP_F32
    if dt == np.float64:
        return DP_F64
    raise TypeError(f"expected float32/float64 feature map, got {dt}")

"""The "cuda" kernel backend: the reference boundary's 7 functions on the B200.

Drop-in for a `backend.kernels()` module (reference backend.py:25-48; function
contract _kernels.pyx:23-247 / _kernels_py.py:19-126): C-contiguous numpy
(C, H, W) float32/float64 in, fresh numpy arrays out, `threads` accepted and
ignored (results never depend on it, tests/test_backends.py:76-89).  Each call
goes through the host-pointer C ABI (dp_host_*, include/denseprop_b200.h):
H2D copy, one sm_100a kernel, D2H copy.  Two extra entry points,
`nonlin_forward` / `nonlin_backward`, move the reference's numpy
nonlinearities (forward.py:69-76, backward.py:172-182) onto the device too.

Numerics: conv_forward, conv_backward_data, both pools, relu are bit-identical
to the compiled reference backend; tanh is within 2 ulp of numpy; dw/db
agree to reduction-order rounding (SURVEY.md 8(c) parity contract).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


def _arr(a, dtype=None):
    if dtype is None:
        a = np.asarray(a)
        if a.dtype not in (np.float32, np.float64):
            raise TypeError(f"expected float32/float64 feature map, got {a.dtype}")
        return np.ascontiguousarray(a)
    return np.ascontiguousarray(a, dtype=dtype)


def _p(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


def _lib_checked():
    return _lib.require_device()


def _ext(k, d):
    return (int(k) - 1) * int(d) + 1


def conv_forward(x, w, b, dilation, threads=1):
    x = _arr(x)
    w, b = _arr(w, x.dtype), _arr(b, x.dtype)
    if x.ndim != 3 or w.ndim != 4 or b.ndim != 1:
        raise ValueError("conv_forward expects x (C,H,W), w (O,C,k,k), b (O,)")
    co, ci, l, l2 = w.shape
    if ci != x.shape[0] or l != l2 or b.shape[0] != co:
        raise ValueError(f"conv_forward: shapes x{x.shape} w{w.shape} b{b.shape} disagree")
    e = _ext(l, dilation)
    if x.shape[1] < e or x.shape[2] < e:
        raise ValueError(f"dilated conv: input {x.shape[1]}x{x.shape[2]} is smaller than the "
                         f"{e}x{e} dilated window")
    y = np.empty((co, x.shape[1] - e + 1, x.shape[2] - e + 1), dtype=x.dtype)
    lib = _lib_checked()
    _lib.check(lib.dp_host_conv_forward(_lib.dtype_code(x.dtype), _p(x), _p(w), _p(b), _p(y),
                                        ci, x.shape[1], x.shape[2], co, l, int(dilation)),
               "conv_forward")
    return y


def conv_backward_data(dy, w, dilation, threads=1):
    dy = _arr(dy)
    w = _arr(w, dy.dtype)
    co, ci, l, _ = w.shape
    if dy.ndim != 3 or dy.shape[0] != co:
        raise ValueError(f"conv_backward_data: delta {dy.shape} vs kernel {w.shape}")
    e = _ext(l, dilation)
    dx = np.empty((ci, dy.shape[1] + e - 1, dy.shape[2] + e - 1), dtype=dy.dtype)
    lib = _lib_checked()
    _lib.check(lib.dp_host_conv_backward_data(_lib.dtype_code(dy.dtype), _p(dy), _p(w), _p(dx),
                                              co, dy.shape[1], dy.shape[2], ci, l,
                                              int(dilation)), "conv_backward_data")
    return dx


def conv_backward_kernel(x, dy, kernel_size, dilation, threads=1):
    x = _arr(x)
    dy = _arr(dy, x.dtype)
    l = int(kernel_size)
    co = dy.shape[0]
    ci, hi, wi = x.shape
    e = _ext(l, dilation)
    if dy.shape[1] != hi - e + 1 or dy.shape[2] != wi - e + 1:
        raise ValueError(f"delta spatial dims {dy.shape[1:]} do not match the conv output for "
                         f"input {x.shape[1:]} (extent {e})")
    dw = np.empty((co, ci, l, l), dtype=x.dtype)
    db = np.empty(co, dtype=x.dtype)
    lib = _lib_checked()
    _lib.check(lib.dp_host_conv_backward_kernel(_lib.dtype_code(x.dtype), _p(x), _p(dy), _p(dw),
                                                _p(db), ci, hi, wi, co, l, int(dilation)),
               "conv_backward_kernel")
    return dw, db


def maxpool_forward(x, p, dilation, threads=1):
    x = _arr(x)
    e = _ext(p, dilation)
    c, h, w = x.shape
    if h < e or w < e:
        raise ValueError(f"dilated max pool: input {h}x{w} is smaller than the {e}x{e} "
                         "dilated window")
    y = np.empty((c, h - e + 1, w - e + 1), dtype=x.dtype)
    arg = np.empty(y.shape, dtype=np.int32)
    lib = _lib_checked()
    _lib.check(lib.dp_host_maxpool_forward(_lib.dtype_code(x.dtype), _p(x), _p(y), _p(arg), c,
                                           h, w, int(p), int(dilation)), "maxpool_forward")
    return y, arg


def maxpool_backward(dy, arg, p, dilation, hi, wi, threads=1):
    dy = _arr(dy)
    arg = _arr(arg, np.int32)
    if arg.shape != dy.shape:
        raise ValueError(f"delta shape {dy.shape} != argmax shape {arg.shape}")
    dx = np.empty((dy.shape[0], int(hi), int(wi)), dtype=dy.dtype)
    lib = _lib_checked()
    _lib.check(lib.dp_host_maxpool_backward(_lib.dtype_code(dy.dtype), _p(dy), _p(arg), _p(dx),
                                            dy.shape[0], dy.shape[1], dy.shape[2], int(p),
                                            int(dilation), int(hi), int(wi)), "maxpool_backward")
    return dx


def avgpool_forward(x, p, dilation, threads=1):
    x = _arr(x)
    e = _ext(p, dilation)
    c, h, w = x.shape
    if h < e or w < e:
        raise ValueError(f"dilated avg pool: input {h}x{w} is smaller than the {e}x{e} "
                         "dilated window")
    y = np.empty((c, h - e + 1, w - e + 1), dtype=x.dtype)
    lib = _lib_checked()
    _lib.check(lib.dp_host_avgpool_forward(_lib.dtype_code(x.dtype), _p(x), _p(y), c, h, w,
                                           int(p), int(dilation)), "avgpool_forward")
    return y


def avgpool_backward(dy, p, dilation, hi, wi, threads=1):
    dy = _arr(dy)
    dx = np.empty((dy.shape[0], int(hi), int(wi)), dtype=dy.dtype)
    lib = _lib_checked()
    _lib.check(lib.dp_host_avgpool_backward(_lib.dtype_code(dy.dtype), _p(dy), _p(dx),
                                            dy.shape[0], dy.shape[1], dy.shape[2], int(p),
                                            int(dilation), int(hi), int(wi)), "avgpool_backward")
    return dx


def nonlin_forward(x, kind):
    if kind not in _lib.NONLIN_CODE:
        raise ValueError(f"unknown nonlinearity {kind!r}")
    if kind == "identity":
        return x
    x = _arr(x)
    y = np.empty_like(x)
    lib = _lib_checked()
    _lib.check(lib.dp_host_nonlin_forward(_lib.dtype_code(x.dtype), _p(x), _p(y), x.size,
                                          _lib.NONLIN_CODE[kind]), "nonlin_forward")
    return y


def nonlin_backward(delta, x_in, kind):
    if kind not in _lib.NONLIN_CODE:
        raise ValueError(f"unknown nonlinearity {kind!r}")
    if np.shape(delta) != np.shape(x_in):
        raise ValueError(f"delta shape {np.shape(delta)} != input shape {np.shape(x_in)}")
    if kind == "identity":
        return delta
    delta = _arr(delta)
    x_in = _arr(x_in, delta.dtype)
    dx = np.empty_like(delta)
    lib = _lib_checked()
    _lib.check(lib.dp_host_nonlin_backward(_lib.dtype_code(delta.dtype), _p(delta), _p(x_in),
                                           _p(dx), delta.size, _lib.NONLIN_CODE[kind]),
               "nonlin_backward")
    return dx

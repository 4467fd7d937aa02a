"""ctypes wrapper exposing oracle/kernels.c as the 7-function boundary module.

Test infrastructure only (see oracle/__init__.py).  Same signatures as the
reference boundary (`backend.kernels()`, reference backend.py:47-48;
_kernels.pyx:23-247): numpy (C, H, W) in, fresh numpy arrays out.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "liboracle_kernels.so")
_lib = None


def build() -> str:
    """Compile kernels.c -> oracle/lib/liboracle_kernels.so (gcc, OpenMP, no FMA)."""
    os.makedirs(os.path.dirname(LIB_PATH), exist_ok=True)
    src = os.path.join(_HERE, "kernels.c")
    if os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= os.path.getmtime(src):
        return LIB_PATH
    cc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
    cmd = (f"{cc} -O3 -march=x86-64-v3 -ffp-contract=off -fopenmp -fPIC -shared "
           f"-o {LIB_PATH} {src}")
    if os.system(cmd) != 0:
        raise RuntimeError(f"oracle C build failed: {cmd}")
    return LIB_PATH


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = ctypes.CDLL(LIB_PATH)
    return _lib


def available() -> bool:
    try:
        _load()
        return True
    except OSError:
        return False


def _sfx(a):
    if a.dtype == np.float32:
        return "f32"
    if a.dtype == np.float64:
        return "f64"
    raise TypeError(f"expected float32/float64, got {a.dtype}")


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _call(name, a, *args):
    fn = getattr(_load(), f"ork_{name}_{_sfx(a)}")
    conv = []
    for v in args:
        if isinstance(v, np.ndarray):
            conv.append(_p(v))
        else:
            conv.append(ctypes.c_ssize_t(int(v)))
    # trailing int threads
    conv[-1] = ctypes.c_int(int(args[-1]))
    fn(*conv)


def _c(a, dt=None):
    return np.ascontiguousarray(a, dtype=dt if dt is not None else a.dtype)


def conv_forward(x, w, b, dilation, threads=1):
    x = _c(x)
    w, b = _c(w, x.dtype), _c(b, x.dtype)
    co, ci, l, _ = w.shape
    e = (l - 1) * dilation + 1
    y = np.empty((co, x.shape[1] - e + 1, x.shape[2] - e + 1), dtype=x.dtype)
    _call("conv_forward", x, x, w, b, y, ci, x.shape[1], x.shape[2], co, l, dilation, threads)
    return y


def conv_backward_data(dy, w, dilation, threads=1):
    dy = _c(dy)
    w = _c(w, dy.dtype)
    co, ci, l, _ = w.shape
    e = (l - 1) * dilation + 1
    dx = np.empty((ci, dy.shape[1] + e - 1, dy.shape[2] + e - 1), dtype=dy.dtype)
    _call("conv_backward_data", dy, dy, w, dx, co, dy.shape[1], dy.shape[2], ci, l,
          dilation, threads)
    return dx


def conv_backward_kernel(x, dy, kernel_size, dilation, threads=1):
    x, dy = _c(x), _c(dy)
    co, ho, wo = dy.shape
    ci = x.shape[0]
    l = int(kernel_size)
    dw = np.empty((co, ci, l, l), dtype=x.dtype)
    db = np.empty(co, dtype=x.dtype)
    _call("conv_backward_kernel", x, x, dy, dw, db, ci, x.shape[1], x.shape[2], co, ho, wo,
          l, dilation, threads)
    return dw, db


def maxpool_forward(x, p, dilation, threads=1):
    x = _c(x)
    e = (p - 1) * dilation + 1
    shp = (x.shape[0], x.shape[1] - e + 1, x.shape[2] - e + 1)
    y = np.empty(shp, dtype=x.dtype)
    arg = np.empty(shp, dtype=np.int32)
    _call("maxpool_forward", x, x, y, arg, x.shape[0], x.shape[1], x.shape[2], p, dilation,
          threads)
    return y, arg


def maxpool_backward(dy, arg, p, dilation, hi, wi, threads=1):
    dy = _c(dy)
    arg = _c(arg, np.int32)
    dx = np.empty((dy.shape[0], hi, wi), dtype=dy.dtype)
    _call("maxpool_backward", dy, dy, arg, dx, dy.shape[0], dy.shape[1], dy.shape[2], p,
          dilation, hi, wi, threads)
    return dx


def avgpool_forward(x, p, dilation, threads=1):
    x = _c(x)
    e = (p - 1) * dilation + 1
    y = np.empty((x.shape[0], x.shape[1] - e + 1, x.shape[2] - e + 1), dtype=x.dtype)
    _call("avgpool_forward", x, x, y, x.shape[0], x.shape[1], x.shape[2], p, dilation, threads)
    return y


def avgpool_backward(dy, p, dilation, hi, wi, threads=1):
    dy = _c(dy)
    dx = np.empty((dy.shape[0], hi, wi), dtype=dy.dtype)
    _call("avgpool_backward", dy, dy, dx, dy.shape[0], dy.shape[1], dy.shape[2], p, dilation,
          hi, wi, threads)
    return dx

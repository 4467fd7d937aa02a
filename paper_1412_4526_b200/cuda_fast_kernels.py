"""The "cuda-fast" kernel backend: the reference boundary's functions with the fp32
convolutions on the tcgen05 fast tier.

Same module contract as `cuda_kernels` (reference backend.py:25-48, _kernels.pyx:23-247):
C-contiguous numpy in, fresh numpy out, `threads` ignored.  The three fp32 convolution
functions run the tensor-core kernels (3xTF32 / fp16-split with its tf32 range guard, the
engine's fast tier) on device copies of the operands; everything else -- fp64 convs, the pools
(argmax bit-exact), the nonlinearities -- is `cuda_kernels`' exact tier.  Numerics of the
three convs: within the north-star 1e-4 normwise of the reference (tests/test_gpu_tc.py,
tests/test_gpu_reference_dropin.py), not bit-identical -- choose "cuda" for that.

Per call: H2D of the operands, the relayout / weight pack and the kernel, D2H of the result;
device workspaces are cached by size.  The reference's per-layer API copies every activation
over PCIe twice, so for whole networks the engine (`engine.DenseNet`) is the fast path; this
backend speeds up the reference's own harness where it spends its time (the convs).
"""

from __future__ import annotations

import numpy as np

from . import _lib, cuda_kernels
from .cuda_kernels import (_arr, _ext, avgpool_backward, avgpool_forward,  # noqa: F401
                           maxpool_backward, maxpool_forward, nonlin_backward, nonlin_forward)

_WS = {}


def _torch():
    import torch
    _lib.require_device()
    return torch


def _ws(nbytes: int):
    torch = _torch()
    buf = _WS.get("ws")
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device="cuda")
        _WS["ws"] = buf
    return buf


def _dev(a):
    return _torch().from_numpy(a).cuda()


def conv_forward(x, w, b, dilation, threads=1):
    x = _arr(x)
    if x.dtype != np.float32:
        return cuda_kernels.conv_forward(x, w, b, dilation, threads)
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
    from .engine import ops
    torch = _torch()
    if not ops.fast_supported(ci, co, l, int(dilation)):
        return cuda_kernels.conv_forward(x, w, b, dilation, threads)
    xt, wt, bt = _dev(x)[None], _dev(w), _dev(b)
    y = torch.empty((1, co, x.shape[1] - e + 1, x.shape[2] - e + 1), device="cuda")
    ws = _ws(ops.fwd_fast_workspace(xt, co, l, int(dilation)))
    ops.conv_forward_fast(xt, wt, bt, y, l, int(dilation), _lib.DP_IDENTITY, ws)
    return y[0].cpu().numpy()


def conv_backward_data(dy, w, dilation, threads=1):
    dy = _arr(dy)
    if dy.dtype != np.float32:
        return cuda_kernels.conv_backward_data(dy, w, dilation, threads)
    w = _arr(w, dy.dtype)
    co, ci, l, _ = w.shape
    if dy.ndim != 3 or dy.shape[0] != co:
        raise ValueError(f"conv_backward_data: delta {dy.shape} vs kernel {w.shape}")
    from .engine import ops
    torch = _torch()
    if not ops.fast_supported(co, ci, l, int(dilation)):
        return cuda_kernels.conv_backward_data(dy, w, dilation, threads)
    e = _ext(l, dilation)
    dyt, wt = _dev(dy)[None], _dev(w)
    dx = torch.empty((1, ci, dy.shape[1] + e - 1, dy.shape[2] + e - 1), device="cuda")
    ws = _ws(ops.bwd_fast_workspace(dyt, ci, l, int(dilation)))
    ops.conv_backward_data_fast(dyt, wt, dx, l, int(dilation), ws)
    return dx[0].cpu().numpy()


def conv_backward_kernel(x, dy, kernel_size, dilation, threads=1):
    x = _arr(x)
    if x.dtype != np.float32:
        return cuda_kernels.conv_backward_kernel(x, dy, kernel_size, dilation, threads)
    dy = _arr(dy, x.dtype)
    l = int(kernel_size)
    co = dy.shape[0]
    ci, hi, wi = x.shape
    e = _ext(l, dilation)
    if dy.shape[1] != hi - e + 1 or dy.shape[2] != wi - e + 1:
        raise ValueError(f"delta spatial dims {dy.shape[1:]} do not match the conv output for "
                         f"input {x.shape[1:]} (extent {e})")
    from .engine import ops
    torch = _torch()
    xt, dyt = _dev(x)[None], _dev(dy)[None]
    nb = ops.wgrad_fast_workspace(xt, co, l, int(dilation))
    if not nb:
        return cuda_kernels.conv_backward_kernel(x, dy, kernel_size, dilation, threads)
    dw = torch.empty((co, ci, l, l), device="cuda")
    db = torch.empty((co,), device="cuda")
    ops.conv_backward_kernel_fast(xt, dyt, dw, db, l, int(dilation), _ws(nb))
    return dw.cpu().numpy(), db.cpu().numpy()

"""Device-resident executors for the dense plan (torch CUDA tensors + the C ABI).

Two executors share the device entry points of libdenseprop_b200.so:

* `run_forward` / `run_backward` -- unfused, every layer input materialised
  (the reference ForwardCache keeps them all, forward.py:19-24); used by the
  drop-in `dense_forward` / `dense_backward` and by per-layer parity tests.

* `DenseNet` -- the throughput engine.  Batches of N images (N, C, H, W) in
  HBM, conv/pool kernels with the following nonlinearity fused into their
  epilogue (plan.fusion_groups()), backward kernels that apply the upstream
  nonlinearity's derivative in their epilogue ("gate"), 1-byte argmax maps,
  a masked squared-error loss kernel (cli.py:218 + backward.py:110-118),
  all buffers preallocated so a whole step can be captured in a CUDA graph,
  and one flat gradient bucket (the data-parallel all-reduce unit).

torch supplies device memory, streams and graphs only; every arithmetic op of
the path is one of this package's sm_100a kernels.
"""

from __future__ import annotations

from dataclasses import dataclass

import os

import numpy as np

from . import _lib
from .netspec import ConvLayerSpec, NonlinLayerSpec
from .plan import DensePlan, DilatedConv, DilatedPool

try:
    import torch
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None

_TORCH_DT = {}
if torch is not None:
    _TORCH_DT = {torch.float32: _lib.DP_F32, torch.float64: _lib.DP_F64}


def _code(t) -> int:
    try:
        return _TORCH_DT[t.dtype]
    except KeyError:
        raise TypeError(f"expected float32/float64 tensor, got {t.dtype}") from None


def _ptr(t):
    return None if t is None else t.data_ptr()


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _lib_dev():
    return _lib.require_device()


# ---------------------------------------------------------------------------
# thin typed wrappers over the device C ABI (batched NCHW tensors)
# ---------------------------------------------------------------------------

class _Rec:
    """Counts kernel launches and, when profiling, brackets each call with CUDA events."""

    def __init__(self, name, kernels, bound, work):
        self.name, self.kernels, self.bound, self.work = name, kernels, bound, work

    def __enter__(self):
        ops.launches += self.kernels
        if ops.profile is not None:
            self.e0 = torch.cuda.Event(enable_timing=True)
            self.e1 = torch.cuda.Event(enable_timing=True)
            self.e0.record(torch.cuda.current_stream())
        return self

    def __exit__(self, *exc):
        if ops.profile is not None and exc[0] is None:
            self.e1.record(torch.cuda.current_stream())
            ops.profile.append((self.name, self.bound, self.work, self.e0, self.e1))


def _repitches(x, dy) -> int:
    """Staging copies the tensor-core weight gradient launches (approximate): x unless it is
    read in place (every tap offset 16-byte aligned and 16-byte rows -- here: d % 4 == 0 is
    not known to this helper, so x staging is counted unless W % 4 == 0), dy when its row
    pitch is not 16-byte aligned."""
    return int(x.shape[3] % 4 != 0) + int(dy.stride(2) % 4 != 0)


def _nbytes(*ts):
    return sum(t.numel() * t.element_size() for t in ts if t is not None)


class ops:
    """Each method enqueues one kernel (two for the weight gradient) on the current
    torch stream.  `ops.launches` counts launches; set `ops.profile = []` to record
    (name, bound, algorithmic work, start event, end event) per call."""

    launches = 0
    profile = None

    @staticmethod
    def conv_forward(x, w, b, y, k, d, nonlin=_lib.DP_IDENTITY):
        with _Rec('conv_forward', 1, 'tensor', 2 * y.numel() * x.shape[1] * k * k):
            n, ci, h, wd = x.shape
            _lib.check(_lib_dev().dp_conv_forward(_code(x), _ptr(x), _ptr(w), _ptr(b), _ptr(y), n,
                                                  ci, h, wd, w.shape[0], k, d, nonlin, _stream()),
                       "conv_forward")

    @staticmethod
    def conv_backward_data(dy, w, dx, k, d, gate=None, gate_kind=_lib.DP_IDENTITY):
        with _Rec('conv_backward_data', 1, 'tensor', 2 * dy.numel() * w.shape[1] * k * k):
            n, co, ho, wo = dy.shape
            _lib.check(_lib_dev().dp_conv_backward_data(_code(dy), _ptr(dy), _ptr(w), _ptr(dx), n,
                                                        co, ho, wo, w.shape[1], k, d, _ptr(gate),
                                                        gate_kind if gate is not None else 0,
                                                        _stream()), "conv_backward_data")

    @staticmethod
    def fast_supported(reduce_c, out_c, k, d) -> bool:
        return bool(_lib_dev().dp_conv_fast_supported(reduce_c, out_c, k, d))

    @staticmethod
    def fast_workspace(reduce_c, out_c, k) -> int:
        return int(_lib_dev().dp_conv_fast_workspace(reduce_c, out_c, k))

    @staticmethod
    def fwd_fast_workspace(x, co, k, d) -> int:
        """Bytes that select the fastest forward kernel for this exact call (tap-stacked:
        packed weights + the input re-laid out as hi/lo channel-quad records)."""
        n, ci, h, w = x.shape
        return int(_lib_dev().dp_conv_forward_fast_workspace(n, ci, h, w, co, k, d))

    @staticmethod
    def bwd_fast_workspace(dy, ci, k, d) -> int:
        n, co, ho, wo = dy.shape
        return int(_lib_dev().dp_conv_backward_data_fast_workspace(n, co, ho, wo, ci, k, d))

    @staticmethod
    def conv_forward_fast(x, w, b, y, k, d, nonlin, ws, fp16_range=False, pack_fwd=False):
        """fp16_range: the caller vouches |x| stays well inside fp16 range (tanh outputs,
        images) -- allows the fp16-split forward (DP_FAST_INPUT_FP16_RANGE); pack_fwd: also for
        <= 8-channel inputs (DP_FAST_PACK_FWD, offset split)."""
        with _Rec('conv_forward_tc', 2, 'tensor', 2 * y.numel() * x.shape[1] * k * k):
            n, ci, h, wd = x.shape
            flags = _lib.DP_FAST_INPUT_FP16_RANGE if fp16_range else 0
            if fp16_range and pack_fwd:
                flags |= _lib.DP_FAST_PACK_FWD
            _lib.check(_lib_dev().dp_conv_forward_fast_ex(
                _ptr(x), _ptr(w), _ptr(b), _ptr(y), n, ci, h, wd, w.shape[0], k, d, nonlin,
                flags, _ptr(ws), ws.numel() * ws.element_size(), _stream()),
                "conv_forward_fast")

    @staticmethod
    def conv_backward_data_fast(dy, w, dx, k, d, ws, gate=None, gate_kind=_lib.DP_IDENTITY):
        with _Rec('conv_backward_data_tc', 2, 'tensor', 2 * dy.numel() * w.shape[1] * k * k):
            n, co, ho, wo = dy.shape
            _lib.check(_lib_dev().dp_conv_backward_data_fast(
                _ptr(dy), _ptr(w), _ptr(dx), n, co, ho, wo, w.shape[1], k, d, _ptr(gate),
                gate_kind if gate is not None else 0, _ptr(ws), ws.numel() * ws.element_size(),
                _stream()), "conv_backward_data_fast")

    @staticmethod
    def wgrad_workspace(x, co, k, d) -> int:
        n, ci, hi, wi = x.shape
        return int(_lib_dev().dp_conv_backward_kernel_workspace(_code(x), n, ci, hi, wi, co, k,
                                                                d))

    @staticmethod
    def conv_backward_kernel(x, dy, dw, db, k, d, ws):
        with _Rec('conv_backward_kernel', 2, 'tensor', 2 * dy.numel() * x.shape[1] * k * k):
            n, ci, hi, wi = x.shape
            co = dy.shape[1]
            _lib.check(_lib_dev().dp_conv_backward_kernel(_code(x), _ptr(x), _ptr(dy), _ptr(dw),
                                                          _ptr(db), n, ci, hi, wi, co, k, d,
                                                          _ptr(ws), ws.numel() * ws.element_size(),
                                                          _stream()), "conv_backward_kernel")

    @staticmethod
    def wgrad_fast_supported(x, co, k, d) -> bool:
        n, ci, hi, wi = x.shape
        return bool(_lib_dev().dp_conv_backward_kernel_fast_supported(n, ci, hi, wi, co, k, d))

    @staticmethod
    def wgrad_fast_workspace(x, co, k, d) -> int:
        n, ci, hi, wi = x.shape
        return int(_lib_dev().dp_conv_backward_kernel_fast_workspace(n, ci, hi, wi, co, k, d))

    @staticmethod
    def wgrad_f16_workspace(x, co, k, d) -> int:
        n, ci, hi, wi = x.shape
        return int(_lib_dev().dp_conv_backward_kernel_fast_f16_workspace(n, ci, hi, wi, co, k,
                                                                         d))

    @staticmethod
    def split_f16(x, x_hi, x_lo, x_hi_s=None, x_lo_s=None, shift=0):
        """x_hi = RN_fp16(x), x_lo = RN_fp16((x - x_hi) * 2^11) (the fp16 weight gradient's
        pre-split operand); x (..., W) -> x_hi / x_lo (..., P) halves, P >= W a multiple of 8
        (zeros past W); x_hi_s / x_lo_s: the same shifted left by `shift` halves (flat)."""
        w, pitch = x.shape[-1], x_hi.shape[-1]
        nout = 2 if x_hi_s is None else 4
        with _Rec('split_f16', 1, 'hbm', x.numel() * 4 + x_hi.numel() * 2 * nout):
            _lib.check(_lib_dev().dp_split_f16(
                _ptr(x), _ptr(x_hi), _ptr(x_lo), _ptr(x_hi_s) if x_hi_s is not None else None,
                _ptr(x_lo_s) if x_lo_s is not None else None, int(shift), x.numel() // w, w,
                pitch, _stream()), "split_f16")

    @staticmethod
    def wgrad_f16_shift(x, co, k, d) -> int:
        n, ci, hi, wi = x.shape
        return int(_lib_dev().dp_conv_backward_kernel_fast_f16_shift(n, ci, hi, wi, co, k, d))

    @staticmethod
    def conv_backward_kernel_fast_f16(x, x_hi, x_lo, dy, dw, db, k, d, ws, x_slack,
                                      dy_pitch=0, x_hi_s=None, x_lo_s=None):
        """fp16-split weight gradient: x_hi / x_lo (N, C, H, P) the fp16 split of x (lo scaled
        by 2^11, rows padded to P, split_f16), read in place (x_slack readable, finite bytes
        after each and after x); x itself feeds the tf32 fallback the device range guard
        selects."""
        # dy split, fp16 kernel, reduce; the gated tf32 fallback's (dy staging,) kernel, reduce
        with _Rec('conv_backward_kernel_tc', 6, 'tensor', 2 * dy.numel() * x.shape[1] * k * k):
            n, ci, hi, wi = x.shape
            co = dy.shape[1]
            _lib.check(_lib_dev().dp_conv_backward_kernel_fast_f16(
                _ptr(x), int(x_slack), _ptr(x_hi), _ptr(x_lo),
                _ptr(x_hi_s) if x_hi_s is not None else None,
                _ptr(x_lo_s) if x_lo_s is not None else None, int(x_slack), x_hi.shape[3],
                _ptr(dy),
                int(dy_pitch), _ptr(dw), _ptr(db), n, ci, hi, wi, co, k, d, _ptr(ws),
                ws.numel() * ws.element_size(), _stream()), "conv_backward_kernel_fast_f16")

    @staticmethod
    def conv_backward_kernel_fast(x, dy, dw, db, k, d, ws, x_slack=0, dy_pitch=0):
        """x_slack: readable bytes after x's storage (engine buffers carry SLACK_BYTES), which
        lets the kernel read x in place instead of staging a copy where the shape allows;
        dy_pitch: dy's row pitch when it is a strided (n, c, h, w) view."""
        with _Rec('conv_backward_kernel_tc', 2 + _repitches(x, dy), 'tensor',
                  2 * dy.numel() * x.shape[1] * k * k):
            n, ci, hi, wi = x.shape
            co = dy.shape[1]
            if x_slack or dy_pitch:
                _lib.check(_lib_dev().dp_conv_backward_kernel_fast_ex(
                    _ptr(x), int(x_slack), _ptr(dy), int(dy_pitch), _ptr(dw), _ptr(db), n, ci,
                    hi, wi, co, k, d, _ptr(ws), ws.numel() * ws.element_size(), _stream()),
                    "conv_backward_kernel_fast_ex")
                return
            _lib.check(_lib_dev().dp_conv_backward_kernel_fast(
                _ptr(x), _ptr(dy), _ptr(dw), _ptr(db), n, ci, hi, wi, co, k, d, _ptr(ws),
                ws.numel() * ws.element_size(), _stream()), "conv_backward_kernel_fast")

    @staticmethod
    def conv_backward_kernel_fast_prepare(x, co, k, d, ws):
        """Stage x for a later conv_backward_kernel_fast_staged on the same workspace."""
        with _Rec('wgrad_stage_x', 1, 'hbm', _nbytes(x)):
            n, ci, hi, wi = x.shape
            _lib.check(_lib_dev().dp_conv_backward_kernel_fast_prepare(
                _ptr(x), n, ci, hi, wi, co, k, d, _ptr(ws), ws.numel() * ws.element_size(),
                _stream()), "conv_backward_kernel_fast_prepare")

    @staticmethod
    def conv_backward_kernel_fast_staged(x, dy, dw, db, k, d, ws):
        with _Rec('conv_backward_kernel_tc', 1 + _repitches(x, dy), 'tensor',
                  2 * dy.numel() * x.shape[1] * k * k):
            n, ci, hi, wi = x.shape
            co = dy.shape[1]
            _lib.check(_lib_dev().dp_conv_backward_kernel_fast_staged(
                _ptr(x), _ptr(dy), _ptr(dw), _ptr(db), n, ci, hi, wi, co, k, d, _ptr(ws),
                ws.numel() * ws.element_size(), _stream()), "conv_backward_kernel_fast_staged")

    @staticmethod
    def maxpool_forward(x, y, arg, p, d, nonlin=_lib.DP_IDENTITY):
        with _Rec('maxpool_forward', 1, 'hbm', _nbytes(x, y, arg)):
            n, c, h, w = x.shape
            _lib.check(_lib_dev().dp_maxpool_forward(_code(x), _ptr(x), _ptr(y), _ptr(arg),
                                                     arg.element_size(), n, c, h, w, p, d, nonlin,
                                                     _stream()), "maxpool_forward")

    @staticmethod
    def maxpool_forward_split(x, y, arg, p, d, nonlin, y_hi, y_lo):
        """maxpool_forward (fp32, uint8 codes) that also writes y's fp16 split (split_f16's
        layout; pad columns untouched), fused into the streaming kernel where it applies."""
        with _Rec('maxpool_forward', 1, 'hbm', _nbytes(x, y, arg, y_hi, y_lo)):
            n, c, h, w = x.shape
            _lib.check(_lib_dev().dp_maxpool_forward_split(
                _ptr(x), _ptr(y), _ptr(arg), n, c, h, w, p, d, nonlin, _ptr(y_hi), _ptr(y_lo),
                y_hi.shape[3], _stream()), "maxpool_forward_split")

    @staticmethod
    def maxpool_backward(dy, arg, dx, p, d, gate=None, gate_kind=_lib.DP_IDENTITY, dx_pitch=0):
        """dx_pitch: write dx with that row pitch (dx a strided (n, c, h, w) view)."""
        with _Rec('maxpool_backward', 1, 'hbm', _nbytes(dy, arg, dx, gate)):
            n, c, ho, wo = dy.shape
            _lib.check(_lib_dev().dp_maxpool_backward_pitched(
                _code(dy), _ptr(dy), _ptr(arg), arg.element_size(), _ptr(dx),
                dx_pitch or dx.shape[3], n, c, ho, wo, p, d, dx.shape[2], dx.shape[3],
                _ptr(gate), gate_kind if gate is not None else 0, _stream()),
                "maxpool_backward")

    @staticmethod
    def avgpool_forward(x, y, p, d, nonlin=_lib.DP_IDENTITY):
        with _Rec('avgpool_forward', 1, 'hbm', _nbytes(x, y)):
            n, c, h, w = x.shape
            _lib.check(_lib_dev().dp_avgpool_forward(_code(x), _ptr(x), _ptr(y), n, c, h, w, p, d,
                                                     nonlin, _stream()), "avgpool_forward")

    @staticmethod
    def avgpool_backward(dy, dx, p, d, gate=None, gate_kind=_lib.DP_IDENTITY):
        with _Rec('avgpool_backward', 1, 'hbm', _nbytes(dy, dx, gate)):
            n, c, ho, wo = dy.shape
            _lib.check(_lib_dev().dp_avgpool_backward(_code(dy), _ptr(dy), _ptr(dx), n, c, ho, wo,
                                                      p, d, dx.shape[2], dx.shape[3], _ptr(gate),
                                                      gate_kind if gate is not None else 0,
                                                      _stream()), "avgpool_backward")

    @staticmethod
    def nonlin_forward(x, y, kind):
        with _Rec('nonlin_forward', 1, 'hbm', _nbytes(x, y)):
            _lib.check(_lib_dev().dp_nonlin_forward(_code(x), _ptr(x), _ptr(y), x.numel(), kind,
                                                    _stream()), "nonlin_forward")

    @staticmethod
    def nonlin_backward(dy, x, dx, kind, x_is_output=False):
        with _Rec('nonlin_backward', 1, 'hbm', _nbytes(dy, x, dx)):
            _lib.check(_lib_dev().dp_nonlin_backward(_code(dy), _ptr(dy), _ptr(x), _ptr(dx),
                                                     dy.numel(), kind, int(x_is_output), _stream()),
                       "nonlin_backward")

    @staticmethod
    def mask_delta(a, mask, out, target=None):
        with _Rec('mask_delta', 1, 'hbm', _nbytes(a, mask, out, target)):
            n, c, h, w = a.shape
            _lib.check(_lib_dev().dp_mask_delta(_code(a), _ptr(a), _ptr(target), _ptr(mask),
                                                _ptr(out), n, c, h, w, _stream()), "mask_delta")

    @staticmethod
    def softmax_xent(logits, labels, mask, delta, loss=None):
        """delta = softmax(logits) - onehot(labels) (per pixel, masked; label 255 = ignore)."""
        with _Rec('softmax_xent', 1, 'hbm', _nbytes(logits, labels, mask, delta, loss)):
            n, q, h, w = logits.shape
            _lib.check(_lib_dev().dp_softmax_xent_delta(
                _code(logits), _ptr(logits), _ptr(labels), _ptr(mask), _ptr(delta), _ptr(loss),
                n, q, h, w, _stream()), "softmax_xent")

    @staticmethod
    def pad(src, dst, top, bottom, left, right):
        with _Rec('pad', 1, 'hbm', _nbytes(src, dst)):
            n, c, h, w = src.shape
            _lib.check(_lib_dev().dp_pad(_code(src), _ptr(src), _ptr(dst), n, c, h, w, top, bottom,
                                         left, right, _stream()), "pad")

    @staticmethod
    def patch_gather(x0, out, patch, w, first, count):
        """out (count, C, patch, patch) <- windows of pixels [first, first+count) of ONE
        padded image x0 (C, Hp, Wp) (patch-by-patch baseline)."""
        with _Rec('patch_gather', 1, 'hbm', 2 * _nbytes(out)):
            c, hp, wp = x0.shape
            _lib.check(_lib_dev().dp_patch_gather(_code(x0), _ptr(x0), _ptr(out), c, hp, wp,
                                                  patch, w, first, count, _stream()),
                       "patch_gather")

    @staticmethod
    def crop(src, dst, top, left):
        with _Rec('crop', 1, 'hbm', 2 * _nbytes(dst)):
            n, c, hs, ws = src.shape
            _lib.check(_lib_dev().dp_crop(_code(src), _ptr(src), _ptr(dst), n, c, hs, ws, top, left,
                                          dst.shape[2], dst.shape[3], _stream()), "crop")

    @staticmethod
    def sgd(param, grad, lr):
        with _Rec('sgd', 1, 'hbm', 3 * _nbytes(param)):
            _lib.check(_lib_dev().dp_sgd_update(_code(param), _ptr(param), _ptr(grad),
                                                param.numel(), float(lr), _stream()), "sgd")


def _nl(kind: str) -> int:
    return _lib.NONLIN_CODE[kind]


# ---------------------------------------------------------------------------
# unfused executor (drop-in semantics)
# ---------------------------------------------------------------------------

def conv_params(plan: DensePlan, k: int, dtype, device):
    w, b = plan.conv_weights(k, dtype)
    return (torch.from_numpy(w).to(device, non_blocking=False),
            torch.from_numpy(b).to(device, non_blocking=False))


def run_forward(plan: DensePlan, x_padded, params=None):
    """All plan layers on (N, C, H, W) padded input; returns (inputs, argmax, output).

    argmax maps are int32 (the API type).  `params[k]` = (w, b) device tensors,
    uploaded from the plan when not given.
    """
    dev, dt = x_padded.device, x_padded.dtype
    np_dt = np.float32 if dt == torch.float32 else np.float64
    x = x_padded
    inputs, argmax = [], {}
    for k, layer in enumerate(plan.layers):
        inputs.append(x)
        n, c, h, w = x.shape
        if isinstance(layer, DilatedConv):
            wt, b = params[k] if params else conv_params(plan, k, np_dt, dev)
            e = layer.extent
            y = torch.empty((n, layer.base.out_channels, h - e + 1, w - e + 1), dtype=dt,
                            device=dev)
            ops.conv_forward(x, wt, b, y, layer.base.kernel_size, layer.dilation)
        elif isinstance(layer, DilatedPool):
            e = layer.extent
            y = torch.empty((n, c, h - e + 1, w - e + 1), dtype=dt, device=dev)
            if layer.base.kind == "max":
                arg = torch.empty(y.shape, dtype=torch.int32, device=dev)
                ops.maxpool_forward(x, y, arg, layer.base.kernel_size, layer.dilation)
                argmax[k] = arg
            else:
                ops.avgpool_forward(x, y, layer.base.kernel_size, layer.dilation)
        else:
            if layer.kind == "identity":
                y = x
            else:
                y = torch.empty_like(x)
                ops.nonlin_forward(x, y, _nl(layer.kind))
        x = y
    return inputs, argmax, x


def run_backward(plan: DensePlan, inputs, argmax, delta, params=None, with_input_grad=False):
    """Reverse sweep over (N, ...) tensors from an already-masked last-layer delta.

    Returns ({k: (dw, db)}, input_delta_padded_or_None).  Gradients are sums over
    the batch and all pixels (backward.py:190-191).
    """
    dev, dt = delta.device, delta.dtype
    np_dt = np.float32 if dt == torch.float32 else np.float64
    grads = {}
    for k in range(len(plan.layers) - 1, -1, -1):
        layer, x_in = plan.layers[k], inputs[k]
        if isinstance(layer, DilatedConv):
            wt, _ = params[k] if params else conv_params(plan, k, np_dt, dev)
            kk, d = layer.base.kernel_size, layer.dilation
            dw = torch.empty(wt.shape, dtype=dt, device=dev)
            db = torch.empty((wt.shape[0],), dtype=dt, device=dev)
            ws = torch.empty(max(1, ops.wgrad_workspace(x_in, wt.shape[0], kk, d)),
                             dtype=torch.uint8, device=dev)
            ops.conv_backward_kernel(x_in, delta, dw, db, kk, d, ws)
            grads[k] = (dw, db)
            if k == 0 and not with_input_grad:
                return grads, None
            dx = torch.empty(x_in.shape, dtype=dt, device=dev)
            ops.conv_backward_data(delta, wt, dx, kk, d)
            delta = dx
        elif isinstance(layer, DilatedPool):
            dx = torch.empty(x_in.shape, dtype=dt, device=dev)
            if layer.base.kind == "max":
                ops.maxpool_backward(delta, argmax[k], dx, layer.base.kernel_size,
                                     layer.dilation)
            else:
                ops.avgpool_backward(delta, dx, layer.base.kernel_size, layer.dilation)
            delta = dx
        else:
            if layer.kind != "identity":
                dx = torch.empty_like(delta)
                ops.nonlin_backward(delta, x_in, dx, _nl(layer.kind), x_is_output=False)
                delta = dx
    return grads, delta


# ---------------------------------------------------------------------------
# fused throughput engine
# ---------------------------------------------------------------------------

# Activation buffers are views of slightly longer allocations, so kernels may read a little
# past a tensor's end (the weight gradient's overlapping in-place tap view of x).
SLACK_BYTES = 64 * 1024


def _slack_empty(shape, kw):
    """The slack is zeroed: overlapping tap views multiply it by zero-filled dy columns, and
    garbage there could be NaN."""
    n = int(np.prod(shape))
    extra = SLACK_BYTES // torch.tensor([], dtype=kw["dtype"]).element_size()
    buf = torch.empty(n + extra, **kw)
    buf[n:].zero_()
    return buf[:n].view(shape)


def _slack_zeros(shape, kw):
    t = _slack_empty(shape, kw)
    t.zero_()
    return t


@dataclass
class _Group:
    first: int                 # plan index of the conv/pool/nonlin
    op: object                 # DilatedConv | DilatedPool | NonlinLayerSpec
    act: str                   # fused trailing nonlinearity kind ("identity" if none)
    out_shape: tuple           # (C, H, W) per image


class DenseNet:
    """Fused, preallocated dense engine for a batch of `batch` images of h x w.

    Buffers live in HBM for the life of the object; `forward`, `loss_delta`,
    `backward` and `sgd_step` only enqueue kernels on the current stream, so a
    whole step can be captured with `capture_step()` and replayed as one graph.
    """

    def __init__(self, plan: DensePlan, batch: int, height: int, width: int,
                 dtype=None, device="cuda", train=True, precision="fast"):
        """precision: "fast" runs fp32 convolutions on the tcgen05 tensor cores with
        3xTF32 products (normwise ~1e-6 vs fp32; reference tolerance 1e-4) wherever the
        layer fits the kernel, "exact" uses the CUDA-core kernels that reproduce the
        reference bit for bit.  fp64 is always exact."""
        if torch is None:
            raise _lib.KernelUnavailable("torch is required for the device engine")
        _lib.require_device()
        self.plan, self.batch, self.h, self.w = plan, batch, height, width
        self.dtype = dtype or torch.float32
        if precision not in ("fast", "exact"):
            raise ValueError("precision must be 'fast' or 'exact'")
        self.precision = precision if self.dtype == torch.float32 else "exact"
        self.device = torch.device(device)
        self.train = train
        self.np_dtype = np.float32 if self.dtype == torch.float32 else np.float64
        shapes = plan.layer_shapes(height, width)
        self.in_shape = shapes[0]
        # ---- fusion groups
        self.groups: list[_Group] = []
        for g in plan.fusion_groups():
            op = plan.layers[g[0]]
            act = plan.layers[g[1]].kind if len(g) == 2 else "identity"
            self.groups.append(_Group(g[0], op, act, shapes[g[-1] + 1]))
        kw = dict(dtype=self.dtype, device=self.device)
        N = batch
        # ---- parameters and the flat gradient bucket (conv layers in order, w then b)
        convs = [(k, l) for k, l in enumerate(plan.layers) if isinstance(l, DilatedConv)]
        sizes = [l.base.weights.size + l.base.bias.size for _, l in convs]
        total = int(sum(sizes))
        self.param_flat = torch.empty(total, **kw)
        self.grad_flat = torch.zeros(total, **kw) if train else None
        self.params, self.grads = {}, {}
        off = 0
        for (k, l), _ in zip(convs, sizes):
            nw, nb = l.base.weights.size, l.base.bias.size
            wv = self.param_flat[off:off + nw].view(l.base.weights.shape)
            bv = self.param_flat[off + nw:off + nw + nb]
            self.params[k] = (wv, bv)
            if train:
                self.grads[k] = (self.grad_flat[off:off + nw].view(l.base.weights.shape),
                                 self.grad_flat[off + nw:off + nw + nb])
            off += nw + nb
        self.load_weights_from_plan()
        # ---- activations: x0 (padded input) and one output per group
        self.x0 = _slack_zeros((N,) + tuple(self.in_shape), kw)
        self.acts = [_slack_empty((N,) + tuple(g.out_shape), kw) for g in self.groups]
        self.args = {}
        for gi, g in enumerate(self.groups):
            if isinstance(g.op, DilatedPool) and g.op.base.kind == "max":
                p = g.op.base.kernel_size
                adt = torch.uint8 if p * p <= 256 else torch.int32
                self.args[gi] = torch.empty((N,) + tuple(g.out_shape), dtype=adt,
                                            device=self.device)
        self.output = self.acts[-1]
        if train:
            biggest = max([int(np.prod(s)) for s in shapes])
            # layer 0's delta goes only to its weight gradient: when a max pool produces it
            # and its rows are not 16-byte aligned, the pool backward writes it with a padded
            # row pitch the weight gradient's TMA reads in place (no re-pitch copy)
            self._l0_pitch = 0
            c0, h0, w0 = self.groups[0].out_shape
            if (len(self.groups) > 1 and isinstance(self.groups[0].op, DilatedConv) and
                    isinstance(self.groups[1].op, DilatedPool) and
                    self.groups[1].op.base.kind == "max" and w0 % 4 and
                    self.dtype == torch.float32 and self.precision == "fast" and
                    not os.environ.get("DP_NO_L0_PITCH")):
                self._l0_pitch = (w0 + 3) // 4 * 4
                biggest = max(biggest, c0 * h0 * self._l0_pitch)
            # three rotating delta buffers: a layer's weight gradient runs on a side stream
            # (overlapping the data-gradient / pool-backward chain) and still reads its
            # delta while the next op writes; the third buffer keeps that delta intact
            # until the op after next (DP_NO_OVERLAP=1: serial, same results)
            self.overlap_wgrad = not os.environ.get("DP_NO_OVERLAP")
            nbuf = 3 if self.overlap_wgrad else 2
            self._dbuf = [torch.empty(N * biggest, **kw) for _ in range(nbuf)]
            self._wg_stream = torch.cuda.Stream(device=self.device) if self.overlap_wgrad else None
            ws = 256
            self.tc_wgrad = {}
            for gi, g in enumerate(self.groups):
                if isinstance(g.op, DilatedConv):
                    xin = self._group_input(gi)
                    co, kk, dd = g.op.base.out_channels, g.op.base.kernel_size, g.op.dilation
                    fast = (self.precision == "fast" and
                            ops.wgrad_fast_supported(xin, co, kk, dd))
                    self.tc_wgrad[gi] = fast
                    ws = max(ws, ops.wgrad_fast_workspace(xin, co, kk, dd) if fast else
                             ops.wgrad_workspace(xin, co, kk, dd))
            # fp16-split weight gradients (DP_WG_F16=0: off): a conv whose input is a tanh
            # output (|x| <= 1, inside fp16's range by construction) and whose shape the fp16
            # kernel takes gets that input split into fp16 hi / lo' once in the forward pass
            self._wg16 = {}
            if not os.environ.get("DP_WG_F16", "1") == "0":
                kw16 = {"dtype": torch.float16, "device": self.device}
                for gi, fast in self.tc_wgrad.items():
                    if not fast or gi == 0 or not self._fp16_input(gi):
                        continue
                    g, xin = self.groups[gi], self._group_input(gi)
                    nb = ops.wgrad_f16_workspace(xin, g.op.base.out_channels,
                                                 g.op.base.kernel_size, g.op.dilation)
                    shift = ops.wgrad_f16_shift(xin, g.op.base.out_channels,
                                                g.op.base.kernel_size, g.op.dilation)
                    if nb and shift >= 0:
                        # rows padded to 16 bytes; a second tap residue reads copies shifted
                        # by `shift` halves (its TMA boxes must start 16-byte aligned)
                        shp = tuple(xin.shape[:3]) + ((xin.shape[3] + 7) // 8 * 8,)
                        # (zeroed: the fused pool forward leaves the pad columns alone)
                        t = [_slack_zeros(shp, kw16) for _ in range(4 if shift else 2)]
                        self._wg16[gi] = {"hi": t[0], "lo": t[1], "nb": nb, "shift": shift,
                                          "hs": t[2] if shift else None,
                                          "ls": t[3] if shift else None}
                        ws = max(ws, nb)
            self._ws = torch.empty(ws, dtype=torch.uint8, device=self.device)
            # overlap mode: each fast weight gradient gets its own workspace so its x staging
            # can run during the forward pass (prepare) and survive until the backward
            self._ws_l = {}
            self._prepared = set()
            if self.overlap_wgrad:
                for gi, fast in self.tc_wgrad.items():
                    if fast:
                        g = self.groups[gi]
                        nb = ops.wgrad_fast_workspace(self._group_input(gi),
                                                      g.op.base.out_channels,
                                                      g.op.base.kernel_size, g.op.dilation)
                        if gi in self._wg16:
                            nb = max(nb, self._wg16[gi]["nb"])
                        self._ws_l[gi] = torch.empty(nb, dtype=torch.uint8, device=self.device)
            self.mask = torch.zeros((N, height, width), dtype=torch.uint8, device=self.device)
            self.target = torch.zeros_like(self.output)
            self.delta_last = torch.empty_like(self.output)
        # ---- tensor-core (fast tier) plan per conv group: (forward ok, data-grad ok)
        self.tc = {}
        tc_ws = 16
        for gi, g in enumerate(self.groups):
            if isinstance(g.op, DilatedConv) and self.precision == "fast":
                ci, co, kk = g.op.base.in_channels, g.op.base.out_channels, g.op.base.kernel_size
                dd = g.op.dilation
                f_ok = ops.fast_supported(ci, co, kk, dd)
                b_ok = train and gi > 0 and ops.fast_supported(co, ci, kk, dd)
                self.tc[gi] = (f_ok, b_ok)
                # one workspace shared by every fast conv call (they run in sequence on one
                # stream), sized for the tap-stacked kernels' relayout planes
                if f_ok:
                    tc_ws = max(tc_ws, ops.fwd_fast_workspace(self._group_input(gi), co, kk, dd))
                if b_ok:
                    tc_ws = max(tc_ws, ops.bwd_fast_workspace(self.acts[gi], ci, kk, dd))
        self._tc_ws = torch.empty(tc_ws, dtype=torch.uint8, device=self.device)
        self.graph = None

    def kernel_plan(self):
        """Which conv kernels run where: {plan layer: {"forward": tier, "data_grad": tier}}."""
        out = {}
        for gi, g in enumerate(self.groups):
            if isinstance(g.op, DilatedConv):
                f_ok, b_ok = self.tc.get(gi, (False, False))
                w_ok = getattr(self, "tc_wgrad", {}).get(gi, False)
                ci, co = g.op.base.in_channels, g.op.base.out_channels
                kk = g.op.base.kernel_size
                # fp16-split (3 passes, tf32 fallback launch when an operand leaves fp16's
                # range): inputs of >= 16 channels declared in range; deltas of >= 16
                # channels, or <= 8 tap-packed at >= 5 taps a row (tc_conv_flat.cu tf_half)
                f16f = (ci >= 16 or (ci <= 8 and self._feeds_tanh(gi))) and self._fp16_input(gi)
                f16b = co >= 16 or (co <= 8 and kk >= 5)
                fwd = ("tcgen05-3xtf32" if not f16f else "tcgen05-fp16x3-offset" if ci <= 8
                       else "tcgen05-fp16x3") if f_ok else "exact"
                dg = ("tcgen05-fp16x3-offset" if f16b else "tcgen05-3xtf32") if b_ok else "exact"
                if gi == 0:
                    dg = "not needed"  # layer 0's input delta is not computed (backward.py:208)
                wg = "cuda-core"
                if w_ok:
                    wg = ("tcgen05-fp16x3-offset" if gi in getattr(self, "_wg16", {})
                          else "tcgen05-3xtf32")
                out[g.first] = {"forward": fwd, "data_grad": dg, "weight_grad": wg}
        return out

    # ------------------------------------------------------------- parameters
    def load_weights_from_plan(self):
        for k, (wv, bv) in self.params.items():
            w, b = self.plan.conv_weights(k, self.np_dtype)
            wv.copy_(torch.from_numpy(w))
            bv.copy_(torch.from_numpy(b))

    def weights_numpy(self):
        return {k: (w.cpu().numpy(), b.cpu().numpy()) for k, (w, b) in self.params.items()}

    # ------------------------------------------------------------- helpers
    def _group_input(self, gi):
        return self.x0 if gi == 0 else self.acts[gi - 1]

    def _fp16_input(self, gi):
        """Is group gi's input bounded well inside fp16 range by construction?  The padded
        image (group 0) and tanh outputs (|x| <= 1) are; relu / identity outputs are not."""
        if gi == 0:
            return True
        prev = self.groups[gi - 1]
        if prev.act == "tanh":
            return True
        return isinstance(prev.op, NonlinLayerSpec) and prev.op.kind == "tanh"

    def _feeds_tanh(self, gi):
        """Does conv group gi's output reach a tanh before any other nonlinearity (directly,
        or through pools)?  Then its <= 8-channel input may take the fp16 offset split
        (DP_FAST_PACK_FWD): on relu nets the extra rounding turned into relu / argmax flips
        past the parity bar (c4), on tanh nets it did not (c3)."""
        if os.environ.get("DP_NO_PACK_FWD"):
            return False
        for g in self.groups[gi:]:
            if g.act != "identity":
                return g.act == "tanh"
            if isinstance(g.op, NonlinLayerSpec):
                return g.op.kind == "tanh"
            if g is not self.groups[gi] and isinstance(g.op, DilatedConv):
                return False
        return False

    def _view(self, buf, shape):
        n = int(np.prod(shape))
        return buf[:n].view(shape)

    # ------------------------------------------------------------- forward
    def set_padded_input(self, x0):
        """x0: (N, C, h + patch - 1, w + patch - 1) device tensor that is ALREADY padded (a
        row band of a bigger padded image in band sharding, trainer.BandParallelTrainer)."""
        if tuple(x0.shape) != tuple(self.x0.shape):
            raise ValueError(f"padded input {tuple(x0.shape)} != {tuple(self.x0.shape)}")
        self.x0.copy_(x0)

    def set_input(self, images):
        """images: (N, C, h, w) device tensor -> zero-padded x0 (forward.py:96-98)."""
        lead, trail = self.plan.lead_margin, self.plan.trail_margin
        ops.pad(images, self.x0, lead, trail, lead, trail)

    def forward(self, images=None, prepare_backward=False):
        """prepare_backward (training steps, with DP_PREPARE=1): stage every fast weight
        gradient's x on the side stream as soon as that x exists, overlapping the rest of the
        forward pass (the backward that follows then runs the staged weight-gradient
        kernels)."""
        if images is not None:
            self.set_input(images)
        # opt-in (DP_PREPARE=1): measured slower on c2 -- the staging copies on the side
        # stream slow the shared-memory-bound forward convs more than they save later
        prep = (prepare_backward and self.train and getattr(self, "overlap_wgrad", False)
                and bool(self._ws_l) and bool(os.environ.get("DP_PREPARE")))
        main = torch.cuda.current_stream(self.device)
        self._prepared = set()
        for gi, g in enumerate(self.groups):
            x, y = self._group_input(gi), self.acts[gi]
            op, act = g.op, _nl(g.act)
            if prep and gi in self._ws_l:
                self._wg_stream.wait_stream(main)
                with torch.cuda.stream(self._wg_stream):
                    ops.conv_backward_kernel_fast_prepare(x, op.base.out_channels,
                                                          op.base.kernel_size, op.dilation,
                                                          self._ws_l[gi])
                self._prepared.add(gi)
            if act == _lib.DP_TANH and self.precision == "fast":
                act = _lib.DP_TANH_FAST  # tanhf (<= 2 ulp) instead of the fp64 evaluation
            # the next conv's fp16 weight-gradient operand (split of y), if it has one
            s16 = getattr(self, "_wg16", {}).get(gi + 1) if self.train else None
            if isinstance(op, DilatedConv):
                wt, b = self.params[g.first]
                if self.tc.get(gi, (False, False))[0]:
                    ops.conv_forward_fast(x, wt, b, y, op.base.kernel_size, op.dilation, act,
                                          self._tc_ws, fp16_range=self._fp16_input(gi),
                                          pack_fwd=self._feeds_tanh(gi))
                else:
                    ops.conv_forward(x, wt, b, y, op.base.kernel_size, op.dilation, act)
            elif isinstance(op, DilatedPool):
                if (op.base.kind == "max" and s16 is not None and not s16["shift"] and
                        self.args[gi].dtype == torch.uint8 and x.dtype == torch.float32 and
                        not os.environ.get("DP_NO_SPLIT_FUSE")):
                    # the next conv's fp16 weight-gradient operand, written with the output
                    ops.maxpool_forward_split(x, y, self.args[gi], op.base.kernel_size,
                                              op.dilation, act, s16["hi"], s16["lo"])
                    s16 = None
                elif op.base.kind == "max":
                    ops.maxpool_forward(x, y, self.args[gi], op.base.kernel_size, op.dilation,
                                        act)
                else:
                    ops.avgpool_forward(x, y, op.base.kernel_size, op.dilation, act)
            else:
                if op.kind == "identity":
                    y.copy_(x)
                else:
                    kind = _nl(op.kind)
                    if kind == _lib.DP_TANH and self.precision == "fast":
                        kind = _lib.DP_TANH_FAST
                    ops.nonlin_forward(x, y, kind)
            if s16 is not None:  # not fused into the producer: a split pass
                ops.split_f16(y, s16["hi"], s16["lo"], s16["hs"], s16["ls"], s16["shift"])
        return self.output

    # ------------------------------------------------------------- loss / mask
    def loss_delta(self, target=None, mask=None, delta=None, labels=None, loss=None):
        """delta_last = mask ? (output - target) : 0 (the reference's squared-error delta,
        cli.py:218), or mask ? delta : 0, or -- with `labels` (uint8 (N, h, w), 255 =
        ignore) -- the softmax cross-entropy delta softmax(output) - onehot(labels) (per-pixel
        losses into `loss` when given)."""
        m = self.mask if mask is None else mask
        if labels is not None:
            ops.softmax_xent(self.output, labels, m, self.delta_last, loss)
        elif delta is not None:
            ops.mask_delta(delta, m, self.delta_last)
        else:
            t = self.target if target is None else target
            ops.mask_delta(self.output, m, self.delta_last, target=t)
        return self.delta_last

    # ------------------------------------------------------------- backward
    def backward(self, delta_last=None, with_input_grad=False):
        """Reverse sweep from the masked delta; fills self.grad_flat (sums)."""
        if not self.train:
            raise RuntimeError("engine built with train=False")
        delta = self.delta_last if delta_last is None else delta_last
        last = self.groups[-1]
        nbuf = len(self._dbuf)
        ping = 0
        main = torch.cuda.current_stream(self.device)
        side = self._wg_stream
        readers = [None] * nbuf  # side-stream event of the last weight gradient per buffer
        side_busy = False

        def out_buf(k, shape):
            # the main stream may overwrite buffer k once the side stream has read it
            if readers[k] is not None:
                main.wait_event(readers[k])
                readers[k] = None
            return self._view(self._dbuf[k], shape)

        def join():
            if side_busy:
                main.wait_stream(side)

        if last.act != "identity":
            # a net ending in conv/pool + nonlin: undo the fused nonlinearity first
            d2 = out_buf(ping, delta.shape)
            ops.nonlin_backward(delta, self.acts[-1], d2, _nl(last.act), x_is_output=True)
            delta, ping = d2, (ping + 1) % nbuf
        for gi in range(len(self.groups) - 1, -1, -1):
            g = self.groups[gi]
            x_in = self._group_input(gi)
            prev = self.groups[gi - 1] if gi > 0 else None
            gate, gk = None, 0
            if prev is not None and prev.act != "identity":
                gate, gk = x_in, _nl(prev.act)
            op = g.op
            if isinstance(op, DilatedConv):
                wt, _ = self.params[g.first]
                dw, db = self.grads[g.first]
                kk, d = op.base.kernel_size, op.dilation
                fast_w = self.tc_wgrad.get(gi, False)
                dyp = delta.stride(2) if (gi == 0 and delta.stride(2) != delta.shape[3]) else 0
                if side is not None:
                    # weight gradient on the side stream (in order; per-layer workspaces for
                    # the fast ones, x staged during the forward pass when prepared)
                    side.wait_stream(main)
                    with torch.cuda.stream(side):
                        if fast_w and gi in self._prepared:
                            ops.conv_backward_kernel_fast_staged(x_in, delta, dw, db, kk, d,
                                                                 self._ws_l[gi])
                        elif gi in self._wg16:
                            s16 = self._wg16[gi]
                            ops.conv_backward_kernel_fast_f16(
                                x_in, s16["hi"], s16["lo"], delta, dw, db, kk, d,
                                self._ws_l.get(gi, self._ws), SLACK_BYTES, dy_pitch=dyp,
                                x_hi_s=s16["hs"], x_lo_s=s16["ls"])
                        elif fast_w:
                            ops.conv_backward_kernel_fast(x_in, delta, dw, db, kk, d,
                                                          self._ws_l.get(gi, self._ws),
                                                          x_slack=SLACK_BYTES, dy_pitch=dyp)
                        else:
                            ops.conv_backward_kernel(x_in, delta, dw, db, kk, d, self._ws)
                    side_busy = True
                    ev = torch.cuda.Event()
                    ev.record(side)
                    src = (ping - 1) % nbuf  # buffer holding `delta` (if it is a buffer)
                    if delta.data_ptr() == self._dbuf[src].data_ptr():
                        readers[src] = ev
                elif gi in self._wg16:
                    s16 = self._wg16[gi]
                    ops.conv_backward_kernel_fast_f16(x_in, s16["hi"], s16["lo"], delta, dw, db,
                                                      kk, d, self._ws, SLACK_BYTES, dy_pitch=dyp,
                                                      x_hi_s=s16["hs"], x_lo_s=s16["ls"])
                elif fast_w:
                    ops.conv_backward_kernel_fast(x_in, delta, dw, db, kk, d, self._ws,
                                                  x_slack=SLACK_BYTES, dy_pitch=dyp)
                else:
                    ops.conv_backward_kernel(x_in, delta, dw, db, kk, d, self._ws)
                if gi == 0 and not with_input_grad:
                    join()
                    self._prepared = set()
                    return None
                dx = out_buf(ping, x_in.shape)
                if self.tc.get(gi, (False, False))[1]:
                    ops.conv_backward_data_fast(delta, wt, dx, kk, d, self._tc_ws, gate, gk)
                else:
                    ops.conv_backward_data(delta, wt, dx, kk, d, gate, gk)
            elif isinstance(op, DilatedPool):
                pitched = (gi == 1 and self._l0_pitch and self.tc_wgrad.get(0, False) and
                           0 not in self._prepared and not with_input_grad)
                if pitched:  # layer 0's delta, rows padded to a 16-byte pitch
                    _ = out_buf(ping, x_in.shape)  # (waits for the buffer's last reader)
                    n_, c_, h_, w_ = x_in.shape
                    pp = self._l0_pitch
                    dx = self._dbuf[ping].as_strided((n_, c_, h_, w_), (c_ * h_ * pp, h_ * pp,
                                                                        pp, 1))
                else:
                    dx = out_buf(ping, x_in.shape)
                if op.base.kind == "max":
                    ops.maxpool_backward(delta, self.args[gi], dx, op.base.kernel_size,
                                         op.dilation, gate, gk,
                                         dx_pitch=self._l0_pitch if pitched else 0)
                else:
                    ops.avgpool_backward(delta, dx, op.base.kernel_size, op.dilation, gate, gk)
            else:
                dx = out_buf(ping, x_in.shape)
                if op.kind == "identity":
                    dx.copy_(delta)
                else:
                    ops.nonlin_backward(delta, x_in, dx, _nl(op.kind), x_is_output=False)
                if gate is not None:
                    # standalone nonlin after a fused group: apply that group's gate too
                    ops.nonlin_backward(dx, x_in, dx, gk, x_is_output=True)
            delta, ping = dx, (ping + 1) % nbuf
        join()
        self._prepared = set()
        return delta

    def sgd_step(self, lr):
        ops.sgd(self.param_flat, self.grad_flat, lr)

    # ------------------------------------------------------------- whole step
    def train_step(self, lr=0.0, allreduce=None):
        """forward -> masked squared-error delta -> backward -> [allreduce] -> SGD."""
        self.forward(prepare_backward=True)
        self.loss_delta()
        self.backward()
        if allreduce is not None:
            allreduce(self.grad_flat)
        if lr:
            self.sgd_step(lr)

    def capture(self, fn, warmup=2):
        """Capture `fn()` (enqueue-only) into a CUDA graph; returns the graph."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                fn()
        torch.cuda.current_stream().wait_stream(s)
        try:  # keep the cudaGraph_t so its kernel nodes can be counted (graph_kernel_nodes)
            g = torch.cuda.CUDAGraph(keep_graph=True)
        except TypeError:
            g = torch.cuda.CUDAGraph()
        before = ops.launches
        with torch.cuda.graph(g):
            fn()
        self.graph_kernels = ops.launches - before
        exact = graph_kernel_nodes(g)
        if exact is not None:
            self.graph_kernels = exact
        return g

    def activation_bytes(self) -> int:
        ts = [self.x0] + list(self.acts) + list(self.args.values())
        if self.train:
            ts += list(self._dbuf) + [self._ws, self.target, self.delta_last, self.mask]
        return _nbytes(*ts)

    def conv_flops_per_image(self) -> dict:
        """Algorithmic conv FLOPs per image: fwd, bwd (no layer-0 dgrad)."""
        fwd = bwd = 0
        for gi, g in enumerate(self.groups):
            if isinstance(g.op, DilatedConv):
                c_out, ho, wo = g.out_shape
                cin = g.op.base.in_channels
                f = 2 * c_out * cin * g.op.base.kernel_size ** 2 * ho * wo
                fwd += f
                bwd += f if gi == 0 else 2 * f
        return {"fwd": fwd, "bwd": bwd}


def graph_kernel_nodes(g):
    """Kernel nodes of OUR library (namespace dp) in a captured CUDA graph, counted from the
    graph itself through the driver API (cuGraphGetNodes / cuGraphKernelNodeGetParams /
    cuFuncGetName: the runtime-API variants cannot resolve functions registered by the
    library's own static runtime); None when that introspection is unavailable (callers then
    keep the per-op estimate)."""
    try:
        from cuda.bindings import driver as drv
        graph = drv.CUgraph(init_value=g.raw_cuda_graph())
        err, _, n = drv.cuGraphGetNodes(graph, 0)
        if int(err) != 0:
            return None
        err, nodes, n = drv.cuGraphGetNodes(graph, n)
        if int(err) != 0:
            return None
        count = 0
        for nd in nodes[:n]:
            err, kind = drv.cuGraphNodeGetType(nd)
            if int(err) != 0 or kind != drv.CUgraphNodeType.CU_GRAPH_NODE_TYPE_KERNEL:
                continue
            err, params = drv.cuGraphKernelNodeGetParams(nd)
            if int(err) != 0:
                return None
            err, name = drv.cuFuncGetName(params.func)
            if int(err) != 0:
                return None
            name = name.decode() if isinstance(name, bytes) else str(name)
            if "2dp" in name or name.startswith("dp::"):
                count += 1
        return count
    except Exception:  # noqa: BLE001 -- introspection is best effort
        return None


def profile_step(trainer, reps=5):
    """Per-kernel CUDA-event durations of eager training steps (forward, loss, backward).

    Returns {"kernels": [{name, bound, ms, flops|bytes, achieved}], "step_ms"}; the
    k-th launch of every step is averaged over `reps` steps.
    """
    net = trainer.net if hasattr(trainer, "net") else trainer
    ops.profile = []
    # serial: per-kernel CUDA-event times are only meaningful without the side-stream overlap
    side, net._wg_stream = getattr(net, "_wg_stream", None), None
    try:
        for _ in range(reps):
            net.forward()
            net.loss_delta()
            net.backward()
        torch.cuda.synchronize()
        rec = ops.profile
    finally:
        ops.profile = None
        net._wg_stream = side
    per = len(rec) // reps
    out = []
    for i in range(per):
        entries = rec[i::per]
        ms = float(np.mean([e0.elapsed_time(e1) for _, _, _, e0, e1 in entries]))
        name, bound, work = entries[0][:3]
        item = {"name": f"{i:02d}:{name}", "bound": bound, "ms": ms}
        if bound == "tensor":
            item["flops"] = int(work)
            item["tflops"] = work / (ms / 1e3) / 1e12 if ms > 0 else None
        else:
            item["bytes"] = int(work)
            item["gbs"] = work / (ms / 1e3) / 1e9 if ms > 0 else None
        out.append(item)
    return {"kernels": out, "step_ms": float(sum(k["ms"] for k in out))}


def ensure_nonlin_spec(layer) -> bool:
    return isinstance(layer, NonlinLayerSpec)


__all__ = ["ops", "run_forward", "run_backward", "DenseNet", "ConvLayerSpec"]

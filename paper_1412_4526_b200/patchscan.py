"""Patch-by-patch evaluation on the GPU: the ORIGINAL strided network on batches of patches.

This is the computation dense propagation eliminates (the paper's baseline, SURVEY.md 8(f)
item 2), restated for the GPU so it can be timed on the same B200 and checked against the
dense path.  Public names follow the reference's patch-by-patch module
(pkg/src/denseprop/oracle.py):

  scan_forward(spec, image, pixels=None)          oracle.py:145-164  -> (Q, h, w) scores
  patch_backward_batch(spec, image, pixels, deltas) oracle.py:237-262  -> GradientSet (sums)
  patch_scan_forward(plan, images, ...)           batched device form used by bench.py

Each patch (patch_size x patch_size, cropped from the zero-padded image around the pixel,
fmap.crop_patch semantics: centre = (n//2, n//2)) goes through the strided layers
(oracle.py:29-91, 167-234):

  conv stride 1 ... the dense conv kernels at dilation 1 (same per-entry order as
                    conv_strided: bias, then (c, i, j) taps -- bit-identical on the exact
                    tier); fast tier = the tcgen05 kernels of the dense path
  conv stride s ... the stride-1 conv sampled every s pixels (dp_subsample); backward of
                    the zero-inserted delta (dp_zero_insert) -- exact, s^2 more MACs
  pool ............ dp_pool_strided_forward / _backward (first-wins max, int32 argmax)
  nonlin .......... dp_nonlin_forward / _backward (numpy semantics)

Weight / bias gradients are summed over every patch of the batch by the batched weight-
gradient kernels (the reference's unweighted per-pixel sum, oracle.py:258-262).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .backward import GradientSet
from .netspec import (ConvLayerSpec, NetworkSpec, PoolLayerSpec, padding_margins,
                      patch_size)

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None


def _dev():
    return _lib.require_device()


def _st():
    return torch.cuda.current_stream().cuda_stream


def _code(t):
    return _lib.DP_F32 if t.dtype == torch.float32 else _lib.DP_F64


class PatchNet:
    """Preallocated strided network for batches of `batch` patches (device tensors)."""

    def __init__(self, spec: NetworkSpec, batch: int, dtype=None, precision: str = "fast",
                 train: bool = False, device="cuda"):
        from .engine import ops
        if torch is None:
            raise _lib.KernelUnavailable("torch is required for the device engine")
        _dev()
        self.spec, self.batch, self.ops = spec, batch, ops
        self.dtype = dtype or torch.float32
        self.precision = precision if self.dtype == torch.float32 else "exact"
        self.device = torch.device(device)
        self.train = train
        self.n = patch_size(spec)
        kw = dict(dtype=self.dtype, device=self.device)
        np_dt = np.float32 if self.dtype == torch.float32 else np.float64
        side, c = self.n, spec.input_channels
        self.inputs, self.full, self.args, self.params, self.fast = [], {}, {}, {}, {}
        ws = 16
        for k, layer in enumerate(spec.layers):
            x = torch.empty((batch, c, side, side), **kw)
            self.inputs.append(x)
            if isinstance(layer, ConvLayerSpec):
                l, s, co = layer.kernel_size, layer.stride, layer.out_channels
                self.params[k] = (torch.from_numpy(np.ascontiguousarray(layer.weights, np_dt)).to(
                    self.device), torch.from_numpy(np.ascontiguousarray(layer.bias, np_dt)).to(
                    self.device))
                if s > 1:  # stride-1 result before sampling (and zero-inserted delta)
                    self.full[k] = torch.empty((batch, co, side - l + 1, side - l + 1), **kw)
                fwd = self.precision == "fast" and ops.fast_supported(c, co, l, 1)
                bwd = (self.precision == "fast" and train and k > 0 and
                       ops.fast_supported(co, c, l, 1))
                wgr = self.precision == "fast" and train and ops.wgrad_fast_supported(x, co, l, 1)
                self.fast[k] = (fwd, bwd, wgr)
                y_full = self.full.get(k, None)
                if fwd:
                    ws = max(ws, ops.fwd_fast_workspace(x, co, l, 1))
                if train:
                    dy = y_full if y_full is not None else torch.empty(
                        (1, co, side - l + 1, side - l + 1), **kw)
                    dyb = dy.expand(batch, -1, -1, -1) if y_full is None else dy
                    if bwd:
                        ws = max(ws, ops.bwd_fast_workspace(dyb, c, l, 1))
                    ws = max(ws, ops.wgrad_fast_workspace(x, co, l, 1) if wgr else
                             ops.wgrad_workspace(x, co, l, 1))
                side, c = (side - l) // s + 1, co
            elif isinstance(layer, PoolLayerSpec):
                p, s = layer.kernel_size, layer.stride
                side = (side - p) // s + 1
                if layer.kind == "max":
                    self.args[k] = torch.empty((batch, c, side, side), dtype=torch.int32,
                                               device=self.device)
        self.output = torch.empty((batch, c, side, side), **kw)
        self.out_channels = c
        self._ws = torch.empty(ws, dtype=torch.uint8, device=self.device)
        if train:
            self.grads = {k: (torch.zeros_like(w), torch.zeros_like(b))
                          for k, (w, b) in self.params.items()}

    # ------------------------------------------------------------------ forward
    def forward(self, patches=None):
        """patches: (batch, C, n, n) device tensor (or already in self.inputs[0])."""
        ops, dev, st = self.ops, _dev(), _st()
        if patches is not None:
            self.inputs[0].copy_(patches)
        L = self.spec.layers
        for k, layer in enumerate(L):
            x = self.inputs[k]
            y = self.inputs[k + 1] if k + 1 < len(L) else self.output
            if isinstance(layer, ConvLayerSpec):
                w, b = self.params[k]
                l, s = layer.kernel_size, layer.stride
                dst = self.full.get(k, y)
                if self.fast[k][0]:
                    ops.conv_forward_fast(x, w, b, dst, l, 1, _lib.DP_IDENTITY, self._ws)
                else:
                    ops.conv_forward(x, w, b, dst, l, 1)
                if s > 1:
                    n, c, h, wd = dst.shape
                    _lib.check(dev.dp_subsample(_code(x), dst.data_ptr(), y.data_ptr(), n, c, h,
                                                wd, s, y.shape[2], y.shape[3], st), "subsample")
            elif isinstance(layer, PoolLayerSpec):
                kind = _lib.DP_POOL_MAX if layer.kind == "max" else _lib.DP_POOL_AVG
                arg = self.args.get(k)
                n, c, h, wd = x.shape
                _lib.check(dev.dp_pool_strided_forward(
                    _code(x), kind, x.data_ptr(), y.data_ptr(),
                    arg.data_ptr() if arg is not None else None, n, c, h, wd,
                    layer.kernel_size, layer.stride, st), "pool_strided_forward")
            else:
                if layer.kind == "identity":
                    y.copy_(x)
                else:
                    ops.nonlin_forward(x, y, _lib.NONLIN_CODE[layer.kind])
        return self.output

    # ------------------------------------------------------------------ backward
    def backward(self, delta, accumulate=True):
        """delta: (batch, Q) or (batch, Q, 1, 1) device tensor of last-layer errors (zero
        rows for padding patches).  Adds every patch's gradients into self.grads."""
        if not self.train:
            raise RuntimeError("PatchNet built with train=False")
        ops, dev, st = self.ops, _dev(), _st()
        delta = delta.reshape(self.output.shape).contiguous()
        if not accumulate:
            for dw, db in self.grads.values():
                dw.zero_()
                db.zero_()
        L = self.spec.layers
        for k in range(len(L) - 1, -1, -1):
            layer, x = L[k], self.inputs[k]
            if isinstance(layer, ConvLayerSpec):
                w, _ = self.params[k]
                l, s = layer.kernel_size, layer.stride
                if s > 1:
                    full = self.full[k]
                    n, c, ho, wo = delta.shape
                    _lib.check(dev.dp_zero_insert(_code(delta), delta.data_ptr(), full.data_ptr(),
                                                  n, c, ho, wo, s, full.shape[2], full.shape[3],
                                                  st), "zero_insert")
                    delta = full
                dw, db = self.grads[k]
                tw, tb = torch.empty_like(dw), torch.empty_like(db)
                if self.fast[k][2]:
                    ops.conv_backward_kernel_fast(x, delta, tw, tb, l, 1, self._ws)
                else:
                    ops.conv_backward_kernel(x, delta, tw, tb, l, 1, self._ws)
                dw.add_(tw)
                db.add_(tb)
                if k == 0:
                    return None
                dx = torch.empty_like(x)
                if self.fast[k][1]:
                    ops.conv_backward_data_fast(delta, w, dx, l, 1, self._ws)
                else:
                    ops.conv_backward_data(delta, w, dx, l, 1)
            elif isinstance(layer, PoolLayerSpec):
                kind = _lib.DP_POOL_MAX if layer.kind == "max" else _lib.DP_POOL_AVG
                arg = self.args.get(k)
                dx = torch.empty_like(x)
                n, c, ho, wo = delta.shape
                _lib.check(dev.dp_pool_strided_backward(
                    _code(delta), kind, delta.data_ptr(),
                    arg.data_ptr() if arg is not None else None, dx.data_ptr(), n, c, ho, wo,
                    layer.kernel_size, layer.stride, x.shape[2], x.shape[3], st),
                    "pool_strided_backward")
            else:
                dx = torch.empty_like(x)
                if layer.kind == "identity":
                    dx.copy_(delta)
                else:
                    ops.nonlin_backward(delta, x, dx, _lib.NONLIN_CODE[layer.kind])
            delta = dx
        return delta


def _padded(spec, image_t):
    """(C, h, w) device tensor -> zero-padded (C, h + n - 1, w + n - 1) (forward.py:96-98)."""
    lead, trail = padding_margins(spec)
    c, h, w = image_t.shape
    x0 = torch.zeros((c, h + lead + trail, w + lead + trail), dtype=image_t.dtype,
                     device=image_t.device)
    x0[:, lead:lead + h, lead:lead + w] = image_t
    return x0


def _gather(x0, out, pix_t, n):
    c, hp, wp = x0.shape
    _lib.check(_dev().dp_patch_gather_pixels(_code(x0), x0.data_ptr(), out.data_ptr(), c, hp, wp,
                                             n, pix_t.data_ptr(), pix_t.numel(), _st()),
               "patch_gather_pixels")


def _pixel_list(pixels, h, w):
    pix = np.asarray(list(pixels), dtype=np.int64).reshape(-1, 2)
    if pix.size and (pix.min() < 0 or (pix[:, 0] >= h).any() or (pix[:, 1] >= w).any()):
        bad = pix[(pix[:, 0] < 0) | (pix[:, 1] < 0) | (pix[:, 0] >= h) | (pix[:, 1] >= w)][0]
        raise ValueError(f"pixel ({bad[0]}, {bad[1]}) outside {h}x{w} image")
    return (pix[:, 0] * w + pix[:, 1]).astype(np.int32)


def _check_image(spec, image):
    image = np.asarray(image)
    if image.dtype not in (np.float32, np.float64):
        raise TypeError(f"expected float32/float64 image, got {image.dtype}")
    if image.ndim != 3 or image.shape[0] != spec.input_channels:
        raise ValueError(f"image has {image.shape[0] if image.ndim == 3 else image.shape} "
                         f"channels, spec wants {spec.input_channels}")
    return np.ascontiguousarray(image)


def scan_forward(spec: NetworkSpec, image, pixels=None, precision: str = "exact",
                 batch: int = 4096) -> np.ndarray:
    """Score the patch of every pixel (or of `pixels`) independently (oracle.py:145-164);
    unscanned pixels stay 0.  numpy in / out, like the reference."""
    image = _check_image(spec, image)
    c, h, w = image.shape
    if pixels is None:
        flat = np.arange(h * w, dtype=np.int32)
    else:
        flat = _pixel_list(pixels, h, w)
    dt = torch.float32 if image.dtype == np.float32 else torch.float64
    x0 = _padded(spec, torch.from_numpy(image).to("cuda"))
    batch = max(1, min(batch, len(flat) or 1))
    net = PatchNet(spec, batch, dtype=dt, precision=precision)
    out = torch.zeros((net.out_channels, h * w), dtype=dt, device="cuda")
    pix_all = torch.from_numpy(flat).to("cuda")
    for first in range(0, len(flat), batch):
        pix = pix_all[first:first + batch]
        cnt = pix.numel()
        _gather(x0, net.inputs[0], pix, net.n)
        if cnt < batch:
            net.inputs[0][cnt:].zero_()
        net.forward()
        out[:, pix.long()] = net.output[:cnt, :, 0, 0].t()
    return out.view(net.out_channels, h, w).cpu().numpy()


def patch_backward_batch(spec: NetworkSpec, image, pixels, deltas, precision: str = "exact",
                         batch: int = 2048) -> GradientSet:
    """Per-patch forward + backward for each selected pixel, gradients summed
    (oracle.py:237-262).  `deltas` holds one (out_channels,) error vector per pixel."""
    image = _check_image(spec, image)
    pixels, deltas = list(pixels), list(deltas)
    if len(pixels) != len(deltas):
        raise ValueError(f"{len(pixels)} pixels but {len(deltas)} delta vectors")
    c, h, w = image.shape
    flat = _pixel_list(pixels, h, w)
    dt = torch.float32 if image.dtype == np.float32 else torch.float64
    grads = GradientSet.zeros(spec, dtype=image.dtype)
    if not len(flat):
        return grads
    d = np.asarray(deltas, dtype=image.dtype).reshape(len(flat), -1)
    x0 = _padded(spec, torch.from_numpy(image).to("cuda"))
    batch = max(1, min(batch, len(flat)))
    net = PatchNet(spec, batch, dtype=dt, precision=precision, train=True)
    pix_all = torch.from_numpy(flat).to("cuda")
    d_all = torch.from_numpy(np.ascontiguousarray(d)).to("cuda")
    dbuf = torch.zeros((batch, net.out_channels), dtype=dt, device="cuda")
    for first in range(0, len(flat), batch):
        pix = pix_all[first:first + batch]
        cnt = pix.numel()
        _gather(x0, net.inputs[0], pix, net.n)
        dbuf.zero_()
        dbuf[:cnt] = d_all[first:first + cnt]
        if cnt < batch:
            net.inputs[0][cnt:].zero_()
        net.forward()
        net.backward(dbuf)
    torch.cuda.current_stream().synchronize()
    for k, (dw, db) in net.grads.items():
        grads.kernel[k] = dw.cpu().numpy()
        grads.bias[k] = db.cpu().numpy()
    return grads


def patch_scan_forward(plan, images, batch: int = 4096, precision: str = "fast", dtype=None):
    """images: (N, C, h, w) CUDA tensor -> (N, Q, h, w): every pixel's patch through the
    strided network, in batches of `batch` patches (the GPU patch-by-patch baseline)."""
    spec = plan.source
    n_img, c, h, w = images.shape
    batch = max(1, min(batch, h * w))
    net = PatchNet(spec, batch, dtype=dtype or images.dtype, precision=precision)
    out = torch.empty((n_img, net.out_channels, h * w), dtype=images.dtype,
                      device=images.device)
    pix_all = torch.arange(h * w, dtype=torch.int32, device=images.device)
    for img in range(n_img):
        x0 = _padded(spec, images[img])
        for first in range(0, h * w, batch):
            pix = pix_all[first:first + batch]
            cnt = pix.numel()
            _gather(x0, net.inputs[0], pix, net.n)
            if cnt < batch:
                net.inputs[0][cnt:].zero_()
            net.forward()
            out[img, :, first:first + cnt] = net.output[:cnt, :, 0, 0].t()
    return out.view(n_img, net.out_channels, h, w)

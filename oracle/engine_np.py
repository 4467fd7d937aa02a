"""Oracle dense engine + patch-by-patch scan (test infrastructure; see oracle/__init__.py).

Restates, against an `ONet` (oracle/netdesc.py) and any kernel module exposing
the 7 boundary functions (kernels_np, kernels_c, or the reference's own
compiled Cython in oracle/_ref):

* dense_forward ........ reference forward.py:96-128 (pad with (lead, trail)
                          margins, run every layer at stride 1 with its dilation,
                          cache every layer input + argmax maps)
* dense_backward ....... backward.py:185-223 (mask the last error map, reverse
                          sweep, unweighted gradient sums, layer-0 data grad
                          skipped unless with_input_grad)
* nonlin fwd/bwd ....... forward.py:69-76, backward.py:172-182 (numpy, outside
                          the kernel boundary in the reference too)
* scan_forward / patch_backward_batch ... oracle.py:145-164, 237-262: the
  ORIGINAL strided network run on one cropped patch per pixel.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import kernels_np
from .netdesc import OConv, ONet, ONonlin, OPool


# ----------------------------------------------------------------------------
# nonlinearities (forward.py:69-76, backward.py:172-182)
# ----------------------------------------------------------------------------

def nonlin_fwd(x, kind):
    if kind == "tanh":
        return np.tanh(x)
    if kind == "relu":
        return np.maximum(x, 0)
    if kind == "identity":
        return x
    raise ValueError(kind)


def nonlin_bwd(delta, x_in, kind):
    if kind == "tanh":
        t = np.tanh(x_in)
        return delta * (1.0 - t * t)
    if kind == "relu":
        return delta * (x_in > 0)
    if kind == "identity":
        return delta
    raise ValueError(kind)


# ----------------------------------------------------------------------------
# dense engine
# ----------------------------------------------------------------------------

@dataclass
class OCache:
    inputs: list
    argmax: dict
    output: np.ndarray


def pad_image(net: ONet, image):
    lead, trail = net.margins()
    c, h, w = image.shape
    out = np.zeros((c, h + lead + trail, w + lead + trail), dtype=image.dtype)
    out[:, lead:lead + h, lead:lead + w] = image
    return out


def _extent(k, d):
    return (k - 1) * d + 1


def dense_forward(net: ONet, image, K=kernels_np, threads=1, padded=False) -> OCache:
    """padded=True: `image` is already the padded input (a row band with its halo in the
    band-sharding tests); the reference always pads (forward.py:96-98)."""
    x = np.ascontiguousarray(image) if padded else pad_image(net, np.ascontiguousarray(image))
    dt = x.dtype
    inputs, argmax = [], {}
    for k, (layer, d) in enumerate(zip(net.layers, net.dilations())):
        inputs.append(x)
        if isinstance(layer, OConv):
            x = K.conv_forward(x, np.ascontiguousarray(layer.w, dtype=dt),
                               np.ascontiguousarray(layer.b, dtype=dt), d, threads)
        elif isinstance(layer, OPool):
            if layer.kind == "max":
                x, argmax[k] = K.maxpool_forward(x, layer.k, d, threads)
            else:
                x = K.avgpool_forward(x, layer.k, d, threads)
        else:
            x = nonlin_fwd(x, layer.kind)
        x = np.ascontiguousarray(x)
    return OCache(inputs, argmax, x)


def mask_from_pixels(h, w, pixels):
    m = np.zeros((h, w), dtype=bool)
    for y, x in pixels:
        m[y, x] = True
    return m


def dense_backward(net: ONet, cache: OCache, delta_last, mask_bool, K=kernels_np,
                   threads=1, with_input_grad=False):
    """Returns (kernel_grads, bias_grads, input_delta) lists aligned with layers."""
    dt = delta_last.dtype
    kgr = [None] * len(net.layers)
    bgr = [None] * len(net.layers)
    delta = np.zeros(delta_last.shape, dtype=dt)
    delta[:, mask_bool] = delta_last[:, mask_bool]
    dils = net.dilations()
    for k in range(len(net.layers) - 1, -1, -1):
        layer, d, x_in = net.layers[k], dils[k], cache.inputs[k]
        if isinstance(layer, OConv):
            kgr[k], bgr[k] = K.conv_backward_kernel(x_in, np.ascontiguousarray(delta),
                                                    layer.k, d, threads)
            if k == 0 and not with_input_grad:
                return kgr, bgr, None
            delta = K.conv_backward_data(np.ascontiguousarray(delta),
                                         np.ascontiguousarray(layer.w, dtype=dt), d, threads)
        elif isinstance(layer, OPool):
            e = _extent(layer.k, d)
            hi, wi = delta.shape[1] + e - 1, delta.shape[2] + e - 1
            if layer.kind == "max":
                delta = K.maxpool_backward(np.ascontiguousarray(delta), cache.argmax[k],
                                           layer.k, d, hi, wi, threads)
            else:
                delta = K.avgpool_backward(np.ascontiguousarray(delta), layer.k, d,
                                           hi, wi, threads)
        else:
            delta = nonlin_bwd(delta, x_in, layer.kind)
    inp = None
    if with_input_grad:
        lead = net.margins()[0]
        h, w = cache.output.shape[1:]
        inp = delta[:, lead:lead + h, lead:lead + w].copy()
    return kgr, bgr, inp


# ----------------------------------------------------------------------------
# patch-by-patch scan: the original strided network (oracle.py:29-262)
# ----------------------------------------------------------------------------

def _taps(x, i, j, s, mo, no):
    return x[:, i:i + (mo - 1) * s + 1:s, j:j + (no - 1) * s + 1:s]


def _strided_layer(layer, x):
    if isinstance(layer, OConv):
        s, l = layer.stride, layer.k
        mo, no = (x.shape[1] - l) // s + 1, (x.shape[2] - l) // s + 1
        w = layer.w.astype(x.dtype)
        y = np.empty((w.shape[0], mo, no), dtype=x.dtype)
        y[...] = layer.b.astype(x.dtype)[:, None, None]
        for c in range(w.shape[1]):
            for i in range(l):
                for j in range(l):
                    y += w[:, c, i, j][:, None, None] * _taps(x[c:c + 1], i, j, s, mo, no)
        return y, None
    if isinstance(layer, OPool):
        s, p = layer.stride, layer.k
        mo, no = (x.shape[1] - p) // s + 1, (x.shape[2] - p) // s + 1
        if layer.kind == "max":
            y = _taps(x, 0, 0, s, mo, no).copy()
            arg = np.zeros(y.shape, dtype=np.int32)
            for t in range(1, p * p):
                tap = _taps(x, t // p, t % p, s, mo, no)
                up = tap > y
                y = np.where(up, tap, y)
                arg = np.where(up, np.int32(t), arg)
            return y, arg
        y = _taps(x, 0, 0, s, mo, no).copy()
        for t in range(1, p * p):
            y = y + _taps(x, t // p, t % p, s, mo, no)
        return y / (p * p), None
    return nonlin_fwd(x, layer.kind), None


def _patch_forward_cached(net, patch):
    inputs, args, x = [], {}, patch
    for k, layer in enumerate(net.layers):
        inputs.append(x)
        x, a = _strided_layer(layer, x)
        if a is not None:
            args[k] = a
    return inputs, args, x


def scan_forward(net: ONet, image, pixels=None):
    n = net.patch()
    lead, _ = net.margins()
    padded = pad_image(net, image)
    h, w = image.shape[1:]
    out = np.zeros((net.out_channels, h, w), dtype=image.dtype)
    if pixels is None:
        pixels = [(y, x) for y in range(h) for x in range(w)]
    for y, x in pixels:
        top, left = y + lead - n // 2, x + lead - n // 2
        _, _, sc = _patch_forward_cached(net, padded[:, top:top + n, left:left + n])
        out[:, y, x] = sc.reshape(-1)
    return out


def patch_backward_batch(net: ONet, image, pixels, deltas):
    """Sum over pixels of the per-patch strided backward (oracle.py:167-262)."""
    n = net.patch()
    lead, _ = net.margins()
    padded = pad_image(net, image)
    dt = image.dtype
    kgr = [np.zeros_like(l.w, dtype=dt) if isinstance(l, OConv) else None for l in net.layers]
    bgr = [np.zeros_like(l.b, dtype=dt) if isinstance(l, OConv) else None for l in net.layers]
    for (y, x), dvec in zip(pixels, deltas):
        top, left = y + lead - n // 2, x + lead - n // 2
        inputs, args, _ = _patch_forward_cached(net, padded[:, top:top + n, left:left + n])
        delta = np.asarray(dvec, dtype=dt).reshape(-1, 1, 1)
        for k in range(len(net.layers) - 1, -1, -1):
            layer, xin = net.layers[k], inputs[k]
            if isinstance(layer, OConv):
                s, l = layer.stride, layer.k
                w = layer.w.astype(dt)
                mo, no = delta.shape[1:]
                dx = np.zeros_like(xin) if k > 0 else None
                for i in range(l):
                    for j in range(l):
                        win = _taps(xin, i, j, s, mo, no)
                        kgr[k][:, :, i, j] += np.tensordot(delta, win, axes=([1, 2], [1, 2]))
                        if dx is not None:
                            dx[:, i:i + (mo - 1) * s + 1:s, j:j + (no - 1) * s + 1:s] += \
                                np.tensordot(w[:, :, i, j], delta, axes=(0, 0))
                bgr[k] += delta.sum(axis=(1, 2))
                if dx is None:
                    break
                delta = dx
            elif isinstance(layer, OPool):
                s, p = layer.stride, layer.k
                mo, no = delta.shape[1:]
                dx = np.zeros(xin.shape, dtype=dt)
                for t in range(p * p):
                    i, j = divmod(t, p)
                    contrib = delta if layer.kind == "avg" else np.where(args[k] == t, delta, 0)
                    if layer.kind == "avg":
                        contrib = delta / (p * p)
                    dx[:, i:i + (mo - 1) * s + 1:s, j:j + (no - 1) * s + 1:s] += contrib
                delta = dx
            else:
                delta = nonlin_bwd(delta, xin, layer.kind)
    return kgr, bgr

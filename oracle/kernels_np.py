"""numpy restatement of the 7 boundary kernels (test infrastructure; see oracle/__init__.py).

Every function follows the *compiled* reference backend's per-entry float
operation order (pkg/src/denseprop/_kernels.pyx), vectorised over output
positions so each entry sees the same scalar op sequence:

* conv_forward .......... _kernels.pyx:23-53  bias, then taps in (c, i, j) order,
                          multiply then add (no FMA: setup.py:15 -ffp-contract=off)
* conv_backward_data .... _kernels.pyx:56-91  gather in (o, i, j) order with the
                          180-degree rotated kernel; taps that fall outside dy
                          are skipped there and add an exact 0.0 here
* conv_backward_kernel .. _kernels.pyx:94-130 reduction over (u, v); NOT
                          order-matched (a sequential 1e5-1e6 term sum cannot be
                          parallelised) -- computed with an fp64 accumulator
* maxpool_forward ....... _kernels.pyx:133-166 best=-inf, strict '>' so the first
                          row-major tap wins ties; argmax = i*p + j (int32)
* maxpool_backward ...... _kernels.pyx:169-191 row-major scatter '+=' ==
                          per-input-pixel gather in DESCENDING tap order
* avgpool_forward ....... _kernels.pyx:194-221 acc=0, += taps row-major, / (p*p)
* avgpool_backward ...... _kernels.pyx:224-247 q = dy/(p*p), descending-tap gather

Arrays are C-contiguous (C, H, W) float32/float64, as at the reference boundary.
"""

from __future__ import annotations

import numpy as np


def _span(size_in: int, k: int, d: int) -> int:
    return size_in - ((k - 1) * d + 1) + 1


def conv_forward(x, w, b, dilation, threads=1):
    d = int(dilation)
    co, ci, l, _ = w.shape
    ho, wo = _span(x.shape[1], l, d), _span(x.shape[2], l, d)
    y = np.empty((co, ho, wo), dtype=x.dtype)
    y[...] = b.astype(x.dtype)[:, None, None]
    for c in range(ci):
        for i in range(l):
            rows = x[c, i * d:i * d + ho]
            for j in range(l):
                tap = rows[:, j * d:j * d + wo]
                y += w[:, c, i, j].astype(x.dtype)[:, None, None] * tap
    return y


def conv_backward_data(dy, w, dilation, threads=1):
    d = int(dilation)
    co, ci, l, _ = w.shape
    e = (l - 1) * d + 1
    ho, wo = dy.shape[1], dy.shape[2]
    hi, wi = ho + e - 1, wo + e - 1
    padded = np.zeros((co, ho + 2 * (e - 1), wo + 2 * (e - 1)), dtype=dy.dtype)
    padded[:, e - 1:e - 1 + ho, e - 1:e - 1 + wo] = dy
    dx = np.zeros((ci, hi, wi), dtype=dy.dtype)
    wt = w.astype(dy.dtype)
    for o in range(co):
        for i in range(l):
            for j in range(l):
                coeff = wt[o, :, l - 1 - i, l - 1 - j][:, None, None]
                dx += coeff * padded[o, i * d:i * d + hi, j * d:j * d + wi]
    return dx


def conv_backward_kernel(x, dy, kernel_size, dilation, threads=1, acc=np.float64):
    d, l = int(dilation), int(kernel_size)
    co, ho, wo = dy.shape
    ci = x.shape[0]
    dy2 = dy.reshape(co, ho * wo).astype(acc)
    dw = np.empty((co, ci, l, l), dtype=acc)
    for i in range(l):
        for j in range(l):
            win = x[:, i * d:i * d + ho, j * d:j * d + wo].reshape(ci, ho * wo).astype(acc)
            dw[:, :, i, j] = dy2 @ win.T
    db = dy2.sum(axis=1)
    return dw.astype(x.dtype), db.astype(x.dtype)


def maxpool_forward(x, p, dilation, threads=1):
    d, p = int(dilation), int(p)
    c = x.shape[0]
    ho, wo = _span(x.shape[1], p, d), _span(x.shape[2], p, d)
    best = np.full((c, ho, wo), -np.inf, dtype=x.dtype)
    arg = np.zeros((c, ho, wo), dtype=np.int32)
    for t in range(p * p):
        i, j = divmod(t, p)
        tap = x[:, i * d:i * d + ho, j * d:j * d + wo]
        win = tap > best
        best = np.where(win, tap, best)
        arg = np.where(win, np.int32(t), arg)
    return best, arg


def maxpool_backward(dy, arg, p, dilation, hi, wi, threads=1):
    d, p = int(dilation), int(p)
    c, ho, wo = dy.shape
    dx = np.zeros((c, hi, wi), dtype=dy.dtype)
    zero = np.zeros((), dtype=dy.dtype)
    for t in range(p * p - 1, -1, -1):
        i, j = divmod(t, p)
        dx[:, i * d:i * d + ho, j * d:j * d + wo] += np.where(arg == t, dy, zero)
    return dx


def avgpool_forward(x, p, dilation, threads=1):
    d, p = int(dilation), int(p)
    c = x.shape[0]
    ho, wo = _span(x.shape[1], p, d), _span(x.shape[2], p, d)
    acc = np.zeros((c, ho, wo), dtype=x.dtype)
    for t in range(p * p):
        i, j = divmod(t, p)
        acc = acc + x[:, i * d:i * d + ho, j * d:j * d + wo]
    return acc / x.dtype.type(p * p)


def avgpool_backward(dy, p, dilation, hi, wi, threads=1):
    d, p = int(dilation), int(p)
    c, ho, wo = dy.shape
    q = dy / dy.dtype.type(p * p)
    dx = np.zeros((c, hi, wi), dtype=dy.dtype)
    for t in range(p * p - 1, -1, -1):
        i, j = divmod(t, p)
        dx[:, i * d:i * d + ho, j * d:j * d + wo] += q
    return dx

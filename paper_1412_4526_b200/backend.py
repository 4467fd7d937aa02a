"""Kernel backend registry -- the drop-in plugin boundary.

Mirrors the reference's selector (backend.py:1-75): `available()`, `use(name)`,
`active()`, `kernels()`, `default_threads()`, env vars DENSEPROP_BACKEND and
DENSEPROP_THREADS.  This package registers "cuda" (`cuda_kernels`, the sm_100a C ABI's
exact tier: bit-identical to the compiled reference) and "cuda-fast" (`cuda_fast_kernels`:
the fp32 convolutions on the tcgen05 fast tier, within the 1e-4 normwise bound).  Unlike the reference there is no silent
CPU fallback: when libdenseprop_b200.so or a CUDA device is missing,
`kernels()` raises `KernelUnavailable` naming the cause.  Unknown names
(including "gpu", tests/test_backends.py:92-95) raise ValueError.

A user of the reference keeps its "compiled"/"python" backends and adds this
one instead; see INTEGRATION.md for the 10-line registration.
"""

from __future__ import annotations

import os
import warnings

from . import _lib, cuda_fast_kernels, cuda_kernels

_BACKENDS = {"cuda": cuda_kernels, "cuda-fast": cuda_fast_kernels}
_active: str | None = None
_why_unavailable: str | None = None


def _usable(name: str) -> bool:
    global _why_unavailable
    if not name.startswith("cuda"):
        return True
    try:
        _lib.require_device()
        return True
    except _lib.KernelUnavailable as exc:
        _why_unavailable = str(exc)
        return False


def registered() -> list[str]:
    return sorted(_BACKENDS)


def available() -> list[str]:
    return sorted(n for n in _BACKENDS if _usable(n))


def use(name: str) -> None:
    global _active
    name = (name or "").strip().lower()
    if name in ("auto", ""):
        name = "cuda"
    if name not in _BACKENDS:
        raise ValueError(f"unknown backend {name!r}; available: {registered()}")
    _active = name


def active() -> str | None:
    return _active


def kernels():
    if _active is None:
        raise _lib.KernelUnavailable("no kernel backend selected")
    if not _usable(_active):
        raise _lib.KernelUnavailable(f"backend {_active!r} unavailable: {_why_unavailable}")
    return _BACKENDS[_active]


def default_threads() -> int:
    raw = os.environ.get("DENSEPROP_THREADS", "").strip()
    if not raw:
        return 1
    try:
        return max(1, int(raw))
    except ValueError:
        warnings.warn(f"DENSEPROP_THREADS={raw!r} is not an integer; using 1", RuntimeWarning)
        return 1


_env = os.environ.get("DENSEPROP_BACKEND", "auto")
try:
    use(_env)
except ValueError:
    # a reference-era setting such as "compiled": this package only has "cuda"
    warnings.warn(f"DENSEPROP_BACKEND={_env!r} is not a backend of this package; using 'cuda'",
                  RuntimeWarning)
    use("cuda")

"""Loader for the reference's own compiled kernels built into oracle/_ref/.

Test infrastructure only (see oracle/__init__.py).  oracle/build_ref.sh compiles
/root/reference/pkg/src/denseprop/_kernels.pyx (the reference's compiled
backend, _kernels.pyx:23-247) into oracle/_ref/_kernels*.so; this module imports
that extension from its file path.  It exposes the same 7 functions as the
reference boundary and is what `bench.py --impl reference` times.
"""

from __future__ import annotations

import glob
import importlib.util
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(_HERE, "_ref")
_mod = None


def path() -> str | None:
    hits = sorted(glob.glob(os.path.join(REF_DIR, "_kernels*.so")))
    return hits[0] if hits else None


def available() -> bool:
    return path() is not None


def load():
    """Return the compiled reference kernel module (raises if not built)."""
    global _mod
    if _mod is None:
        p = path()
        if p is None:
            raise ImportError("oracle/_ref not built (run oracle/build_ref.sh)")
        spec = importlib.util.spec_from_file_location("_kernels", p)
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _mod = mod
    return _mod

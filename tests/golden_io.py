"""Helpers to read the committed golden fixtures (tests/golden/)."""

from __future__ import annotations

import functools
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=None)
def manifest():
    with open(os.path.join(GOLDEN, "manifest.json")) as fh:
        return json.load(fh)


@functools.lru_cache(maxsize=None)
def npz(kind: str, tag: str):
    with np.load(os.path.join(GOLDEN, f"{kind}_{tag}.npz")) as z:
        return {k: z[k] for k in z.files}


def net_names():
    return sorted(manifest()["nets"])


def conv_cases(tag):
    z = npz("kernels", tag)
    n = 0
    while f"conv{n}/meta" in z:
        yield {k.split("/", 1)[1]: v for k, v in z.items() if k.startswith(f"conv{n}/")}
        n += 1


def pool_cases(tag):
    z = npz("kernels", tag)
    n = 0
    while f"pool{n}/meta" in z:
        yield {k.split("/", 1)[1]: v for k, v in z.items() if k.startswith(f"pool{n}/")}
        n += 1


def net_case(name: str, tag: str):
    z = npz("nets", tag)
    pre = name + "/"
    return {k[len(pre):]: v for k, v in z.items() if k.startswith(pre)}


def rel_err(a, b) -> float:
    """Normwise relative error max|a-b| / max|b| (SURVEY.md 8(c) fast tier)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = float(np.max(np.abs(b))) if b.size else 0.0
    diff = float(np.max(np.abs(a - b))) if b.size else 0.0
    return diff / scale if scale > 0 else diff

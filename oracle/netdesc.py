"""Oracle-side network description (test infrastructure; see oracle/__init__.py).

Deliberately independent of the product's parser so a bug there cannot hide
behind a shared helper.  Restates:

* spec grammar + seeded weights ... reference netspec.py:9-18, 114-120, 180-250
* patch size / padding margins .... netspec.py:274-284, 320-323
* Alg. 1 dilation schedule ........ plan.py:80-105 (nonlin layers record the
  running d as well, plan.py:94-96)
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class OConv:
    w: np.ndarray        # (out, in, k, k) float64
    b: np.ndarray        # (out,) float64
    stride: int

    @property
    def k(self) -> int:
        return self.w.shape[2]


@dataclass
class OPool:
    kind: str            # "max" | "avg"
    k: int
    stride: int


@dataclass
class ONonlin:
    kind: str            # "tanh" | "relu" | "identity"


@dataclass
class ONet:
    in_channels: int
    layers: list = field(default_factory=list)

    # ---- receptive-field arithmetic (netspec.py:274-284, 320-323) ----
    def patch(self) -> int:
        n = 1
        for layer in self.layers[::-1]:
            if isinstance(layer, OConv):
                n = (n - 1) * layer.stride + layer.k
            elif isinstance(layer, OPool):
                n = (n - 1) * layer.stride + layer.k
        return n

    def margins(self) -> tuple[int, int]:
        n = self.patch()
        return n // 2, n - 1 - n // 2

    # ---- Alg. 1 (plan.py:80-105) ----
    def dilations(self) -> list[int]:
        out, d = [], 1
        for layer in self.layers:
            out.append(d)
            if isinstance(layer, (OConv, OPool)):
                d *= layer.stride
        return out

    @property
    def out_channels(self) -> int:
        c = self.in_channels
        for layer in self.layers:
            if isinstance(layer, OConv):
                c = layer.w.shape[0]
        return c


def seeded(out: int, inc: int, k: int, seed: int):
    """Weights then bias, U[-0.5, 0.5], numpy default_rng (netspec.py:114-120)."""
    g = np.random.default_rng(seed)
    return g.uniform(-0.5, 0.5, (out, inc, k, k)), g.uniform(-0.5, 0.5, out)


def read_spec(text: str) -> ONet:
    """Parse the spec grammar (seed: weights only -- all oracle cases are seeded)."""
    net = None
    for raw in text.splitlines():
        line = raw.split("#", 1)[0].split()
        if not line:
            continue
        kv = dict(tok.split("=", 1) for tok in line[1:])
        if line[0] == "input":
            net = ONet(int(kv["channels"]))
        elif line[0] == "conv":
            tok = kv["weights"]
            if not tok.startswith("seed:"):
                raise ValueError("oracle spec reader supports seed: weights only")
            w, b = seeded(int(kv["out"]), int(kv["in"]), int(kv["k"]), int(tok[5:]))
            net.layers.append(OConv(w, b, int(kv["stride"])))
        elif line[0] == "pool":
            net.layers.append(OPool(kv["kind"], int(kv["k"]), int(kv["stride"])))
        elif line[0] == "nonlin":
            net.layers.append(ONonlin(kv["kind"]))
        else:
            raise ValueError(f"unknown directive {line[0]!r}")
    return net

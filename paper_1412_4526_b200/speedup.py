"""Analytic redundancy model of the dense plan (reference bench.py:129-140).

Per conv layer, patch-by-patch scanning of an s x s image costs s^2 * m^2
window evaluations where the dense plan costs (s + m)^2, m being the patch
side entering that layer: speedup s^2 m^2 / (s + m)^2.
"""

from __future__ import annotations

from .netspec import ConvLayerSpec, NetworkSpec, layer_input_sizes


def theoretical_speedup(spec: NetworkSpec, image_side: int) -> dict:
    if image_side < 1:
        raise ValueError("image_side must be >= 1")
    sides = layer_input_sizes(spec)
    s = float(image_side)
    return {k: (s * s * sides[k] ** 2) / (s + sides[k]) ** 2
            for k, layer in enumerate(spec.layers) if isinstance(layer, ConvLayerSpec)}

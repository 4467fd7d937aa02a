"""Generate the golden fixtures under tests/golden/ from the REAL reference.

Run here (not on the GPU box -- /root/reference does not exist there):

    ./oracle/build_ref.sh && python tests/golden/make_golden.py

It imports the reference package from /root/reference/pkg/src with its
*compiled* backend: the Cython extension is the one oracle/build_ref.sh
compiled from the reference's own _kernels.pyx into oracle/_ref/, injected as
`denseprop._kernels` before `denseprop` is imported (the reference's
backend.py:20-23 then picks it up and `use("auto")` selects "compiled").

Outputs (committed):
  kernels_<dtype>.npz   per-kernel cases for the 7 boundary functions
  nets_<dtype>.npz      dense_forward / dense_backward cases on seeded specs
  manifest.json         spec texts, sides, seeds, plan metadata per case
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
REF_SRC = os.environ.get("REF_SRC", "/root/reference/pkg/src")


def _import_reference():
    from oracle import ref_kernels
    sys.modules["denseprop._kernels"] = ref_kernels.load()
    sys.path.insert(0, REF_SRC)
    import denseprop  # noqa: F401
    from denseprop import backend
    backend.use("compiled")
    assert backend.active() == "compiled"
    return denseprop


MIXED_NET = (
    "input channels=3\n"
    "conv out=4 in=3 k=3 stride=1 weights=seed:21\n"
    "pool kind=max k=2 stride=2\n"
    "nonlin kind=relu\n"
    "conv out=3 in=4 k=2 stride=1 weights=seed:22\n"
    "pool kind=avg k=2 stride=2\n"
    "nonlin kind=tanh\n"
    "conv out=2 in=3 k=3 stride=1 weights=seed:23\n"
)

# SURVEY.md Appendix A c1 (1 channel, patch 29) -- same net as c2 with in=1
C1_NET = (
    "input channels=1\n"
    "conv out=16 in=1 k=6 stride=1 weights=seed:1\n"
    "pool kind=max k=2 stride=2\n"
    "nonlin kind=tanh\n"
    "conv out=32 in=16 k=5 stride=1 weights=seed:2\n"
    "pool kind=max k=2 stride=2\n"
    "nonlin kind=tanh\n"
    "conv out=10 in=32 k=4 stride=1 weights=seed:3\n"
)

# c4-shaped chain (strided convs, relu) with small channel counts
STRIDED_NET = (
    "input channels=3\n"
    "conv out=6 in=3 k=5 stride=2 weights=seed:1\n"
    "nonlin kind=relu\n"
    "conv out=8 in=6 k=3 stride=1 weights=seed:2\n"
    "nonlin kind=relu\n"
    "pool kind=max k=2 stride=2\n"
    "conv out=8 in=8 k=3 stride=1 weights=seed:3\n"
    "nonlin kind=relu\n"
    "pool kind=max k=2 stride=2\n"
    "conv out=8 in=8 k=3 stride=2 weights=seed:4\n"
    "nonlin kind=relu\n"
    "pool kind=max k=2 stride=2\n"
    "conv out=4 in=8 k=3 stride=1 weights=seed:5\n"
)


def net_cases(dp):
    from denseprop import fixtures
    sys.path.insert(0, os.path.join(os.path.dirname(REF_SRC), "tests"))
    import specgen
    cases = [
        ("mixed", MIXED_NET, 13),
        ("example", fixtures.example_net_text(0), 7),
        ("plain_small", fixtures.plain_cnn1_text(3, channels=(4, 4, 2), pool1=(2, 2)), 9),
        ("plain69_small", fixtures.plain_cnn1_text(0, channels=(5, 6, 3), pool1=(4, 4)), 6),
        ("c1", C1_NET, 24),
        ("strided", STRIDED_NET, 10),
        ("even_patch", "input channels=1\nconv out=1 in=1 k=2 stride=1 weights=seed:3\n"
                       "nonlin kind=tanh\n", 4),
    ]
    for s in (1000, 1003, 1007, 1011, 1017, 1023):
        cases.append((f"rand{s}", specgen.random_spec_text(s), 9))
    return cases


def make_nets(dp, dtype, manifest):
    from denseprop import ErrorMask, compile_plan, dense_backward, dense_forward, parse_spec
    out = {}
    for ci, (name, text, side) in enumerate(net_cases(dp)):
        spec = parse_spec(text)
        plan = compile_plan(spec)
        rng = np.random.default_rng(9000 + ci)
        img = rng.uniform(-0.5, 0.5, (spec.input_channels, side, side)).astype(dtype)
        cache = dense_forward(plan, img)
        delta = rng.uniform(-1.0, 1.0, cache.output.shape).astype(dtype)
        npix = side * side
        flat = rng.choice(npix, size=min(5, npix), replace=False)
        pixels = sorted((int(f) // side, int(f) % side) for f in flat)
        masks = {"m5": ErrorMask.of(side, side, pixels), "all": ErrorMask.full(side, side)}
        key = f"{name}"
        out[f"{key}/image"] = img
        for k, x in enumerate(cache.inputs):
            out[f"{key}/in{k:02d}"] = x
        for k, a in cache.argmax.items():
            out[f"{key}/arg{k:02d}"] = a
        out[f"{key}/output"] = cache.output
        out[f"{key}/delta"] = delta
        for mname, mask in masks.items():
            out[f"{key}/mask_{mname}"] = mask._bool.copy()
            g = dense_backward(plan, cache, delta, mask, with_input_grad=True)
            for k, (kw, kb) in enumerate(zip(g.kernel, g.bias)):
                if kw is not None:
                    out[f"{key}/{mname}/dw{k:02d}"] = kw
                    out[f"{key}/{mname}/db{k:02d}"] = kb
            out[f"{key}/{mname}/input_delta"] = g.input_delta
        manifest["nets"][name] = {
            "spec": text, "side": side,
            "patch_size": plan.patch_size,
            "margins": [plan.lead_margin, plan.trail_margin],
            "dilations": plan.dilations,
            "extents": [getattr(l, "extent", None) for l in plan.layers],
            "argmax_layers": sorted(cache.argmax),
            "n_layers": len(plan.layers),
        }
    return out


KERNEL_SHAPES = [
    # (cin, cout, l, d, h, w)
    (3, 4, 3, 1, 12, 13),
    (2, 3, 2, 3, 11, 9),
    (1, 1, 1, 4, 6, 6),
    (4, 2, 3, 2, 5, 5),       # output 1x1
    (5, 7, 4, 2, 17, 15),
    (3, 5, 5, 1, 9, 30),
]
POOL_SHAPES = [
    # (c, p, d, h, w)
    (2, 2, 1, 9, 10),
    (3, 3, 2, 11, 12),
    (1, 4, 1, 8, 8),
    (2, 2, 3, 7, 9),
    (2, 1, 5, 4, 4),
    (1, 8, 1, 12, 12),
]


def make_kernels(dp, dtype):
    K = sys.modules["denseprop._kernels"]
    out = {}
    rng = np.random.default_rng(77 if dtype == np.float64 else 78)
    for n, (cin, cout, l, d, h, w) in enumerate(KERNEL_SHAPES):
        x = rng.uniform(-1, 1, (cin, h, w)).astype(dtype)
        wt = rng.uniform(-0.5, 0.5, (cout, cin, l, l)).astype(dtype)
        b = rng.uniform(-0.5, 0.5, cout).astype(dtype)
        y = K.conv_forward(x, wt, b, d, 1)
        dy = rng.uniform(-1, 1, y.shape).astype(dtype)
        dx = K.conv_backward_data(dy, wt, d, 1)
        dw, db = K.conv_backward_kernel(x, dy, l, d, 1)
        for nm, v in dict(x=x, w=wt, b=b, y=y, dy=dy, dx=dx, dw=dw, db=db).items():
            out[f"conv{n}/{nm}"] = v
        out[f"conv{n}/meta"] = np.array([cin, cout, l, d, h, w])
    for n, (c, p, d, h, w) in enumerate(POOL_SHAPES):
        x = rng.uniform(-1, 1, (c, h, w)).astype(dtype)
        if n == 2:       # exact ties everywhere: first tap must win
            x[:] = np.round(x * 2) / 2
        y, arg = K.maxpool_forward(x, p, d, 1)
        dy = rng.uniform(-1, 1, y.shape).astype(dtype)
        dxm = K.maxpool_backward(dy, arg, p, d, h, w, 1)
        ya = K.avgpool_forward(x, p, d, 1)
        dxa = K.avgpool_backward(dy, p, d, h, w, 1)
        for nm, v in dict(x=x, y=y, arg=arg, dy=dy, dxm=dxm, ya=ya, dxa=dxa).items():
            out[f"pool{n}/{nm}"] = v
        out[f"pool{n}/meta"] = np.array([c, p, d, h, w])
    return out


def main():
    dp = _import_reference()
    manifest = {"generator": "tests/golden/make_golden.py",
                "reference": "/root/reference/pkg (denseprop 0.1.0), compiled backend "
                             "built by oracle/build_ref.sh",
                "nets": {}}
    for dtype, tag in ((np.float32, "f32"), (np.float64, "f64")):
        np.savez_compressed(os.path.join(HERE, f"kernels_{tag}.npz"), **make_kernels(dp, dtype))
        np.savez_compressed(os.path.join(HERE, f"nets_{tag}.npz"), **make_nets(dp, dtype, manifest))
    with open(os.path.join(HERE, "manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=1, sort_keys=True)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()

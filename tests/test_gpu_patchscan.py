"""GPU patch-by-patch baseline: the ORIGINAL strided network on
batches of patches (paper_1412_4526_b200.patchscan), checked against the oracle's restatement
of the reference's patch scan (oracle/engine_np.py scan_forward / patch_backward_batch ->
reference oracle.py:145-164, 237-262) and against dense propagation.

* exact tier: scan_forward equal to the oracle's strided scan bit for bit on relu nets
  (fp32 and fp64; tanh nets to the 2-ulp tanh bound), including stride-2 convolutions,
  overlapping and average pools;
* patch_backward_batch: summed per-patch gradients vs the oracle (fp64 1e-12, fast tier
  fp32 1e-4 normwise), and equal to dense masked backward with the same pixels / deltas
  (the identity the paper's method rests on);
* errors: pixel outside the image, pixel / delta count mismatch.
"""

import numpy as np
import pytest

from golden_io import rel_err
from oracle import engine_np
from oracle.netdesc import read_spec

pytestmark = pytest.mark.gpu

NETS = {
    # conv stride 2 (subsample / zero-insert path), relu, max pool
    "strided": ("input channels=2\n"
                "conv out=3 in=2 k=3 stride=2 weights=seed:31\n"
                "nonlin kind=relu\n"
                "pool kind=max k=2 stride=2\n"
                "conv out=2 in=3 k=2 stride=1 weights=seed:32\n"),
    # overlapping avg pool (k=3, s=2) and a max pool, tanh
    "avg_overlap": ("input channels=3\n"
                    "conv out=4 in=3 k=2 stride=1 weights=seed:41\n"
                    "pool kind=avg k=3 stride=2\n"
                    "nonlin kind=tanh\n"
                    "conv out=5 in=4 k=2 stride=1 weights=seed:42\n"
                    "pool kind=max k=2 stride=2\n"
                    "nonlin kind=relu\n"
                    "conv out=3 in=5 k=2 stride=1 weights=seed:43\n"),
    # the c2 network (BASELINE configs[1])
    "c2": ("input channels=3\n"
           "conv out=16 in=3 k=6 stride=1 weights=seed:1\n"
           "pool kind=max k=2 stride=2\nnonlin kind=tanh\n"
           "conv out=32 in=16 k=5 stride=1 weights=seed:2\n"
           "pool kind=max k=2 stride=2\nnonlin kind=tanh\n"
           "conv out=10 in=32 k=4 stride=1 weights=seed:3\n"),
}


def _img(spec_c, side, dt, seed=0):
    return np.random.default_rng(seed).uniform(-0.5, 0.5, (spec_c, side, side)).astype(dt)


@pytest.mark.parametrize("name", sorted(NETS))
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_scan_forward_exact_vs_oracle(name, dt):
    import paper_1412_4526_b200 as dp
    text = NETS[name]
    spec = dp.parse_spec(text)
    side = 13
    img = _img(spec.input_channels, side, dt)
    got = dp.scan_forward(spec, img, precision="exact", batch=50)
    want = engine_np.scan_forward(read_spec(text), img)
    assert got.dtype == want.dtype and got.shape == want.shape
    if "tanh" in text:
        assert rel_err(got, want) < (1e-6 if dt == np.float32 else 1e-14)
    else:
        assert np.array_equal(got, want)


def test_scan_forward_pixel_subset_and_dense_equality():
    """Scanning a pixel subset fills just those pixels; the full scan equals dense forward
    bit for bit on the exact tier (dense == patch scan)."""
    import paper_1412_4526_b200 as dp
    text = NETS["c2"]
    spec = dp.parse_spec(text)
    img = _img(3, 24, np.float64, seed=2)
    pix = [(0, 0), (5, 17), (23, 23), (11, 3)]
    sub = dp.scan_forward(spec, img, pixels=pix, precision="exact")
    dense = dp.dense_forward(dp.compile_plan(spec), img).output
    mask = np.zeros(img.shape[1:], bool)
    for y, x in pix:
        mask[y, x] = True
    assert np.array_equal(sub[:, mask], dense[:, mask])
    assert not sub[:, ~mask].any()
    assert np.array_equal(dp.scan_forward(spec, img, precision="exact"), dense)


@pytest.mark.parametrize("name", sorted(NETS))
def test_patch_backward_batch_vs_oracle(name):
    import paper_1412_4526_b200 as dp
    text = NETS[name]
    spec = dp.parse_spec(text)
    net = read_spec(text)
    side = 12
    rng = np.random.default_rng(7)
    img = _img(spec.input_channels, side, np.float64, seed=3)
    flat = rng.choice(side * side, 30, replace=False)
    pix = [(int(i) // side, int(i) % side) for i in flat]
    deltas = rng.uniform(-1, 1, (len(pix), spec.output_channels))
    got = dp.patch_backward_batch(spec, img, pix, deltas, precision="exact", batch=7)
    kw, kb = engine_np.patch_backward_batch(net, img, pix, deltas)[:2]
    for k, _ in spec.conv_layers():
        assert rel_err(got.kernel[k], kw[k]) < 1e-12, k
        assert rel_err(got.bias[k], kb[k]) < 1e-12, k
    # fast tier, fp32
    got32 = dp.patch_backward_batch(spec, img.astype(np.float32), pix,
                                    deltas.astype(np.float32), precision="fast", batch=16)
    for k, _ in spec.conv_layers():
        assert rel_err(got32.kernel[k], kw[k]) < 1e-4, k
        assert rel_err(got32.bias[k], kb[k]) < 1e-4, k


def test_patch_backward_equals_dense_backward():
    """Dense masked backward over a pixel set == the sum of per-patch backward passes
    (the identity the dense method rests on; reference check.py / test_backward.py)."""
    import paper_1412_4526_b200 as dp
    from paper_1412_4526_b200.backward import ErrorMask, dense_backward
    text = NETS["c2"]
    spec = dp.parse_spec(text)
    plan = dp.compile_plan(spec)
    side = 20
    rng = np.random.default_rng(9)
    img = _img(3, side, np.float64, seed=5)
    cache = dp.dense_forward(plan, img)
    delta = rng.uniform(-1, 1, cache.output.shape)
    flat = rng.choice(side * side, 25, replace=False)
    pix = [(int(i) // side, int(i) % side) for i in flat]
    dense = dense_backward(plan, cache, delta, ErrorMask.of(side, side, pix))
    patch = dp.patch_backward_batch(spec, img, pix, [delta[:, y, x] for y, x in pix],
                                    precision="exact")
    for k, _ in spec.conv_layers():
        assert rel_err(patch.kernel[k], dense.kernel[k]) < 1e-12
        assert rel_err(patch.bias[k], dense.bias[k]) < 1e-12


def test_patch_scan_errors():
    import paper_1412_4526_b200 as dp
    spec = dp.parse_spec(NETS["strided"])
    img = _img(2, 8, np.float64)
    with pytest.raises(ValueError, match="outside"):
        dp.patch_backward_batch(spec, img, [(8, 0)], [np.zeros(2)])
    with pytest.raises(ValueError, match="delta vectors"):
        dp.patch_backward_batch(spec, img, [(1, 1), (2, 2)], [np.zeros(2)])
    with pytest.raises(ValueError, match="channels"):
        dp.scan_forward(spec, _img(3, 8, np.float64))
    assert not dp.patch_backward_batch(spec, img, [], []).max_abs()

"""Pin the CPU oracle to the reference's own outputs (tests/golden/, CPU only).

The oracle (numpy restatement and C/OpenMP port) must reproduce every golden
vector generated from the real reference with its compiled backend:
bit-exact for forward maps, argmax, conv data-gradients and pool backward,
and within reduction-order noise for the weight/bias gradients (the
reference sums 1e2-1e6 terms sequentially).
"""

import numpy as np
import pytest

from golden_io import conv_cases, manifest, net_case, net_names, pool_cases, rel_err
from oracle import engine_np, kernels_c, kernels_np
from oracle.netdesc import read_spec

TAGS = {"f32": np.float32, "f64": np.float64}
DW_TOL = {"f32": 1e-5, "f64": 1e-12}

KMODS = [pytest.param(kernels_np, id="numpy"), pytest.param(kernels_c, id="cport")]


@pytest.mark.parametrize("tag", TAGS)
@pytest.mark.parametrize("K", KMODS)
def test_conv_kernels_match_golden(K, tag):
    for case in conv_cases(tag):
        cin, cout, l, d, h, w = (int(v) for v in case["meta"])
        y = K.conv_forward(case["x"], case["w"], case["b"], d, 1)
        assert y.dtype == case["y"].dtype and np.array_equal(y, case["y"])
        dx = K.conv_backward_data(case["dy"], case["w"], d, 1)
        assert np.array_equal(dx, case["dx"])
        dw, db = K.conv_backward_kernel(case["x"], case["dy"], l, d, 1)
        assert dw.shape == (cout, cin, l, l) and db.shape == (cout,)
        assert rel_err(dw, case["dw"]) < DW_TOL[tag]
        assert rel_err(db, case["db"]) < DW_TOL[tag]


@pytest.mark.parametrize("tag", TAGS)
@pytest.mark.parametrize("K", KMODS)
def test_pool_kernels_match_golden(K, tag):
    for case in pool_cases(tag):
        c, p, d, h, w = (int(v) for v in case["meta"])
        y, arg = K.maxpool_forward(case["x"], p, d, 1)
        assert np.array_equal(y, case["y"])
        assert arg.dtype == np.int32 and np.array_equal(arg, case["arg"])
        assert np.array_equal(K.maxpool_backward(case["dy"], case["arg"], p, d, h, w, 1),
                              case["dxm"])
        assert np.array_equal(K.avgpool_forward(case["x"], p, d, 1), case["ya"])
        assert np.array_equal(K.avgpool_backward(case["dy"], p, d, h, w, 1), case["dxa"])


def test_cport_dw_is_bit_exact_with_reference():
    # the C port keeps the compiled backend's sequential (u, v) sum order
    for tag in TAGS:
        for case in conv_cases(tag):
            l, d = int(case["meta"][2]), int(case["meta"][3])
            dw, db = kernels_c.conv_backward_kernel(case["x"], case["dy"], l, d, 3)
            assert np.array_equal(dw, case["dw"]) and np.array_equal(db, case["db"])


@pytest.mark.parametrize("name", net_names())
def test_oracle_plan_metadata(name):
    meta = manifest()["nets"][name]
    net = read_spec(meta["spec"])
    assert net.patch() == meta["patch_size"]
    assert list(net.margins()) == meta["margins"]
    assert net.dilations() == meta["dilations"]


@pytest.mark.parametrize("tag", TAGS)
@pytest.mark.parametrize("name", net_names())
def test_oracle_engine_matches_golden(name, tag):
    meta = manifest()["nets"][name]
    g = net_case(name, tag)
    net = read_spec(meta["spec"])
    cache = engine_np.dense_forward(net, g["image"], kernels_c, threads=2)
    assert len(cache.inputs) == meta["n_layers"]
    for k, x in enumerate(cache.inputs):
        assert np.array_equal(x, g[f"in{k:02d}"]), f"layer {k} input"
    assert sorted(cache.argmax) == meta["argmax_layers"]
    for k, a in cache.argmax.items():
        assert np.array_equal(a, g[f"arg{k:02d}"])
    assert np.array_equal(cache.output, g["output"])
    for m in ("m5", "all"):
        kgr, bgr, inp = engine_np.dense_backward(net, cache, g["delta"], g[f"mask_{m}"],
                                                 kernels_c, threads=2, with_input_grad=True)
        for k in range(len(net.layers)):
            if kgr[k] is None:
                assert f"{m}/dw{k:02d}" not in g
                continue
            assert np.array_equal(kgr[k], g[f"{m}/dw{k:02d}"])
            assert np.array_equal(bgr[k], g[f"{m}/db{k:02d}"])
        assert np.array_equal(inp, g[f"{m}/input_delta"])


@pytest.mark.parametrize("name", ["mixed", "example", "plain_small", "even_patch", "rand1017"])
def test_dense_equals_patch_scan(name):
    """Paper claim: dense == patch-by-patch, exact in fp64."""
    meta = manifest()["nets"][name]
    g = net_case(name, "f64")
    net = read_spec(meta["spec"])
    scanned = engine_np.scan_forward(net, g["image"])
    assert np.array_equal(scanned, g["output"])
    side = meta["side"]
    pixels = [(y, x) for y in range(side) for x in range(side) if g["mask_m5"][y, x]]
    kgr, bgr = engine_np.patch_backward_batch(net, g["image"], pixels,
                                              [g["delta"][:, y, x] for y, x in pixels])
    for k in range(len(net.layers)):
        if kgr[k] is not None:
            assert np.max(np.abs(kgr[k] - g[f"m5/dw{k:02d}"])) < 1e-10
            assert np.max(np.abs(bgr[k] - g[f"m5/db{k:02d}"])) < 1e-10

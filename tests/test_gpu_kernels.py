"""Per-kernel parity of the sm_100a C ABI against the reference (GPU).

Every call goes through the host-pointer C ABI (cuda_kernels -> dp_host_*),
i.e. exactly what a reference backend module would bind.  Bar:
bit-exact for conv forward, conv data-gradient, max/avg pool forward and
backward and argmax; dw/db within reduction-order noise (fp32 normwise 1e-5
vs the golden, fp64 1e-12).  Golden vectors come from the real reference
(tests/golden/make_golden.py); bigger random shapes are checked against the
oracle's C port, which is pinned bit-exact to the reference in
tests/test_oracle_golden.py.
"""

import numpy as np
import pytest

from golden_io import conv_cases, pool_cases, rel_err
from oracle import kernels_c

pytestmark = pytest.mark.gpu

TAGS = {"f32": np.float32, "f64": np.float64}
DW_TOL = {"f32": 1e-5, "f64": 1e-12}


@pytest.fixture(scope="module")
def K():
    from paper_1412_4526_b200 import cuda_kernels
    return cuda_kernels


@pytest.mark.parametrize("tag", TAGS)
def test_conv_golden(K, tag):
    for case in conv_cases(tag):
        cin, cout, l, d, h, w = (int(v) for v in case["meta"])
        y = K.conv_forward(case["x"], case["w"], case["b"], d)
        assert y.dtype == case["y"].dtype and np.array_equal(y, case["y"]), case["meta"]
        dx = K.conv_backward_data(case["dy"], case["w"], d)
        assert np.array_equal(dx, case["dx"]), case["meta"]
        dw, db = K.conv_backward_kernel(case["x"], case["dy"], l, d)
        assert rel_err(dw, case["dw"]) < DW_TOL[tag]
        assert rel_err(db, case["db"]) < DW_TOL[tag]


@pytest.mark.parametrize("tag", TAGS)
def test_pool_golden(K, tag):
    for case in pool_cases(tag):
        c, p, d, h, w = (int(v) for v in case["meta"])
        y, arg = K.maxpool_forward(case["x"], p, d)
        assert np.array_equal(y, case["y"]) and arg.dtype == np.int32
        assert np.array_equal(arg, case["arg"]), case["meta"]
        assert np.array_equal(K.maxpool_backward(case["dy"], case["arg"], p, d, h, w),
                              case["dxm"])
        assert np.array_equal(K.avgpool_forward(case["x"], p, d), case["ya"])
        assert np.array_equal(K.avgpool_backward(case["dy"], p, d, h, w), case["dxa"])


CONV_SHAPES = [
    # cin, cout, k, d, h, w  -- paper/config-like layers, odd sizes, many tiles
    (3, 16, 6, 1, 70, 75),      # c2 conv1
    (16, 32, 5, 2, 60, 66),     # c2 conv2
    (32, 10, 4, 4, 61, 57),     # c2 conv3 (Cout not a multiple of 8)
    (8, 8, 7, 8, 70, 70),       # plain CNN1 FC head (k=7, d=8)
    (5, 20, 3, 16, 50, 40),     # large dilation
    (2, 3, 1, 5, 9, 9),         # 1x1 at any dilation
]


@pytest.mark.parametrize("shape", CONV_SHAPES)
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_conv_vs_cport(K, shape, dt):
    cin, cout, k, d, h, w = shape
    rng = np.random.default_rng(hash(shape) % 2**32)
    x = rng.uniform(-1, 1, (cin, h, w)).astype(dt)
    wt = rng.uniform(-0.5, 0.5, (cout, cin, k, k)).astype(dt)
    b = rng.uniform(-0.5, 0.5, cout).astype(dt)
    y = K.conv_forward(x, wt, b, d)
    assert np.array_equal(y, kernels_c.conv_forward(x, wt, b, d, 8))
    dy = rng.uniform(-1, 1, y.shape).astype(dt)
    assert np.array_equal(K.conv_backward_data(dy, wt, d), kernels_c.conv_backward_data(dy, wt, d, 8))
    dw, db = K.conv_backward_kernel(x, dy, k, d)
    # fp64 reference accumulation as the yardstick
    from oracle import kernels_np
    dw64, db64 = kernels_np.conv_backward_kernel(x.astype(np.float64), dy.astype(np.float64), k, d)
    tol = 1e-5 if dt == np.float32 else 1e-12
    assert rel_err(dw, dw64) < tol and rel_err(db, db64) < tol


POOL_SHAPES = [(4, 2, 1, 40, 41), (3, 3, 2, 33, 35), (2, 8, 1, 40, 40), (5, 2, 16, 60, 50),
               (1, 4, 4, 30, 31), (2, 1, 3, 7, 7),
               # several shared-memory tiles (128 x 32) per plane, halos up to 48, p <= 8
               (2, 4, 1, 150, 300), (2, 8, 1, 99, 270), (2, 5, 3, 90, 170), (3, 2, 4, 70, 290),
               (1, 7, 8, 80, 400), (1, 9, 1, 40, 50), (1, 3, 25, 60, 60),
               # d = 1, p = 3..8: the vectorised kernels (4-column groups, ragged tile edges)
               (2, 3, 1, 50, 77), (3, 5, 1, 45, 140), (2, 6, 1, 37, 131), (1, 7, 1, 70, 263),
               # output widths of 4k: the warp-streaming kernels (pool_stream.cu) forward and
               # backward, several 64-row items and column strips, halos 1..16
               (2, 4, 1, 150, 303), (2, 2, 4, 140, 264), (2, 2, 16, 90, 276),
               (2, 3, 8, 100, 272), (2, 4, 4, 80, 140), (2, 3, 1, 70, 130), (2, 2, 2, 66, 258),
               (2, 2, 8, 70, 136), (3, 4, 2, 67, 70), (2, 2, 1, 129, 253), (1, 4, 1, 200, 579)]


@pytest.mark.parametrize("shape", POOL_SHAPES)
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_pools_vs_cport(K, shape, dt):
    c, p, d, h, w = shape
    rng = np.random.default_rng(sum(shape))
    x = rng.uniform(-1, 1, (c, h, w)).astype(dt)
    x[:, ::3, ::2] = 0.25  # plenty of exact ties
    y, arg = K.maxpool_forward(x, p, d)
    y2, arg2 = kernels_c.maxpool_forward(x, p, d, 4)
    assert np.array_equal(y, y2) and np.array_equal(arg, arg2)
    dy = rng.uniform(-1, 1, y.shape).astype(dt)
    assert np.array_equal(K.maxpool_backward(dy, arg, p, d, h, w),
                          kernels_c.maxpool_backward(dy, arg, p, d, h, w, 4))
    # a bigger target map than needed: extra rows/cols receive zeros
    big = K.maxpool_backward(dy, arg, p, d, h + 2, w + 3)
    assert np.array_equal(big[:, :h, :w], kernels_c.maxpool_backward(dy, arg, p, d, h, w, 4))
    assert not big[:, h:, :].any() and not big[:, :, w:].any()
    assert np.array_equal(K.avgpool_forward(x, p, d), kernels_c.avgpool_forward(x, p, d, 4))
    assert np.array_equal(K.avgpool_backward(dy, p, d, h, w),
                          kernels_c.avgpool_backward(dy, p, d, h, w, 4))


@pytest.mark.parametrize("p,d", [(2, 1), (3, 1), (4, 1), (5, 1), (8, 1), (3, 5)])
def test_pool_nan_signed_zero(K, p, d):
    # NaN never wins (strict '>'), -0.0 / +0.0 ties keep the row-major first (the separable
    # shared-memory forward must pick exactly the reference's element)
    rng = np.random.default_rng(p * 10 + d)
    x = rng.choice(np.array([0.0, -0.0, 1.0, -1.0, np.nan], np.float32), size=(2, 60, 150))
    x[1, :20, :40] = np.nan
    y, arg = K.maxpool_forward(x, p, d)
    y2, arg2 = kernels_c.maxpool_forward(x, p, d, 4)
    assert np.array_equal(y.view(np.uint32), y2.view(np.uint32))
    assert np.array_equal(arg, arg2)
    dy = rng.uniform(-1, 1, y.shape).astype(np.float32)
    h, w = x.shape[1:]
    assert np.array_equal(K.maxpool_backward(dy, arg, p, d, h, w).view(np.uint32),
                          kernels_c.maxpool_backward(dy, arg, p, d, h, w, 4).view(np.uint32))


@pytest.mark.parametrize("p,d", [(2, 1), (4, 1), (2, 4), (3, 2), (2, 16)])
def test_pool_stream_nan_signed_zero(K, p, d):
    # the same special values through the warp-streaming kernels (output width 4k)
    rng = np.random.default_rng(p * 100 + d)
    w = 144 + (p - 1) * d
    x = rng.choice(np.array([0.0, -0.0, 1.0, -1.0, np.nan, np.inf, -np.inf], np.float32),
                   size=(2, 90, w))
    x[1, :20, :40] = np.nan
    y, arg = K.maxpool_forward(x, p, d)
    y2, arg2 = kernels_c.maxpool_forward(x, p, d, 4)
    assert np.array_equal(y.view(np.uint32), y2.view(np.uint32))
    assert np.array_equal(arg, arg2)
    dy = rng.choice(np.array([0.0, -0.0, 0.5, -0.25, 1e-30], np.float32), size=y.shape)
    h = x.shape[1]
    assert np.array_equal(K.maxpool_backward(dy, arg, p, d, h, w).view(np.uint32),
                          kernels_c.maxpool_backward(dy, arg, p, d, h, w, 4).view(np.uint32))


def test_maxpool_special_values(K):
    x = np.full((1, 4, 4), -np.inf, dtype=np.float32)
    y, arg = K.maxpool_forward(x, 2, 1)
    assert np.all(y == -np.inf) and not arg.any()          # -inf start, nothing beats it
    x = np.zeros((1, 3, 3), dtype=np.float64)
    x[0, 1, 1] = 5.0
    y, arg = K.maxpool_forward(x, 2, 1)
    dx = K.maxpool_backward(np.ones_like(y), arg, 2, 1, 3, 3)
    assert dx[0, 1, 1] == 4.0 and dx.sum() == 4.0          # overlap accumulates


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_nonlin(K, dt):
    rng = np.random.default_rng(5)
    x = rng.normal(size=(3, 17, 19)).astype(dt)
    x[0, 0, :4] = [0.0, -0.0, 1e-30, -1e-30]
    r = K.nonlin_forward(x, "relu")
    assert np.array_equal(r, np.maximum(x, 0))
    assert np.array_equal(np.signbit(r), np.signbit(np.maximum(x, 0)))
    t = K.nonlin_forward(x, "tanh")
    ref = np.tanh(x)
    assert np.all(np.abs(t - ref) <= 2 * np.spacing(np.abs(ref)))   # <= 2 ulp of numpy
    assert K.nonlin_forward(x, "identity") is x
    dy = rng.normal(size=x.shape).astype(dt)
    assert np.array_equal(K.nonlin_backward(dy, x, "relu"), dy * (x > 0))
    tb = K.nonlin_backward(dy, x, "tanh")
    th = np.tanh(x)
    assert rel_err(tb, dy * (1.0 - th * th)) < (1e-6 if dt == np.float32 else 1e-15)
    assert np.array_equal(K.nonlin_backward(dy, np.zeros_like(x), "tanh"), dy)


def test_errors(K):
    x = np.zeros((1, 4, 4), dtype=np.float32)
    w = np.zeros((1, 1, 3, 3), dtype=np.float32)
    b = np.zeros(1, dtype=np.float32)
    with pytest.raises(ValueError, match="smaller"):
        K.conv_forward(x, w, b, 2)
    with pytest.raises(TypeError):
        K.conv_forward(x.astype(np.int32), w, b, 1)
    with pytest.raises(ValueError):
        K.maxpool_forward(x, 5, 1)
    with pytest.raises(ValueError):
        K.maxpool_backward(np.zeros((1, 3, 3), np.float32), np.zeros((1, 3, 3), np.int32),
                           2, 1, 3, 3)
    with pytest.raises(ValueError):
        K.conv_backward_kernel(x, np.zeros((1, 3, 3), np.float32), 3, 1)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_sgd_update_matches_numpy(dt):
    """dp_sgd_update (the trainer's SGD step, DataParallelTrainer.step) is p - lr*g rounded
    exactly as numpy rounds it (one multiply, one subtract, no FMA contraction), in place,
    over a ragged length that is not a multiple of the grid stride."""
    import torch
    from paper_1412_4526_b200 import engine
    rng = np.random.default_rng(3)
    n = 148 * 256 * 3 + 17
    p = rng.standard_normal(n).astype(dt)
    g = rng.standard_normal(n).astype(dt)
    lr = 0.0123
    pt, gt = torch.from_numpy(p).cuda(), torch.from_numpy(g).cuda()
    engine.ops.sgd(pt, gt, lr)
    want = p - dt(lr) * g
    assert np.array_equal(pt.cpu().numpy(), want)
    assert np.array_equal(gt.cpu().numpy(), g)


@pytest.mark.parametrize("act", [0, 1, 3])  # identity, tanh (fp64), tanh (fast)
@pytest.mark.parametrize("shape", [(2, 6, 4, 1, 70, 135), (2, 5, 2, 4, 66, 128),
                                   (1, 4, 8, 1, 80, 139), (2, 3, 3, 2, 40, 68)])
def test_pool_stream_fused_act_gate_pitch(shape, act, monkeypatch):
    """The engine-facing device pools (batched, fused nonlinearity, fused backward gate, pitched
    dx): the warp-streaming kernels are bit-identical to pool.cu's (DP_POOL_STREAM=0) -- the
    gate staged as 16-byte rows (aligned maps) and word by word otherwise."""
    import torch
    from paper_1412_4526_b200 import _lib
    from paper_1412_4526_b200.engine import ops
    n, c, p, d, h, w = shape
    e = (p - 1) * d + 1
    ho, wo = h - e + 1, w - e + 1
    g = torch.Generator(device="cuda").manual_seed(sum(shape) + act)
    x = torch.rand((n, c, h, w), device="cuda", generator=g) - 0.5
    x[:, :, ::3, ::2] = 0.125  # ties
    dy = torch.rand((n, c, ho, wo), device="cuda", generator=g) - 0.5
    gate = torch.tanh(torch.rand((n, c, h, w), device="cuda", generator=g) - 0.5)
    pitch = (w + 7) // 4 * 4
    out = {}
    for mode in ("smem", "stream"):
        if mode == "smem":
            monkeypatch.setenv("DP_POOL_STREAM", "0")
        else:
            monkeypatch.delenv("DP_POOL_STREAM", raising=False)
        y = torch.empty((n, c, ho, wo), device="cuda")
        arg = torch.empty((n, c, ho, wo), device="cuda", dtype=torch.uint8)
        ops.maxpool_forward(x, y, arg, p, d, act)
        dxs = torch.full((n, c, h, pitch), 7.0, device="cuda")
        dx = dxs[..., :w]
        ops.maxpool_backward(dy, arg, dx, p, d, gate, _lib.DP_TANH_FAST, dx_pitch=pitch)
        dx2 = torch.empty((n, c, h, w), device="cuda")
        ops.maxpool_backward(dy, arg, dx2, p, d)
        torch.cuda.synchronize()
        out[mode] = (y.clone(), arg.clone(), dxs.clone(), dx2.clone())
    for a, b in zip(out["smem"], out["stream"]):
        assert torch.equal(a.view(torch.int32) if a.dtype == torch.float32 else a,
                           b.view(torch.int32) if b.dtype == torch.float32 else b)

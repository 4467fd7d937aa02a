"""Fast tier: tcgen05 3xTF32 conv (forward and data gradient) vs the exact tier (GPU).

The exact CUDA-core kernels are bit-identical to the reference (test_gpu_kernels.py); run in
fp64 they are the yardstick here (the fp32 exact tier carries its own rounding: on the c3 head
at its real widths, K = 2450, fast-vs-fp32-exact differences reach 1.5e-4 after tanh).
Bound: the north-star 1e-4 normwise relative.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# normwise vs fp64 (north-star bound)
TOL = 1e-4

SHAPES = [
    # n, cin, cout, k, d, h, w
    (2, 3, 16, 6, 1, 70, 75),       # c2 conv1 (Cin=3 -> one zero-padded chunk of 8)
    (2, 16, 32, 5, 2, 62, 66),      # c2 conv2 (3-MMA mode, Npad=32)
    (2, 32, 10, 4, 4, 61, 57),      # c2 conv3 (stacked mode, Q=10 -> Npad=16)
    (1, 8, 8, 7, 8, 70, 71),        # FC head k=7 d=8
    (1, 5, 20, 3, 16, 50, 40),      # large dilation, Npad=32 with Q=20
    (3, 2, 3, 1, 5, 9, 9),          # 1x1 kernel, tiny image (MT clamps)
    (1, 48, 64, 3, 2, 40, 45),      # c4-like L2: R=48, Q=64 (acc 64 cols)
    (1, 12, 48, 5, 1, 33, 37),      # Npad=48
    (1, 16, 8, 3, 32, 80, 90),      # d=32: tap-row / tap-column halo layout
    (1, 8, 16, 7, 8, 60, 66),       # 7x7 FC-style head, d=8
    (4, 3, 16, 6, 1, 20, 23),       # tiny images: one M tile, several images per CTA
    (1, 50, 8, 7, 8, 96, 90),       # c3 head at its real widths (tap stride QS = 8, N = 64)
    (2, 16, 6, 4, 4, 50, 52),       # Q < 8, even l: QS = 8, N = 32 (8-column TMEM loads)
    (1, 24, 8, 2, 3, 40, 41),       # Q = 8, l = 2: N = 16
]


def _t(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _rel(a, b):
    a = a.double()
    b = b.double()
    return float((a - b).abs().max() / max(b.abs().max(), 1e-30))


@pytest.fixture
def force_env(monkeypatch):
    """Select a fallback kernel for one test through its (per-call) environment switch."""
    def _set(kernel):
        if kernel == "halo":
            monkeypatch.setenv("DP_TC_HALO", "1")    # halo-buffer / converter kernel
        elif kernel == "tmem":
            monkeypatch.setenv("DP_WG_TMEM", "1")    # TMEM-operand weight gradient
        elif kernel == "flat_packlast":
            monkeypatch.setenv("DP_TF_PACK_LAST", "1")  # tap-packed last channel chunk
        elif kernel.startswith("ss_j"):
            monkeypatch.setenv("DP_WG_J", kernel[4:])  # column-tap stacking factor J
    return _set


@pytest.mark.parametrize("fp16", [False, True])
@pytest.mark.parametrize("kernel", ["flat", "tap", "halo", "flat_packlast"])
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("act", [0, 1, 2])
def test_tc_forward_matches_exact(shape, act, kernel, fp16, force_env):
    """kernel="tap" passes the shape-aware workspace, which selects the tap-stacked kernel
    where it applies (else the flat one runs again); fp16: the input is declared in fp16
    range, selecting the fp16-split forward for inputs of >= 16 channels."""
    import torch
    from paper_1412_4526_b200.engine import ops
    n, ci, co, k, d, h, w = shape
    force_env(kernel)
    if not ops.fast_supported(ci, co, k, d):
        pytest.skip("weights exceed the tensor-core kernel's shared-memory budget")
    rng = np.random.default_rng(sum(shape) + act)
    x = _t(rng.uniform(-1, 1, (n, ci, h, w)).astype(np.float32))
    # weights scaled so pre-activations stay O(1) for long reductions (K = ci*k*k up to 2450):
    # a saturated tanh turns the normwise measure into a relative error of tiny outputs
    ws_ = min(1.0, 4.0 / np.sqrt(ci * k * k))
    wt = _t((rng.uniform(-0.5, 0.5, (co, ci, k, k)) * ws_).astype(np.float32))
    b = _t(rng.uniform(-0.5, 0.5, co).astype(np.float32))
    e = (k - 1) * d + 1
    y_ref = torch.empty((n, co, h - e + 1, w - e + 1), device="cuda", dtype=torch.float64)
    y = torch.full(y_ref.shape, float("nan"), device="cuda")
    ops.conv_forward(x.double(), wt.double(), b.double(), y_ref, k, d, act)
    nb = ops.fast_workspace(ci, co, k) if kernel != "tap" else ops.fwd_fast_workspace(x, co, k, d)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    ops.conv_forward_fast(x, wt, b, y, k, d, act, ws, fp16_range=fp16)
    torch.cuda.synchronize()
    assert torch.isfinite(y).all()
    assert _rel(y, y_ref) < TOL


@pytest.mark.parametrize("kernel", ["flat", "tap", "halo", "flat_packlast"])
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("gate_kind", [None, 1, 2])
def test_tc_backward_data_matches_exact(shape, gate_kind, kernel, force_env):
    import torch
    from paper_1412_4526_b200.engine import ops
    n, ci, co, k, d, h, w = shape
    force_env(kernel)
    if not ops.fast_supported(co, ci, k, d):
        pytest.skip("weights exceed the tensor-core kernel's shared-memory budget")
    rng = np.random.default_rng(sum(shape) + 7)
    e = (k - 1) * d + 1
    ho, wo = h - e + 1, w - e + 1
    dy = _t(rng.uniform(-1, 1, (n, co, ho, wo)).astype(np.float32))
    wt = _t(rng.uniform(-0.5, 0.5, (co, ci, k, k)).astype(np.float32))
    gate = None
    if gate_kind is not None:
        gate = _t(np.tanh(rng.normal(size=(n, ci, h, w))).astype(np.float32))
    dx_ref = torch.empty((n, ci, h, w), device="cuda", dtype=torch.float64)
    dx = torch.full(dx_ref.shape, float("nan"), device="cuda")
    ops.conv_backward_data(dy.double(), wt.double(), dx_ref, k, d,
                           None if gate is None else gate.double(), gate_kind or 0)
    nb = ops.fast_workspace(co, ci, k) if kernel != "tap" else ops.bwd_fast_workspace(dy, ci, k, d)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    ops.conv_backward_data_fast(dy, wt, dx, k, d, ws, gate, gate_kind or 0)
    torch.cuda.synchronize()
    assert torch.isfinite(dx).all()
    assert _rel(dx, dx_ref) < TOL


def test_tc_deterministic_and_large_batch():
    import torch
    from paper_1412_4526_b200.engine import ops
    rng = np.random.default_rng(3)
    x = _t(rng.uniform(-1, 1, (16, 16, 278, 278)).astype(np.float32))
    wt = _t(rng.uniform(-0.5, 0.5, (32, 16, 5, 5)).astype(np.float32))
    b = _t(rng.uniform(-0.5, 0.5, 32).astype(np.float32))
    y1 = torch.empty((16, 32, 270, 270), device="cuda")
    y2 = torch.empty_like(y1)
    yr = torch.empty_like(y1)
    ws = torch.empty(ops.fast_workspace(16, 32, 5), dtype=torch.uint8, device="cuda")
    ops.conv_forward_fast(x, wt, b, y1, 5, 2, 1, ws)
    ops.conv_forward_fast(x, wt, b, y2, 5, 2, 1, ws)
    ops.conv_forward(x, wt, b, yr, 5, 2, 1)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    assert _rel(y1, yr) < TOL


WGRAD_SHAPES = [
    # n, cin, cout, k, d, h, w   (x is (n, cin, h, w); dy is the valid-conv output size)
    (2, 3, 16, 6, 1, 70, 75),       # c2 conv1: Cin=3 -> Cpad 8, odd widths (row re-pitch)
    (2, 16, 32, 5, 2, 62, 66),      # c2 conv2: 4 tiles of 128 rows, Npad=32
    (2, 32, 10, 4, 4, 61, 57),      # c2 conv3: 512 rows, Npad=16
    (1, 48, 64, 3, 2, 40, 45),      # c4 L2-like: Cpad 48 (box 16), G=2 -> 2 tile groups
    (1, 96, 128, 3, 8, 50, 52),     # c4 L8-like: Npad=128, G=1, 7 tile groups
    (1, 128, 8, 3, 32, 70, 68),     # c4 head-like: large dilation, 9 tiles
    (3, 2, 3, 1, 5, 9, 9),          # 1x1 kernel, tiny image (fewer K blocks than SMs)
    (1, 12, 48, 5, 1, 33, 37),      # Npad=48 (G=3)
    (4, 16, 32, 5, 2, 140, 140),    # larger batch, aligned widths (no re-pitch)
]


@pytest.mark.parametrize("kernel", ["ss", "ss_j1", "ss_j2", "ss_j3", "ss_j4", "tmem"])
@pytest.mark.parametrize("shape", WGRAD_SHAPES)
def test_tc_weight_gradient_matches_fp64(shape, kernel, force_env):
    """kernel="ss": shared-memory-operand kernel (tc_wgrad_ss.cu, the default, column-tap
    stacking factor J from its cost model); "ss_jN": the same with J forced to N (where the
    plan allows it); "tmem": the TMEM-operand fallback (tc_wgrad.cu)."""
    force_env(kernel)
    import torch
    from paper_1412_4526_b200.engine import ops
    n, ci, co, k, d, h, w = shape
    x = _t(np.random.default_rng(sum(shape)).uniform(-1, 1, (n, ci, h, w)).astype(np.float32))
    e = (k - 1) * d + 1
    ho, wo = h - e + 1, w - e + 1
    if not ops.wgrad_fast_supported(x, co, k, d):
        pytest.skip("outside the tensor-core weight-gradient envelope")
    rng = np.random.default_rng(sum(shape) + 1)
    dy = _t(rng.uniform(-1, 1, (n, co, ho, wo)).astype(np.float32))
    # ground truth: the exact-tier kernel in fp64 on the same (fp32-valued) inputs
    dw64 = torch.empty((co, ci, k, k), dtype=torch.float64, device="cuda")
    db64 = torch.empty(co, dtype=torch.float64, device="cuda")
    ws64 = torch.empty(max(1, ops.wgrad_workspace(x.double(), co, k, d)), dtype=torch.uint8,
                       device="cuda")
    ops.conv_backward_kernel(x.double(), dy.double(), dw64, db64, k, d, ws64)
    dw = torch.full((co, ci, k, k), float("nan"), device="cuda")
    db = torch.full((co,), float("nan"), device="cuda")
    ws = torch.empty(ops.wgrad_fast_workspace(x, co, k, d), dtype=torch.uint8, device="cuda")
    ops.conv_backward_kernel_fast(x, dy, dw, db, k, d, ws)
    dw2, db2 = torch.empty_like(dw), torch.empty_like(db)
    ops.conv_backward_kernel_fast(x, dy, dw2, db2, k, d, ws)
    torch.cuda.synchronize()
    assert torch.isfinite(dw).all() and torch.isfinite(db).all()
    assert torch.equal(dw, dw2) and torch.equal(db, db2)   # deterministic split-K
    assert _rel(dw, dw64) < 1e-5, _rel(dw, dw64)
    assert _rel(db, db64) < 1e-5, _rel(db, db64)


@pytest.mark.parametrize("shape", [WGRAD_SHAPES[0], WGRAD_SHAPES[1], WGRAD_SHAPES[2]])
def test_tc_weight_gradient_split_prepare_staged(shape):
    """dp_conv_backward_kernel_fast_prepare (stage x) + _staged (the rest) on one workspace
    == the single call, bit for bit."""
    import torch
    from paper_1412_4526_b200.engine import ops
    n, ci, co, k, d, h, w = shape
    e = (k - 1) * d + 1
    rng = np.random.default_rng(3)
    x = _t(rng.uniform(-1, 1, (n, ci, h, w)).astype(np.float32))
    dy = _t(rng.uniform(-1, 1, (n, co, h - e + 1, w - e + 1)).astype(np.float32))
    nb = ops.wgrad_fast_workspace(x, co, k, d)
    ws1 = torch.empty(nb, dtype=torch.uint8, device="cuda")
    ws2 = torch.empty(nb, dtype=torch.uint8, device="cuda")
    dw1 = torch.empty((co, ci, k, k), device="cuda")
    db1 = torch.empty(co, device="cuda")
    dw2, db2 = torch.empty_like(dw1), torch.empty_like(db1)
    ops.conv_backward_kernel_fast(x, dy, dw1, db1, k, d, ws1)
    ops.conv_backward_kernel_fast_prepare(x, co, k, d, ws2)
    ops.conv_backward_kernel_fast_staged(x, dy, dw2, db2, k, d, ws2)
    torch.cuda.synchronize()
    assert torch.equal(dw1, dw2) and torch.equal(db1, db2)


DIRECT_SHAPES = [
    # n, cin, cout, k, d, h, w  -- tap offsets j*d multiples of 4 floats, W % 4 == 0
    (2, 32, 10, 4, 4, 61, 60),      # c2 conv3-like
    (2, 50, 50, 3, 4, 70, 72),      # c3 conv2 widths
    (1, 50, 8, 7, 8, 90, 96),       # c3 head widths (J = 7 column-tap stacking)
    (3, 16, 32, 3, 8, 45, 44),      # Ho % d != 0: a column phase runs past the image
]


@pytest.mark.parametrize("shape", DIRECT_SHAPES)
def test_tc_weight_gradient_x_in_place(shape):
    """dp_conv_backward_kernel_fast_ex with readable slack after x: x is read in place
    (5-D NCHW tensor map, no staged copy) -- bit-identical to the staged call (rows past an
    image's end are now TMA zero fill instead of the next image's rows; they meet zero dy
    either way)."""
    import torch
    from paper_1412_4526_b200.engine import ops
    n, ci, co, k, d, h, w = shape
    e = (k - 1) * d + 1
    rng = np.random.default_rng(sum(shape))
    slack = 64 * 1024
    buf = torch.zeros(n * ci * h * w + slack // 4, device="cuda")
    x = buf[:n * ci * h * w].view(n, ci, h, w)
    x.copy_(_t(rng.uniform(-1, 1, (n, ci, h, w)).astype(np.float32)))
    dy = _t(rng.uniform(-1, 1, (n, co, h - e + 1, w - e + 1)).astype(np.float32))
    if not ops.wgrad_fast_supported(x, co, k, d):
        pytest.skip("outside the tensor-core weight-gradient envelope")
    ws = torch.empty(ops.wgrad_fast_workspace(x, co, k, d), dtype=torch.uint8, device="cuda")
    out = {}
    for mode in ("staged", "direct"):
        dw = torch.full((co, ci, k, k), float("nan"), device="cuda")
        db = torch.full((co,), float("nan"), device="cuda")
        ops.conv_backward_kernel_fast(x, dy, dw, db, k, d, ws,
                                      x_slack=slack if mode == "direct" else 0)
        out[mode] = (dw, db)
    torch.cuda.synchronize()
    assert torch.isfinite(out["direct"][0]).all()
    assert torch.equal(out["direct"][0], out["staged"][0])
    assert torch.equal(out["direct"][1], out["staged"][1])


F16_WGRAD_SHAPES = [
    # n, cin, cout, k, d, h, w  -- tap offsets j*d multiples of 8 halves, W % 8 == 0
    (1, 50, 8, 7, 8, 90, 96),       # c3 head widths (J = 7 column-tap stacking)
    (2, 32, 16, 3, 8, 60, 64),
    (3, 16, 32, 3, 8, 45, 48),      # Ho % d != 0: a column phase runs past the image
    (2, 32, 10, 4, 8, 70, 72),      # Q = 10 -> Npad 16
    (2, 24, 48, 1, 3, 20, 24),      # 1x1 kernel
    (1, 8, 8, 2, 16, 50, 48),       # d = 16
    # two residues (tap offsets 0 / 4 mod 8 halves): one in-place box each
    (2, 50, 50, 3, 4, 70, 76),      # c3 conv2 widths, W % 8 = 4 (split rows padded to 80)
    (1, 32, 16, 7, 8, 60, 61),      # W odd
    (1, 16, 24, 5, 4, 60, 64),      # residues of 3 and 2 taps
    (2, 16, 16, 3, 12, 80, 88),     # d = 12: offsets 0, 12, 24
    (2, 8, 16, 2, 2, 40, 48),       # d = 2, two taps
]


def _f16_case(shape, seed):
    import torch
    from paper_1412_4526_b200.engine import SLACK_BYTES, _slack_empty, ops
    n, ci, co, k, d, h, w = shape
    e = (k - 1) * d + 1
    rng = np.random.default_rng(seed)
    kw = {"dtype": torch.float32, "device": "cuda"}
    x = _slack_empty((n, ci, h, w), kw)
    x.copy_(_t(np.tanh(rng.normal(size=(n, ci, h, w))).astype(np.float32)))
    dy = _t(rng.uniform(-1, 1, (n, co, h - e + 1, w - e + 1)).astype(np.float32))
    nb = ops.wgrad_f16_workspace(x, co, k, d)
    if not nb:
        pytest.skip("outside the fp16 weight-gradient envelope")
    kw16 = {"dtype": torch.float16, "device": "cuda"}
    wp = (w + 7) // 8 * 8  # 16-byte rows of halves
    shift = ops.wgrad_f16_shift(x, co, k, d)
    assert shift >= 0
    t = [_slack_empty((n, ci, h, wp), kw16) for _ in range(4 if shift else 2)]
    ops.split_f16(x, t[0], t[1], *(t[2:] + [shift] if shift else []))
    if shift:  # the second residue's copies: the padded arrays shifted left (flat)
        for a, s in ((t[0], t[2]), (t[1], t[3])):
            fa, fs = a.reshape(-1), s.reshape(-1)
            assert torch.equal(fs[:-shift], fa[shift:]) and not fs[-shift:].any()
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    xs = {"x_hi_s": t[2], "x_lo_s": t[3]} if shift else {}
    return x, t[0], t[1], dy, ws, SLACK_BYTES, xs


@pytest.mark.parametrize("scale", [1.0, 1e-3, 1e4])
@pytest.mark.parametrize("kernel", ["ss", "ss_j1", "ss_j2", "ss_j3", "ilv"])
@pytest.mark.parametrize("shape", F16_WGRAD_SHAPES)
def test_tc_weight_gradient_fp16_split(shape, kernel, scale, force_env, monkeypatch):
    """dp_conv_backward_kernel_fast_f16 (x pre-split by dp_split_f16, dy split on the device,
    kind::f16 offset-split MMAs) vs the fp64 exact tier: tighter than the tf32 kernel's bound
    (fp16's 11-bit hi), deterministic, at dy magnitudes across the guarded range.  Two-residue
    shapes (shifted copies) are opt-in in production (DP_WG_F16_RES2) and enabled here;
    kernel "ilv": the same layouts through interleaved taps + dy copies (DP_WG_F16_ILV)."""
    monkeypatch.setenv("DP_WG_F16_RES2", "1")
    if kernel == "ilv":
        monkeypatch.setenv("DP_WG_F16_ILV", "1")
        monkeypatch.delenv("DP_WG_F16_RES2")
    else:
        force_env(kernel)
    import torch
    from paper_1412_4526_b200.engine import ops
    n, ci, co, k, d, h, w = shape
    x, xh, xl, dy, ws, slack, xs = _f16_case(shape, sum(shape))
    dy = dy * scale
    assert torch.equal(xh[..., :w], x.half())
    assert torch.equal(xl[..., :w], ((x - xh[..., :w].float()) * 2048.0).half())
    assert not xh[..., w:].any() and not xl[..., w:].any()
    dw64 = torch.empty((co, ci, k, k), dtype=torch.float64, device="cuda")
    db64 = torch.empty(co, dtype=torch.float64, device="cuda")
    ws64 = torch.empty(max(1, ops.wgrad_workspace(x.double(), co, k, d)), dtype=torch.uint8,
                       device="cuda")
    ops.conv_backward_kernel(x.double(), dy.double(), dw64, db64, k, d, ws64)
    outs = []
    for _ in range(2):
        dw = torch.full((co, ci, k, k), float("nan"), device="cuda")
        db = torch.full((co,), float("nan"), device="cuda")
        ops.conv_backward_kernel_fast_f16(x, xh, xl, dy, dw, db, k, d, ws, slack, **xs)
        outs.append((dw, db))
    torch.cuda.synchronize()
    dw, db = outs[0]
    assert torch.isfinite(dw).all() and torch.isfinite(db).all()
    assert torch.equal(dw, outs[1][0]) and torch.equal(db, outs[1][1])
    assert _rel(dw, dw64) < 5e-6, _rel(dw, dw64)
    assert _rel(db, db64) < 5e-6, _rel(db, db64)


@pytest.mark.parametrize("bad", [4e4, float("inf")])
@pytest.mark.parametrize("shape", F16_WGRAD_SHAPES[:3] + F16_WGRAD_SHAPES[6:7])
def test_tc_weight_gradient_fp16_range_fallback(shape, bad, monkeypatch):
    """One dy element outside fp16's range (or not finite) trips the device flag: the fp16
    launches exit and the gated tf32 kernel runs -- bit-identical to calling it directly."""
    monkeypatch.setenv("DP_WG_F16_RES2", "1")
    import torch
    from paper_1412_4526_b200.engine import ops
    n, ci, co, k, d, h, w = shape
    x, xh, xl, dy, ws, slack, xs = _f16_case(shape, 7)
    dy[n - 1, co - 1, 1, 2] = bad
    dw = torch.full((co, ci, k, k), float("nan"), device="cuda")
    db = torch.full((co,), float("nan"), device="cuda")
    ops.conv_backward_kernel_fast_f16(x, xh, xl, dy, dw, db, k, d, ws, slack, **xs)
    ws32 = torch.empty(ops.wgrad_fast_workspace(x, co, k, d), dtype=torch.uint8, device="cuda")
    dw2, db2 = torch.empty_like(dw), torch.empty_like(db)
    ops.conv_backward_kernel_fast(x, dy, dw2, db2, k, d, ws32, x_slack=slack)
    torch.cuda.synchronize()
    if bad == 4e4:
        assert torch.isfinite(dw).all()
        assert torch.equal(dw, dw2) and torch.equal(db, db2)
    else:
        assert torch.equal(torch.isfinite(dw), torch.isfinite(dw2))
        assert torch.equal(torch.isfinite(db), torch.isfinite(db2))


@pytest.mark.parametrize("p,d", [(2, 1), (4, 1), (2, 2)])
def test_layer0_pitched_delta_path(p, d):
    """Layer 0's delta handed over with a 16-byte row pitch: the max-pool backward writes dx
    with row pitch P (gate still read at pitch W) and the weight gradient reads dy through
    that pitch in place -- both bit-identical to the contiguous path (which re-pitches dy)."""
    import torch
    from paper_1412_4526_b200 import _lib
    from paper_1412_4526_b200.engine import ops
    n, ci, co, k, kd, h, w = 2, 3, 50, 6, 1, 80, 86   # conv x (n, ci, h, w), d = 1
    e = (k - 1) * kd + 1
    ho, wo = h - e + 1, w - e + 1                        # conv output = pool input (81 wide)
    assert wo % 4
    rng = np.random.default_rng(p * 7 + d)
    x = _t(rng.uniform(-1, 1, (n, ci, h, w)).astype(np.float32))
    a = _t(rng.uniform(-1, 1, (n, co, ho, wo)).astype(np.float32))
    ep = (p - 1) * d + 1
    y = torch.empty((n, co, ho - ep + 1, wo - ep + 1), device="cuda")
    arg = torch.empty(y.shape, dtype=torch.uint8, device="cuda")
    ops.maxpool_forward(a, y, arg, p, d)
    g = _t(rng.uniform(-1, 1, y.shape).astype(np.float32))
    dx = torch.empty_like(a)
    ops.maxpool_backward(g, arg, dx, p, d)
    pp = (wo + 3) // 4 * 4
    buf = torch.full((n * co * ho * pp,), float("nan"), device="cuda")
    dxp = buf.as_strided((n, co, ho, wo), (co * ho * pp, ho * pp, pp, 1))
    ops.maxpool_backward(g, arg, dxp, p, d, dx_pitch=pp)
    assert torch.equal(dxp, dx)
    ws = torch.empty(ops.wgrad_fast_workspace(x, co, k, kd), dtype=torch.uint8, device="cuda")
    dw1, db1 = torch.empty((co, ci, k, k), device="cuda"), torch.empty(co, device="cuda")
    dw2, db2 = torch.empty_like(dw1), torch.empty_like(db1)
    ops.conv_backward_kernel_fast(x, dx, dw1, db1, k, kd, ws)
    ops.conv_backward_kernel_fast(x, dxp, dw2, db2, k, kd, ws, dy_pitch=pp)
    torch.cuda.synchronize()
    assert torch.equal(dw1, dw2) and torch.equal(db1, db2)


@pytest.mark.parametrize("scale", [1e-3, 1e-6, 1e3, 1e5])
def test_tc_backward_data_fp16_offset_split_range(scale):
    """The fp16 data gradient (offset split, lo' = RN((dy - hi) * 2^11), cross products in
    their own accumulator half) stays within the north-star bound for deltas far from 1 in
    magnitude -- where an unscaled fp16 lo would fall into subnormals; at 1e5 (beyond fp16's
    range) the relayout's range flag sends the layer to the tf32 fallback launch."""
    import torch
    from paper_1412_4526_b200.engine import ops
    n, ci, co, k, d, h, w = 2, 50, 50, 3, 4, 60, 64
    rng = np.random.default_rng(11)
    e = (k - 1) * d + 1
    dy = _t((rng.uniform(-1, 1, (n, co, h - e + 1, w - e + 1)) * scale).astype(np.float32))
    wt = _t((rng.uniform(-0.5, 0.5, (co, ci, k, k)) * 4.0 / np.sqrt(co * k * k))
            .astype(np.float32))
    ref = torch.empty((n, ci, h, w), device="cuda", dtype=torch.float64)
    ops.conv_backward_data(dy.double(), wt.double(), ref, k, d)
    dx = torch.full((n, ci, h, w), float("nan"), device="cuda")
    ws = torch.empty(ops.bwd_fast_workspace(dy, ci, k, d), dtype=torch.uint8, device="cuda")
    ops.conv_backward_data_fast(dy, wt, dx, k, d, ws)
    torch.cuda.synchronize()
    assert torch.isfinite(dx).all()
    assert _rel(dx, ref) < TOL


@pytest.mark.parametrize("scale", [1.0, 1e5])
@pytest.mark.parametrize("shape", [(2, 50, 50, 3, 4, 60, 64), (1, 50, 8, 7, 8, 90, 96)])
def test_tc_forward_fp16_range_fallback(shape, scale):
    """Inputs declared in fp16 range but exceeding it (1e5): the fp16-split forward's range
    flag makes its kernel exit and the paired tf32 launch compute the layer (flat and
    tap-stacked paths) -- results within the bound either way."""
    import torch
    from paper_1412_4526_b200.engine import ops
    n, ci, co, k, d, h, w = shape
    rng = np.random.default_rng(5)
    x = _t((rng.uniform(-1, 1, (n, ci, h, w)) * scale).astype(np.float32))
    wt = _t((rng.uniform(-0.5, 0.5, (co, ci, k, k)) * 4.0 / np.sqrt(ci * k * k)).astype(np.float32))
    b = _t(rng.uniform(-0.5, 0.5, co).astype(np.float32))
    e = (k - 1) * d + 1
    ref = torch.empty((n, co, h - e + 1, w - e + 1), device="cuda", dtype=torch.float64)
    ops.conv_forward(x.double(), wt.double(), b.double(), ref, k, d, 0)
    y = torch.full(ref.shape, float("nan"), device="cuda")
    ws = torch.empty(ops.fwd_fast_workspace(x, co, k, d), dtype=torch.uint8, device="cuda")
    ops.conv_forward_fast(x, wt, b, y, k, d, 0, ws, fp16_range=True)
    torch.cuda.synchronize()
    assert torch.isfinite(y).all()
    assert _rel(y, ref) < TOL


PACKED_FWD = [(2, 3, 16, 6, 1, 70, 75), (4, 3, 16, 6, 1, 20, 23), (1, 8, 8, 7, 8, 70, 71),
              (1, 5, 20, 3, 16, 50, 40), (3, 2, 3, 1, 5, 9, 9), (1, 8, 16, 7, 8, 60, 66),
              (1, 3, 50, 6, 1, 80, 90), (4, 1, 16, 6, 1, 40, 40)]
PACKED_BWD = [(1, 8, 8, 7, 8, 70, 71), (1, 50, 8, 7, 8, 96, 90), (2, 16, 6, 4, 4, 50, 52),
              (1, 24, 8, 2, 3, 40, 41), (1, 16, 8, 3, 32, 80, 90), (3, 2, 3, 1, 5, 9, 9)]


@pytest.mark.parametrize("scale", [1.0, 1e5])
@pytest.mark.parametrize("shape", PACKED_FWD)
def test_tc_forward_fp16_tap_packed(shape, scale, monkeypatch):
    """Inputs of <= 8 channels in the fp16 split (opt-in DP_TF_F16_PACK_FWD): 16 / R column
    taps per K step (slot t*R + c), TMA-fed from a packed relayout; 1e5 trips the range flag
    (tf32 fallback)."""
    import torch
    from paper_1412_4526_b200.engine import ops
    monkeypatch.setenv("DP_TF_F16_PACK_FWD", "1")
    n, ci, co, k, d, h, w = shape
    rng = np.random.default_rng(sum(shape))
    x = _t((rng.uniform(-1, 1, (n, ci, h, w)) * scale).astype(np.float32))
    wt = _t((rng.uniform(-0.5, 0.5, (co, ci, k, k)) * 4.0 / np.sqrt(ci * k * k)).astype(np.float32))
    b = _t(rng.uniform(-0.5, 0.5, co).astype(np.float32))
    e = (k - 1) * d + 1
    ref = torch.empty((n, co, h - e + 1, w - e + 1), device="cuda", dtype=torch.float64)
    ops.conv_forward(x.double(), wt.double(), b.double(), ref, k, d, 0)
    y = torch.full(ref.shape, float("nan"), device="cuda")
    ws = torch.empty(ops.fwd_fast_workspace(x, co, k, d), dtype=torch.uint8, device="cuda")
    ops.conv_forward_fast(x, wt, b, y, k, d, 0, ws, fp16_range=True)
    torch.cuda.synchronize()
    assert torch.isfinite(y).all()
    assert _rel(y, ref) < TOL


@pytest.mark.parametrize("scale", [1.0, 1e-4, 1e5])
@pytest.mark.parametrize("gate_kind", [None, 1])
@pytest.mark.parametrize("shape", PACKED_BWD)
def test_tc_backward_data_fp16_tap_packed(shape, gate_kind, scale):
    """Deltas of <= 8 channels: the offset-split fp16 data gradient on tap-packed records
    (c3's 8-channel head); 1e5 sends the layer to the tf32 fallback."""
    import torch
    from paper_1412_4526_b200.engine import ops
    n, ci, co, k, d, h, w = shape
    rng = np.random.default_rng(sum(shape) + 3)
    e = (k - 1) * d + 1
    dy = _t((rng.uniform(-1, 1, (n, co, h - e + 1, w - e + 1)) * scale).astype(np.float32))
    wt = _t((rng.uniform(-0.5, 0.5, (co, ci, k, k)) * 4.0 / np.sqrt(co * k * k))
            .astype(np.float32))
    gate = None
    if gate_kind is not None:
        gate = _t(np.tanh(rng.normal(size=(n, ci, h, w))).astype(np.float32))
    ref = torch.empty((n, ci, h, w), device="cuda", dtype=torch.float64)
    ops.conv_backward_data(dy.double(), wt.double(), ref, k, d,
                           None if gate is None else gate.double(), gate_kind or 0)
    dx = torch.full((n, ci, h, w), float("nan"), device="cuda")
    ws = torch.empty(ops.bwd_fast_workspace(dy, ci, k, d), dtype=torch.uint8, device="cuda")
    ops.conv_backward_data_fast(dy, wt, dx, k, d, ws, gate, gate_kind or 0)
    torch.cuda.synchronize()
    assert torch.isfinite(dx).all()
    assert _rel(dx, ref) < TOL


PACK_LAST = [(2, 50, 50, 3, 4, 60, 64), (1, 20, 16, 5, 2, 40, 44), (1, 24, 32, 3, 1, 33, 40),
             (1, 40, 8, 7, 8, 90, 96), (1, 66, 24, 2, 3, 30, 31), (2, 18, 10, 4, 4, 50, 52)]


@pytest.mark.parametrize("mode", ["fwd", "bwd"])
@pytest.mark.parametrize("shape", PACK_LAST)
def test_tc_fp16_pack_last_chunk(shape, mode):
    """fp16 split with a tap-packed LAST chunk (R = 16k + r, r <= 8: slot t*r + c holds channel
    16k + c at column tap t), next to the full 16-channel chunks -- forward (input declared in
    range) and the offset-split data gradient (deltas of R channels)."""
    import torch
    from paper_1412_4526_b200.engine import ops
    n, ci, co, k, d, h, w = shape
    rng = np.random.default_rng(sum(shape) + (0 if mode == "fwd" else 1))
    e = (k - 1) * d + 1
    if mode == "fwd":
        x = _t(rng.uniform(-1, 1, (n, ci, h, w)).astype(np.float32))
        wt = _t((rng.uniform(-0.5, 0.5, (co, ci, k, k)) * 4.0 / np.sqrt(ci * k * k))
                .astype(np.float32))
        b = _t(rng.uniform(-0.5, 0.5, co).astype(np.float32))
        ref = torch.empty((n, co, h - e + 1, w - e + 1), device="cuda", dtype=torch.float64)
        ops.conv_forward(x.double(), wt.double(), b.double(), ref, k, d, 0)
        y = torch.full(ref.shape, float("nan"), device="cuda")
        ws = torch.empty(ops.fwd_fast_workspace(x, co, k, d), dtype=torch.uint8, device="cuda")
        ops.conv_forward_fast(x, wt, b, y, k, d, 0, ws, fp16_range=True)
    else:  # deltas of ci channels flow back to co inputs: R = ci here
        dy = _t(rng.uniform(-1, 1, (n, ci, h - e + 1, w - e + 1)).astype(np.float32))
        wt = _t((rng.uniform(-0.5, 0.5, (ci, co, k, k)) * 4.0 / np.sqrt(ci * k * k))
                .astype(np.float32))
        ref = torch.empty((n, co, h, w), device="cuda", dtype=torch.float64)
        ops.conv_backward_data(dy.double(), wt.double(), ref, k, d)
        y = torch.full(ref.shape, float("nan"), device="cuda")
        ws = torch.empty(ops.bwd_fast_workspace(dy, co, k, d), dtype=torch.uint8, device="cuda")
        ops.conv_backward_data_fast(dy, wt, y, k, d, ws)
    torch.cuda.synchronize()
    assert torch.isfinite(y).all()
    assert _rel(y, ref) < TOL


@pytest.mark.parametrize("shape", [
    # n, c, h, w, p, d
    (2, 50, 70, 72, 2, 4),     # c3 pool2-like: warp-streaming kernel, split fused
    (1, 8, 61, 67, 2, 8),      # ragged width (pitch padded, scalar tail stores)
    (2, 5, 40, 45, 4, 1),      # p = 4 streaming
    (1, 6, 30, 33, 2, 1),      # p = 2, d = 1: pool.cu kernel + split pass
])
def test_maxpool_forward_split(shape):
    """dp_maxpool_forward_split: y and the argmax codes bit-identical to dp_maxpool_forward,
    the split equal to dp_split_f16 of y (fused or as a second pass), pad columns untouched."""
    import torch
    from paper_1412_4526_b200 import _lib
    from paper_1412_4526_b200.engine import ops
    n, c, h, w, p, d = shape
    e = (p - 1) * d + 1
    ho, wo = h - e + 1, w - e + 1
    rng = np.random.default_rng(sum(shape))
    x = _t(rng.normal(size=(n, c, h, w)).astype(np.float32))
    y1 = torch.empty((n, c, ho, wo), device="cuda")
    a1 = torch.empty((n, c, ho, wo), dtype=torch.uint8, device="cuda")
    ops.maxpool_forward(x, y1, a1, p, d, _lib.DP_TANH_FAST)
    wp = (wo + 7) // 8 * 8
    y2, a2 = torch.empty_like(y1), torch.empty_like(a1)
    kw16 = {"dtype": torch.float16, "device": "cuda"}
    hi = torch.full((n, c, ho, wp), 7.0, **kw16)
    lo = torch.full((n, c, ho, wp), 7.0, **kw16)
    ops.maxpool_forward_split(x, y2, a2, p, d, _lib.DP_TANH_FAST, hi, lo)
    hr, lr = torch.zeros_like(hi), torch.zeros_like(lo)
    ops.split_f16(y1, hr, lr)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2) and torch.equal(a1, a2)
    assert torch.equal(hi[..., :wo], hr[..., :wo]) and torch.equal(lo[..., :wo], lr[..., :wo])


def test_fp16_split_and_weight_gradient_errors():
    """The ABI-6 entry points fail loudly (DP_ERR_ARG -> ValueError) on bad layouts instead of
    computing garbage."""
    import torch
    from paper_1412_4526_b200.engine import SLACK_BYTES, _slack_zeros, ops
    x = torch.rand((1, 8, 40, 48), device="cuda")
    kw16 = {"dtype": torch.float16, "device": "cuda"}
    bad = torch.zeros((1, 8, 40, 50), **kw16)  # pitch 50: not a multiple of 8 halves
    with pytest.raises(ValueError, match="pitch"):
        ops.split_f16(x, bad, bad.clone())
    short = torch.zeros((1, 8, 40, 40), **kw16)  # pitch < width
    with pytest.raises(ValueError, match="pitch"):
        ops.split_f16(x, short, short.clone())
    # fp16 weight gradient: a workspace one byte short, then an unsupported dy pitch
    co, k, d = 16, 3, 8
    nb = ops.wgrad_f16_workspace(x, co, k, d)
    assert nb > 0
    xh, xl = _slack_zeros((1, 8, 40, 48), kw16), _slack_zeros((1, 8, 40, 48), kw16)
    ops.split_f16(x, xh, xl)
    dy = torch.rand((1, co, 40 - 16, 48 - 16), device="cuda")
    dw = torch.empty((co, 8, k, k), device="cuda")
    db = torch.empty((co,), device="cuda")
    ws = torch.empty(nb - 1, dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError, match="workspace"):
        ops.conv_backward_kernel_fast_f16(x, xh, xl, dy, dw, db, k, d, ws, SLACK_BYTES)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError, match="pitch"):
        ops.conv_backward_kernel_fast_f16(x, xh, xl, dy, dw, db, k, d, ws, SLACK_BYTES,
                                          dy_pitch=3)
    # and the good call still works after the errors
    ops.conv_backward_kernel_fast_f16(x, xh, xl, dy, dw, db, k, d, ws, SLACK_BYTES)
    torch.cuda.synchronize()
    assert torch.isfinite(dw).all()

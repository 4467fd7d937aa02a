"""Whole-network parity of the B200 path (GPU).

* drop-in `dense_forward` / `dense_backward` against the golden vectors of the
  real reference (tests/golden/): bit-exact maps/argmax/input-delta for
  relu/identity nets, toleranced where np.tanh's last bit or the weight-gradient
  reduction order enters;
* teacher-forced layers: each plan layer fed the reference's own layer input
  reproduces the reference's output and argmax bit-for-bit;
* the fused batched engine (DenseNet) against per-image oracle runs, the config
  networks at full size against the oracle C port, and size-independent
  properties (determinism, mask additivity) at the largest sizes;
* dense == patch-by-patch scan on small cases.
"""

import numpy as np
import pytest

from golden_io import manifest, net_case, net_names, rel_err
from oracle import engine_np, kernels_c
from oracle.netdesc import read_spec

pytestmark = pytest.mark.gpu

TAGS = {"f32": np.float32, "f64": np.float64}
# normwise tolerances (north star: fp32 rel err <= 1e-4)
FWD_TOL = {"f32": 1e-5, "f64": 1e-12}
GRAD_TOL = {"f32": 1e-4, "f64": 1e-10}


@pytest.fixture(scope="module")
def dp():
    import paper_1412_4526_b200 as dp
    return dp


def _has_tanh(spec):
    return any(getattr(l, "kind", None) == "tanh" for l in spec.layers)


@pytest.mark.parametrize("tag", TAGS)
@pytest.mark.parametrize("name", net_names())
def test_dropin_matches_reference(dp, name, tag):
    meta = manifest()["nets"][name]
    g = net_case(name, tag)
    spec = dp.parse_spec(meta["spec"])
    plan = dp.compile_plan(spec)
    cache = dp.dense_forward(plan, g["image"])
    exact = not _has_tanh(spec)
    assert len(cache.inputs) == meta["n_layers"]
    assert sorted(cache.argmax) == meta["argmax_layers"]
    for k, x in enumerate(cache.inputs):
        ref = g[f"in{k:02d}"]
        assert x.shape == ref.shape and x.dtype == ref.dtype
        if exact:
            assert np.array_equal(x, ref), f"layer {k} input"
        else:
            assert rel_err(x, ref) < FWD_TOL[tag], f"layer {k} input"
    if exact:
        for k, a in cache.argmax.items():
            assert np.array_equal(a, g[f"arg{k:02d}"])
        assert np.array_equal(cache.output, g["output"])
    else:
        assert rel_err(cache.output, g["output"]) < FWD_TOL[tag]
    for m in ("m5", "all"):
        mask = dp.ErrorMask.from_bitmap(g[f"mask_{m}"])
        grads = dp.dense_backward(plan, cache, g["delta"], mask, with_input_grad=True)
        for k in range(len(spec.layers)):
            if grads.kernel[k] is None:
                assert f"{m}/dw{k:02d}" not in g
                continue
            assert grads.kernel[k].dtype == g["delta"].dtype
            assert rel_err(grads.kernel[k], g[f"{m}/dw{k:02d}"]) < GRAD_TOL[tag]
            assert rel_err(grads.bias[k], g[f"{m}/db{k:02d}"]) < GRAD_TOL[tag]
        ref_in = g[f"{m}/input_delta"]
        if exact:
            assert np.array_equal(grads.input_delta, ref_in)
        else:
            assert rel_err(grads.input_delta, ref_in) < GRAD_TOL[tag]


@pytest.mark.parametrize("tag", TAGS)
@pytest.mark.parametrize("name", net_names())
def test_teacher_forced_layers_bit_exact(dp, name, tag):
    """Each layer fed the reference's own input: conv/pool outputs and argmax bit-exact."""
    from paper_1412_4526_b200.forward import run_plan_layer
    meta = manifest()["nets"][name]
    g = net_case(name, tag)
    plan = dp.compile_plan(dp.parse_spec(meta["spec"]))
    n = meta["n_layers"]
    for k, layer in enumerate(plan.layers):
        y, arg = run_plan_layer(plan, k, g[f"in{k:02d}"])
        ref = g[f"in{k + 1:02d}"] if k + 1 < n else g["output"]
        if getattr(layer, "kind", None) == "tanh":
            # within 2 ulp of numpy's tanh elementwise (each side is <= 1 ulp from exact)
            assert np.all(np.abs(y - ref) <= 2 * np.spacing(np.abs(ref)))
        else:
            assert np.array_equal(y, ref), f"layer {k}"
        if arg is not None:
            assert np.array_equal(arg, g[f"arg{k:02d}"])


@pytest.mark.parametrize("name", ["mixed", "example", "plain_small", "even_patch", "rand1017",
                                  "strided"])
def test_gpu_dense_equals_patch_scan(dp, name):
    meta = manifest()["nets"][name]
    g = net_case(name, "f64")
    plan = dp.compile_plan(dp.parse_spec(meta["spec"]))
    net = read_spec(meta["spec"])
    side = meta["side"]
    pixels = [(y, x) for y in range(side) for x in range(0, side, 3)]
    dense = dp.dense_forward(plan, g["image"]).output
    scanned = engine_np.scan_forward(net, g["image"], pixels)
    ys, xs = zip(*pixels)
    assert np.max(np.abs(dense[:, ys, xs] - scanned[:, ys, xs])) < 1e-13


def _c1_text(cin):
    return (f"input channels={cin}\n"
            f"conv out=16 in={cin} k=6 stride=1 weights=seed:1\n"
            "pool kind=max k=2 stride=2\nnonlin kind=tanh\n"
            "conv out=32 in=16 k=5 stride=1 weights=seed:2\n"
            "pool kind=max k=2 stride=2\nnonlin kind=tanh\n"
            "conv out=10 in=32 k=4 stride=1 weights=seed:3\n")


C4_TEXT = ("input channels=3\n"
           "conv out=48 in=3 k=5 stride=2 weights=seed:1\nnonlin kind=relu\n"
           "conv out=64 in=48 k=3 stride=1 weights=seed:2\nnonlin kind=relu\n"
           "pool kind=max k=2 stride=2\n"
           "conv out=96 in=64 k=3 stride=1 weights=seed:3\nnonlin kind=relu\n"
           "pool kind=max k=2 stride=2\n"
           "conv out=128 in=96 k=3 stride=2 weights=seed:4\nnonlin kind=relu\n"
           "pool kind=max k=2 stride=2\n"
           "conv out=8 in=128 k=3 stride=1 weights=seed:5\n")


def _fast_vs_exact_forced(dp, text, imgs, targets, masks, max_flips=None):
    """Fast tier vs exact tier on the same inputs with the exact tier's forward state
    (activations = nonlinearity gates, max-pool argmax maps) forced into the fast engine.

    3xTF32 convs differ from fp32 by ~1e-6, which flips the occasional near-tied max-pool
    window or near-zero relu input; each flip routes a whole delta
    elsewhere.  Forcing the forward state makes both backward passes see identical inputs,
    so every gradient must agree within 1e-4.  The exact tier itself is pinned to the
    oracle by the precision="exact" tests.  Returns (exact, fast) engines."""
    import torch
    from paper_1412_4526_b200.engine import DenseNet
    from paper_1412_4526_b200 import trainer
    spec = dp.parse_spec(text)
    plan = dp.compile_plan(spec)
    batch, _, h, w = imgs.shape
    tdt = torch.float32 if imgs.dtype == np.float32 else torch.float64
    engs = {}
    for prec in ("exact", "fast"):
        e = DenseNet(plan, batch, h, w, dtype=tdt, precision=prec)
        e.set_input(torch.from_numpy(imgs).cuda())
        e.forward()
        engs[prec] = e
    ex, fa = engs["exact"], engs["fast"]
    assert rel_err(fa.output.cpu().numpy(), ex.output.cpu().numpy()) < 5e-5
    flips = sum(int((ex.args[g] != fa.args[g]).sum()) for g in ex.args)
    total = sum(ex.args[g].numel() for g in ex.args)
    assert flips <= (max_flips if max_flips is not None else max(20, total // 100000)), (flips, total)
    for g in ex.args:
        fa.args[g].copy_(ex.args[g])
    for x_e, x_f in zip(ex.acts, fa.acts):
        x_f.copy_(x_e)
    for e in (ex, fa):
        e.target.copy_(torch.from_numpy(targets))
        e.mask.copy_(torch.from_numpy(masks))
        e.loss_delta()
        e.backward()
    torch.cuda.synchronize()
    gk_e, gb_e = trainer.unflatten(spec, ex.grad_flat.double().cpu().numpy())
    gk_f, gb_f = trainer.unflatten(spec, fa.grad_flat.double().cpu().numpy())
    for k in range(len(spec.layers)):
        if gk_e[k] is not None:
            assert rel_err(gk_f[k], gk_e[k]) < 1e-4, f"dw layer {k}"
            assert rel_err(gb_f[k], gb_e[k]) < 1e-4, f"db layer {k}"
    return ex, fa


def _engine_vs_oracle(dp, text, side, batch, dt, frac, seed=0, tol_f=None, tol_g=None,
                      precision="fast", oracle_f64=False):
    """Fused engine vs per-image oracle runs.  oracle_f64 evaluates the oracle in fp64
    (at large activations the fp32 reference's own sequential
    weight-gradient sums drift by ~1e-4, so fp64 is the yardstick there)."""
    import torch
    from paper_1412_4526_b200.engine import DenseNet
    spec = dp.parse_spec(text)
    plan = dp.compile_plan(spec)
    net = read_spec(text)
    rng = np.random.default_rng(seed)
    imgs = rng.uniform(-0.5, 0.5, (batch, spec.input_channels, side, side)).astype(dt)
    co = spec.output_channels
    targets = rng.uniform(-1, 1, (batch, co, side, side)).astype(dt)
    masks = np.zeros((batch, side, side), dtype=np.uint8)
    for b in range(batch):
        k = max(1, int(frac * side * side))
        flat = rng.choice(side * side, size=k, replace=False)
        masks[b].flat[flat] = 1
    tdt = torch.float32 if dt == np.float32 else torch.float64
    eng = DenseNet(plan, batch, side, side, dtype=tdt, precision=precision)
    if tol_f is None and precision == "fast" and dt == np.float32:
        tol_f = 5e-5  # 3xTF32 tensor-core convs: fp32 reassociation-level differences
    eng.set_input(torch.from_numpy(imgs).cuda())
    eng.target.copy_(torch.from_numpy(targets))
    eng.mask.copy_(torch.from_numpy(masks))
    eng.forward()
    eng.loss_delta()
    eng.backward()
    torch.cuda.synchronize()
    out = eng.output.cpu().numpy()
    from paper_1412_4526_b200 import trainer
    ks, bs = trainer.unflatten(spec, eng.grad_flat.cpu().numpy())
    acc_k = [None] * len(spec.layers)
    acc_b = [None] * len(spec.layers)
    # fp32 fast tier: gradients through the teacher-forced comparison with the exact tier
    forced = precision == "fast" and dt == np.float32 and tol_g is None
    for b in range(batch):
        odt = np.float64 if oracle_f64 else dt
        cache = engine_np.dense_forward(net, imgs[b].astype(odt), kernels_c, threads=8)
        assert rel_err(out[b], cache.output) < (tol_f or FWD_TOL["f32" if dt == np.float32 else "f64"])
        if forced:
            continue
        delta = (cache.output - targets[b].astype(odt)).astype(odt)
        kg, bg, _ = engine_np.dense_backward(net, cache, delta, masks[b].astype(bool), kernels_c,
                                             threads=8)
        for k in range(len(spec.layers)):
            if kg[k] is not None:
                acc_k[k] = kg[k].astype(np.float64) + (0 if acc_k[k] is None else acc_k[k])
                acc_b[k] = bg[k].astype(np.float64) + (0 if acc_b[k] is None else acc_b[k])
    if forced:
        _fast_vs_exact_forced(dp, text, imgs, targets, masks)
    for k in range(len(spec.layers)):
        if acc_k[k] is not None:
            tg = tol_g or GRAD_TOL["f32" if dt == np.float32 else "f64"]
            assert rel_err(ks[k], acc_k[k]) < tg, f"dw layer {k}"
            assert rel_err(bs[k], acc_b[k]) < tg, f"db layer {k}"
    return eng


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("precision", ["fast", "exact"])
def test_fused_engine_batch_small(dp, dt, precision):
    _engine_vs_oracle(dp, _c1_text(1), 40, 3, dt, 0.05, precision=precision)


def test_fused_engine_mixed_pools(dp):
    text = manifest()["nets"]["mixed"]["spec"]
    _engine_vs_oracle(dp, text, 33, 2, np.float64, 0.2)
    _engine_vs_oracle(dp, text, 33, 2, np.float32, 1.0)


def test_config_c2_full_size(dp):
    """c2: 3x256x256, forward + masked backward with 1% of pixels (BASELINE.json configs[1])."""
    eng = _engine_vs_oracle(dp, _c1_text(3), 256, 2, np.float32, 0.01)
    plan = eng.kernel_plan()
    assert all(v["forward"].startswith("tcgen05-") for v in plan.values())
    _engine_vs_oracle(dp, _c1_text(3), 256, 1, np.float32, 0.01, precision="exact")


def test_config_c4_reduced_side(dp):
    """c4 network (strided convs, relu) vs the fp64 oracle at side 160, exact tier.

    The exact tier reproduces the reference's fp32 arithmetic, so its max-pool argmax maps
    are the reference's.  (The fast tier is checked against it below: its 3xTF32 convs
    differ from fp32 by ~1e-6, which flips a handful of near-tied max-pool windows out of
    ~1.7e7 -- SURVEY.md 0 fact 5 -- and each flip moves a whole delta to another tap.)"""
    _engine_vs_oracle(dp, C4_TEXT, 160, 1, np.float32, 0.02, oracle_f64=True,
                      precision="exact")


def test_config_c4_fast_tier_teacher_forced(dp):
    """c4 at side 160: fast tier (tcgen05 3xTF32 forward, data and weight gradients) vs
    the exact tier.  Forward within 5e-5; argmax flips are rare.  With the exact tier's
    forward state (activations = relu gates, argmax maps) forced into the fast engine,
    the backward kernels see identical inputs and every gradient agrees within 1e-4.
    (Without it, near-zero relu inputs and near-tied max windows that the ~1e-6 3xTF32
    differences flip route whole deltas differently through the 12-layer net.)"""
    side = 160
    rng = np.random.default_rng(0)
    img = rng.uniform(-0.5, 0.5, (2, 3, side, side)).astype(np.float32)
    tgt = rng.uniform(-1, 1, (2, 8, side, side)).astype(np.float32)
    mask = (rng.random((2, side, side)) < 0.05).astype(np.uint8)
    _, fa = _fast_vs_exact_forced(dp, C4_TEXT, img, tgt, mask)
    assert any(v["weight_grad"] == "tcgen05-3xtf32" for v in fa.kernel_plan().values())


def test_config_c4_full_size_properties(dp):
    """c4 at 1024x1024: determinism and mask additivity (oracle too slow at this size)."""
    import torch
    from paper_1412_4526_b200.engine import DenseNet
    spec = dp.parse_spec(C4_TEXT)
    plan = dp.compile_plan(spec)
    side = 1024
    eng = DenseNet(plan, 1, side, side)
    rng = np.random.default_rng(3)
    img = torch.from_numpy(rng.uniform(-0.5, 0.5, (1, 3, side, side)).astype(np.float32)).cuda()
    eng.set_input(img)
    eng.target.copy_(torch.from_numpy(rng.uniform(-1, 1, (1, 8, side, side)).astype(np.float32)))
    a = np.zeros((1, side, side), np.uint8)
    b = np.zeros((1, side, side), np.uint8)
    a.flat[rng.choice(side * side, 5000, replace=False)] = 1
    b.flat[rng.choice(side * side, 5000, replace=False)] = 1
    b[a == 1] = 0
    grads = {}
    for name, m in (("a", a), ("b", b), ("ab", a | b), ("a2", a)):
        eng.mask.copy_(torch.from_numpy(m))
        eng.forward()
        eng.loss_delta()
        eng.backward()
        grads[name] = eng.grad_flat.double().cpu().numpy()
        if name == "a":
            out1 = eng.output.clone()
    torch.cuda.synchronize()
    assert np.array_equal(grads["a"], grads["a2"])                 # run-to-run bitwise
    assert torch.equal(out1, eng.output)
    assert rel_err(grads["a"] + grads["b"], grads["ab"]) < 1e-4    # linearity in the mask
    assert np.isfinite(grads["ab"]).all() and np.abs(grads["ab"]).max() > 0


def test_graph_capture_replays_same_step(dp):
    import torch
    from paper_1412_4526_b200.trainer import DataParallelTrainer
    spec = dp.parse_spec(_c1_text(3))
    plan = dp.compile_plan(spec)
    tr = DataParallelTrainer(plan, 2, 64, 64, lr=0.0, use_graph=True)
    rng = np.random.default_rng(1)
    imgs = torch.from_numpy(rng.uniform(-0.5, 0.5, (2, 3, 64, 64)).astype(np.float32)).cuda()
    tgts = torch.from_numpy(rng.uniform(-1, 1, (2, 10, 64, 64)).astype(np.float32)).cuda()
    masks = torch.from_numpy((rng.random((2, 64, 64)) < 0.3).astype(np.uint8)).cuda()
    tr.load_batch(imgs, tgts, masks)
    tr.net.forward()
    tr.net.loss_delta()
    tr.net.backward()
    eager = tr.net.grad_flat.clone()
    tr.step()
    tr.step()
    torch.cuda.synchronize()
    assert torch.equal(eager, tr.net.grad_flat)


def test_dropin_errors(dp):
    plan = dp.compile_plan(dp.parse_spec(manifest()["nets"]["example"]["spec"]))
    with pytest.raises(ValueError, match="channels"):
        dp.dense_forward(plan, np.zeros((2, 5, 5)))
    with pytest.raises(TypeError):
        dp.dense_forward(plan, np.zeros((1, 5, 5), dtype=np.int64))
    cache = dp.dense_forward(plan, np.zeros((1, 5, 5)))
    with pytest.raises(ValueError):
        dp.dense_backward(plan, cache, np.zeros((1, 4, 4)), dp.ErrorMask.full(5, 5))
    with pytest.raises(ValueError):
        dp.dense_backward(plan, cache, np.zeros((1, 5, 5)), dp.ErrorMask.full(4, 4))
    g = dp.dense_backward(plan, cache, np.ones((1, 5, 5)), dp.ErrorMask.of(5, 5, []))
    assert g.max_abs() == 0.0


def test_h2d_pipeline_matches_direct_steps(dp):
    """The double-buffered host->device feeder gives the same gradients as loading each
    batch synchronously (trainer.H2DPipeline, used by bench.py's e2e leg)."""
    import torch
    from paper_1412_4526_b200.trainer import DataParallelTrainer, H2DPipeline
    spec = dp.parse_spec(_c1_text(3))
    plan = dp.compile_plan(spec)
    side, B = 40, 2
    rng = np.random.default_rng(5)
    host = []
    for _ in range(3):
        imgs = torch.from_numpy(rng.uniform(-0.5, 0.5, (B, 3, side, side)).astype(np.float32))
        tgts = torch.from_numpy(rng.uniform(-1, 1, (B, 10, side, side)).astype(np.float32))
        masks = torch.from_numpy((rng.random((B, side, side)) < 0.1).astype(np.uint8))
        host.append(tuple(t.pin_memory() for t in (imgs, tgts, masks)))
    direct = DataParallelTrainer(plan, B, side, side, lr=1e-3, use_graph=False)
    ref = []
    for h in host:
        direct.load_batch(*(t.cuda() for t in h))
        direct.step()
        ref.append(direct.net.grad_flat.clone())
    piped = DataParallelTrainer(plan, B, side, side, lr=1e-3, use_graph=True)
    feed = H2DPipeline(piped, *(t.cuda() for t in host[0]))
    got = []
    feed.submit(*host[0])
    for s in range(3):
        if s + 1 < 3:
            feed.submit(*host[s + 1])
        feed.step()
        got.append(piped.net.grad_flat.clone())
    torch.cuda.synchronize()
    for a, b in zip(got, ref):
        assert torch.equal(a, b)


@pytest.mark.parametrize("precision", ["exact", "fast"])
def test_band_sharding_equals_full_image(dp, precision):
    """SURVEY.md 8(e) fallback (fewer images than ranks): the engine on each rank's
    output-row band + (patch - 1)-row halo (trainer.BandParallelTrainer), buckets summed as
    the all-reduce would, equals the full-image engine; band outputs tile its output map."""
    import torch
    from paper_1412_4526_b200 import trainer
    from paper_1412_4526_b200.engine import DenseNet
    text = _c1_text(3)
    spec = dp.parse_spec(text)
    plan = dp.compile_plan(spec)
    side, world = 48, 3
    dt = torch.float64 if precision == "exact" else torch.float32
    rng = np.random.default_rng(9)
    img = torch.from_numpy(rng.uniform(-0.5, 0.5, (1, 3, side, side))).to(dt).cuda()
    tgt = torch.from_numpy(rng.uniform(-1, 1, (1, 10, side, side))).to(dt).cuda()
    mask = torch.from_numpy((rng.random((1, side, side)) < 0.2).astype(np.uint8)).cuda()
    full = DenseNet(plan, 1, side, side, dtype=dt, precision=precision)
    full.set_input(img)
    full.target.copy_(tgt)
    full.mask.copy_(mask)
    full.forward()
    full.loss_delta()
    full.backward()
    total = torch.zeros_like(full.grad_flat)
    outs = []
    for r in range(world):
        t = trainer.BandParallelTrainer(plan, 1, side, side, rank=r, world=world, dtype=dt,
                                        precision=precision)
        t.load(full.x0, tgt, mask)
        t.step()
        total += t.net.grad_flat
        outs.append(t.net.output.clone())
    torch.cuda.synchronize()
    got_out = torch.cat(outs, dim=2)
    if precision == "exact":
        assert torch.equal(got_out, full.output)
        assert rel_err(total.cpu().numpy(), full.grad_flat.cpu().numpy()) < 1e-12
    else:
        assert rel_err(got_out.cpu().numpy(), full.output.cpu().numpy()) < 5e-5
        assert rel_err(total.cpu().numpy(), full.grad_flat.cpu().numpy()) < 1e-4


@pytest.mark.parametrize("precision", ["exact", "fast"])
def test_gpu_patch_scan_equals_dense(dp, precision):
    """the patch-by-patch baseline on the GPU (every pixel's window
    classified on its own, oracle.py scan_forward:145-164) equals dense evaluation --
    bit-identical on the exact tier, within the fast-tier tolerance otherwise."""
    import torch
    from paper_1412_4526_b200.engine import DenseNet
    plan = dp.compile_plan(dp.parse_spec(_c1_text(3)))
    side = 20
    dt = torch.float64 if precision == "exact" else torch.float32
    rng = np.random.default_rng(4)
    img = torch.from_numpy(rng.uniform(-0.5, 0.5, (2, 3, side, side))).to(dt).cuda()
    net = DenseNet(plan, 2, side, side, dtype=dt, train=False, precision=precision)
    net.set_input(img)
    net.forward()
    scan = dp.patch_scan_forward(plan, img, batch=96, precision=precision)
    torch.cuda.synchronize()
    if precision == "exact":
        assert torch.equal(scan, net.output)
    else:
        assert rel_err(scan.cpu().numpy(), net.output.cpu().numpy()) < 5e-5


@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_softmax_xent_delta_matches_autograd(dp, dtype):
    """SURVEY.md 8(f) item 4 (8-class labelling loss, not in the reference -- parity
    unpinned, checked against torch fp64): delta = d(sum of masked per-pixel cross-entropy) /
    d logits, per-pixel loss = -log softmax[label]; label 255 and mask 0 contribute nothing."""
    import torch
    from paper_1412_4526_b200.engine import ops
    dt = getattr(torch, dtype)
    g = torch.Generator().manual_seed(5)
    n, q, h, w = 2, 8, 17, 19
    logits = (torch.randn((n, q, h, w), generator=g, dtype=torch.float64) * 3).to(dt)
    labels = torch.randint(0, q, (n, h, w), generator=g, dtype=torch.uint8)
    labels[0, :3] = 255
    mask = (torch.rand((n, h, w), generator=g) < 0.7).to(torch.uint8)
    delta = torch.empty_like(logits).cuda()
    loss = torch.empty((n, h, w), dtype=dt).cuda()
    ops.softmax_xent(logits.cuda(), labels.cuda(), mask.cuda(), delta, loss)
    torch.cuda.synchronize()
    z = logits.double().clone().requires_grad_(True)
    on = (mask.bool() & (labels != 255))
    lab = labels.long().clamp(max=q - 1)
    lp = torch.log_softmax(z, dim=1)
    px = -lp.gather(1, lab[:, None]).squeeze(1) * on
    px.sum().backward()
    tol = 1e-12 if dtype == "float64" else 2e-6
    assert rel_err(delta.double().cpu().numpy(), z.grad.numpy()) < tol
    assert rel_err(loss.double().cpu().numpy(), px.detach().numpy()) < tol


def test_engine_step_with_softmax_xent(dp):
    """The fused engine trains with the cross-entropy delta (fast tier): one step runs and its
    gradient equals the exact tier's with the forward state forced (same protocol as above)."""
    import torch
    from paper_1412_4526_b200.engine import DenseNet
    from paper_1412_4526_b200 import trainer
    spec = dp.parse_spec(_c1_text(3))
    plan = dp.compile_plan(spec)
    side = 32
    rng = np.random.default_rng(2)
    img = torch.from_numpy(rng.uniform(-0.5, 0.5, (2, 3, side, side)).astype(np.float32)).cuda()
    labels = torch.from_numpy(rng.integers(0, 10, (2, side, side)).astype(np.uint8)).cuda()
    mask = torch.from_numpy((rng.random((2, side, side)) < 0.05).astype(np.uint8)).cuda()
    engs = {}
    for prec in ("exact", "fast"):
        e = DenseNet(plan, 2, side, side, precision=prec)
        e.set_input(img)
        e.forward()
        engs[prec] = e
    ex, fa = engs["exact"], engs["fast"]
    for gname in ex.args:
        fa.args[gname].copy_(ex.args[gname])
    for x_e, x_f in zip(ex.acts, fa.acts):
        x_f.copy_(x_e)
    for e in (ex, fa):
        e.mask.copy_(mask)
        e.loss_delta(labels=labels)
        e.backward()
    torch.cuda.synchronize()
    ke, be = trainer.unflatten(spec, ex.grad_flat.double().cpu().numpy())
    kf, bf = trainer.unflatten(spec, fa.grad_flat.double().cpu().numpy())
    for k in range(len(spec.layers)):
        if ke[k] is not None:
            assert np.abs(ke[k]).max() > 0
            assert rel_err(kf[k], ke[k]) < 1e-4
            assert rel_err(bf[k], be[k]) < 1e-4


_C3 = ("input channels=3\n"
       "conv out=50 in=3 k=6 stride=1 weights=seed:0\n"
       "pool kind=max k=4 stride=4\nnonlin kind=tanh\n"
       "conv out=50 in=50 k=3 stride=1 weights=seed:3\n"
       "pool kind=max k=2 stride=2\nnonlin kind=tanh\n"
       "conv out=8 in=50 k=7 stride=1 weights=seed:6\n")


@pytest.mark.parametrize("split", ["fused", "pass"])
@pytest.mark.parametrize("target_scale", [1.0, 1e6])
def test_engine_fp16_weight_gradient_and_its_guard(dp, monkeypatch, target_scale, split):
    """c3 widths (the head's weight gradient on the fp16 split, its input split in the pool2
    forward -- or by a separate split pass, DP_NO_SPLIT_FUSE) vs the same engine with
    DP_WG_F16=0 (3xTF32 weight gradients): within 1e-4 at ordinary deltas; with deltas beyond
    fp16's range the device flag sends that layer to its tf32 launches, which then give
    bit-identical gradients."""
    if split == "pass":
        monkeypatch.setenv("DP_NO_SPLIT_FUSE", "1")
    import torch
    from paper_1412_4526_b200.engine import DenseNet
    spec = dp.parse_spec(_C3)
    plan = dp.compile_plan(spec)
    side, batch = 96, 2
    rng = np.random.default_rng(5)
    imgs = torch.from_numpy(rng.uniform(-0.5, 0.5, (batch, 3, side, side)).astype(np.float32))
    tgt = torch.from_numpy((rng.uniform(-1, 1, (batch, 8, side, side)) * target_scale)
                           .astype(np.float32))
    grads, plans = {}, {}
    for mode in ("f16", "tf32"):
        if mode == "tf32":
            monkeypatch.setenv("DP_WG_F16", "0")
        e = DenseNet(plan, batch, side, side, dtype=torch.float32, precision="fast")
        e.set_input(imgs.cuda())
        e.forward()
        e.target.copy_(tgt)
        e.mask.fill_(1)
        e.loss_delta()
        e.backward()
        torch.cuda.synchronize()
        grads[mode] = e.grad_flat.clone()
        plans[mode] = e.kernel_plan()
    head = max(plans["f16"])
    assert plans["f16"][head]["weight_grad"] == "tcgen05-fp16x3-offset"
    assert plans["tf32"][head]["weight_grad"] == "tcgen05-3xtf32"
    g16, g32 = grads["f16"], grads["tf32"]
    assert torch.isfinite(g16).all()
    if target_scale > 1e5:
        assert torch.equal(g16, g32)
    else:
        assert rel_err(g16.double().cpu().numpy(), g32.double().cpu().numpy()) < 1e-4

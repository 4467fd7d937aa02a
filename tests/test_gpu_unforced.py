"""Un-forced end-to-end parity of the BENCHMARKED fast tier at the BASELINE configs (GPU).

The throughput engine exactly as bench.py runs it (precision="fast": tcgen05 split-product
convolutions, fused epilogues, 1-byte argmax maps, side-stream weight gradients) on
seeded inputs, compared with the fp64 oracle (oracle/kernels.c, pinned to the reference in
tests/test_oracle_golden.py) run through the reference's dense_forward / dense_backward
algorithm (forward.py:101-128, backward.py:185-223).  Nothing is teacher-forced: the fast
tier's own activations and argmax maps drive its backward pass.

Bar (BASELINE.json north star): per-tensor normwise max|d| / max|ref| <= 1e-4 for the
output score maps, every dw and every db -- except where the reference's own fp32 result
(the exact tier, bit-identical to it) also misses 1e-4 against fp64 because near-tied
max-pool windows and relu gates flip (measured: c4 at 2% mask); there the fast tier must be
within 3x of the reference's own error.  Argmax maps are bit-exact only where the pool
inputs are bit-identical; the number of windows whose argmax differs
from the exact tier (which reproduces the fp32 reference bit for bit) is reported per pool
layer and bounded.  Set DP_PARITY_LOG=<file> to append the measured numbers as JSON lines.
"""

import json
import os

import numpy as np
import pytest

from golden_io import rel_err
from oracle import engine_np, kernels_c
from oracle.netdesc import read_spec

pytestmark = pytest.mark.gpu

TOL = 1e-4

C2 = ("input channels=3\n"
      "conv out=16 in=3 k=6 stride=1 weights=seed:1\n"
      "pool kind=max k=2 stride=2\nnonlin kind=tanh\n"
      "conv out=32 in=16 k=5 stride=1 weights=seed:2\n"
      "pool kind=max k=2 stride=2\nnonlin kind=tanh\n"
      "conv out=10 in=32 k=4 stride=1 weights=seed:3\n")
# fixtures.plain_cnn1_text(channels=(50, 50, 8), pool1=(4, 4)) -- BASELINE configs[2]
C3 = ("input channels=3\n"
      "conv out=50 in=3 k=6 stride=1 weights=seed:0\n"
      "pool kind=max k=4 stride=4\nnonlin kind=tanh\n"
      "conv out=50 in=50 k=3 stride=1 weights=seed:3\n"
      "pool kind=max k=2 stride=2\nnonlin kind=tanh\n"
      "conv out=8 in=50 k=7 stride=1 weights=seed:6\n")
C4 = ("input channels=3\n"
      "conv out=48 in=3 k=5 stride=2 weights=seed:1\nnonlin kind=relu\n"
      "conv out=64 in=48 k=3 stride=1 weights=seed:2\nnonlin kind=relu\n"
      "pool kind=max k=2 stride=2\n"
      "conv out=96 in=64 k=3 stride=1 weights=seed:3\nnonlin kind=relu\n"
      "pool kind=max k=2 stride=2\n"
      "conv out=128 in=96 k=3 stride=2 weights=seed:4\nnonlin kind=relu\n"
      "pool kind=max k=2 stride=2\n"
      "conv out=8 in=128 k=3 stride=1 weights=seed:5\n")
# plain CNN1 with the paper's 8x8 first pool (patch 133) -- BASELINE configs[4] family
PLAIN8 = C3.replace("out=8 in=50 k=7", "out=32 in=50 k=7").replace("k=4 stride=4", "k=8 stride=8")
# the other configs[4] points: 2x2 first pool (patch 37) and the k = 2 first conv (patch 65)
PLAIN2 = C3.replace("out=8 in=50 k=7", "out=32 in=50 k=7").replace("k=4 stride=4", "k=2 stride=2")
PLAIN4_K2 = C3.replace("out=8 in=50 k=7", "out=32 in=50 k=7").replace("in=3 k=6", "in=3 k=2")


def _run(text, side, batch, frac, seed):
    import torch
    import paper_1412_4526_b200 as dp
    from paper_1412_4526_b200 import trainer
    from paper_1412_4526_b200.engine import DenseNet
    spec = dp.parse_spec(text)
    plan = dp.compile_plan(spec)
    net = read_spec(text)
    rng = np.random.default_rng(seed)
    imgs = rng.uniform(-0.5, 0.5, (batch, spec.input_channels, side, side)).astype(np.float32)
    targets = rng.uniform(-1, 1, (batch, spec.output_channels, side, side)).astype(np.float32)
    masks = np.ones((batch, side, side), np.uint8) if frac >= 1 else \
        (rng.random((batch, side, side)) < frac).astype(np.uint8)
    engs = {}
    for prec in ("fast", "exact"):
        e = DenseNet(plan, batch, side, side, precision=prec)
        e.set_input(torch.from_numpy(imgs).cuda())
        e.target.copy_(torch.from_numpy(targets))
        e.mask.copy_(torch.from_numpy(masks))
        e.forward()
        e.loss_delta()
        e.backward()
        engs[prec] = e
    torch.cuda.synchronize()
    fast, exact = engs["fast"], engs["exact"]
    assert all(v["forward"].startswith("tcgen05") for v in fast.kernel_plan().values())
    out = fast.output.cpu().numpy()
    ks, bs = trainer.unflatten(spec, fast.grad_flat.double().cpu().numpy())
    eks, ebs = trainer.unflatten(spec, exact.grad_flat.double().cpu().numpy())
    eout = exact.output.cpu().numpy()
    flips, fast_args = {}, {}
    for gi, a in fast.args.items():
        layer = fast.groups[gi].first
        flips[str(layer)] = {"differ": int((a != exact.args[gi]).sum()), "windows": int(a.numel())}
        fast_args[layer] = a.cpu().numpy().astype(np.int32)
    # fp64 oracle, image by image, gradients summed (backward.py:190-191): once with its own
    # argmax maps (un-forced truth) and once following the fast tier's routing decisions
    threads = os.cpu_count() or 1
    acc = {"truth": ([None] * len(spec.layers), [None] * len(spec.layers)),
           "routed": ([None] * len(spec.layers), [None] * len(spec.layers))}
    out_err = eout_err = 0.0
    for b in range(batch):
        cache = engine_np.dense_forward(net, imgs[b].astype(np.float64), kernels_c, threads)
        out_err = max(out_err, rel_err(out[b], cache.output))
        eout_err = max(eout_err, rel_err(eout[b], cache.output))
        delta = cache.output - targets[b].astype(np.float64)
        for name in acc:
            if name == "routed":
                cache.argmax = {k: np.ascontiguousarray(v[b]) for k, v in fast_args.items()}
            kg, bg, _ = engine_np.dense_backward(net, cache, delta, masks[b].astype(bool),
                                                 kernels_c, threads)
            ak, ab = acc[name]
            for k in range(len(spec.layers)):
                if kg[k] is not None:
                    ak[k] = kg[k] + (0 if ak[k] is None else ak[k])
                    ab[k] = bg[k] + (0 if ab[k] is None else ab[k])
    errs = {"output": out_err}
    exact_errs = {"output": eout_err}
    routed = {}
    tk, tb = acc["truth"]
    rk, rb = acc["routed"]
    for k in range(len(spec.layers)):
        if tk[k] is not None:
            errs[f"dw{k}"], errs[f"db{k}"] = rel_err(ks[k], tk[k]), rel_err(bs[k], tb[k])
            exact_errs[f"dw{k}"] = rel_err(eks[k], tk[k])
            exact_errs[f"db{k}"] = rel_err(ebs[k], tb[k])
            routed[f"dw{k}"], routed[f"db{k}"] = rel_err(ks[k], rk[k]), rel_err(bs[k], rb[k])
    rec = {"side": side, "batch": batch, "mask_fraction": frac,
           "normwise_fast_vs_fp64": errs,
           "normwise_exact_tier_vs_fp64": exact_errs,
           "normwise_fast_vs_fp64_on_fast_routing": routed,
           "argmax_vs_exact_tier": flips}
    print(json.dumps(rec))
    log = os.environ.get("DP_PARITY_LOG")
    if log:
        with open(log, "a") as fh:
            fh.write(json.dumps(rec) + "\n")
    return errs, exact_errs, routed, flips


def _check(errs, exact_errs, routed, flips, flip_frac=1e-4):
    """Fast tier vs the fp64 truth: <= 1e-4, or -- where the exact tier (the reference's own
    fp32 result, bit for bit) itself is not far below 1e-4 against fp64 -- no worse than 3x
    the reference's own error.  (Measured on c4 at a 2 % mask: the exact tier's dw0 is 2.6e-4
    off fp64, the fast tier's 4.4e-4; dw2 4.5e-5 vs 1.0e-4 -- near-tied max-pool windows and
    relu inputs near 0 change sign between fp32 and fp64, and a sparse mask leaves few pixels
    to average them out.)  `routed` (the fp64
    backward along the fast tier's own argmax choices) is reported, not bounded: the relu
    gates still flip there."""
    assert errs["output"] <= TOL
    for name, e in errs.items():
        assert e <= max(TOL, 3.0 * exact_errs[name]), (name, e, exact_errs[name])
    for layer, f in flips.items():
        assert f["differ"] <= max(50, flip_frac * f["windows"]), (layer, f)


def test_unforced_c2_256():
    """BASELINE configs[1]: c2, 3x256x256, 1%-masked backward, batch 2."""
    _check(*_run(C2, 256, 2, 0.01, seed=11))


def test_unforced_c3_512():
    """BASELINE configs[2] (the bench headline): c3 at its real 50/50/8 widths, 3x512x512,
    full-image forward + full-mask backward."""
    _check(*_run(C3, 512, 1, 1.0, seed=12))


def test_unforced_c4_512():
    """BASELINE configs[3] network (5 conv with strides 2,1,1,2,1, relu, 3 max-pools) at
    side 512, 2%-masked backward."""
    _check(*_run(C4, 512, 1, 0.02, seed=13))


def test_unforced_plain_p8_256():
    """BASELINE configs[4] family: plain CNN1 with the 8x8 first pool (patch 133)."""
    _check(*_run(PLAIN8, 256, 1, 1.0, seed=14))


def test_unforced_plain_p2_256():
    """BASELINE configs[4] family: plain CNN1 with the 2x2 first pool (patch 37)."""
    _check(*_run(PLAIN2, 256, 1, 1.0, seed=15))


def test_unforced_plain_p4_k2_256():
    """BASELINE configs[4] family: plain CNN1 with a 2x2 first convolution (patch 65)."""
    _check(*_run(PLAIN4_K2, 256, 1, 1.0, seed=16))

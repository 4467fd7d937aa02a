"""Benchmark: classified pixels/s of dense fwd + masked bwd on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one process per GPU, NCCL)

Workload of the headline line (N=1): BASELINE.json configs[2] = "c3": the scene-labelling
Plain CNN1 of the reference's fixtures (`fixtures.plain_cnn1_text(channels=(50, 50, 8),
pool1=(4, 4))`: conv6(3->50)/maxpool4/tanh/conv3(50->50)/maxpool2/tanh/conv7(50->8),
patch 69, 8 classes) on 3x512x512 synthetic RGB images, full-image forward + backward
(every pixel in the error mask), squared-error delta against a synthetic target map
(cli.py:218), gradients summed per image, one NCCL all-reduce(SUM) of the gradient bucket
per step when N > 1, and a plain SGD update.  A "step" = one such training pass over a
batch of B images per GPU (weak scaling: per-GPU work fixed).

value  = whole-job training throughput, images*h*w / time over all ranks, inputs already
         resident in HBM (device-timed, CUDA events, max over ranks)
e2e    = the same through the public trainer API from pinned HOST buffers: per step H2D of
         images + targets + masks and D2H of the gradient bucket
forward = forward-only inference throughput (no collective); forward.e2e adds the H2D of
         the images and the D2H of the score maps
roofline = the dominant kernel of the step, timed per launch with CUDA events
cpu_baseline = the UNMODIFIED reference package (baseline/_ref) through its own API
         (dense_forward + dense_backward, compiled backend) on the host cores, one image of
         the same config (all threads), plus a 1-thread band sample and the patch-by-patch
         scan on sampled pixels (rank 0, N=1 only)
lines  = the other BASELINE configs (c1 fwd-only, c2, c4) on the same GPU, each with a
         sampled CPU reference beside it;  sizes = the c5 image/patch-size sweep.

`--impl reference` times the reference's CPU path alone (c3@512, one image per step) as the
driver's reference arm.
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "classified pixels/sec fwd and fwd+bwd per image size at 1/2/4/8 B200 vs CPU"


def plain_cnn1_text(channels=(50, 50, 32), pool1=2, k1=6, in_channels=3, seed=0):
    """The reference's fixtures.plain_cnn1_text (fixtures.py:45-63), with conv1 k=2 variants
    (SURVEY.md Appendix A): pool1 p -> patch 37 / 69 / 133 (k1 = 6) or 33 / 65 / 129 (k1 = 2)."""
    c1, c2, c3 = channels
    s = lambda k: f"seed:{seed * 10000 + k}"  # noqa: E731  (fixtures._seed_token)
    return (f"input channels={in_channels}\n"
            f"conv out={c1} in={in_channels} k={k1} stride=1 weights={s(0)}\n"
            f"pool kind=max k={pool1} stride={pool1}\nnonlin kind=tanh\n"
            f"conv out={c2} in={c1} k=3 stride=1 weights={s(3)}\n"
            "pool kind=max k=2 stride=2\nnonlin kind=tanh\n"
            f"conv out={c3} in={c2} k=7 stride=1 weights={s(6)}\n")


C1_TEXT = ("input channels=1\n"
           "conv out=16 in=1 k=6 stride=1 weights=seed:1\n"
           "pool kind=max k=2 stride=2\nnonlin kind=tanh\n"
           "conv out=32 in=16 k=5 stride=1 weights=seed:2\n"
           "pool kind=max k=2 stride=2\nnonlin kind=tanh\n"
           "conv out=10 in=32 k=4 stride=1 weights=seed:3\n")
C2_TEXT = C1_TEXT.replace("input channels=1", "input channels=3").replace(
    "conv out=16 in=1", "conv out=16 in=3")
# BASELINE.json configs[2] / configs[3]
C3_TEXT = plain_cnn1_text(channels=(50, 50, 8), pool1=4)
C4_TEXT = ("input channels=3\n"
           "conv out=48 in=3 k=5 stride=2 weights=seed:1\nnonlin kind=relu\n"
           "conv out=64 in=48 k=3 stride=1 weights=seed:2\nnonlin kind=relu\n"
           "pool kind=max k=2 stride=2\n"
           "conv out=96 in=64 k=3 stride=1 weights=seed:3\nnonlin kind=relu\n"
           "pool kind=max k=2 stride=2\n"
           "conv out=128 in=96 k=3 stride=2 weights=seed:4\nnonlin kind=relu\n"
           "pool kind=max k=2 stride=2\n"
           "conv out=8 in=128 k=3 stride=1 weights=seed:5\n")

# name -> (spec text, side, images per GPU per step, mask fraction (None = forward only), net)
CONFIGS = {
    "c1": (C1_TEXT, 64, 1024, None,
           "conv6/maxpool2/tanh/conv5/maxpool2/tanh/conv4 (16,32,10 ch), 1 ch, patch 29"),
    "c2": (C2_TEXT, 256, 64, 0.01,
           "conv6/maxpool2/tanh/conv5/maxpool2/tanh/conv4 (16,32,10 ch), patch 29"),
    "c3": (C3_TEXT, 512, 16, 1.0,
           "plain CNN1 (50,50,8): conv6/maxpool4/tanh/conv3/maxpool2/tanh/conv7, patch 69"),
    "c4": (C4_TEXT, 1024, 2, 0.01,
           "5 conv (strides 2,1,1,2,1) / 3 max-pool, relu, patch 119"),
}
HEADLINE = "c3"
WORKLOAD = {
    "c1": "c1: 1x64x64, forward only",
    "c2": "c2: 3x256x256, fwd + 1%-masked bwd (655 px/image), squared-error delta",
    "c3": "c3: 3x512x512 RGB, 8 classes, patch 69, full-image fwd + bwd (full mask), "
          "squared-error delta, grad all-reduce, SGD",
    "c4": "c4: 3x1024x1024, 5-conv/3-pool (strides 2,1,1,2,1), fwd + 1%-masked bwd",
}


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            j = json.load(fh)
        return {"hbm_gbs": j["hbm_gbs"], "bf16_tflops": j["bf16_tflops"],
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0,
            "source": "fallback (B200_PROFILING.md)"}


def host_info():
    model = platform.processor() or ""
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True,
                                   timeout=10).stdout.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
                break
    except (OSError, subprocess.SubprocessError):
        pass
    return {"cpu_model": model, "nproc": os.cpu_count() or 1}


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 25 ms during the timed region
    (nvidia-smi is started and its first sample awaited before the region begins; rows
    taken before the region are discarded)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "25"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5 and self.proc.poll() is None:
                time.sleep(0.01)
            self.rows.clear()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [s.strip() for s in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ----------------------------------------------------------------------------- CPU arm

def _ref_package():
    """The UNMODIFIED reference package installed into baseline/_ref (DESIGN.md recipe), with
    its compiled backend selected, or None."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "denseprop")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import denseprop
        from denseprop import backend
        if "compiled" not in backend.available():
            return None
        backend.use("compiled")
        return denseprop
    except Exception:  # noqa: BLE001 -- fall back to the oracle glue
        return None


def conv_flops(text, rows, side):
    """(forward, backward) algorithmic conv FLOPs of the dense plan for `rows` output rows of a
    `side`-wide image (backward = data + weight gradients, no layer-0 data gradient)."""
    import paper_1412_4526_b200 as dp
    from paper_1412_4526_b200.plan import DilatedConv
    plan = dp.compile_plan(dp.parse_spec(text))
    shapes = plan.layer_shapes(rows, side)
    fwd = bwd = 0
    first = True
    for k, layer in enumerate(plan.layers):
        if isinstance(layer, DilatedConv):
            co, ho, wo = shapes[k + 1]
            f = 2 * co * layer.base.in_channels * layer.base.kernel_size ** 2 * ho * wo
            fwd += f
            bwd += f if first else 2 * f
            first = False
    return fwd, bwd


def cpu_dense_seconds(text, side, mask_frac, threads, rows=None, seed=0):
    """(forward s, backward s, output pixels, kind, how) of ONE image of `side` on the CPU.

    With `rows` < side only a band of that many output rows is run (its padded input rows
    plus the (patch - 1)-row halo); a band costs MORE per output pixel than the full image
    (every layer also computes the halo rows still needed below it), so the band's times are
    scaled to the full image by the ratio of the dense plan's conv FLOPs, full image / band
    (forward and backward separately), and `output pixels` is the full image's.
    """
    f, b, px, kind, how = _cpu_dense_band(text, side, mask_frac, threads, rows, seed)
    band = rows if rows is not None and rows < side else side
    if band < side:
        ff, fb = conv_flops(text, side, side)
        bf, bb = conv_flops(text, band, side)
        f *= ff / bf
        b *= fb / bb if bb else 1.0
        px = side * side
        how += f", band of {band} rows scaled to the full image by conv FLOPs"
    return f, b, px, kind, how


def _cpu_dense_band(text, side, mask_frac, threads, rows=None, seed=0):
    """The unscaled measurement behind cpu_dense_seconds (a band when rows < side).

    Through the reference package's own public API (compile_plan, pad_image,
    run_plan_layer = the body of dense_forward, forward.py:101-128, then dense_backward,
    backward.py:185-223) on its compiled backend when baseline/_ref is installed, else the
    reference's compiled kernels (oracle/_ref) or the oracle C port via the oracle glue."""
    rng = np.random.default_rng(seed)
    img_c = 3 if "input channels=3" in text else 1
    band = rows if rows is not None and rows < side else side
    img = rng.uniform(-0.5, 0.5, (img_c, side, side)).astype(np.float32)
    pkg = _ref_package()
    if pkg is not None:
        from denseprop.backward import ErrorMask, dense_backward
        from denseprop.forward import ForwardCache, pad_image, run_plan_layer
        from denseprop.netspec import parse_spec
        from denseprop.plan import compile_plan
        plan = compile_plan(parse_spec(text))
        patch = plan.lead_margin + plan.trail_margin + 1
        t0 = time.perf_counter()
        x = pad_image(plan, img)[:, :band + patch - 1, :]
        inputs, argmax = [], {}
        for k in range(len(plan.layers)):
            inputs.append(x)
            x, arg = run_plan_layer(plan, k, x, threads)
            if arg is not None:
                argmax[k] = arg
        cache = ForwardCache(plan=plan, inputs=inputs, argmax=argmax, output=x)
        t1 = time.perf_counter()
        if mask_frac is None:
            return t1 - t0, 0.0, band * side, "reference", \
                "unmodified reference package (baseline/_ref), compiled backend"
        q = cache.output.shape[0]
        tgt = rng.uniform(-1, 1, (q, band, side)).astype(np.float32)
        if mask_frac >= 1.0:
            mask = ErrorMask.full(band, side)
        else:
            n = max(1, int(mask_frac * band * side))
            flat = rng.choice(band * side, n, replace=False)
            mask = ErrorMask.of(band, side, [(int(i) // side, int(i) % side) for i in flat])
        t2 = time.perf_counter()
        dense_backward(plan, cache, (cache.output - tgt).astype(np.float32), mask, threads)
        t3 = time.perf_counter()
        return t1 - t0, t3 - t2, band * side, "reference", \
            "unmodified reference package (baseline/_ref), compiled backend"
    # fallback: the reference's compiled kernels / the oracle C port through the oracle glue
    from oracle import engine_np, kernels_c, ref_kernels
    from oracle.netdesc import read_spec
    if ref_kernels.available():
        K, kind = ref_kernels.load(), "reference"
    else:
        kernels_c.build()
        K, kind = kernels_c, "port"
    net = read_spec(text)
    t0 = time.perf_counter()
    xp = engine_np.pad_image(net, img)[:, :band + net.patch() - 1, :]
    cache = engine_np.dense_forward(net, xp, K, threads, padded=True)
    t1 = time.perf_counter()
    how = "reference compiled kernels (oracle/_ref) via the oracle glue" if kind == "reference" \
        else "oracle C port"
    if mask_frac is None:
        return t1 - t0, 0.0, band * side, kind, how
    tgt = rng.uniform(-1, 1, cache.output.shape).astype(np.float32)
    mask = np.ones(cache.output.shape[1:], bool)
    if mask_frac < 1.0:
        mask[:] = rng.random(mask.shape) < mask_frac
    t2 = time.perf_counter()
    engine_np.dense_backward(net, cache, (cache.output - tgt).astype(np.float32), mask, K,
                             threads)
    t3 = time.perf_counter()
    return t1 - t0, t3 - t2, band * side, kind, how


def cpu_patch_scan_px_per_s(text, side, budget_s=3.0):
    """Patch-by-patch scan (oracle.py:145-164 restated), 1 thread, sampled pixels."""
    from oracle import engine_np
    from oracle.netdesc import read_spec
    net = read_spec(text)
    img_c = 3 if "input channels=3" in text else 1
    img = np.random.default_rng(1).uniform(-0.5, 0.5, (img_c, side, side)).astype(np.float32)
    step = max(1, side // 16)
    pixels = [(y, x) for y in range(0, side, step) for x in range(0, side, step)]
    done, t0 = 0, time.perf_counter()
    for px in pixels:
        engine_np.scan_forward(net, img, [px])
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return done / dt, done


def run_reference_arm(args, rank):
    """The driver's reference arm: the unmodified reference package on the headline config
    (c3@512, one full image per step, fwd + full-mask bwd), all host threads."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(threads))
    text, side, _, mask_frac, net = CONFIGS[HEADLINE]
    for s in range(max(0, args.warmup)):
        cpu_dense_seconds(text, side, mask_frac, threads, seed=100 + s)
    fw, bw = [], []
    kind = how = None
    for s in range(args.steps):
        f, b, px, kind, how = cpu_dense_seconds(text, side, mask_frac, threads, seed=s)
        fw.append(f)
        bw.append(b)
    step = float(np.sum(fw) + np.sum(bw)) / args.steps
    value = side * side / step
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "pixels/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD[HEADLINE], "images_per_step": 1, "side": side,
                   "mask_fraction": mask_frac, "net": net},
        "forward": {"value": side * side / float(np.mean(fw)), "unit": "pixels/s"},
        "cpu_baseline": {"value": value, "unit": "pixels/s", "cores": threads, "kind": kind,
                         "sample": f"{args.steps} images of {HEADLINE}@{side} (fwd + "
                                   f"full-mask bwd), {how}, {threads} threads",
                         **host_info()},
        "e2e": {"value": value, "unit": "pixels/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm

def stable_lr(batch, side, mask_frac):
    """SGD step size that keeps the synthetic training run finite: the loss is a SUM over the
    masked pixels, so the gradient grows with their count (a fixed 1e-7 diverges to NaN within
    ~8 c3 steps, and a NaN/overflowing step is a degenerate workload: the fp16-split convs
    see out-of-range operands and fall back to tf32)."""
    frac = 1.0 if mask_frac is None else mask_frac
    return 1e-4 / max(1.0, batch * side * side * frac)


def _synthetic(spec, batch, side, mask_frac, seed, dev):
    import torch
    rng = np.random.default_rng(seed)
    imgs = torch.from_numpy(rng.uniform(-0.5, 0.5, (batch, spec.input_channels, side, side))
                            .astype(np.float32))
    tgts = torch.from_numpy(rng.uniform(-1, 1, (batch, spec.output_channels, side, side))
                            .astype(np.float32))
    m = np.zeros((batch, side, side), np.uint8)
    frac = 1.0 if mask_frac is None else mask_frac
    if frac >= 1.0:
        m[:] = 1
    else:
        n = max(1, int(frac * side * side))
        for b in range(batch):
            m[b].flat[rng.choice(side * side, n, replace=False)] = 1
    return imgs, tgts, torch.from_numpy(m)


def measure_config(text, side, batch, mask_frac, steps=5, warmup=3, seed=7):
    """Device-timed fwd and fwd+masked-bwd throughput (pixels/s) of one net / image size on
    this GPU: CUDA-graph replays over synthetic HBM-resident inputs (SGD included)."""
    import torch
    import paper_1412_4526_b200 as dp
    from paper_1412_4526_b200.engine import DenseNet
    from paper_1412_4526_b200.trainer import DataParallelTrainer
    spec = dp.parse_spec(text)
    plan = dp.compile_plan(spec)
    imgs, tgts, masks = (t.cuda() for t in _synthetic(spec, batch, side, mask_frac, seed, "cuda"))
    stream = torch.cuda.current_stream()

    def timed(fn):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps

    px = batch * side * side
    out = {"side": side, "images": batch, "mask_fraction": mask_frac}
    if mask_frac is None:
        net = DenseNet(plan, batch, side, side, train=False)
        net.set_input(imgs)
        g = net.capture(net.forward)
        ms_fwd = timed(g.replay)
        out.update({"forward": px / (ms_fwd / 1e3), "ms_forward": ms_fwd})
        flops = net.conv_flops_per_image()["fwd"] * batch
    else:
        tr = DataParallelTrainer(plan, batch, side, side, lr=stable_lr(batch, side, mask_frac),
                                 use_graph=True)
        net = tr.net
        tr.load_batch(imgs, tgts, masks)
        ms_train = timed(tr.step)
        ms_fwd = timed(net.forward)
        f = net.conv_flops_per_image()
        flops = (f["fwd"] + f["bwd"]) * batch
        out.update({"train": px / (ms_train / 1e3), "forward": px / (ms_fwd / 1e3),
                    "ms_train": ms_train, "ms_forward": ms_fwd,
                    "conv_tflops_train": flops / (ms_train / 1e3) / 1e12})
        del tr
    out["conv_tiers"] = {str(k): v["forward"] for k, v in net.kernel_plan().items()}
    del net
    torch.cuda.empty_cache()
    return out


def sizes_sweep(budget_cpu=True):
    """BASELINE configs[4] (c5): the Plain CNN1 family, pool1 p in {2, 4, 8} with conv1 k = 6
    (patch 37 / 69 / 133) and k = 2 (33 / 65 / 129), sides 128 .. 2048; GPU fwd and train
    (full-image fwd + full-mask bwd), plus a sampled CPU reference (and patch scan) per net."""
    nets = [(p, k1) for p in (2, 4, 8) for k1 in (6, 2)]
    sides = (128, 256, 512, 1024, 2048)
    batch = {128: 64, 256: 16, 512: 4, 1024: 1, 2048: 1}
    points = []
    threads = os.cpu_count() or 1
    for p, k1 in nets:
        text = plain_cnn1_text(pool1=p, k1=k1)
        patch = {(2, 6): 37, (4, 6): 69, (8, 6): 133, (2, 2): 33, (4, 2): 65, (8, 2): 129}[(p, k1)]
        for side in sides:
            pt = {"patch": patch, "pool1": p, "conv1_k": k1,
                  **measure_config(text, side, batch[side], 1.0, steps=3, warmup=2)}
            if budget_cpu and side in (128, 512, 2048):
                rows = side if side <= 128 else 8
                f, b, px, kind, _ = cpu_dense_seconds(text, side, 1.0, threads, rows=rows)
                pt["cpu"] = {"train": px / (f + b), "forward": px / f, "cores": threads,
                             "kind": kind,
                             "sample": ("1 full image" if rows == side else
                                        f"band of {rows} output rows x {side} (+{patch - 1}-row "
                                        "halo), scaled to the full image by conv FLOPs")}
                pt["train_over_cpu"] = pt["train"] / pt["cpu"]["train"]
            points.append(pt)
        if budget_cpu:
            ps, n = cpu_patch_scan_px_per_s(text, 256, budget_s=1.5)
            points[-1]["patch_scan_cpu"] = {"forward": ps, "cores": 1,
                                            "sample": f"{n} pixels of a 256^2 image"}
    return points


def mask_sweep(tr, batch_tensors, side, timed, steps=5):
    """Training-step time (CUDA-graph replay: fwd + masked bwd + SGD) per error-mask size,
    1 pixel .. the full image per image; spread = (max - min) / min, the reference's budget is
    10 % (bench.py:311-343).  Restores the full mask afterwards."""
    import torch
    imgs, tgts, masks = batch_tensors
    tr.load_batch(imgs, tgts, masks)
    total = side * side
    sizes = [1, total // 1000, total // 100, total // 10, total // 2, total]
    rng = np.random.default_rng(5)
    ms = []
    for k in sizes:
        m = np.zeros((masks.shape[0], total), np.uint8)
        for b in range(masks.shape[0]):
            m[b, rng.choice(total, k, replace=False)] = 1
        tr.net.mask.copy_(torch.from_numpy(m.reshape(masks.shape)))
        ms.append(timed(lambda s: tr.step(), steps) / steps)
    tr.net.mask.copy_(masks)
    spread = (max(ms) - min(ms)) / min(ms)
    return {"mask_pixels_per_image": sizes, "ms_per_step": ms, "spread": spread,
            "ok": spread <= 0.10, "steps_per_size": steps}


def patch_scan_gpu(text, side, n_pix, dev, batch=4096, reps=2):
    """GPU patch-by-patch baseline: n_pix patches of one synthetic image through the strided
    network (same tcgen05 conv kernels at dilation 1), forward only and forward + backward
    (per-patch gradients summed), device-timed with CUDA events."""
    import torch
    import paper_1412_4526_b200 as dp
    from paper_1412_4526_b200 import patchscan
    spec = dp.parse_spec(text)
    img = (torch.rand((spec.input_channels, side, side), device=dev) - 0.5)
    x0 = patchscan._padded(spec, img)
    batch = min(batch, n_pix)
    net = patchscan.PatchNet(spec, batch, train=True, precision="fast")
    pix = torch.arange(n_pix, dtype=torch.int32, device=dev)
    delta = torch.rand((batch, net.out_channels), device=dev) - 0.5

    def run(train):
        for first in range(0, n_pix, batch):
            patchscan._gather(x0, net.inputs[0], pix[first:first + batch], net.n)
            net.forward()
            if train:
                net.backward(delta)

    out = {"unit": "pixels/s", "patch": net.n, "side": side,
           "sample": f"{n_pix} patches of one {side}x{side} image, batches of {batch}"}
    for key, train in (("forward", False), ("train", True)):
        run(train)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            run(train)
        e1.record()
        torch.cuda.synchronize()
        out[key] = reps * n_pix / (e0.elapsed_time(e1) / 1e3)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=HEADLINE, choices=sorted(CONFIGS),
                    help="workload of the main line (default: the c3@512 headline)")
    ap.add_argument("--batch", type=int, default=0, help="images per GPU per step")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-sweep", action="store_true",
                    help="skip the c5 size sweep and the other config lines")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference_arm(args, rank)
        return

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    dist_info = {"world_size": world, "backend": None}
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        # force the NCCL communicator up now (a 1-element all-reduce), outside the timings
        t = torch.ones(1, device="cuda")
        dist.all_reduce(t)
        torch.cuda.synchronize()
        dist_info = {"world_size": dist.get_world_size(), "backend": dist.get_backend(),
                     "nccl_version": ".".join(map(str, torch.cuda.nccl.version())),
                     "allreduce_check": float(t.item())}
        if rank == 0:
            print(f"[bench] NCCL communicator up: world {world}, nccl "
                  f"{dist_info['nccl_version']}", file=sys.stderr, flush=True)

    import paper_1412_4526_b200 as dp
    from paper_1412_4526_b200 import engine
    from paper_1412_4526_b200.trainer import DataParallelTrainer, H2DPipeline

    text, SIDE, B, MASK_FRAC, NET = CONFIGS[args.config]
    if args.batch:
        B = args.batch
    if MASK_FRAC is None:
        raise SystemExit("the main line needs a training config (c2, c3 or c4)")
    spec = dp.parse_spec(text)
    plan = dp.compile_plan(spec)
    dev = torch.device("cuda", local)
    # synthetic inputs, resident in HBM: two batches alternated step to step
    pool = [_synthetic(spec, B, SIDE, MASK_FRAC, 1234 + 17 * rank + i, dev) for i in range(2)]
    dpool = [tuple(t.to(dev) for t in p) for p in pool]
    hpool = [tuple(t.pin_memory() for t in p) for p in pool]

    tr = DataParallelTrainer(plan, B, SIDE, SIDE, lr=stable_lr(B, SIDE, MASK_FRAC),
                            use_graph=not args.no_graph)
    net = tr.net
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    def maxrank(ms):
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    def timed(fn, steps):
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s in range(steps):
            fn(s)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        return maxrank(e0.elapsed_time(e1))

    # ---- training step, inputs resident in HBM
    def train_step(s):
        imgs, tgts, masks = dpool[s & 1]
        tr.load_batch(imgs, tgts, masks)
        tr.step()

    for s in range(args.warmup):
        train_step(s)
    engine.ops.launches = 0
    with ClockSampler(local) as clk:
        ms_train = timed(train_step, args.steps)
    # eager launches (pad, SGD) counted by the ops wrappers + kernels inside each graph replay
    launches_in_region = engine.ops.launches + \
        (tr.graph_kernel_count * args.steps if tr._graph is not None else 0)
    clocks = clk.summary()

    # ---- forward only (inference shards images, no collective)
    def fwd_step(s):
        net.set_input(dpool[s & 1][0])
        net.forward()

    for s in range(args.warmup):
        fwd_step(s)
    ms_fwd = timed(fwd_step, args.steps)

    # ---- e2e through the public trainer API from pinned host buffers: every step copies
    # its images + targets + masks H2D (double-buffered: the copy of batch s+1 overlaps
    # step s) and reads the gradient bucket back D2H
    grad_host = torch.empty(net.grad_flat.shape, dtype=net.grad_flat.dtype).pin_memory()
    feed = H2DPipeline(tr, *dpool[0])

    def e2e_run(steps):
        feed.submit(*hpool[0])
        for s in range(steps):
            if s + 1 < steps:
                feed.submit(*hpool[(s + 1) & 1])
            feed.step()
            grad_host.copy_(net.grad_flat, non_blocking=True)

    e2e_run(args.warmup)
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    feed.copy_stream.wait_event(e0)  # every H2D copy of the run lies inside [e0, e1]
    e2e_run(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms_e2e = maxrank(e0.elapsed_time(e1))
    h2d = sum(t.numel() * t.element_size() for t in hpool[0])
    d2h = grad_host.numel() * grad_host.element_size()

    # ---- forward e2e (inference from host): H2D images, forward, D2H score maps; the
    # copies of image s+1 and the read-back of scores s-1 overlap forward s (two streams)
    out_host = [torch.empty(net.output.shape, dtype=net.output.dtype).pin_memory()
                for _ in range(2)]
    img_dev = [torch.empty_like(dpool[0][0]) for _ in range(2)]
    cs = torch.cuda.Stream(device=dev)
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]

    def fwd_e2e_run(steps):
        with torch.cuda.stream(cs):
            img_dev[0].copy_(hpool[0][0], non_blocking=True)
            ev_in[0].record(cs)
        for s in range(steps):
            k = s & 1
            if s + 1 < steps:
                with torch.cuda.stream(cs):
                    cs.wait_event(ev_out[k ^ 1]) if s >= 1 else None
                    img_dev[k ^ 1].copy_(hpool[(s + 1) & 1][0], non_blocking=True)
                    ev_in[k ^ 1].record(cs)
            stream.wait_event(ev_in[k])
            net.set_input(img_dev[k])
            net.forward()
            out_host[k].copy_(net.output, non_blocking=True)
            ev_out[k].record(stream)

    fwd_e2e_run(args.warmup)
    barrier()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    cs.wait_event(f0)
    fwd_e2e_run(args.steps)
    f1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms_fwd_e2e = maxrank(f0.elapsed_time(f1))

    # ---- mask-size sweep (reference bench.py:311-343): the training step's
    # cost must not depend on how many pixels the error mask keeps
    msweep = mask_sweep(tr, dpool[0], SIDE, timed) if not args.no_sweep else None

    # ---- per-kernel timing of one eager step (roofline of the dominant kernel)
    prof = engine.profile_step(tr, reps=5)

    px_per_step = B * SIDE * SIDE * world
    value = px_per_step / (ms_train / args.steps / 1e3)
    peaks = _peaks()
    top = max(prof["kernels"], key=lambda k: k["ms"])
    if top["bound"] == "tensor":
        achieved = top["flops"] / (top["ms"] / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": peaks["bf16_tflops"],
                "unit": "TFLOP/s", "frac": achieved / peaks["bf16_tflops"]}
    else:
        achieved = top["bytes"] / (top["ms"] / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"]}
    if top["bound"] == "tensor" and "_tc" in top["name"]:
        # 3xTF32 issues 3 TF32 MACs per algorithmic MAC; dense TF32 is half of dense bf16
        ceil = peaks["bf16_tflops"] / 2 / 3
        roof["derived_3xtf32_ceiling_tflops"] = ceil
        roof["frac_of_3xtf32_ceiling"] = roof["achieved"] / ceil
        # measured tcgen05 SS-MMA throughput (tools/mma_peak.cu, profiles/r02_mma_peak.json):
        # the split kernels issue 3 MMAs per algorithmic MAC at N = 64 / 128
        mpath = os.path.join(ROOT, "profiles", "r02_mma_peak.json")
        if os.path.exists(mpath):
            with open(mpath) as fh:
                pts = json.load(fh)["points"]
            ss = {f"{p['kind']}_n{p['N']}": p["tflops"] for p in pts
                  if p.get("operands", "SS") == "SS" and p.get("layout", "none") == "none"}
            roof["tcgen05_ss_peak_tflops"] = ss
            roof["mma_rate_tflops"] = 3 * roof["achieved"]  # split products issued per s
            for kind in ("tf32", "f16"):  # the weight gradients are 3xTF32
                if f"{kind}_n128" in ss:
                    roof[f"frac_of_ss_{kind}_n128"] = 3 * roof["achieved"] / ss[f"{kind}_n128"]
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", f"r02_traffic_{args.config}.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            tj = json.load(fh)
        if top["name"] in tj.get("kernels", {}):
            traffic = tj["kernels"][top["name"]]["dram_bytes"]
            traffic_src = tj.get("source")
        # the committed ncu capture's per-launch tensor-pipe / DRAM / issue percentages
        # beside each record's CUDA-event time (cold-cache, serialised: indicative)
        for k in prof["kernels"]:
            rec = tj.get("kernels", {}).get(k["name"])
            if rec:
                k["ncu"] = [{"kernel": ln["kernel"].split("(")[0][:60],
                             **{m: round(ln[m], 1) for m in ("tensor_pct", "dram_pct",
                                                            "issue_pct") if m in ln}}
                            for ln in rec["launches"]]
    roof.update({"kernel": top["name"], "ms_per_launch": top["ms"],
                 "share_of_step": top["ms"] / prof["step_ms"], "peak_source": peaks["source"],
                 "traffic": traffic, "traffic_source": traffic_src,
                 "note": ("tcgen05 conv: algorithmic FLOPs (each MAC issues 3 split "
                          "products); peak = measured dense bf16"
                          if "_tc" in top["name"] else
                          "measured against the peak named in `bound`")})
    conv = net.conv_flops_per_image()

    line = {
        "metric": METRIC, "value": value, "unit": "pixels/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_train / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": WORKLOAD[args.config], "config": args.config,
                   "images_per_gpu_per_step": B, "side": SIDE, "mask_fraction": MASK_FRAC,
                   "net": NET,
                   "parallelism": f"dp{world} (images sharded, NCCL all-reduce SUM)",
                   "l2": "working set >> L2 (activations %.1f GB per GPU)" %
                         (net.activation_bytes() / 1e9),
                   "cuda_graph": tr._graph is not None,
                   "precision": net.precision,
                   "conv_tiers": {str(k): v for k, v in net.kernel_plan().items()}},
        "forward": {"value": px_per_step / (ms_fwd / args.steps / 1e3), "unit": "pixels/s",
                    "ms_per_step": ms_fwd / args.steps,
                    "e2e": {"value": px_per_step / (ms_fwd_e2e / args.steps / 1e3),
                            "unit": "pixels/s",
                            "h2d_bytes_per_step": hpool[0][0].numel() * 4,
                            "d2h_bytes_per_step": out_host[0].numel() * 4}},
        "e2e": {"value": px_per_step / (ms_e2e / args.steps / 1e3), "unit": "pixels/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches_in_region,
        "conv_tflops_step": (conv["fwd"] + conv["bwd"]) * B * world /
                            (ms_train / args.steps / 1e3) / 1e12,
        "roofline": roof,
        "kernels": prof["kernels"],
        "clocks": clocks,
        "distributed": dist_info,
    }
    if msweep is not None:
        line["mask_sweep"] = msweep

    if rank == 0 and world == 1 and not args.no_sweep:
        # patch-by-patch baseline on the same GPU: the ORIGINAL
        # strided network on every pixel's patch (patchscan.PatchNet), fwd and fwd + bwd
        line["patch_scan_gpu"] = {
            name: patch_scan_gpu(CONFIGS[name][0], CONFIGS[name][1], n_pix, dev)
            for name, n_pix in (("c2", 65536), (args.config, 16384))}
        for name, ps in line["patch_scan_gpu"].items():
            if name == args.config:
                ps["dense_over_scan_forward"] = line["forward"]["value"] / ps["forward"]
                ps["dense_over_scan_train"] = value / ps["train"]

        # the other BASELINE configs on the same GPU, a sampled CPU reference beside each
        threads = os.cpu_count() or 1
        lines = {}
        for name in ("c1", "c2", "c4"):
            t, side, b, mf, netd = CONFIGS[name]
            m = measure_config(t, side, b, mf)
            m.update({"workload": WORKLOAD[name], "net": netd})
            if not args.no_cpu_baseline:
                rows = None if name in ("c1", "c2") else 64
                f, bk, px, kind, how = cpu_dense_seconds(t, side, mf, threads, rows=rows)
                m["cpu"] = {"forward": px / f, "cores": threads, "kind": kind,
                            "sample": ("1 full image, " if rows is None else "") + how}
                if mf is not None:
                    m["cpu"]["train"] = px / (f + bk)
                    m["train_over_cpu"] = m["train"] / m["cpu"]["train"]
                m["forward_over_cpu"] = m["forward"] / m["cpu"]["forward"]
            lines[f"{name}_{side}"] = m
        line["lines"] = lines
        line["sizes"] = {
            "net": "plain CNN1 (50,50,32), 3 ch; pool1 p in {2,4,8}, conv1 k in {6,2}",
            "unit": "pixels/s", "note": "train = full-image fwd + full-mask bwd + SGD",
            "points": sizes_sweep(budget_cpu=not args.no_cpu_baseline)}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        f, b, px, kind, how = cpu_dense_seconds(text, SIDE, MASK_FRAC, threads)
        f1, b1, px1, _, _ = cpu_dense_seconds(text, SIDE, MASK_FRAC, 1, rows=32)
        scan_px_s, scan_n = cpu_patch_scan_px_per_s(text, SIDE)
        line["cpu_baseline"] = {
            "value": px / (f + b), "unit": "pixels/s", "cores": threads, "kind": kind,
            "sample": f"1 image of {args.config}@{SIDE} (fwd + bwd), {how}, {threads} threads",
            "forward_value": px / f, **host_info(),
            "single_thread": {"value": px1 / (f1 + b1), "forward_value": px1 / f1,
                              "cores": 1,
                              "sample": f"band of 32 output rows x {SIDE}, 1 thread, "
                                        "scaled to the full image by conv FLOPs"},
            "patch_scan_forward": {"value": scan_px_s, "unit": "pixels/s", "cores": 1,
                                   "sample": f"{scan_n} pixels on a 16-px grid"},
        }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

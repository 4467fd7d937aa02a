"""Benchmark: classified pixels/s of dense fwd + masked bwd on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one process per GPU, NCCL)

Workload (N=1 line): BASELINE.json configs[1] = "c2": the c1/c2 CNN of SURVEY.md
Appendix A (conv6-maxpool2-tanh-conv5-maxpool2-tanh-conv4, patch 29) on 3x256x256
synthetic images, forward + masked backward with 1% sampled pixels (655 per
image), squared-error delta against a synthetic target map (cli.py:218),
gradients summed per image, one NCCL all-reduce(SUM) of the gradient bucket
per step when N > 1, and a plain SGD update.  A "step" = one such training pass
over a batch of B images per GPU (weak scaling: per-GPU work fixed).

value  = whole-job training throughput, images*h*w / time over all ranks, with the
         inputs already resident in HBM (device-timed, CUDA events, max over ranks)
e2e    = the same through the public trainer API from pinned HOST buffers:
         per step H2D of images + targets + masks and D2H of the gradient bucket
forward = forward-only inference throughput (no collective), same batch
roofline = the dominant kernel of the step, timed per launch with CUDA events
cpu_baseline = the reference's own compiled kernels (oracle/_ref, built from
         /root/reference) driving the dense path on the host cores, one image
         (rank 0, N=1 only); plus the patch-by-patch scan on a sampled pixel grid.

`--impl reference` times that reference CPU path alone as the driver's reference arm.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "classified pixels/sec fwd and fwd+bwd per image size at 1/2/4/8 B200 vs CPU"
C2_TEXT = ("input channels=3\n"
           "conv out=16 in=3 k=6 stride=1 weights=seed:1\n"
           "pool kind=max k=2 stride=2\nnonlin kind=tanh\n"
           "conv out=32 in=16 k=5 stride=1 weights=seed:2\n"
           "pool kind=max k=2 stride=2\nnonlin kind=tanh\n"
           "conv out=10 in=32 k=4 stride=1 weights=seed:3\n")
SIDE = 256
MASK_FRAC = 0.01
# BASELINE.json configs[2] / configs[3]
C3_TEXT = ("input channels=3\n"
           "conv out=50 in=3 k=6 stride=1 weights=seed:0\n"
           "pool kind=max k=4 stride=4\nnonlin kind=tanh\n"
           "conv out=50 in=50 k=3 stride=1 weights=seed:3\n"
           "pool kind=max k=2 stride=2\nnonlin kind=tanh\n"
           "conv out=8 in=50 k=7 stride=1 weights=seed:6\n")
C4_TEXT = ("input channels=3\n"
           "conv out=48 in=3 k=5 stride=2 weights=seed:1\nnonlin kind=relu\n"
           "conv out=64 in=48 k=3 stride=1 weights=seed:2\nnonlin kind=relu\n"
           "pool kind=max k=2 stride=2\n"
           "conv out=96 in=64 k=3 stride=1 weights=seed:3\nnonlin kind=relu\n"
           "pool kind=max k=2 stride=2\n"
           "conv out=128 in=96 k=3 stride=2 weights=seed:4\nnonlin kind=relu\n"
           "pool kind=max k=2 stride=2\n"
           "conv out=8 in=128 k=3 stride=1 weights=seed:5\n")


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            j = json.load(fh)
        return {"hbm_gbs": j["hbm_gbs"], "bf16_tflops": j["bf16_tflops"],
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0,
            "source": "fallback (B200_PROFILING.md)"}


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

def _cpu_kernels():
    """The reference's own compiled kernels when built (oracle/_ref), else the oracle C port."""
    from oracle import kernels_c, ref_kernels
    if ref_kernels.available():
        try:
            return ref_kernels.load(), "reference"
        except ImportError:
            pass
    kernels_c.build()
    return kernels_c, "port"


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


def cpu_dense_step_seconds(threads, images=1, seed=0):
    """Time fwd + 1%-masked bwd of c2@256 on the CPU, per image: through the reference
    package's own public API (dense_forward / dense_backward, compiled backend) when it is
    installed in baseline/_ref, else through its compiled kernels via the oracle glue."""
    pkg = _ref_package()
    if pkg is not None:
        from denseprop.backward import ErrorMask, dense_backward
        from denseprop.forward import dense_forward
        from denseprop.netspec import parse_spec
        from denseprop.plan import compile_plan
        plan = compile_plan(parse_spec(C2_TEXT))
        rng = np.random.default_rng(seed)
        times_f, times_b = [], []
        for _ in range(images):
            img = rng.uniform(-0.5, 0.5, (3, SIDE, SIDE)).astype(np.float32)
            tgt = rng.uniform(-1, 1, (10, SIDE, SIDE)).astype(np.float32)
            flat = rng.choice(SIDE * SIDE, int(MASK_FRAC * SIDE * SIDE), replace=False)
            mask = ErrorMask.of(SIDE, SIDE, [(int(i) // SIDE, int(i) % SIDE) for i in flat])
            t0 = time.perf_counter()
            cache = dense_forward(plan, img, threads)
            t1 = time.perf_counter()
            dense_backward(plan, cache, (cache.output - tgt).astype(np.float32), mask, threads)
            t2 = time.perf_counter()
            times_f.append(t1 - t0)
            times_b.append(t2 - t1)
        return (float(np.median(times_f)), float(np.median(times_b)), "reference",
                "unmodified reference package (baseline/_ref): dense_forward + dense_backward, "
                "compiled backend")
    from oracle import engine_np
    from oracle.netdesc import read_spec
    K, kind = _cpu_kernels()
    net = read_spec(C2_TEXT)
    rng = np.random.default_rng(seed)
    times_f, times_b = [], []
    for _ in range(images):
        img = rng.uniform(-0.5, 0.5, (3, SIDE, SIDE)).astype(np.float32)
        tgt = rng.uniform(-1, 1, (10, SIDE, SIDE)).astype(np.float32)
        mask = np.zeros((SIDE, SIDE), bool)
        mask.flat[rng.choice(SIDE * SIDE, int(MASK_FRAC * SIDE * SIDE), replace=False)] = True
        t0 = time.perf_counter()
        cache = engine_np.dense_forward(net, img, K, threads)
        t1 = time.perf_counter()
        engine_np.dense_backward(net, cache, (cache.output - tgt).astype(np.float32), mask, K,
                                 threads)
        t2 = time.perf_counter()
        times_f.append(t1 - t0)
        times_b.append(t2 - t1)
    how = ("reference compiled kernels (oracle/_ref) via oracle/ engine glue" if kind == "reference"
           else "oracle C port")
    return float(np.median(times_f)), float(np.median(times_b)), kind, how


def cpu_patch_scan_px_per_s(budget_s=4.0):
    """Patch-by-patch scan (oracle.py:145-164 restated), 1 thread, sampled pixels."""
    from oracle import engine_np
    from oracle.netdesc import read_spec
    net = read_spec(C2_TEXT)
    img = np.random.default_rng(1).uniform(-0.5, 0.5, (3, SIDE, SIDE)).astype(np.float32)
    pixels = [(y, x) for y in range(0, SIDE, 16) for x in range(0, SIDE, 16)]
    done, t0 = 0, time.perf_counter()
    for px in pixels:
        engine_np.scan_forward(net, img, [px])
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return done / dt, done


def run_reference_arm(args, rank):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(threads))
    for _ in range(max(0, args.warmup)):
        cpu_dense_step_seconds(threads, 1)
    fw, bw = [], []
    kind = how = None
    for s in range(args.steps):
        f, b, kind, how = cpu_dense_step_seconds(threads, 1, seed=s)
        fw.append(f)
        bw.append(b)
    step = float(np.sum(fw) + np.sum(bw)) / args.steps
    value = SIDE * SIDE / step
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "pixels/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "c2: 3x256x256, fwd + 1%-masked bwd, squared-error delta",
                   "images_per_step": 1, "side": SIDE, "mask_fraction": MASK_FRAC,
                   "net": "conv6/maxpool2/tanh/conv5/maxpool2/tanh/conv4 (16,32,10 ch), patch 29"},
        "forward": {"value": SIDE * SIDE / float(np.mean(fw)), "unit": "pixels/s"},
        "cpu_baseline": {"value": value, "unit": "pixels/s", "cores": threads, "kind": kind,
                         "sample": f"{args.steps} images of c2@256 (fwd+bwd, 1% mask), {how}, "
                                   f"{threads} threads"},
        "e2e": {"value": value, "unit": "pixels/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm

def measure_config(text, side, batch, mask_frac, steps=5, warmup=2, seed=7):
    """Device-timed fwd and fwd+masked-bwd throughput (pixels/s) of one net / image size on
    this GPU: CUDA-graph replays over synthetic HBM-resident inputs (SGD included)."""
    import torch
    import paper_1412_4526_b200 as dp
    from paper_1412_4526_b200.trainer import DataParallelTrainer
    spec = dp.parse_spec(text)
    plan = dp.compile_plan(spec)
    rng = np.random.default_rng(seed)
    gen = torch.Generator(device="cuda").manual_seed(seed)
    imgs = torch.rand((batch, spec.input_channels, side, side), device="cuda", generator=gen) - 0.5
    tgts = torch.rand((batch, spec.output_channels, side, side), device="cuda", generator=gen)
    masks = torch.from_numpy((rng.random((batch, side, side)) < mask_frac).astype(np.uint8)).cuda()
    tr = DataParallelTrainer(plan, batch, side, side, lr=1e-9, use_graph=True)
    net = tr.net
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

    tr.load_batch(imgs, tgts, masks)
    ms_train = timed(tr.step)
    ms_fwd = timed(net.forward)
    px = batch * side * side
    tiers = net.kernel_plan()
    out = {"side": side, "images": batch, "mask_fraction": mask_frac,
           "train": px / (ms_train / 1e3), "forward": px / (ms_fwd / 1e3),
           "ms_train": ms_train, "ms_forward": ms_fwd,
           "conv_tiers": {str(k): v for k, v in tiers.items()}}
    del tr, net
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=64, help="images per GPU per step")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-sweep", action="store_true",
                    help="skip the image-size sweep and the c3 / c4 config lines")
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
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_1412_4526_b200 as dp
    from paper_1412_4526_b200 import engine
    from paper_1412_4526_b200.trainer import DataParallelTrainer

    spec = dp.parse_spec(C2_TEXT)
    plan = dp.compile_plan(spec)
    B = args.batch
    dev = torch.device("cuda", local)
    rng = np.random.default_rng(1234 + rank)
    # synthetic inputs, resident in HBM: two batches alternated step to step
    pool = []
    for _ in range(2):
        imgs = torch.from_numpy(rng.uniform(-0.5, 0.5, (B, 3, SIDE, SIDE)).astype(np.float32))
        tgts = torch.from_numpy(rng.uniform(-1, 1, (B, 10, SIDE, SIDE)).astype(np.float32))
        m = np.zeros((B, SIDE, SIDE), np.uint8)
        for b in range(B):
            m[b].flat[rng.choice(SIDE * SIDE, int(MASK_FRAC * SIDE * SIDE), replace=False)] = 1
        pool.append((imgs, tgts, torch.from_numpy(m)))
    dpool = [tuple(t.to(dev) for t in p) for p in pool]
    hpool = [tuple(t.pin_memory() for t in p) for p in pool]

    tr = DataParallelTrainer(plan, B, SIDE, SIDE, lr=1e-7, use_graph=not args.no_graph)
    net = tr.net
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

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
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

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
    from paper_1412_4526_b200.trainer import H2DPipeline
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
    ms_e2e = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms_e2e], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
    h2d = sum(t.numel() * t.element_size() for t in hpool[0])
    d2h = grad_host.numel() * grad_host.element_size()

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
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "r01_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            tj = json.load(fh)
        if top["name"] in tj.get("kernels", {}):
            traffic = tj["kernels"][top["name"]]["dram_bytes"]
            traffic_src = tj.get("source")
    roof.update({"kernel": top["name"], "ms_per_launch": top["ms"],
                 "share_of_step": top["ms"] / prof["step_ms"], "peak_source": peaks["source"],
                 "traffic": traffic, "traffic_source": traffic_src,
                 "note": ("tcgen05 kind::tf32 3xTF32 conv: algorithmic FLOPs (each MAC issues 3 "
                          "TF32 MACs); peak = measured dense bf16 (TF32 dense is half of it)"
                          if "_tc" in top["name"] else
                          "CUDA-core conv measured against the dense bf16 tensor peak")})

    line = {
        "metric": METRIC, "value": value, "unit": "pixels/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_train / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": "c2: 3x256x256 RGB, fwd + 1%-masked bwd (655 px/image), "
                               "squared-error delta, grad all-reduce, SGD",
                   "images_per_gpu_per_step": B, "side": SIDE, "mask_fraction": MASK_FRAC,
                   "net": "conv6/maxpool2/tanh/conv5/maxpool2/tanh/conv4 (16,32,10 ch), patch 29",
                   "parallelism": f"dp{world} (images sharded, NCCL all-reduce SUM)",
                   "l2": "working set >> L2 (activations %.1f GB per GPU)" %
                         (net.activation_bytes() / 1e9),
                   "cuda_graph": tr._graph is not None,
                   "precision": net.precision,
                   "conv_tiers": {str(k): v for k, v in net.kernel_plan().items()}},
        "forward": {"value": px_per_step / (ms_fwd / args.steps / 1e3), "unit": "pixels/s",
                    "ms_per_step": ms_fwd / args.steps},
        "e2e": {"value": px_per_step / (ms_e2e / args.steps / 1e3), "unit": "pixels/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches_in_region,
        "roofline": roof,
        "kernels": prof["kernels"],
        "clocks": clocks,
    }

    if rank == 0 and world == 1 and not args.no_sweep:
        # patch-by-patch baseline on the same GPU: every pixel's
        # 29x29 window classified on its own through the same fast-tier kernels
        import paper_1412_4526_b200 as dp_pkg
        one = dpool[0][0][:1]
        dp_pkg.patch_scan_forward(net.plan, one, batch=8192)
        torch.cuda.synchronize()
        q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        q0.record()
        dp_pkg.patch_scan_forward(net.plan, one, batch=8192)
        q1.record()
        torch.cuda.synchronize()
        ps = SIDE * SIDE / (q0.elapsed_time(q1) / 1e3)
        line["patch_scan_gpu"] = {
            "value": ps, "unit": "pixels/s",
            "dense_forward_over_patch_scan": line["forward"]["value"] / ps,
            "sample": "1 image of c2@256: 65536 windows, batches of 8192, same kernels"}

        # "per image size" (BASELINE metric) and the other BASELINE configs, same GPU
        sizes = []
        for side, b in ((128, 256), (512, 16), (1024, 4)):
            sizes.append(measure_config(C2_TEXT, side, b, MASK_FRAC))
        line["sizes"] = {"net": "c2 (conv6/pool2/tanh/conv5/pool2/tanh/conv4, 3 ch)",
                         "unit": "pixels/s", "points": sizes,
                         "note": "train = fwd + 1%-masked bwd + SGD; 256 is the headline line"}
        line["configs"] = {
            "c3_512": dict(measure_config(C3_TEXT, 512, 4, 1.0),
                           net="plain CNN1 (50,50,8), pool1 4x4, patch 69, full-image fwd/bwd"),
            "c4_1024": dict(measure_config(C4_TEXT, 1024, 2, MASK_FRAC),
                            net="5 conv (strides 2,1,1,2,1) / 3 max-pool, relu, patch 119"),
        }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        f, b, kind, how = cpu_dense_step_seconds(threads, 1)
        scan_px_s, scan_n = cpu_patch_scan_px_per_s()
        line["cpu_baseline"] = {
            "value": SIDE * SIDE / (f + b), "unit": "pixels/s", "cores": threads, "kind": kind,
            "sample": f"1 image of c2@256 (fwd + 1%-masked bwd), {how}, {threads} threads",
            "forward_value": SIDE * SIDE / f,
            "patch_scan_forward": {"value": scan_px_s, "unit": "pixels/s", "cores": 1,
                                   "sample": f"{scan_n} pixels on a 16-px grid, extrapolated"},
        }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

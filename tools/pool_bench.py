"""Pool kernels: the smem-tiled path (DP_POOL_STREAM=0) vs the warp-streaming max-pool
kernels (default; avg pools are smem in both) on config shapes -- bit-identity of the two and
CUDA-event GB/s.  python tools/pool_bench.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1412_4526_b200 import _lib  # noqa: E402
from paper_1412_4526_b200.engine import ops  # noqa: E402

# (name, n, c, h, w, p, d) -- pool INPUT shapes of the configs' pools
SHAPES = [
    ("c2 pool1", 64, 16, 266, 266, 2, 1),
    ("c2 pool2", 64, 32, 260, 260, 2, 2),
    ("c3 pool1", 8, 50, 575, 575, 4, 1),
    ("c3 pool2", 8, 50, 564, 564, 2, 4),
    ("c4 L4", 2, 64, 1134, 1134, 2, 2),
    ("c4 L7", 2, 96, 1124, 1124, 2, 4),
    ("c4 L10", 2, 128, 1104, 1104, 2, 16),
    ("plain p8 @512", 2, 50, 639, 639, 8, 1),
    ("plain p2 @512", 8, 50, 543, 543, 2, 1),
    ("c3 pool1 bs16", 16, 50, 575, 575, 4, 1),
    ("c3 pool2 bs16", 16, 50, 564, 564, 2, 4),
]


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run():
    for name, n, c, h, w, p, d in SHAPES:
        e = (p - 1) * d + 1
        ho, wo = h - e + 1, w - e + 1
        g = torch.Generator(device="cuda").manual_seed(1)
        x = torch.rand((n, c, h, w), device="cuda", generator=g) - 0.5
        x[:, :, ::5, ::3] = 0.125  # ties
        dy = torch.rand((n, c, ho, wo), device="cuda", generator=g) - 0.5
        gate = torch.rand((n, c, h, w), device="cuda", generator=g) - 0.5
        res = {}
        for mode in ("smem", "stream"):
            if mode == "smem":
                os.environ["DP_POOL_STREAM"] = "0"
            else:
                os.environ.pop("DP_POOL_STREAM", None)
            y = torch.empty((n, c, ho, wo), device="cuda")
            arg = torch.empty((n, c, ho, wo), device="cuda", dtype=torch.uint8)
            if "bs16" in name:
                # as in the c3 step: no gate; pool1's dx is the pitched layer-0 delta
                pitch = (w + 3) // 4 * 4
                dxs = torch.zeros((n, c, h, pitch), device="cuda")
                dx = dxs[..., :w]
                tf = timeit(lambda: ops.maxpool_forward(x, y, arg, p, d, _lib.DP_TANH_FAST))
                tb = timeit(lambda: ops.maxpool_backward(dy, arg, dx, p, d, dx_pitch=pitch))
            else:
                dx = torch.empty_like(x)
                tf = timeit(lambda: ops.maxpool_forward(x, y, arg, p, d, _lib.DP_TANH_FAST))
                tb = timeit(lambda: ops.maxpool_backward(dy, arg, dx, p, d, gate,
                                                         _lib.DP_TANH_FAST))
            ya = torch.empty_like(y)
            dxa = torch.empty_like(x)
            ta = timeit(lambda: ops.avgpool_forward(x, ya, p, d))
            tab = timeit(lambda: ops.avgpool_backward(dy, dxa, p, d, gate, _lib.DP_TANH_FAST))
            res[mode] = (tf, tb, ta, tab, y.clone(), arg.clone(), dx.clone(), ya.clone(), dxa.clone())
        same = all(torch.equal(a, b) for a, b in zip(res["smem"][4:], res["stream"][4:]))
        bf = 4 * (x.numel() + y.numel()) + arg.numel()
        bb = 4 * (dy.numel() + 2 * x.numel()) + arg.numel()
        ba = 4 * (x.numel() + y.numel())
        bab = 4 * (dy.numel() + 2 * x.numel())
        out = [f"{name:15s} same={same}"]
        for mode in ("smem", "stream"):
            tf, tb, ta, tab = res[mode][:4]
            out.append(f"{mode}: fwd {tf*1e3:7.1f}us {bf/tf/1e6:6.0f} GB/s  bwd {tb*1e3:7.1f}us "
                       f"{bb/tb/1e6:6.0f} GB/s  avg {ba/ta/1e6:5.0f}/{bab/tab/1e6:5.0f} GB/s")
        print("  ".join(out), flush=True)


if __name__ == "__main__":
    run()

"""c3 max-pool A/B: smem-tiled (DP_POOL_STREAM=0) vs warp-streaming kernels, forward with and
without the fused tanh, backward as in the step (no gate; pool1 dx pitched).
python tools/pool_ab.py [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1412_4526_b200 import _lib  # noqa: E402
from paper_1412_4526_b200.engine import ops  # noqa: E402

SHAPES = [("c3 pool1", 16, 50, 575, 575, 4, 1), ("c3 pool2", 16, 50, 564, 564, 2, 4),
          ("plain p8", 4, 50, 639, 639, 8, 1)]


def timeit(fn, reps):
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


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    for name, n, c, h, w, p, d in SHAPES:
        e = (p - 1) * d + 1
        ho, wo = h - e + 1, w - e + 1
        g = torch.Generator(device="cuda").manual_seed(1)
        x = torch.rand((n, c, h, w), device="cuda", generator=g) - 0.5
        dy = torch.rand((n, c, ho, wo), device="cuda", generator=g) - 0.5
        y = torch.empty((n, c, ho, wo), device="cuda")
        arg = torch.empty((n, c, ho, wo), device="cuda", dtype=torch.uint8)
        pitch = (w + 3) // 4 * 4
        dx = torch.zeros((n, c, h, pitch), device="cuda")[..., :w]
        bf = 4 * (x.numel() + y.numel()) + arg.numel()
        bb = 4 * (dy.numel() + x.numel()) + arg.numel()
        for mode in ("smem", "stream"):
            if mode == "smem":
                os.environ["DP_POOL_STREAM"] = "0"
            else:
                os.environ.pop("DP_POOL_STREAM", None)
            ti = timeit(lambda: ops.maxpool_forward(x, y, arg, p, d, _lib.DP_IDENTITY), reps)
            tt = timeit(lambda: ops.maxpool_forward(x, y, arg, p, d, _lib.DP_TANH_FAST), reps)
            tb = timeit(lambda: ops.maxpool_backward(dy, arg, dx, p, d, dx_pitch=pitch), reps)
            print(f"{name} {mode:6s} fwd id {ti*1e3:6.1f}us {bf/ti/1e6:5.0f} GB/s  "
                  f"fwd tanh {tt*1e3:6.1f}us {bf/tt/1e6:5.0f} GB/s  "
                  f"bwd {tb*1e3:6.1f}us {bb/tb/1e6:5.0f} GB/s", flush=True)


if __name__ == "__main__":
    main()

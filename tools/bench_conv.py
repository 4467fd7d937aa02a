"""Per-layer conv timing: exact CUDA-core tier vs tcgen05 3xTF32 tier (CUDA events).

    python tools/bench_conv.py [--batch 64]

Shapes are the c2 network's convs at 256x256, forward and
data gradient.  Prints ms per call and algorithmic TFLOP/s (2*Cout*Cin*k^2*Ho*Wo*N).
"""

import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1412_4526_b200.engine import ops  # noqa: E402

LAYERS = [  # name, cin, cout, k, d, Hin (square)
    ("conv1", 3, 16, 6, 1, 284),
    ("conv2", 16, 32, 5, 2, 278),
    ("conv3", 32, 10, 4, 4, 268),
]


def timeit(fn, reps=10):
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
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    a = ap.parse_args()
    N = a.batch
    for name, ci, co, k, d, H in LAYERS:
        e = (k - 1) * d + 1
        Ho = H - e + 1
        x = torch.randn(N, ci, H, H, device="cuda")
        w = torch.randn(co, ci, k, k, device="cuda") * 0.1
        b = torch.randn(co, device="cuda")
        y = torch.empty(N, co, Ho, Ho, device="cuda")
        dy = torch.randn(N, co, Ho, Ho, device="cuda")
        dx = torch.empty(N, ci, H, H, device="cuda")
        flops = 2.0 * co * ci * k * k * Ho * Ho * N
        t_ex = timeit(lambda: ops.conv_forward(x, w, b, y, k, d, 1))
        t_exb = timeit(lambda: ops.conv_backward_data(dy, w, dx, k, d))
        line = f"{name}: fwd exact {t_ex:.3f} ms ({flops / t_ex / 1e9:.1f} TF/s)"
        if ops.fast_supported(ci, co, k, d):
            ws = torch.empty(ops.fwd_fast_workspace(x, co, k, d) if os.environ.get("TAP", "1") == "1" else ops.fast_workspace(ci, co, k), dtype=torch.uint8, device="cuda")
            t_tc = timeit(lambda: ops.conv_forward_fast(x, w, b, y, k, d, 1, ws))
            line += f" | fwd tc {t_tc:.3f} ms ({flops / t_tc / 1e9:.1f} TF/s)"
        line += f" | dgrad exact {t_exb:.3f} ms ({flops / t_exb / 1e9:.1f} TF/s)"
        if ops.fast_supported(co, ci, k, d):
            wsb = torch.empty(ops.bwd_fast_workspace(dy, ci, k, d) if os.environ.get("TAP", "1") == "1" else ops.fast_workspace(co, ci, k), dtype=torch.uint8, device="cuda")
            t_tcb = timeit(lambda: ops.conv_backward_data_fast(dy, w, dx, k, d, wsb))
            line += f" | dgrad tc {t_tcb:.3f} ms ({flops / t_tcb / 1e9:.1f} TF/s)"
        print(line, flush=True)


if __name__ == "__main__":
    main()

"""Time the weight-gradient kernels (fast tcgen05 vs CUDA-core) on the c2 layer shapes.

    python tools/bench_wgrad.py [batch]
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1412_4526_b200.engine import ops  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 64
# (cin, hi, cout, k, d): c2 layer inputs at 256x256 (padded 284)
LAYERS = [(3, 284, 16, 6, 1), (16, 278, 32, 5, 2), (32, 268, 10, 4, 4)]


def timeit(f, reps=5):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for ci, hi, co, k, d in LAYERS:
    e = (k - 1) * d + 1
    ho = hi - e + 1
    x = torch.randn(N, ci, hi, hi, device="cuda")
    dy = torch.randn(N, co, ho, ho, device="cuda")
    dw = torch.empty(co, ci, k, k, device="cuda")
    db = torch.empty(co, device="cuda")
    flops = 2.0 * N * ho * ho * co * ci * k * k
    ws = torch.empty(ops.wgrad_fast_workspace(x, co, k, d), dtype=torch.uint8, device="cuda")
    tf = timeit(lambda: ops.conv_backward_kernel_fast(x, dy, dw, db, k, d, ws))
    ws2 = torch.empty(ops.wgrad_workspace(x, co, k, d), dtype=torch.uint8, device="cuda")
    te = timeit(lambda: ops.conv_backward_kernel(x, dy, dw, db, k, d, ws2))
    print(f"cin={ci:3d} cout={co:3d} k={k} d={d} hi={hi}: fast {tf:7.3f} ms "
          f"({flops / tf / 1e9:6.1f} TF/s)  cuda-core {te:7.3f} ms ({flops / te / 1e9:6.1f} TF/s)",
          flush=True)

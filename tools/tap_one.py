"""Run one fast conv (fwd or bwd) with the shape-aware (tap-stacked) workspace:
python tools/tap_one.py <fwd|bwd> n,ci,co,k,d,h [reps]"""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_1412_4526_b200.engine import ops  # noqa: E402

mode = sys.argv[1]
n, ci, co, k, d, h = [int(v) for v in sys.argv[2].split(",")]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
e = (k - 1) * d + 1
ho = h - e + 1
x = torch.randn(n, ci, h, h, device="cuda")
w = torch.randn(co, ci, k, k, device="cuda") * 0.1
b = torch.randn(co, device="cuda")
if mode == "fwd":
    y = torch.empty(n, co, ho, ho, device="cuda")
    ws = torch.empty(ops.fwd_fast_workspace(x, co, k, d), dtype=torch.uint8, device="cuda")
    f = lambda: ops.conv_forward_fast(x, w, b, y, k, d, 1, ws)  # noqa: E731
else:
    dy = torch.randn(n, co, ho, ho, device="cuda")
    ws = torch.empty(ops.bwd_fast_workspace(dy, ci, k, d), dtype=torch.uint8, device="cuda")
    f = lambda: ops.conv_backward_data_fast(dy, w, x, k, d, ws)  # noqa: E731
for _ in range(reps):
    f()
torch.cuda.synchronize()

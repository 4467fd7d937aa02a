"""One c2 layer's fast weight gradient (for ncu): python tools/wg_one.py <layer 0|1|2> [batch]"""
import sys
import torch
sys.path.insert(0, ".")
from paper_1412_4526_b200.engine import ops
LAYERS = [(3, 284, 16, 6, 1), (16, 278, 32, 5, 2), (32, 268, 10, 4, 4)]
ci, hi, co, k, d = LAYERS[int(sys.argv[1])]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 64
e = (k - 1) * d + 1
ho = hi - e + 1
x = torch.randn(N, ci, hi, hi, device="cuda")
dy = torch.randn(N, co, ho, ho, device="cuda")
dw = torch.empty(co, ci, k, k, device="cuda"); db = torch.empty(co, device="cuda")
ws = torch.empty(ops.wgrad_fast_workspace(x, co, k, d), dtype=torch.uint8, device="cuda")
for _ in range(2):
    ops.conv_backward_kernel_fast(x, dy, dw, db, k, d, ws)
torch.cuda.synchronize()
print("done")

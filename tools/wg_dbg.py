import sys
import torch
sys.path.insert(0, ".")
from paper_1412_4526_b200.engine import ops
n, ci, co, k, d, h, w = 2, 3, 16, 6, 1, 70, 75
x = torch.randn(n, ci, h, w, device="cuda")
e = (k - 1) * d + 1
dy = torch.randn(n, co, h - e + 1, w - e + 1, device="cuda")
dw = torch.empty(co, ci, k, k, device="cuda"); db = torch.empty(co, device="cuda")
ws = torch.empty(ops.wgrad_fast_workspace(x, co, k, d), dtype=torch.uint8, device="cuda")
ops.conv_backward_kernel_fast(x, dy, dw, db, k, d, ws)
torch.cuda.synchronize()
print("ok", dw.abs().max().item())

import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1412_4526_b200.engine import ops
shape = tuple(int(v) for v in sys.argv[1].split(","))
n, ci, co, k, d, h, w = shape
e = (k - 1) * d + 1
rng = np.random.default_rng(1)
x = torch.from_numpy(rng.uniform(-1, 1, (n, ci, h, w)).astype(np.float32)).cuda()
dy = torch.from_numpy(rng.uniform(-1, 1, (n, co, h - e + 1, w - e + 1)).astype(np.float32)).cuda()
dw64 = torch.empty((co, ci, k, k), dtype=torch.float64, device="cuda")
db64 = torch.empty(co, dtype=torch.float64, device="cuda")
ws64 = torch.empty(max(1, ops.wgrad_workspace(x.double(), co, k, d)), dtype=torch.uint8, device="cuda")
ops.conv_backward_kernel(x.double(), dy.double(), dw64, db64, k, d, ws64)
dw = torch.full((co, ci, k, k), float("nan"), device="cuda")
db = torch.full((co,), float("nan"), device="cuda")
ws = torch.empty(ops.wgrad_fast_workspace(x, co, k, d), dtype=torch.uint8, device="cuda")
ops.conv_backward_kernel_fast(x, dy, dw, db, k, d, ws)
torch.cuda.synchronize()
rel = float((dw.double() - dw64).abs().max() / dw64.abs().max())
bad = (dw.double() - dw64).abs() > 1e-4 * dw64.abs().max()
print(sys.argv[1], os.environ.get("DP_WG_J"), "rel", rel, "db", float((db.double()-db64).abs().max()), "bad idx", bad.nonzero()[:6].tolist())

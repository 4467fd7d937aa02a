"""Flat-conv forward vs the exact tier for one shape: python tools/flat_one.py n,ci,co,k,d,h,w"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
from paper_1412_4526_b200.engine import ops  # noqa: E402

n, ci, co, k, d, h, w = (int(v) for v in sys.argv[1].split(","))
rng = np.random.default_rng(1)
x = torch.from_numpy(rng.uniform(-1, 1, (n, ci, h, w)).astype(np.float32)).cuda()
wt = torch.from_numpy(rng.uniform(-0.5, 0.5, (co, ci, k, k)).astype(np.float32)).cuda()
b = torch.from_numpy(rng.uniform(-0.5, 0.5, co).astype(np.float32)).cuda()
e = (k - 1) * d + 1
yr = torch.empty((n, co, h - e + 1, w - e + 1), device="cuda")
y = torch.full_like(yr, float("nan"))
ops.conv_forward(x, wt, b, yr, k, d, 0)
ws = torch.empty(ops.fast_workspace(ci, co, k), dtype=torch.uint8, device="cuda")
ops.conv_forward_fast(x, wt, b, y, k, d, 0, ws)
torch.cuda.synchronize()
err = (y - yr).abs()
print(sys.argv[1], os.environ.get("DP_TF_MT"), "rel", float(err.max() / yr.abs().max()),
      "bad frac", float((err > 1e-3).float().mean()))

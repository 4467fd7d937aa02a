"""Timeline of the fast weight-gradient kernel (CTA 0): DP_WG_TRACE=1 python tools/wg_trace.py [layer]"""
import ctypes
import os
import sys

import numpy as np
import torch

os.environ["DP_WG_TRACE"] = "1"
sys.path.insert(0, ".")
from paper_1412_4526_b200 import _lib  # noqa: E402
from paper_1412_4526_b200.engine import ops  # noqa: E402

# c2 conv1..conv3 (N = 64), then c3 conv1..conv3 (N = 16)
LAYERS = [(3, 284, 16, 6, 1), (16, 278, 32, 5, 2), (32, 268, 10, 4, 4),
          (3, 580, 50, 6, 1), (50, 572, 50, 3, 4), (50, 560, 8, 7, 8)]
li = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ci, hi, co, k, d = LAYERS[li]
N = 64 if li < 3 else 16
e = (k - 1) * d + 1
ho = hi - e + 1
x = torch.randn(N, ci, hi, hi, device="cuda")
dy = torch.randn(N, co, ho, ho, device="cuda")
dw = torch.empty(co, ci, k, k, device="cuda")
db = torch.empty(co, device="cuda")
ws = torch.empty(ops.wgrad_fast_workspace(x, co, k, d), dtype=torch.uint8, device="cuda")
for _ in range(2):
    ops.conv_backward_kernel_fast(x, dy, dw, db, k, d, ws)
torch.cuda.synchronize()
buf = np.zeros((256, 16), dtype=np.uint64)
_lib.check(_lib.load().dp_debug_wgrad_trace(buf.ctypes.data_as(ctypes.c_void_p), buf.nbytes))
t0 = buf[0, 0]
names = ["tma", "prodrdy", "sfull", "Blo", "cvdone", "-", "-", "-", "mmwait", "mmissued", "mmrdy", "-",
         "-", "-", "-", "-"]
print("K-block  " + " ".join(f"{n:>7}" for n in names))
for kl in list(range(0, 12)) + list(range(100, 106)):
    row = buf[kl]
    print(f"{kl:7d}  " + " ".join(f"{int(v) - int(t0):7d}" if v else "      -" for v in row[:16]))
per = (int(buf[200, 9]) - int(buf[100, 9])) / 100 if buf[200, 9] and buf[100, 9] else 0
print(f"steady-state cycles per K-block (MMA issue, kb 100->200): {per:.0f}")

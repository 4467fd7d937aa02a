"""Per-unit timeline of the flat conv kernel (CTA 0):
python tools/tf_trace.py <fwd|bwd> <n,ci,co,k,d,h>
TF_CTA=<n>: trace CTA n instead of 0.  TF_FP16=1: forward input declared in fp16 range (the fp16-split TMA-fed kernel); TF_ACT=<code>
fused nonlinearity (default 0).  (An fp16 launch's tf32 fallback exits before tracing.)"""
import ctypes
import os
import sys

import numpy as np
import torch

os.environ["DP_TC_TRACE"] = os.environ.get("TF_CTA", "0")  # the CTA traced
sys.path.insert(0, ".")
from paper_1412_4526_b200 import _lib  # noqa: E402
from paper_1412_4526_b200.engine import ops  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "fwd"
n, ci, co, k, d, h = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "16,16,32,5,2,278").split(",")]
e = (k - 1) * d + 1
x = torch.randn(n, ci, h, h, device="cuda")
w = torch.randn(co, ci, k, k, device="cuda") * 0.1
b = torch.randn(co, device="cuda")
ho = h - e + 1
if mode == "fwd":
    y = torch.empty(n, co, ho, ho, device="cuda")
    x = x.clamp(-1, 1)
    ws = torch.empty(ops.fwd_fast_workspace(x, co, k, d), dtype=torch.uint8, device="cuda")
    act = int(os.environ.get("TF_ACT", "0"))
    f16 = os.environ.get("TF_FP16", "0") == "1"
    f = lambda: ops.conv_forward_fast(x, w, b, y, k, d, act, ws, fp16_range=f16)  # noqa: E731
else:
    dy = torch.randn(n, co, ho, ho, device="cuda")
    ws = torch.empty(ops.bwd_fast_workspace(dy, ci, k, d), dtype=torch.uint8, device="cuda")
    f = lambda: ops.conv_backward_data_fast(dy, w, x, k, d, ws)  # noqa: E731
f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
f()
e1.record()
torch.cuda.synchronize()
print(f"{mode} n={n} ci={ci} co={co} k={k} d={d} h={h}: {e0.elapsed_time(e1):.3f} ms")
buf = np.zeros((1024, 8), dtype=np.uint64)
_lib.check(_lib.load().dp_debug_conv_trace(buf.ctypes.data_as(ctypes.c_void_p), buf.nbytes))
t0 = int(buf[0, 0])
print("unit  ld_start  ld_done | mm_wait  mm_got  mm_done | ep_wait  ep_got  ep_done")
nz = [u for u in range(1024) if buf[u, 2]]
last = nz[-1] if nz else 0
rows = os.environ.get('ROWS')
sel = [int(v) for v in rows.split(',')] if rows else list(range(0, 12)) + list(range(last // 2, last // 2 + 12))
for u in (list(range(sel[0], sel[1])) if rows else sel):
    r = [int(v) - t0 if v else -1 for v in buf[u]]
    print(f"{u:4d} {r[0]:9d} {r[1]:8d} | {r[2]:8d} {r[3]:7d} {r[4]:8d} | {r[5]:8d} {r[6]:7d} {r[7]:8d}")
if last > 20:
    a, bb = last // 4, 3 * last // 4
    print(f"steady cycles per unit: {(int(buf[bb, 4]) - int(buf[a, 4])) / (bb - a):.0f} "
          f"(MMA issue {np.mean([int(buf[u, 4]) - int(buf[u, 3]) for u in range(a, bb)]):.0f}, "
          f"wait {np.mean([int(buf[u, 3]) - int(buf[u, 2]) for u in range(a, bb)]):.0f}, "
          f"load {np.mean([int(buf[u, 1]) - int(buf[u, 0]) for u in range(a, bb)]):.0f})")

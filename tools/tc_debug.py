"""Run tensor-core conv configs one per subprocess with a watchdog; report ok/hang/err."""

import subprocess
import sys

CASES = [
    # n, cin, cout, k, d, H
    (1, 16, 32, 5, 2, 40), (1, 16, 32, 5, 2, 120), (1, 16, 32, 5, 2, 278), (4, 16, 32, 5, 2, 278),
    (1, 3, 16, 6, 1, 284), (4, 3, 16, 6, 1, 284),
    (1, 32, 10, 4, 4, 268), (4, 32, 10, 4, 4, 268),
    (1, 16, 16, 3, 1, 278), (1, 8, 32, 3, 1, 278), (1, 16, 32, 4, 1, 278),
]

CODE = """
import sys, torch
sys.path.insert(0, '.')
from paper_1412_4526_b200.engine import ops
n, ci, co, k, d, H = {case}
e = (k - 1) * d + 1
x = torch.randn(n, ci, H, H, device='cuda'); w = torch.randn(co, ci, k, k, device='cuda') * .1
b = torch.randn(co, device='cuda'); y = torch.empty(n, co, H - e + 1, H - e + 1, device='cuda')
yr = torch.empty_like(y)
ws = torch.empty(ops.fast_workspace(ci, co, k), dtype=torch.uint8, device='cuda')
ops.conv_forward_fast(x, w, b, y, k, d, 0, ws); ops.conv_forward(x, w, b, yr, k, d, 0)
torch.cuda.synchronize()
print('relerr', float((y - yr).abs().max() / yr.abs().max()))
"""

for case in CASES:
    try:
        r = subprocess.run([sys.executable, "-c", CODE.format(case=case)], capture_output=True,
                           text=True, timeout=40)
        out = (r.stdout.strip() or r.stderr.strip().splitlines()[-1:])
        print(case, "rc", r.returncode, out, flush=True)
    except subprocess.TimeoutExpired:
        print(case, "HANG", flush=True)

"""SM clock / power / throttle reasons sampled WHILE one fast conv runs back to back for a few
seconds (power-cap check): python tools/clock_probe.py <n,ci,co,k,d,h> [seconds]"""
import os
import subprocess
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1412_4526_b200.engine import ops  # noqa: E402


def main():
    n, ci, co, k, d, h = [int(v) for v in sys.argv[1].split(",")]
    secs = float(sys.argv[2]) if len(sys.argv) > 2 else 4.0
    e = (k - 1) * d + 1
    ho = h - e + 1
    x = torch.rand((n, ci, h, h), device="cuda") * 2 - 1
    w = (torch.rand((co, ci, k, k), device="cuda") - 0.5) * 0.2
    b = torch.rand((co,), device="cuda") - 0.5
    y = torch.empty((n, co, ho, ho), device="cuda")
    ws = torch.empty(ops.fwd_fast_workspace(x, co, k, d), dtype=torch.uint8, device="cuda")

    def f():
        ops.conv_forward_fast(x, w, b, y, k, d, 0, ws, fp16_range=True)

    for _ in range(5):
        f()
    torch.cuda.synchronize()
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,"
                            "clocks_throttle_reasons.active", "--format=csv,noheader",
                            "-lms", "100"], stdout=subprocess.PIPE, text=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0, cnt = time.time(), 0
    e0.record()
    while time.time() - t0 < secs:
        for _ in range(20):
            f()
        cnt += 20
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    smi.terminate()
    lines = [ln.strip() for ln in smi.stdout.read().splitlines() if ln.strip()]
    mhz = sorted(int(ln.split(",")[0].split()[0]) for ln in lines)
    watts = sorted(float(ln.split(",")[1].split()[0]) for ln in lines)
    print(f"{sys.argv[1]}: {e0.elapsed_time(e1) / cnt:.3f} ms per call over {cnt}; "
          f"SM MHz median {mhz[len(mhz) // 2]} (min {mhz[0]}, max {mhz[-1]}), "
          f"power median {watts[len(watts) // 2]:.0f} W, reasons {sorted(set(ln.split(',')[2].strip() for ln in lines))}")


if __name__ == "__main__":
    main()

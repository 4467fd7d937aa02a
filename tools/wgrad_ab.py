"""A/B the fast weight gradient (x read in place as in the engine: buffers with slack) under
environment settings: python tools/wgrad_ab.py n,ci,co,k,d,h "DP_WG_PF=0" ...
Prints CUDA-event ms per call and the normwise difference of dw from the default."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1412_4526_b200.engine import SLACK_BYTES, _slack_empty, ops  # noqa: E402


def main():
    n, ci, co, k, d, h = [int(v) for v in sys.argv[1].split(",")]
    e = (k - 1) * d + 1
    ho = h - e + 1
    kw = {"dtype": torch.float32, "device": "cuda"}
    g = torch.Generator(device="cuda").manual_seed(0)
    x = _slack_empty((n, ci, h, h), kw)
    x.copy_(torch.rand((n, ci, h, h), generator=g, **kw) * 2 - 1)
    dy = torch.rand((n, co, ho, ho), generator=g, **kw) - 0.5
    dw = torch.empty((co, ci, k, k), **kw)
    db = torch.empty((co,), **kw)
    ws = torch.empty(ops.wgrad_fast_workspace(x, co, k, d), dtype=torch.uint8, device="cuda")
    base = None
    for var in [""] + sys.argv[2:]:
        keys = []
        for kv in filter(None, var.split(",")):
            kk, vv = kv.split("=")
            os.environ[kk] = vv
            keys.append(kk)
        f = lambda: ops.conv_backward_kernel_fast(x, dy, dw, db, k, d, ws,  # noqa: E731
                                                  x_slack=SLACK_BYTES)
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        if base is None:
            base = dw.clone()
        diff = float((dw - base).abs().max() / base.abs().max())
        print(f"wgrad {sys.argv[1]} [{var or 'default'}]: {ms:.3f} ms  diff {diff:.2e}", flush=True)
        for kk in keys:
            os.environ.pop(kk)


if __name__ == "__main__":
    main()

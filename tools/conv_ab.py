"""A/B one fast conv call (forward or data gradient, relayout + kernel) under several
environment settings in one process (the switches are read per call):

    python tools/conv_ab.py fwd n,ci,co,k,d,h "DP_TT_TR=1" "DP_TT_TR=2" "DP_TT_QS16=1" ...

AB_ACT=<code> fuses a nonlinearity into the forward (default 0: none, as in front of a pool);
AB_FP16=0 does not declare the forward input in fp16 range (default: declared, |x| <= 1).
Prints CUDA-event ms per call for the default and each setting, and the normwise difference
of each output from the default one."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1412_4526_b200.engine import ops  # noqa: E402


def main():
    mode = sys.argv[1]
    n, ci, co, k, d, h = [int(v) for v in sys.argv[2].split(",")]
    variants = [""] + sys.argv[3:]
    e = (k - 1) * d + 1
    ho = h - e + 1
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand((n, ci, h, h), device="cuda", generator=g) * 2 - 1
    w = (torch.rand((co, ci, k, k), device="cuda", generator=g) - 0.5) * 0.2
    b = torch.rand((co,), device="cuda", generator=g) - 0.5
    dy = torch.rand((n, co, ho, ho), device="cuda", generator=g) * 2 - 1
    base = None
    for var in variants:
        keys = []
        for kv in filter(None, var.split(",")):
            kk, vv = kv.split("=")
            os.environ[kk] = vv
            keys.append(kk)
        if mode == "fwd":
            out = torch.empty((n, co, ho, ho), device="cuda")
            ws = torch.empty(ops.fwd_fast_workspace(x, co, k, d), dtype=torch.uint8, device="cuda")
            act = int(os.environ.get("AB_ACT", "0"))  # fused nonlinearity code (0 = none)
            f16 = os.environ.get("AB_FP16", "1") == "1"  # input declared in fp16 range
            f = lambda: ops.conv_forward_fast(x, w, b, out, k, d, act, ws,  # noqa: E731
                                              fp16_range=f16)
        else:
            out = torch.empty((n, ci, h, h), device="cuda")
            ws = torch.empty(ops.bwd_fast_workspace(dy, ci, k, d), dtype=torch.uint8,
                             device="cuda")
            f = lambda: ops.conv_backward_data_fast(dy, w, out, k, d, ws)  # noqa: E731
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
            base = out.clone()
            diff = 0.0
        else:
            diff = float((out - base).abs().max() / base.abs().max())
        print(f"{mode} {sys.argv[2]} [{var or 'default'}]: {ms:.3f} ms  diff {diff:.2e}",
              flush=True)
        for kk in keys:
            os.environ.pop(kk)


if __name__ == "__main__":
    main()

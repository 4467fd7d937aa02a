"""fp16-split weight gradient vs the tf32 one (x read in place in both): normwise error vs
fp64 and CUDA-event time.  python tools/wgrad_f16_ab.py n,ci,co,k,d,h [...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1412_4526_b200.engine import SLACK_BYTES, _slack_empty, ops  # noqa: E402


def split16(x, kw16, shift):
    w = x.shape[3]
    shp = tuple(x.shape[:3]) + ((w + 7) // 8 * 8,)
    t = [_slack_empty(shp, kw16) for _ in range(4 if shift else 2)]
    ops.split_f16(x, *t, shift) if shift else ops.split_f16(x, *t)
    hi, lo = t[0], t[1]
    assert torch.equal(hi[..., :w], x.half())
    assert torch.equal(lo[..., :w], ((x - hi[..., :w].float()) * 2048.0).half())
    return t + [None, None] if not shift else t


def timeit(f, reps=10):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    for arg in sys.argv[1:]:
        n, ci, co, k, d, h = [int(v) for v in arg.split(",")]
        e = (k - 1) * d + 1
        ho = h - e + 1
        kw = {"dtype": torch.float32, "device": "cuda"}
        g = torch.Generator(device="cuda").manual_seed(0)
        x = _slack_empty((n, ci, h, h), kw)
        x.copy_(torch.tanh(torch.randn((n, ci, h, h), generator=g, **kw)))
        dy = (torch.rand((n, co, ho, ho), generator=g, **kw) - 0.5) * 1e-2
        if os.environ.get("BIG_DY"):  # one delta outside fp16's range: the tf32 fallback runs
            dy[0, 0, 0, 0] = 4e4
        shift = max(0, ops.wgrad_f16_shift(x, co, k, d))
        xh, xl, xhs, xls = split16(x, {"dtype": torch.float16, "device": "cuda"}, shift)
        ref_w = torch.empty((co, ci, k, k), dtype=torch.float64, device="cuda")
        ref_b = torch.empty((co,), dtype=torch.float64, device="cuda")
        ws64 = torch.empty(max(1, ops.wgrad_workspace(x.double(), co, k, d)), dtype=torch.uint8,
                           device="cuda")
        ops.conv_backward_kernel(x.double(), dy.double(), ref_w, ref_b, k, d, ws64)
        res = {}
        ws32 = torch.empty(ops.wgrad_fast_workspace(x, co, k, d), dtype=torch.uint8, device="cuda")
        nb16 = ops.wgrad_f16_workspace(x, co, k, d)
        ws16 = torch.empty(max(nb16, 16), dtype=torch.uint8, device="cuda")
        for name in ("tf32", "f16"):
            dw = torch.empty((co, ci, k, k), **kw)
            db = torch.empty((co,), **kw)
            if name == "tf32":
                f = lambda: ops.conv_backward_kernel_fast(x, dy, dw, db, k, d, ws32,  # noqa
                                                          x_slack=SLACK_BYTES)
            else:
                if not nb16:
                    print(arg, "f16 unsupported")
                    continue
                f = lambda: ops.conv_backward_kernel_fast_f16(x, xh, xl, dy, dw, db, k, d,  # noqa
                                                              ws16, SLACK_BYTES, x_hi_s=xhs,
                                                              x_lo_s=xls)
            ms = timeit(f)
            ew = float((dw.double() - ref_w).abs().max() / ref_w.abs().max())
            eb = float((db.double() - ref_b).abs().max() / ref_b.abs().max())
            print(f"{arg} {name}: {ms:.3f} ms  dw err {ew:.2e}  db err {eb:.2e}", flush=True)


if __name__ == "__main__":
    main()

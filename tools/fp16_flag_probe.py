"""Does an engine activation trip the fp16-split range flag?  Times the c3 head forward on the
engine's real conv3 input (after one c3 forward) with and without the fp16 path, and prints
the input's range.   python tools/fp16_flag_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1412_4526_b200 as dp  # noqa: E402
from paper_1412_4526_b200.engine import DenseNet, ops  # noqa: E402


def timed(f, reps=5):
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
    text = bench.C3_TEXT
    plan = dp.compile_plan(dp.parse_spec(text))
    net = DenseNet(plan, 4, 512, 512, train=False)
    x = torch.rand((4, 3, 512, 512), device="cuda") - 0.5
    net.set_input(x)
    net.forward()
    torch.cuda.synchronize()
    for gi, g in enumerate(net.groups):
        a = net._group_input(gi)
        print(gi, type(g.op).__name__, g.act, tuple(a.shape), "max|x| %.3g" % a.abs().max().item(),
              "finite", bool(torch.isfinite(a).all()), "fp16 input", net._fp16_input(gi))
    gi = 4
    xin = net._group_input(gi)
    op = net.groups[gi].op
    wt, b = net.params[net.groups[gi].first]
    y = torch.empty_like(net.acts[gi])
    for f16 in (True, False):
        ms = timed(lambda: ops.conv_forward_fast(xin, wt, b, y, op.base.kernel_size, op.dilation,
                                                 0, net._tc_ws, fp16_range=f16))
        print("head fwd fp16_range", f16, "%.3f ms" % ms)


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def train_probe(steps=40):
    """bench's c3 trainer: weight / activation range per step (NaN / overflow trips the flag)"""
    from paper_1412_4526_b200.trainer import DataParallelTrainer
    text, side, B, mf, _ = bench.CONFIGS["c3"]
    spec = dp.parse_spec(text)
    plan = dp.compile_plan(spec)
    imgs, tgts, masks = [t.cuda() for t in bench._synthetic(spec, B, side, mf, 1234, "cuda")]
    tr = DataParallelTrainer(plan, B, side, side, lr=bench.stable_lr(B, side, mf), use_graph=False)
    for s in range(steps):
        tr.load_batch(imgs, tgts, masks)
        tr.step()
        torch.cuda.synchronize()
        wmax = max(float(w.abs().max()) for w, _ in tr.net.params.values())
        amax = [float(a.abs().max()) for a in tr.net.acts]
        if s % 8 and s != steps - 1:
            continue
        print("step", s, "max|w| %.3g" % wmax, "max|act|", ["%.3g" % v for v in amax], flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "train":
    train_probe()

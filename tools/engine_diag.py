"""Fast vs exact fused engine on a small c1 case: argmax flips and teacher-forced grads."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import test_gpu_engine as t
import paper_1412_4526_b200 as dp
from paper_1412_4526_b200.engine import DenseNet
from paper_1412_4526_b200 import trainer

text, side, batch = t._c1_text(1), 40, 3
spec = dp.parse_spec(text); plan = dp.compile_plan(spec)
rng = np.random.default_rng(0)
imgs = rng.uniform(-0.5, 0.5, (batch, 1, side, side)).astype(np.float32)
tg = rng.uniform(-1, 1, (batch, 10, side, side)).astype(np.float32)
masks = (rng.random((batch, side, side)) < 0.05).astype(np.uint8)
engs = {}
for prec in ("exact", "fast"):
    e = DenseNet(plan, batch, side, side, precision=prec)
    e.set_input(torch.from_numpy(imgs).cuda()); e.forward(); engs[prec] = e
ex, fa = engs["exact"], engs["fast"]
for g in ex.args:
    print("argmax group", g, "flips", int((ex.args[g] != fa.args[g]).sum()), "of", ex.args[g].numel())
for forced in (False, True):
    if forced:
        for g in ex.args: fa.args[g].copy_(ex.args[g])
        for xe, xf in zip(ex.acts, fa.acts): xf.copy_(xe)
    for e in (ex, fa):
        e.target.copy_(torch.from_numpy(tg)); e.mask.copy_(torch.from_numpy(masks)); e.loss_delta(); e.backward()
    torch.cuda.synchronize()
    ke, be = trainer.unflatten(spec, ex.grad_flat.double().cpu().numpy())
    kf, bf = trainer.unflatten(spec, fa.grad_flat.double().cpu().numpy())
    for k in range(len(spec.layers)):
        if ke[k] is not None:
            print("forced" if forced else "free", k, t.rel_err(kf[k], ke[k]), t.rel_err(bf[k], be[k]))

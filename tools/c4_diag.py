"""c4 at side 160: exact vs fast tier -- forward agreement and argmax-map flips."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1412_4526_b200 as dp  # noqa: E402
from paper_1412_4526_b200.engine import DenseNet  # noqa: E402
sys.path.insert(0, "tests")
from test_gpu_engine import C4_TEXT  # noqa: E402

spec = dp.parse_spec(C4_TEXT)
plan = dp.compile_plan(spec)
side = 160
rng = np.random.default_rng(0)
img = torch.from_numpy(rng.uniform(-0.5, 0.5, (1, 3, side, side)).astype(np.float32)).cuda()
engs = {}
for prec in ("exact", "fast"):
    e = DenseNet(plan, 1, side, side, precision=prec)
    e.set_input(img)
    e.forward()
    engs[prec] = e
torch.cuda.synchronize()
a, b = engs["exact"], engs["fast"]
for gi in a.args:
    diff = (a.args[gi] != b.args[gi]).sum().item()
    print(f"group {gi}: argmax flips {diff} of {a.args[gi].numel()}")
for gi, (x, y) in enumerate(zip(a.acts, b.acts)):
    r = ((x.double() - y.double()).abs().max() / y.double().abs().max()).item()
    print(f"group {gi} act rel diff {r:.3e}")

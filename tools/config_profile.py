"""Per-kernel CUDA-event breakdown of one eager training step for a bench config:
python tools/config_profile.py <c2|c3|c4> [side] [batch]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1412_4526_b200 as dp  # noqa: E402
from paper_1412_4526_b200 import engine  # noqa: E402
from paper_1412_4526_b200.trainer import DataParallelTrainer  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
text = {"c2": bench.C2_TEXT, "c3": bench.C3_TEXT, "c4": bench.C4_TEXT}[name]
side = int(sys.argv[2]) if len(sys.argv) > 2 else {"c2": 256, "c3": 512, "c4": 1024}[name]
batch = int(sys.argv[3]) if len(sys.argv) > 3 else {"c2": 64, "c3": 4, "c4": 2}[name]
spec = dp.parse_spec(text)
plan = dp.compile_plan(spec)
tr = DataParallelTrainer(plan, batch, side, side, lr=bench.stable_lr(batch, side, 0.01),
                        use_graph=False)
imgs = torch.rand((batch, spec.input_channels, side, side), device="cuda") - 0.5
tgts = torch.rand((batch, spec.output_channels, side, side), device="cuda")
masks = (torch.rand((batch, side, side), device="cuda") < 0.01).to(torch.uint8)
tr.load_batch(imgs, tgts, masks)
for _ in range(2):
    tr.step()
prof = engine.profile_step(tr, reps=3)
print(json.dumps({"config": name, "side": side, "batch": batch,
                  "plan": {str(k): v for k, v in tr.net.kernel_plan().items()}}))
tot = 0
for k in prof["kernels"]:
    tot += k["ms"]
    extra = f"{k['tflops']:.1f} TF/s" if k["bound"] == "tensor" else f"{k['gbs']:.0f} GB/s"
    print(f"{k['name']:32s} {k['ms']:8.3f} ms  {extra}")
print(f"total {tot:.3f} ms")

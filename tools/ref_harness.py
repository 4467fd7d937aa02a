"""The reference's own bench harness with this repo's backends registered (drop-in, per-call
H2D/D2H: "cuda" = exact tier through dp_host_*, "cuda-fast" = fp32 convs on the tcgen05
tier): python tools/ref_harness.py [side] [reps] [c2|c3] > report.txt"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
from denseprop import backend, bench  # noqa: E402
from denseprop.netspec import parse_spec  # noqa: E402

import bench as our_bench  # noqa: E402
from paper_1412_4526_b200 import cuda_fast_kernels, cuda_kernels  # noqa: E402

backend._BACKENDS["cuda"] = cuda_kernels
backend._BACKENDS["cuda-fast"] = cuda_fast_kernels
side = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = sys.argv[3] if len(sys.argv) > 3 else "c2"
spec = parse_spec({"c2": our_bench.C2_TEXT, "c3": our_bench.C3_TEXT}[cfg])
threads = os.cpu_count() or 1
rep = bench.compare_backends(spec, image_side=side, reps=reps, dtype=np.float32, threads=threads)
print(f"# reference bench.compare_backends, {cfg} at {side}x{side}, fp32, full mask, "
      f"{threads} host threads for the CPU backends; cuda / cuda-fast = drop-in per-call path")
print(rep.format_table())

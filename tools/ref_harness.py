"""The reference's own bench harness with this repo's backend registered (drop-in, per-call
H2D/D2H through dp_host_*): python tools/ref_harness.py [side] [reps] > report.txt"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
from denseprop import backend, bench  # noqa: E402
from denseprop.netspec import parse_spec  # noqa: E402

import bench as our_bench  # noqa: E402
from paper_1412_4526_b200 import cuda_kernels  # noqa: E402

backend._BACKENDS["cuda"] = cuda_kernels
side = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
spec = parse_spec(our_bench.C2_TEXT)
threads = os.cpu_count() or 1
rep = bench.compare_backends(spec, image_side=side, reps=reps, dtype=np.float32, threads=threads)
print(f"# reference bench.compare_backends, c2 at {side}x{side}, fp32, full mask, "
      f"{threads} host threads for the CPU backends; cuda = drop-in per-call path")
print(rep.format_table())

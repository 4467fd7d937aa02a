#!/usr/bin/env bash
# One GPU-box pass: gpu tests, smoke, bench, launch list, full ncu captures of the top kernels.
# usage: bash tools/gpu_check.sh <tag> [ncu-kernel-regex ...]
set -u
TAG=${1:-run}; shift || true
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph > $OUT/ncu_bench.log 2>&1
for k in "$@"; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 3 -c 1 \
     -o $OUT/full_${k//[^a-zA-Z0-9]/_} python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph \
     > $OUT/ncu_full_${k//[^a-zA-Z0-9]/_}.log 2>&1
done
echo done

#!/usr/bin/env bash
# One GPU-box pass for a round checkpoint: full gpu tests (parity numbers logged), smoke, the
# default bench, the reference arm, the c3 launch list and full ncu captures of one step.
# usage: bash tools/round_check.sh <tag>
TAG=${1:-check}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
DP_PARITY_LOG=$OUT/parity.jsonl timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
bash tools/profile_c3.sh $OUT/prof 16
echo done

#!/usr/bin/env bash
# c3@512 headline: launch list of 2 eager steps + one full ncu capture per conv/pool launch of
# one eager training step.  usage: bash tools/profile_c3.sh <outdir> [batch]
OUT=${1:-gpurun_out/prof_c3}; B=${2:-16}; mkdir -p $OUT
ARGS="--config c3 --batch $B --no-cpu-baseline --no-graph --no-sweep"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
   python bench.py --steps 2 --warmup 3 $ARGS > $OUT/ncu_launch.log 2>&1
# warm-up steps are eager too: skip the first 2 steps' launches of our kernels (capture step 3)
timeout 1500 ncu --set full --clock-control none --import-source on \
   -k "regex:tc_conv|tc_wgrad|maxpool|tc_stage|tc_relayout|mask" -s 40 -c 20 \
   -o $OUT/full_step python bench.py --steps 1 --warmup 3 $ARGS > $OUT/ncu_full.log 2>&1
echo done

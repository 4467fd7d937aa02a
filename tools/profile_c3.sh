#!/usr/bin/env bash
# c3@512 headline: launch list of 2 eager steps + one full ncu capture of one eager training
# step's conv / pool / staging launches, summarised on the box (gpurun copies back <= 64 MiB,
# so the .ncu-rep is reduced to its raw CSV + the step summary and removed).
# usage: bash tools/profile_c3.sh <outdir> [batch]
OUT=${1:-gpurun_out/prof_c3}; B=${2:-16}; mkdir -p $OUT
ARGS="--config c3 --batch $B --no-cpu-baseline --no-graph --no-sweep"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
   python bench.py --steps 2 --warmup 3 $ARGS > $OUT/ncu_launch.log 2>&1
# warm-up steps are eager too: skip the first steps' launches of our kernels
timeout 1500 ncu --set full --clock-control none --import-source on \
   -k "regex:tc_conv|tc_wgrad|maxpool|tc_stage|tc_relayout|mask" -s 40 -c 31 \
   -o $OUT/full_step python bench.py --steps 1 --warmup 3 $ARGS > $OUT/ncu_full.log 2>&1
ncu -i $OUT/full_step.ncu-rep --page raw --csv > $OUT/full_step_raw.csv 2>/dev/null
python tools/step_traffic.py $OUT/full_step.ncu-rep $OUT/traffic_c3.json $OUT/ncu_c3.md \
   "$OUT (tools/profile_c3.sh)" > $OUT/step_traffic.log 2>&1
python tools/ncu_summary.py launches $OUT/launches.csv > $OUT/launches.md 2>&1
SZ=$(stat -c %s $OUT/full_step.ncu-rep 2>/dev/null || echo 0)
if [ "$SZ" -gt 30000000 ]; then rm -f $OUT/full_step.ncu-rep; fi
echo done

#!/usr/bin/env bash
# Launch list (all kernels of 2 eager steps) + full ncu captures of the top kernels.
# usage: bash tools/profile_round.sh <outdir>
OUT=${1:-gpurun_out/prof}; mkdir -p $OUT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph --no-sweep > $OUT/ncu_launch.log 2>&1
# full captures: skip the warm-up launches of each kernel, take one
for k in "tc_conv_flat_kernel<true, false>" "tc_conv_flat_kernel<true, true>" tc_wgrad_kernel \
         maxpool_fwd_tile maxpool_bwd_tile tc_stage_x; do
  tag=$(echo "$k" | tr -c 'a-zA-Z0-9' '_')
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${k//</\\<}" -s 5 -c 1 \
     -o $OUT/full_$tag python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph --no-sweep \
     > $OUT/ncu_$tag.log 2>&1
done
echo done

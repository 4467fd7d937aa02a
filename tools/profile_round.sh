#!/usr/bin/env bash
# Launch list (all kernels of 2 eager steps) + full ncu captures of the step's main launches.
# usage: bash tools/profile_round.sh <outdir>
# The -s skip counts pick, in the eager training warm-up, the launch the bench line names:
#   flat conv 3/step (fwd 00, 02; data grad 07): skip 4 = 02 (conv2);
#   tap-stacked conv 2/step (fwd 04; data grad 10): skip 4 = 04, skip 5 = 10;
#   weight grad 3/step (06,09,12) -> skip 4 = 09; pool fwd 2/step (01,03) -> skip 5 = 03;
#   pool bwd 2/step (08,11) -> skip 4 = 08; x staging 3/step -> skip 4 (conv2's)
OUT=${1:-gpurun_out/prof}; mkdir -p $OUT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph --no-sweep > $OUT/ncu_launch.log 2>&1
cap() {  # name regex skip
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$2" -s $3 -c 1 \
     -o $OUT/full_$1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph --no-sweep \
     > $OUT/ncu_$1.log 2>&1
}
cap 02_conv_forward_tc tc_conv_flat_kernel 4
cap 04_conv_forward_tc tc_conv_tap_kernel 4
cap 10_conv_backward_data_tc tc_conv_tap_kernel 5
cap 09_conv_backward_kernel_tc tc_wgrad_ss_kernel 4
cap 03_maxpool_forward maxpool_fwd_tile 5
cap 08_maxpool_backward maxpool_bwd_tile 4
cap stage_x tc_stage_x 2
cap relayout tc_relayout 5
echo done

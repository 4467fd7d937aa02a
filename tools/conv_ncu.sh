#!/usr/bin/env bash
# ncu --set full of single c3 conv launches (tools/conv_ab.py), source + details pages
# summarised on the box: bash tools/conv_ncu.sh <outdir>
OUT=${1:-gpurun_out/conv_ncu}; mkdir -p $OUT
run() {  # name mode shape kernel-regex skip
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$4 -s $5 -c 1 \
     -o $OUT/$1 -f python tools/conv_ab.py $2 $3 > $OUT/$1.log 2>&1
  ncu -i $OUT/$1.ncu-rep --page source --csv > $OUT/$1.src.csv 2>&1
  ncu -i $OUT/$1.ncu-rep --page details --csv > $OUT/$1.details.csv 2>&1
  rm -f $OUT/$1.ncu-rep
}
run conv1_fwd fwd 16,3,50,6,1,580 tc_conv_flat_kernel 3
run conv2_fwd fwd 16,50,50,3,4,572 tc_conv_flat_kernel 4
run conv2_dgrad bwd 16,50,50,3,4,572 tc_conv_flat_kernel 4
run conv3_dgrad bwd 16,50,8,7,8,560 tc_conv_flat_kernel 3
run conv3_fwd fwd 16,50,8,7,8,560 tc_conv_tap_kernel 3
ls -la $OUT

#!/usr/bin/env bash
# ncu --set full of one streaming max-pool forward launch per c3 pool (tanh fused):
# bash tools/pool_ncu2.sh <outdir>
OUT=${1:-gpurun_out/pool_ncu2}; mkdir -p $OUT
# pool_ab launch order per mode: fwd id x4, fwd tanh x4, bwd x4; stream mode follows smem
timeout 300 ncu --set full --clock-control none --import-source on -k regex:maxpool_fwd_stream \
   -s 4 -c 1 -o $OUT/fwd1 -f python tools/pool_ab.py 1 > $OUT/fwd1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:maxpool_fwd_stream \
   -s 12 -c 1 -o $OUT/fwd2 -f python tools/pool_ab.py 1 > $OUT/fwd2.log 2>&1
for K in fwd1 fwd2; do
  ncu -i $OUT/$K.ncu-rep --page source --csv > $OUT/$K.src.csv 2>&1
  ncu -i $OUT/$K.ncu-rep --page details --csv > $OUT/$K.details.csv 2>&1
done
ls -la $OUT

timeout 300 python -m pytest tests/test_gpu_tc.py -q -x 2>&1 | tail -2
for c in "fwd 64,32,10,4,4,268" "fwd 64,16,32,5,2,278" "bwd 64,16,32,5,2,278" "bwd 64,32,10,4,4,268" "fwd 64,3,16,6,1,284" "fwd 1,96,128,3,8,1124" "bwd 1,96,128,3,8,1120" "fwd 4,50,8,7,8,560"; do timeout 60 python tools/tc_trace.py $c | sed -n "1p"; done

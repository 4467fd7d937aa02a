timeout 200 python -m pytest tests/test_gpu_tc.py -q -x -k weight 2>&1 | tail -3
timeout 60 python tools/bench_wgrad.py 64 2>&1
for l in 0 1 2; do timeout 60 python tools/wg_trace.py $l 2>&1 | tail -1; done
timeout 60 python tools/wg_trace.py 1 2>&1 | sed -n '1p;14,17p'

timeout 120 python -m pytest tests/test_gpu_tc.py -q -x -k weight 2>&1 | tail -2
for v in 0 42; do echo "== dbg $v"; DP_WG_DBG=$v timeout 60 python tools/wg_trace.py 1 2>&1 | sed -n '1p;14,17p;20p'; done
timeout 60 python tools/bench_wgrad.py 64 2>&1

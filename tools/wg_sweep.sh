for v in 34 32 2 0; do echo "== dbg $v"; DP_WG_DBG=$v timeout 60 python tools/wg_trace.py 1 2>&1 | sed -n '1p;14,16p;20p'; done

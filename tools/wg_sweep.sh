for gg in 2 1; do echo "G<=$gg"; DP_WG_G=$gg timeout 60 python tools/bench_wgrad.py 64 2>&1; done

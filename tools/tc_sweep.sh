for v in 15 8 9; do timeout 60 tools/tc_trace 64,16,32,5,2,278 $v 120 | sed -n '2p;100,104p'; done

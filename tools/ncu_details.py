"""Print selected rows of an `ncu --page details --csv` export (first kernel):
python tools/ncu_details.py <details.csv> [regex]"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[0]
pat = re.compile(sys.argv[2] if len(sys.argv) > 2 else
                 "Duration|Throughput|Issue|Occupancy|Warp Cycles|Eligible|Active Warps|"
                 "Executed Ipc|Registers|Shared Memory|Stall|Block Limit", re.I)
iS, iN, iU, iV = (h.index(k) for k in ("Section Name", "Metric Name", "Metric Unit",
                                        "Metric Value"))
first = rows[1][h.index("ID")] if "ID" in h else None
for r in rows[1:]:
    if first is not None and r[h.index("ID")] != first:
        break
    if pat.search(r[iN]):
        print(f"{r[iS][:28]:28s} {r[iN][:48]:48s} {r[iV]:>14s} {r[iU]}")

"""Summarise an `ncu --page source --csv` (SASS view) export: instructions executed per opcode
and the instructions with the most warp-stall samples.  python tools/sass_hot.py <src.csv> [n]"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    rows = list(csv.reader(open(path)))
    h = rows[1]
    body = [r for r in rows[2:] if len(r) == len(h)]
    iS, iE, iW = h.index("Source"), h.index("Instructions Executed"), h.index(
        "Warp Stall Sampling (All Samples)")
    ops = collections.Counter()
    tot = 0
    for r in body:
        e = int(r[iE] or 0)
        op = r[iS].split()[0] if r[iS].split() else "?"
        if op.startswith("@"):
            op = r[iS].split()[1]
        ops[op.split(".")[0]] += e
        tot += e
    print(f"total warp instructions executed: {tot}")
    for op, e in ops.most_common(n):
        print(f"  {op:10s} {e:12d} {100 * e / tot:5.1f} %")
    print("hottest (stall samples):")
    for r in sorted(body, key=lambda r: -int(r[iW] or 0))[:n]:
        print(f"  {int(r[iW] or 0):7d} {int(r[iE] or 0):10d}  {r[iS].strip()[:90]}")


if __name__ == "__main__":
    main()

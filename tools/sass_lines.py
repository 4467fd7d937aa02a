"""Attribute an `ncu --page source --csv` (SASS view) export to CUDA source lines using the
-lineinfo of the built library:

    python tools/sass_lines.py <src.csv> <file.cu> [n]

Extracts the kernel's cubin from paper_1412_4526_b200/libdenseprop_b200.so (cuobjdump),
maps each SASS offset to its source line (nvdisasm -g) and prints, per source line, the
instructions executed and warp-stall samples, hottest first."""
import collections
import csv
import glob
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1412_4526_b200", "libdenseprop_b200.so")


def demangle_match(kernel_name, mangled):
    return True


def main():
    src_csv, cu = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    rows = list(csv.reader(open(src_csv)))
    kname = rows[0][1]
    h = rows[1]
    body = [r for r in rows[2:] if len(r) == len(h)]
    iA, iS, iE, iW = (h.index(k) for k in ("Address", "Source", "Instructions Executed",
                                           "Warp Stall Sampling (All Samples)"))
    base = int(body[0][iA], 16)
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", LIB], cwd=tmp, capture_output=True)
    stem = os.path.splitext(os.path.basename(cu))[0]
    cub = glob.glob(os.path.join(tmp, stem + ".*.cubin"))[0]
    dis = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    # functions: pick the one whose SASS matches the ncu listing (first 8 instructions)
    funcs = re.split(r"\n(?=\.text\.)", dis)
    # the kernel: the function whose whole SASS listing matches the ncu one
    want = [r[iS].replace(" ", "").rstrip(";") for r in body]
    best = None
    for f in funcs:
        ins = re.findall(r"/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", f)
        got = [t.replace(" ", "") for _, t in ins]
        if abs(len(got) - len(want)) > 8:
            continue
        score = sum(a == b for a, b in zip(want, got))
        if best is None or score > best[0]:
            best = (score, f)
    f = best[1]
    line_of = {}
    cur = None
    for ln in f.splitlines():
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            line_of[int(m.group(1), 16)] = cur
    agg = collections.defaultdict(lambda: [0, 0])
    for r in body:
        off = int(r[iA], 16) - base
        key = line_of.get(off, ("?", 0))
        agg[key][0] += int(r[iE] or 0)
        agg[key][1] += int(r[iW] or 0)
    texts = {}
    for fn in set(k[0] for k in agg):
        p = os.path.join(ROOT, "paper_1412_4526_b200", "csrc", fn)
        if os.path.exists(p):
            texts[fn] = open(p).read().splitlines()
    tot_e = sum(v[0] for v in agg.values())
    tot_w = sum(v[1] for v in agg.values())
    print(f"{kname[:100]}\nmatch score {best[0]}/{len(want)}, instructions {tot_e}, stall samples {tot_w}")
    print("   stall%  inst%   file:line  source")
    for (fn, ln), (e, w) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:n]:
        t = texts.get(fn, [])
        s = t[ln - 1].strip()[:80] if 0 < ln <= len(t) else ""
        print(f"  {100 * w / max(tot_w, 1):6.1f} {100 * e / max(tot_e, 1):6.1f}  {fn}:{ln:<5d} {s}")


if __name__ == "__main__":
    main()

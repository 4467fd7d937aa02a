"""Write profiles/<name>_traffic.json: per bench-line kernel name, the DRAM bytes of one launch
from the full ncu captures made by tools/profile_round.sh.

    python tools/traffic_json.py <capture dir> <out json> [source note]
"""
import csv
import glob
import io
import json
import os
import subprocess
import sys


def one(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rd = list(csv.reader(io.StringIO(raw)))
    d = dict(zip(rd[0], rd[2]))
    u = dict(zip(rd[0], rd[1]))

    def val(k):
        v = float(d[k].replace(",", ""))
        unit = u.get(k, "")
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)

    return {"kernel": d.get("Kernel Name", "?")[:160],
            "dram_bytes": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
            "gpu_time_us": float(d["gpu__time_duration.sum"].replace(",", "")) *
            (1e3 if u.get("gpu__time_duration.sum") == "ms" else 1)}


def main():
    src, out = sys.argv[1], sys.argv[2]
    note = sys.argv[3] if len(sys.argv) > 3 else src
    ks = {}
    for p in sorted(glob.glob(os.path.join(src, "full_*.ncu-rep"))):
        tag = os.path.basename(p)[5:-8]
        if tag[:2].isdigit():
            name = tag[:2] + ":" + tag[3:]
            ks[name] = one(p)
    with open(out, "w") as fh:
        json.dump({"source": note, "kernels": ks}, fh, indent=1)
    print(json.dumps(ks, indent=1))


if __name__ == "__main__":
    main()

"""Summarise ncu outputs brought back from the GPU box into profiles/ (markdown).

    python tools/ncu_summary.py launches <launches.csv>            # per-kernel time shares
    python tools/ncu_summary.py report <prof.ncu-rep> [...]        # key metrics of a full capture
"""

from __future__ import annotations

import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__occupancy_limit_registers",
    "smsp__average_warp_latency_issue_stalled_barrier",
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_mio_throttle",
    "smsp__pcsamp_warps_issue_stalled_barrier",
    "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
    "smsp__pcsamp_warps_issue_stalled_wait",
    "smsp__pcsamp_warps_issue_stalled_lg_throttle",
]


def launches(path):
    rows = []
    with open(path) as fh:
        text = fh.read()
    start = text.index('"ID"')
    for r in csv.DictReader(io.StringIO(text[start:])):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((r["Kernel Name"], float(r["Metric Value"])))
    agg = defaultdict(lambda: [0, 0.0])
    for name, ns in rows:
        short = re.sub(r"\(.*", "", name)
        short = re.sub(r"^void ", "", short)
        agg[short][0] += 1
        agg[short][1] += ns
    total = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | total ms | mean us | share |", "|---|---|---|---|---|"]
    for name, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{name[:90]}` | {n} | {ns / 1e6:.3f} | {ns / n / 1e3:.1f} | "
                   f"{100 * ns / total:.1f}% |")
    out.append(f"\n{len(rows)} launches, {total / 1e6:.3f} ms total (cold-cache, serialised by ncu)")
    return "\n".join(out)


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rd = list(csv.reader(io.StringIO(raw)))
    if len(rd) < 3:
        return f"(no data in {path})"
    hdr, units = rd[0], rd[1]
    out = []
    for row in rd[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        out.append(f"### `{d.get('Kernel Name', '?')[:120]}`\n")
        out.append("| metric | value |\n|---|---|")
        for k in KEYS:
            if k in d:
                out.append(f"| {k} | {d[k]} {u.get(k, '')} |")
        out.append("")
    return "\n".join(out)


if __name__ == "__main__":
    mode = sys.argv[1]
    for p in sys.argv[2:]:
        print(launches(p) if mode == "launches" else report(p))

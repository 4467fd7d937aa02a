"""Per bench-record DRAM traffic from a one-step full ncu capture (tools/profile_c3.sh):

    python tools/step_traffic.py <full_step.ncu-rep | raw.csv> <out json> <out md> [source note]

The capture holds ~one eager c3 training step (`-s 40 -c 20`) starting anywhere in it; SEQ,
the step's launch sequence, assigns each captured launch to the bench `kernels` record that
times it (a record = the staging / relayout launches + the main kernel of one op).  Writes the json
bench.py reads for `roofline.traffic` and a markdown summary for profiles/."""
import csv
import io
import json
import subprocess
import sys

# one c3 training step in issue order: (kernel-name fragment, bench record); weight packs and
# reductions are outside the capture's kernel filter, an fp16-split layer's tf32 fallback
# launch (which exits at once) is inside.  The capture starts anywhere in a step; the
# sequence is matched cyclically against it.
SEQ = [("tc_relayout_f16_pk<1, 3", "00:conv_forward_tc"),
       ("tc_conv_flat_kernel<1, 0, 1, 1, 1>", "00:conv_forward_tc"),
       ("tc_conv_flat_kernel<1, 0, 3, 0, 0>", "00:conv_forward_tc"),
       ("maxpool_fwd_stream", "01:maxpool_forward"),
       ("tc_relayout_f16<0>", "02:conv_forward_tc"), ("tc_relayout_f16_pk<0,", "02:conv_forward_tc"),
       ("tc_conv_flat_kernel<0, 0, 1, 1, 0>", "02:conv_forward_tc"),
       ("tc_conv_flat_kernel<0, 0, 0, 0, 0>", "02:conv_forward_tc"),
       ("maxpool_fwd_stream", "03:maxpool_forward"),
       ("tc_relayout_f16<0>", "04:conv_forward_tc"), ("tc_conv_tap_kernel<0, 1>", "04:conv_forward_tc"),
       ("tc_conv_flat_kernel<1, 0, 0, 0, 0>", "04:conv_forward_tc"),
       ("mask_delta", "05:mask_delta"), ("tc_stage_dy16", "06:conv_backward_kernel_tc"),
       ("tc_wgrad_ss", "06:conv_backward_kernel_tc"),
       # the fp16 weight gradient's gated tf32 fallback (dy staging, kernel: exit at once)
       ("tc_stage_dy", "06:conv_backward_kernel_tc"), ("tc_wgrad_ss", "06:conv_backward_kernel_tc"),
       ("tc_relayout_f16_pk<1,", "07:conv_backward_data_tc"),
       ("tc_conv_flat_kernel<1, 1, 1, 1, 0>", "07:conv_backward_data_tc"),
       ("tc_conv_flat_kernel<1, 1, 0, 0, 0>", "07:conv_backward_data_tc"),
       ("maxpool_bwd_stream", "08:maxpool_backward"), ("tc_wgrad_ss", "09:conv_backward_kernel_tc"),
       ("tc_relayout_f16<1>", "10:conv_backward_data_tc"),
       ("tc_relayout_f16_pk<1,", "10:conv_backward_data_tc"),
       ("tc_conv_flat_kernel<1, 1, 1, 1, 0>", "10:conv_backward_data_tc"),
       ("tc_conv_flat_kernel<0, 1, 0, 0, 0>", "10:conv_backward_data_tc"),
       ("maxpool_bwd_stream", "11:maxpool_backward"), ("tc_stage_x_taps", "12:conv_backward_kernel_tc"),
       ("tc_wgrad_ss", "12:conv_backward_kernel_tc")]


def assign(names):
    """records for the captured launches (None where the sequence does not match)"""
    n = len(SEQ)
    for start in range(len(names)):
        for rot in range(n):
            k_max = min(n, len(names) - start)
            if all(SEQ[(rot + k) % n][0] in names[start + k] for k in range(k_max)):
                out = [None] * len(names)
                for k in range(k_max):
                    out[start + k] = SEQ[(rot + k) % n][1]
                return out
    raise SystemExit("capture does not match the expected c3 step sequence")


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__issue_active.avg.pct_of_peak_sustained_active"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1e3, "us": 1, "usecond": 1,
         "msecond": 1e3, "nsecond": 1e-3}


def main():
    rep, out_json, out_md = sys.argv[1:4]
    note = sys.argv[4] if len(sys.argv) > 4 else rep
    if rep.endswith(".csv"):  # a saved `ncu -i <rep> --page raw --csv` export
        with open(rep) as fh:
            raw = fh.read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                              ",".join(METRICS)], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]

    def val(r, k):
        i = h.index(k)
        return float(r[i].replace(",", "")) * SCALE.get(units[i], 1)

    recs = {}
    body = rows[2:]
    mapping = assign([r[h.index("Kernel Name")] for r in body])
    lines = ["| # | kernel | record | us | DRAM read GB | write GB | tensor % | DRAM % | L2 % | "
             "issue % |", "|---|---|---|---|---|---|---|---|---|---|"]
    for i, r in enumerate(body):
        name = r[h.index("Kernel Name")]
        rec = mapping[i]
        if rec is None:
            continue
        rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
        t = val(r, "gpu__time_duration.sum")
        e = recs.setdefault(rec, {"launches": [], "dram_bytes": 0.0, "gpu_time_us": 0.0})
        e["launches"].append({"kernel": name[:120], "dram_bytes": rd + wr, "gpu_time_us": t,
                              "tensor_pct": val(r, METRICS[3]), "dram_pct": val(r, METRICS[4]),
                              "issue_pct": val(r, METRICS[6])})
        e["dram_bytes"] += rd + wr
        e["gpu_time_us"] += t
        pct = [r[h.index(k)][:5] for k in METRICS[3:]]
        lines.append(f"| {i} | `{name.split('(')[0][:48]}` | {rec} | {t:.0f} | {rd / 1e9:.3f} | "
                     f"{wr / 1e9:.3f} | " + " | ".join(pct) + " |")
    with open(out_json, "w") as fh:
        json.dump({"source": note, "note": "dram_bytes = all launches of the bench record "
                   "(staging / relayout + kernel), one eager step, ncu --set full",
                   "kernels": recs}, fh, indent=1)
    with open(out_md, "w") as fh:
        fh.write(f"# One c3 training step under ncu --set full ({note})\n\n")
        fh.write("Cold-cache, serialised launches; percentages are ncu's (tensor = "
                 "sm__pipe_tensor_cycles_active, DRAM = gpu__dram_throughput, L2 = "
                 "lts__throughput, issue = smsp__issue_active).\n\n")
        fh.write("\n".join(lines) + "\n\n## Per bench record\n\n| record | launches | us | DRAM GB |\n"
                 "|---|---|---|---|\n")
        for k in sorted(recs):
            e = recs[k]
            fh.write(f"| {k} | {len(e['launches'])} | {e['gpu_time_us']:.0f} | "
                     f"{e['dram_bytes'] / 1e9:.3f} |\n")


if __name__ == "__main__":
    main()

"""Condense an ncu --set full report: per kernel duration, DRAM bytes, throughputs, occupancy, issue
efficiency and the top warp-stall reasons.  Usage: ncu_summary.py report.ncu-rep [out.csv]"""
import csv
import io
import re
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio"]


def main(rep, out=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    # tensor-pipe utilisation (tcgen05 kernels): every percent-of-peak metric of the tensor pipes
    tkeys = [k for k in hdr if re.search(r"pipe_(tensor|tc|uma|imma)", k) and k.endswith("pct_of_peak_sustained_active")]
    lines = []
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        name = d["Kernel Name"].split("(")[0].replace("void ", "")[:60]
        stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): float(v)
                  for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_")
                  and k.endswith("_per_issue_active.ratio") and v}
        top = sorted(stalls.items(), key=lambda x: -x[1])[:4]
        vals = {k: f"{d.get(k, '')} {u.get(k, '')}".strip() for k in KEYS}
        lines.append([name] + [vals[k] for k in KEYS] + ["; ".join(f"{k}={v:.2f}" for k, v in top)] +
                     [d.get(k, "") for k in tkeys])
    head = ["kernel"] + KEYS + ["top_stalls(cycles/issue)"] + tkeys
    buf = io.StringIO()
    w = csv.writer(buf)
    w.writerow(head)
    w.writerows(lines)
    if out:
        open(out, "w").write(buf.getvalue())
    print(buf.getvalue())


if __name__ == "__main__":
    main(*sys.argv[1:])

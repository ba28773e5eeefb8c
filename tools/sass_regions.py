"""Summarise an `ncu --page source --csv --print-source sass` dump: contiguous SASS regions grouped by how often a
warp executes them, with their share of executed instructions and of stall samples, plus headline raw metrics.

    python tools/sass_regions.py gpurun_out/src_x.csv [gpurun_out/raw_x.csv]
"""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    for k, r in enumerate(rows):
        if "Source" in r and any("Instructions Executed" in c for c in r):
            hdr, start = r, k + 1
            break
    ie, src, ws = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    L = [(r[src], int(r[ie]), int(r[ws])) for r in rows[start:] if len(r) > ie and r[ie].isdigit()]
    tot, st = sum(x[1] for x in L), sum(x[2] for x in L)
    warps = L[0][1]
    seg, cur = [], None
    for j, (s, n, w) in enumerate(L):
        lvl = round(n / warps, 1)
        if cur is None or abs(lvl - cur[2]) > 0.25 * max(cur[2], 0.2):
            cur = [j, j, lvl, 0, 0, collections.Counter()]
            seg.append(cur)
        cur[1] = j
        cur[3] += n
        cur[4] += w
        cur[5][s.split()[0] if not s.startswith("@") else s.split()[1]] += 1
    print(f"{len(L)} SASS lines, {tot} warp instructions, {warps} warps")
    for a, b, lvl, n, w, c in seg:
        if n / tot > 0.01:
            print(f"{a}-{b} exec/warp {lvl} inst% {100 * n / tot:.1f} stall% {100 * w / st:.1f}", c.most_common(8))
    if len(sys.argv) > 2:
        rows = list(csv.reader(open(sys.argv[2])))
        hdr, r = rows[0], rows[2]
        want = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
                "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
                "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum")
        for i, h in enumerate(hdr):
            if h in want:
                print(h, r[i])
            if "issue_stalled" in h and h.endswith("per_issue_active.ratio"):
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                if v > 0.3:
                    print("  stall", h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), round(v, 2))


if __name__ == "__main__":
    main()

"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel launches, mean
time and share of the layer's kernel time (wl:: kernels only count toward the share)."""
import collections
import csv
import re
import sys


def main(path, out):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, vi, gi, bi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size"), hdr.index("Block Size")
    agg = collections.OrderedDict()
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        name = re.sub(r"\(.*$", "", r[ki]).replace("void ", "")[:90]
        key = (name, r[gi], r[bi])
        agg.setdefault(key, []).append(float(r[vi].replace(",", "")) / 1e3)
    ours = {k: v for k, v in agg.items() if k[0].startswith("wl::") or "gemm_i8" in k[0]}
    # per forward: each wl kernel's launches / number of forwards (the input cast runs once per forward)
    nfwd = max(len(v) for k, v in ours.items() if "quant_input" in k[0] or "cast_input" in k[0])
    step = sum(sum(v) for v in ours.values()) / nfwd
    with open(out, "w") as f:
        f.write("kernel,grid,block,launches,mean_us,per_forward_us,share_of_forward\n")
        for (name, grid, block), v in agg.items():
            mine = (name, grid, block) in ours
            pf = sum(v) / nfwd if mine else ""
            share = f"{sum(v) / nfwd / step:.4f}" if mine else ""
            f.write(f"\"{name}\",\"{grid}\",\"{block}\",{len(v)},{sum(v) / len(v):.1f},"
                    f"{pf if pf == '' else f'{pf:.1f}'},{share}\n")
        f.write(f"# forwards={nfwd}, serialized wl kernel time per forward = {step:.1f} us (cold-cache, ncu-serialised)\n")
    print(open(out).read())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])

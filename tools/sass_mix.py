"""Opcode mix (executed warp instructions) and top stall lines per kernel from an ncu source CSV
(--page source --csv --print-source sass).  Usage: sass_mix.py source.csv [kernel-substring]"""
import csv
import sys
from collections import Counter

def main(path, want=None):
    kern, mix, stalls, total = None, Counter(), [], 0
    out = []
    def flush():
        if kern and (not want or want in kern) and total:
            out.append((kern, total, mix.copy(), sorted(stalls, key=lambda x: -x[0])[:12]))
    with open(path) as fh:
        rd = csv.reader(fh)
        hdr = None
        for row in rd:
            if row and row[0] == "Kernel Name":
                flush()
                kern, mix, stalls, total, hdr = row[1], Counter(), [], 0, None
                continue
            if row and row[0] == "Address":
                hdr = row
                ie = hdr.index("Instructions Executed"); ss = hdr.index("Warp Stall Sampling (All Samples)")
                continue
            if hdr is None or len(row) < len(hdr):
                continue
            n = int(row[ie] or 0)
            op = row[1].strip().split()[0] if row[1].strip() else "?"
            if op.startswith("@"):
                op = row[1].strip().split()[1]
            op = op.split(".")[0]
            mix[op] += n
            total += n
            stalls.append((int(row[ss] or 0), row[1].strip()[:70], n))
    flush()
    for k, tot, m, st in out:
        print(f"== {k[:110]}\n   total warp-instr {tot}")
        print("   " + ", ".join(f"{o}:{100*c/tot:.1f}%" for o, c in m.most_common(25)))
        for s in st:
            print(f"   stall {s[0]:6d}  exec {s[2]:10d}  {s[1]}")

if __name__ == "__main__":
    main(*sys.argv[1:])

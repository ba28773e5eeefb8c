"""Side-by-side per-kernel times (last iteration) of two ncu launch lists of tools/prof_backward.py."""
import csv
import re
import sys


def last_iter(path, marker="FillFunctor"):
    rows = [r for r in csv.reader(open(path)) if len(r) > 8 and r[0].isdigit()]
    names = [r[4] for r in rows]
    vals = [float(r[-1]) for r in rows]
    s = [i for i, n in enumerate(names) if marker in n][-1]
    return [(re.sub(r"\(.*", "", n).replace("void ", "").replace("wl::", "")[:40], v / 1000) for n, v in zip(names[s:], vals[s:])]


a, b = last_iter(sys.argv[1]), last_iter(sys.argv[2])
for x, y in zip(a, b):
    print(f"  {x[0]:42s} {x[1]:8.1f}   {y[0]:30s} {y[1]:8.1f}")
print("  total", round(sum(v for _, v in a), 1), round(sum(v for _, v in b), 1))

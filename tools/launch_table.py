"""Per-kernel table (ms) from an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
kn, mv, mu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}
tot = 0.0
for r in rows[h + 1:]:
    ms = float(r[mv].replace(",", "")) * scale.get(r[mu], 1.0)
    tot += ms
    print(f"{ms:8.4f}  {r[kn][:90]}")
print(f"{tot:8.4f}  total")

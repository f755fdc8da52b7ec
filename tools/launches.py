"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, data = rows[0], rows[1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
tot, cnt, seq = collections.OrderedDict(), collections.Counter(), []
for r in data:
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3)
    name = r[ki].split("(")[0].replace("void ", "")
    seq.append((name, v))
    tot[name] = tot.get(name, 0) + v
    cnt[name] += 1
T = sum(tot.values())
print(f"total {T:.1f} us over {len(seq)} launches")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"  {k:45s} {cnt[k]:4d} {v:9.1f} us {100 * v / T:5.1f}%")
if "-v" in sys.argv:
    for n, v in seq:
        print(f"    {n:45s} {v:8.1f}")

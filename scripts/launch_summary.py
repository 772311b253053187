"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[hi + 1:]:
    try:
        v = float(r[mi].replace(",", "")) * scale.get(r[ui], 1e-6)
    except (ValueError, IndexError):
        continue
    name = r[ki].split("(")[0].replace("void ", "").replace("fsgg::<unnamed>::", "")[:70]
    tot[name] += v
    cnt[name] += 1
allt = sum(tot.values())
print(f"total {allt:.2f} ms over {sum(cnt.values())} launches")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{v:10.3f} ms {100 * v / allt:5.1f}% {cnt[k]:5d}  {k}")

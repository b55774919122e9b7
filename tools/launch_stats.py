"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui, idi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("ID")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= vi or int(r[idi]) < skip:
        continue
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    name = r[ki].split("(")[0]
    name = name.replace("void ", "")[:70]
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
print("total %.1f us over %d launches" % (T, sum(cnt.values())))
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 40]:
    print("%10.1f us %5.1f%% %6d  %s" % (v, 100 * v / T, cnt[k], k))

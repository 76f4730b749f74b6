"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_*) per kernel."""
import csv, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]; idx = {k: i for i, k in enumerate(h)}
per = defaultdict(lambda: defaultdict(dict))
for r in rows[hi + 1:]:
    per[r[idx["ID"]]][r[idx["Metric Name"]]] = (float(r[idx["Metric Value"]].replace(",", "")), r[idx["Metric Unit"]])
    per[r[idx["ID"]]]["name"] = r[idx["Kernel Name"]]
agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for lid, m in per.items():
    name = m["name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").replace("acg::", "")
    t, u = m["gpu__time_duration.sum"]
    t = t / 1e3 if u in ("ns", "nsecond") else (t * 1e3 if u in ("ms", "msecond") else t)  # -> usecond
    a = agg[name]
    a[0] += 1; a[1] += t
    a[2] += m.get("dram__bytes_read.sum", (0.0, ""))[0]; a[3] += m.get("dram__bytes_write.sum", (0.0, ""))[0]
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':60s} {'launches':>8s} {'mean_us':>10s} {'share':>7s} {'rd/launch':>10s} {'wr/launch':>10s}")
for name, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    unit = 1.0
    print(f"{name[:60]:60s} {a[0]:8d} {a[1]/a[0]:10.1f} {a[1]/tot*100:6.1f}% {a[2]/a[0]:10.3g} {a[3]/a[0]:10.3g}")

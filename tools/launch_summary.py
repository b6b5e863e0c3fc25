"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv), per pass."""
import collections
import csv
import sys

rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"'))
        if r["Metric Name"] == "gpu__time_duration.sum"]
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    n = r["Kernel Name"].split("(")[0].replace("void ", "").split("::")[-1][:48]
    agg[n][0] += 1
    agg[n][1] += float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]
npass = agg["k_conn_mis"][0] or 1
tot = sum(v[1] for v in agg.values())
print(f"{npass} passes, {len(rows)} launches, {tot / npass:.3f} ms/pass serialised")
for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{v / npass:8.3f} ms/pass {100 * v / tot:5.1f}% {c:6d} {n}")

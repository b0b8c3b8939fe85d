"""Aggregate an ncu --metrics gpu__time_duration.sum --csv log by kernel name."""
import csv, collections, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = next(r for r in rows if r[0] == "ID")
data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    k = d["Kernel Name"].split("(")[0].replace("eh::", "").replace("<unnamed>::", "")
    agg[k][0] += 1
    agg[k][1] += float(d["Metric Value"]) * scale[d["Metric Unit"]]
tot = sum(v[1] for v in agg.values())
print(f"total {tot:.3f} ms over {sum(v[0] for v in agg.values())} launches")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[1]:9.3f} ms {100 * v[1] / tot:5.1f}%  n={v[0]:4d}  {k[:90]}")

"""Summarise an ncu --csv launch list (gpu__time_duration.sum per kernel)."""
import collections, csv, sys
path = sys.argv[1]
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.DictReader(lines))
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("spamm::<unnamed>::", "")
    v = float(r["Metric Value"].replace(",", ""))
    v = {"ns": v / 1e3, "nsecond": v / 1e3, "us": v, "usecond": v, "ms": v * 1e3, "msecond": v * 1e3}[r["Metric Unit"]]
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{len(rows)} launches, {tot:.1f} us total")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:10.1f} us {100 * t / tot:5.1f}%  n={n:4d}  {k[:90]}")

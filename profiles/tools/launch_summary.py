"""Aggregate an ncu gpu__time_duration launch list into per-kernel shares."""
import csv, sys, collections
rows = [l for l in open(sys.argv[1]) if l.startswith('"')]
r = csv.DictReader(rows)
agg = collections.defaultdict(lambda: [0, 0.0])
for row in r:
    if row["Metric Name"] != "gpu__time_duration.sum":
        continue
    k = row["Kernel Name"].split("(")[0]
    v = float(row["Metric Value"]) * (1e-3 if row["Metric Unit"] == "ns" else 1.0 if row["Metric Unit"] == "us" else 1e3)
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(v[1] for v in agg.values())
print(f"| kernel | launches | total us | share |\n|---|---|---|---|")
for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| `{k}` | {n} | {us:.0f} | {100*us/tot:.1f}% |")
print(f"| **total** | {sum(v[0] for v in agg.values())} | {tot:.0f} | 100% |")

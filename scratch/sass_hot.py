"""Print SASS instructions with the most stall samples from an ncu source page (sass) CSV."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)"); iSrc = h.index("Source")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(float(r[iS] or 0) for r in data)
print("total samples", tot, "instructions", len(data))
top = sorted(range(len(data)), key=lambda i: -float(data[i][iS] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]
for i in sorted(top):
    r = data[i]
    st = sorted(((float(r[h.index(c)] or 0), c[6:]) for c in cols), reverse=True)[:2]
    print(f"{i:5d} {float(r[iS]):7.0f} {100*float(r[iS])/tot:5.1f}% {r[iSrc][:60]:60s} {st}")

"""Summarise an ncu `--page source --csv --print-source sass` dump: stall samples by reason
and by code region (bucket of consecutive SASS lines)."""
import csv, gzip, sys, collections
path = sys.argv[1]; bucket = int(sys.argv[2]) if len(sys.argv) > 2 else 256
op = gzip.open if path.endswith(".gz") else open
rows = list(csv.reader(op(path, "rt")))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]; data = rows[hdr_i + 1:]
col = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter(); 
per = []
for k, r in enumerate(data):
    if len(r) < len(hdr): continue
    s = {h: int(r[col[h]] or 0) for h in stalls}
    for h, v in s.items(): tot[h] += v
    per.append((k, r[col["Source"]].strip(), int(r[col["# Samples"]] or 0), int(r[col["Instructions Executed"]] or 0), s))
allsmp = sum(p[2] for p in per)
print("instructions", len(per), "samples", allsmp)
print("by reason:", ", ".join(f"{h[6:]} {v} ({100*v/allsmp:.1f}%)" for h, v in tot.most_common(10)))
print(f"\nregions of {bucket} SASS lines: first-line | samples % | exec/line | top stalls")
for b0 in range(0, len(per), bucket):
    blk = per[b0:b0 + bucket]
    smp = sum(p[2] for p in blk)
    ex = sum(p[3] for p in blk) / max(len(blk), 1)
    c = collections.Counter()
    for p in blk:
        for h, v in p[4].items(): c[h] += v
    top = ", ".join(f"{h[6:]} {v}" for h, v in c.most_common(3))
    print(f"{b0:6d} {blk[0][1][:38]:38s} | {smp:6d} {100*smp/allsmp:5.1f}% | {ex:8.0f} | {top}")

"""Executed-instruction mix (warp level) from an ncu sass source page CSV."""
import csv, sys, collections, re
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]; d = rows[2:]
iE = h.index("Instructions Executed"); iSrc = h.index("Source")
mix = collections.Counter()
for r in d:
    op = re.sub(r"^@!?U?P\w+\s+", "", r[iSrc].strip()).split(" ")[0].split(".")[0]
    mix[op] += float(r[iE] or 0)
tot = sum(mix.values())
print("total", tot)
for k, v in mix.most_common(25):
    print(f"{k:10s} {v:12.0f} {100*v/tot:5.1f}%")

"""Backward branches (loops) and local-memory traffic of a cuobjdump -sass function listing."""
import re, sys
lines = [l for l in open(sys.argv[1]) if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l)]
addr = [int(re.match(r"\s+/\*([0-9a-f]+)\*/", l).group(1), 16) for l in lines]
idx = {a: i for i, a in enumerate(addr)}
for i, l in enumerate(lines):
    m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d,\s*)?0x([0-9a-f]+)", l)
    if m:
        t = int(m.group(1), 16)
        if t < addr[i] and t in idx:
            body = lines[idx[t]:i + 1]
            loc = sum(("LDL" in b) or ("STL" in b) for b in body)
            dfma = sum("DFMA" in b for b in body)
            print(f"loop lines {idx[t]+1}..{i+1} ({i+1-idx[t]} instr, {dfma} DFMA, {loc} LDL/STL)")
print("total", len(lines), "LDL/STL", sum(("LDL" in b) or ("STL" in b) for b in lines))

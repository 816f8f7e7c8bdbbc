"""Static SASS listings + instruction mix of the hot kernels of libfractime_b200.so.

    python profiles/tools/sass_listing.py <out dir>

Writes <name>.sass.gz (cuobjdump -sass of the kernel) and a mix table
(sass_mix.md): static counts of FP64 (DFMA/DADD/DMUL), memory (LDG/STG/LDS/STS,
128-bit forms), shuffles, barriers and special ops -- the proof of what the
compiled code actually does (no tcgen05 / TMA: this path is FP64 FFTs and scans).
"""
import collections, gzip, os, re, subprocess, sys

LIB = os.path.join(os.path.dirname(__file__), "..", "..", "paper_1710_11593_b200", "libfractime_b200.so")
KERNELS = {
    "mp_split_kernel_16": r"_ZN3ftb15mp_split_kernelILi16ELi12EEEvNS_6MpArgsENS_6SplitQE",
    "mp_split_kernel_8": r"_ZN3ftb15mp_split_kernelILi8ELi12EEEvNS_6MpArgsENS_6SplitQE",
    "leaf_pair_tridiag": r"_ZN3ftb9leaf_pairILi2ELi2ELi32EEEvNS_8LeafArgsE",
    "leaf_fused_tridiag": r"_ZN3ftb10leaf_fusedILi2ELi2ELi32ELb1ELb1EEEvNS_8LeafArgsE",
    "leaf_chain_upwind": r"_ZN3ftb10leaf_chainILi1ELi2ELi32ELb1ELb1EEEvNS_8LeafArgsE",
    "mp1g_kernel_9": r"_ZN3ftb11mp1g_kernelILi9EEEvNS_6MpArgsE",
    "mp1p_kernel_12_tma": r"_ZN3ftb11mp1p_kernelILi12EEEvNS_6MpArgsEi",
    "mp8_kernel_9_radix8": r"_ZN3ftb10mp8_kernelILi9EEEvNS_6MpArgsE",
    "mp_direct_kernel_64": r"_ZN3ftb16mp_direct_kernelILi64EEEvNS_6MpArgsE",
    "mp1g_kernel_12": r"_ZN3ftb11mp1g_kernelILi12EEEvNS_6MpArgsE",
    "mp_kernel_cluster4": r"_ZN3ftb9mp_kernelILi4ELi12ELb0ELb0EEEvNS_6MpArgsE",
    "direct_multi_kernel": r"_ZN3ftb19direct_multi_kernelENS_10DirectArgsEPjii",
}


def main():
    out = sys.argv[1]
    os.makedirs(out, exist_ok=True)
    rows = []
    for name, sym in KERNELS.items():
        r = subprocess.run(["cuobjdump", "-sass", "-fun", sym, LIB], capture_output=True, text=True)
        text = r.stdout
        if "Function" not in text:
            print("missing", name, r.stderr[:200])
            continue
        with gzip.open(os.path.join(out, name + ".sass.gz"), "wt") as f:
            f.write(text)
        mix = collections.Counter()
        for line in text.splitlines():
            m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
            if m:
                op = m.group(1)
                mix[op.split(".")[0]] += 1
                if op.startswith(("LDG", "STG", "LDS", "STS")) and ".128" in op:
                    mix[op.split(".")[0] + ".128"] += 1
        total = sum(v for k, v in mix.items() if not k.endswith(".128"))
        rows.append((name, total, mix))
    keys = ["DFMA", "DADD", "DMUL", "LDG", "LDG.128", "STG", "STG.128", "LDS", "LDS.128", "STS", "STS.128", "SHFL",
            "BAR", "ATOMG", "RED", "MUFU", "UTMALDG", "UBLKCP", "LDGSTS", "HMMA", "DMMA"]
    with open(os.path.join(out, "sass_mix.md"), "w") as f:
        f.write("| kernel | SASS instr. (static) | " + " | ".join(keys) + " |\n")
        f.write("|---|---|" + "---|" * len(keys) + "\n")
        for name, total, mix in rows:
            f.write(f"| `{name}` | {total} | " + " | ".join(str(mix.get(k, 0)) for k in keys) + " |\n")
    print(open(os.path.join(out, "sass_mix.md")).read())


if __name__ == "__main__":
    main()

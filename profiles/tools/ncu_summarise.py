"""Summarise ncu --set full raw-page CSVs (one launch each) into kernels.json.

    python profiles/tools/ncu_summarise.py <dir with cap_*_raw.csv> <out dir>
"""
import csv, glob, gzip, json, os, shutil, sys

KEYS = {"duration": "gpu__time_duration.sum", "dram_read": "dram__bytes_read.sum", "dram_write": "dram__bytes_write.sum",
        "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
        "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
        "dram_throughput_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l2_hit_pct": "lts__t_sector_hit_rate.pct",
        "registers": "launch__registers_per_thread", "grid": "launch__grid_size", "block": "launch__block_size",
        "warp_instructions": "smsp__inst_executed.sum", "fp64_warp_instructions": "smsp__inst_executed_pipe_fp64.sum"}


def main():
    src, dst = sys.argv[1], sys.argv[2]
    os.makedirs(os.path.join(dst, "raw"), exist_ok=True)
    out = {}
    for f in sorted(glob.glob(os.path.join(src, "cap_*_raw.csv"))):
        rows = [r for r in csv.reader(open(f))]
        if len(rows) < 3:
            continue
        h, u, v = rows[0], rows[1], rows[2]
        d = {"kernel": v[h.index("Kernel Name")]}
        for name, k in KEYS.items():
            if k in h:
                d[name] = f"{v[h.index(k)].replace(',', '')} {u[h.index(k)]}".strip()
        st = {}
        for i, k in enumerate(h):
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    val = float(v[i])
                except ValueError:
                    continue
                if val >= 0.05:
                    st[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(val, 3)
        d["stalls_per_issue"] = dict(sorted(st.items(), key=lambda t: -t[1]))
        tag = os.path.basename(f)[4:-8]
        out[tag] = d
        with open(f, "rb") as a, gzip.open(os.path.join(dst, "raw", os.path.basename(f) + ".gz"), "wb") as b:
            shutil.copyfileobj(a, b)
    json.dump(out, open(os.path.join(dst, "kernels.json"), "w"), indent=1)
    for k, d in out.items():
        print(k, d["kernel"][:60], d.get("duration"), d.get("dram_read"), d.get("dram_write"), d.get("fp64_pipe_pct"))


if __name__ == "__main__":
    main()

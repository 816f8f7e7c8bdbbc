"""Summarise the round's ncu --set full captures (raw-page CSVs) into profiles/ncu_r01/kernels.json."""
import csv, glob, gzip, json, os, shutil, sys
out = {}
KEYS = {"duration": "gpu__time_duration.sum", "dram_read": "dram__bytes_read.sum", "dram_write": "dram__bytes_write.sum",
        "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
        "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
        "dram_throughput_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "registers": "launch__registers_per_thread", "grid": "launch__grid_size", "block": "launch__block_size",
        "warp_instructions": "smsp__inst_executed.sum"}
for f in sorted(glob.glob(sys.argv[1] + "/ev_*_raw.csv")):
    rows = list(csv.reader(open(f)))
    if len(rows) < 3:
        continue
    h, u, v = rows[0], rows[1], rows[2]
    d = {"kernel": v[h.index("Kernel Name")]}
    for name, k in KEYS.items():
        if k in h:
            x = v[h.index(k)].replace(",", "")
            d[name] = f"{x} {u[h.index(k)]}".strip()
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
    for i, k in enumerate(h):
        if k in ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
                 "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"):
            d[k] = v[i]
    tag = os.path.basename(f)[3:-8]
    out[tag] = d
    with open(f, "rb") as src, gzip.open(os.path.join(sys.argv[2], "raw", os.path.basename(f) + ".gz"), "wb") as dst:
        shutil.copyfileobj(src, dst)
json.dump(out, open(os.path.join(sys.argv[2], "kernels.json"), "w"), indent=1)
print(json.dumps({k: (v["kernel"][:40], v.get("duration"), v["stalls_per_issue"]) for k, v in out.items()}, indent=0)[:4000])

"""Summarise ncu --set full reports: duration, DRAM bytes, occupancy, pipe utilisation."""
import csv, subprocess, sys, json
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
        "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]
pipes = ["fp64", "xu", "alu", "fma", "lsu", "adu", "cbu", "uniform", "fp16", "tensor"]
out = {}
for rep in sys.argv[1:]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, units, vals = rows[0], rows[1], rows[2]
    d = {"kernel": vals[h.index("Kernel Name")][:60]}
    for k in keys:
        if k in h:
            d[k] = f"{vals[h.index(k)]} {units[h.index(k)]}".strip()
    for p in pipes:
        k = f"sm__inst_executed_pipe_{p}.avg.pct_of_peak_sustained_active"
        if k in h:
            d[f"pipe_{p}_%"] = vals[h.index(k)]
    out[rep] = d
    print(rep, json.dumps(d, indent=0))
json.dump(out, open("profiles/ncu_r01/kernels.json", "w"), indent=1)

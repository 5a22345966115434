"""Summarize an ncu report: per kernel duration, DRAM bytes, throughput, issue, occupancy, top stalls."""
import csv, io, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
for d in data:
    name = d[col["Kernel Name"]][:60]
    print("==", name)
    for w in want:
        if w in col:
            print(f"   {w:70s} {d[col[w]]} {units[col[w]]}")
    st = [(h, float(d[i] or 0)) for h, i in col.items() if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
    st = sorted(st, key=lambda x: -x[1])[:6]
    print("   stalls (cycles/issued):", ", ".join(f"{h.replace("smsp__average_warps_issue_stalled_","").replace("_per_issue_active.ratio","")}={v:.2f}" for h, v in st))

"""Summarise an ncu report: per kernel duration, DRAM bytes, throughputs, stalls."""
import csv, subprocess, sys, io, collections

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, units = r[0], r[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "launch__grid_size", "launch__block_size"]
for row in r[2:]:
    name = row[h.index("Kernel Name")][:60]
    print(name)
    for m in want:
        if m in h:
            print(f"   {m:65s} {row[h.index(m)]:>14s} {units[h.index(m)]}")
    st = [(h[i].replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
           float(row[i].replace(",", ""))) for i in range(len(h))
          if h[i].startswith("smsp__average_warps_issue_stalled_") and h[i].endswith("per_issue_active.ratio")
          and row[i] not in ("", "n/a")]
    st.sort(key=lambda x: -x[1])
    print("   stalls:", ", ".join(f"{k}={v:.2f}" for k, v in st[:6]))

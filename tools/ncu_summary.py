"""Summarise an ncu --set full report: per kernel time, DRAM bytes, key throughputs, stalls."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct", "launch__grid_size", "launch__block_size"]
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    print(name[:70])
    print("   " + "  ".join(f"{w.split('__')[1][:24]}={r[hdr.index(w)]}" for w in want if w in hdr))
    st = [(hdr[i], float(r[i] or 0)) for i in range(len(hdr))
          if "smsp__pcsamp_warps_issue_stalled" in hdr[i] and not hdr[i].endswith("not_issued")]
    tot = sum(v for _, v in st) or 1.0
    st.sort(key=lambda x: -x[1])
    print("   stalls: " + ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100*v/tot:.0f}%"
                                    for k, v in st[:6]))

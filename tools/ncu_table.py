"""Summarise an .ncu-rep: one line per launch with the metrics that matter
for the gather-bound kernels (time, DRAM bytes, occupancy, L2/L1 hit rate,
issue activity) — python tools/ncu_table.py <report.ncu-rep>."""
import csv
import io
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
     "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
     "smsp__issue_active.avg.pct_of_peak_sustained_active",
     "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--metrics", ",".join(M)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
cols = [h.index("Kernel Name")] + [h.index(m) for m in M if m in h]
print("\t".join(["kernel", "ms", "dramR_GB", "dramW_GB", "regs", "warps%", "L2hit%", "L1hit%",
                 "issue%", "occ_smem", "occ_regs"][:len(cols)]))
for r in rows[2:]:
    name = r[cols[0]].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
    print("\t".join([name[:48]] + [r[c][:8] for c in cols[1:]]))

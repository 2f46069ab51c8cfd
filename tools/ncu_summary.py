"""Summarise an ncu report: one block of key metrics per profiled kernel."""
import csv
import subprocess
import sys

KEYS = [
    ("time_us", "gpu__time_duration.sum"),
    ("dram_read_MB", "dram__bytes_read.sum"),
    ("dram_write_MB", "dram__bytes_write.sum"),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("l2_read_sectors", "lts__t_sectors_srcunit_tex_op_read.sum"),
    ("l2_hit_pct", "lts__t_sector_hit_rate.pct"),
    ("l1_hit_pct", "l1tex__t_sector_hit_rate.pct"),
    ("l1_ld_requests", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"),
    ("l1_ld_sectors", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"),
    ("l1_ld_wavefronts", "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum"),
    ("l1_pct", "l1tex__throughput.avg.pct_of_peak_sustained_active"),
    ("l2_pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("sm_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("issue_active_pct", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
    ("inst", "smsp__inst_executed.sum"),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("stall_long_sb", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"),
    ("stall_short_sb", "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio"),
    ("stall_lg_throttle", "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio"),
    ("stall_wait", "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio"),
    ("stall_math", "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio"),
    ("stall_barrier", "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio"),
    ("stall_membar", "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio"),
    ("stall_tex", "smsp__average_warps_issue_stalled_tex_throttle_per_issue_active.ratio"),
    ("cycles_per_issue", "smsp__average_warp_latency_per_inst_issued.ratio"),
    ("regs", "launch__registers_per_thread"),
    ("tensor_pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        print("no data")
        return
    h = rows[0]
    for r in rows[2:]:
        d = dict(zip(h, r))
        print("==", d.get("Kernel Name", "?")[:110])
        for label, key in KEYS:
            if key in d and d[key] not in ("", "n/a"):
                print(f"   {label:18s} {d[key]}")


if __name__ == "__main__":
    main(sys.argv[1])

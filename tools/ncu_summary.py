"""Summarise an ncu report (.ncu-rep) into the numbers we track (run here, no GPU)."""
import csv
import re
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_%"),
    ("l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct", "l1_ld_hit_%"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "l1_wavefronts_%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem_wavefronts_%"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts"),
    ("lts__t_sectors.sum.pct_of_peak_sustained_elapsed", "l2_sectors_%"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"== {name[:90]}")
        for k, label in KEYS:
            if k in h:
                i = h.index(k)
                print(f"  {label:22s} {v[i]} {u[i]}")
        stalls = [(h[i], float(v[i])) for i in range(len(h))
                  if re.match(r"smsp__average_warps_issue_stalled_.*_per_issue_active.ratio", h[i]) and v[i]]
        stalls.sort(key=lambda x: -x[1])
        print("  stalls/issue:", ", ".join(f"{n.split('stalled_')[1].split('_per')[0]}={x:.2f}" for n, x in stalls[:6]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)

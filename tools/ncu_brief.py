"""Print the key metrics of an .ncu-rep (first kernel): time, pipes, occupancy, traffic and the
stall reasons above a threshold.   python tools/ncu_brief.py gpurun_out/prof_x.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ("Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem")


def main():
    out = subprocess.check_output(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"]).decode()
    rows = list(csv.reader(io.StringIO(out)))
    h, units, v = rows[0], rows[1], rows[2]
    for k, u, x in zip(h, units, v):
        stall = "issue_stalled" in k and k.endswith("per_issue_active.ratio")
        if k in KEYS or (stall and float(x or 0) > 0.3):
            print(f"{k:80s} {x} {u}")


if __name__ == "__main__":
    main()

"""Summarise an `ncu --page raw --csv` export: one block of key metrics per launch.

usage: ncu -i X.ncu-rep --page raw --csv > raw.csv; python profiles/ncu_summary.py raw.csv
"""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__grid_size", "launch__block_size",
        "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed"]


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    name = hdr.index("Kernel Name")
    for r in rows[2:]:
        print(r[name])
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:70s} {r[i]:>16s} {units[i]}")
        if "dram__bytes_read.sum" in hdr:
            rd = float(r[hdr.index("dram__bytes_read.sum")])
            wr = float(r[hdr.index("dram__bytes_write.sum")])
            mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            ur = mul.get(units[hdr.index("dram__bytes_read.sum")], 1)
            uw = mul.get(units[hdr.index("dram__bytes_write.sum")], 1)
            print(f"  {'traffic (read+write) bytes':70s} {rd * ur + wr * uw:16.4e}")


if __name__ == "__main__":
    main(sys.argv[1])

"""Print selected raw metrics of an .ncu-rep (dev tool): python tools/ncu_raw.py REP [metric ...]"""
import csv
import subprocess
import sys

DEFAULT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
           "l1tex__t_sector_hit_rate.pct", "l1tex__throughput.avg.pct_of_peak_sustained_active",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "smsp__thread_inst_executed_per_inst_executed.ratio",
           "sm__inst_executed.avg.per_cycle_active", "launch__grid_size", "lts__t_sectors_op_red.sum",
           "lts__t_sectors_op_atom.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
           "l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum"]


def main():
    rep = sys.argv[1]
    want = sys.argv[2:] or DEFAULT
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    for v in rows[2:]:
        print("--", v[h.index("Kernel Name")][:60] if "Kernel Name" in h else "")
        for w in want:
            for i, n in enumerate(h):
                if n == w or (w.endswith("*") and n.startswith(w[:-1])):
                    print(f"  {n} = {v[i]} {units[i]}")


if __name__ == "__main__":
    main()

"""Summarise ncu outputs (launch list CSV + --set full reports) into profiles/ (dev tool)."""
import collections
import csv
import io
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
           "l1tex__t_sector_hit_rate.pct", "l1tex__throughput.avg.pct_of_peak_sustained_active",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "sm__maximum_warps_per_active_cycle_pct", "launch__registers_per_thread",
           "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__inst_executed.avg.per_cycle_active",
           "launch__grid_size", "launch__block_size",
           # L2 operation counts (the texture walks' roofline: corner fetches and adjoint REDs)
           "lts__t_requests_srcunit_tex_op_red.sum", "lts__t_sectors_srcunit_tex_op_red.sum",
           "lts__t_requests_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
           "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
           "l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct",
           "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hd = rows[h]
    ki, vi, ui = hd.index("Kernel Name"), hd.index("Metric Value"), hd.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[h + 1:]:
        k = r[ki].split("(")[0].split("::")[-1]
        v = float(r[vi].replace(",", ""))
        v = v / 1e6 if r[ui] == "ns" else (v / 1e3 if r[ui] in ("us", "usecond") else v)
        tot[k] += v
        cnt[k] += 1
    s = sum(tot.values())
    out = ["| kernel | launches | ms (sum, serialised, cold) | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"| {k} | {cnt[k]} | {v:.3f} | {100 * v / s:.1f}% |")
    out.append(f"| total | {sum(cnt.values())} | {s:.3f} | 100% |")
    return "\n".join(out)


def report(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u = rows[0], rows[1]
    out = []
    for row in rows[2:]:
        name = row[h.index("Kernel Name")].split("(")[0].split("::")[-1]
        out.append(f"### {name}\n\n| metric | value | unit |\n|---|---|---|")
        for m in METRICS:
            if m in h:
                i = h.index(m)
                out.append(f"| {m} | {row[i]} | {u[i]} |")
    return "\n".join(out)


if __name__ == "__main__":
    tag, launch_csv, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    md = [f"# ncu summary {tag}", ""]
    if launch_csv != "-":
        md += ["Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`):", "", launches(launch_csv), ""]
    for r in reps:
        md += [f"## {r}", "", report(r), ""]
    print("\n".join(md))

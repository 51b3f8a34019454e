"""DRAM traffic per launch from an ncu --set full capture -> JSON read by bench.py (dev tool).
python tools/ncu_traffic.py REP CONFIG KERNEL OUT.json"""
import csv
import io
import json
import subprocess
import sys

rep, config, kernel, out = sys.argv[1:5]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h, u = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tscale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
launches = []
for r in rows[2:]:
    if kernel not in r[h.index("Kernel Name")]:
        continue
    rd = float(r[h.index("dram__bytes_read.sum")]) * scale[u[h.index("dram__bytes_read.sum")]]
    wr = float(r[h.index("dram__bytes_write.sum")]) * scale[u[h.index("dram__bytes_write.sum")]]
    ms = float(r[h.index("gpu__time_duration.sum")]) * tscale[u[h.index("gpu__time_duration.sum")]]
    def g(name):
        return float(r[h.index(name)]) if name in h and r[h.index(name)] not in ("", "n/a") else None
    launches.append({"dram_read": rd, "dram_write": wr, "ms_cold_serialised": ms,
                     "l2_hit_pct": g("lts__t_sector_hit_rate.pct"), "l1_hit_pct": g("l1tex__t_sector_hit_rate.pct"),
                     "lanes_per_inst": g("smsp__thread_inst_executed_per_inst_executed.ratio"),
                     "ipc": g("sm__inst_executed.avg.per_cycle_active"),
                     "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active")})
avg = sum(x["dram_read"] + x["dram_write"] for x in launches) / max(len(launches), 1)


def mean(k):
    v = [x[k] for x in launches if x[k] is not None]
    return round(sum(v) / len(v), 3) if v else None


json.dump({"config": config, "kernel": kernel, "source": rep.split("/")[-1],
           "capture": "ncu --set full --clock-control none, the timed step's launches of the kernel",
           "dram_bytes_per_launch": avg, **{k: mean(k) for k in ("l2_hit_pct", "l1_hit_pct", "lanes_per_inst", "ipc",
                                                                  "issue_active_pct")},
           "launches": launches}, open(out, "w"), indent=1)
print(f"{len(launches)} launches, {avg / 1e9:.3f} GB per launch")

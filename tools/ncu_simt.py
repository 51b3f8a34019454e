"""SIMT efficiency per CUDA source line of an .ncu-rep (dev tool; needs -lineinfo builds):
warp instructions issued, thread instructions, and the issue slots lost to idle lanes.
python tools/ncu_simt.py REP [N] [--sass]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = collections.defaultdict(lambda: [0.0, 0.0])
src = {}
fname, line, hdr = "?", None, None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ii, ti = hdr.index("Instructions Executed"), hdr.index("Thread Instructions Executed")
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0]:
        line = (fname, int(r[0]))
        src[line] = r[1].strip()[:70]
        continue
    try:
        agg[line][0] += float(r[ii] or 0)
        agg[line][1] += float(r[ti] or 0)
    except ValueError:
        pass
W = sum(v[0] for v in agg.values())
Tt = sum(v[1] for v in agg.values())
print(f"warp inst {W:.3e}  thread inst {Tt:.3e}  lanes/inst {Tt / W:.2f}")
print(f"{'line':>24s} {'inst%':>6s} {'lanes':>6s} {'lost%':>6s}  source")
for k, v in sorted(agg.items(), key=lambda kv: -(32 * kv[1][0] - kv[1][1]))[:n]:
    if v[0] == 0:
        continue
    print(f"{k[0][:16]:>16s}:{k[1]:<7d} {v[0] / W * 100:6.2f} {v[1] / v[0]:6.1f} {(32 * v[0] - v[1]) / (32 * W) * 100:6.2f}  {src.get(k, '')}")

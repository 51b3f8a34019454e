"""Warp-stall samples aggregated per CUDA source line (dev tool; needs -lineinfo builds).
python tools/ncu_lines.py REP [N]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = collections.Counter()
why = collections.defaultdict(collections.Counter)
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
        si = hdr.index("Warp Stall Sampling (All Samples)")
        stall_cols = [i for i, c in enumerate(hdr) if c.startswith("stall_") and "Not Issued" not in c]
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0]:
        line = (fname, int(r[0]))
        src[line] = r[1].strip()
    elif line is not None and r[2] not in ("", "-"):
        try:
            agg[line] += float(r[si])
            for i in stall_cols:
                why[line][hdr[i][6:]] += float(r[i])
        except ValueError:
            pass
tot = sum(agg.values()) or 1
print(f"total samples {tot:.0f}")
for (f, l), v in agg.most_common(n):
    top = ", ".join(f"{k}={c / v * 100:.0f}%" for k, c in why[(f, l)].most_common(2))
    print(f"{v / tot * 100:5.1f}%  {f}:{l:<5d} {src.get((f, l), '')[:70]:70s} [{top}]")

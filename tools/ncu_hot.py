"""Top SASS instructions by warp-stall samples of an .ncu-rep (dev tool).
python tools/ncu_hot.py REP [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
si, ai = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_")]
body = [r for r in rows[2:] if len(r) == len(h)]
tot = sum(float(r[si]) for r in body)
print(f"total samples {tot:.0f}, instructions {len(body)}")
for idx, r in sorted(enumerate(body), key=lambda x: -float(x[1][si]))[:n]:
    top = sorted(((float(r[i]), h[i][6:]) for i in stall_cols), reverse=True)[:2]
    print(f"{idx:5d} {float(r[si]) / tot * 100:5.1f}%  {r[ai].strip()[:60]:60s} {top[0][1]}={top[0][0]:.0f} {top[1][1]}={top[1][0]:.0f}")

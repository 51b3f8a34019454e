"""Dev tool: copy the round's bench lines from gpurun_out/ into profiles/ and regenerate the
per-config tables of BASELINE.md §4 and DESIGN.md §10, and the C3 ncu summary files.
python tools/refresh_docs.py TAG   (TAG: the tools/profile_round.sh tag of the C3 capture)"""
import glob
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else None
for f in glob.glob(os.path.join(ROOT, "gpurun_out", "r02_bench_*.json")):
    shutil.copy(f, os.path.join(ROOT, "profiles"))
if tag:
    g = lambda n: os.path.join(ROOT, "gpurun_out", f"{tag}_{n}")
    subprocess.run([sys.executable, "tools/ncu_traffic.py", g("traverse.ncu-rep"), "C3", "k_traverse_level",
                    "profiles/r02_traffic_c3.json"], cwd=ROOT, check=True)
    with open(os.path.join(ROOT, "profiles", "r02_c3_ncu_summary.md"), "w") as out:
        subprocess.run([sys.executable, "tools/ncu_summary.py", "r02 final", g("launches.csv"), g("traverse.ncu-rep"),
                        g("shade.ncu-rep"), g("bwd.ncu-rep"), g("primary.ncu-rep")], cwd=ROOT, check=True, stdout=out)
    shutil.copy(g("launches.csv"), os.path.join(ROOT, "profiles", "r02_c3_launches.csv"))
    with open(os.path.join(ROOT, "profiles", "r02_traverse_simt_by_line.txt"), "w") as out:
        subprocess.run([sys.executable, "tools/ncu_simt.py", g("traverse.ncu-rep"), "30"], cwd=ROOT, check=True, stdout=out)

names = {"C1": "C1 icosphere 320 tris, 1×64², D2, analytic env", "C2": "C2 50.7k tris, 8×256², D4, voxel+triplane env",
         "C3": "C3 499k tris, 100×800², D4", "C4": "C4 torus knot + gems 263k tris, 64³ σ grid, 50×800², D6",
         "C5": "C5 1M tris, 200×1024², D4 (1 GPU)", "C4H": "C4H = C4 + 16-level hash σ, 8 views",
         "C3V": "C3V = C3 + volumetric env", "C3R_infer": "C3R inference (fwd only, D8)"}
rows = {c: json.load(open(os.path.join(ROOT, "profiles", f"r02_bench_{c}.json"))) for c in names}
out = ["| Config | GPU Mray·bounce/s (device / e2e) | ms/step | segments/step | Oracle seg/s, 16 cores / 1 core (sample) "
       "| Oracle time for one full step (16 cores) | GPU / oracle (16 cores) | Dominant kernel, roofline frac |",
       "|---|---|---|---|---|---|---|---|"]
for c, d in rows.items():
    cb, r = d["cpu_baseline"], d["roofline"]
    seg = d["config"]["segments_per_step"]
    o, o1 = cb["value"] * 1e6, cb["value_1thread"] * 1e6
    t = seg / o
    ts = f"{t * 1e3:.0f} ms" if t < 1 else (f"{t:.1f} s" if t < 120 else (f"{t / 60:.0f} min" if t < 7200 else f"{t / 3600:.1f} h"))
    out.append(f"| {names[c]} | {d['value']:.0f} / {d['e2e']['value']:.0f} | {d['ms_per_step']:.2f} | {seg:,} | "
               f"{o:,.0f} / {o1:,.0f} | {ts} | {d['value'] / cb['value']:.2e} | {r['kernel']} ({r['bound']}), {r['frac']} |")
p = os.path.join(ROOT, "BASELINE.md")
s = open(p).read()
a = s.index("| Config | GPU Mray·bounce/s (device / e2e)")
s = s[:a] + "\n".join(out) + s[s.index("\n\n", a):]
open(p, "w").write(s)

b = json.load(open(os.path.join(ROOT, "profiles", "r02_bench_C3_batch5000.json")))


def line(c, label):
    d, r = rows[c], rows[c]["roofline"]
    k = r["kernel"].replace("k_traverse_level", "traverse").replace("k_backward_level", "backward")
    return (f"| {label} | {d['config']['segments_per_step'] / 1e6:.1f} M | {d['ms_per_step']:.1f} | {d['value']:.0f} | "
            f"{d['e2e']['value']:.0f} | {k}, {r['bound']} {r['frac']:.2f} |")


tab = "\n".join(["| Config | segments/step | ms/step | value | e2e | dominant kernel, roofline |", "|---|---|---|---|---|---|",
                 line("C2", "C2 (50.7k tris, 8 × 256², D 4)"), line("C3", "**C3** (499k tris, 100 × 800², D 4)"),
                 line("C4", "C4 (263k tris, σ grid, D 6)"), line("C5", "C5 (1M tris, 200 × 1024², D 4)"),
                 line("C4H", "C4H (C4 + 16-level hash texture, 8 views)"),
                 line("C3V", "C3V (C3 + volumetric env, 32 samples)"),
                 line("C3R_infer", "C3R inference (forward only, D 8, swapped env)"),
                 f"| C3, the paper's 5,000-ray batch (`--batch 5000`, CUDA graph) | 15 k | {b['ms_per_step']:.2f} | "
                 f"{b['value']:.1f} | — | build / launch bound; {b['iterations_per_s']:.0f} it/s, graph "
                 f"{b['graph_speedup']:.2f}× eager |"])
p = os.path.join(ROOT, "DESIGN.md")
s = open(p).read()
a = s.index("| Config | segments/step | ms/step | value | e2e | dominant kernel, roofline |")
s = s[:a] + tab + s[s.index("\n\n", a):]
open(p, "w").write(s)
print(tab)

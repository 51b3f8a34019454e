"""Which stage's float32 rounding moves the radiance?  ("sources of error")

Builds the oracle with -DDTO_PRECISION_STUDY (a separate .so under /tmp; liboracle.so is
untouched), then renders the parity pixels of a config with the value at ONE stage rounded to
float32 (camera ray, hit point, child directions, vertex normals, shading normal, env shell
point, barycentrics) and counts the pixels whose radiance moves by more than 1e-4 (or whose
path topology changes) against the unrounded float64 render.  CPU only; test infrastructure.

    python tools/precision_study.py C5 [n_pixels]
"""
import ctypes as C
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
from paper_2603_00413_b200 import scenes as S  # noqa: E402

STAGES = [(0, "none (fp64)"), (1, "camera ray"), (2, "hit point"), (4, "child directions"), (8, "vertex normals"),
          (16, "shading normal"), (32, "env shell point"), (64, "barycentrics"), (127, "all stages")]


def study_lib():
    so = "/tmp/liboracle_study.so"
    src = os.path.join(ROOT, "oracle", "oracle.cpp")
    if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-pthread", "-DDTO_PRECISION_STUDY", src,
                        "-o", so], check=True)
    lib = C.CDLL(so)
    for name in ("dto_render", "dto_camera_rays"):
        getattr(lib, name).restype = C.c_int
    return lib


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    seeds = dict(C1=None, C2=2, C3=3, C4=4, C5=6)
    sc = S.CONFIGS[cfg]()
    pid = np.arange(sc.n_pixels) if cfg == "C1" else S.central_pixels(sc.cams, n, seeds[cfg])
    O._lib = study_lib()
    osc = O.OracleScene(sc)
    O._lib.dto_study_set_mask(0)
    base = O.render(osc, pid)
    print(f"{cfg}: {len(pid)} pixels, oracle flags (edge/grazing/near-TIR) on {int((base['flags'] != 0).sum())}")
    for mask, name in STAGES:
        O._lib.dto_study_set_mask(mask)
        r = O.render(osc, pid)
        err = np.abs(r["rgb"] - base["rgb"]).max(1)
        topo = r["sig_topo"] != base["sig_topo"]
        moved = topo | (err > 1e-4)
        print(f"  {name:18s} moved>1e-4: {int(moved.sum()):4d} ({100 * moved.mean():5.1f}%)  topology: {int(topo.sum()):3d}"
              f"  max|d rgb| (same topology): {err[~topo].max() if (~topo).any() else 0:.2e}")
    O._lib.dto_study_set_mask(0)


if __name__ == "__main__":
    main()

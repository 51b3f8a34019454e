"""Per-depth radiance of one pixel, GPU vs oracle (dev tool)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle as O
from paper_2603_00413_b200 import scenes as S
from paper_2603_00413_b200.tracer import DeviceScene, Tracer
from tests import _scenes as T

V, F = S.icosphere(2)
cams = T.one_view(40, 28, (0.6, -0.4, 2.6), fov_deg=55)
px = int(sys.argv[1]) if len(sys.argv) > 1 else 68
dev = torch.device("cuda:0")
tr = Tracer(dev)
for cap in (0, 1):
    for D in range(0, 6):
        sc = T.scene(V, F, cams, env=T.small_volume_env(), D=D, cap=cap)
        o = O.render(O.OracleScene(sc), np.array([px]))["rgb"][0]
        ds = DeviceScene(sc, dev)
        tr.build_bvh(ds.V, ds.F)
        g = tr.trace_forward(ds, torch.as_tensor([px], device=dev)).rgb.cpu().numpy()[0]
        print("cap", cap, "D", D, "err", np.abs(g - o).max(), g, o)

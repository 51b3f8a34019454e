"""Pixel 68 at D=4/CAP_ZERO under variants of the volume env (dev tool)."""
import dataclasses
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
dev = torch.device("cuda:0")
tr = Tracer(dev)
px = 68
def run(env, D=4, cap=0, label=""):
    sc = T.scene(V, F, cams, env=env, D=D, cap=cap)
    orc = O.render(O.OracleScene(sc), np.array([px]))
    ds = DeviceScene(sc, dev)
    tr.build_bvh(ds.V, ds.F)
    out = tr.trace_forward(ds, torch.as_tensor([px], device=dev), want_capped=True)
    g = out.rgb.cpu().numpy()[0]
    print(label, "err", np.abs(g - orc["rgb"][0]).max(), "capw", float(out.capped_w.cpu()[0]), orc["capped_w"][0])
base = T.small_volume_env()
run(base, label="base")
z = T.small_volume_env(); z.voxel[..., 3] = 0; z.planes[..., 3] = 0
run(z, label="zero-density")
run(dataclasses.replace(z, kind=S.ENV_GRID), label="grid-env")
c = T.small_volume_env(); c.voxel[..., :3] = 0.5; c.planes[..., :3] = 0.0
run(c, label="const-colour")

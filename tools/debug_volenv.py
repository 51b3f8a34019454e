"""Worst pixels of the volumetric-env parity case (dev tool, GPU)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle as O
from paper_2603_00413_b200 import scenes as S
from paper_2603_00413_b200.tracer import DeviceScene, Tracer
from tests import _scenes as T
from tests._parity import oracle_forward, compare_forward

V, F = S.icosphere(2)
cams = T.one_view(40, 28, (0.6, -0.4, 2.6), fov_deg=55)
for M in (12, 48):
    sc = T.scene(V, F, cams, env=T.small_volume_env(n_samples=M), D=4)
    pid = np.arange(sc.n_pixels)
    osc = O.OracleScene(sc)
    orc = oracle_forward(O, osc, pid)
    dev = torch.device("cuda:0")
    ds = DeviceScene(sc, dev)
    tr = Tracer(dev)
    tr.build_bvh(ds.V, ds.F)
    out = tr.trace_forward(ds, torch.as_tensor(pid, device=dev), want_sig=True)
    rgb = out.rgb.cpu().numpy()
    cmp = compare_forward(rgb, out.sig_topo.cpu().numpy(), orc)
    print("M", M, {k: v for k, v in cmp.items() if "mask" not in k})
    err = np.abs(rgb - orc["rgb"]).max(1)
    for i in np.argsort(-err)[:6]:
        print(i, err[i], rgb[i], orc["rgb"][i], "flags", orc["flags"][i], "segs", orc["segments"][i],
              "sig_ok", out.sig_topo.cpu().numpy()[i] == orc["sig_topo"][i])

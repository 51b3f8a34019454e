"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck) on the GPU box:
every kernel family of libdifftrans.so on small seeded scenes -- the LBVH build with the
persistent wide collapse (C2 mesh, 50.7k triangles), forward + backward at C1 and on a reduced
C2 (2 views 64x64), the sigma-grid, hash-texture and volumetric-env kernels, the debug
closest-hit (BVH and brute force), one optimiser step with the periodic mesh pass.
    compute-sanitizer --tool racecheck python tools/sanitize_run.py"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_00413_b200 import scenes as S  # noqa: E402
from paper_2603_00413_b200.optim import RefineConfig, RefineOptimizer  # noqa: E402
from paper_2603_00413_b200.tracer import DeviceScene, Tracer  # noqa: E402

dev = torch.device("cuda:0")
tr = Tracer(dev)
cases = [("C1", S.config_c1()), ("C2s", S.config_c2(n_views=2, res=64)),
         ("C4s", S.config_c4(n_views=1, res=48)), ("C4Hs", S.config_c4h(n_views=1, res=48)),
         ("C3Vs", S.config_c3v(n_views=1, res=32, vres=32, pres=64))]
for name, sc in cases:
    ds = DeviceScene(sc, dev)
    tr.build_bvh(ds.V, ds.F)
    out = tr.trace_forward(ds, want_sig=True, stats=True)
    g = torch.as_tensor(S.upstream_grad(sc.n_pixels, 1), device=dev)
    tr.trace_backward(g)
    torch.cuda.synchronize()
    print(name, "segments", out.stats["segments"], flush=True)
# debug closest hit: BVH and brute force
sc = S.config_c2(n_views=1, res=32)
ds = DeviceScene(sc, dev)
tr.build_bvh(ds.V, ds.F)
rays = torch.randn(512, 6, device=dev)
rays[:, :3] *= 0.2
tr.closest_hit(rays, 0.0, brute_force=False)
tr.closest_hit(rays, 0.0, brute_force=True)
tr.bvh_check()
# one optimiser step (async forward, loss, backward, regularisers, Adam) + the mesh pass
sc = S.config_c2(n_views=2, res=48)
ds = DeviceScene(sc, dev)
tr.build_bvh(ds.V, ds.F)
target = tr.trace_forward(ds).rgb.clone() * 0.9
_, _, masks = tr.mask_loss(ds, torch.zeros(sc.n_pixels, device=dev), 0.0, want_mask=True)
opt = RefineOptimizer(tr, ds, RefineConfig(freeze_iters=0, reg_every=1, reg_inner=1), seed=1)
opt.step(target, async_=True, gt_masks=masks.contiguous())
opt.step(target, async_=True)
torch.cuda.synchronize()
print("sanitize workload done", flush=True)

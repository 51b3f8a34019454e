"""Dev diagnostic (GPU box): where does the L_mask gradient of the CUDA path differ from the
oracle's?  Per-vertex error concentration and, per silhouette sample, whether its visibility
decision flips when the sample point moves by +-delta px along the edge normal.
python tools/mask_diag.py [delta]"""
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
from oracle import mask as OM  # noqa: E402
from paper_2603_00413_b200 import scenes as S  # noqa: E402
from paper_2603_00413_b200.tracer import DeviceScene, Tracer  # noqa: E402
from tests import _scenes as T  # noqa: E402

delta = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-4
V, F = S.icosphere(2)
cams = T.one_view(48, 48, (0.3, 0.2, 3.0), fov_deg=50, up=(0.0, 1.0, 0.0))
sc = T.scene(V, F, cams, D=0)
osc = O.OracleScene(sc)
m = OM.rendered_mask(osc, cams, 0)
ys, xs = np.mgrid[0:48, 0:48]
gt = ((xs + 0.5 - 26) ** 2 + (ys + 0.5 - 22) ** 2 <= (0.8 * np.sqrt(m.sum() / np.pi)) ** 2).astype(np.float32)[None]
tr = Tracer("cuda:0")
ds = DeviceScene(sc, torch.device("cuda:0"))
tr.build_bvh(ds.V, ds.F)
loss, gV, mask = tr.mask_loss(ds, torch.as_tensor(gt, device="cuda:0").contiguous(), 1.0, want_mask=True)
gg = gV.cpu().numpy().astype(np.float64)
go = OM.gradient(osc, sc, gt)
err = gg - go
print("rel-L2", np.linalg.norm(err) / np.linalg.norm(go), "mask diff", int((mask.cpu().numpy()[0] != m).sum()))
en = np.linalg.norm(err, axis=1)
order = np.argsort(-en)
print("top vertex errors (|err|, |g_oracle|):")
for i in order[:12]:
    print(f"  v{i:4d} {en[i]:.3e} {np.linalg.norm(go[i]):.3e}  err={err[i]}")
print("share of err^2 in top 4 vertices:", (en[order[:4]] ** 2).sum() / (en ** 2).sum())

# per-sample ambiguity in the oracle
Vd, Fd = np.asarray(sc.V, np.float64), np.asarray(sc.F, np.int64)
W, H = cams.width, cams.height
cam = np.asarray(cams.c2w[0], np.float64)[:, 3]
n_s = n_amb = 0
amb_g = np.zeros_like(go)
for a, b, fr in OM.silhouette_edges(Vd, Fd, cam):
    c = [int(x) for x in Fd[fr] if x != a and x != b][0]
    pa, Ja = OM.project(cams, 0, Vd[a])
    pb, Jb = OM.project(cams, 0, Vd[b])
    pc, _ = OM.project(cams, 0, Vd[c])
    e = pb - pa
    L = float(np.hypot(*e))
    nrm = np.array([-e[1], e[0]]) / L
    if nrm @ (pc - pa) > 0:
        nrm = -nrm
    K = max(1, math.ceil(L / 0.5))
    s = (np.arange(K) + 0.5) / K
    x = pa[None] + s[:, None] * e[None]
    for sgn_o in (1,):
        pass
    res = {}
    for tag, off in (("o", 0.02), ("i", -0.02)):
        for dd in (-delta, 0.0, delta):
            pts = x + (off + dd) * nrm
            f, _, _ = O.closest_hit(osc, OM._rays_at(cams, 0, pts))
            res[(tag, dd)] = f >= 0
    for k in range(K):
        xo = x[k] + 0.02 * nrm
        if not (0 <= xo[0] < W and 0 <= xo[1] < H):
            continue
        acc = (not res[("o", 0.0)][k]) and res[("i", 0.0)][k]
        flip = any(res[(t, dd)][k] != res[(t, 0.0)][k] for t in ("o", "i") for dd in (-delta, delta))
        # gt pixel near a boundary?
        gflip = abs(xo[0] - round(xo[0])) < delta or abs(xo[1] - round(xo[1])) < delta
        n_s += 1
        if flip or gflip:
            n_amb += 1
            gtv = gt[0][int(xo[1]), int(xo[0])]
            w = (1.0 - 2.0 * gtv) * (L / K) / (W * H)
            amb_g[a] += w * (1 - s[k]) * (Ja.T @ nrm)
            amb_g[b] += w * s[k] * (Jb.T @ nrm)
            print(f"  ambiguous sample edge ({a},{b}) k={k} accepted={acc} vis-flip={flip} gt-edge={gflip}")
print(f"samples {n_s}, ambiguous at delta={delta}: {n_amb}; |amb contribution| / |g| = "
      f"{np.linalg.norm(amb_g) / np.linalg.norm(go):.3e}")

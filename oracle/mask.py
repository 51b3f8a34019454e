"""Oracle of the mask regulariser L_mask and its silhouette-edge-sampling gradient (SURVEY
NEXT-4, reading R32).  TEST INFRASTRUCTURE ONLY; float64, plain loops.

  rendered mask  M^(x, y) = 1 iff the camera ray through the pixel centre hits the mesh (R19)
  L_mask         (1 / (n_views W H)) sum_pixels |M^ - M|  (mean form)
  gradient       of the area-coverage relaxation: moving the projected outer boundary of the
                 mesh by dn (outward) at a point x changes the loss by (1 - 2 M(x+)) dn / N,
                 M(x+) = the ground-truth pixel just outside.  The outer boundary is made of
                 silhouette edges (shared by a front- and a back-facing face, or boundary edges),
                 projected; a point at screen parameter s of edge (a, b) moves by
                 (1 - s) dP(v_a) + s dP(v_b) (P = pinhole projection).  The boundary integral is
                 taken with midpoint samples every `spacing` pixels; a sample counts when the
                 screen point eps inside is covered and the point eps outside is not.
Visibility uses the fp64 oracle's brute-force closest hit.  Shares no code with csrc.
"""
from __future__ import annotations

import math

import numpy as np

from . import OracleScene, closest_hit


def _rays_at(cams, v, uv):
    """camera rays [n][6] through continuous image points uv [n][2] of view v (R19)."""
    fx, fy, cx, cy = [float(a) for a in cams.K[v]]
    c2w = np.asarray(cams.c2w[v], np.float64)
    d = np.stack([(uv[:, 0] - cx) / fx, (uv[:, 1] - cy) / fy, np.ones(len(uv))], 1) @ c2w[:, :3].T
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    o = np.broadcast_to(c2w[:, 3], d.shape)
    return np.concatenate([o, d], 1)


def rendered_mask(osc: OracleScene, cams, v):
    W, H = cams.width, cams.height
    ys, xs = np.mgrid[0:H, 0:W]
    uv = np.stack([xs.ravel() + 0.5, ys.ravel() + 0.5], 1).astype(np.float64)
    face, _, _ = closest_hit(osc, _rays_at(cams, v, uv))
    return (face >= 0).reshape(H, W).astype(np.float64)


def loss(osc: OracleScene, cams, gt):
    n = cams.n_views * cams.width * cams.height
    return float(sum(np.abs(rendered_mask(osc, cams, v) - gt[v]).sum() for v in range(cams.n_views)) / n)


def project(cams, v, X):
    """(uv [2], J [2][3] = d uv / d X) of world point X in view v."""
    fx, fy, cx, cy = [float(a) for a in cams.K[v]]
    c2w = np.asarray(cams.c2w[v], np.float64)
    R, t = c2w[:, :3], c2w[:, 3]
    Xc = R.T @ (np.asarray(X, np.float64) - t)
    x, y, z = Xc
    uv = np.array([fx * x / z + cx, fy * y / z + cy])
    Jc = np.array([[fx / z, 0.0, -fx * x / (z * z)], [0.0, fy / z, -fy * y / (z * z)]])
    return uv, Jc @ R.T


def silhouette_edges(V, F, cam_pos):
    """(a, b, front face) for edges whose incident faces disagree in facing (or boundary edges)."""
    V = np.asarray(V, np.float64)
    F = np.asarray(F, np.int64)
    n = np.cross(V[F[:, 1]] - V[F[:, 0]], V[F[:, 2]] - V[F[:, 0]])
    front = ((cam_pos - V[F[:, 0]]) * n).sum(1) > 0
    faces_of = {}
    for f in range(len(F)):
        for k in range(3):
            a, b = int(F[f, k]), int(F[f, (k + 1) % 3])
            faces_of.setdefault((min(a, b), max(a, b)), []).append(f)
    out = []
    for (a, b), fs in faces_of.items():
        fr = [f for f in fs if front[f]]
        if len(fs) == 1 and fr:
            out.append((a, b, fr[0]))
        elif len(fs) == 2 and len(fr) == 1:
            out.append((a, b, fr[0]))
    return out


def gradient(osc: OracleScene, sc, gt, spacing: float = 0.5, eps: float = 0.02):
    """dL_mask/dV [nv][3] by silhouette edge sampling (R32)."""
    V = np.asarray(sc.V, np.float64)
    F = np.asarray(sc.F, np.int64)
    cams = sc.cams
    W, H = cams.width, cams.height
    N = cams.n_views * W * H
    g = np.zeros_like(V)
    for v in range(cams.n_views):
        cam = np.asarray(cams.c2w[v], np.float64)[:, 3]
        for a, b, fr in silhouette_edges(V, F, cam):
            c = [int(x) for x in F[fr] if x != a and x != b][0]
            pa, Ja = project(cams, v, V[a])
            pb, Jb = project(cams, v, V[b])
            pc, _ = project(cams, v, V[c])
            e = pb - pa
            L = float(np.hypot(*e))
            if L == 0.0:
                continue
            nrm = np.array([-e[1], e[0]]) / L
            if nrm @ (pc - pa) > 0:                      # outward: away from the front face
                nrm = -nrm
            K = max(1, math.ceil(L / spacing))
            s = (np.arange(K) + 0.5) / K
            x = pa[None] + s[:, None] * e[None]
            xo, xi = x + eps * nrm, x - eps * nrm
            ok = (xo[:, 0] >= 0) & (xo[:, 0] < W) & (xo[:, 1] >= 0) & (xo[:, 1] < H)
            if not ok.any():
                continue
            fo, _, _ = closest_hit(osc, _rays_at(cams, v, xo))
            fi, _, _ = closest_hit(osc, _rays_at(cams, v, xi))
            for k in np.flatnonzero(ok & (fo < 0) & (fi >= 0)):
                gtv = gt[v][int(xo[k, 1]), int(xo[k, 0])]
                w = (1.0 - 2.0 * gtv) * (L / K) / N
                g[a] += w * (1.0 - s[k]) * (Ja.T @ nrm)
                g[b] += w * s[k] * (Jb.T @ nrm)
    return g

"""Pins of the mask-regulariser oracle (NEXT-4; reading R32):

(i)   a front-facing quad against an empty / full ground truth: the edge-sampling gradient is
      (+/-) the derivative of the quad's projected area (shoelace formula, chained through the
      pinhole Jacobian) divided by the pixel count -- the exact derivative of the coverage
      relaxation;
(ii)  a sphere inside a larger ground-truth disk: the descent direction -dL/dV points outward
      on the silhouette, and a small step along it lowers the pixel mask loss;
(iii) the loss value: |M^ - M| averaged over pixels, zero when the ground truth is the render.
"""
import numpy as np

import oracle as O
from oracle import mask as OM
from paper_2603_00413_b200 import scenes as S
from tests import _scenes as T


def quad_scene(W=48, H=40):
    V = np.array([[-0.5, -0.4, 0.0], [0.6, -0.5, 0.0], [0.5, 0.45, 0.0], [-0.45, 0.5, 0.0]], np.float32)
    F = np.array([[0, 1, 2], [0, 2, 3]], np.int32)
    cams = T.one_view(W, H, (0.1, 0.05, 3.0), fov_deg=40, up=(0.0, 1.0, 0.0))
    sc = T.scene(V, F, cams, D=0)
    cam = np.asarray(cams.c2w[0], np.float64)[:, 3]
    n = np.cross(V[1] - V[0], V[2] - V[0])
    if n @ (cam - V[0]) < 0:                                   # make the faces front-facing
        sc = T.scene(V, F[:, ::-1].copy(), cams, D=0)
    return sc


def area_gradient(sc):
    cams = sc.cams
    P, J = zip(*[OM.project(cams, 0, x) for x in sc.V.astype(np.float64)])
    P = np.array(P)
    order = [0, 1, 2, 3]
    A = 0.5 * sum(P[order[i]][0] * P[order[(i + 1) % 4]][1] - P[order[(i + 1) % 4]][0] * P[order[i]][1] for i in range(4))
    sg = np.sign(A)
    g = np.zeros((4, 3))
    for i in range(4):
        nx, pv = P[(i + 1) % 4], P[(i - 1) % 4]
        dA = sg * 0.5 * np.array([nx[1] - pv[1], pv[0] - nx[0]])
        g[i] = J[i].T @ dA
    return g, abs(A)


def test_quad_gradient_is_the_area_derivative():
    sc = quad_scene()
    osc = O.OracleScene(sc)
    N = sc.cams.width * sc.cams.height
    gA, A = area_gradient(sc)
    for gtv, sign in ((0.0, 1.0), (1.0, -1.0)):
        gt = np.full((1, sc.cams.height, sc.cams.width), gtv)
        g = OM.gradient(osc, sc, gt, spacing=0.25)
        np.testing.assert_allclose(g, sign * gA / N, rtol=2e-2, atol=2e-3 * np.abs(gA).max() / N)
    # loss: the rendered mask's pixel count ~ the projected area
    gt = np.zeros((1, sc.cams.height, sc.cams.width))
    L = OM.loss(osc, sc.cams, gt)
    assert abs(L * N - A) < 0.05 * A
    assert OM.loss(osc, sc.cams, OM.rendered_mask(osc, sc.cams, 0)[None]) == 0.0


def test_sphere_in_larger_disk_grows():
    V, F = S.icosphere(2)
    cams = T.one_view(48, 48, (0.0, 0.0, 3.0), fov_deg=50, up=(0.0, 1.0, 0.0))
    sc = T.scene(V, F, cams, D=0)
    osc = O.OracleScene(sc)
    m = OM.rendered_mask(osc, cams, 0)
    ys, xs = np.mgrid[0:48, 0:48]
    r = np.sqrt(m.sum() / np.pi)
    gt = ((xs + 0.5 - 24) ** 2 + (ys + 0.5 - 24) ** 2 <= (1.3 * r) ** 2).astype(np.float64)[None]
    g = OM.gradient(osc, sc, gt)
    act = np.linalg.norm(g, axis=1) > 0
    assert act.sum() >= 10
    radial = V.astype(np.float64)[act]
    radial[:, 2] = 0.0                                   # outward in the image plane
    out = ((-g[act]) * radial).sum(1) > 0
    assert out.mean() >= 0.95, out.mean()
    L0 = OM.loss(osc, cams, gt)
    step = 0.05 / np.abs(g).max()
    sc2 = T.scene((V - step * g).astype(np.float32), F, cams, D=0)
    assert OM.loss(O.OracleScene(sc2), cams, gt) < L0

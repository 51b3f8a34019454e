"""Pins of the oracle's geometry and recursive transport against closed forms
(P:154-174 recursive tracing, P:124-137 Beer-Lambert, P:165-174 intersection)."""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
from paper_2603_00413_b200 import scenes as S
from tests import _scenes as T

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "closed_forms.json")))


# ----------------------------------------------------------------------------- geometry
def test_vertex_normals_closed_forms():
    # flat fan: every vertex normal is the plane normal
    V = np.array([[0, 0, 0], [1, 0, 0], [0.5, 0.8, 0], [-0.6, 0.7, 0], [-0.9, -0.3, 0]], np.float32)
    F = np.array([[0, 1, 2], [0, 2, 3], [0, 3, 4]], np.int32)
    cams = T.one_view(2, 2, (0, 0, 3))
    n = O.vertex_normals(O.OracleScene(T.scene(V, F, cams)))
    np.testing.assert_allclose(n, np.tile([0, 0, 1.0], (5, 1)), atol=1e-15)
    # right-angle corner, each of the 3 faces contributes once -> -(1,1,1)/sqrt3 (S: vertex_normals)
    V = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], np.float32)
    F = np.array([[0, 2, 1], [0, 1, 3], [0, 3, 2]], np.int32)
    n = O.vertex_normals(O.OracleScene(T.scene(V, F, cams)))
    np.testing.assert_allclose(n[0], -np.ones(3) / math.sqrt(3), atol=1e-15)


def test_icosphere_vertex_normals_near_radial():
    V, F = S.icosphere(2)
    n = O.vertex_normals(O.OracleScene(T.scene(V, F, T.one_view(2, 2, (0, 0, 3)))))
    radial = V / np.linalg.norm(V, axis=1, keepdims=True)
    ang = np.degrees(np.arccos(np.clip((n * radial).sum(1), -1, 1)))
    assert ang.max() < 2.0


def test_closest_hit_centroid_and_sphere():
    V = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], np.float32)
    F = np.array([[0, 1, 2]], np.int32)
    osc = O.OracleScene(T.scene(V, F, T.one_view(2, 2, (0, 0, 3))))
    c = V.mean(0).astype(np.float64)
    face, tuv, _ = O.closest_hit(osc, [[c[0], c[1], 2.0, 0, 0, -1]])
    assert face[0] == 0 and abs(tuv[0, 0] - 2.0) < 1e-15
    np.testing.assert_allclose(tuv[0, 1:], [1 / 3, 1 / 3], atol=1e-15)
    # miss outside, and t_lo offset contract
    face, _, _ = O.closest_hit(osc, [[1.0, 1.0, 2.0, 0, 0, -1]])
    assert face[0] == -1
    # icosphere s3: ray from the centre along a face axis meets the face at its inradius
    for s, gold in zip(GOLD["icosphere_axis_face_distance"]["subdiv"], GOLD["icosphere_axis_face_distance"]["value"]):
        V, F = S.icosphere(s, face_axis_to_z=True)
        osc = O.OracleScene(T.scene(V, F, T.one_view(2, 2, (0, 0, 3))))
        face, tuv, _ = O.closest_hit(osc, [[0, 0, 0, 0, 0, 1.0], [0, 0, 0, 0, 0, -1.0]])
        np.testing.assert_allclose(tuv[:, 0], gold, atol=2e-7)  # float32 vertices
    # sphere mesh from (0,0,3) toward the centre: t ~ 2 up to the chord error (S: intersect)
    V, F = S.icosphere(3)
    osc = O.OracleScene(T.scene(V, F, T.one_view(2, 2, (0, 0, 3))))
    g = np.random.default_rng(1)
    dirs = g.normal(size=(200, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    o = 3 * dirs
    face, tuv, _ = O.closest_hit(osc, np.concatenate([o, -dirs], 1))
    assert (face >= 0).all()
    assert np.abs(tuv[:, 0] - 2.0).max() < 1 - 0.9954716324  # within the sagitta at s3
    # secondary-ray offset: from the hit point, t_lo = 1e-4 re-hits the far side (S: intersect)
    x = o + tuv[:, :1] * -dirs
    f2, t2, _ = O.closest_hit(osc, np.concatenate([x, -dirs], 1), t_lo=1e-4)
    assert (f2 != face).all() and (t2[:, 0] > 1.9).all()


def test_brute_force_tie_break_lowest_id():
    """Two coincident triangles: equal t resolves to the lower face id (R18), and the
    hit is flagged as a tie."""
    V = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], np.float32)
    F = np.array([[0, 1, 2], [0, 1, 2], [0, 2, 1]], np.int32)
    osc = O.OracleScene(T.scene(V, F, T.one_view(2, 2, (0, 0, 3))))
    face, _, flags = O.closest_hit(osc, [[0.2, 0.3, 1.0, 0, 0, -1]])
    assert face[0] == 0 and flags[0] & O.FLAG_EDGE


# ----------------------------------------------------------------------------- media / env
def test_transmittance_closed_forms():
    V, F = S.icosphere(1)
    sc = T.scene(V, F, T.one_view(2, 2, (0, 0, 3)), sigma=(1.0, 1.0, 1.0))
    tau = O.transmittance(O.OracleScene(sc), [0.1, 0.2, 0.3], [0.1, 0.2, 1.3])
    np.testing.assert_allclose(tau, GOLD["unit_medium_transmittance"]["value"], atol=1e-15)
    # linear ramp field on the grid: midpoint quadrature is exact for linear integrands
    res = 5
    lo, hi = np.array([-1, -1, -1.0]), np.array([1, 1, 1.0])
    ax = np.linspace(-1, 1, res)
    zz, yy, xx = np.meshgrid(ax, ax, ax, indexing="ij")
    sig = np.stack([1 + 0.5 * xx, 1 + 0.25 * yy - 0.2 * zz, 2 + 0.3 * xx + 0.3 * zz], -1).astype(np.float32)
    for N in (1, 7, 64):
        ab = S.Absorption(S.ABS_GRID, sig, lo.astype(np.float32), hi.astype(np.float32), N)
        osc = O.OracleScene(T.scene(V, F, T.one_view(2, 2, (0, 0, 3)), absorption=ab))
        o, x = np.array([-0.7, 0.3, -0.4]), np.array([0.8, -0.6, 0.5])
        mid = (o + x) / 2
        L = np.linalg.norm(x - o)
        exact = np.exp(-L * np.array([1 + 0.5 * mid[0], 1 + 0.25 * mid[1] - 0.2 * mid[2], 2 + 0.3 * mid[0] + 0.3 * mid[2]]))
        np.testing.assert_allclose(O.transmittance(osc, o, x), exact, rtol=2e-7)  # float32 texels
        # outside the box the field is zero (R11)
        np.testing.assert_allclose(O.transmittance(osc, [2, 2, 2], [3, 2.5, 2]), 1.0, atol=0)


def test_env_closed_forms():
    V, F = S.icosphere(0)
    cams = T.one_view(2, 2, (0, 0, 3))
    # analytic: a lobe at its own axis returns ambient + w (+ other lobes), at -mu w e^{-2 kappa}
    env = S.Env(S.ENV_ANALYTIC, ambient=np.array([0.1, 0.2, 0.3], np.float32),
                lobes=np.array([[0, 0, 1, 5.0, 1.0, 2.0, 3.0]], np.float32))
    osc = O.OracleScene(T.scene(V, F, cams, env=env))
    np.testing.assert_allclose(O.env(osc, [0, 0, 0], [0, 0, 2.0]), [1.1, 2.2, 3.3], atol=1e-7)
    np.testing.assert_allclose(O.env(osc, [0, 0, 0], [0, 0, -1.0]),
                               np.array([0.1, 0.2, 0.3]) + np.array([1, 2, 3.0]) * math.exp(-10), atol=1e-7)
    # grid: a linear voxel field returns the shell point p itself: |p| = R_e, p on the ray
    osc = O.OracleScene(T.scene(V, F, cams, env=T.linear_grid_env()))
    g = np.random.default_rng(2)
    for _ in range(50):
        o = g.uniform(-2, 2, 3)
        d = g.normal(size=3)
        p = O.env(osc, o, d)
        assert abs(np.linalg.norm(p) - 10.0) < 1e-12 * 10 * 4
        dh = d / np.linalg.norm(d)
        t = (p - o) @ dh
        assert t > 0 and np.linalg.norm(o + t * dh - p) < 1e-11
    # constant field -> constant
    e = S.grid_env(3, 6, 8)
    e.voxel[..., :3] = 0.5
    e.planes[..., :3] = 0.25
    osc = O.OracleScene(T.scene(V, F, cams, env=e))
    np.testing.assert_allclose(O.env(osc, [0.3, 0, 1], [1, 2, 3.0]), 0.5 + 3 * 0.25, atol=1e-15)


# ----------------------------------------------------------------------------- transport
def slab_expected(eta, sig, d, D, Lf, Lb):
    R = ((eta - 1) / (eta + 1)) ** 2
    Tt = 1 - R
    sig = np.asarray(sig, np.float64)
    fwd = sum(Tt * Tt * R ** (2 * k) * np.exp(-(2 * k + 1) * sig * d) for k in range(0, (D - 2) // 2 + 1))
    back = R + sum(Tt * Tt * R ** (2 * k + 1) * np.exp(-(2 * k + 2) * sig * d) for k in range(0, (D - 3) // 2 + 1))
    return Lf * fwd + Lb * back


@pytest.mark.parametrize("eta", [1.3, 1.5])
@pytest.mark.parametrize("sig", [(0, 0, 0), (0.5, 0.5, 0.5), (2.0, 0.5, 0.0)])
@pytest.mark.parametrize("D", [2, 4, 6, 8])
def test_slab_series(eta, sig, D):
    """Normal incidence on a tessellated slab (exact float32 geometry, vertex normals equal
    the face normal): the tree sums the truncated multi-bounce series."""
    V, F = S.slab(0.5, 4.0, 4)
    sc = T.scene(V, F, T.one_view(2, 2, (0, 0, 3)), env=T.lobe_env(), ior=eta, sigma=sig, D=D)
    osc = O.OracleScene(sc)
    ray = [[0.3, 0.2, 3.0, 0, 0, -1.0]]
    out = O.render(osc, rays=ray)
    Lf = O.env(osc, [0, 0, 0], [0, 0, -1.0])
    Lb = O.env(osc, [0, 0, 0], [0, 0, 1.0])
    np.testing.assert_allclose(out["rgb"][0], slab_expected(eta, sig, 0.5, D, Lf, Lb), atol=1e-12)
    if eta == 1.5 and sig == (0, 0, 0):
        i = GOLD["slab_W_fwd"]["D"].index(D)
        # the same numbers through the printed tables (one lobe env up = 1, down = 0 etc.)
        wf = slab_expected(1.5, (0, 0, 0), 0.5, D, 1.0, 0.0)[0]
        wb = slab_expected(1.5, (0, 0, 0), 0.5, D, 0.0, 1.0)[0]
        assert abs(wf - GOLD["slab_W_fwd"]["value"][i]) < 1e-12
        assert abs(wb - GOLD["slab_W_back"]["value"][i]) < 1e-12
        assert abs(wf - GOLD["slab_W_fwd"]["printed"][i]) < 1e-9     # SURVEY's rounded table
        assert abs(wb - GOLD["slab_W_back"]["printed"][i]) < 1e-9
        if D in GOLD["slab_W_cap"]["D"]:
            assert abs(out["capped_w"][0] - GOLD["slab_W_cap"]["value"][GOLD["slab_W_cap"]["D"].index(D)]) < 1e-15
        assert abs(wf + wb + out["capped_w"][0] - 1.0) < 1e-12
    assert out["segments"][0] <= 2 ** (D + 1) - 1


def test_slab_full_series_limit():
    wf = slab_expected(1.5, (0, 0, 0), 0.5, 60, 1.0, 0.0)[0]
    assert abs(wf - GOLD["slab_full_series"]["value"]) < 1e-6


def test_c1_axis_pixel_is_slab_series():
    """C1's own mesh: pixel (31,31) is the face-axis ray; the two hit faces are parallel at
    distance 2*0.98224694.  float32 vertices bound the agreement to 1e-7."""
    sc = S.config_c1()
    osc = O.OracleScene(sc)
    out = O.render(osc, [31 * 64 + 31])
    Lf = O.env(osc, [0, 0, 0], [0, 0, -1.0])
    Lb = O.env(osc, [0, 0, 0], [0, 0, 1.0])
    d = 2 * GOLD["icosphere_axis_face_distance"]["value"][2]
    np.testing.assert_allclose(out["rgb"][0], slab_expected(1.5, (0.2, 0.5, 1.0), d, 2, Lf, Lb), atol=1e-7)
    assert out["flags"][0] == 0


def test_energy_conservation_and_cap_policies():
    """sigma = 0, constant env L0 = 1: every event has R + T = 1, so CAP_ZERO gives
    1 - W_cap and CAP_ENV gives exactly 1 (SURVEY §8c.3 'Energy')."""
    base = S.config_c1()
    env = S.constant_env((1.0, 1.0, 1.0))
    for D in (2, 4):
        sc = T.scene(base.V, base.F, base.cams, env=env, sigma=(0, 0, 0), D=D)
        out = O.render(O.OracleScene(sc), np.arange(64 * 64))
        np.testing.assert_allclose(out["rgb"], np.repeat(1 - out["capped_w"][:, None], 3, 1), atol=1e-12)
        assert (out["segments"] <= 2 ** (D + 1) - 1).all()
        assert (out["capped_w"] >= 0).all() and (out["capped_w"] <= 1 + 1e-12).all()
        sc = T.scene(base.V, base.F, base.cams, env=env, sigma=(0, 0, 0), D=D, cap=S.CAP_ENV)
        out = O.render(O.OracleScene(sc), np.arange(64 * 64))
        np.testing.assert_allclose(out["rgb"], 1.0, atol=1e-12)


def test_optical_absence():
    """eta = 1, sigma = 0: the object is optically absent."""
    base = S.config_c1()
    sc = T.scene(base.V, base.F, base.cams, env=base.env, ior=1.0, sigma=(0, 0, 0), D=2)
    osc = O.OracleScene(sc)
    pid = np.arange(64 * 64)
    out = O.render(osc, pid)
    empty = T.scene(np.array([[100, 100, 100], [101, 100, 100], [100, 101, 100]]), np.array([[0, 1, 2]]),
                    base.cams, env=base.env)
    ref = O.render(O.OracleScene(empty), pid)
    np.testing.assert_allclose(out["rgb"], ref["rgb"], atol=1e-12)
    assert (out["segments"] > 1).sum() > 1000   # the object is hit, just invisible


def test_absorption_scales_inside_paths_only():
    """Doubling sigma on the slab multiplies the k-th inside branch by e^{-(...) sigma d}
    exactly as the series says; sigma never touches exterior paths (R9)."""
    V, F = S.slab(0.5, 4.0, 4)
    for sig in (0.1, 0.7):
        sc = T.scene(V, F, T.one_view(2, 2, (0, 0, 3)), env=T.lobe_env(), sigma=(sig,) * 3, D=4)
        osc = O.OracleScene(sc)
        out = O.render(osc, rays=[[0.3, 0.2, 3.0, 0, 0, -1.0]])
        Lb = O.env(osc, [0, 0, 0], [0, 0, 1.0])
        Lf = O.env(osc, [0, 0, 0], [0, 0, -1.0])
        np.testing.assert_allclose(out["rgb"][0], slab_expected(1.5, (sig,) * 3, 0.5, 4, Lf, Lb), atol=1e-12)


# ----------------------------------------------------------------------------- discriminating pins
def test_vertex_normal_uniform_not_area_weighted():
    """R6: n_v = normalize(sum of incident UNIT face normals).  The apex is shared
    by a tiny face in the plane z = 0 (normal +z, area 2e-6) and a large face in the plane
    x = 0 (normal +x, area 50): uniform weights give (1, 0, 1)/sqrt 2 exactly, area weights
    (summing raw cross products) would give ~+x."""
    V = np.array([[0, 0, 0], [1e-3, 0, 0], [0, 1e-3, 0], [0, 10, 0], [0, 0, 10]], np.float32)
    F = np.array([[0, 1, 2], [0, 3, 4]], np.int32)
    n = O.vertex_normals(O.OracleScene(T.scene(V, F, T.one_view(2, 2, (0, 0, 3)))))
    np.testing.assert_allclose(n[0], [1 / math.sqrt(2), 0, 1 / math.sqrt(2)], atol=1e-15)
    np.testing.assert_allclose(n[1:3], [[0, 0, 1.0]] * 2, atol=1e-15)
    np.testing.assert_allclose(n[3:], [[1.0, 0, 0]] * 2, atol=1e-15)
    # three unequal faces around a corner: still the normalised sum of the three axes
    V = np.array([[0, 0, 0], [5, 0, 0], [0, 0.01, 0], [0, 0, 2]], np.float32)
    F = np.array([[0, 2, 1], [0, 1, 3], [0, 3, 2]], np.int32)
    n = O.vertex_normals(O.OracleScene(T.scene(V, F, T.one_view(2, 2, (0, 0, 3)))))
    np.testing.assert_allclose(n[0], -np.ones(3) / math.sqrt(3), atol=1e-15)


def triplane_linear_env(pres=5, radius=10.0, far_field=0):
    """Zero voxel; each plane holds a distinct linear function of ITS OWN two axes, written
    in the documented layout P_xy[y][x], P_xz[z][x], P_yz[z][y] (row index = second axis).
    Per channel c: P_xy = A[c] (x, y), P_xz = B[c] (x, z), P_yz = C[c] (y, z)."""
    ax = np.linspace(-radius, radius, pres)
    row, col = np.meshgrid(ax, ax, indexing="ij")          # [row][col] coordinates
    A = np.array([[1.0, 2.0], [0.5, -1.0], [3.0, 0.25]])    # (x, y) coefficients per channel
    B = np.array([[-2.0, 0.75], [1.5, 4.0], [0.1, -3.0]])   # (x, z)
    Cc = np.array([[0.3, -0.6], [-2.5, 1.0], [2.0, 5.0]])   # (y, z)
    planes = np.zeros((3, pres, pres, 4), np.float32)
    for c in range(3):
        planes[0, :, :, c] = A[c, 0] * col + A[c, 1] * row   # P_xy[y][x]: col = x, row = y
        planes[1, :, :, c] = B[c, 0] * col + B[c, 1] * row   # P_xz[z][x]: col = x, row = z
        planes[2, :, :, c] = Cc[c, 0] * col + Cc[c, 1] * row  # P_yz[z][y]: col = y, row = z
    vox = np.zeros((3, 3, 3, 4), np.float32)
    env = S.Env(S.ENV_GRID, voxel=vox, planes=planes, radius=radius, far_field=far_field)

    def expected(p):
        x, y, z = p
        return np.array([A[c, 0] * x + A[c, 1] * y + B[c, 0] * x + B[c, 1] * z + Cc[c, 0] * y + Cc[c, 1] * z
                         for c in range(3)])
    return env, expected


def test_env_triplane_layout_and_far_field():
    """R14 / P:91 triplane layout: every plane reproduces its own linear function exactly, so a
    swapped row/column on any plane changes the value.  Far field (R14): the lookup point is
    R_e d/|d| whatever the origin."""
    V, F = S.icosphere(0)
    cams = T.one_view(2, 2, (0, 0, 3))
    g = np.random.default_rng(4)
    for ff in (0, 1):
        env, expected = triplane_linear_env(far_field=ff)
        osc = O.OracleScene(T.scene(V, F, cams, env=env))
        for _ in range(40):
            o = g.uniform(-2, 2, 3)
            d = g.normal(size=3)
            dh = d / np.linalg.norm(d)
            if ff:
                p = 10.0 * dh
            else:                                               # |o + t dh| = R_e, t > 0
                b = o @ dh
                p = o + (-b + math.sqrt(b * b - o @ o + 100.0)) * dh
            np.testing.assert_allclose(O.env(osc, o, d), expected(p), atol=1e-11)
    # far field with a linear voxel field: the value is R_e d^ for any origin
    env = T.linear_grid_env()
    env.far_field = 1
    osc = O.OracleScene(T.scene(V, F, cams, env=env))
    for _ in range(20):
        o, d = g.uniform(-3, 3, 3), g.normal(size=3)
        np.testing.assert_allclose(O.env(osc, o, d), 10.0 * d / np.linalg.norm(d), atol=1e-12)


def test_camera_axes_opencv():
    """R19: pinhole with OpenCV axes (+x right, +y down, +z forward) and +0.5 pixel centres.
    A camera at the origin looking down +z (identity rotation) images the world point
    (0.5, -0.25, 2) at column cx + fx*0.25 + ... (right of centre) and row above centre;
    checked on the rays themselves and by rendering a small off-centre triangle."""
    W, H, f = 40, 30, 30.0
    K = np.array([[f, f, 19.5, 14.5]], np.float32)
    c2w = np.zeros((1, 3, 4), np.float32)
    c2w[0, :, :3] = np.eye(3)
    cams = S.Cameras(W, H, K, c2w)
    V = np.array([[0.45, -0.3, 2.0], [0.55, -0.3, 2.0], [0.5, -0.2, 2.0]], np.float32)
    F = np.array([[0, 2, 1]], np.int32)
    osc = O.OracleScene(T.scene(V, F, cams, env=T.lobe_env(), D=0, cap=S.CAP_ENV))
    rays = O.camera_rays(osc, [0, W - 1, (H - 1) * W])
    assert rays[0, 3] < 0 and rays[0, 4] < 0                     # top-left: -x, -y (up)
    assert rays[1, 3] > 0 and rays[2, 4] > 0                     # top-right +x, bottom-left +y
    # pixel centre (x + 0.5): pixel (19, 14) looks at ((19.5 - 19.5)/f, 0, 1) = +z exactly
    r = O.camera_rays(osc, [14 * W + 19])
    np.testing.assert_allclose(r[0, 3:], [0, 0, 1], atol=1e-15)
    # the triangle around (0.5, -0.25, 2) projects to column 19.5 + 30*0.25 = 27, row 14.5 - 30*0.125 = 10.75
    hit = O.render(osc, np.arange(W * H))["sig_topo"] != O.render(osc, [14 * W + 19])["sig_topo"][0]
    ys, xs = np.divmod(np.flatnonzero(hit), W)
    assert len(xs) > 0 and abs(xs.mean() + 0.5 - 27.0) < 1.0 and abs(ys.mean() + 0.5 - 10.75) < 1.0

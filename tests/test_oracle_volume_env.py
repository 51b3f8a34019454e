"""Pins of the oracle's volumetric environment (NEXT-3; P:91 MERF grid + triplanes, P:155 /
P:161 "mixed with the environmental radiance prior to the intersection point"; reading R30):

(i)   zero density: the volume env IS the shell env of R14 (identical radiance);
(ii)  constant density sigma and a linear colour field c(p) = C p along a ray that escapes:
      the emission-absorption integral has the closed form
        L = C o (1 - e^{-s l}) + C dh [(1 - e^{-s l})/s - l e^{-s l}] + e^{-s l} C p_s,
      which the midpoint quadrature must reach within its O(Delta^2) error (1e-6 at M = 4000,
      1e-3 at M = 32), and the transmittance part is exact at any M;
(iii) the reverse mode: FD and dot tests in test_oracle_gradients.py (ico1_volenv*).
"""
import dataclasses
import math

import numpy as np

import oracle as O
from paper_2603_00413_b200 import scenes as S
from tests import _scenes as T


def test_zero_density_is_the_shell_env():
    V, F = S.icosphere(1)
    cams = T.one_view(16, 16, (0.4, -0.3, 3.0), fov_deg=60)
    vol = T.small_volume_env(density=0.0)
    vol.voxel[..., 3] = 0.0
    vol.planes[..., 3] = 0.0
    shell = dataclasses.replace(vol, kind=S.ENV_GRID)
    a = O.render(O.OracleScene(T.scene(V, F, cams, env=vol, D=3)), np.arange(256))["rgb"]
    b = O.render(O.OracleScene(T.scene(V, F, cams, env=shell, D=3)), np.arange(256))["rgb"]
    np.testing.assert_array_equal(a, b)


def _linear_volume_env(sigma, M, radius=10.0):
    env = T.linear_grid_env(radius=radius, coeff=((0.05, 0.0, 0.02), (0.0, 0.04, 0.0), (0.01, 0.01, 0.03)))
    env.voxel[..., 3] = sigma
    return dataclasses.replace(env, kind=S.ENV_VOLUME, n_samples=M)


def test_constant_density_linear_colour_closed_form():
    C = np.array([[0.05, 0.0, 0.02], [0.0, 0.04, 0.0], [0.01, 0.01, 0.03]])
    sg, R = 0.3, 10.0
    V, F = S.icosphere(0)
    V = V * 0.1 + np.array([0.0, 0.0, -5.0], np.float32)          # a small mesh off the rays' paths
    g = np.random.default_rng(4)
    o = g.uniform(-1, 1, (6, 3))
    d = g.normal(size=(6, 3))
    d[:, 2] = np.abs(d[:, 2])                                       # away from the mesh
    dh = d / np.linalg.norm(d, axis=1, keepdims=True)
    rays = np.concatenate([o, d], 1)
    for M, tol in ((4000, 1e-6), (32, 1e-3)):
        sc = T.scene(V, F, T.one_view(2, 2, (0, 0, 3)), env=_linear_volume_env(sg, M, R), D=1)
        L = O.render(O.OracleScene(sc), rays=rays)["rgb"]
        for i in range(len(o)):
            b = o[i] @ dh[i]
            ts = -b + math.sqrt(b * b - o[i] @ o[i] + R * R)
            ps = o[i] + ts * dh[i]
            e = math.exp(-sg * ts)
            exact = C @ o[i] * (1 - e) + C @ dh[i] * ((1 - e) / sg - ts * e) + e * (C @ ps)
            np.testing.assert_allclose(L[i], exact, rtol=tol, atol=tol * 1e-2)

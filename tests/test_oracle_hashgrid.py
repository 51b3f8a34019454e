"""Pins of the oracle's hash-grid absorption texture (NEXT-2; "differentiable 3D
texture" with the iNGP citation; reading R29 in DESIGN.md):

(i)   the spatial hash: a table with one non-zero entry lights up exactly the cell corner
      that iNGP's hash (x * 1) ^ (y * 2654435761) ^ (z * 805459861) mod T sends there
      (the hash is recomputed here in plain Python integers);
(ii)  special case: one dense level (T >= (N+1)^3) IS the vertex-centred R^3 grid of R11,
      so it must reproduce the grid oracle's transmittance;
(iii) linearity over levels: the optical depth of tables A + B is the sum of A's and B's.
The reverse mode is pinned by FD and the dot test in test_oracle_gradients.py (ico0_hashgrid).
"""
import dataclasses
import math

import numpy as np

import oracle as O
from paper_2603_00413_b200 import scenes as S
from tests import _scenes as T

P1, P2, P3 = 1, 2654435761, 805459861


def ingp_hash(x, y, z, T_):
    return ((x * P1) ^ (y * P2) ^ (z * P3)) % (1 << 32) % T_


def optical_depth(sc, o, x):
    osc = O.OracleScene(sc)
    tau = np.zeros(3)
    a0, a1 = np.ascontiguousarray(o, np.float64), np.ascontiguousarray(x, np.float64)   # keep alive for the call
    O.lib().dto_transmittance(osc.ref, O._p(a0), O._p(a1), O._p(tau))
    return -np.log(tau)


def base_scene(ab):
    V, F = S.icosphere(0)
    return T.scene(V, F, T.one_view(4, 4, (0, 0, 3)), absorption=ab)


def test_hash_function_selects_the_ingp_entry():
    N, log2T = 40, 10                       # (N+1)^3 = 68921 > 1024: hashed level
    Tn = 1 << log2T
    lo, hi = np.zeros(3, np.float32), np.full(3, float(N), np.float32)
    checked = 0
    for (x, y, z) in [(3, 5, 7), (0, 0, 0), (39, 1, 22), (17, 33, 2)]:
        e = ingp_hash(x, y, z, Tn)
        # the other 7 corners of the cell must not collide into e (else the pin is ambiguous)
        others = {ingp_hash(x + dx, y + dy, z + dz, Tn) for dx in (0, 1) for dy in (0, 1) for dz in (0, 1)} - {e}
        if e in others or len(others) < 7:
            continue
        tab = np.zeros((1, Tn, 3), np.float32)
        tab[0, e] = (1.0, 2.0, 4.0)
        ab = S.Absorption(S.ABS_HASH, tab, lo, hi, 1, np.array([N], np.int32))
        p = np.array([x + 0.25, y + 0.25, z + 0.25])
        d = np.array([1e-3, 0, 0])          # one midpoint sample at p: depth = mu(p) * |d|
        mu = optical_depth(base_scene(ab), p - d / 2, p + d / 2) / 1e-3
        np.testing.assert_allclose(mu, np.array([1.0, 2.0, 4.0]) * 0.75 ** 3, rtol=1e-9)
        checked += 1
    assert checked >= 3


def test_one_dense_level_is_the_vertex_grid():
    V, _ = S.icosphere(0)
    grid = T.small_sigma_grid(V, 6)
    R = grid.sigma.shape[0]
    tab = np.zeros((1, 256, 3), np.float32)             # (R-1+1)^3 = 216 <= 256: dense
    tab[0, :R ** 3] = grid.sigma.reshape(-1, 3)          # dense index x + R (y + R z) = [z][y][x]
    hashed = S.Absorption(S.ABS_HASH, tab, grid.box_lo, grid.box_hi, grid.n_samples, np.array([R - 1], np.int32))
    g = np.random.default_rng(0)
    for _ in range(20):
        o, x = g.uniform(grid.box_lo - 0.1, grid.box_hi + 0.1, (2, 3))
        a = optical_depth(base_scene(grid), o, x)
        b = optical_depth(base_scene(hashed), o, x)
        np.testing.assert_allclose(b, a, rtol=1e-12, atol=1e-14)


def test_levels_add():
    V, _ = S.icosphere(0)
    ab = T.small_hash_grid(V, levels=3, log2_size=6)
    A = dataclasses.replace(ab, sigma=ab.sigma * np.array([1, 0, 0], np.float32)[:, None, None])
    B = dataclasses.replace(ab, sigma=ab.sigma * np.array([0, 1, 1], np.float32)[:, None, None])
    g = np.random.default_rng(1)
    for _ in range(10):
        o, x = g.uniform(ab.box_lo, ab.box_hi, (2, 3))
        ab_ = optical_depth(base_scene(ab), o, x)
        a_ = optical_depth(base_scene(A), o, x)
        b_ = optical_depth(base_scene(B), o, x)
        np.testing.assert_allclose(ab_, a_ + b_, rtol=1e-11)
        assert np.all(a_ > 0) and np.all(b_ > 0)


def test_level_resolutions_geometric():
    r = S.hash_level_res(16, 16, 512)
    assert r[0] == 16 and r[-1] == 512 and np.all(np.diff(r) > 0)
    b = math.exp((math.log(512) - math.log(16)) / 15)
    assert all(r[l] == math.floor(16 * b ** l + 1e-9) for l in range(16))

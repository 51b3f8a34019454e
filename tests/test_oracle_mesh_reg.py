"""Pins of the mesh-regulariser oracle (NEXT-4; R31): closed forms on the regular
icosahedron (every vertex normal radial, every neighbour ring at cos = 1/sqrt 5), a flat
triangulated patch (all normals equal: L_edge = 0), translation/scale invariances, and
central finite differences of both hand-derived gradients."""
import math

import numpy as np

from oracle import mesh_reg as MR
from paper_2603_00413_b200 import scenes as S


def exact_icosahedron():
    """S.icosphere(0)'s faces with its (float32) vertices snapped to the exact float64
    icosahedron (0, +-1, +-phi) and cyclic permutations, normalised."""
    V32, F = S.icosphere(0)
    phi = (1 + math.sqrt(5.0)) / 2
    ex = []
    for a in (-1, 1):
        for b in (-phi, phi):
            ex += [(0, a, b), (a, b, 0), (b, 0, a)]
    ex = np.array(ex, np.float64)
    ex /= np.linalg.norm(ex, axis=1, keepdims=True)
    d = np.linalg.norm(V32[:, None, :] / np.linalg.norm(V32, axis=1)[:, None, None] - ex[None], axis=2)
    assert d.min(1).max() < 1e-6, "icosphere(0) must be a rotated copy of the standard icosahedron"
    return ex[d.argmin(1)], F


def test_icosahedron_closed_forms():
    V, F = exact_icosahedron()
    assert len(MR.edges(F)) == 30
    n = MR.vertex_normals(V, F)
    np.testing.assert_allclose(n, V, atol=1e-12)                     # radial normals
    c = 1.0 / math.sqrt(5.0)
    Le, _ = MR.loss_edge(V, F)
    assert abs(Le - (1 - c) ** 2) < 1e-12
    Ll, _ = MR.loss_lap(V, F)
    assert abs(Ll - (1 - c) ** 2) < 1e-12                             # delta = v (1 - cos theta)


def test_flat_patch_and_invariances():
    xs, ys = np.meshgrid(np.arange(5.0), np.arange(4.0))
    V = np.stack([xs.ravel(), ys.ravel(), np.zeros(20)], 1)
    F = []
    for y in range(3):
        for x in range(4):
            a = y * 5 + x
            F += [[a, a + 1, a + 6], [a, a + 6, a + 5]]
    F = np.array(F)
    Le, ge = MR.loss_edge(V, F)
    assert Le == 0.0 and np.abs(ge).max() < 1e-12
    g = np.random.default_rng(0)
    W, Fw = S.icosphere(1)
    W = W.astype(np.float64) * (1 + 0.1 * g.normal(size=W.shape))
    a, _ = MR.loss_edge(W, Fw)
    b, _ = MR.loss_edge(W * 3.0 + 1.5, Fw)                          # normals: scale/translation invariant
    assert abs(a - b) < 1e-12
    la, _ = MR.loss_lap(W, Fw)
    lb, _ = MR.loss_lap(W * 3.0 + 1.5, Fw)                          # Laplacian: quadratic in scale
    assert abs(lb - 9 * la) < 1e-10 * lb


def test_gradients_central_differences():
    g = np.random.default_rng(1)
    V, F = S.icosphere(1)
    V = V.astype(np.float64) * (1 + 0.15 * g.normal(size=V.shape))
    for fn in (MR.loss_edge, MR.loss_lap):
        L, gV = fn(V, F)
        h = 1e-6
        for c in g.choice(V.size, 20, replace=False):
            a, b = V.copy().ravel(), V.copy().ravel()
            a[c] += h
            b[c] -= h
            fd = (fn(a.reshape(V.shape), F)[0] - fn(b.reshape(V.shape), F)[0]) / (2 * h)
            assert abs(fd - gV.ravel()[c]) < 1e-6 * max(1.0, abs(fd)), (fn.__name__, c, fd, gV.ravel()[c])

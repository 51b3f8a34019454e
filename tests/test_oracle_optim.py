"""Pins of the optimisation-step oracle (oracle/optim.py): SPEC/paper worked values,
closed forms and float64 central differences of the hand-written gradients."""
import json
import os

import numpy as np

from oracle import optim as OO
from paper_2603_00413_b200 import scenes as S
from tests import _scenes as T

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "closed_forms.json")))


def test_loss_values_spec_examples():
    # S: l_color single ray (c^-c = 0.1, c = 1) -> 0.03 (golden), black target -> 0
    Lc, _, _ = OO.loss_rt([[1.1, 1.1, 1.1]], [[1.0, 1.0, 1.0]])
    assert abs(Lc - GOLD["loss_color_single_ray"]["value"]) < 1e-12
    Lc, _, g = OO.loss_rt([[0.7, 0.2, 0.9]], [[0.0, 0.0, 0.0]])
    assert Lc == 0.0 and np.abs(g).max() == 0.0
    # S: l_tone orthogonal -> 1 - var((0,1,0)) = 1 - 2/9; c^ = 2c -> -var(c); grey c^ = c -> 0
    _, Lt, _ = OO.loss_rt([[1.0, 0.0, 0.0]], [[0.0, 1.0, 0.0]])
    assert abs(Lt - (1 - 2 / 9)) < 1e-12
    c = np.array([[0.2, 0.5, 0.3]])
    _, Lt, _ = OO.loss_rt(2 * c, c)
    assert abs(Lt - (-0.0155555555555556)) < 1e-12
    _, Lt, _ = OO.loss_rt([[0.4, 0.4, 0.4]], [[0.4, 0.4, 0.4]])
    assert abs(Lt) < 1e-15


def test_loss_gradient_central_differences():
    g = np.random.default_rng(0)
    rgb = g.uniform(0.05, 2, (6, 3))
    tgt = g.uniform(0.05, 2, (6, 3))
    mask = g.uniform(0, 1, 6)
    lc, lt = 1.0, 0.37
    _, _, grad = OO.loss_rt(rgb, tgt, mask, lc, lt)
    h = 1e-6
    for i in range(6):
        for k in range(3):
            a, b = rgb.copy(), rgb.copy()
            a[i, k] += h
            b[i, k] -= h
            fa = np.dot([lc, lt], OO.loss_rt(a, tgt, mask, lc, lt)[:2])
            fb = np.dot([lc, lt], OO.loss_rt(b, tgt, mask, lc, lt)[:2])
            assert abs((fa - fb) / (2 * h) - grad[i, k]) < 1e-8


def test_sigma_regularizers_closed_forms_and_fd():
    V, _ = S.icosphere(1)
    ab = T.small_sigma_grid(V, 6)
    # constant field: smoothness 0, volume 3k^2
    ab_c = S.Absorption(S.ABS_GRID, np.full_like(ab.sigma, 0.7), ab.box_lo, ab.box_hi, 8)
    g = np.random.default_rng(1)
    pts = g.uniform(ab.box_lo, ab.box_hi, (50, 3))
    xi = g.normal(size=(50, 3)) * 0.05
    Lm, Lv, _ = OO.sigma_regularizers(ab_c, pts, xi * 0, 0.1, 0.2)
    assert abs(Lm) < 1e-12 and abs(Lv - 3 * 0.7 ** 2) < 1e-6
    # FD of the gradient on a random field (points away from cell faces are differentiable)
    sig = ab.sigma.astype(np.float64)
    ls, lv = 0.3, 0.7
    _, _, grad = OO.sigma_regularizers(S.Absorption(S.ABS_GRID, sig, ab.box_lo, ab.box_hi, 8), pts, xi, ls, lv)
    idx = np.argsort(-np.abs(grad.ravel()))[:15]
    h = 1e-7
    for j in idx:
        a, b = sig.copy().ravel(), sig.copy().ravel()
        a[j] += h
        b[j] -= h
        fa = np.dot([ls, lv], OO.sigma_regularizers(S.Absorption(S.ABS_GRID, a.reshape(sig.shape), ab.box_lo,
                                                                  ab.box_hi, 8), pts, xi, ls, lv)[:2])
        fb = np.dot([ls, lv], OO.sigma_regularizers(S.Absorption(S.ABS_GRID, b.reshape(sig.shape), ab.box_lo,
                                                                  ab.box_hi, 8), pts, xi, ls, lv)[:2])
        assert abs((fa - fb) / (2 * h) - grad.ravel()[j]) < 1e-6 * max(1, abs(grad.ravel()[j]))
    # constant sigma: L_vol = |sigma|^2, gradient 2 lambda sigma
    Lm, Lv, gc = OO.sigma_regularizers(S.const_absorption((0.2, 0.5, 1.0)), None, None, 0.1, 0.5)
    assert Lm == 0 and abs(Lv - (0.04 + 0.25 + 1.0)) < 1e-7
    np.testing.assert_allclose(gc, [0.2, 0.5, 1.0], rtol=1e-6)


def test_adam_closed_forms():
    # zero gradient and no weight decay: unchanged (S: adam_step)
    p, m, v = OO.adam(np.ones(4), np.zeros(4), np.zeros(4), np.zeros(4), 1, 0.1)
    np.testing.assert_array_equal(p, np.ones(4))
    # first step: bias correction makes the step lr * g / (|g| + eps)
    g = np.array([3.0, -0.5, 1e-3, 40.0])
    p, _, _ = OO.adam(np.zeros(4), g, np.zeros(4), np.zeros(4), 1, 0.01, eps=0.0)
    np.testing.assert_allclose(p, -0.01 * np.sign(g), rtol=1e-12)
    # f(x) = x^2 from 1, lr 0.1, 200 steps -> |x| < 1e-3 (S: adam_step convergence example)
    x, m, v = np.array([1.0]), np.zeros(1), np.zeros(1)
    for t in range(1, 201):
        x, m, v = OO.adam(x, 2 * x, m, v, t, 0.1)
    assert abs(x[0]) < 1e-3
    # AdamUniform: a uniform gradient field gives identical per-coordinate steps; one large and
    # one small gradient keep their ratio (per-coordinate Adam equalises them)
    p, _, _ = OO.adam(np.zeros(6), np.full(6, 0.3), np.zeros(6), np.zeros(1), 1, 0.01, uniform=True, eps=0.0)
    assert np.allclose(p, p[0])
    pu, _, _ = OO.adam(np.zeros(2), np.array([1.0, 0.01]), np.zeros(2), np.zeros(1), 1, 0.01, uniform=True, eps=0.0)
    pa, _, _ = OO.adam(np.zeros(2), np.array([1.0, 0.01]), np.zeros(2), np.zeros(2), 1, 0.01, eps=0.0)
    assert abs(pu[0] / pu[1] - 100.0) < 1e-9 and abs(pa[0] / pa[1] - 1.0) < 1e-12
    # clamp projection
    p, _, _ = OO.adam(np.array([1.0]), np.array([5.0]), np.zeros(1), np.zeros(1), 1, 0.5, clamp=(0.9, 3.0))
    assert p[0] == 0.9


def test_adam_converges_on_quadratic():
    x, m, v = np.array([1.0, -2.0]), np.zeros(2), np.zeros(2)
    for t in range(1, 2001):
        x, m, v = OO.adam(x, 2 * x, m, v, t, 0.01)
    assert np.abs(x).max() < 1e-3


def test_hash_regularizers_match_cpp_oracle_and_fd():
    """oracle/optim.py's numpy hash lookup (R29) against the C++ oracle's mu (an independent
    implementation: one midpoint sample of a tiny segment), and FD of its gradient."""
    import oracle as O
    V, F = S.icosphere(1)
    ab = T.small_hash_grid(V, levels=3, log2_size=6)
    sc = T.scene(V, F, T.one_view(4, 4, (0, 0, 3)), absorption=ab)
    osc = O.OracleScene(sc)
    g = np.random.default_rng(2)
    sig = ab.sigma.astype(np.float64)
    lo, hi = np.asarray(ab.box_lo, np.float64), np.asarray(ab.box_hi, np.float64)
    for p in g.uniform(lo, hi, (20, 3)):
        d = np.array([0.0, 0.0, 1e-4])
        tau = np.zeros(3)
        a0, a1 = np.ascontiguousarray(p - d / 2), np.ascontiguousarray(p + d / 2)   # keep alive
        O.lib().dto_transmittance(osc.ref, O._p(a0), O._p(a1), O._p(tau))
        mu_cpp = -np.log(tau) / 1e-4
        mu_np, _ = OO._hash_lookup(ab, sig, lo, hi, p)
        np.testing.assert_allclose(mu_np, mu_cpp, rtol=1e-9)
    pts = g.uniform(lo, hi, (30, 3))
    xi = g.normal(size=(30, 3)) * 0.05
    ls, lv = 0.3, 0.7
    _, _, grad = OO.sigma_regularizers(ab, pts, xi, ls, lv)
    import dataclasses
    h = 1e-7
    for j in np.argsort(-np.abs(grad.ravel()))[:10]:
        a, b = sig.copy().ravel(), sig.copy().ravel()
        a[j] += h
        b[j] -= h
        fa = np.dot([ls, lv], OO.sigma_regularizers(dataclasses.replace(ab, sigma=a.reshape(sig.shape)), pts, xi, ls, lv)[:2])
        fb = np.dot([ls, lv], OO.sigma_regularizers(dataclasses.replace(ab, sigma=b.reshape(sig.shape)), pts, xi, ls, lv)[:2])
        assert abs((fa - fb) / (2 * h) - grad.ravel()[j]) < 1e-6 * max(1, abs(grad.ravel()[j]))

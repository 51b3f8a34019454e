"""Pins of the oracle's hand-derived reverse mode (Appendix B of DESIGN.md).

(i)   closed-form gradients of the slab series (dR/deta = 0.128, d/dsigma, d/dthickness);
(ii)  central finite differences in float64 on tiny meshes (topology-stable coordinates);
(iii) a dot-product test against an independent forward mode (dual numbers):
      <VJP(g), t> == <g, JVP(t)> to 1e-10 relative.
A dropped term, a sign or a transposed operand in the reverse code fails (ii) and (iii).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
from paper_2603_00413_b200 import scenes as S
from tests import _scenes as T

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "closed_forms.json")))


def fd_scenes():
    out = {}
    V, F = S.icosphere(1)
    cams = T.one_view(12, 12, (0.4, -0.3, 3.0), fov_deg=50)
    out["ico1_lobes_const"] = T.scene(V, F, cams, env=T.lobe_env(kappa=2.0), D=3)
    out["ico1_gridenv"] = T.scene(V, F, cams, env=T.small_grid_env(), D=3)
    out["ico1_farfield"] = T.scene(V, F, cams, env=T.small_grid_env(far_field=1), D=2)
    V0, F0 = S.icosphere(0)
    out["ico0_sigmagrid"] = T.scene(V0, F0, cams, env=T.lobe_env(kappa=2.0),
                                    absorption=T.small_sigma_grid(V0, 5), D=3)
    out["ico1_volenv"] = T.scene(V, F, cams, env=T.small_volume_env(), D=3)
    out["ico1_volenv_capenv"] = T.scene(V, F, cams, env=T.small_volume_env(seed=8), D=2, cap=S.CAP_ENV)
    out["ico0_hashgrid"] = T.scene(V0, F0, cams, env=T.lobe_env(kappa=2.0),
                                   absorption=T.small_hash_grid(V0), D=3)
    Vt, Ft = S.tetrahedron()
    out["tet_capenv"] = T.scene(Vt, Ft, T.one_view(10, 10, (0.5, 0.7, 2.5), fov_deg=60),
                                env=T.lobe_env(kappa=2.0), D=2, cap=S.CAP_ENV)
    return out


SCENES = fd_scenes()


@pytest.mark.parametrize("name", sorted(SCENES))
def test_dot_product_reverse_vs_forward_mode(name):
    sc = SCENES[name]
    osc = O.OracleScene(sc)
    pid = np.arange(sc.n_pixels)
    g = S.upstream_grad(len(pid), 5)
    gV, gi, gs = O.backward(osc, g, pid)
    for k in range(3):
        tV = S.tangent(sc.V.shape, 9, k)
        ti = [0.7, -0.4, 0.0][k]
        ts = S.tangent(osc.sigma.shape, 9, 10 + k)
        _, j = O.jvp(osc, tV, ti, ts, pid)
        lhs = float((g * j).sum())
        rhs = float((gV * tV).sum() + gi * ti + (gs * ts).sum())
        assert abs(lhs - rhs) <= 1e-10 * max(abs(lhs), abs(rhs), 1e-3), (lhs, rhs)
    assert np.abs(gV).max() > 0 and gi != 0


def loss_and_sig(sc, pid, g, V64=None, ior=None, sigma64=None):
    osc = O.OracleScene(sc, ior=ior, V64=V64, sigma64=sigma64)
    out = O.render(osc, pid)
    return float((g * out["rgb"]).sum()), out["sig_face"]


@pytest.mark.parametrize("name", sorted(SCENES))
def test_central_finite_differences(name):
    sc = SCENES[name]
    pid = np.arange(sc.n_pixels)
    g = S.upstream_grad(len(pid), 6)
    osc = O.OracleScene(sc)
    gV, gi, gs = O.backward(osc, g, pid)
    _, sig0 = loss_and_sig(sc, pid, g)
    rng = np.random.default_rng(0)
    V64 = sc.V.astype(np.float64)
    h = 1e-6
    cand = np.flatnonzero(np.abs(gV).ravel() > 1e-3 * np.abs(gV).max())
    coords = rng.choice(cand, size=min(25, len(cand)), replace=False)
    checked = 0
    scale = np.abs(gV).max()
    for c in coords:
        Vp, Vm = V64.copy().ravel(), V64.copy().ravel()
        Vp[c] += h
        Vm[c] -= h
        lp, sp = loss_and_sig(sc, pid, g, V64=Vp)
        lm, sm = loss_and_sig(sc, pid, g, V64=Vm)
        if not (np.array_equal(sp, sig0) and np.array_equal(sm, sig0)):
            continue  # path topology changed within +-h: not differentiable there
        fd = (lp - lm) / (2 * h)
        an = gV.ravel()[c]
        assert abs(fd - an) <= 1e-6 * max(abs(an), 1e-2 * scale) + 1e-7, (c, fd, an)
        checked += 1
    assert checked >= 0.8 * len(coords)
    # ior
    lp, sp = loss_and_sig(sc, pid, g, ior=sc.ior + h)
    lm, sm = loss_and_sig(sc, pid, g, ior=sc.ior - h)
    assert np.array_equal(sp, sig0) and np.array_equal(sm, sig0)
    fd = (lp - lm) / (2 * h)
    assert abs(fd - gi) <= 1e-6 * abs(gi) + 1e-7, (fd, gi)
    # sigma
    s64 = osc.sigma.astype(np.float64).ravel()
    idx = np.argsort(-np.abs(gs.ravel()))[:6]
    for c in idx:
        sp_, sm_ = s64.copy(), s64.copy()
        sp_[c] += h
        sm_[c] -= h
        lp, _ = loss_and_sig(sc, pid, g, sigma64=sp_)
        lm, _ = loss_and_sig(sc, pid, g, sigma64=sm_)
        fd = (lp - lm) / (2 * h)
        an = gs.ravel()[c]
        assert abs(fd - an) <= 1e-6 * max(abs(an), 1e-2 * np.abs(gs).max()) + 1e-7, (c, fd, an)


def test_slab_gradients_closed_form():
    """Slab, D = 2, normal incidence: L = Lf T^2 e^{-sigma d} + Lb R with
    dR/deta = 4(eta-1)/(eta+1)^3 = 0.128 (golden), so
    dL/deta = -2 T 0.128 Lf e^{-sigma d} + 0.128 Lb;  dL/dsigma_c = -d T^2 e^{-sigma_c d} Lf_c;
    moving the bottom face down by delta lengthens the interior segment: sum of the bottom
    vertices' z-gradients = sigma T^2 e^{-sigma d} Lf (SURVEY §8c.3 'Slab gradients')."""
    V, F = S.slab(0.5, 4.0, 4)
    sig = np.array([0.25, 0.75, 1.5])     # exact in float32
    sc = T.scene(V, F, T.one_view(2, 2, (0, 0, 3)), env=T.lobe_env(), sigma=tuple(sig), D=2)
    osc = O.OracleScene(sc)
    ray = [[0.3, 0.2, 3.0, 0, 0, -1.0]]
    Lf = O.env(osc, [0, 0, 0], [0, 0, -1.0])
    Lb = O.env(osc, [0, 0, 0], [0, 0, 1.0])
    dR = GOLD["dR_deta_normal_1p5"]["value"]
    assert abs(4 * 0.5 / 2.5 ** 3 - dR) < 1e-15
    Tt, d = 0.96, 0.5
    bottom = np.abs(V[:, 2] + 0.25) < 1e-6
    for c in range(3):
        gsel = np.zeros((1, 3))
        gsel[0, c] = 1.0
        gV, gi, gs = O.backward(osc, gsel, rays=ray)
        e = math.exp(-sig[c] * d)
        assert abs(gi - (-2 * Tt * dR * Lf[c] * e + dR * Lb[c])) < 1e-12
        assert abs(gs[c] - (-d * Tt * Tt * e * Lf[c])) < 1e-12
        assert abs(gs[(c + 1) % 3]) == 0.0
        assert abs(gV[bottom, 2].sum() - sig[c] * Tt * Tt * e * Lf[c]) < 1e-12
        assert np.abs(gV[bottom, :2]).max() < 1e-12


def test_miss_and_no_absorption_gives_zero_gradients():
    """A ray that misses the object has zero parameter gradients (S: backward examples)."""
    sc = S.config_c1()
    osc = O.OracleScene(sc)
    gV, gi, gs = O.backward(osc, np.ones((1, 3)), [0])    # corner pixel misses the sphere
    assert np.abs(gV).max() == 0 and gi == 0 and np.abs(gs).max() == 0

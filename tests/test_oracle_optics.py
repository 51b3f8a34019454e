"""Pins of the oracle's interface physics against closed forms.

Nothing here compares the oracle with itself: every expected value is a printed
number (tests/golden/closed_forms.json, with citations) or an independent textbook
formula (trigonometric Fresnel forms, Snell's law in angle form, critical angle).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "closed_forms.json")))
Z = np.array([0.0, 0.0, 1.0])


def incoming(theta):
    """incoming direction d making angle theta with the normal +z (omega_i = -d)."""
    return np.array([-math.sin(theta), 0.0, -math.cos(theta)])


def trig_fresnel(ti, n1, n2):
    """Textbook trigonometric Fresnel forms (independent of P:113-122's cosine form)."""
    st = n1 / n2 * math.sin(ti)
    if st >= 1.0:
        return 1.0
    tt = math.asin(st)
    if ti == 0.0:
        return ((n1 - n2) / (n1 + n2)) ** 2
    rs = -math.sin(ti - tt) / math.sin(ti + tt)
    rp = math.tan(ti - tt) / math.tan(ti + tt)
    return 0.5 * (rs * rs + rp * rp)


def test_normal_incidence_R_is_0p04_and_reciprocal():
    g = GOLD["fresnel_normal_incidence_1_to_1p5"]["value"]
    a = O.interface(incoming(0.0), Z, 1.0, 1.5)
    b = O.interface(incoming(0.0), Z, 1.5, 1.0)
    assert abs(a["R"] - g) < 1e-15 and abs(b["R"] - g) < 1e-15
    assert abs(a["R"] + a["T"] - 1.0) < 1e-15
    np.testing.assert_allclose(a["wt"], -Z, atol=1e-15)     # straight through
    np.testing.assert_allclose(a["wr"], Z, atol=1e-15)


def test_30deg_fresnel_and_snell():
    th = math.radians(30.0)
    a = O.interface(incoming(th), Z, 1.0, 1.5)
    gold = GOLD["fresnel_30deg_1_to_1p5"]["value"]
    assert abs(a["R"] - gold) < 1e-12
    assert abs(a["R"] - trig_fresnel(th, 1.0, 1.5)) < 1e-14
    tt = math.degrees(math.acos(-a["wt"][2]))
    assert abs(tt - GOLD["snell_30deg_theta_t_deg"]["value"]) < 1e-9
    # Snell residual eta_i sin(ti) - eta_t sin(tt) and unit length
    st = math.hypot(a["wt"][0], a["wt"][1])
    assert abs(1.0 * math.sin(th) - 1.5 * st) < 1e-12
    assert abs(np.linalg.norm(a["wt"]) - 1.0) < 1e-12


def test_brewster_exact():
    th = math.atan(1.5)
    assert abs(math.degrees(th) - GOLD["brewster_angle_deg"]["value"]) < 1e-9
    a = O.interface(incoming(th), Z, 1.0, 1.5)
    assert abs(a["R"] - 25.0 / 338.0) < 1e-15
    assert abs(a["R"] - GOLD["brewster_R"]["value"]) < 1e-15


def test_tir_at_critical_angle():
    crit = math.asin(1.0 / 1.5)
    assert abs(math.degrees(crit) - GOLD["critical_angle_deg"]["value"]) < 1e-9
    below = O.interface(incoming(crit - 1e-9), Z, 1.5, 1.0)
    above = O.interface(incoming(crit + 1e-9), Z, 1.5, 1.0)
    assert not below["tir"] and above["tir"]
    assert above["R"] == 1.0 and above["T"] == 0.0
    assert O.interface(incoming(math.radians(45)), Z, 1.5, 1.0)["tir"]   # S:139 example
    assert below["R"] > 0.999   # R -> 1 continuously at the critical angle (R5)


@pytest.mark.parametrize("n1,n2", [(1.0, 1.5), (1.5, 1.0), (1.0, 1.3), (1.4, 1.0), (1.0, 2.4)])
def test_random_interfaces_energy_snell_unit_reflection(n1, n2):
    g = np.random.default_rng(0)
    for _ in range(300):
        th = g.uniform(0.0, math.pi / 2 * 0.999)
        ph = g.uniform(0, 2 * math.pi)
        d = np.array([-math.sin(th) * math.cos(ph), -math.sin(th) * math.sin(ph), -math.cos(th)])
        a = O.interface(d, Z, n1, n2)
        assert abs(a["R"] + a["T"] - 1.0) < 1e-12
        assert abs(a["R"] - trig_fresnel(th, n1, n2)) < 1e-12
        wi = -d
        # reflection: unit, same normal component, tangential part negated
        assert abs(np.linalg.norm(a["wr"]) - 1) < 1e-12
        assert abs(a["wr"] @ Z - wi @ Z) < 1e-12
        np.testing.assert_allclose(a["wr"][:2], -wi[:2], atol=1e-12)
        if not a["tir"]:
            wt = a["wt"]
            assert abs(np.linalg.norm(wt) - 1) < 1e-12
            assert abs(n1 * math.sin(th) - n2 * math.hypot(wt[0], wt[1])) < 1e-12
            # reciprocity: refracting back recovers -omega_i (SPEC optics invariants)
            b = O.interface(-wt, -Z, n2, n1)
            np.testing.assert_allclose(b["wt"], -d, atol=1e-9)


def test_equal_media_no_interface():
    a = O.interface(incoming(0.7), Z, 1.3, 1.3)
    assert abs(a["R"]) < 1e-15
    np.testing.assert_allclose(a["wt"], incoming(0.7), atol=1e-15)


def test_clamp_reading_R3():
    """Shading normal facing away (omega_i . n < 0): c_i clamps to 0, R = 1, omega_r = d."""
    d = np.array([0.6, 0.0, 0.8])          # moving along +z, n = +z: omega_i . n = -0.8
    a = O.interface(d, Z, 1.0, 1.5)
    assert a["ci"] == 0.0 and abs(a["R"] - 1.0) < 1e-15
    np.testing.assert_allclose(a["wr"], d, atol=1e-15)

"""Oracle of the optimisation step, float64 numpy.  TEST INFRASTRUCTURE ONLY.

Plain restatements, one function per formula:
  loss_rt            L_color and L_tone and d/dc^ of lambda-weighted sum
  sigma_regularizers L_mat-smooth, L_vol (mean form) and d/dsigma
  adam               torch.optim.Adam semantics (beta, weight decay), and the
                     AdamUniform variant (block-shared second moment, R26)
Shares no code with paper_2603_00413_b200/csrc.
"""
from __future__ import annotations

import numpy as np


def loss_rt(rgb, target, mask=None, lambda_color=1.0, lambda_tone=0.001, eps=1e-6):
    ch = np.asarray(rgb, np.float64)
    c = np.asarray(target, np.float64)
    n = ch.shape[0]
    m = np.ones(n) if mask is None else np.asarray(mask, np.float64)
    Lc = Lt = 0.0
    g = np.zeros_like(ch)
    for i in range(n):
        e = (ch[i] - c[i]) * c[i]
        Lc += m[i] * float(e @ e)
        gi = lambda_color * 2.0 * (ch[i] - c[i]) * c[i] * c[i]
        nh, nc = np.linalg.norm(ch[i]), np.linalg.norm(c[i])
        if nh > eps and nc > eps:
            cos = float(ch[i] @ c[i]) / (nh * nc)
            Lt += m[i] * ((1.0 - cos) ** 2 - np.var(c[i]))       # population variance
            dcos = c[i] / (nh * nc) - cos * ch[i] / (nh * nh)
            gi = gi + lambda_tone * (-2.0 * (1.0 - cos)) * dcos
        g[i] = gi * m[i] / n
    return Lc / n, Lt / n, g


def _trilinear(sig, lo, hi, p):
    """value and (node, weight) list of the R^3 vertex-centred grid at p (zero outside, R11)."""
    R = sig.shape[0]
    g = (np.asarray(p, np.float64) - lo) / (hi - lo) * (R - 1)
    if np.any(g < 0) or np.any(g > R - 1):
        return np.zeros(3), []
    i0 = np.minimum(np.floor(g).astype(int), R - 2)
    f = g - i0
    val = np.zeros(3)
    nodes = []
    for dz in (0, 1):
        for dy in (0, 1):
            for dx in (0, 1):
                w = (f[0] if dx else 1 - f[0]) * (f[1] if dy else 1 - f[1]) * (f[2] if dz else 1 - f[2])
                z, y, x = i0[2] + dz, i0[1] + dy, i0[0] + dx
                val += w * sig[z, y, x]
                nodes.append(((z, y, x), w))
    return val, nodes


def _hash_lookup(ab, sig, lo, hi, p):
    """value and (entry, weight) list of the hash texture at p (R29): the sum over levels of
    the trilinear lookup, corner (x, y, z) of level l stored at x + (N+1)(y + (N+1) z) while
    (N+1)^3 <= T, else at iNGP's hash (x * 1 ^ y * 2654435761 ^ z * 805459861) mod T."""
    u = (np.asarray(p, np.float64) - lo) / (hi - lo)
    if np.any(u < 0) or np.any(u > 1):
        return np.zeros(3), []
    T = sig.shape[1]
    val = np.zeros(3)
    ents = []
    for l, N in enumerate(ab.level_res):
        N = int(N)
        g = u * N
        i0 = np.minimum(np.floor(g).astype(int), N - 1)
        f = g - i0
        for dz in (0, 1):
            for dy in (0, 1):
                for dx in (0, 1):
                    x, y, z = int(i0[0] + dx), int(i0[1] + dy), int(i0[2] + dz)
                    if (N + 1) ** 3 <= T:
                        e = x + (N + 1) * (y + (N + 1) * z)
                    else:
                        e = ((x * 1) ^ (y * 2654435761) ^ (z * 805459861)) % (1 << 32) % T
                    w = (f[0] if dx else 1 - f[0]) * (f[1] if dy else 1 - f[1]) * (f[2] if dz else 1 - f[2])
                    val += w * sig[l, e]
                    ents.append(((l, e), w))
    return val, ents


def sigma_regularizers(absorption, points, xi, lambda_smooth, lambda_vol):
    """(L_mat, L_vol, grad) for scenes.Absorption; grad has sigma's shape."""
    sig = np.asarray(absorption.sigma, np.float64)
    if absorption.kind == 0:
        return 0.0, float(sig @ sig), 2.0 * lambda_vol * sig
    lo = np.asarray(absorption.box_lo, np.float64)
    hi = np.asarray(absorption.box_hi, np.float64)
    if absorption.kind == 2:
        lookup = lambda p: _hash_lookup(absorption, sig, lo, hi, p)
    else:
        lookup = lambda p: _trilinear(sig, lo, hi, p)
    pts = np.asarray(points, np.float64)
    n = pts.shape[0]
    grad = np.zeros_like(sig)
    Lm = Lv = 0.0
    for i in range(n):
        mv, nv = lookup(pts[i])
        mu, nu = lookup(pts[i] + np.asarray(xi[i], np.float64))
        d = mv - mu
        Lm += float(np.abs(d).sum())
        Lv += float(mv @ mv)
        s = np.sign(d) * lambda_smooth / n
        for node, w in nv:
            grad[node] += w * (s + 2.0 * lambda_vol * mv / n)
        for node, w in nu:
            grad[node] -= w * s
    return Lm / n, Lv / n, grad


def adam(p, g, m, v, step, lr, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.0, uniform=False,
         clamp=(-np.inf, np.inf)):
    """One Adam step; returns (p, m, v).  uniform: v is a scalar, v = b2 v + (1-b2) max g^2."""
    b1, b2 = betas
    p = np.asarray(p, np.float64).copy()
    g = np.asarray(g, np.float64) + weight_decay * p
    m = b1 * np.asarray(m, np.float64) + (1 - b1) * g
    if uniform:
        v = b2 * float(np.asarray(v).ravel()[0]) + (1 - b2) * float(np.max(g * g))
        v = np.array([v])
        vh = v[0] / (1 - b2 ** step)
    else:
        v = b2 * np.asarray(v, np.float64) + (1 - b2) * g * g
        vh = v / (1 - b2 ** step)
    mh = m / (1 - b1 ** step)
    p = np.clip(p - lr * mh / (np.sqrt(vh) + eps), clamp[0], clamp[1])
    return p, m, v

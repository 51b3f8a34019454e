"""Oracle of the periodic mesh regularisers, float64 numpy.  TEST INFRASTRUCTURE ONLY.

Plain restatements, one function per formula, gradients hand-derived (pinned by FD in
tests/test_oracle_mesh_reg.py):
  edges          the undirected edge set E' of the triangle mesh
  vertex_normals n_v = normalize(sum of incident unit face normals) (R6)
  loss_edge      L_edge = (1/|E'|) sum_{(i,j) in E'} (1 - n_i . n_j)^2       (P:451-455 / P:428-430)
  loss_lap       L_lap  = (1/|V|) sum_i |v_i - mean_{j in N(i)} v_j|^2      (R31: the
                 uniform graph Laplacian energy of Nicolet et al.'s uniformity term)
Shares no code with paper_2603_00413_b200/csrc.
"""
from __future__ import annotations

import numpy as np


def edges(F):
    F = np.asarray(F, np.int64)
    e = np.concatenate([F[:, [0, 1]], F[:, [1, 2]], F[:, [2, 0]]], 0)
    e.sort(axis=1)
    return np.unique(e, axis=0)


def neighbours(nv, E):
    nb = [set() for _ in range(nv)]
    for i, j in E:
        nb[i].add(int(j))
        nb[j].add(int(i))
    return [sorted(s) for s in nb]


def _face_terms(V, F):
    v0, v1, v2 = V[F[:, 0]], V[F[:, 1]], V[F[:, 2]]
    c = np.cross(v1 - v0, v2 - v0)
    lc = np.linalg.norm(c, axis=1)
    return v0, v1, v2, c, lc


def vertex_normals(V, F):
    V = np.asarray(V, np.float64)
    F = np.asarray(F, np.int64)
    _, _, _, c, lc = _face_terms(V, F)
    h = c / lc[:, None]
    s = np.zeros_like(V)
    for k in range(3):
        np.add.at(s, F[:, k], h)
    return s / np.linalg.norm(s, axis=1, keepdims=True)


def normals_vjp(V, F, gn):
    """d/dV of <gn, vertex_normals(V, F)>: n = s/|s|, s = sum h_f, h = c/|c|, c = e1 x e2."""
    V = np.asarray(V, np.float64)
    F = np.asarray(F, np.int64)
    v0, v1, v2, c, lc = _face_terms(V, F)
    h = c / lc[:, None]
    s = np.zeros_like(V)
    for k in range(3):
        np.add.at(s, F[:, k], h)
    ls = np.linalg.norm(s, axis=1)
    n = s / ls[:, None]
    gs = (gn - n * (gn * n).sum(1, keepdims=True)) / ls[:, None]
    gh = gs[F[:, 0]] + gs[F[:, 1]] + gs[F[:, 2]]
    gc = (gh - h * (gh * h).sum(1, keepdims=True)) / lc[:, None]
    e1, e2 = v1 - v0, v2 - v0
    ge1 = np.cross(e2, gc)          # d(e1 x e2)/de1 ^T gc = e2 x gc
    ge2 = np.cross(gc, e1)          # d(e1 x e2)/de2 ^T gc = gc x e1
    gV = np.zeros_like(V)
    np.add.at(gV, F[:, 1], ge1)
    np.add.at(gV, F[:, 2], ge2)
    np.add.at(gV, F[:, 0], -(ge1 + ge2))
    return gV


def loss_edge(V, F):
    """(L_edge, dL/dV)."""
    E = edges(F)
    n = vertex_normals(V, F)
    d = 1.0 - (n[E[:, 0]] * n[E[:, 1]]).sum(1)
    L = float((d * d).sum() / len(E))
    gn = np.zeros_like(n)
    w = (-2.0 * d / len(E))[:, None]
    np.add.at(gn, E[:, 0], w * n[E[:, 1]])
    np.add.at(gn, E[:, 1], w * n[E[:, 0]])
    return L, normals_vjp(V, F, gn)


def loss_lap(V, F):
    """(L_lap, dL/dV); vertices without neighbours contribute nothing."""
    V = np.asarray(V, np.float64)
    nb = neighbours(len(V), edges(F))
    delta = np.zeros_like(V)
    for i, N in enumerate(nb):
        if N:
            delta[i] = V[i] - V[N].mean(0)
    L = float((delta * delta).sum() / len(V))
    g = 2.0 * delta / len(V)
    gV = g.copy()
    for i, N in enumerate(nb):
        for j in N:
            gV[j] -= g[i] / len(N)
    return L, gV

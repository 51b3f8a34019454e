"""Seeded synthetic inputs shared by the CUDA path and the CPU oracle.

This module is the ONLY code both sides use.  It builds raw inputs (meshes,
cameras, environment fields, absorption fields, upstream gradients) and holds
none of the method's arithmetic: no intersection, no optics, no transport, no
gradients.  Every array is float32 / int32 in the layouts `include/difftrans.h`
and `oracle/oracle.h` document, so the two sides read identical bytes.

Workload shapes follow BASELINE.json `configs` and SURVEY.md §8(d):

  C1  icosphere subdiv 2 (320 tris), IOR 1.5, constant sigma, 1 view 64x64,
      D_max 2, analytic env                       (P:531 bounce caps)
  C2  cube-sphere n=65 (50,700 tris) with noise displacement + tangential
      jitter ("FlexiCubes-extracted ~50k"), 8 views 256x256, D 4, voxel+triplane env
  C3  cube-sphere n=204 (499,392 tris), 100 views 800x800 (~100 object
      views), D 4, voxel+triplane env
  C4  (2,3) torus knot 1024x128 quads + 12 unwelded brilliant-cut gems,
      64^3 sigma grid, 50 views 800x800, D 6
  C5  cube-sphere n=289 (1,002,252 tris), 200 views 1024x1024, D 4

Cameras sit uniformly on the upper hemisphere ("camera views sampled from
a uniform distribution ... on the upper hemisphere") looking at the origin.
Random numbers come from numpy PCG64 with sub-seeds seed*1000 + tag.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

ENV_ANALYTIC = 0
ENV_GRID = 1
ENV_VOLUME = 2
ABS_CONST = 0
ABS_GRID = 1
ABS_HASH = 2
CAP_ZERO = 0
CAP_ENV = 1


def rng(seed: int, tag: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed * 1000 + tag))


# --------------------------------------------------------------------------- meshes
def icosahedron():
    p = (1.0 + math.sqrt(5.0)) / 2.0
    v = np.array([[-1, p, 0], [1, p, 0], [-1, -p, 0], [1, -p, 0],
                  [0, -1, p], [0, 1, p], [0, -1, -p], [0, 1, -p],
                  [p, 0, -1], [p, 0, 1], [-p, 0, -1], [-p, 0, 1]], dtype=np.float64)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    f = np.array([[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11],
                  [1, 5, 9], [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8],
                  [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
                  [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]], dtype=np.int64)
    return v, f


def icosphere(subdiv: int, radius: float = 1.0, face_axis_to_z: bool = False):
    """Welded icosphere: F = 20*4^s, V = 10*4^s + 2, CCW = outward.

    face_axis_to_z rotates the mesh so that the centre of base face 0 lies on +z
    (and, by central symmetry, its antipodal face on -z): the axis ray through
    the centre then meets two parallel faces at their centroids.
    """
    v, f = icosahedron()
    verts = [tuple(x) for x in v]
    for _ in range(subdiv):
        cache = {}
        nf = []

        def mid(a, b):
            key = (min(a, b), max(a, b))
            if key not in cache:
                m = (np.array(verts[a]) + np.array(verts[b])) / 2.0
                m /= np.linalg.norm(m)
                verts.append(tuple(m))
                cache[key] = len(verts) - 1
            return cache[key]

        for a, b, c in f:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nf += [[a, ab, ca], [b, bc, ab], [c, ca, bc], [ab, bc, ca]]
        f = np.array(nf, dtype=np.int64)
    V = np.array(verts, dtype=np.float64)
    if face_axis_to_z:
        c = v[[0, 11, 5]].mean(axis=0)
        V = V @ rotation_to(c / np.linalg.norm(c), np.array([0.0, 0.0, 1.0])).T
    return (V * radius).astype(np.float32), f.astype(np.int32)


def rotation_to(a, b):
    """Rotation matrix taking unit a onto unit b (Rodrigues)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    v = np.cross(a, b)
    c = float(np.dot(a, b))
    if np.linalg.norm(v) < 1e-15:
        if c > 0:
            return np.eye(3)
        ax = np.array([1.0, 0, 0]) if abs(a[0]) < 0.9 else np.array([0, 1.0, 0])
        ax = ax - a * np.dot(ax, a)
        ax /= np.linalg.norm(ax)
        return 2 * np.outer(ax, ax) - np.eye(3)
    vx = np.array([[0, -v[2], v[1]], [v[2], 0, -v[0]], [-v[1], v[0], 0]])
    return np.eye(3) + vx + vx @ vx * (1.0 / (1.0 + c))


def cube_sphere(n: int, seed: int, displace: float = 0.15, jitter: float = 0.2):
    """Welded cube-sphere with 6n^2+2 vertices and 12n^2 CCW faces.

    Low-frequency radial noise (amplitude `displace`, creates concavities) plus
    tangential jitter of `jitter` x edge length mimic an iso-surface-extracted
    mesh (BASELINE.json configs[1] "FlexiCubes-extracted mesh").
    """
    faces_def = [  # (fixed axis, sign, u axis, v axis) with u x v = outward
        (0, +1, 1, 2), (0, -1, 2, 1), (1, +1, 2, 0), (1, -1, 0, 2), (2, +1, 0, 1), (2, -1, 1, 0)]
    keys_all, tris_all = [], []
    ii, jj = np.meshgrid(np.arange(n + 1), np.arange(n + 1), indexing="ij")
    base = 0
    for ax, sg, ua, va in faces_def:
        lat = np.zeros((n + 1, n + 1, 3), np.int64)
        lat[..., ax] = n if sg > 0 else 0
        lat[..., ua] = ii
        lat[..., va] = jj
        keys_all.append(lat.reshape(-1, 3))
        idx = base + (ii * (n + 1) + jj)
        a = idx[:-1, :-1].ravel()
        b = idx[1:, :-1].ravel()
        c = idx[1:, 1:].ravel()
        d = idx[:-1, 1:].ravel()
        t = np.stack([np.stack([a, b, c], 1), np.stack([a, c, d], 1)], 1).reshape(-1, 3)
        tris_all.append(t)
        base += (n + 1) ** 2
    keys = np.concatenate(keys_all)
    tris = np.concatenate(tris_all)
    code = (keys[:, 0] * (n + 1) + keys[:, 1]) * (n + 1) + keys[:, 2]
    uniq, first, inv = np.unique(code, return_index=True, return_inverse=True)
    F = inv[tris]
    cube = keys[first].astype(np.float64) / n * 2.0 - 1.0
    # equal-angle warp keeps cells near-uniform on the sphere
    cube = np.tan(cube * (math.pi / 4.0))
    P = cube / np.linalg.norm(cube, axis=1, keepdims=True)
    g = rng(seed, 11)
    if displace > 0:
        k = 6
        dirs = g.normal(size=(k, 3))
        dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
        freq = g.uniform(1.5, 4.0, size=k)
        phase = g.uniform(0, 2 * math.pi, size=k)
        amp = g.uniform(0.5, 1.0, size=k)
        noise = (np.cos(P @ dirs.T * freq + phase) * amp).sum(1) / amp.sum()
        P = P * (1.0 + displace * noise)[:, None]
    if jitter > 0:
        edge = (math.pi / 2.0) / n
        t = g.normal(size=P.shape)
        nrm = P / np.linalg.norm(P, axis=1, keepdims=True)
        t -= nrm * (t * nrm).sum(1, keepdims=True)
        t /= np.maximum(np.linalg.norm(t, axis=1, keepdims=True), 1e-12)
        mag = g.uniform(0, jitter * edge, size=(P.shape[0], 1)) * np.linalg.norm(P, axis=1, keepdims=True)
        P = P + t * mag
    return P.astype(np.float32), F.astype(np.int32)


def torus_knot(p: int = 2, q: int = 3, n_u: int = 1024, n_v: int = 128, tube: float = 0.15,
               scale: float = 0.32):
    """Welded (p,q) torus-knot tube: 2*n_u*n_v CCW (outward) triangles."""
    t = np.arange(n_u) / n_u * 2 * math.pi

    def curve(t):
        r = 2.0 + np.cos(q * t)
        return np.stack([r * np.cos(p * t), r * np.sin(p * t), -np.sin(q * t)], -1) * scale

    c = curve(t)
    h = 1e-4
    T = curve(t + h) - curve(t - h)
    T /= np.linalg.norm(T, axis=1, keepdims=True)
    A = curve(t + h) - 2 * c + curve(t - h)
    N = A - T * (A * T).sum(1, keepdims=True)
    N /= np.linalg.norm(N, axis=1, keepdims=True)
    B = np.cross(T, N)
    s = np.arange(n_v) / n_v * 2 * math.pi
    P = (c[:, None, :] + tube * (np.cos(s)[None, :, None] * N[:, None, :]
                                  + np.sin(s)[None, :, None] * B[:, None, :]))
    P = P.reshape(-1, 3)
    i, j = np.meshgrid(np.arange(n_u), np.arange(n_v), indexing="ij")
    a = i * n_v + j
    b = ((i + 1) % n_u) * n_v + j
    cc = ((i + 1) % n_u) * n_v + (j + 1) % n_v
    d = i * n_v + (j + 1) % n_v
    F = np.stack([np.stack([a, b, cc], -1), np.stack([a, cc, d], -1)], 2).reshape(-1, 3)
    # orient outward: compare the first face normal with the radial offset
    v0, v1, v2 = P[F[0, 0]], P[F[0, 1]], P[F[0, 2]]
    if np.dot(np.cross(v1 - v0, v2 - v0), v0 - c[0]) < 0:
        F = F[:, [0, 2, 1]]
    return P.astype(np.float32), F.astype(np.int32)


def gem(n_girdle: int = 16):
    """Brilliant-cut-like gem, UNWELDED facets (each triangle owns its 3 vertices),
    so vertex normals equal face normals (flat facets).  Unit girdle radius."""
    m = n_girdle
    g = [(math.cos(2 * math.pi * k / m), math.sin(2 * math.pi * k / m), 0.0) for k in range(m)]
    tr = [(0.55 * math.cos(2 * math.pi * (k + 0.5) / (m // 2)), 0.55 * math.sin(2 * math.pi * (k + 0.5) / (m // 2)), 0.35)
          for k in range(m // 2)]
    pm = [(0.5 * math.cos(2 * math.pi * k / m), 0.5 * math.sin(2 * math.pi * k / m), -0.45) for k in range(m)]
    top = (0.0, 0.0, 0.35)
    cul = (0.0, 0.0, -0.85)
    tris = []
    h = m // 2
    for k in range(h):  # table fan
        tris.append((top, tr[k], tr[(k + 1) % h]))
    for k in range(h):  # crown: table edge to girdle
        tris.append((tr[k], g[2 * k + 1], tr[(k + 1) % h]))
        tris.append((tr[k], g[2 * k], g[2 * k + 1]))
        tris.append((tr[(k + 1) % h], g[2 * k + 1], g[(2 * k + 2) % m]))
    for k in range(m):  # upper pavilion
        tris.append((g[k], pm[k], g[(k + 1) % m]))
        tris.append((g[(k + 1) % m], pm[k], pm[(k + 1) % m]))
    for k in range(m):  # lower pavilion
        tris.append((pm[k], cul, pm[(k + 1) % m]))
    V = np.array(tris, dtype=np.float64).reshape(-1, 3)
    F = np.arange(V.shape[0]).reshape(-1, 3)
    # orient outward (convex: centroid test)
    cen = V.mean(0)
    for i, (a, b, c) in enumerate(F):
        if np.dot(np.cross(V[b] - V[a], V[c] - V[a]), V[a] - cen) < 0:
            F[i] = [a, c, b]
    return V, F


def knot_and_gems(seed: int):
    """BASELINE.json configs[3]: torus knot + 12 disjoint unwelded gems (~263k tris)."""
    Vk, Fk = torus_knot()
    Vs, Fs = [Vk.astype(np.float64)], [Fk.astype(np.int64)]
    off = Vk.shape[0]
    g = rng(seed, 12)
    Vg, Fg = gem()
    for k in range(12):
        ang = 2 * math.pi * (k + 0.5) / 12
        z = 0.55 if k % 2 == 0 else -0.55
        cen = np.array([1.25 * math.cos(ang), 1.25 * math.sin(ang), z])
        R = rotation_to(np.array([0, 0, 1.0]), g.normal(size=3) / 1.0 + np.array([0, 0, 2.0]))
        R = R / np.cbrt(np.linalg.det(R))
        Vs.append((Vg @ R.T) * 0.11 + cen)
        Fs.append(Fg + off)
        off += Vg.shape[0]
    return np.concatenate(Vs).astype(np.float32), np.concatenate(Fs).astype(np.int32)


def slab(thickness: float = 0.5, extent: float = 4.0, tess: int = 4):
    """Axis-aligned closed box [-e/2,e/2]^2 x [-d/2,d/2]; the two large faces are
    tessellated (tess x tess quads) so interior vertices carry the face normal."""
    e, d = extent / 2.0, thickness / 2.0
    Vs, Fs = [], []
    off = 0

    def quad_grid(o, u, v, nu, nv):
        nonlocal off
        pts = np.array([o + u * (i / nu) + v * (j / nv) for i in range(nu + 1) for j in range(nv + 1)])
        f = []
        for i in range(nu):
            for j in range(nv):
                a = i * (nv + 1) + j
                b = (i + 1) * (nv + 1) + j
                c = (i + 1) * (nv + 1) + j + 1
                dd = i * (nv + 1) + j + 1
                f += [[a, b, c], [a, c, dd]]
        Vs.append(pts)
        Fs.append(np.array(f) + off)
        off += pts.shape[0]

    X, Y, Z = np.eye(3)
    quad_grid(np.array([-e, -e, d]), 2 * e * X, 2 * e * Y, tess, tess)        # top  (+z)
    quad_grid(np.array([-e, -e, -d]), 2 * e * Y, 2 * e * X, tess, tess)       # bottom (-z)
    quad_grid(np.array([-e, -e, -d]), 2 * e * X, 2 * d * Z, 1, 1)             # -y
    quad_grid(np.array([e, e, -d]), -2 * e * X, 2 * d * Z, 1, 1)              # +y
    quad_grid(np.array([e, -e, -d]), 2 * e * Y, 2 * d * Z, 1, 1)              # +x
    quad_grid(np.array([-e, e, -d]), -2 * e * Y, 2 * d * Z, 1, 1)             # -x
    V = np.concatenate(Vs)
    F = np.concatenate(Fs)
    # weld duplicated points
    key = np.round(V * 1e6).astype(np.int64)
    _, first, inv = np.unique(key, axis=0, return_index=True, return_inverse=True)
    return V[first].astype(np.float32), inv.reshape(-1)[F].astype(np.int32)


def tetrahedron():
    V = np.array([[0.9, 0.1, -0.3], [-0.5, 0.8, -0.35], [-0.45, -0.75, -0.3], [0.05, -0.02, 0.85]], np.float32)
    F = np.array([[0, 2, 1], [0, 1, 3], [1, 2, 3], [2, 0, 3]], np.int32)
    return V, F


# --------------------------------------------------------------------------- cameras
def look_at(pos, target=(0.0, 0.0, 0.0), up=(0.0, 0.0, 1.0)):
    """camera-to-world 3x4, OpenCV axes: +z forward, +y down, +x right."""
    pos = np.asarray(pos, np.float64)
    f = np.asarray(target, np.float64) - pos
    f /= np.linalg.norm(f)
    up = np.asarray(up, np.float64)
    if abs(np.dot(f, up)) > 0.999:
        up = np.array([0.0, 1.0, 0.0])
    x = np.cross(f, up)
    x /= np.linalg.norm(x)
    y = np.cross(f, x)
    return np.concatenate([np.stack([x, y, f], 1), pos[:, None]], 1)


@dataclasses.dataclass
class Cameras:
    width: int
    height: int
    K: np.ndarray     # [n,4] fx, fy, cx, cy (float32)
    c2w: np.ndarray   # [n,3,4] row-major (float32)

    @property
    def n_views(self):
        return self.K.shape[0]

    @property
    def n_pixels(self):
        return self.n_views * self.width * self.height


def hemisphere_cameras(n: int, W: int, H: int, dist: float, bound_radius: float, seed: int,
                       fill: float = 0.7) -> Cameras:
    g = rng(seed, 21)
    z = g.uniform(0.05, 0.95, size=n)
    phi = g.uniform(0, 2 * math.pi, size=n)
    s = np.sqrt(1 - z * z)
    pos = np.stack([s * np.cos(phi), s * np.sin(phi), z], 1) * dist
    half = math.asin(min(bound_radius / dist, 0.999))
    fx = (fill * W / 2.0) / math.tan(half)
    K = np.tile(np.array([[fx, fx, W / 2.0 - 0.5, H / 2.0 - 0.5]]), (n, 1))
    c2w = np.stack([look_at(p) for p in pos])
    return Cameras(W, H, K.astype(np.float32), c2w.astype(np.float32))


# --------------------------------------------------------------------------- fields
@dataclasses.dataclass
class Env:
    kind: int
    ambient: np.ndarray = None      # [3]
    lobes: np.ndarray = None        # [n,7]: mu(3), kappa, w(3)
    voxel: np.ndarray = None        # [vres,vres,vres,4] = [z][y][x][rgb_]
    planes: np.ndarray = None       # [3,pres,pres,4]: P_xy[y][x], P_xz[z][x], P_yz[z][y]
    radius: float = 10.0
    far_field: int = 0
    n_samples: int = 32             # ENV_VOLUME: midpoint samples per exterior segment (R30)


def analytic_env(seed: int, n_lobes: int = 8, ambient: float = 0.2) -> Env:
    g = rng(seed, 31)
    mu = g.normal(size=(n_lobes, 3))
    mu /= np.linalg.norm(mu, axis=1, keepdims=True)
    kappa = g.uniform(4, 40, size=(n_lobes, 1))
    w = g.uniform(0.5, 3.0, size=(n_lobes, 3))
    lobes = np.concatenate([mu, kappa, w], 1).astype(np.float32)
    return Env(ENV_ANALYTIC, ambient=np.full(3, ambient, np.float32), lobes=lobes)


def _smooth_field(g, coords, n_waves, lo, hi, scale):
    """sum of random low-frequency cosines over coords [...,k], mapped to [lo,hi] per channel."""
    k = coords.shape[-1]
    out = np.zeros(coords.shape[:-1] + (3,), np.float64)
    for c in range(3):
        acc = np.zeros(coords.shape[:-1])
        for _ in range(n_waves):
            w = g.normal(size=k) * scale
            acc += np.cos(coords @ w + g.uniform(0, 2 * math.pi)) * g.uniform(0.3, 1.0)
        acc = (acc - acc.min()) / max(acc.max() - acc.min(), 1e-12)
        out[..., c] = lo + (hi - lo) * acc
    return out


def volume_env(seed: int, vres: int, pres: int, radius: float = 10.0, density: float = 0.12,
               n_samples: int = 32) -> Env:
    """Volumetric env (P:91 MERF coarse grid + fine triplanes; R30): grid_env's colour
    textures plus a density channel (w): a smooth voxel field in [0, density] and plane
    fields in [0, density / 4] (per unit length), so a camera-to-object segment loses a few
    percent and an escaping ray tens of percent before the shell."""
    env = grid_env(seed, vres, pres, radius, 0)
    g = rng(seed, 33)
    ax = np.linspace(-1.0, 1.0, vres)
    zz, yy, xx = np.meshgrid(ax, ax, ax, indexing="ij")
    env.voxel[..., 3] = _smooth_field(g, np.stack([xx, yy, zz], -1), 4, 0.0, density, 3.0)[..., 0]
    ap = np.linspace(-1.0, 1.0, pres)
    bb, aa = np.meshgrid(ap, ap, indexing="ij")
    for i in range(3):
        env.planes[i, ..., 3] = _smooth_field(g, np.stack([aa, bb], -1), 6, 0.0, density / 4, 8.0)[..., 0]
    env.kind = ENV_VOLUME
    env.n_samples = n_samples
    return env


def grid_env(seed: int, vres: int, pres: int, radius: float = 10.0, far_field: int = 0) -> Env:
    """Frozen voxel + triplane env field: HDR-ish positive texels."""
    g = rng(seed, 32)
    ax = np.linspace(-1.0, 1.0, vres)
    zz, yy, xx = np.meshgrid(ax, ax, ax, indexing="ij")
    vox = _smooth_field(g, np.stack([xx, yy, zz], -1), 4, 0.05, 2.5, 3.0)
    voxel = np.zeros((vres, vres, vres, 4), np.float32)
    voxel[..., :3] = vox
    ap = np.linspace(-1.0, 1.0, pres)
    bb, aa = np.meshgrid(ap, ap, indexing="ij")    # row = second coord, col = first
    planes = np.zeros((3, pres, pres, 4), np.float32)
    for i in range(3):
        planes[i, ..., :3] = _smooth_field(g, np.stack([aa, bb], -1), 6, 0.0, 0.8, 8.0)
    return Env(ENV_GRID, voxel=voxel, planes=planes, radius=float(radius), far_field=int(far_field))


def constant_env(value=(1.0, 1.0, 1.0)) -> Env:
    """Analytic env with no lobes: L(d) = ambient for every direction."""
    return Env(ENV_ANALYTIC, ambient=np.asarray(value, np.float32), lobes=np.zeros((0, 7), np.float32))


@dataclasses.dataclass
class Absorption:
    kind: int
    sigma: np.ndarray                # [3], [R,R,R,3] = [z][y][x][c], or hash tables [L,T,3]
    box_lo: np.ndarray = None
    box_hi: np.ndarray = None
    n_samples: int = 64
    level_res: np.ndarray = None     # hash: int32 [L] cells per axis of each level (N_l)

    @property
    def res(self):
        if self.kind == ABS_CONST:
            return 0
        return self.sigma.shape[1] if self.kind == ABS_HASH else self.sigma.shape[0]

    @property
    def levels(self):
        return 0 if self.level_res is None else len(self.level_res)


def const_absorption(sigma=(0.2, 0.5, 1.0)) -> Absorption:
    return Absorption(ABS_CONST, np.asarray(sigma, np.float32))


def grid_absorption(V: np.ndarray, res: int, seed: int, n_samples: int = 64, vmax: float = 3.0) -> Absorption:
    """Two-tone smooth absorption field over the object box + 5%."""
    lo = V.min(0).astype(np.float64)
    hi = V.max(0).astype(np.float64)
    pad = 0.05 * (hi - lo)
    lo, hi = lo - pad, hi + pad
    g = rng(seed, 41)
    ax = [np.linspace(lo[i], hi[i], res) for i in range(3)]
    zz, yy, xx = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
    zmid = 0.5 * (lo[2] + hi[2])
    s = 1.0 / (1.0 + np.exp(-6.0 * (zz - zmid) / (hi[2] - lo[2])))
    top = g.uniform(0.2, vmax, 3)
    bot = g.uniform(0.0, vmax * 0.5, 3)
    ripple = 0.15 * np.cos(3.0 * xx + 2.0 * yy)
    sig = s[..., None] * top + (1 - s[..., None]) * bot
    sig = np.clip(sig * (1.0 + ripple[..., None]), 0.0, vmax)
    return Absorption(ABS_GRID, sig.astype(np.float32), lo.astype(np.float32), hi.astype(np.float32), n_samples)


def hash_level_res(levels: int, base: int, top: int) -> np.ndarray:
    """N_l = floor(N_min b^l), b = exp((ln N_max - ln N_min) / (L - 1)) (iNGP's geometric
    progression of grid resolutions; R29).  Integers, computed once here."""
    if levels == 1:
        return np.array([base], np.int32)
    b = np.exp((np.log(top) - np.log(base)) / (levels - 1))
    return np.floor(base * b ** np.arange(levels) + 1e-9).astype(np.int32)


def hash_absorption(V: np.ndarray, seed: int, levels: int = 16, log2_size: int = 19, base: int = 16, top: int = 512,
                    n_samples: int = 64, vmax: float = 3.0, detail: float = 0.05) -> Absorption:
    """Multiresolution hash-grid absorption (the paper's iNGP "3D texture"; R29) over
    the object box + 5%: level 0 (dense) holds the two-tone field of grid_absorption at its
    (N_0 + 1)^3 vertices, every finer level small non-negative noise U[0, detail vmax / L]
    (all entries >= 0, so mu >= 0).  Tables [L][T][3], T = 2^log2_size."""
    res = hash_level_res(levels, base, top)
    T = 1 << log2_size
    coarse = grid_absorption(V, int(res[0]) + 1, seed, n_samples, vmax)
    g = rng(seed, 43)
    tab = g.uniform(0.0, detail * vmax / levels, (levels, T, 3)).astype(np.float32)
    n0 = (int(res[0]) + 1) ** 3
    assert n0 <= T, "level 0 must be dense"
    tab[0, :n0] = coarse.sigma.reshape(-1, 3)
    tab[0, n0:] = 0.0
    return Absorption(ABS_HASH, tab, coarse.box_lo, coarse.box_hi, n_samples, res)


# --------------------------------------------------------------------------- scene
@dataclasses.dataclass
class Scene:
    name: str
    V: np.ndarray
    F: np.ndarray
    ior: float
    absorption: Absorption
    env: Env
    cams: Cameras
    max_depth: int
    cap_policy: int = CAP_ZERO
    t_eps: float = 1e-4

    @property
    def n_pixels(self):
        return self.cams.n_pixels


def config_c1(seed: int = 1) -> Scene:
    V, F = icosphere(2, 1.0, face_axis_to_z=True)
    W = H = 64
    fx = (W / 2.0) / math.tan(math.radians(22.5))
    K = np.array([[fx, fx, 31.5, 31.5]], np.float32)
    c2w = look_at((0.0, 0.0, 3.0), up=(0.0, 1.0, 0.0))[None].astype(np.float32)
    return Scene("C1", V, F, 1.5, const_absorption(), analytic_env(seed), Cameras(W, H, K, c2w), 2)


def config_c2(seed: int = 2, n_views: int = 8, res: int = 256, vres: int = 64, pres: int = 512) -> Scene:
    V, F = cube_sphere(65, seed)
    r = float(np.linalg.norm(V, axis=1).max())
    cams = hemisphere_cameras(n_views, res, res, 3.0 * r, r, seed)
    return Scene("C2", V, F, 1.5, const_absorption(), grid_env(seed, vres, pres), cams, 4)


def config_c3(seed: int = 3, n_views: int = 100, res: int = 800, vres: int = 128, pres: int = 1024) -> Scene:
    V, F = cube_sphere(204, seed)
    r = float(np.linalg.norm(V, axis=1).max())
    cams = hemisphere_cameras(n_views, res, res, 3.0 * r, r, seed)
    return Scene("C3", V, F, 1.5, const_absorption(), grid_env(seed, vres, pres), cams, 4)


def config_c3r(seed: int = 3, n_views: int = 100, res: int = 800, vres: int = 128, pres: int = 1024,
               env_seed: int = 1003) -> Scene:
    """NEXT-3 inference workload (relighting / novel views): C3's mesh and
    cameras, D_max = 8, and the environment swapped for another (seeded) one."""
    V, F = cube_sphere(204, seed)
    r = float(np.linalg.norm(V, axis=1).max())
    cams = hemisphere_cameras(n_views, res, res, 3.0 * r, r, seed)
    return Scene("C3R", V, F, 1.5, const_absorption(), grid_env(env_seed, vres, pres), cams, 8)


def config_c3v(seed: int = 3, n_views: int = 100, res: int = 800, vres: int = 128, pres: int = 1024,
               env_samples: int = 32) -> Scene:
    """NEXT-3 volumetric-env workload: C3's mesh and cameras with the MERF-style env volume
    rendered along every exterior segment (R30)."""
    V, F = cube_sphere(204, seed)
    r = float(np.linalg.norm(V, axis=1).max())
    cams = hemisphere_cameras(n_views, res, res, 3.0 * r, r, seed)
    env = volume_env(seed, vres, pres, n_samples=env_samples)
    return Scene("C3V", V, F, 1.5, const_absorption(), env, cams, 4)


def config_c4(seed: int = 4, n_views: int = 50, res: int = 800, vres: int = 128, pres: int = 1024,
              sigma_res: int = 64) -> Scene:
    V, F = knot_and_gems(seed)
    r = float(np.linalg.norm(V, axis=1).max())
    cams = hemisphere_cameras(n_views, res, res, 3.0 * r, r, seed)
    return Scene("C4", V, F, 1.5, grid_absorption(V, sigma_res, seed), grid_env(seed, vres, pres), cams, 6)


def config_c4h(seed: int = 4, n_views: int = 8, res: int = 800, vres: int = 128, pres: int = 1024,
               levels: int = 16, log2_size: int = 19) -> Scene:
    """NEXT-2 workload: C4's geometry with the paper's hash-grid absorption texture (R29),
    8 views (each interior sample reads 16 levels x 8 corners)."""
    V, F = knot_and_gems(seed)
    r = float(np.linalg.norm(V, axis=1).max())
    cams = hemisphere_cameras(n_views, res, res, 3.0 * r, r, seed)
    return Scene("C4H", V, F, 1.5, hash_absorption(V, seed, levels, log2_size), grid_env(seed, vres, pres), cams, 6)


def config_c5(seed: int = 5, n_views: int = 200, res: int = 1024, vres: int = 128, pres: int = 1024) -> Scene:
    V, F = cube_sphere(289, seed)
    r = float(np.linalg.norm(V, axis=1).max())
    cams = hemisphere_cameras(n_views, res, res, 3.0 * r, r, seed)
    return Scene("C5", V, F, 1.5, const_absorption(), grid_env(seed, vres, pres), cams, 4)


CONFIGS = {"C1": config_c1, "C2": config_c2, "C3": config_c3, "C3R": config_c3r, "C3V": config_c3v, "C4": config_c4,
           "C4H": config_c4h,
           "C5": config_c5}


# --------------------------------------------------------------------------- sampling helpers
def central_pixels(cams: Cameras, n: int, seed: int, frac: float = 0.6) -> np.ndarray:
    """Seeded pixel ids (view*H*W + y*W + x) drawn inside a centred disc of radius
    frac*W/2 in each view, i.e. mostly object-covering pixels.  Sorted, unique."""
    g = rng(seed, 51)
    out = set()
    W, H = cams.width, cams.height
    while len(out) < n:
        m = 2 * (n - len(out)) + 8
        v = g.integers(0, cams.n_views, m)
        a = g.uniform(0, 2 * math.pi, m)
        rr = np.sqrt(g.uniform(0, 1, m)) * frac * W / 2.0
        x = np.clip(np.floor(W / 2.0 + rr * np.cos(a)), 0, W - 1).astype(np.int64)
        y = np.clip(np.floor(H / 2.0 + rr * np.sin(a)), 0, H - 1).astype(np.int64)
        for pid in (v * H * W + y * W + x):
            if len(out) < n:
                out.add(int(pid))
    return np.array(sorted(out), np.int64)


def upstream_grad(n_rays: int, seed: int) -> np.ndarray:
    """Seeded dL/d(rgb) ~ U[-1,1]^3."""
    return rng(seed, 61).uniform(-1.0, 1.0, size=(n_rays, 3)).astype(np.float32)


def tangent(shape, seed: int, tag: int) -> np.ndarray:
    return rng(seed, 70 + tag).uniform(-1.0, 1.0, size=shape)

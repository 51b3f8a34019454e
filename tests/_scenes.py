"""Small hand-built scenes for the pins (inputs only; no method arithmetic)."""
import math

import numpy as np

from paper_2603_00413_b200 import scenes as S


def one_view(W, H, pos, fov_deg=45.0, target=(0.0, 0.0, 0.0), up=(0.0, 0.0, 1.0)):
    fx = (W / 2.0) / math.tan(math.radians(fov_deg / 2.0))
    K = np.array([[fx, fx, W / 2.0 - 0.5, H / 2.0 - 0.5]], np.float32)
    c2w = S.look_at(pos, target, up)[None].astype(np.float32)
    return S.Cameras(W, H, K, c2w)


def lobe_env(up=(0.7, 0.2, 0.5), down=(0.3, 0.9, 0.4), ambient=(0.05, 0.1, 0.15), kappa=3.0):
    """Analytic env with one lobe along +z and one along -z (radiances `up`, `down` at the poles
    plus small cross terms), smooth for finite differences."""
    lobes = np.array([[0, 0, 1, kappa, *up], [0, 0, -1, kappa, *down]], np.float32)
    return S.Env(S.ENV_ANALYTIC, ambient=np.array(ambient, np.float32), lobes=lobes)


def scene(V, F, cams, env=None, ior=1.5, sigma=(0.2, 0.5, 1.0), absorption=None, D=2, cap=S.CAP_ZERO, name="t"):
    ab = absorption if absorption is not None else S.const_absorption(sigma)
    return S.Scene(name, np.asarray(V, np.float32), np.asarray(F, np.int32), ior, ab,
                   env if env is not None else S.analytic_env(1), cams, D, cap)


def small_grid_env(seed=7, vres=8, pres=16, radius=10.0, far_field=0):
    return S.grid_env(seed, vres, pres, radius, far_field)


def linear_grid_env(vres=5, pres=4, radius=10.0, coeff=((1, 0, 0), (0, 1, 0), (0, 0, 1))):
    """voxel texels whose RGB = coeff @ p (a linear field), zero planes: the shell lookup
    then returns coeff @ p exactly (trilinear reproduces linear functions)."""
    ax = np.linspace(-radius, radius, vres)
    zz, yy, xx = np.meshgrid(ax, ax, ax, indexing="ij")
    P = np.stack([xx, yy, zz], -1)
    vox = np.zeros((vres, vres, vres, 4), np.float32)
    vox[..., :3] = P @ np.asarray(coeff, np.float64).T
    planes = np.zeros((3, pres, pres, 4), np.float32)
    return S.Env(S.ENV_GRID, voxel=vox, planes=planes, radius=radius, far_field=0)


def small_volume_env(seed=7, vres=8, pres=16, radius=6.0, density=0.15, n_samples=12):
    """Tiny volumetric env (R30): grid_env colours plus a smooth density channel."""
    return S.volume_env(seed, vres, pres, radius, density, n_samples)


def small_sigma_grid(V, res=6, seed=3):
    return S.grid_absorption(np.asarray(V), res, seed, n_samples=16)


def small_hash_grid(V, levels=3, log2_size=6, base=2, top=8, seed=3, n_samples=16):
    """Tiny hash-grid absorption (R29): level 0 dense, finer levels hashed with collisions."""
    return S.hash_absorption(np.asarray(V), seed, levels, log2_size, base, top, n_samples=n_samples, detail=0.6)

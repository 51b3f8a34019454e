"""ctypes front-end of the fp64 CPU oracle (oracle/oracle.cpp).

TEST INFRASTRUCTURE ONLY: may be imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product package.
It shares no code with paper_2603_00413_b200/csrc; both read the same raw arrays
made by paper_2603_00413_b200/scenes.py (the shared seeded input generator).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "oracle.cpp")
HDR = os.path.join(HERE, "oracle.h")
LIB = os.path.join(HERE, "liboracle.so")

FLAG_EDGE, FLAG_GRAZING, FLAG_NEARTIR = 1, 2, 4


def build(force: bool = False) -> str:
    """Compile liboracle.so with g++ (plain -O2, no fast-math) if missing or stale."""
    stale = (not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(SRC), os.path.getmtime(HDR)))
    if force or stale:
        cmd = ["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-pthread", SRC, "-o", LIB + ".tmp"]
        subprocess.run(cmd, check=True)
        os.replace(LIB + ".tmp", LIB)
    return LIB


class _Scene(C.Structure):
    _fields_ = [
        ("nv", C.c_int32), ("nf", C.c_int32), ("V", C.c_void_p), ("F", C.c_void_p),
        ("ior", C.c_double),
        ("abs_kind", C.c_int32), ("sigma", C.c_void_p), ("sigma_res", C.c_int32),
        ("sigma_lo", C.c_float * 3), ("sigma_hi", C.c_float * 3), ("n_samples", C.c_int32),
        ("env_kind", C.c_int32), ("ambient", C.c_float * 3), ("lobes", C.c_void_p), ("n_lobes", C.c_int32),
        ("voxel", C.c_void_p), ("vres", C.c_int32), ("planes", C.c_void_p), ("pres", C.c_int32),
        ("env_radius", C.c_float), ("far_field", C.c_int32),
        ("n_views", C.c_int32), ("width", C.c_int32), ("height", C.c_int32), ("K", C.c_void_p),
        ("c2w", C.c_void_p),
        ("max_depth", C.c_int32), ("cap_policy", C.c_int32), ("t_eps", C.c_double),
        ("V64", C.c_void_p), ("sigma64", C.c_void_p),
        ("hash_levels", C.c_int32), ("hash_log2_size", C.c_int32), ("hash_res", C.c_int32 * 32),
        ("env_samples", C.c_int32),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        for name in ("dto_render", "dto_backward", "dto_jvp", "dto_closest_hit", "dto_vertex_normals", "dto_camera_rays",
                     "dto_interface", "dto_env", "dto_transmittance"):
            getattr(_lib, name).restype = C.c_int
    return _lib


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


class OracleScene:
    """Holds contiguous copies of a scenes.Scene's arrays and the dto_scene struct."""

    def __init__(self, sc, ior=None, V64=None, sigma64=None):
        """V64 / sigma64: optional float64 overrides (finite-difference pins)."""
        self.V = np.ascontiguousarray(sc.V, np.float32)
        self.V64 = None if V64 is None else np.ascontiguousarray(V64, np.float64).reshape(-1, 3)
        self.sigma64 = None if sigma64 is None else np.ascontiguousarray(sigma64, np.float64)
        self.F = np.ascontiguousarray(sc.F, np.int32)
        ab = sc.absorption
        self.sigma = np.ascontiguousarray(ab.sigma, np.float32)
        env = sc.env
        self.lobes = np.ascontiguousarray(env.lobes if env.lobes is not None else np.zeros((0, 7)), np.float32)
        self.voxel = None if env.voxel is None else np.ascontiguousarray(env.voxel, np.float32)
        self.planes = None if env.planes is None else np.ascontiguousarray(env.planes, np.float32)
        self.K = np.ascontiguousarray(sc.cams.K, np.float32)
        self.c2w = np.ascontiguousarray(sc.cams.c2w, np.float32)
        s = _Scene()
        s.nv, s.nf = self.V.shape[0], self.F.shape[0]
        s.V, s.F = _p(self.V), _p(self.F)
        s.ior = float(sc.ior if ior is None else ior)
        s.abs_kind = ab.kind
        s.sigma = _p(self.sigma)
        s.sigma_res = ab.res
        if ab.box_lo is not None:
            s.sigma_lo = (C.c_float * 3)(*[float(x) for x in ab.box_lo])
            s.sigma_hi = (C.c_float * 3)(*[float(x) for x in ab.box_hi])
        s.n_samples = ab.n_samples
        if ab.kind == 2:                                   # hash grid (R29)
            T = ab.sigma.shape[1]
            assert T & (T - 1) == 0 and len(ab.level_res) <= 32
            s.hash_levels, s.hash_log2_size = len(ab.level_res), T.bit_length() - 1
            s.hash_res = (C.c_int32 * 32)(*[int(x) for x in ab.level_res])
        s.env_kind = env.kind
        amb = env.ambient if env.ambient is not None else np.zeros(3)
        s.ambient = (C.c_float * 3)(*[float(x) for x in amb])
        s.lobes, s.n_lobes = _p(self.lobes), self.lobes.shape[0]
        s.voxel = _p(self.voxel)
        s.vres = 0 if self.voxel is None else self.voxel.shape[0]
        s.planes = _p(self.planes)
        s.pres = 0 if self.planes is None else self.planes.shape[1]
        s.env_radius = env.radius
        s.far_field = env.far_field
        s.env_samples = env.n_samples
        s.n_views, s.width, s.height = self.K.shape[0], sc.cams.width, sc.cams.height
        s.K, s.c2w = _p(self.K), _p(self.c2w)
        s.max_depth, s.cap_policy, s.t_eps = sc.max_depth, sc.cap_policy, sc.t_eps
        s.V64, s.sigma64 = _p(self.V64), _p(self.sigma64)
        self.s = s

    @property
    def ref(self):
        return C.byref(self.s)


def _src(pixel_ids, rays):
    if rays is not None:
        rays = np.ascontiguousarray(rays, np.float64).reshape(-1, 6)
        return None, rays, rays.shape[0]
    pixel_ids = np.ascontiguousarray(pixel_ids, np.int64)
    return pixel_ids, None, pixel_ids.shape[0]


def render(osc: OracleScene, pixel_ids=None, rays=None, nthreads: int = 0):
    """Forward: dict(rgb, capped_w, sig_topo, sig_face, flags, segments)."""
    pid, rays, n = _src(pixel_ids, rays)
    out = dict(rgb=np.zeros((n, 3)), capped_w=np.zeros(n), sig_topo=np.zeros(n, np.uint64),
               sig_face=np.zeros(n, np.uint64), flags=np.zeros(n, np.int32), segments=np.zeros(n, np.int64))
    rc = lib().dto_render(osc.ref, _p(pid), _p(rays), C.c_int64(n), _p(out["rgb"]), _p(out["capped_w"]),
                          _p(out["sig_topo"]), _p(out["sig_face"]), _p(out["flags"]), _p(out["segments"]),
                          C.c_int(nthreads))
    assert rc == 0, rc
    return out


def backward(osc: OracleScene, grad_rgb, pixel_ids=None, rays=None, nthreads: int = 0):
    """Reverse mode: (gV [nv,3], gior float, gsigma same shape as sigma)."""
    pid, rays, n = _src(pixel_ids, rays)
    g = np.ascontiguousarray(grad_rgb, np.float64).reshape(n, 3)
    gV = np.zeros((osc.V.shape[0], 3))
    gior = np.zeros(1)
    gs = np.zeros(osc.sigma.shape)
    rc = lib().dto_backward(osc.ref, _p(pid), _p(rays), C.c_int64(n), _p(g), _p(gV), _p(gior), _p(gs),
                            C.c_int(nthreads))
    assert rc == 0, rc
    return gV, float(gior[0]), gs


def jvp(osc: OracleScene, tV, tior, tsigma, pixel_ids=None, rays=None, nthreads: int = 0):
    """Forward mode along (tV, tior, tsigma): (rgb [n,3], jvp [n,3])."""
    pid, rays, n = _src(pixel_ids, rays)
    tV = np.ascontiguousarray(tV, np.float64)
    ts = np.ascontiguousarray(tsigma, np.float64)
    rgb = np.zeros((n, 3))
    j = np.zeros((n, 3))
    rc = lib().dto_jvp(osc.ref, _p(pid), _p(rays), C.c_int64(n), _p(tV), C.c_double(tior), _p(ts), _p(rgb),
                       _p(j), C.c_int(nthreads))
    assert rc == 0, rc
    return rgb, j


def closest_hit(osc: OracleScene, rays, t_lo: float = 0.0, nthreads: int = 0):
    rays = np.ascontiguousarray(rays, np.float64).reshape(-1, 6)
    n = rays.shape[0]
    face = np.zeros(n, np.int32)
    tuv = np.zeros((n, 3))
    flags = np.zeros(n, np.int32)
    rc = lib().dto_closest_hit(osc.ref, _p(rays), C.c_int64(n), C.c_double(t_lo), _p(face), _p(tuv), _p(flags),
                               C.c_int(nthreads))
    assert rc == 0, rc
    return face, tuv, flags


def camera_rays(osc: OracleScene, pixel_ids):
    pid = np.ascontiguousarray(pixel_ids, np.int64)
    out = np.zeros((pid.shape[0], 6))
    assert lib().dto_camera_rays(osc.ref, _p(pid), C.c_int64(pid.shape[0]), _p(out)) == 0
    return out


def vertex_normals(osc: OracleScene):
    out = np.zeros((osc.V.shape[0], 3))
    assert lib().dto_vertex_normals(osc.ref, _p(out)) == 0
    return out


def interface(d, n, eta_i, eta_t):
    """dict(ci, R, T, tir, wr, wt, ct, q) for one specular interface."""
    d = np.ascontiguousarray(d, np.float64)
    n = np.ascontiguousarray(n, np.float64)
    out = np.zeros(12)
    lib().dto_interface(_p(d), _p(n), C.c_double(eta_i), C.c_double(eta_t), _p(out))
    return dict(ci=out[0], R=out[1], T=out[2], tir=bool(out[3]), wr=out[4:7].copy(), wt=out[7:10].copy(),
                ct=out[10], q=out[11])


def env(osc: OracleScene, o, d):
    o = np.ascontiguousarray(o, np.float64)
    d = np.ascontiguousarray(d, np.float64)
    out = np.zeros(3)
    lib().dto_env(osc.ref, _p(o), _p(d), _p(out))
    return out


def transmittance(osc: OracleScene, o, x):
    o = np.ascontiguousarray(o, np.float64)
    x = np.ascontiguousarray(x, np.float64)
    out = np.zeros(3)
    lib().dto_transmittance(osc.ref, _p(o), _p(x), _p(out))
    return out

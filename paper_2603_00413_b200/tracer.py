"""Python front-end of libdifftrans: the same calls as include/difftrans.h, taking torch
CUDA tensors.  Every step of the path runs in the library's kernels; this module only
marshals pointers, shapes and the current CUDA stream.  PyTorch supplies device memory,
streams and (in dist.py) process groups.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _native as N
from . import scenes as S


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _dev(a, dtype, device):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype).to(device).contiguous()


class DeviceScene:
    """Device copies of a scenes.Scene's inputs plus the ABI parameter blocks.

    The mesh (V, F), IOR and sigma are the differentiable parameters; they can be
    replaced between steps (set_vertices / ior / set_sigma).  Env and cameras are frozen."""

    def __init__(self, sc: S.Scene, device: torch.device):
        self.device = device
        self.name = sc.name
        self.V = _dev(sc.V, torch.float32, device)
        self.F = _dev(sc.F, torch.int32, device)
        self.ior = float(sc.ior)
        ab = sc.absorption
        self.sigma = _dev(ab.sigma, torch.float32, device)
        self.absorption = N.Absorption()
        self.absorption.kind = ab.kind
        self.absorption.res = ab.res
        if ab.box_lo is not None:
            self.absorption.box_lo = (C.c_float * 3)(*map(float, ab.box_lo))
            self.absorption.box_hi = (C.c_float * 3)(*map(float, ab.box_hi))
        self.absorption.n_samples = ab.n_samples
        if ab.kind == 2:                      # hash-grid texture (R29)
            T = ab.sigma.shape[1]
            self.absorption.levels = len(ab.level_res)
            self.absorption.log2_size = T.bit_length() - 1
            self.absorption.level_res = (C.c_int32 * 32)(*[int(x) for x in ab.level_res])
        env = sc.env
        self.env = N.Env()
        self.env.kind = env.kind
        self.env.ambient = (C.c_float * 3)(*map(float, env.ambient if env.ambient is not None else (0, 0, 0)))
        self.lobes = _dev(env.lobes if env.lobes is not None else np.zeros((0, 7)), torch.float32, device)
        self.voxel = None if env.voxel is None else _dev(env.voxel, torch.float32, device)
        self.planes = None if env.planes is None else _dev(env.planes, torch.float32, device)
        self.env.lobes = _ptr(self.lobes) if self.lobes.numel() else None
        self.env.n_lobes = self.lobes.shape[0]
        self.env.voxel = _ptr(self.voxel)
        self.env.vres = 0 if self.voxel is None else self.voxel.shape[0]
        self.env.planes = _ptr(self.planes)
        self.env.pres = 0 if self.planes is None else self.planes.shape[1]
        self.env.radius = float(env.radius)
        self.env.far_field = int(env.far_field)
        self.env.n_samples = int(getattr(env, "n_samples", 0))
        cams = sc.cams
        self.K = _dev(cams.K, torch.float32, device)
        self.c2w = _dev(cams.c2w, torch.float32, device)
        self.width, self.height, self.n_views = cams.width, cams.height, cams.n_views
        self.max_depth = sc.max_depth
        self.cap_policy = sc.cap_policy
        self.t_eps = sc.t_eps

    @property
    def n_pixels(self):
        return self.n_views * self.width * self.height

    def set_vertices(self, V: torch.Tensor):
        self.V = V.to(self.device, torch.float32).contiguous()

    def set_sigma(self, sigma: torch.Tensor):
        assert sigma.numel() == self.sigma.numel()
        self.sigma = sigma.to(self.device, torch.float32).contiguous()

    def cameras(self, pixel_ids=None) -> N.Cameras:
        """pixel_ids: None (every pixel), a device int64 tensor of pixel ids, or a TileShard."""
        c = N.Cameras()
        c.n_views, c.width, c.height = self.n_views, self.width, self.height
        c.K, c.c2w = _ptr(self.K), _ptr(self.c2w)
        if isinstance(pixel_ids, TileShard):
            sh = pixel_ids
            c.tile, c.shard_rank, c.shard_count = sh.tile, sh.rank, sh.count
            if sh.tile_ids is not None:
                assert sh.tile_ids.is_cuda and sh.tile_ids.dtype == torch.int32 and sh.tile_ids.is_contiguous()
                ids = sh.tile_ids
                if ids.numel() == 0:         # an empty list is not "the cyclic rule" (NULL)
                    self._empty_tiles = ids = torch.zeros(1, dtype=torch.int32, device=ids.device)
                c.tile_ids, c.n_tiles = _ptr(ids), sh.tile_ids.numel()
            c.n_rays = sh.n_rays(self.n_views, self.width, self.height)
            return c
        if pixel_ids is not None:
            assert pixel_ids.dtype == torch.int64 and pixel_ids.is_cuda and pixel_ids.is_contiguous()
            if pixel_ids.numel() == 0:       # an empty list is not "all pixels" (NULL)
                self._empty_ids = torch.zeros(1, dtype=torch.int64, device=pixel_ids.device)
                pixel_ids = self._empty_ids
                c.pixel_ids, c.n_rays = _ptr(pixel_ids), 0
                return c
            c.pixel_ids, c.n_rays = _ptr(pixel_ids), pixel_ids.numel()
        else:
            c.pixel_ids, c.n_rays = None, self.n_pixels
        return c


@dataclass
class TileShard:
    """A data-parallel shard of the image plane (dt_cameras.tile): the tile x tile
    pixel tiles listed in tile_ids (device int32, e.g. dist.lpt_assign) or, when None, every tile
    with id % count == rank; rays in tile order, 8 x 4 micro-tiles inside a tile (the order of
    dist.tiles_pixel_ids).  Width and height must be multiples of tile."""
    tile: int = 32
    rank: int = 0
    count: int = 1
    tile_ids: Optional[torch.Tensor] = None

    def n_tiles(self, n_views: int, W: int, H: int) -> int:
        if self.tile_ids is not None:
            return int(self.tile_ids.numel())
        total = n_views * (W // self.tile) * (H // self.tile)
        return max(0, (total - self.rank + self.count - 1) // self.count)

    def n_rays(self, n_views: int, W: int, H: int) -> int:
        return self.n_tiles(n_views, W, H) * self.tile * self.tile


@dataclass
class ForwardOut:
    rgb: torch.Tensor
    capped_w: Optional[torch.Tensor] = None
    sig_topo: Optional[torch.Tensor] = None
    sig_face: Optional[torch.Tensor] = None
    stats: Optional[dict] = None


class Tracer:
    """One libdifftrans context (one per GPU)."""

    def __init__(self, device=None):
        self.device = torch.device(device if device is not None else f"cuda:{torch.cuda.current_device()}")
        self._lib = N.lib()
        h = C.c_void_p()
        self._check(self._lib.dt_create(self.device.index or 0, C.byref(h)), None)
        self.h = h
        self.n_rays = 0
        self._keep = []

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self._lib.dt_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def _check(self, rc, h):
        if rc != N.DT_OK:
            msg = self._lib.dt_last_error(h).decode() if h else ""
            raise N.DiffTransError(f"{N.STATUS.get(rc, rc)}: {msg}", rc)

    # ------------------------------------------------------------------ path
    def set_bvh_quality(self, treelet_passes: int):
        """Treelet-restructuring passes of the following builds (0..4, default 2)."""
        self._check(self._lib.dt_set_bvh_quality(self.h, int(treelet_passes)), self.h)

    def build_bvh(self, V: torch.Tensor, F: torch.Tensor, stream=None):
        assert V.is_cuda and V.dtype == torch.float32 and V.is_contiguous() and V.shape[-1] == 3
        assert F.is_cuda and F.dtype == torch.int32 and F.is_contiguous() and F.shape[-1] == 3
        self._check(self._lib.dt_build_bvh(self.h, _ptr(V), V.shape[0], _ptr(F), F.shape[0], _stream(stream)), self.h)
        self._nv_built = V.shape[0]

    def trace_forward(self, ds: DeviceScene, pixel_ids: Optional[torch.Tensor] = None, ior: Optional[float] = None,
                      max_depth: Optional[int] = None, cap_policy: Optional[int] = None, want_capped=False,
                      want_sig=False, stats=False, check_finite=False, rgb: Optional[torch.Tensor] = None,
                      async_: bool = False, ior_device: Optional[torch.Tensor] = None,
                      seg_count: Optional[torch.Tensor] = None, stream=None) -> ForwardOut:
        """async_: no end-of-call synchronisation (see dt_trace_opts.async); an arena overflow
        of this call is reported by the next call as DiffTransError('DT_ERR_RETRY ...').
        ior_device: a device float32[1] the kernels read the IoR from (no host round trip when an
        on-device optimiser updates it); it must not change before the matching backward.
        seg_count: optional device int32[n_rays], accumulated with each ray's traced segments."""
        cams = ds.cameras(pixel_ids)
        n = cams.n_rays
        dev = self.device
        if rgb is None:
            rgb = torch.empty((n, 3), dtype=torch.float32, device=dev)
        capw = torch.empty(n, dtype=torch.float32, device=dev) if want_capped else None
        st = torch.empty(n, dtype=torch.int64, device=dev) if want_sig else None
        sf = torch.empty(n, dtype=torch.int64, device=dev) if want_sig else None
        opts = N.TraceOpts()
        opts.max_depth = ds.max_depth if max_depth is None else max_depth
        opts.cap_policy = ds.cap_policy if cap_policy is None else cap_policy
        opts.t_eps = ds.t_eps
        opts.check_finite = int(check_finite)
        opts.async_ = int(async_)
        if ior_device is not None:
            assert ior_device.is_cuda and ior_device.dtype == torch.float32 and ior_device.numel() >= 1
            opts.ior_device = ior_device.data_ptr()
        if seg_count is not None:
            assert seg_count.is_cuda and seg_count.dtype == torch.int32 and seg_count.numel() == n
            opts.seg_count = seg_count.data_ptr()
        ds.absorption.sigma = _ptr(ds.sigma)
        st_out = N.Stats() if stats else None
        rc = self._lib.dt_trace_forward(self.h, float(ds.ior if ior is None else ior), C.byref(ds.absorption),
                                        C.byref(ds.env), C.byref(cams), C.byref(opts), _ptr(rgb), _ptr(capw),
                                        _ptr(st), _ptr(sf), C.byref(st_out) if stats else None, _stream(stream))
        self._check(rc, self.h)
        self.n_rays = n
        self._last_depth = opts.max_depth
        self._sigma_shape = tuple(ds.sigma.shape)
        self._nv = ds.V.shape[0]
        self._keep = [ds]          # env buffers must outlive the backward
        return ForwardOut(rgb, capw, st, sf, st_out.as_dict(opts.max_depth) if stats else None)

    def trace_backward(self, grad_rgb: torch.Tensor, grad_V=None, grad_ior=None, grad_sigma=None,
                       accumulate: bool = False, stream=None):
        assert grad_rgb.is_cuda and grad_rgb.dtype == torch.float32 and grad_rgb.is_contiguous()
        assert grad_rgb.numel() == 3 * self.n_rays
        dev = self.device
        if grad_V is None:
            grad_V = torch.empty((self._nv, 3), dtype=torch.float32, device=dev)
        if grad_ior is None:
            grad_ior = torch.empty(1, dtype=torch.float32, device=dev)
        if grad_sigma is None:
            grad_sigma = torch.empty(self._sigma_shape, dtype=torch.float32, device=dev)
        rc = self._lib.dt_trace_backward(self.h, _ptr(grad_rgb), _ptr(grad_V), _ptr(grad_ior), _ptr(grad_sigma),
                                         int(accumulate), _stream(stream))
        self._check(rc, self.h)
        return grad_V, grad_ior, grad_sigma

    def loss_color(self, rgb: torch.Tensor, target: torch.Tensor, grad_rgb: Optional[torch.Tensor] = None,
                   loss: Optional[torch.Tensor] = None, stream=None):
        n = rgb.shape[0]
        if grad_rgb is None:
            grad_rgb = torch.empty_like(rgb)
        if loss is None:
            loss = torch.empty(1, dtype=torch.float32, device=rgb.device)
        self._check(self._lib.dt_loss_color(self.h, _ptr(rgb), _ptr(target), n, _ptr(grad_rgb), _ptr(loss),
                                            _stream(stream)), self.h)
        return loss, grad_rgb

    def get_stats(self) -> dict:
        st = N.Stats()
        rc = self._lib.dt_get_stats(self.h, C.byref(st))
        self._check(rc, self.h)
        return st.as_dict(self._last_depth)

    # ------------------------------------------------------------------ optimisation step (NEXT-1)
    def loss_rt(self, rgb: torch.Tensor, target: torch.Tensor, lambda_color: float = 1.0, lambda_tone: float = 0.001,
                mask: Optional[torch.Tensor] = None, grad_rgb: Optional[torch.Tensor] = None,
                loss: Optional[torch.Tensor] = None, stream=None):
        """Fused L_color + L_tone: returns (loss[2] = [L_color, L_tone], grad_rgb)."""
        n = rgb.shape[0]
        if grad_rgb is None:
            grad_rgb = torch.empty_like(rgb)
        if loss is None:
            loss = torch.empty(2, dtype=torch.float32, device=rgb.device)
        self._check(self._lib.dt_loss_rt(self.h, _ptr(rgb), _ptr(target), _ptr(mask), n, float(lambda_color),
                                         float(lambda_tone), _ptr(grad_rgb), _ptr(loss), _stream(stream)), self.h)
        return loss, grad_rgb

    def sigma_regularizers(self, ds: "DeviceScene", points: torch.Tensor, xi: torch.Tensor, grad_sigma: torch.Tensor,
                           lambda_smooth: float, lambda_vol: float, loss: Optional[torch.Tensor] = None, stream=None):
        """L_mat-smooth / L_vol; accumulates into grad_sigma."""
        if loss is None:
            loss = torch.empty(2, dtype=torch.float32, device=grad_sigma.device)
        ds.absorption.sigma = _ptr(ds.sigma)
        self._check(self._lib.dt_sigma_regularizers(self.h, C.byref(ds.absorption), _ptr(points), _ptr(xi),
                                                    points.shape[0] if points is not None else 0, float(lambda_smooth),
                                                    float(lambda_vol), _ptr(grad_sigma), _ptr(loss),
                                                    _stream(stream)), self.h)
        return loss

    def mesh_regularizers(self, lambda_edge: float, lambda_lap: float, grad_V: Optional[torch.Tensor] = None,
                          loss: Optional[torch.Tensor] = None, stream=None):
        """L_edge and L_lap of the last built mesh (NEXT-4): returns (loss[2], grad_V);
        grad_V is accumulated into (a new zero tensor if None)."""
        if grad_V is None:
            grad_V = torch.zeros((self._nv_built, 3), dtype=torch.float32, device=self.device)
        if loss is None:
            loss = torch.empty(2, dtype=torch.float32, device=self.device)
        self._check(self._lib.dt_mesh_regularizers(self.h, float(lambda_edge), float(lambda_lap), _ptr(grad_V),
                                                   _ptr(loss), _stream(stream)), self.h)
        return loss, grad_V

    def mask_loss(self, ds: DeviceScene, gt_mask: torch.Tensor, lam: float = 1.0, grad_V: Optional[torch.Tensor] = None,
                  want_mask: bool = False, stream=None):
        """L_mask of the last built mesh over ds's full images (NEXT-4, R32): returns
        (loss[1], grad_V (accumulated; new zeros if None), rendered mask or None)."""
        assert gt_mask.is_cuda and gt_mask.dtype == torch.float32 and gt_mask.is_contiguous()
        assert gt_mask.numel() == ds.n_pixels
        if grad_V is None:
            grad_V = torch.zeros((self._nv_built, 3), dtype=torch.float32, device=self.device)
        loss = torch.empty(1, dtype=torch.float32, device=self.device)
        mask = torch.empty_like(gt_mask) if want_mask else None
        cams = ds.cameras(None)
        self._check(self._lib.dt_mask_loss(self.h, C.byref(cams), _ptr(gt_mask), float(lam), _ptr(grad_V), _ptr(loss),
                                           _ptr(mask), _stream(stream)), self.h)
        self._keep_mask = (ds, cams)
        return loss, grad_V, mask

    def overflow_flag(self) -> int:
        """Device address of the int that is nonzero iff the last forward overflowed its record
        arena (dt_forward_overflow_flag): pass as adam_step(skip_if=...)."""
        return self._lib.dt_forward_overflow_flag(self.h)

    def adam_step(self, param: torch.Tensor, grad: torch.Tensor, m: torch.Tensor, v: torch.Tensor, step: int,
                  lr: float, betas=(0.9, 0.999), eps: float = 1e-8, weight_decay: float = 0.0, uniform=False,
                  clamp=(-float("inf"), float("inf")), skip_if: Optional[int] = None,
                  step_device: Optional[torch.Tensor] = None, stream=None):
        """In-place Adam / AdamUniform update of `param`.  skip_if: device int
        address (e.g. overflow_flag()); the update is skipped when it holds a nonzero value.
        step_device: device int32[1] holding t, read at run time and incremented after the update
        (CUDA-graph replays); `step` is then ignored."""
        for t in (param, grad, m, v):
            assert t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()
        cfg = N.Adam()
        cfg.lr, cfg.beta1, cfg.beta2, cfg.eps, cfg.weight_decay = lr, betas[0], betas[1], eps, weight_decay
        cfg.step, cfg.uniform = int(step), int(uniform)
        cfg.clamp_lo, cfg.clamp_hi = float(clamp[0]), float(clamp[1])
        cfg.skip_if = skip_if
        if step_device is not None:
            assert step_device.is_cuda and step_device.dtype == torch.int32
            cfg.step_device = step_device.data_ptr()
        self._check(self._lib.dt_adam_step(self.h, _ptr(param), _ptr(grad), _ptr(m), _ptr(v), param.numel(),
                                           C.byref(cfg), _stream(stream)), self.h)

    # ------------------------------------------------------------------ profiling
    def set_profiling(self, enable: bool):
        self._check(self._lib.dt_set_profiling(self.h, int(enable)), self.h)

    def profile(self, reset: bool = False) -> dict:
        p = N.Profile()
        self._check(self._lib.dt_get_profile(self.h, C.byref(p), int(reset)), self.h)
        return p.as_dict()

    # ------------------------------------------------------------------ test hooks
    def closest_hit(self, rays: torch.Tensor, t_lo: float = 0.0, brute_force: bool = False, stream=None):
        rays = rays.to(self.device, torch.float32).contiguous()
        n = rays.shape[0]
        face = torch.empty(n, dtype=torch.int32, device=self.device)
        tuv = torch.empty((n, 3), dtype=torch.float32, device=self.device)
        self._check(self._lib.dt_debug_closest_hit(self.h, _ptr(rays), n, float(t_lo), int(brute_force), _ptr(face),
                                                   _ptr(tuv), _stream(stream)), self.h)
        return face, tuv

    def bvh_check(self, stream=None):
        out = (C.c_int64 * 4)()
        self._check(self._lib.dt_debug_bvh_check(self.h, out, _stream(stream)), self.h)
        return dict(bad_boxes=out[0], leaves=out[1], distinct_faces=out[2], depth=out[3])

    def vertex_normals(self, nv: int, stream=None):
        out = torch.empty((nv, 3), dtype=torch.float32, device=self.device)
        self._check(self._lib.dt_debug_vertex_normals(self.h, _ptr(out), _stream(stream)), self.h)
        return out


class DiffTraceFunction(torch.autograd.Function):
    """autograd wrapper: rgb = trace(V, ior, sigma); backward through dt_trace_backward."""

    @staticmethod
    def forward(ctx, V, ior, sigma, tracer: Tracer, ds: DeviceScene, pixel_ids):
        ds.set_vertices(V.detach())
        ds.set_sigma(sigma.detach())
        ds.ior = float(ior.detach().item())
        tracer.build_bvh(ds.V, ds.F)
        out = tracer.trace_forward(ds, pixel_ids)
        ctx.tracer = tracer
        return out.rgb

    @staticmethod
    def backward(ctx, grad_rgb):
        gV, gi, gs = ctx.tracer.trace_backward(grad_rgb.contiguous())
        return gV, gi.reshape(()), gs, None, None, None

"""ctypes declarations of libdifftrans (include/difftrans.h).  Argument marshalling only.

The product path has no fallback: if the shared library is missing or cannot be loaded,
importing the tracer raises.  It never loads or calls anything under oracle/.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdifftrans.so")

DT_OK = 0
STATUS = {0: "DT_OK", 1: "DT_ERR_INVALID_ARG", 2: "DT_ERR_EMPTY_GEOMETRY", 3: "DT_ERR_CUDA", 4: "DT_ERR_OOM",
          5: "DT_ERR_NOT_BUILT", 6: "DT_ERR_NO_FORWARD", 7: "DT_ERR_NONFINITE", 8: "DT_ERR_STACK",
          9: "DT_ERR_RETRY"}
DT_ERR_RETRY = 9
DT_MAX_DEPTH = 15


class Absorption(C.Structure):
    _fields_ = [("kind", C.c_int32), ("sigma", C.c_void_p), ("res", C.c_int32), ("box_lo", C.c_float * 3),
                ("box_hi", C.c_float * 3), ("n_samples", C.c_int32), ("levels", C.c_int32), ("log2_size", C.c_int32),
                ("level_res", C.c_int32 * 32)]


class Env(C.Structure):
    _fields_ = [("kind", C.c_int32), ("ambient", C.c_float * 3), ("lobes", C.c_void_p), ("n_lobes", C.c_int32),
                ("voxel", C.c_void_p), ("vres", C.c_int32), ("planes", C.c_void_p), ("pres", C.c_int32),
                ("radius", C.c_float), ("far_field", C.c_int32), ("n_samples", C.c_int32)]


class Cameras(C.Structure):
    _fields_ = [("n_views", C.c_int32), ("width", C.c_int32), ("height", C.c_int32), ("K", C.c_void_p),
                ("c2w", C.c_void_p), ("pixel_ids", C.c_void_p), ("n_rays", C.c_int64), ("tile", C.c_int32),
                ("shard_rank", C.c_int32), ("shard_count", C.c_int32), ("tile_ids", C.c_void_p),
                ("n_tiles", C.c_int32)]


class TraceOpts(C.Structure):
    _fields_ = [("max_depth", C.c_int32), ("cap_policy", C.c_int32), ("t_eps", C.c_float),
                ("check_finite", C.c_int32), ("async_", C.c_int32), ("ior_device", C.c_void_p),
                ("seg_count", C.c_void_p)]


class Stats(C.Structure):
    _fields_ = [("segments_per_depth", C.c_int64 * (DT_MAX_DEPTH + 1)), ("primaries", C.c_int64),
                ("primaries_traced", C.c_int64), ("segments", C.c_int64), ("arena_capacity", C.c_int64),
                ("arena_retries", C.c_int32), ("bvh_depth", C.c_int32)]

    def as_dict(self, max_depth: int):
        return dict(segments_per_depth=[int(self.segments_per_depth[k]) for k in range(max_depth + 1)],
                    primaries=int(self.primaries), primaries_traced=int(self.primaries_traced),
                    segments=int(self.segments), arena_capacity=int(self.arena_capacity),
                    arena_retries=int(self.arena_retries))


class Adam(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("weight_decay", C.c_float), ("step", C.c_int32), ("uniform", C.c_int32), ("clamp_lo", C.c_float),
                ("clamp_hi", C.c_float), ("skip_if", C.c_void_p), ("step_device", C.c_void_p)]


PHASES = ["build", "trace0", "shade", "trace", "gather", "bwd", "normals_bwd", "loss"]


class Profile(C.Structure):
    _fields_ = [("ms", C.c_double * len(PHASES)), ("launches", C.c_int64 * len(PHASES)),
                ("kernel_launches", C.c_int64), ("node_visits", C.c_int64), ("tri_tests", C.c_int64),
                ("node_visits_primary", C.c_int64), ("tri_tests_primary", C.c_int64), ("segments", C.c_int64),
                ("walk_cells_fwd", C.c_int64), ("walk_cells_bwd", C.c_int64), ("env_samples_bwd", C.c_int64)]

    def as_dict(self):
        return dict(ms={p: float(self.ms[i]) for i, p in enumerate(PHASES)},
                    launches={p: int(self.launches[i]) for i, p in enumerate(PHASES)},
                    kernel_launches=int(self.kernel_launches), node_visits=int(self.node_visits),
                    tri_tests=int(self.tri_tests), node_visits_primary=int(self.node_visits_primary),
                    tri_tests_primary=int(self.tri_tests_primary), segments=int(self.segments),
                    walk_cells_fwd=int(self.walk_cells_fwd), walk_cells_bwd=int(self.walk_cells_bwd),
                    env_samples_bwd=int(self.env_samples_bwd))


_P = C.c_void_p
SIGNATURES = {
    "dt_set_profiling": (C.c_int, [_P, C.c_int32]),
    "dt_get_stats": (C.c_int, [_P, C.POINTER(Stats)]),
    "dt_get_profile": (C.c_int, [_P, C.POINTER(Profile), C.c_int32]),
    "dt_create": (C.c_int, [C.c_int32, C.POINTER(C.c_void_p)]),
    "dt_destroy": (None, [_P]),
    "dt_last_error": (C.c_char_p, [_P]),
    "dt_status_string": (C.c_char_p, [C.c_int]),
    "dt_build_bvh": (C.c_int, [_P, _P, C.c_int32, _P, C.c_int32, _P]),
    "dt_set_bvh_quality": (C.c_int, [_P, C.c_int32]),
    "dt_trace_forward": (C.c_int, [_P, C.c_float, C.POINTER(Absorption), C.POINTER(Env), C.POINTER(Cameras),
                                   C.POINTER(TraceOpts), _P, _P, _P, _P, C.POINTER(Stats), _P]),
    "dt_trace_backward": (C.c_int, [_P, _P, _P, _P, _P, C.c_int32, _P]),
    "dt_loss_color": (C.c_int, [_P, _P, _P, C.c_int64, _P, _P, _P]),
    "dt_loss_rt": (C.c_int, [_P, _P, _P, _P, C.c_int64, C.c_float, C.c_float, _P, _P, _P]),
    "dt_sigma_regularizers": (C.c_int, [_P, C.POINTER(Absorption), _P, _P, C.c_int64, C.c_float, C.c_float, _P, _P,
                                        _P]),
    "dt_adam_step": (C.c_int, [_P, _P, _P, _P, _P, C.c_int64, C.POINTER(Adam), _P]),
    "dt_mesh_regularizers": (C.c_int, [_P, C.c_float, C.c_float, _P, _P, _P]),
    "dt_mask_loss": (C.c_int, [_P, C.POINTER(Cameras), _P, C.c_float, _P, _P, _P, _P]),
    "dt_debug_closest_hit": (C.c_int, [_P, _P, C.c_int64, C.c_float, C.c_int32, _P, _P, _P]),
    "dt_debug_bvh_check": (C.c_int, [_P, C.POINTER(C.c_int64), _P]),
    "dt_debug_vertex_normals": (C.c_int, [_P, _P, _P]),
    "dt_forward_overflow_flag": (C.c_void_p, [_P]),
    "dt_debug_check_status": (C.c_int, [C.POINTER(C.c_int32)]),
}


def check_status():
    """Bounds-checked build (DT_CHECKED): first failed check line per translation unit
    (bvh, trace, optim, meshreg, api; 0 = none), cleared; all -1 in the product build."""
    out = (C.c_int32 * 5)()
    rc = lib().dt_debug_check_status(out)
    if rc != 0:
        raise DiffTransError(f"dt_debug_check_status failed ({rc})", rc)
    return dict(zip(["bvh", "trace", "optim", "meshreg", "api"], list(out)))

_lib = None
_lib_path = LIB_PATH


def use_library(path: str) -> None:
    """Tuning sweeps only (tools/bench_variant.py): load a variant build of libdifftrans.so
    (same ABI, other compile-time constants) instead of the in-tree one.  Must be called
    before the first lib()."""
    global _lib_path
    assert _lib is None, "libdifftrans already loaded"
    _lib_path = path


def lib():
    """Load libdifftrans.so (building it with nvcc first if it is absent)."""
    global _lib
    if _lib is None:
        path = _lib_path
        if not os.path.exists(path):
            if path != LIB_PATH:
                raise FileNotFoundError(path)
            from . import build as _build
            _build.build()
        _lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(_lib, name)
            fn.restype = res
            fn.argtypes = args
    return _lib


class DiffTransError(RuntimeError):
    """A non-DT_OK status; .status holds the dt_status code."""

    def __init__(self, msg: str, status: int = -1):
        super().__init__(msg)
        self.status = status

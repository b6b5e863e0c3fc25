"""ctypes binding of libpxg.so (include/pxg.h). Loads the in-tree library and fails loudly
when it is missing: there is no CPU fallback on the product path."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# PXG_LIBRARY: an alternative build of the same library (A/B tuning experiments only)
LIB_PATH = os.environ.get("PXG_LIBRARY") or os.path.join(HERE, "libpxg.so")


class PxgError(RuntimeError):
    """A nonzero libpxg return code (the reference would have thrown)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"pxg error {code}: {msg}")
        self.code = code


class PxgValidationError(PxgError, ValueError):
    pass


class SceneDesc(C.Structure):
    _fields_ = [
        ("n_prims", C.c_int),
        ("shape", C.POINTER(C.c_int)),
        ("material", C.POINTER(C.c_int)),
        ("a", C.POINTER(C.c_double)),
        ("b", C.POINTER(C.c_double)),
        ("c", C.POINTER(C.c_double)),
        ("radius", C.POINTER(C.c_double)),
        ("n_materials", C.c_int),
        ("materials", C.POINTER(C.c_double)),
        ("n_emitters", C.c_int),
        ("emitter_prim", C.POINTER(C.c_int)),
        ("emitter_radiance", C.POINTER(C.c_double)),
        ("cam_position", C.c_double * 3),
        ("cam_look_at", C.c_double * 3),
        ("cam_up", C.c_double * 3),
        ("fov_y", C.c_double),
        ("width", C.c_int),
        ("height", C.c_int),
        ("max_depth", C.c_int),
    ]


class Params(C.Structure):
    _fields_ = [
        ("enabled", C.c_int),
        ("pool_budget", C.c_int),
        ("recip_repeats", C.c_int),
        ("freeze_iteration", C.c_int),
        ("recursion_cap", C.c_longlong),
        ("pretrace_paths", C.c_int),
        ("light_walks", C.c_int),
        ("gate_high", C.c_double),
        ("gate_low", C.c_double),
        ("gate_threshold", C.c_double),
    ]


class Shard(C.Structure):
    _fields_ = [("row_begin", C.c_int), ("row_end", C.c_int), ("walk_begin", C.c_int), ("walk_end", C.c_int)]


_lib = None
_DP = C.POINTER(C.c_double)
_IP = C.POINTER(C.c_int)
_LP = C.POINTER(C.c_longlong)


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing; run `python -m paper_2503_23412_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    L.pxg_last_error.restype = C.c_char_p
    L.pxg_last_error.argtypes = [C.c_void_p]
    L.pxg_default_params.argtypes = [C.POINTER(Params)]
    L.pxg_device_count.restype = C.c_int
    L.pxg_create.argtypes = [C.POINTER(SceneDesc), C.POINTER(Params), C.c_uint64, C.c_int, C.POINTER(Shard),
                             C.POINTER(C.c_void_p)]
    L.pxg_destroy.argtypes = [C.c_void_p]
    L.pxg_scene_create.argtypes = [C.POINTER(SceneDesc), C.POINTER(C.c_void_p)]
    L.pxg_scene_destroy.argtypes = [C.c_void_p]
    L.pxg_scene_device_bytes.argtypes = [C.c_void_p]
    L.pxg_scene_device_bytes.restype = C.c_longlong
    L.pxg_create_from_scene.argtypes = [C.c_void_p, C.POINTER(Params), C.c_uint64, C.c_int, C.POINTER(Shard),
                                        C.POINTER(C.c_void_p)]
    L.pxg_render_pass.argtypes = [C.c_void_p]
    L.pxg_render_passes.argtypes = [C.c_void_p, C.c_int]
    L.pxg_render_pass_traced.argtypes = [C.c_void_p]
    L.pxg_synchronize.argtypes = [C.c_void_p]
    L.pxg_set_pass_limit.argtypes = [C.c_void_p, C.c_int]
    L.pxg_render_passes_async.argtypes = [C.c_void_p, C.c_int]
    L.pxg_snapshot_mean.argtypes = [C.c_void_p, C.c_int]
    L.pxg_read_snapshot.argtypes = [C.c_void_p, C.c_int, _DP, _IP]
    L.pxg_measure_traversal.argtypes = [C.c_void_p, C.c_int, _DP]
    L.pxg_read_mean.argtypes = [C.c_void_p, _DP, _IP]
    L.pxg_read_accum.argtypes = [C.c_void_p, _DP, _IP]
    L.pxg_accum_to_device.argtypes = [C.c_void_p, C.c_void_p, _IP]
    L.pxg_accum_to_device_async.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, _IP]
    L.pxg_read_diag.argtypes = [C.c_void_p, _LP, _IP, _LP]
    L.pxg_read_stats.argtypes = [C.c_void_p, _DP, _LP, _DP]
    L.pxg_dump_pass.argtypes = [C.c_void_p, _DP, _DP, _DP, _IP]
    L.pxg_dump_prims.argtypes = [C.c_void_p, _IP, _IP]
    L.pxg_dump_pool.argtypes = [C.c_void_p, C.c_int, _IP, _LP, _IP, _IP, _IP, _DP, _DP, _DP]
    L.pxg_dump_paths.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, _DP]
    L.pxg_intersect.argtypes = [C.c_void_p, C.c_int, _DP, _DP, _IP, _DP]
    L.pxg_occluded.argtypes = [C.c_void_p, C.c_int, _DP, _IP]
    L.pxg_trace_rays.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _DP, _DP, _IP, _DP]
    L.pxg_proxy_probe.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_uint64, _IP, _DP,
                                  _DP, _DP, C.c_void_p, _DP, _IP]
    L.pxg_proxy_recip.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_double, C.c_int, _DP, _LP, _IP]
    L.pxg_node_bytes.argtypes = [C.c_void_p]
    L.pxg_render_pt.argtypes = [C.c_void_p, C.c_int, C.c_uint64, C.c_int, _DP]
    L.pxg_recip_twopoint.argtypes = [C.c_int, C.c_double, C.c_longlong, C.c_uint64, _DP, _LP, _IP]
    L.pxg_rng_draws.argtypes = [C.c_uint64, C.c_uint, C.c_uint, C.c_uint64, C.c_int, C.POINTER(C.c_uint)]
    L.pxg_read_timing.argtypes = [C.c_void_p, _DP, _LP]
    L.pxg_read_recip_counts.argtypes = [C.c_void_p, _LP]
    L.pxg_sincos_2pi.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_uint), _DP, _DP]
    _lib = L
    return L


EXPORTED_SYMBOLS = [
    "pxg_default_params", "pxg_abi_version", "pxg_node_bytes", "pxg_device_count", "pxg_create", "pxg_scene_create", "pxg_scene_destroy", "pxg_scene_device_bytes", "pxg_create_from_scene", "pxg_destroy", "pxg_last_error",
    "pxg_render_pass", "pxg_render_passes", "pxg_render_pass_traced", "pxg_set_pass_limit", "pxg_render_passes_async", "pxg_snapshot_mean", "pxg_read_snapshot",
    "pxg_measure_traversal", "pxg_synchronize", "pxg_read_mean", "pxg_read_accum", "pxg_accum_to_device", "pxg_accum_to_device_async", "pxg_read_diag",
    "pxg_read_stats", "pxg_dump_pass", "pxg_dump_prims", "pxg_dump_pool", "pxg_dump_paths", "pxg_intersect", "pxg_occluded", "pxg_trace_rays", "pxg_proxy_probe", "pxg_proxy_recip",
    "pxg_render_pt", "pxg_recip_twopoint", "pxg_rng_draws", "pxg_read_timing", "pxg_read_recip_counts", "pxg_sincos_2pi",
]


def check(rc: int, ctx=None):
    if rc != 0:
        msg = lib().pxg_last_error(ctx).decode()
        if rc == -1:
            raise PxgValidationError(rc, msg)
        raise PxgError(rc, msg)

"""ctypes binding of the C ABI in include/screloc_gpu.h (libscreloc_gpu.so, sm_100a).

The library is the product: there is no CPU fallback. Loading fails loudly if the
shared object is missing, and every call that returns a non-zero status raises the
screloc exception class mapped from it (proj/include/screloc/core.hpp:24-72).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libscreloc_gpu.so")


class Intrinsics(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double)]


class Pose(C.Structure):
    _fields_ = [("R", C.c_double * 9), ("t", C.c_double * 3)]


class Frame(C.Structure):
    _fields_ = [("depth", C.c_void_p), ("rgb", C.c_void_p), ("width", C.c_int32), ("height", C.c_int32),
                ("pose_reliable", C.c_int32), ("pad", C.c_int32)]


class ForestParams(C.Structure):
    _fields_ = [("sigma", C.c_float), ("tau", C.c_float), ("max_clusters", C.c_int32),
                ("min_cluster_size", C.c_int32), ("capacity", C.c_int32)]


class RansacParams(C.Structure):
    _fields_ = [("max_gen_iters", C.c_int32), ("n_max", C.c_int32), ("n_cull", C.c_int32), ("eta", C.c_int32),
                ("pose_update", C.c_int32), ("use_cov", C.c_int32), ("min_sq_dist", C.c_double),
                ("colour_thresh", C.c_float), ("pad0", C.c_float), ("rigidity_tol", C.c_double),
                ("n_out", C.c_int32), ("pad1", C.c_int32)]


class Result(C.Structure):
    _fields_ = [("has_pose", C.c_int32), ("status", C.c_int32), ("pose", Pose), ("score", C.c_double),
                ("stage_used", C.c_int32), ("n_candidates", C.c_int32), ("stage_ms", C.c_float * 4)]


MODE_DTYPE = np.dtype([("mu", "<f4", 3), ("colour", "<f4", 3), ("cov", "<f4", 6), ("icov", "<f4", 6),
                       ("isqrt", "<f4", 6), ("size", "<i4")])
ENTRY_DTYPE = np.dtype([("xyz", "<f4", 3), ("rgb", "u1", 3), ("pad", "u1")])
PRIM_DTYPE = np.dtype([("type", "<i4"), ("a", "<f4", 3), ("b", "<f4", 3), ("colour", "<f4", 3), ("cell", "<f4"),
                       ("tex_seed", "<u4")])
assert C.sizeof(Result) == 136 and C.sizeof(RansacParams) == 56 and C.sizeof(Intrinsics) == 40
assert MODE_DTYPE.itemsize == 100 and ENTRY_DTYPE.itemsize == 16 and PRIM_DTYPE.itemsize == 48

MODE_RAW, MODE_ICP, MODE_RANKED = 0, 1, 2

# ---- error mapping (core.hpp:24-72) -------------------------------------------------------


class ScrelocError(RuntimeError):
    """screloc::Error"""


class InvalidDepth(ScrelocError):
    pass


class InvalidCentrePixel(ScrelocError):
    pass


class UnreliablePose(ScrelocError):
    pass


class NoHypotheses(ScrelocError):
    pass


class AllCandidatesFailed(ScrelocError):
    pass


class DimensionMismatch(ScrelocError):
    pass


class MalformedData(ScrelocError):
    pass


class CudaError(ScrelocError):
    pass


STATUS_ERRORS = {1: ScrelocError, 2: InvalidDepth, 3: InvalidCentrePixel, 4: UnreliablePose, 5: NoHypotheses,
                 6: AllCandidatesFailed, 7: DimensionMismatch, 8: MalformedData, 9: CudaError, 10: CudaError}

# Every symbol include/screloc_gpu.h declares: (restype, argtypes)
_vp, _i32, _i64, _u64, _dbl, _flt, _sz = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_float, C.c_size_t
_P = C.POINTER
SIGNATURES = {
    "scr_last_error": (C.c_char_p, []),
    "scr_version": (C.c_char_p, []),
    "scr_device_open": (C.c_int, [C.c_int, _P(_vp)]),
    "scr_device_close": (None, [_vp]),
    "scr_scene_create": (C.c_int, [_vp, _P(C.c_uint8), _sz, _P(ForestParams), _P(Intrinsics), _u64, C.c_int,
                                   _P(_vp)]),
    "scr_scene_destroy": (None, [_vp]),
    "scr_scene_fork": (C.c_int, [_vp, C.c_int, _P(_vp)]),
    "scr_tsdf_create": (C.c_int, [_vp, _P(C.c_float), C.c_float, C.c_int, C.c_int, C.c_int, C.c_float, _P(_vp)]),
    "scr_tsdf_destroy": (None, [_vp]),
    "scr_tsdf_fuse": (C.c_int, [_vp, _P(Intrinsics), _P(C.c_float), _P(Pose)]),
    "scr_tsdf_raycast": (C.c_int, [_vp, _P(Intrinsics), _P(Pose), _P(C.c_float), _P(C.c_uint32)]),
    "scr_tsdf_download": (C.c_int, [_vp, _P(C.c_float), _P(C.c_float)]),
    "scr_scene_set_tsdf_model": (C.c_int, [_vp, _vp]),
    "scr_scene_total_leaves": (_i64, [_vp]),
    "scr_scene_stream": (_vp, [_vp]),
    "scr_scene_set_analytic_model": (C.c_int, [_vp, _vp, C.c_int]),
    "scr_train": (C.c_int, [_vp, _P(Frame), _P(Pose)]),
    "scr_train_batch": (C.c_int, [_vp, _P(Frame), _P(Pose), C.c_int]),
    "scr_update": (C.c_int, [_vp, _i64]),
    "scr_reset": (C.c_int, [_vp]),
    "scr_relocalise_batch": (C.c_int, [_vp, _P(Frame), C.c_int, _P(RansacParams), C.c_int, _P(_u64), _P(Result)]),
    "scr_cascade_batch": (C.c_int, [_vp, _P(Frame), C.c_int, _P(RansacParams), _P(_i32), _P(_dbl), C.c_int,
                                    _P(_u64), _P(Result)]),
    "scr_frameset_create": (C.c_int, [_vp, C.c_int, _P(_vp)]),
    "scr_frameset_destroy": (None, [_vp]),
    "scr_frameset_upload": (C.c_int, [_vp, C.c_int, _P(Frame), C.c_int]),
    "scr_frameset_render": (C.c_int, [_vp, C.c_int, _P(Pose), C.c_int]),
    "scr_frameset_download": (C.c_int, [_vp, C.c_int, C.c_int, _vp, _vp]),
    "scr_train_frameset": (C.c_int, [_vp, _vp, _P(_i32), _P(Pose), C.c_int]),
    "scr_cascade_frameset": (C.c_int, [_vp, _vp, _P(_i32), C.c_int, _P(RansacParams), _P(_i32), _P(_dbl), C.c_int,
                                       _P(_u64), _P(Result)]),
    "scr_predictions_bytes": (_sz, [_vp]),
    "scr_predictions_export": (C.c_int, [_vp, _vp]),
    "scr_predictions_import": (C.c_int, [_vp, _vp]),
    "scr_broadcast_predictions": (C.c_int, [_P(_vp), C.c_int, C.c_int]),
    "scr_debug_leaves": (C.c_int, [_vp, _P(Frame), _P(_i32), _P(_i32), _P(C.c_int)]),
    "scr_debug_features": (C.c_int, [_vp, _P(Frame), _P(_i32), C.c_int, _P(_flt)]),
    "scr_dump_seen": (C.c_int, [_vp, _P(C.c_uint32)]),
    "scr_dump_entries": (C.c_int, [_vp, _i64, _i64, _vp]),
    "scr_dump_predictions": (C.c_int, [_vp, _P(_i32), _vp]),
    "scr_load_predictions": (C.c_int, [_vp, _P(_i32), _vp]),
    "scr_update_cursor": (_i64, [_vp]),
    "scr_debug_cluster": (C.c_int, [_vp, _vp, C.c_int, _vp, _P(_i32), _P(C.c_int)]),
    "scr_debug_ransac": (C.c_int, [_vp, _P(Frame), _P(RansacParams), _u64, _P(_i32), _P(Pose), _P(C.c_int),
                                   _P(_i32), _P(Pose), _P(_flt), _P(C.c_int)]),
    "scr_debug_generation_mode": (C.c_int, [_vp, C.c_int]),
    "scr_debug_generation_stats": (C.c_int, [_vp, _P(Frame), _P(RansacParams), _u64, _P(_i64), _P(C.c_int)]),
    "scr_debug_icp": (C.c_int, [_vp, _P(Frame), _P(Pose), _P(Pose), _P(C.c_int), _P(_dbl), _P(_dbl), _P(_dbl)]),
    "scr_kernel_launches": (_i64, [_vp]),
    "scr_profile_enable": (C.c_int, [_vp, C.c_int]),
    "scr_profile_read": (C.c_int, [_vp, _P(C.c_char_p), _P(_dbl), _P(_i64), _P(_u64), C.c_int]),
    "scr_generate_random_forest": (_sz, [_u64, C.c_int, _dbl, C.c_int, C.c_int, _P(C.c_uint8), _sz]),
    "scr_generate_synthetic_scene": (C.c_int, [_u64, C.c_int, _vp, C.c_int]),
    "scr_generate_trajectory": (None, [_u64, C.c_int, C.c_int, _P(Pose)]),
}

_LIB = None


def load(path: str = LIB_PATH):
    """Loads libscreloc_gpu.so; raises if it has not been built (no fallback exists)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise OSError(f"{path} is missing: build it with `python -m paper_1810_12163_b200.build` "
                      "(there is no CPU fallback for the product path)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def check(status: int, what: str = "") -> None:
    if status == 0:
        return
    msg = load().scr_last_error().decode(errors="replace")
    raise STATUS_ERRORS.get(status, ScrelocError)(f"{what}: {msg} (status {status})")


def ptr(a: np.ndarray, ctype=C.c_uint8):
    return a.ctypes.data_as(C.POINTER(ctype))

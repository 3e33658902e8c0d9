"""ORACLE — test infrastructure only.

ctypes bindings for oracle/lib/liboracle.so (the CPU restatement of the reference
path). Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "liboracle.so")


class Intrinsics(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double)]


class Pose(C.Structure):
    _fields_ = [("R", C.c_double * 9), ("t", C.c_double * 3)]


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
assert MODE_DTYPE.itemsize == 100 and ENTRY_DTYPE.itemsize == 16 and PRIM_DTYPE.itemsize == 48

# Table 4 profiles; colour threshold 30, rigidity 0.05.
PROFILES = {
    "default": dict(max_gen_iters=6000, n_max=1024, n_cull=64, eta=512, pose_update=1, use_cov=1,
                    min_sq_dist=0.09, n_out=16),
    "fast": dict(max_gen_iters=500, n_max=2048, n_cull=64, eta=256, pose_update=0, use_cov=0,
                 min_sq_dist=0.0, n_out=1),
    "intermediate": dict(max_gen_iters=1000, n_max=2048, n_cull=64, eta=256, pose_update=1, use_cov=0,
                         min_sq_dist=0.09, n_out=1),
    "slow": dict(max_gen_iters=250, n_max=2048, n_cull=64, eta=256, pose_update=1, use_cov=0,
                 min_sq_dist=0.0225, n_out=16),
}
FOREST_DEFAULT = dict(sigma=0.1, tau=0.05, max_clusters=50, min_cluster_size=20, capacity=1024)
FOREST_CASCADE = dict(sigma=0.1, tau=0.2, max_clusters=50, min_cluster_size=5, capacity=2048)
CASCADE_MODES = (1, 1, 2)          # Fast w/ICP, Intermediate w/ICP, Slow w/Ranking
CASCADE_THRESHOLDS = (0.05, 0.075)


def ransac_params(name_or_dict, **over) -> RansacParams:
    d = dict(PROFILES[name_or_dict]) if isinstance(name_or_dict, str) else dict(name_or_dict)
    d.update(over)
    p = RansacParams()
    p.colour_thresh = 30.0
    p.rigidity_tol = 0.05
    for k, v in d.items():
        setattr(p, k, v)
    return p


def intrinsics(width=640, height=480, fx=585.0, fy=585.0, cx=None, cy=None) -> Intrinsics:
    return Intrinsics(width, height, fx, fy, width / 2.0 if cx is None else cx, height / 2.0 if cy is None else cy)


def pose_from(R, t) -> Pose:
    p = Pose()
    for i, v in enumerate(np.asarray(R, dtype=np.float64).reshape(9)):
        p.R[i] = float(v)
    for i, v in enumerate(np.asarray(t, dtype=np.float64).reshape(3)):
        p.t[i] = float(v)
    return p


def pose_np(p: Pose):
    return np.array(p.R[:], dtype=np.float64).reshape(3, 3), np.array(p.t[:], dtype=np.float64)


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _ptr(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


class Oracle:
    def __init__(self, path: str = LIB_PATH):
        if not os.path.exists(path):
            build()
        self.lib = L = C.CDLL(path)
        vp, i32, i64, u64, dbl, flt = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_float
        P = C.POINTER
        sig = {
            "or_last_error": (C.c_char_p, []),
            "or_rng_u64": (None, [u64, C.c_int, u64, C.c_int, P(u64)]),
            "or_rng_uniform_int": (None, [u64, C.c_int, u64, u64, C.c_int, P(u64)]),
            "or_rng_uniform": (None, [u64, C.c_int, u64, C.c_int, P(dbl)]),
            "or_det_expf": (flt, [flt]),
            "or_det_sincos": (None, [dbl, P(dbl), P(dbl)]),
            "or_svd3": (None, [P(dbl)] * 4),
            "or_eig3": (None, [P(dbl)] * 3),
            "or_chol6": (C.c_int, [P(dbl)] * 3),
            "or_exp_se3": (None, [P(dbl), P(Pose)]),
            "or_log_se3": (C.c_int, [P(Pose), P(dbl)]),
            "or_kabsch": (C.c_int, [P(dbl), P(dbl), C.c_int, P(Pose)]),
            "or_backproject": (C.c_int, [C.c_int, C.c_int, dbl, P(Intrinsics), P(dbl)]),
            "or_pose_error": (None, [P(Pose), P(Pose), P(dbl), P(dbl)]),
            "or_compose": (None, [P(Pose), P(Pose), P(Pose)]),
            "or_invert": (None, [P(Pose), P(Pose)]),
            "or_feature_specs": (None, [u64, C.c_int, P(i32)]),
            "or_compute_feature": (C.c_int, [P(flt), P(C.c_uint8), C.c_int, C.c_int, C.c_int, C.c_int, P(i32),
                                             P(flt)]),
            "or_grid": (C.c_int, [P(flt), C.c_int, C.c_int, C.c_int, P(i32), C.c_int]),
            "or_forest_random": (vp, [u64, C.c_int, dbl, C.c_int, C.c_int]),
            "or_forest_deserialize": (vp, [P(C.c_uint8), C.c_size_t]),
            "or_forest_serialize": (C.c_size_t, [vp, P(C.c_uint8), C.c_size_t]),
            "or_forest_free": (None, [vp]),
            "or_forest_total_leaves": (i64, [vp]),
            "or_forest_trees": (C.c_int, [vp]),
            "or_forest_nodes": (C.c_int, [vp, C.c_int]),
            "or_forest_dump_tree": (None, [vp, C.c_int, P(i32)]),
            "or_forest_specs": (None, [vp, P(i32)]),
            "or_forest_leaves": (C.c_int, [vp, P(flt), P(C.c_uint8), C.c_int, C.c_int, P(i32), C.c_int, P(i32)]),
            "or_scene_generate": (vp, [u64, C.c_int]),
            "or_scene_from_prims": (vp, [vp, C.c_int]),
            "or_scene_free": (None, [vp]),
            "or_scene_prims": (C.c_int, [vp, vp, C.c_int]),
            "or_render": (None, [vp, P(Pose), P(Intrinsics), P(flt), P(C.c_uint8)]),
            "or_render_batch": (None, [vp, P(Pose), C.c_int, P(Intrinsics), P(flt), P(C.c_uint8), C.c_int]),
            "or_trajectory": (None, [u64, C.c_int, C.c_int, P(Pose)]),
            "or_state_create": (vp, [vp, flt, flt, C.c_int, C.c_int, C.c_int, u64]),
            "or_state_free": (None, [vp]),
            "or_integrate": (C.c_int, [vp, vp, P(flt), P(C.c_uint8), P(Intrinsics), C.c_int, P(Pose)]),
            "or_update": (None, [vp, i64]),
            "or_update_all_parallel": (None, [vp, C.c_int]),
            "or_clear": (None, [vp]),
            "or_cursor": (i64, [vp]),
            "or_dump_seen": (None, [vp, P(C.c_uint32)]),
            "or_dump_entries": (None, [vp, i64, i64, vp]),
            "or_dump_predictions": (None, [vp, P(i32), vp]),
            "or_load_predictions": (None, [vp, P(i32), vp]),
            "or_cluster": (C.c_int, [vp, C.c_int, flt, flt, C.c_int, C.c_int, vp, P(i32)]),
            "or_ransac": (C.c_int, [vp, vp, P(flt), P(C.c_uint8), P(Intrinsics), P(RansacParams), u64, P(i32),
                                    P(Pose), P(C.c_int), P(i32), P(Pose), P(flt), P(C.c_int)]),
            "or_relocalise": (C.c_int, [vp, vp, vp, P(flt), P(C.c_uint8), P(Intrinsics), P(RansacParams),
                                        C.c_int, u64, P(Result)]),
            "or_cascade_batch": (C.c_int, [vp, vp, vp, P(flt), P(C.c_uint8), P(Intrinsics), C.c_int,
                                           P(RansacParams), P(i32), P(dbl), C.c_int, P(u64), C.c_int, P(Result)]),
            "or_icp": (C.c_int, [vp, P(flt), P(C.c_uint8), P(Intrinsics), P(Pose), P(Pose), P(C.c_int), P(dbl),
                                 P(dbl)]),
            "or_depth_diff": (dbl, [vp, P(flt), P(C.c_uint8), P(Intrinsics), P(Pose)]),
            "or_depth_diff_images": (dbl, [P(flt), P(flt), C.c_int, C.c_int]),
            "or_raycast_depth": (None, [vp, P(Pose), P(Intrinsics), P(flt)]),
            "or_stage_seed": (u64, [u64, C.c_int]),
            "or_check_triplet": (C.c_int, [P(dbl), P(dbl), P(RansacParams), P(Pose)]),
            "or_lm_residual_jacobian": (None, [P(Pose), P(dbl), vp, C.c_int, P(dbl), P(dbl)]),
            "or_generation_stats": (C.c_int, [vp, vp, P(flt), P(C.c_uint8), P(Intrinsics), P(RansacParams), u64,
                                              P(Pose), dbl, P(C.c_int64), P(C.c_int), P(dbl), P(dbl)]),
            "or_energy": (C.c_int, [vp, vp, P(flt), P(C.c_uint8), P(Intrinsics), P(Pose), P(i32), C.c_int, P(flt)]),
            "or_lm": (C.c_int, [vp, vp, P(flt), P(C.c_uint8), P(Intrinsics), P(Pose), P(i32), C.c_int, C.c_int,
                                P(dbl)]),
            "or_integrate_batch": (C.c_int, [vp, vp, P(flt), P(C.c_uint8), P(Intrinsics), P(Pose), C.c_int,
                                             C.c_int]),
            "or_grid_count": (C.c_int, [vp, vp, P(flt), P(C.c_uint8), P(Intrinsics), P(i32), C.c_int]),
            "or_tsdf_create": (vp, [P(flt), flt, C.c_int, C.c_int, C.c_int, flt]),
            "or_tsdf_free": (None, [vp]),
            "or_tsdf_fuse": (None, [vp, P(flt), P(Intrinsics), P(Pose)]),
            "or_tsdf_dump": (None, [vp, P(flt), P(flt)]),
            "or_tsdf_raycast": (None, [vp, P(Pose), P(Intrinsics), P(flt), P(C.c_uint32)]),
            "or_scene_set_tsdf": (None, [vp, vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args

    def err(self) -> str:
        return self.lib.or_last_error().decode()

    # ---- convenience wrappers -------------------------------------------------
    def trajectory(self, seed: int, n: int, kind: int):
        arr = (Pose * n)()
        self.lib.or_trajectory(seed, n, kind, arr)
        return list(arr)

    def render(self, scene, poses, k: Intrinsics, threads: int = 8):
        n = len(poses)
        depth = np.zeros((n, k.height, k.width), np.float32)
        rgb = np.zeros((n, k.height, k.width, 3), np.uint8)
        arr = (Pose * n)(*poses)
        self.lib.or_render_batch(scene, arr, n, C.byref(k), _ptr(depth, C.c_float), _ptr(rgb, C.c_uint8), threads)
        return depth, rgb

    def scene_prims(self, scene):
        n = self.lib.or_scene_prims(scene, None, 0)
        out = np.zeros(n, PRIM_DTYPE)
        self.lib.or_scene_prims(scene, out.ctypes.data, n)
        return out

    def feature_specs(self, seed: int, radius: int = 130):
        out = np.zeros((256, 4), np.int32)
        self.lib.or_feature_specs(seed, radius, _ptr(out, C.c_int32))
        return out

    def grid(self, depth, spacing=4):
        h, w = depth.shape
        d = np.ascontiguousarray(depth, np.float32)
        out = np.zeros(((h + spacing - 1) // spacing) * ((w + spacing - 1) // spacing), np.int32)
        n = self.lib.or_grid(_ptr(d, C.c_float), w, h, spacing, _ptr(out, C.c_int32), out.size)
        return out[:n]

    def forest_leaves(self, forest, depth, rgb, px):
        h, w = depth.shape
        T = self.lib.or_forest_trees(forest)
        px = np.ascontiguousarray(px, np.int32)
        out = np.zeros((px.size, T), np.int32)
        d = np.ascontiguousarray(depth, np.float32)
        c = np.ascontiguousarray(rgb, np.uint8)
        rc = self.lib.or_forest_leaves(forest, _ptr(d, C.c_float), _ptr(c, C.c_uint8), w, h, _ptr(px, C.c_int32),
                                       px.size, _ptr(out, C.c_int32))
        if rc:
            raise RuntimeError(self.err())
        return out

    def serialize(self, forest) -> bytes:
        n = self.lib.or_forest_serialize(forest, None, 0)
        buf = (C.c_uint8 * n)()
        self.lib.or_forest_serialize(forest, buf, n)
        return bytes(buf)

    def state_create(self, forest, fp: dict, seed: int = 7):
        return self.lib.or_state_create(forest, fp["sigma"], fp["tau"], fp["max_clusters"], fp["min_cluster_size"],
                                        fp["capacity"], seed)

    def integrate(self, state, forest, depth, rgb, k, pose, reliable=1):
        d = np.ascontiguousarray(depth, np.float32)
        c = np.ascontiguousarray(rgb, np.uint8)
        return self.lib.or_integrate(state, forest, _ptr(d, C.c_float), _ptr(c, C.c_uint8), C.byref(k), reliable,
                                     C.byref(pose))

    def predictions(self, state, total_leaves: int, with_modes=True):
        counts = np.zeros(total_leaves, np.int32)
        modes = np.zeros(total_leaves * 50, MODE_DTYPE) if with_modes else None
        self.lib.or_dump_predictions(state, _ptr(counts, C.c_int32), modes.ctypes.data if with_modes else None)
        return counts, modes

    def load_predictions(self, state, counts, modes):
        counts = np.ascontiguousarray(counts, np.int32)
        modes = np.ascontiguousarray(modes, MODE_DTYPE)
        self.lib.or_load_predictions(state, _ptr(counts, C.c_int32), modes.ctypes.data)

    def seen(self, state, total_leaves: int):
        out = np.zeros(total_leaves, np.uint32)
        self.lib.or_dump_seen(state, _ptr(out, C.c_uint32))
        return out

    def entries(self, state, slot0: int, nslots: int, capacity: int):
        out = np.zeros(nslots * capacity, ENTRY_DTYPE)
        self.lib.or_dump_entries(state, slot0, nslots, out.ctypes.data)
        return out.reshape(nslots, capacity)

    def cluster(self, entries, fp: dict):
        e = np.ascontiguousarray(entries, ENTRY_DTYPE)
        out = np.zeros(fp["max_clusters"], MODE_DTYPE)
        labels = np.zeros(max(1, e.size), np.int32)
        n = self.lib.or_cluster(e.ctypes.data, e.size, fp["sigma"], fp["tau"], fp["min_cluster_size"],
                                fp["max_clusters"], out.ctypes.data, _ptr(labels, C.c_int32))
        return out[:n], labels[:e.size]

    def relocalise(self, forest, state, scene, depth, rgb, k, params, mode, seed):
        d = np.ascontiguousarray(depth, np.float32)
        c = np.ascontiguousarray(rgb, np.uint8)
        r = Result()
        rc = self.lib.or_relocalise(forest, state, scene, _ptr(d, C.c_float), _ptr(c, C.c_uint8), C.byref(k),
                                    C.byref(params), mode, seed, C.byref(r))
        if rc:
            raise RuntimeError(self.err())
        return r

    def cascade_batch(self, forest, state, scene, depth, rgb, k, stages, modes, thresholds, seeds, threads=8):
        n = depth.shape[0]
        d = np.ascontiguousarray(depth, np.float32)
        c = np.ascontiguousarray(rgb, np.uint8)
        st = (RansacParams * len(stages))(*stages)
        md = np.asarray(modes, np.int32)
        th = np.asarray(list(thresholds) + [0.0], np.float64)
        sd = np.asarray(seeds, np.uint64)
        out = (Result * n)()
        rc = self.lib.or_cascade_batch(forest, state, scene, _ptr(d, C.c_float), _ptr(c, C.c_uint8), C.byref(k), n,
                                       st, _ptr(md, C.c_int32), _ptr(th, C.c_double), len(stages),
                                       _ptr(sd, C.c_uint64), threads, out)
        if rc:
            raise RuntimeError(self.err())
        return list(out)

    REJECTION_TAGS = ("OK", "NoModes", "ColourCheckFailed", "TooClose", "NotRigid", "DegenerateKabsch")

    def generation_stats(self, forest, state, depth, rgb, k, params, seed, gt=None, radius=0.05):
        """Per-attempt rejection-tag histogram of generate_hypothesis over all slots of one frame
        ({tag: attempts}, slots ok, fraction of modes within `radius` of the true point, fraction
        of moded grid pixels with such a mode)."""
        tags = (C.c_int64 * 6)()
        ok = C.c_int()
        mf, pf = C.c_double(), C.c_double()
        d = np.ascontiguousarray(depth, np.float32)
        c = np.ascontiguousarray(rgb, np.uint8)
        rc = self.lib.or_generation_stats(forest, state, _ptr(d, C.c_float), _ptr(c, C.c_uint8), C.byref(k),
                                          C.byref(params), seed, C.byref(gt) if gt is not None else None, radius,
                                          tags, C.byref(ok), C.byref(mf), C.byref(pf))
        if rc:
            raise RuntimeError(self.err())
        return dict(zip(self.REJECTION_TAGS, list(tags))), ok.value, mf.value, pf.value

    def check_triplet(self, cam, world, params):
        cm = np.ascontiguousarray(cam, np.float64).reshape(9)
        w = np.ascontiguousarray(world, np.float64).reshape(9)
        out = Pose()
        tag = self.lib.or_check_triplet(_ptr(cm, C.c_double), _ptr(w, C.c_double), C.byref(params), C.byref(out))
        return self.REJECTION_TAGS[tag], out

    def lm_residual_jacobian(self, H, x, mode, use_cov):
        xx = np.ascontiguousarray(x, np.float64)
        m = np.ascontiguousarray(mode, MODE_DTYPE)
        r = np.zeros(3)
        J = np.zeros(18)
        self.lib.or_lm_residual_jacobian(C.byref(H), _ptr(xx, C.c_double), m.ctypes.data, int(use_cov),
                                         _ptr(r, C.c_double), _ptr(J, C.c_double))
        return r, J.reshape(3, 6)

    # ---- TSDF model ----
    def tsdf_create(self, origin, voxel, dims, trunc=None):
        o = np.ascontiguousarray(origin, np.float32)
        return self.lib.or_tsdf_create(_ptr(o, C.c_float), float(voxel), int(dims[0]), int(dims[1]), int(dims[2]),
                                       float(4 * voxel if trunc is None else trunc))

    def tsdf_fuse(self, vol, depth, k, pose):
        d = np.ascontiguousarray(depth, np.float32)
        self.lib.or_tsdf_fuse(vol, _ptr(d, C.c_float), C.byref(k), C.byref(pose))

    def tsdf_dump(self, vol, dims):
        n = int(dims[0]) * int(dims[1]) * int(dims[2])
        t, w = np.zeros(n, np.float32), np.zeros(n, np.float32)
        self.lib.or_tsdf_dump(vol, _ptr(t, C.c_float), _ptr(w, C.c_float))
        return t, w

    def tsdf_raycast(self, vol, pose, k):
        d = np.zeros((k.height, k.width), np.float32)
        nrm = np.zeros((k.height, k.width), np.uint32)
        self.lib.or_tsdf_raycast(vol, C.byref(pose), C.byref(k), _ptr(d, C.c_float), _ptr(nrm, C.c_uint32))
        return d, nrm

    def ransac(self, forest, state, depth, rgb, k, params, seed):
        d = np.ascontiguousarray(depth, np.float32)
        c = np.ascontiguousarray(rgb, np.uint8)
        nmax = params.n_max
        gs = np.zeros(nmax, np.int32)
        gp = (Pose * nmax)()
        ng = C.c_int()
        ss = np.zeros(nmax, np.int32)
        sp = (Pose * nmax)()
        se = np.zeros(nmax, np.float32)
        ns = C.c_int()
        rc = self.lib.or_ransac(forest, state, _ptr(d, C.c_float), _ptr(c, C.c_uint8), C.byref(k), C.byref(params),
                                seed, _ptr(gs, C.c_int32), gp, C.byref(ng), _ptr(ss, C.c_int32), sp,
                                _ptr(se, C.c_float), C.byref(ns))
        return rc, gs[:ng.value], list(gp)[:ng.value], ss[:ns.value], list(sp)[:ns.value], se[:ns.value]


_ORACLE = None


def get() -> Oracle:
    global _ORACLE
    if _ORACLE is None:
        _ORACLE = Oracle()
    return _ORACLE

"""Host-side mirror of the reference relocaliser interface (namespace screloc).

Names, argument meaning and error behaviour follow the reference API:
  integrate_frame(state, forest, frame, pose)
  update_leaves_round_robin(state, 256)
  clear_adaptation(state)
  relocalise(profile, frame, state, forest, model, mode)
  run_cascade(config, frame, ...)
A `Scene` bundles ForestModel + AdaptationState + SceneModel on one GPU; every call
goes through the C ABI (include/screloc_gpu.h) into the sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

from . import native as N

# Table 4; colour threshold 30 and rigidity 0.05 m are the
# artifact defaults of SPEC.md:501-502.
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
FOREST_PROFILES = {
    "default": dict(sigma=0.1, tau=0.05, max_clusters=50, min_cluster_size=20, capacity=1024),
    "cascade": dict(sigma=0.1, tau=0.2, max_clusters=50, min_cluster_size=5, capacity=2048),
}
MODES = {"raw": N.MODE_RAW, "icp": N.MODE_ICP, "ranked": N.MODE_RANKED}


def ransac_params(profile="default", **override) -> N.RansacParams:
    d = dict(PROFILES[profile]) if isinstance(profile, str) else dict(profile)
    d.update(override)
    p = N.RansacParams()
    p.colour_thresh = 30.0
    p.rigidity_tol = 0.05
    for k, v in d.items():
        setattr(p, k, v)
    return p


def forest_params(profile="default", **override) -> N.ForestParams:
    d = dict(FOREST_PROFILES[profile]) if isinstance(profile, str) else dict(profile)
    d.update(override)
    fp = N.ForestParams()
    for k, v in d.items():
        setattr(fp, k, v)
    return fp


def intrinsics(width=640, height=480, fx=585.0, fy=585.0, cx=None, cy=None) -> N.Intrinsics:
    return N.Intrinsics(width, height, fx, fy, width / 2.0 if cx is None else cx, height / 2.0 if cy is None else cy)


def to_pose(pose) -> N.Pose:
    if isinstance(pose, N.Pose):
        return pose
    if hasattr(pose, "R") and hasattr(pose, "t"):
        R, t = pose.R, pose.t
    elif isinstance(pose, np.ndarray) and pose.shape == (4, 4):  # camera->world matrix
        R, t = pose[:3, :3], pose[:3, 3]
    else:
        R, t = pose
    p = N.Pose()
    p.R[:] = [float(v) for v in np.asarray(R, np.float64).reshape(9)]
    p.t[:] = [float(v) for v in np.asarray(t, np.float64).reshape(3)]
    return p


def pose_arrays(p: N.Pose):
    return np.array(p.R[:], np.float64).reshape(3, 3), np.array(p.t[:], np.float64)


@dataclass
class CascadeConfig:
    """CascadeConfig: stages + fallback thresholds (metres)."""
    stages: Sequence[N.RansacParams]
    modes: Sequence[int]
    thresholds: Sequence[float]

    @staticmethod
    def paper_three_stage() -> "CascadeConfig":
        # F(5 cm) -> I(7.5 cm) -> S with ICP, ICP, ranking
        return CascadeConfig([ransac_params("fast"), ransac_params("intermediate"), ransac_params("slow")],
                             [N.MODE_ICP, N.MODE_ICP, N.MODE_RANKED], [0.05, 0.075])


@dataclass
class RelocalisationResult:
    """RelocalisationResult."""
    final_pose: tuple | None
    best_score: float
    stage_used: int
    status: int
    n_candidates: int
    stage_ms: list = field(default_factory=list)

    @staticmethod
    def from_c(r: N.Result) -> "RelocalisationResult":
        return RelocalisationResult(pose_arrays(r.pose) if r.has_pose else None, float(r.score), int(r.stage_used),
                                    int(r.status), int(r.n_candidates), list(r.stage_ms))


class Device:
    def __init__(self, ordinal: int = 0):
        self.lib = N.load()
        h = C.c_void_p()
        N.check(self.lib.scr_device_open(ordinal, C.byref(h)), "scr_device_open")
        self.handle = h
        self.ordinal = ordinal

    def close(self):
        if self.handle:
            self.lib.scr_device_close(self.handle)
            self.handle = None


def _frames(depths, rgbs, reliable=1, k: N.Intrinsics | None = None):
    """C frame views of (H, W) depth and (H, W, 3) colour arrays. Shapes that disagree with each
    other or with the scene's intrinsics raise DimensionMismatch (core.hpp:57) before any
    native call reads them."""
    if len(depths) != len(rgbs):
        raise N.DimensionMismatch(f"{len(depths)} depth images but {len(rgbs)} colour images")
    depths = [np.ascontiguousarray(d, np.float32) for d in depths]
    rgbs = [np.ascontiguousarray(c, np.uint8) for c in rgbs]
    arr = (N.Frame * len(depths))()
    for i, (d, c) in enumerate(zip(depths, rgbs)):
        if d.ndim != 2 or c.shape != d.shape + (3,):
            raise N.DimensionMismatch(f"frame {i}: depth {d.shape} and colour {c.shape} are not (H, W) / (H, W, 3)")
        if k is not None and d.shape != (k.height, k.width):
            raise N.DimensionMismatch(f"frame {i} is {d.shape[1]}x{d.shape[0]}, the scene's intrinsics are "
                                      f"{k.width}x{k.height}")
        arr[i].depth = d.ctypes.data
        arr[i].rgb = c.ctypes.data
        arr[i].height, arr[i].width = d.shape
        arr[i].pose_reliable = reliable
    return arr, (depths, rgbs)  # keep buffers alive


def _seeds(seeds, n: int) -> np.ndarray:
    sd = np.ascontiguousarray(seeds, np.uint64)
    if sd.ndim != 1 or sd.size != n:
        raise N.DimensionMismatch(f"{sd.size} seeds for {n} frames")
    return sd


class Scene:
    """ForestModel + AdaptationState + SceneModel resident on one B200."""

    def __init__(self, device: Device, forest_blob: bytes, fparams: N.ForestParams, k: N.Intrinsics,
                 adapt_seed: int = 7, max_batch: int = 64):
        self.lib = device.lib
        self.device = device
        self.k = k
        self.fparams = fparams
        blob = np.frombuffer(forest_blob, np.uint8).copy()
        h = C.c_void_p()
        N.check(self.lib.scr_scene_create(device.handle, N.ptr(blob), blob.size, C.byref(fparams), C.byref(k),
                                          adapt_seed, max_batch, C.byref(h)), "scr_scene_create")
        self.handle = h
        self.total_leaves = int(self.lib.scr_scene_total_leaves(h))
        self.trees = int(np.frombuffer(forest_blob[8:12], "<u4")[0])
        self.max_batch = max_batch
        self._lanes = []

    def fork(self, max_batch: int | None = None) -> "Scene":
        """A relocalisation lane: same forest / predictions / model, own stream + workspace
        (scr_scene_fork). Lanes let several host threads relocalise concurrently."""
        lane = Scene.__new__(Scene)
        lane.lib, lane.device, lane.k, lane.fparams = self.lib, self.device, self.k, self.fparams
        h = C.c_void_p()
        N.check(self.lib.scr_scene_fork(self.handle, max_batch or self.max_batch, C.byref(h)), "scr_scene_fork")
        lane.handle = h
        lane.total_leaves, lane.trees, lane.max_batch = self.total_leaves, self.trees, max_batch or self.max_batch
        lane.root = self  # the root must outlive its lanes
        self._lanes.append(lane)
        return lane

    def close(self):
        for lane in getattr(self, "_lanes", []):
            lane.close()
        if self.handle:
            self.lib.scr_scene_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return int(self.lib.scr_scene_stream(self.handle) or 0)

    @property
    def kernel_launches(self) -> int:
        return int(self.lib.scr_kernel_launches(self.handle))

    def profile(self, enable: bool = True):
        """Enables the in-library per-kernel CUDA-event profiler (and resets its totals)."""
        N.check(self.lib.scr_profile_enable(self.handle, 1 if enable else 0), "scr_profile_enable")

    WORK_NAMES = ("mode_evals", "sample_evals", "lm_terms", "icp_terms", "rays", "node_visits", "gen_attempts",
                  "lm_assoc_evals", "ray_prim_tests")

    def profile_read(self) -> dict:
        cap = 32
        names = (C.c_char_p * cap)()
        ms = (C.c_double * cap)()
        n = (C.c_int64 * cap)()
        work = (C.c_uint64 * 16)()
        k = self.lib.scr_profile_read(self.handle, names, ms, n, work, cap)
        kernels = {names[i].decode(): {"ms": ms[i], "launches": n[i]} for i in range(k)}
        return {"kernels": kernels, "work": {w: int(work[i]) for i, w in enumerate(self.WORK_NAMES)}}

    def set_tsdf_model(self, volume: "TsdfVolume | None"):
        """ICP and ranking use the fused volume (None: back to the analytic model)."""
        N.check(self.lib.scr_scene_set_tsdf_model(self.handle, volume.handle if volume else None),
                "scr_scene_set_tsdf_model")
        self._tsdf = volume  # keep it alive while the scene uses it

    def set_model(self, prims: np.ndarray):
        prims = np.ascontiguousarray(prims, N.PRIM_DTYPE)
        N.check(self.lib.scr_scene_set_analytic_model(self.handle, prims.ctypes.data, prims.size),
                "scr_scene_set_analytic_model")

    # ---- adaptation -------------------------------------------------------------------
    def integrate_frame(self, depth, rgb, pose, pose_reliable: bool = True):
        arr, keep = _frames([depth], [rgb], 1 if pose_reliable else 0, self.k)
        p = to_pose(pose)
        N.check(self.lib.scr_train(self.handle, arr, C.byref(p)), "integrate_frame")

    def integrate_frames(self, depths, rgbs, poses):
        if len(poses) != len(depths):
            raise N.DimensionMismatch(f"{len(poses)} poses for {len(depths)} frames")
        arr, keep = _frames(depths, rgbs, 1, self.k)
        ps = (N.Pose * len(poses))(*[to_pose(p) for p in poses])
        N.check(self.lib.scr_train_batch(self.handle, arr, ps, len(poses)), "integrate_frame")

    def update_leaves_round_robin(self, leaves_per_call: int = 256):
        N.check(self.lib.scr_update(self.handle, leaves_per_call), "update_leaves_round_robin")

    def clear_adaptation(self):
        N.check(self.lib.scr_reset(self.handle), "clear_adaptation")

    @property
    def update_cursor(self) -> int:
        return int(self.lib.scr_update_cursor(self.handle))

    # ---- relocalisation -----------------------------------------------------------------
    def relocalise_batch(self, depths, rgbs, profile, mode, seeds) -> list[N.Result]:
        arr, keep = _frames(depths, rgbs, 1, self.k)
        n = len(depths)
        p = profile if isinstance(profile, N.RansacParams) else ransac_params(profile)
        sd = _seeds(seeds, n)
        out = (N.Result * n)()
        m = MODES[mode] if isinstance(mode, str) else int(mode)
        N.check(self.lib.scr_relocalise_batch(self.handle, arr, n, C.byref(p), m, N.ptr(sd, C.c_uint64), out),
                "relocalise")
        return list(out)

    def relocalise(self, depth, rgb, profile="default", mode="icp", seed: int = 0) -> RelocalisationResult:
        return RelocalisationResult.from_c(self.relocalise_batch([depth], [rgb], profile, mode, [seed])[0])

    def run_cascade_batch(self, depths, rgbs, config: CascadeConfig, seeds) -> list[N.Result]:
        arr, keep = _frames(depths, rgbs, 1, self.k)
        n = len(depths)
        st = (N.RansacParams * len(config.stages))(*config.stages)
        md = np.asarray(config.modes, np.int32)
        th = np.asarray(list(config.thresholds) + [0.0], np.float64)
        sd = _seeds(seeds, n)
        out = (N.Result * n)()
        N.check(self.lib.scr_cascade_batch(self.handle, arr, n, st, N.ptr(md, C.c_int32), N.ptr(th, C.c_double),
                                           len(config.stages), N.ptr(sd, C.c_uint64), out), "run_cascade")
        return list(out)

    def run_cascade(self, depth, rgb, config: CascadeConfig, seed: int = 0) -> RelocalisationResult:
        return RelocalisationResult.from_c(self.run_cascade_batch([depth], [rgb], config, [seed])[0])

    # ---- parity hooks -----------------------------------------------------------------
    def debug_leaves(self, depth, rgb):
        arr, keep = _frames([depth], [rgb], 1, self.k)
        h, w = np.asarray(depth).shape
        gmax = ((w + 3) // 4) * ((h + 3) // 4)
        T = 8
        px = np.zeros(gmax, np.int32)
        leaves = np.zeros(gmax * T, np.int32)
        n = C.c_int()
        N.check(self.lib.scr_debug_leaves(self.handle, arr, N.ptr(px, C.c_int32), N.ptr(leaves, C.c_int32),
                                          C.byref(n)), "debug_leaves")
        g = n.value
        return px[:g], leaves[: g * self.trees].reshape(g, self.trees)

    def debug_features(self, depth, rgb, px):
        arr, keep = _frames([depth], [rgb], 1, self.k)
        px = np.ascontiguousarray(px, np.int32)
        out = np.zeros((px.size, 256), np.float32)
        N.check(self.lib.scr_debug_features(self.handle, arr, N.ptr(px, C.c_int32), px.size, N.ptr(out, C.c_float)),
                "compute_feature_vector")
        return out

    def seen(self):
        out = np.zeros(self.total_leaves, np.uint32)
        N.check(self.lib.scr_dump_seen(self.handle, N.ptr(out, C.c_uint32)), "dump_seen")
        return out

    def entries(self, slot0: int, nslots: int):
        out = np.zeros(nslots * self.fparams.capacity, N.ENTRY_DTYPE)
        N.check(self.lib.scr_dump_entries(self.handle, slot0, nslots, out.ctypes.data), "dump_entries")
        return out.reshape(nslots, self.fparams.capacity)

    def predictions(self, with_modes: bool = True):
        counts = np.zeros(self.total_leaves, np.int32)
        modes = np.zeros(self.total_leaves * 50, N.MODE_DTYPE) if with_modes else None
        N.check(self.lib.scr_dump_predictions(self.handle, N.ptr(counts, C.c_int32),
                                              modes.ctypes.data if with_modes else None), "dump_predictions")
        return counts, modes

    def load_predictions(self, counts, modes):
        counts = np.ascontiguousarray(counts, np.int32)
        modes = np.ascontiguousarray(modes, N.MODE_DTYPE)
        N.check(self.lib.scr_load_predictions(self.handle, N.ptr(counts, C.c_int32), modes.ctypes.data),
                "load_predictions")

    def debug_cluster(self, entries):
        e = np.ascontiguousarray(entries, N.ENTRY_DTYPE)
        out = np.zeros(50, N.MODE_DTYPE)
        labels = np.zeros(max(1, e.size), np.int32)
        n = C.c_int()
        N.check(self.lib.scr_debug_cluster(self.handle, e.ctypes.data, e.size, out.ctypes.data,
                                           N.ptr(labels, C.c_int32), C.byref(n)), "cluster_reservoir")
        return out[: n.value], labels[: e.size]

    def debug_ransac(self, depth, rgb, params: N.RansacParams, seed: int):
        arr, keep = _frames([depth], [rgb], 1, self.k)
        nmax = params.n_max
        gs = np.zeros(nmax, np.int32)
        gp = (N.Pose * nmax)()
        ng = C.c_int()
        ss = np.zeros(nmax, np.int32)
        sp = (N.Pose * nmax)()
        se = np.zeros(nmax, np.float32)
        ns = C.c_int()
        st = self.lib.scr_debug_ransac(self.handle, arr, C.byref(params), seed, N.ptr(gs, C.c_int32), gp,
                                       C.byref(ng), N.ptr(ss, C.c_int32), sp, N.ptr(se, C.c_float), C.byref(ns))
        return st, gs[: ng.value], list(gp)[: ng.value], ss[: ns.value], list(sp)[: ns.value], se[: ns.value]

    def debug_generation_mode(self, mode: int) -> None:
        """Test hook: 1 = every passing triplet goes through the exact suspect/continuation path."""
        N.check(self.lib.scr_debug_generation_mode(self.handle, int(mode)), "debug_generation_mode")

    REJECTION_TAGS = ("OK", "NoModes", "ColourCheckFailed", "TooClose", "NotRigid", "DegenerateKabsch")

    def debug_generation_stats(self, depth, rgb, params: N.RansacParams, seed: int):
        """Per-attempt outcome histogram of hypothesis generation on one frame:
        ({tag: attempts}, slots that generated a hypothesis)."""
        arr, keep = _frames([depth], [rgb], 1, self.k)
        tags = np.zeros(6, np.int64)
        ok = C.c_int()
        N.check(self.lib.scr_debug_generation_stats(self.handle, arr, C.byref(params), seed, N.ptr(tags, C.c_int64),
                                                    C.byref(ok)), "generation_stats")
        return dict(zip(self.REJECTION_TAGS, (int(v) for v in tags))), ok.value

    def debug_icp(self, depth, rgb, init):
        arr, keep = _frames([depth], [rgb], 1, self.k)
        p = to_pose(init)
        out = N.Pose()
        conv = C.c_int()
        rms, inl, score = C.c_double(), C.c_double(), C.c_double()
        N.check(self.lib.scr_debug_icp(self.handle, arr, C.byref(p), C.byref(out), C.byref(conv), C.byref(rms),
                                       C.byref(inl), C.byref(score)), "icp_refine")
        return out, conv.value, rms.value, inl.value, score.value


def broadcast_predictions(scenes: list, root: int = 0) -> None:
    """One process, several GPUs: ncclBroadcast of root's adapted prediction table to the
    other scenes (scr_broadcast_predictions; one root scene per GPU, same forest)."""
    arr = (C.c_void_p * len(scenes))(*[s.handle.value if isinstance(s.handle, C.c_void_p) else s.handle
                                        for s in scenes])
    lib = scenes[0].lib if scenes else N.load()
    N.check(lib.scr_broadcast_predictions(arr, len(scenes), root), "scr_broadcast_predictions")


def generate_random_forest(seed: int = 42, height: int = 14, p_depth: float = 0.4, trees: int = 5,
                           radius: int = 130) -> bytes:
    """generate_random_forest (forest.hpp:104-106) -> serialised ForestModel."""
    lib = N.load()
    n = lib.scr_generate_random_forest(seed, height, p_depth, trees, radius, None, 0)
    if n == 0:
        raise N.ScrelocError("generate_random_forest: bad arguments")
    buf = (C.c_uint8 * n)()
    lib.scr_generate_random_forest(seed, height, p_depth, trees, radius, buf, n)
    return bytes(buf)


def generate_synthetic_scene(seed: int, complexity: int = 20) -> np.ndarray:
    lib = N.load()
    n = lib.scr_generate_synthetic_scene(seed, complexity, None, 0)
    out = np.zeros(n, N.PRIM_DTYPE)
    lib.scr_generate_synthetic_scene(seed, complexity, out.ctypes.data, n)
    return out


def generate_trajectory(seed: int, n: int, kind: int) -> list:
    arr = (N.Pose * n)()
    N.load().scr_generate_trajectory(seed, n, kind, arr)
    return list(arr)


class TsdfVolume:
    """Dense TSDF scene model on the device (scr_tsdf_*). fuse = fuse_frame,
    raycast = raycast_depth (z-depth + packed normals)."""

    def __init__(self, device: Device, origin, voxel: float, dims, trunc: float | None = None):
        self.lib, self.device = device.lib, device
        self.dims = tuple(int(d) for d in dims)
        o = np.ascontiguousarray(origin, np.float32)
        h = C.c_void_p()
        N.check(self.lib.scr_tsdf_create(device.handle, N.ptr(o, C.c_float), float(voxel), *self.dims,
                                         float(4 * voxel if trunc is None else trunc), C.byref(h)), "scr_tsdf_create")
        self.handle = h

    def fuse(self, depth, pose, k: N.Intrinsics):
        d = np.ascontiguousarray(depth, np.float32)
        p = to_pose(pose)
        N.check(self.lib.scr_tsdf_fuse(self.handle, C.byref(k), N.ptr(d, C.c_float), C.byref(p)), "fuse_frame")

    def raycast(self, pose, k: N.Intrinsics):
        d = np.zeros((k.height, k.width), np.float32)
        n = np.zeros((k.height, k.width), np.uint32)
        p = to_pose(pose)
        N.check(self.lib.scr_tsdf_raycast(self.handle, C.byref(k), C.byref(p), N.ptr(d, C.c_float),
                                          N.ptr(n, C.c_uint32)), "raycast_depth")
        return d, n

    def download(self):
        n = self.dims[0] * self.dims[1] * self.dims[2]
        t, w = np.zeros(n, np.float32), np.zeros(n, np.float32)
        N.check(self.lib.scr_tsdf_download(self.handle, N.ptr(t, C.c_float), N.ptr(w, C.c_float)), "tsdf download")
        return t, w

    def close(self):
        if self.handle:
            self.lib.scr_tsdf_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class FrameSet:
    """Frames resident in HBM (inputs for the device-timed bench path)."""

    def __init__(self, scene: Scene, capacity: int):
        self.scene = scene
        self.lib = scene.lib
        h = C.c_void_p()
        N.check(self.lib.scr_frameset_create(scene.handle, capacity, C.byref(h)), "scr_frameset_create")
        self.handle = h
        self.capacity = capacity

    def close(self):
        if self.handle:
            self.lib.scr_frameset_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def render(self, poses, first: int = 0):
        ps = (N.Pose * len(poses))(*[to_pose(p) for p in poses])
        N.check(self.lib.scr_frameset_render(self.handle, first, ps, len(poses)), "render_frame")

    def upload(self, depths, rgbs, first: int = 0):
        arr, keep = _frames(depths, rgbs, 1, self.scene.k)
        N.check(self.lib.scr_frameset_upload(self.handle, first, arr, len(depths)), "frameset_upload")

    def download(self, first: int, n: int):
        k = self.scene.k
        d = np.zeros((n, k.height, k.width), np.float32)
        c = np.zeros((n, k.height, k.width, 3), np.uint8)
        N.check(self.lib.scr_frameset_download(self.handle, first, n, d.ctypes.data, c.ctypes.data), "download")
        return d, c

    def train(self, idx: Iterable[int], poses):
        idx = np.ascontiguousarray(list(idx), np.int32)
        if len(poses) != idx.size:
            raise N.DimensionMismatch(f"{len(poses)} poses for {idx.size} frames")
        ps = (N.Pose * len(poses))(*[to_pose(p) for p in poses])
        N.check(self.lib.scr_train_frameset(self.scene.handle, self.handle, N.ptr(idx, C.c_int32), ps, idx.size),
                "integrate_frame")

    def cascade(self, idx, config: CascadeConfig, seeds, scene: "Scene | None" = None) -> list[N.Result]:
        """run_cascade over resident frames idx; `scene` may be a lane of the owning scene."""
        idx = np.ascontiguousarray(list(idx), np.int32)
        n = idx.size
        st = (N.RansacParams * len(config.stages))(*config.stages)
        md = np.asarray(config.modes, np.int32)
        th = np.asarray(list(config.thresholds) + [0.0], np.float64)
        sd = _seeds(seeds, n)
        out = (N.Result * n)()
        N.check(self.lib.scr_cascade_frameset((scene or self.scene).handle, self.handle, N.ptr(idx, C.c_int32), n, st,
                                              N.ptr(md, C.c_int32), N.ptr(th, C.c_double), len(config.stages),
                                              N.ptr(sd, C.c_uint64), out), "run_cascade")
        return list(out)

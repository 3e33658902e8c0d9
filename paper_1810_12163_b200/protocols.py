"""Evaluation protocols that drive the relocalisation hot path (the
reference's bench_cli module, §4.1-4.3).

* `run_headline_eval`: adapt on a training sequence (integrate every
  reliable frame, then refresh until every leaf is clustered), relocalise every test frame
  independently, report Table-1 aggregates.
* `run_tracking_loss_protocol` (§4.2): on one sequence, assume
  tracking is lost at every frame but the first: relocalise with the state available so
  far, then integrate the frame (ground-truth pose) and continue adapting. Relocalisation
  runs on a lane of the scene, adaptation on the scene itself, so the lane always sees the
  last *published* prediction state.
* `compute_novelty_bins` (§4.3).
* `perturb_missing_depth`, `perturb_noisy_depth` (§A.4.1-A.4.2): the
  depth perturbations of the robustness experiments (host-side, seeded numpy).

Every relocalisation goes through the B200 library (`Scene` / lanes); this module only
sequences calls and does the report arithmetic.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import native as N
from .relocaliser import CascadeConfig, Scene, pose_arrays, ransac_params, to_pose

SUCCESS_T_M = 0.05   # Table 1: <= 5 cm
SUCCESS_R_DEG = 5.0  # Table 1: <= 5 degrees


def pose_error(R_est, t_est, R_gt, t_gt) -> tuple[float, float]:
    """pose_error (geometry.hpp:206-216): translation distance (m) and rotation angle (deg)."""
    R_est, R_gt = np.asarray(R_est, float).reshape(3, 3), np.asarray(R_gt, float).reshape(3, 3)
    te = float(np.linalg.norm(np.asarray(t_est, float) - np.asarray(t_gt, float)))
    c = (np.trace(R_gt.T @ R_est) - 1.0) / 2.0
    ae = math.degrees(math.acos(min(1.0, max(-1.0, c))))
    return te, ae


def is_success(t_err: float, r_err_deg: float) -> bool:
    return t_err <= SUCCESS_T_M and r_err_deg <= SUCCESS_R_DEG


@dataclass
class FrameOutcome:
    has_pose: bool
    t_err: float = math.inf
    r_err: float = math.inf
    success: bool = False
    stage_used: int = 0
    score: float = math.inf
    pose: N.Pose | None = None  # the estimate (camera -> world)


@dataclass
class EvalReport:
    frames: list[FrameOutcome] = field(default_factory=list)

    @property
    def success_fraction(self) -> float:
        return sum(f.success for f in self.frames) / max(1, len(self.frames))

    @staticmethod
    def _lower_median(v: list[float]) -> float:
        if not v:
            return math.inf
        s = sorted(v)
        return s[(len(s) - 1) // 2]

    @property
    def median_t_err(self) -> float:
        return self._lower_median([f.t_err for f in self.frames])

    @property
    def median_r_err(self) -> float:
        return self._lower_median([f.r_err for f in self.frames])


def _outcome(r: N.Result, gt) -> FrameOutcome:
    if not r.has_pose:
        return FrameOutcome(False, stage_used=int(r.stage_used), score=float(r.score))
    R, t = pose_arrays(r.pose)
    Rg, tg = pose_arrays(to_pose(gt))
    te, ae = pose_error(R, t, Rg, tg)
    return FrameOutcome(True, te, ae, is_success(te, ae), int(r.stage_used), float(r.score), r.pose)


def _relocalise(scene: Scene, depths, rgbs, config, seeds) -> list[N.Result]:
    if isinstance(config, CascadeConfig):
        return scene.run_cascade_batch(depths, rgbs, config, seeds)
    profile, mode = config
    return scene.relocalise_batch(depths, rgbs, profile if isinstance(profile, N.RansacParams) else
                                  ransac_params(profile), mode, seeds)


def run_headline_eval(scene: Scene, adapt: tuple, test: tuple, config, seeds: Sequence[int],
                      batch: int | None = None) -> EvalReport:
    """adapt = (depths, rgbs, poses[, reliable flags]); test = (depths, rgbs, gt poses);
    config = CascadeConfig or (profile, mode)."""
    depths, rgbs, poses = adapt[:3]
    reliable = adapt[3] if len(adapt) > 3 else [True] * len(poses)
    keep = [i for i, r in enumerate(reliable) if r]  # integrate_frame rejects unreliable poses
    step = batch or scene.max_batch
    for i0 in range(0, len(keep), step):
        sel = keep[i0:i0 + step]
        scene.integrate_frames([depths[i] for i in sel], [rgbs[i] for i in sel], [poses[i] for i in sel])
    scene.update_leaves_round_robin(scene.total_leaves)  # every leaf clustered at least once
    tdepths, trgbs, tposes = test
    report = EvalReport()
    for i0 in range(0, len(tposes), step):
        res = _relocalise(scene, tdepths[i0:i0 + step], trgbs[i0:i0 + step], config, list(seeds[i0:i0 + step]))
        report.frames += [_outcome(r, tposes[i0 + j]) for j, r in enumerate(res)]
    return report


def run_tracking_loss_protocol(scene: Scene, seq: tuple, config, seeds: Sequence[int],
                               leaves_per_frame: int = 256) -> list[FrameOutcome | None]:
    """seq = (depths, rgbs, gt poses[, reliable flags]). Returns one outcome per frame; frame 0
    (empty forest) is never relocalised (None)."""
    depths, rgbs, poses = seq[:3]
    reliable = seq[3] if len(seq) > 3 else [True] * len(poses)
    lane = scene.fork(1)
    out: list[FrameOutcome | None] = []
    try:
        for i in range(len(poses)):
            if i == 0:
                out.append(None)
            else:
                r = _relocalise(lane, [depths[i]], [rgbs[i]], config, [seeds[i]])[0]
                out.append(_outcome(r, poses[i]))
            if reliable[i]:  # "use examples from the current frame to continue training"
                scene.integrate_frame(depths[i], rgbs[i], poses[i])
            scene.update_leaves_round_robin(leaves_per_frame)
    finally:
        lane.close()
        scene._lanes.remove(lane)
    return out


def success_curve(outcomes: Sequence[FrameOutcome | None], window: int = 0) -> np.ndarray:
    """Cumulative (window = 0) or windowed success fraction over the relocalised frames."""
    s = np.array([o.success for o in outcomes if o is not None], float)
    if s.size == 0:
        return s
    if window <= 0:
        return np.cumsum(s) / np.arange(1, s.size + 1)
    k = np.ones(window)
    return np.convolve(s, k, "full")[: s.size] / np.minimum(np.arange(1, s.size + 1), window)


def novelty_bin_keys(test_poses, training_poses, step: int = 5, last: int = 55) -> np.ndarray:
    """Novelty bin of every test pose: the first b in (5, 10, ..., `last`)
    such that some training pose is within b cm AND b degrees, else `last` + `step`.
    Vectorised over the training poses (same pose_error arithmetic, geometry.hpp:206-216)."""
    tr = [pose_arrays(to_pose(p)) for p in training_poses]
    Rt = np.stack([r for r, _ in tr])            # (n, 3, 3)
    tt = np.stack([t for _, t in tr])            # (n, 3)
    edges = np.arange(step, last + step, step, dtype=float)
    keys = np.empty(len(test_poses), np.int64)
    for i, tp in enumerate(test_poses):
        R, t = pose_arrays(to_pose(tp))
        te = np.linalg.norm(tt - t, axis=1) * 100.0
        c = (np.einsum("nij,ij->n", Rt, R) - 1.0) / 2.0  # trace(R_t^T R)
        ae = np.degrees(np.arccos(np.clip(c, -1.0, 1.0)))
        need = np.maximum(te, ae).min()  # smallest b with te <= b and ae <= b for one pose
        hit = edges[edges >= need]
        keys[i] = int(hit[0]) if hit.size else last + step
    return keys


def compute_novelty_bins(test_poses, outcomes: Sequence[FrameOutcome], training_poses, step: int = 5,
                         last: int = 55) -> dict:
    """A test pose belongs to the first bin b (5, 10, ..., `last` cm/deg) such that some
    training pose is within b cm AND b degrees of it; otherwise to the open bin `last`+.
    Returns {bin: (count, success fraction)}; the open bin is keyed by `last` + `step`."""
    keys = novelty_bin_keys(test_poses, training_poses, step, last)
    bins: dict[int, list[bool]] = {b: [] for b in range(step, last + 2 * step, step)}
    for key, o in zip(keys, outcomes):
        bins[int(key)].append(bool(o.success))
    return {b: (len(v), (sum(v) / len(v)) if v else math.nan) for b, v in bins.items()}


def perturb_missing_depth(depth: np.ndarray, p: float, rng: np.random.Generator) -> np.ndarray:
    """PAPER.md §A.4.1: draw r_i ~ U[0, 1] per pixel and set the pixel to 0 iff r_i <= p
    (invalid pixels stay invalid)."""
    if not (0.0 <= p <= 1.0):
        raise ValueError("p must be in [0, 1]")
    d = np.array(depth, np.float32, copy=True)
    r = rng.random(d.shape)
    d[r <= p] = 0.0
    return d


def perturb_noisy_depth(depth: np.ndarray, sigma: float, rng: np.random.Generator) -> np.ndarray:
    """PAPER.md §A.4.2: d_i <- d_i + n_i d_i with n_i ~ N(0, sigma^2); invalid pixels stay
    invalid."""
    if sigma < 0:
        raise ValueError("sigma must be >= 0")
    d = np.array(depth, np.float32, copy=True)
    valid = (d > 0) & (d <= 20.0) & np.isfinite(d)
    n = rng.normal(0.0, sigma, d.shape).astype(np.float32) if sigma > 0 else np.zeros(d.shape, np.float32)
    d[valid] = d[valid] + n[valid] * d[valid]
    return d

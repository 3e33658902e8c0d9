"""Appendix-B parameter tuner over the GPU relocaliser (the reference's
tuning module).

* `cost` (Appendix B): (1 - score)^2 if time <= t_max else inf.
* `coordinate_descent`: sweeps the coordinates in declaration order; per coordinate every
  value is evaluated with the others fixed and the argmin kept (ties keep the current
  value); stops after a sweep without change or `max_sweeps`; every evaluation is memoised
  by assignment. Evaluations of one coordinate scan are independent, so they run
  concurrently on relocalisation lanes of the scene (one host thread per lane).
* `sharded_parallel`: the same scans sharded across GPUs (one process per GPU,
  torch.distributed): the uncached assignments of a scan go to rank i mod N, each rank
  evaluates its share (on its own lanes), and the costs are all-gathered into every rank's
  memo, so all ranks take identical decisions.
* `tune_single`: objective = sum over (adapt, validation) sequence pairs of the cost of the
  profile on the validation frames after adapting on the training frames.
* `tune_cascade`: the four-step procedure of Appendix B.2 (tune the fastest stage fully,
  fix its forest parameters, tune the RANSAC parameters of the other stages, then the
  depth-difference thresholds against the amortised cost).

Relocalisation and adaptation run on the B200 library; this module is host-side control.
"""
from __future__ import annotations

import math
import threading
from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np

from . import native as N
from .protocols import is_success, pose_error
from .relocaliser import CascadeConfig, Scene, pose_arrays, ransac_params, to_pose

RANSAC_FIELDS = ("max_gen_iters", "n_max", "n_cull", "eta", "pose_update", "use_cov", "min_sq_dist", "n_out",
                 "colour_thresh", "rigidity_tol")
FOREST_FIELDS = ("sigma", "tau", "max_clusters", "min_cluster_size", "capacity")


@dataclass
class ParamDomain:
    name: str
    values: list

    def __post_init__(self):
        if not self.values:
            raise ValueError(f"ParamDomain {self.name}: empty value list")


def cost(score: float, time_ms: float, t_max: float) -> float:
    """Appendix B: (1 - score)^2 if time <= t_max, else infinity."""
    if not (0.0 <= score <= 1.0) or time_ms < 0:
        raise ValueError("score must be in [0, 1] and time >= 0")
    return (1.0 - score) ** 2 if time_ms <= t_max else math.inf


class Memo:
    """Evaluation memo keyed by assignment, safe under concurrent insert-or-get."""

    def __init__(self, fn: Callable[[dict], float]):
        self.fn = fn
        self.table: dict[tuple, float] = {}
        self.evaluations = 0
        self._lock = threading.Lock()
        self._pending: dict[tuple, threading.Event] = {}

    @staticmethod
    def key(a: dict) -> tuple:
        return tuple(sorted(a.items()))

    def __call__(self, a: dict) -> float:
        k = self.key(a)
        with self._lock:
            if k in self.table:
                return self.table[k]
            ev = self._pending.get(k)
            owner = ev is None
            if owner:
                ev = self._pending[k] = threading.Event()
        if not owner:
            ev.wait()
            return self.table[k]
        try:
            v = self.fn(dict(a))
        except Exception:  # evaluation failures count as infinite cost (SPEC.md tune_single)
            v = math.inf
        with self._lock:
            self.table[k] = v
            self.evaluations += 1
            del self._pending[k]
        ev.set()
        return v

    def cached(self, a: dict) -> bool:
        with self._lock:
            return self.key(a) in self.table

    def put(self, k: tuple, v: float) -> None:
        """Inserts a cost computed elsewhere (another rank); never overwrites."""
        with self._lock:
            self.table.setdefault(k, v)


def sharded_parallel(memo: Memo, dist=None, local: Callable[[list], list] | None = None) -> Callable[[list], list]:
    """`parallel` for coordinate_descent over N ranks: the scan's uncached assignments (in scan
    order, deduplicated) go to rank i mod N; each rank evaluates its share with `local` (e.g.
    GpuObjective.parallel on its lanes) or sequentially, then every rank all-gathers the
    (assignment, cost) pairs into its memo. Every rank therefore holds the same table and
    takes the same decisions; no rank evaluates an assignment another rank owns."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return local or (lambda cands: [memo(c) for c in cands])
    rank, world = dist.get_rank(), dist.get_world_size()

    def run(cands: list) -> list:
        todo, seen = [], set()
        for c in cands:
            k = Memo.key(c)
            if k not in seen and not memo.cached(c):
                seen.add(k)
                todo.append(c)
        mine = todo[rank::world]
        if local:
            local(mine)
        else:
            for c in mine:
                memo(c)
        pairs = [(Memo.key(c), memo(c)) for c in mine]
        parts = [None] * world
        dist.all_gather_object(parts, pairs)
        for part in parts:
            for k, v in part:
                memo.put(k, v)
        return [memo(c) for c in cands]

    return run


@dataclass
class DescentResult:
    assignment: dict
    cost: float
    sweeps: int
    evaluations: int
    history: list = field(default_factory=list)  # best cost after every sweep


def coordinate_descent(domains: Sequence[ParamDomain], objective: Callable[[dict], float], start: dict,
                       max_sweeps: int = 10, parallel: Callable[[list], list] | None = None) -> DescentResult:
    """`parallel(list of assignments) -> list of costs` evaluates one coordinate scan (e.g. on
    relocalisation lanes); default is sequential."""
    memo = objective if isinstance(objective, Memo) else Memo(objective)
    cur = dict(start)
    best = memo(cur)
    history = []
    sweeps = 0
    for sweeps in range(1, max_sweeps + 1):
        changed = False
        for d in domains:
            cands = [dict(cur, **{d.name: v}) for v in d.values]
            if parallel:
                parallel(cands)  # fills the memo concurrently
            costs = [memo(c) for c in cands]
            i_best = None
            for i, (c, v) in enumerate(zip(cands, costs)):
                if v < best:  # strict: ties keep the current value
                    best, i_best = v, i
            if i_best is not None and cands[i_best][d.name] != cur[d.name]:
                cur = cands[i_best]
                changed = True
        history.append(best)
        if not changed:
            break
    return DescentResult(cur, best, sweeps, memo.evaluations, history)


# ---- GPU objectives ------------------------------------------------------------------------
@dataclass
class Sequences:
    """(adapt, validation) pairs; each sequence = (depths, rgbs, poses)."""
    pairs: list


def _split(assignment: dict) -> tuple[dict, dict]:
    rp = {k: v for k, v in assignment.items() if k in RANSAC_FIELDS}
    fp = {k: v for k, v in assignment.items() if k in FOREST_FIELDS}
    return rp, fp


def _evaluate(scene: Scene, params: N.RansacParams, mode, val, seeds) -> tuple[float, float]:
    """Success fraction and mean per-frame GPU time (ms) of one profile on one validation set."""
    depths, rgbs, poses = val
    res = scene.relocalise_batch(depths, rgbs, params, mode, seeds)
    ok = 0
    t = 0.0
    for r, gt in zip(res, poses):
        t += float(r.stage_ms[0])
        if r.has_pose:
            R, tt = pose_arrays(r.pose)
            Rg, tg = pose_arrays(to_pose(gt))
            ok += is_success(*pose_error(R, tt, Rg, tg))
    return ok / max(1, len(poses)), t / max(1, len(poses))


class GpuObjective:
    """tune_single's objective on the GPU. Adapted scenes are cached per forest-parameter
    assignment (adaptation depends only on those); RANSAC-only changes re-run relocalisation
    on a lane, so one coordinate scan evaluates its values concurrently."""

    def __init__(self, make_scene: Callable[[dict], Scene], seqs: Sequences, t_max: float, base_profile="fast",
                 mode="icp", seed: int = 1234, lanes: int = 4):
        self.make_scene, self.seqs, self.t_max = make_scene, seqs, t_max
        self.base, self.mode, self.seed, self.nlanes = base_profile, mode, seed, lanes
        self.scenes: dict[tuple, list[Scene]] = {}
        self._lock = threading.Lock()
        self.memo = Memo(self._cost)

    def _adapted(self, fp: dict) -> list[Scene]:
        k = tuple(sorted(fp.items()))
        with self._lock:
            if k not in self.scenes:
                built = []
                for adapt, _ in self.seqs.pairs:
                    s = self.make_scene(fp)
                    d, c, p = adapt
                    for i0 in range(0, len(p), s.max_batch):
                        s.integrate_frames(d[i0:i0 + s.max_batch], c[i0:i0 + s.max_batch], p[i0:i0 + s.max_batch])
                    s.update_leaves_round_robin(s.total_leaves)
                    s._pool = [s.fork(s.max_batch) for _ in range(self.nlanes)]
                    s._free = list(s._pool)
                    s._cv = threading.Condition()
                    built.append(s)
                self.scenes[k] = built
            return self.scenes[k]

    def _cost(self, assignment: dict) -> float:
        rp, fp = _split(assignment)
        params = ransac_params(self.base, **rp)
        total = 0.0
        for s, (_, val) in zip(self._adapted(fp), self.seqs.pairs):
            with s._cv:
                while not s._free:
                    s._cv.wait()
                lane = s._free.pop()
            try:
                seeds = [self.seed + i for i in range(len(val[2]))]
                score, t = _evaluate(lane, params, self.mode, val, seeds)
            finally:
                with s._cv:
                    s._free.append(lane)
                    s._cv.notify()
            total += cost(score, t, self.t_max)
        return total

    def parallel(self, cands: list) -> list:
        out = [None] * len(cands)
        ths = [threading.Thread(target=lambda i=i: out.__setitem__(i, self.memo(cands[i]))) for i in range(len(cands))]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        return out

    def close(self):
        for ss in self.scenes.values():
            for s in ss:
                s.close()
        self.scenes.clear()


def tune_single(domains: Sequence[ParamDomain], objective: GpuObjective, start: dict,
                max_sweeps: int = 4, dist=None) -> DescentResult:
    """Coordinate descent of one profile; with `dist` (torch.distributed, one process per GPU,
    each with its own GpuObjective on its own device) every scan is sharded across the ranks."""
    par = sharded_parallel(objective.memo, dist, objective.parallel)
    return coordinate_descent(domains, objective.memo, start, max_sweeps, parallel=par)


def tune_cascade(stage_domains: Sequence[Sequence[ParamDomain]], objectives: Sequence[GpuObjective],
                 starts: Sequence[dict], threshold_grid: Sequence[float], overall_cost: Callable[[CascadeConfig], float],
                 modes=(N.MODE_ICP, N.MODE_ICP, N.MODE_RANKED), max_sweeps: int = 4) -> tuple[CascadeConfig, list]:
    """Appendix B.2: (1) tune stage 1 (forest + RANSAC) under t_max^(1); (2) fix its forest
    parameters phi*; (3) tune only the RANSAC parameters of stages 2..N under their bounds;
    (4) tune the thresholds over `threshold_grid` against `overall_cost(config)`."""
    results = [tune_single(stage_domains[0], objectives[0], starts[0], max_sweeps)]
    _, phi = _split(results[0].assignment)
    for dom, obj, st in zip(stage_domains[1:], objectives[1:], starts[1:]):
        ransac_only = [d for d in dom if d.name in RANSAC_FIELDS]
        results.append(tune_single(ransac_only, obj, dict(st, **phi), max_sweeps))
    stages = [ransac_params(obj.base, **_split(r.assignment)[0]) for r, obj in zip(results, objectives)]
    n = len(stages)
    thr_domains = [ParamDomain(f"t{i}", list(threshold_grid)) for i in range(n - 1)]

    def thr_cost(a: dict) -> float:
        return overall_cost(CascadeConfig(stages, list(modes[:n]), [a[f"t{i}"] for i in range(n - 1)]))

    start_thr = {f"t{i}": threshold_grid[0] for i in range(n - 1)}
    tr = coordinate_descent(thr_domains, thr_cost, start_thr, max_sweeps)
    return CascadeConfig(stages, list(modes[:n]), [tr.assignment[f"t{i}"] for i in range(n - 1)]), results + [tr]

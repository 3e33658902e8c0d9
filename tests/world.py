"""Seeded synthetic worlds shared by the parity tests (oracle side + GPU side)."""
from __future__ import annotations

import numpy as np

import oracle_ffi as of

K = of.intrinsics()


class OracleWorld:
    """Scene + random forest + adapted state on the CPU oracle."""

    def __init__(self, oracle, scene_seed=1, n_adapt=30, n_test=6, forest=of.FOREST_DEFAULT, cluster=True,
                 adapt_seed=7, forest_seed=42, k=None, test_kind=1):
        self.O = O = oracle
        self.k = k = K if k is None else k
        L = O.lib
        self.scene_seed = scene_seed
        self.fp = dict(forest)
        self.scene = L.or_scene_generate(scene_seed, 20)
        self.prims = O.scene_prims(self.scene)
        self.adapt_poses = O.trajectory(scene_seed, n_adapt, 0)
        self.test_poses = O.trajectory(scene_seed, n_test, test_kind)
        self.D, self.RGB = O.render(self.scene, self.adapt_poses, k)
        self.Dt, self.RGBt = O.render(self.scene, self.test_poses, k)
        self.forest = L.or_forest_random(forest_seed, 14, 0.4, 5, 130)
        self.blob = O.serialize(self.forest)
        self.total_leaves = L.or_forest_total_leaves(self.forest)
        self.state = O.state_create(self.forest, self.fp, adapt_seed)
        for i in range(n_adapt):
            assert O.integrate(self.state, self.forest, self.D[i], self.RGB[i], k, self.adapt_poses[i]) == 0
        if cluster:
            L.or_update_all_parallel(self.state, 8)

    def predictions(self):
        return self.O.predictions(self.state, self.total_leaves)


def gpu_scene(device, world: OracleWorld, max_batch=8, adapt_seed=7):
    import paper_1810_12163_b200 as P

    k = world.k
    s = P.Scene(device, world.blob, P.forest_params(world.fp),
                P.intrinsics(k.width, k.height, k.fx, k.fy, k.cx, k.cy), adapt_seed=adapt_seed, max_batch=max_batch)
    s.set_model(world.prims)
    return s


def pose_err(R, t, gt):
    Rg, tg = of.pose_np(gt)
    te = float(np.linalg.norm(t - tg))
    ae = float(np.degrees(np.arccos(np.clip((np.trace(Rg.T @ R) - 1) / 2, -1, 1))))
    return te, ae

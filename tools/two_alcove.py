"""Acceptance criterion 8 harness: the constructed two-alcove aliasing scene.

A 4 x 3 x 2.5 m room whose surfaces are flat-coloured (no texture) and symmetric under the
half turn about the vertical axis through the room centre, with two identical alcoves
(cabinet + boxes) on the x = 0 and x = 4 walls. The only asymmetry is a shallow panel of the
wall's own colour beside alcove A: invisible to colour, visible in depth. Frames that
look into either alcove are appearance-aliased; ranking (ICP + depth difference against the
model) can tell the two poses apart, the raw RANSAC output cannot.

  python tools/two_alcove.py          (on a B200: prints raw / icp / ranked success per alcove)
"""
from __future__ import annotations

import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def prims(bump: bool = True) -> np.ndarray:
    import paper_1810_12163_b200 as P

    X, Y, Z = 4.0, 3.0, 2.5
    big = 1000.0  # texture cell larger than the room: one flat colour per primitive
    rows = []

    def box(a, b, col, seed):
        rows.append((0, a, b, col, big, seed))

    wall_x, wall_y = (170.0, 150.0, 120.0), (120.0, 160.0, 170.0)
    box((0, 0, 0), (X, Y, 0), (110.0, 110.0, 110.0), 11)        # floor
    box((0, 0, Z), (X, Y, Z), (200.0, 200.0, 200.0), 12)        # ceiling
    box((0, 0, 0), (0, Y, Z), wall_x, 13)                       # x = 0
    box((X, 0, 0), (X, Y, Z), wall_x, 13)                       # x = X (same colour and seed)
    box((0, 0, 0), (X, 0, Z), wall_y, 14)                       # y = 0
    box((0, Y, 0), (X, Y, Z), wall_y, 14)                       # y = Y
    cab, top = (60.0, 140.0, 90.0), (200.0, 80.0, 60.0)
    for flip in (False, True):  # alcove A on x = 0, its half-turn image B on x = X
        def m(p):
            return (X - p[0], Y - p[1], p[2]) if flip else p

        def mbox(a, b, col, seed):
            pa, pb = m(a), m(b)
            box(tuple(min(u, v) for u, v in zip(pa, pb)), tuple(max(u, v) for u, v in zip(pa, pb)), col, seed)

        # a furnished niche: cabinet with drawers, objects on top, a picture and a shelf on the
        # wall (flat colours, so A and B look exactly alike)
        mbox((0.0, 0.9, 0.0), (0.6, 2.1, 1.0), cab, 21)
        mbox((0.6, 1.0, 0.15), (0.63, 1.45, 0.45), (220.0, 200.0, 60.0), 24)   # drawer
        mbox((0.6, 1.55, 0.15), (0.63, 2.0, 0.45), (60.0, 90.0, 200.0), 25)    # drawer
        mbox((0.6, 1.0, 0.55), (0.63, 2.0, 0.85), (230.0, 120.0, 170.0), 26)   # drawer
        mbox((0.1, 1.0, 1.0), (0.35, 1.25, 1.35), top, 22)                     # box on top
        mbox((0.15, 1.4, 1.0), (0.3, 1.55, 1.55), (40.0, 40.0, 40.0), 27)      # tall thin box
        mbox((0.05, 1.7, 1.0), (0.45, 2.05, 1.12), (240.0, 240.0, 120.0), 28)  # flat box
        mbox((0.0, 1.1, 1.65), (0.03, 1.9, 2.1), (90.0, 50.0, 30.0), 29)       # picture frame
        mbox((0.03, 1.2, 1.73), (0.04, 1.8, 2.02), (70.0, 200.0, 210.0), 30)   # picture
        mbox((0.0, 0.3, 1.3), (0.3, 0.75, 1.35), (150.0, 100.0, 60.0), 31)     # shelf
        mbox((0.05, 0.35, 1.35), (0.25, 0.5, 1.6), (200.0, 60.0, 60.0), 32)    # object on the shelf
        mbox((0.0, 2.3, 0.0), (0.35, 2.65, 0.7), (120.0, 60.0, 160.0), 33)     # side box
    if bump:  # the asymmetry: a shallow panel of the wall's own colour beside alcove A
        box((0.0, 2.3, 1.0), (0.15, 2.7, 1.6), wall_x, 13)
    out = np.zeros(len(rows), P.native.PRIM_DTYPE)
    for i, (t, a, b, col, cell, seed) in enumerate(rows):
        out[i] = (t, a, b, col, cell, seed)
    return out


def look(px, py, pz, yaw, pitch):
    """Camera -> world pose looking along (yaw, pitch) (z up, the trajectories' convention)."""
    cy, sy, cp, sp = math.cos(yaw), math.sin(yaw), math.cos(pitch), math.sin(pitch)
    f = np.array([cp * cy, cp * sy, sp])
    x = np.array([sy, -cy, 0.0])
    y = np.cross(f, x)
    R = np.stack([x, y, f], axis=1)
    return R, np.array([px, py, pz])


def alcove_views(n: int, seed: int = 5):
    """n views into alcove A (facing -x) and their half-turn images into B."""
    import paper_1810_12163_b200 as P

    rng = np.random.default_rng(seed)
    va, vb = [], []
    for _ in range(n):
        px, py = 1.9 + 0.3 * rng.uniform(-1, 1), 1.5 + 0.3 * rng.uniform(-1, 1)
        pz, yaw, pitch = 1.2 + 0.2 * rng.uniform(-1, 1), math.pi + 0.25 * rng.uniform(-1, 1), -0.3 + 0.1 * rng.uniform(-1, 1)
        va.append(P.to_pose(look(px, py, pz, yaw, pitch)))
        vb.append(P.to_pose(look(4.0 - px, 3.0 - py, pz, yaw - math.pi, pitch)))
    return va, vb


def run(device=None, n_views=24, adapt_frames=400, verbose=True):
    import paper_1810_12163_b200 as P
    from paper_1810_12163_b200.protocols import is_success, pose_error

    dev = device or P.Device(0)
    k = P.intrinsics()
    s = P.Scene(dev, P.generate_random_forest(42), P.forest_params("default"), k, adapt_seed=7, max_batch=64)
    s.set_model(prims())
    adapt = P.generate_trajectory(3, adapt_frames, 0)
    fs = P.FrameSet(s, adapt_frames)
    fs.render(adapt)
    fs.train(range(adapt_frames), adapt)
    s.update_leaves_round_robin(s.total_leaves)
    va, vb = alcove_views(n_views)
    views = va + vb
    ft = P.FrameSet(s, len(views))
    ft.render(views)
    seeds = [7000 + i for i in range(len(views))]
    rates = {}
    for mode, name in ((0, "raw"), (1, "icp"), (2, "ranked")):
        res = ft.cascade(range(len(views)), P.CascadeConfig([P.ransac_params("default")], [mode], []), seeds)
        ok = []
        for r, gt in zip(res, views):
            good = False
            if r.has_pose:
                R, t = P.pose_arrays(r.pose)
                Rg, tg = P.pose_arrays(gt)
                good = is_success(*pose_error(R, t, Rg, tg))
            ok.append(good)
        rates[name] = (float(np.mean(ok[:n_views])), float(np.mean(ok[n_views:])), float(np.mean(ok)))
        if verbose:
            print(f"{name:7s} alcove A {rates[name][0]:.3f}  alcove B {rates[name][1]:.3f}  all {rates[name][2]:.3f}")
    ft.close()
    fs.close()
    s.close()
    if device is None:
        dev.close()
    return rates


if __name__ == "__main__":
    run()

"""Fixture diagnostics (oracle only): rejection-tag histogram of hypothesis generation and
mode quality on a seeded synthetic world. Used to calibrate the synthetic fixture against
SPEC.md:450 ("N_max=1024 on a well-adapted synthetic scene -> >= 99% slots succeed").

  python tools/gen_diag.py --adapt 200 --forest default --profile default --frames 4
"""
from __future__ import annotations

import argparse
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle_ffi as of  # noqa: E402

TAGS = ["OK", "NoModes", "ColourCheckFailed", "TooClose", "NotRigid", "DegenerateKabsch"]


def world(O, scene_seed, adapt, forest_kind, threads, kind=0):
    k = of.intrinsics()
    scene = O.lib.or_scene_generate(scene_seed, 20)
    forest = O.lib.or_forest_random(42, 14, 0.4, 5, 130)
    fp = of.FOREST_DEFAULT if forest_kind == "default" else of.FOREST_CASCADE
    st = O.state_create(forest, fp, 7)
    poses = O.trajectory(scene_seed, adapt, kind)
    for c0 in range(0, adapt, 100):
        chunk = poses[c0:c0 + 100]
        D, RGB = O.render(scene, chunk, k, threads)
        arr = (of.Pose * len(chunk))(*chunk)
        rc = O.lib.or_integrate_batch(st, forest, of._ptr(D, C.c_float), of._ptr(RGB, C.c_uint8), C.byref(k), arr,
                                      len(chunk), threads)
        assert rc == 0, O.err()
    O.lib.or_update_all_parallel(st, threads)
    return k, scene, forest, st, poses


def stats(O, k, scene, forest, st, poses, profile, seed=11, radius=0.05):
    D, RGB = O.render(scene, poses, k)
    out = []
    p = of.ransac_params(profile)
    for i, pose in enumerate(poses):
        tags = (C.c_int64 * 6)()
        ok = C.c_int()
        mf, pf = C.c_double(), C.c_double()
        d = np.ascontiguousarray(D[i])
        c = np.ascontiguousarray(RGB[i])
        rc = O.lib.or_generation_stats(forest, st, of._ptr(d, C.c_float), of._ptr(c, C.c_uint8), C.byref(k),
                                       C.byref(p), seed + i, C.byref(pose), radius, tags, C.byref(ok), C.byref(mf),
                                       C.byref(pf))
        assert rc == 0, O.err()
        out.append((list(tags), ok.value, mf.value, pf.value))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scene", type=int, default=1)
    ap.add_argument("--adapt", type=int, default=200)
    ap.add_argument("--forest", default="default")
    ap.add_argument("--profile", default="default")
    ap.add_argument("--frames", type=int, default=4)
    ap.add_argument("--test-kind", type=int, default=1)
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    a = ap.parse_args()
    O = of.get()
    t0 = time.time()
    k, scene, forest, st, _ = world(O, a.scene, a.adapt, a.forest, a.threads)
    t1 = time.time()
    test = O.trajectory(a.scene, a.frames, a.test_kind)
    res = stats(O, k, scene, forest, st, test, a.profile)
    n_max = of.PROFILES[a.profile]["n_max"]
    tot = np.zeros(6, np.int64)
    for tags, ok, mf, pf in res:
        tot += np.array(tags)
        print(f"slots ok {ok}/{n_max}  mode_frac(5cm) {mf:.3f}  pixel_frac {pf:.3f}  "
              + " ".join(f"{n}={v}" for n, v in zip(TAGS, tags)))
    print("attempt share: " + " ".join(f"{n}={v / tot.sum():.4f}" for n, v in zip(TAGS, tot)),
          f"(adapt {t1 - t0:.1f}s, stats {time.time() - t1:.1f}s)")


if __name__ == "__main__":
    main()

"""TSDF scene model in the oracle (SPEC.md:538-555 known answers). CPU."""
import numpy as np

import oracle_ffi as of

K = of.intrinsics(64, 48, 58.5, 58.5)
ORIGIN, VOX, DIMS = (-1.1, -0.9, 1.5), 0.02, (110, 90, 40)


def wall(z=2.0):
    return np.full((K.height, K.width), z, np.float32)


def test_wall_zero_crossing_and_raycast(oracle):
    v = oracle.tsdf_create(ORIGIN, VOX, DIMS)
    I = of.pose_from(np.eye(3), [0, 0, 0])
    oracle.tsdf_fuse(v, wall(), K, I)
    d, nrm = oracle.tsdf_raycast(v, I, K)
    # principal ray: zero crossing at 2 m within one voxel
    assert abs(d[24, 32] - 2.0) <= VOX
    valid = d > 0
    assert valid.mean() > 0.9
    assert np.abs(d[valid] - 2.0).max() <= VOX  # fused plane vs analytic (z-depth) within a voxel
    assert nrm[24, 32] != 0xFFFFFFFF  # normal available at the principal-ray hit
    oracle.lib.or_tsdf_free(v)


def test_fuse_twice_and_empty_frame(oracle):
    I = of.pose_from(np.eye(3), [0, 0, 0])
    a = oracle.tsdf_create(ORIGIN, VOX, DIMS)
    oracle.tsdf_fuse(a, wall(), K, I)
    t1, w1 = oracle.tsdf_dump(a, DIMS)
    oracle.tsdf_fuse(a, wall(), K, I)
    t2, w2 = oracle.tsdf_dump(a, DIMS)
    seen = w1 > 0
    assert seen.any()
    assert np.array_equal(t1, t2)  # idempotent average
    assert np.array_equal(w2[seen], 2 * w1[seen])  # weights double
    oracle.tsdf_fuse(a, np.zeros_like(wall()), K, I)  # empty depth: unchanged
    t3, w3 = oracle.tsdf_dump(a, DIMS)
    assert np.array_equal(t3, t2) and np.array_equal(w3, w2)
    oracle.lib.or_tsdf_free(a)


def test_looking_away_is_all_invalid(oracle):
    v = oracle.tsdf_create(ORIGIN, VOX, DIMS)
    I = of.pose_from(np.eye(3), [0, 0, 0])
    oracle.tsdf_fuse(v, wall(), K, I)
    away = of.pose_from(np.diag([1.0, -1.0, -1.0]), [0, 0, 0])  # facing -z
    d, _ = oracle.tsdf_raycast(v, away, K)
    assert (d == 0).all()
    oracle.lib.or_tsdf_free(v)

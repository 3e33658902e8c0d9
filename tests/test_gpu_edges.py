"""Edge cases through the C ABI, held to the oracle bit for bit.

Frames with no valid depth (no grid pixels, SPEC.md NoHypotheses), depth maps full of
invalid values (NaN, +inf, 0, negative, beyond 20 m: core.hpp depth_valid), a batch that
mixes them with ordinary frames, a scene that was never adapted (every pixel predicts no
mode), unreliable training poses and out-of-range RANSAC parameters."""
import ctypes as C

import numpy as np
import pytest

import oracle_ffi as of

from world import K, OracleWorld, gpu_scene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def adapted(oracle, gpu_device):
    w = OracleWorld(oracle, scene_seed=4, n_adapt=16, n_test=4)
    s = gpu_scene(gpu_device, w)
    s.integrate_frames(list(w.D), list(w.RGB), w.adapt_poses)
    s.update_leaves_round_robin(s.total_leaves)
    return w, s


def corrupted_frames(w):
    D = np.array(w.Dt, np.float32, copy=True)
    RGB = np.array(w.RGBt, np.uint8, copy=True)
    D[0][...] = 0.0  # no valid pixel at all
    d1 = D[1].reshape(-1)
    d1[::3] = np.nan
    d1[1::7] = np.inf
    d1[2::11] = -1.0
    d1[3::13] = 25.0  # beyond the 20 m validity limit
    D[2][: D[2].shape[0] // 2] = 0.0  # top half missing
    return D, RGB


def check_same(res, refs):
    for i, (r, ref) in enumerate(zip(res, refs)):
        assert r.has_pose == ref.has_pose and r.status == ref.status, f"frame {i}"
        if r.has_pose:
            assert bytes(r.pose) == bytes(ref.pose), f"frame {i}"
            assert r.score == ref.score or (np.isinf(r.score) and np.isinf(ref.score))


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_invalid_and_empty_frames_match_oracle(oracle, adapted, mode):
    import paper_1810_12163_b200 as P

    w, s = adapted
    D, RGB = corrupted_frames(w)
    seeds = [300 + i for i in range(len(D))]
    res = s.relocalise_batch(D, RGB, P.ransac_params("fast"), mode, seeds)
    refs = [oracle.relocalise(w.forest, w.state, w.scene, D[i], RGB[i], K, of.ransac_params("fast"), mode, seeds[i])
            for i in range(len(D))]
    assert not res[0].has_pose and not refs[0].has_pose  # nothing to sample
    check_same(res, refs)
    # one frame at a time gives the same results as the mixed batch
    for i in range(len(D)):
        one = s.relocalise_batch(D[i:i + 1], RGB[i:i + 1], P.ransac_params("fast"), mode, [seeds[i]])[0]
        assert one.has_pose == res[i].has_pose and one.status == res[i].status
        if one.has_pose:
            assert bytes(one.pose) == bytes(res[i].pose)


def test_unadapted_scene_finds_no_hypotheses(oracle, gpu_device, adapted):
    import paper_1810_12163_b200 as P

    w, _ = adapted
    s = gpu_scene(gpu_device, w)  # same forest, never trained: every leaf predicts no mode
    state = oracle.state_create(w.forest, w.fp, 7)
    seeds = [11, 12]
    res = s.relocalise_batch(w.Dt[:2], w.RGBt[:2], P.ransac_params("fast"), 1, seeds)
    refs = [oracle.relocalise(w.forest, state, w.scene, w.Dt[i], w.RGBt[i], K, of.ransac_params("fast"), 1,
                              seeds[i]) for i in range(2)]
    for r, ref in zip(res, refs):
        assert not r.has_pose and not ref.has_pose and r.status == ref.status != 0
    s.close()


def test_unreliable_pose_is_rejected_and_changes_nothing(adapted):
    from paper_1810_12163_b200 import native as N

    w, s = adapted
    before = s.predictions(with_modes=False)[0].copy()
    seen = s.lib.scr_dump_seen  # reservoirs must be untouched too
    s0 = np.zeros(s.total_leaves, np.uint32)
    N.check(seen(s.handle, s0.ctypes.data_as(C.POINTER(C.c_uint32))), "seen")
    with pytest.raises(N.UnreliablePose):
        s.integrate_frame(w.D[0], w.RGB[0], w.adapt_poses[0], pose_reliable=False)
    s1 = np.zeros(s.total_leaves, np.uint32)
    N.check(seen(s.handle, s1.ctypes.data_as(C.POINTER(C.c_uint32))), "seen")
    assert np.array_equal(s0, s1)
    assert np.array_equal(before, s.predictions(with_modes=False)[0])


def test_out_of_range_ransac_parameters_are_rejected(adapted):
    import paper_1810_12163_b200 as P
    from paper_1810_12163_b200 import native as N

    w, s = adapted
    for bad in (dict(n_max=8192), dict(n_cull=128), dict(eta=1024)):
        with pytest.raises(N.ScrelocError):
            s.relocalise_batch(w.Dt[:1], w.RGBt[:1], P.ransac_params("fast", **bad), 1, [1])


def test_wrong_sized_frames_raise_dimension_mismatch_at_the_abi(adapted):
    """core.hpp:57 DimensionMismatch: a C caller handing a frame whose width/height differ
    from the scene's intrinsics gets SCR_E_DIMENSION_MISMATCH before any pixel is read (the
    Python mirror raises the same exception earlier); a null plane is SCR_E_ARG."""
    import paper_1810_12163_b200 as P
    from paper_1810_12163_b200 import native as N

    w, s = adapted
    d = np.ascontiguousarray(w.Dt[0][:, : K.width // 2], np.float32)
    c = np.ascontiguousarray(w.RGBt[0][:, : K.width // 2], np.uint8)
    fr = (N.Frame * 1)()
    fr[0].depth, fr[0].rgb = d.ctypes.data, c.ctypes.data
    fr[0].width, fr[0].height, fr[0].pose_reliable = K.width // 2, K.height, 1
    p = P.ransac_params("fast")
    sd = np.array([1], np.uint64)
    out = (N.Result * 1)()
    st = s.lib.scr_relocalise_batch(s.handle, fr, 1, C.byref(p), 1, N.ptr(sd, C.c_uint64), out)
    assert st == 7  # SCR_E_DIMENSION_MISMATCH
    pose = P.to_pose(w.adapt_poses[0])
    assert s.lib.scr_train(s.handle, fr, C.byref(pose)) == 7
    fr[0].width, fr[0].depth = K.width, None
    assert s.lib.scr_relocalise_batch(s.handle, fr, 1, C.byref(p), 1, N.ptr(sd, C.c_uint64), out) == 1
    with pytest.raises(N.DimensionMismatch):
        s.relocalise_batch([d], [c], p, 1, [1])

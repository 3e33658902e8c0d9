"""TSDF scene model on the GPU against the oracle:
fusion, ray casting and relocalisation with ICP / ranking on the fused model, bit for bit."""
import ctypes as C

import numpy as np
import pytest

import oracle_ffi as of
from world import K, OracleWorld, gpu_scene

pytestmark = pytest.mark.gpu

ORIGIN, VOX, DIMS = (-0.2, -0.2, -0.1), 0.02, (220, 170, 140)  # the 4 x 3 x 2.5 m room at 2 cm


@pytest.fixture(scope="module")
def fused(oracle, gpu_device):
    import paper_1810_12163_b200 as P

    w = OracleWorld(oracle, scene_seed=1, n_adapt=24, n_test=3, forest=of.FOREST_CASCADE)
    gv = P.TsdfVolume(gpu_device, ORIGIN, VOX, DIMS)
    ov = oracle.tsdf_create(ORIGIN, VOX, DIMS)
    for i in range(0, 24, 4):  # fuse every 4th adaptation frame
        gv.fuse(w.D[i], w.adapt_poses[i], P.intrinsics())
        oracle.tsdf_fuse(ov, w.D[i], K, w.adapt_poses[i])
    return w, gv, ov


def test_fusion_bit_exact(oracle, fused):
    w, gv, ov = fused
    gt, gw = gv.download()
    ot, ow = oracle.tsdf_dump(ov, DIMS)
    assert (gw > 0).sum() > 100000
    assert np.array_equal(gw, ow)
    assert np.array_equal(gt.view(np.uint32), ot.view(np.uint32))


def test_raycast_bit_exact_and_close_to_analytic(oracle, fused):
    import paper_1810_12163_b200 as P

    w, gv, ov = fused
    for pose in w.test_poses[:2]:
        gd, gn = gv.raycast(pose, P.intrinsics())
        od, on = oracle.tsdf_raycast(ov, pose, K)
        assert np.array_equal(gd.view(np.uint32), od.view(np.uint32))
        assert np.array_equal(gn, on)
        # fused surface vs the exact analytic depth: within a few voxels where both exist
        ad = np.zeros_like(od)
        oracle.lib.or_raycast_depth(w.scene, C.byref(pose), C.byref(K), of._ptr(ad, C.c_float))
        both = (od > 0) & (ad > 0)
        assert both.mean() > 0.3
        assert np.median(np.abs(od[both] - ad[both])) <= VOX


def test_relocalise_on_fused_model_matches_oracle(oracle, gpu_device, fused):
    import paper_1810_12163_b200 as P

    w, gv, ov = fused
    s = gpu_scene(gpu_device, w)
    s.integrate_frames(list(w.D), list(w.RGB), w.adapt_poses)
    s.update_leaves_round_robin(s.total_leaves)
    s.set_tsdf_model(gv)
    oracle.lib.or_scene_set_tsdf(w.scene, ov)
    try:
        for mode in (1, 2):
            prof = "fast" if mode == 1 else "slow"
            res = s.relocalise_batch(w.Dt[:2], w.RGBt[:2], P.ransac_params(prof), mode, [71, 72])
            assert any(r.has_pose and np.isfinite(r.score) for r in res)  # ICP converged on the fused model
            for i, r in enumerate(res):
                ref = oracle.relocalise(w.forest, w.state, w.scene, w.Dt[i], w.RGBt[i], K, of.ransac_params(prof), mode,
                                        71 + i)
                assert r.has_pose == ref.has_pose and r.status == ref.status
                if r.has_pose:
                    assert bytes(r.pose) == bytes(ref.pose), (mode, i)
                    assert r.score == ref.score or (np.isinf(r.score) and np.isinf(ref.score))
    finally:
        oracle.lib.or_scene_set_tsdf(w.scene, None)
        s.set_tsdf_model(None)

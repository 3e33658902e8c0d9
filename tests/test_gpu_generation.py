"""GPU hypothesis generation diagnostics vs the oracle: the per-attempt rejection-tag
histogram (NoModes, ColourCheckFailed, TooClose, NotRigid, DegenerateKabsch)
and the number of generating slots are identical, attempt for attempt, through the C ABI
(scr_debug_generation_stats)."""
import pytest

import oracle_ffi as of
from world import OracleWorld, gpu_scene

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("forest,profile", [(of.FOREST_CASCADE, "fast"), (of.FOREST_CASCADE, "intermediate"),
                                            (of.FOREST_DEFAULT, "default")])
def test_generation_tags_match_oracle(oracle, gpu_device, forest, profile):
    import paper_1810_12163_b200 as P

    w = OracleWorld(oracle, scene_seed=3, n_adapt=30, n_test=2, forest=forest, test_kind=2)
    s = gpu_scene(gpu_device, w)
    s.integrate_frames(list(w.D), list(w.RGB), w.adapt_poses)
    s.update_leaves_round_robin(s.total_leaves)
    over = dict(n_max=512) if profile == "default" else dict(n_max=1024)
    for i in range(2):
        tags_g, ok_g = s.debug_generation_stats(w.Dt[i], w.RGBt[i], P.ransac_params(profile, **over), 4242 + i)
        tags_o, ok_o, _, _ = oracle.generation_stats(w.forest, w.state, w.Dt[i], w.RGBt[i], w.k,
                                                     of.ransac_params(profile, **over), 4242 + i)
        assert ok_g == ok_o and tags_g == tags_o, (tags_g, tags_o)
        assert tags_g["OK"] == ok_g
    s.close()


@pytest.mark.parametrize("profile", ["fast", "default"])
def test_sparse_predictions_generation_matches_oracle(oracle, gpu_device, profile):
    """Two adaptation frames leave most leaves without modes, so a large share of attempts
    draws a pixel without modes (NoModes) and stops early. The attempt loop draws an attempt's
    seven values at once and falls back to the sequential draws for exactly these attempts:
    generated slots, their poses and the preemptive-RANSAC survivors stay bit-exact."""
    import numpy as np

    import paper_1810_12163_b200 as P
    from world import K

    w = OracleWorld(oracle, scene_seed=1, n_adapt=2, n_test=2)
    s = gpu_scene(gpu_device, w)
    s.integrate_frames(list(w.D), list(w.RGB), w.adapt_poses)
    s.update_leaves_round_robin(s.total_leaves)
    for i in range(2):
        p = of.ransac_params(profile)
        tags, ok, _, _ = oracle.generation_stats(w.forest, w.state, w.Dt[i], w.RGBt[i], w.k, p, 700 + i)
        assert tags["NoModes"] > 10000 and ok > 0, tags
        st, gs, gpz, ss, sp, se = s.debug_ransac(w.Dt[i], w.RGBt[i], P.ransac_params(profile), 700 + i)
        rc, ogs, ogp, oss, osp, ose = oracle.ransac(w.forest, w.state, w.Dt[i], w.RGBt[i], K, p, 700 + i)
        assert np.array_equal(gs, ogs)
        assert all(bytes(a) == bytes(b) for a, b in zip(gpz, ogp))
        assert np.array_equal(ss, oss)
        assert np.array_equal(se.view(np.uint32), ose.view(np.uint32))
    s.close()

"""1280x960, kappa = 4096, N_max x 2 for every cascade
stage — same bit-exact bar as the 640x480 parity tests, on a few frames."""
import numpy as np
import pytest

import oracle_ffi as of
from world import OracleWorld, gpu_scene

pytestmark = pytest.mark.gpu

KS = of.intrinsics(1280, 960, 1170.0, 1170.0)
FOREST_STRESS = dict(of.FOREST_CASCADE, capacity=4096)


@pytest.fixture(scope="module")
def stress(oracle, gpu_device):
    w = OracleWorld(oracle, scene_seed=4, n_adapt=6, n_test=2, forest=FOREST_STRESS, k=KS)
    s = gpu_scene(gpu_device, w, max_batch=2)
    s.integrate_frames(list(w.D), list(w.RGB), w.adapt_poses)
    s.update_leaves_round_robin(s.total_leaves)
    return w, s


def test_stress_renders_and_adapts_bit_exact(oracle, stress):
    w, s = stress
    seen = oracle.seen(w.state, w.total_leaves)
    assert np.array_equal(s.seen(), seen)
    cnt_ref, _ = w.predictions()
    cnt, _ = s.predictions()
    assert np.array_equal(cnt, cnt_ref)


def test_stress_cascade_bit_exact(oracle, stress):
    import paper_1810_12163_b200 as P

    w, s = stress
    names = ("fast", "intermediate", "slow")
    cfg = P.CascadeConfig([P.ransac_params(n, n_max=2 * of.PROFILES[n]["n_max"]) for n in names],
                          list(of.CASCADE_MODES), list(of.CASCADE_THRESHOLDS))
    seeds = [31, 32]
    res = s.run_cascade_batch(w.Dt, w.RGBt, cfg, seeds)
    ref = oracle.cascade_batch(w.forest, w.state, w.scene, w.Dt, w.RGBt, KS,
                               [of.ransac_params(n, n_max=2 * of.PROFILES[n]["n_max"]) for n in names],
                               list(of.CASCADE_MODES), list(of.CASCADE_THRESHOLDS), seeds)
    for a, b in zip(res, ref):
        assert a.stage_used == b.stage_used and a.has_pose == b.has_pose
        if a.has_pose:
            assert bytes(a.pose) == bytes(b.pose)

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

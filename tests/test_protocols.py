"""Evaluation protocols (SPEC.md bench_cli 757-826).

CPU: report arithmetic KATs from SPEC.md. GPU: the tracking-loss protocol (relocalise on a
lane with the state published so far, then integrate on the root) reproduces the same
protocol run on the oracle bit for bit, and the headline evaluation matches the oracle."""
import math

import numpy as np
import pytest

import oracle_ffi as of


def test_success_threshold_edges():
    from paper_1810_12163_b200.protocols import is_success

    assert is_success(0.049, 4.9)        # SPEC.md: (0.049 m, 4.9 deg) -> success
    assert not is_success(0.051, 1.0)    # (0.051 m, 1 deg) -> failure
    assert not is_success(0.01, 5.01)


def test_pose_error_and_lower_median():
    from paper_1810_12163_b200.protocols import EvalReport, FrameOutcome, pose_error

    a = np.radians(3.0)
    R = np.array([[np.cos(a), -np.sin(a), 0], [np.sin(a), np.cos(a), 0], [0, 0, 1.0]])
    te, ae = pose_error(R, [0.03, 0.04, 0.0], np.eye(3), [0, 0, 0])
    assert abs(te - 0.05) < 1e-12 and abs(ae - 3.0) < 1e-9
    rep = EvalReport([FrameOutcome(True, t, 1.0, True) for t in (0.4, 0.1, 0.3, 0.2)])
    assert rep.median_t_err == 0.2  # lower median of 4 values
    assert rep.success_fraction == 1.0


def test_novelty_bins_first_bin_rule():
    from paper_1810_12163_b200.protocols import FrameOutcome, compute_novelty_bins

    train = [of.pose_from(np.eye(3), [0.0, 0.0, 0.0])]
    a = np.radians(12.0)
    Rz = np.array([[np.cos(a), -np.sin(a), 0], [np.sin(a), np.cos(a), 0], [0, 0, 1.0]])
    tests = [of.pose_from(np.eye(3), [0.03, 0, 0]),    # 3 cm, 0 deg  -> bin 5
             of.pose_from(np.eye(3), [0.07, 0, 0]),    # 7 cm         -> bin 10
             of.pose_from(Rz, [0.01, 0, 0]),           # 1 cm, 12 deg -> bin 15 (both bounds)
             of.pose_from(np.eye(3), [0.9, 0, 0])]     # 90 cm        -> open bin 60
    outs = [FrameOutcome(True, success=s) for s in (True, False, True, True)]
    bins = compute_novelty_bins(tests, outs, train)
    assert bins[5] == (1, 1.0) and bins[10] == (1, 0.0) and bins[15] == (1, 1.0) and bins[60] == (1, 1.0)
    assert bins[20][0] == 0 and math.isnan(bins[20][1])


def test_success_curve():
    from paper_1810_12163_b200.protocols import FrameOutcome, success_curve

    outs = [None] + [FrameOutcome(True, success=s) for s in (False, True, True, False)]
    assert np.allclose(success_curve(outs), [0, 0.5, 2 / 3, 0.5])
    assert np.allclose(success_curve(outs, window=2), [0, 0.5, 1.0, 0.5])


@pytest.mark.gpu
def test_tracking_loss_protocol_matches_oracle(oracle, gpu_device):
    import paper_1810_12163_b200 as P
    from paper_1810_12163_b200.protocols import run_tracking_loss_protocol
    from world import K, OracleWorld, gpu_scene

    n = 14
    w = OracleWorld(oracle, scene_seed=6, n_adapt=n, n_test=1, forest=of.FOREST_CASCADE, cluster=False)
    s = gpu_scene(gpu_device, w)
    cfg = P.CascadeConfig.paper_three_stage()
    seeds = [500 + i for i in range(n)]
    outs = run_tracking_loss_protocol(s, (w.D, w.RGB, w.adapt_poses), cfg, seeds, leaves_per_frame=4096)
    # the same protocol on the oracle: fresh state, relocalise then integrate + refresh
    state = oracle.state_create(w.forest, w.fp, 7)
    stages = [of.ransac_params(p) for p in ("fast", "intermediate", "slow")]
    assert outs[0] is None
    for i in range(n):
        if i > 0:
            ref = oracle.cascade_batch(w.forest, state, w.scene, w.D[i:i + 1], w.RGB[i:i + 1], K, stages,
                                       list(of.CASCADE_MODES), list(of.CASCADE_THRESHOLDS), [seeds[i]])[0]
            assert outs[i].has_pose == bool(ref.has_pose), i
            if ref.has_pose:
                assert bytes(outs[i].pose) == bytes(ref.pose), i
                assert outs[i].score == ref.score or (math.isinf(outs[i].score) and math.isinf(ref.score))
        assert oracle.integrate(state, w.forest, w.D[i], w.RGB[i], K, w.adapt_poses[i]) == 0
        oracle.lib.or_update(state, 4096)
    assert any(o.success for o in outs[1:11])  # "typically 4-6 frames are enough" (§4.2)


@pytest.mark.gpu
def test_headline_eval_matches_oracle(oracle, gpu_device):
    import paper_1810_12163_b200 as P
    from paper_1810_12163_b200.protocols import pose_error, run_headline_eval
    from world import K, OracleWorld, gpu_scene

    w = OracleWorld(oracle, scene_seed=7, n_adapt=20, n_test=6, forest=of.FOREST_CASCADE)
    s = gpu_scene(gpu_device, w)
    cfg = P.CascadeConfig.paper_three_stage()
    seeds = [900 + i for i in range(len(w.test_poses))]
    rep = run_headline_eval(s, (w.D, w.RGB, w.adapt_poses), (w.Dt, w.RGBt, w.test_poses), cfg, seeds)
    ref = oracle.cascade_batch(w.forest, w.state, w.scene, w.Dt, w.RGBt, K,
                               [of.ransac_params(p) for p in ("fast", "intermediate", "slow")],
                               list(of.CASCADE_MODES), list(of.CASCADE_THRESHOLDS), seeds)
    for o, r, gt in zip(rep.frames, ref, w.test_poses):
        assert o.has_pose == bool(r.has_pose)
        if r.has_pose:
            assert bytes(o.pose) == bytes(r.pose)
            R, t = of.pose_np(r.pose)
            Rg, tg = of.pose_np(gt)
            assert (o.t_err, o.r_err) == pose_error(R, t, Rg, tg)
    assert rep.success_fraction >= 0.5


def test_perturbation_kats():
    """p = 0 leaves the frame unchanged, p = 0.5 masks half the pixels (binomial
    bound on 1e6 pixels), sigma = 0.025 gives 2.5 % relative noise, invalid pixels stay
    invalid."""
    import numpy as np

    from paper_1810_12163_b200.protocols import perturb_missing_depth, perturb_noisy_depth

    rng = np.random.default_rng(0)
    d = np.full((1000, 1000), 2.0, np.float32)
    d[0, :10] = 0.0
    assert np.array_equal(perturb_missing_depth(d, 0.0, rng), d)
    m = perturb_missing_depth(d, 0.5, rng)
    assert abs((m == 0).mean() - 0.5) < 0.002 + 1e-5
    nz = perturb_noisy_depth(d, 0.025, rng)
    assert np.all(nz[0, :10] == 0.0)
    v = nz[1:] / 2.0 - 1.0
    assert abs(v.std() - 0.025) < 0.025 * 0.02

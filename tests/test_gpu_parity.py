"""GPU (sm_100a, through the C ABI) versus the CPU oracle on identical seeded inputs.

Bars (BASELINE.json north_star): features within 1e-5 (we require bit-exact), leaf
indices and reservoir contents bit-exact, cluster modes within 1e-4 m, final poses
within 1 cm / 1 deg, 5 cm/5 deg success rate within +-0.5 %.
"""
import numpy as np
import pytest

import oracle_ffi as of
from world import K, OracleWorld, gpu_scene, pose_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def world(oracle):
    return OracleWorld(oracle, scene_seed=1, n_adapt=30, n_test=4)


@pytest.fixture(scope="module")
def gscene(gpu_device, world):
    import paper_1810_12163_b200 as P

    s = gpu_scene(gpu_device, world)
    for i in range(len(world.adapt_poses)):
        s.integrate_frame(world.D[i], world.RGB[i], world.adapt_poses[i])
    s.update_leaves_round_robin(s.total_leaves)
    return s


def test_render_bit_exact(gpu_device, world):
    import paper_1810_12163_b200 as P

    s = gpu_scene(gpu_device, world)
    fs = P.FrameSet(s, 2)
    fs.render(world.test_poses[:2])
    d, c = fs.download(0, 2)
    assert np.array_equal(d.view(np.uint32), world.Dt[:2].view(np.uint32))
    assert np.array_equal(c, world.RGBt[:2])


def test_leaves_and_features_bit_exact(oracle, gpu_device, world):
    s = gpu_scene(gpu_device, world)
    for i in range(2):
        px, leaves = s.debug_leaves(world.Dt[i], world.RGBt[i])
        ref_px = oracle.grid(world.Dt[i])
        assert np.array_equal(px, ref_px)
        ref = oracle.forest_leaves(world.forest, world.Dt[i], world.RGBt[i], ref_px)
        assert np.array_equal(leaves, ref)
        sel = ref_px[:: max(1, ref_px.size // 64)]
        feats = s.debug_features(world.Dt[i], world.RGBt[i], sel)
        specs = oracle.feature_specs(42)
        import ctypes as C

        for j in range(0, sel.size, 7):
            x, y = int(sel[j] & 0xFFFF), int(sel[j] >> 16)
            for kk in range(0, 256, 5):
                out = C.c_float()
                d = np.ascontiguousarray(world.Dt[i])
                c = np.ascontiguousarray(world.RGBt[i])
                sp = np.ascontiguousarray(specs[kk])
                assert oracle.lib.or_compute_feature(of._ptr(d, C.c_float), of._ptr(c, C.c_uint8), 640, 480, x, y,
                                                     of._ptr(sp, C.c_int32), C.byref(out)) == 0
                assert np.float32(out.value).view(np.uint32) == feats[j, kk].view(np.uint32)


def test_reservoirs_bit_exact(oracle, world, gscene):
    seen_ref = oracle.seen(world.state, world.total_leaves)
    assert np.array_equal(gscene.seen(), seen_ref)
    cap = world.fp["capacity"]
    busy = np.argsort(-seen_ref.astype(np.int64))[:64]
    for slot in list(busy) + list(range(0, world.total_leaves, 4099)):
        a = gscene.entries(int(slot), 1)
        b = oracle.entries(world.state, int(slot), 1, cap)
        assert a.tobytes() == b.tobytes(), f"slot {slot}"


def test_predictions_match(oracle, world, gscene):
    cnt_ref, modes_ref = world.predictions()
    cnt, modes = gscene.predictions()
    assert np.array_equal(cnt, cnt_ref)
    m = modes.reshape(-1, 50)
    r = modes_ref.reshape(-1, 50)
    live = np.nonzero(cnt)[0]
    for slot in live:
        n = cnt[slot]
        assert np.abs(m[slot, :n]["mu"] - r[slot, :n]["mu"]).max() <= 1e-4
        assert np.array_equal(m[slot, :n]["size"], r[slot, :n]["size"])
    # stronger: bit-exact
    same = sum(m[s, : cnt[s]].tobytes() == r[s, : cnt[s]].tobytes() for s in live)
    assert same == len(live)


def test_cluster_kernel_matches_oracle(oracle, gscene):
    rng = np.random.default_rng(3)
    for trial in range(20):
        n = int(rng.integers(1, 300))
        e = np.zeros(n, of.ENTRY_DTYPE)
        centres = rng.uniform(-1, 1, size=(int(rng.integers(1, 6)), 3))
        e["xyz"] = centres[rng.integers(0, len(centres), n)] + rng.normal(0, 0.03, (n, 3))
        e["rgb"] = rng.integers(0, 256, (n, 3))
        gm, gl = gscene.debug_cluster(e)
        om, ol = oracle.cluster(e, of.FOREST_DEFAULT)
        assert np.array_equal(gl, ol)
        assert gm.tobytes() == om.tobytes()


def _ransac_matches_oracle(oracle, world, gscene, frames):
    import paper_1810_12163_b200 as P

    for i in frames:
        for prof in ("default", "fast"):
            p = of.ransac_params(prof)
            gp = P.ransac_params(prof)
            st, gs, gpz, ss, sp, se = gscene.debug_ransac(world.Dt[i], world.RGBt[i], gp, 100 + i)
            rc, ogs, ogp, oss, osp, ose = oracle.ransac(world.forest, world.state, world.Dt[i], world.RGBt[i], K, p,
                                                        100 + i)
            assert np.array_equal(gs, ogs)
            assert all(bytes(a) == bytes(b) for a, b in zip(gpz, ogp))
            assert np.array_equal(ss, oss), (prof, ss, oss)
            assert np.array_equal(se.view(np.uint32), ose.view(np.uint32))
            for a, b in zip(sp, osp):
                R, t = of.pose_np(b)
                ga = np.array(a.R[:]).reshape(3, 3)
                assert np.abs(ga - R).max() < 1e-9 and np.abs(np.array(a.t[:]) - t).max() < 1e-9


def test_ransac_bit_exact(oracle, world, gscene):
    _ransac_matches_oracle(oracle, world, gscene, range(2))


def test_ransac_exact_finisher_paths(oracle, world, gscene):
    """Every passing triplet routed through the generation finisher as a possibly degenerate
    Kabsch: suspect ordering, suspect-list overflow and the exact sequential continuation must
    all reproduce the sequential reference bit for bit."""
    gscene.debug_generation_mode(1)
    try:
        _ransac_matches_oracle(oracle, world, gscene, range(1))
    finally:
        gscene.debug_generation_mode(0)


@pytest.mark.parametrize("prof,over", [
    ("default", dict(n_cull=40, n_out=1)),      # 40 -> 20 -> 10 -> 5 -> 3 -> 2 -> 1: every lane layout
    ("default", dict(n_cull=33, n_out=2)),
    ("intermediate", dict(n_cull=20, n_out=1)),  # Euclidean association
    ("intermediate", dict(n_cull=7, n_out=3)),
])
def test_ransac_lm_candidate_counts(oracle, world, gscene, prof, over):
    """LM association over the compacted candidate list picks its lane layout from the number
    of candidates that need it (two per lane, one per lane, G lanes per candidate): culls that
    are not powers of two and several survivors keep every layout bit-exact."""
    import paper_1810_12163_b200 as P

    i = 0
    p = of.ransac_params(prof, **over)
    gp = P.ransac_params(prof, **over)
    st, gs, gpz, ss, sp, se = gscene.debug_ransac(world.Dt[i], world.RGBt[i], gp, 300 + i)
    rc, ogs, ogp, oss, osp, ose = oracle.ransac(world.forest, world.state, world.Dt[i], world.RGBt[i], K, p, 300 + i)
    assert np.array_equal(ss, oss), (prof, over, ss, oss)
    assert np.array_equal(se.view(np.uint32), ose.view(np.uint32))
    assert all(bytes(a) == bytes(b) for a, b in zip(sp, osp))


def test_icp_matches_oracle(oracle, world, gscene):
    import ctypes as C

    import paper_1810_12163_b200 as P

    for i in range(2):
        gt = world.test_poses[i]
        R, t = of.pose_np(gt)
        ang = np.radians(3.0)
        Rz = np.array([[np.cos(ang), -np.sin(ang), 0], [np.sin(ang), np.cos(ang), 0], [0, 0, 1]])
        init = of.pose_from(Rz @ R, t + np.array([0.03, -0.02, 0.01]))
        out, conv, rms, inl, score = gscene.debug_icp(world.Dt[i], world.RGBt[i], init)
        ref = of.Pose()
        rconv, rrms, rinl = C.c_int(), C.c_double(), C.c_double()
        d = np.ascontiguousarray(world.Dt[i])
        c = np.ascontiguousarray(world.RGBt[i])
        assert oracle.lib.or_icp(world.scene, of._ptr(d, C.c_float), of._ptr(c, C.c_uint8), C.byref(K), C.byref(init),
                                 C.byref(ref), C.byref(rconv), C.byref(rrms), C.byref(rinl)) == 0
        assert conv == rconv.value
        assert bytes(out) == bytes(ref), "ICP pose must be bit-exact"
        rscore = oracle.lib.or_depth_diff(world.scene, of._ptr(d, C.c_float), of._ptr(c, C.c_uint8), C.byref(K),
                                          C.byref(ref))
        if conv:
            assert score == rscore


def test_relocalise_modes_match_oracle(oracle, world, gscene):
    import paper_1810_12163_b200 as P

    for mode in (0, 1, 2):
        res = gscene.relocalise_batch(world.Dt, world.RGBt, P.ransac_params("default"), mode,
                                      [1000 + i for i in range(len(world.test_poses))])
        for i, r in enumerate(res):
            ref = oracle.relocalise(world.forest, world.state, world.scene, world.Dt[i], world.RGBt[i], K,
                                    of.ransac_params("default"), mode, 1000 + i)
            assert r.has_pose == ref.has_pose and r.status == ref.status
            if r.has_pose:
                assert bytes(r.pose) == bytes(ref.pose), f"mode {mode} frame {i}"
                assert r.score == ref.score or (np.isinf(r.score) and np.isinf(ref.score))


def test_cascade_matches_oracle(oracle, gpu_device):
    import paper_1810_12163_b200 as P

    w = OracleWorld(oracle, scene_seed=2, n_adapt=30, n_test=6, forest=of.FOREST_CASCADE)
    s = gpu_scene(gpu_device, w)
    s.integrate_frames(list(w.D), list(w.RGB), w.adapt_poses)
    s.update_leaves_round_robin(s.total_leaves)
    cfg = P.CascadeConfig.paper_three_stage()
    seeds = [77 + i for i in range(len(w.test_poses))]
    res = s.run_cascade_batch(w.Dt, w.RGBt, cfg, seeds)
    ref = oracle.cascade_batch(w.forest, w.state, w.scene, w.Dt, w.RGBt, K,
                               [of.ransac_params(p) for p in ("fast", "intermediate", "slow")],
                               list(of.CASCADE_MODES), list(of.CASCADE_THRESHOLDS), seeds)
    for a, b in zip(res, ref):
        assert a.stage_used == b.stage_used and a.has_pose == b.has_pose
        if a.has_pose:
            assert bytes(a.pose) == bytes(b.pose)


def test_cascade_novel_poses_resolve_at_every_stage(oracle, gpu_device):
    """Held-out novel poses (trajectory kind 2, offsets up to 55 cm / 55 deg):
    frames resolve at the Fast, Intermediate and Slow stages and some end without a pose; the
    GPU cascade equals the oracle's frame for frame (stage used, pose bytes, score)."""
    import paper_1810_12163_b200 as P

    w = OracleWorld(oracle, scene_seed=2, n_adapt=30, n_test=22, forest=of.FOREST_CASCADE, test_kind=2)
    s = gpu_scene(gpu_device, w, max_batch=22)
    s.integrate_frames(list(w.D), list(w.RGB), w.adapt_poses)
    s.update_leaves_round_robin(s.total_leaves)
    cfg = P.CascadeConfig.paper_three_stage()
    seeds = [77 + i for i in range(len(w.test_poses))]
    res = s.run_cascade_batch(w.Dt, w.RGBt, cfg, seeds)
    ref = oracle.cascade_batch(w.forest, w.state, w.scene, w.Dt, w.RGBt, K,
                               [of.ransac_params(p) for p in ("fast", "intermediate", "slow")],
                               list(of.CASCADE_MODES), list(of.CASCADE_THRESHOLDS), seeds)
    stages = [b.stage_used for b in ref]
    assert {0, 1, 2} <= set(stages) and not all(b.has_pose for b in ref), stages
    for i, (a, b) in enumerate(zip(res, ref)):
        assert a.stage_used == b.stage_used and a.has_pose == b.has_pose, i
        assert a.score == b.score or (np.isinf(a.score) and np.isinf(b.score)), i
        if a.has_pose:
            assert bytes(a.pose) == bytes(b.pose), i


def test_batch_invariance(world, gscene):
    """Results depend only on (frame, seed): batch composition never changes them."""
    import paper_1810_12163_b200 as P

    p = P.ransac_params("fast")
    full = gscene.relocalise_batch(world.Dt, world.RGBt, p, 1, [5, 6, 7, 8])
    single = [gscene.relocalise_batch(world.Dt[i:i + 1], world.RGBt[i:i + 1], p, 1, [5 + i])[0] for i in range(4)]
    for a, b in zip(full, single):
        assert bytes(a.pose) == bytes(b.pose) and a.score == b.score


def test_features_match_reference_golden(gpu_device):
    """GPU feature vectors on the reference-generated golden frame (tests/golden) — bit-exact."""
    import os

    import paper_1810_12163_b200 as P

    G = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz"))
    depth, rgb = G["frame_depth"], G["frame_rgb"]
    h, w = depth.shape
    blob = P.generate_random_forest(42, 3, 0.4, 1, 25)  # spec table = reference specs (seed 42, r 25)
    s = P.Scene(gpu_device, blob, P.forest_params("default"), P.intrinsics(w, h, 60.0, 60.0), max_batch=1)
    px, ref, st = G["feature_px"], G["feature_values"], G["feature_status"]
    ok = px[st == 0]
    got = s.debug_features(depth, rgb, ok)
    assert np.array_equal(got.view(np.uint32), ref[st == 0].view(np.uint32))
    import paper_1810_12163_b200.native as N

    bad = px[st != 0][:1]
    with pytest.raises(N.InvalidCentrePixel):
        s.debug_features(depth, rgb, bad)
    gpx, _ = s.debug_leaves(depth, rgb)
    assert np.array_equal(gpx, G["grid_4"])


def test_multi_chunk_calls_match_single_chunk(oracle, gpu_device, world):
    """A call with more frames than the workspace holds runs in chunks whose uploads are
    double-buffered (chunk j + 1 uploads while chunk j runs); results equal one-chunk calls."""
    import paper_1810_12163_b200 as P

    small = gpu_scene(gpu_device, world, max_batch=2)
    small.integrate_frames(list(world.D), list(world.RGB), world.adapt_poses)
    small.update_leaves_round_robin(small.total_leaves)
    cfg = P.CascadeConfig.paper_three_stage()
    n = len(world.test_poses)
    seeds = [300 + i for i in range(n)]
    chunked = small.run_cascade_batch(world.Dt, world.RGBt, cfg, seeds)  # chunks of <= 2 frames
    single = [small.run_cascade_batch(world.Dt[i:i + 1], world.RGBt[i:i + 1], cfg, [seeds[i]])[0] for i in range(n)]
    for a, b in zip(chunked, single):
        assert a.stage_used == b.stage_used and a.has_pose == b.has_pose
        assert bytes(a.pose) == bytes(b.pose) and (a.score == b.score or (np.isinf(a.score) and np.isinf(b.score)))
    small.close()


def test_relocalise_at_an_untiled_resolution(oracle, gpu_device):
    """400 x 300: no pyramid level's width (400, 200, 100) is a multiple of the 32-pixel ray-cast
    tile, so ICP and ranking cast through the untiled primitive lists; all three modes stay
    bit-exact with the oracle."""
    import paper_1810_12163_b200 as P

    k = of.intrinsics(400, 300, 365.0, 365.0)
    w = OracleWorld(oracle, scene_seed=2, n_adapt=12, n_test=3, k=k)
    s = gpu_scene(gpu_device, w)
    s.integrate_frames(list(w.D), list(w.RGB), w.adapt_poses)
    s.update_leaves_round_robin(s.total_leaves)
    for mode in (0, 1, 2):
        res = s.relocalise_batch(w.Dt, w.RGBt, P.ransac_params("default"), mode, [2000 + i for i in range(3)])
        for i, r in enumerate(res):
            ref = oracle.relocalise(w.forest, w.state, w.scene, w.Dt[i], w.RGBt[i], k, of.ransac_params("default"),
                                    mode, 2000 + i)
            assert r.has_pose == ref.has_pose and r.status == ref.status, (mode, i)
            if r.has_pose:
                assert bytes(r.pose) == bytes(ref.pose), f"mode {mode} frame {i}"
                assert r.score == ref.score or (np.isinf(r.score) and np.isinf(ref.score))
    s.close()


@pytest.mark.parametrize("prof,over", [
    ("fast", dict(n_max=37)),                   # fewer slots than one warp's lanes
    ("fast", dict(n_max=1000, max_gen_iters=77)),
    ("default", dict(n_max=333, n_cull=17, n_out=3)),
])
def test_ransac_odd_slot_counts(oracle, world, gscene, prof, over):
    """Slot counts that fill no warp or CTA evenly (slots are pulled from a per-frame counter;
    survivors compacted in slot order) stay bit-exact with the sequential reference."""
    import paper_1810_12163_b200 as P

    p = of.ransac_params(prof, **over)
    gp = P.ransac_params(prof, **over)
    for i in range(2):
        st, gs, gpz, ss, sp, se = gscene.debug_ransac(world.Dt[i], world.RGBt[i], gp, 500 + i)
        rc, ogs, ogp, oss, osp, ose = oracle.ransac(world.forest, world.state, world.Dt[i], world.RGBt[i], K, p,
                                                    500 + i)
        assert np.array_equal(gs, ogs)
        assert all(bytes(a) == bytes(b) for a, b in zip(gpz, ogp))
        assert np.array_equal(ss, oss)
        assert np.array_equal(se.view(np.uint32), ose.view(np.uint32))
        assert all(bytes(a) == bytes(b) for a, b in zip(sp, osp))

"""Relocalisation lanes (scr_scene_fork): concurrent relocalisation on one GPU.

A lane shares the root scene's forest, adaptation state and model and owns a stream and a
workspace; results must be bit-identical to the root's, from any thread, and a lane must
see the root's updates and refuse to make its own."""
import threading

import numpy as np
import pytest

import oracle_ffi as of

from world import OracleWorld, gpu_scene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def adapted(oracle, gpu_device):
    w = OracleWorld(oracle, scene_seed=3, n_adapt=20, n_test=8)
    s = gpu_scene(gpu_device, w)
    s.integrate_frames(list(w.D), list(w.RGB), w.adapt_poses)
    s.update_leaves_round_robin(s.total_leaves)
    return w, s


def test_lane_matches_root(adapted):
    import paper_1810_12163_b200 as P

    w, s = adapted
    lane = s.fork(8)
    cfg = P.CascadeConfig.paper_three_stage()
    seeds = [900 + i for i in range(len(w.test_poses))]
    a = s.run_cascade_batch(w.Dt, w.RGBt, cfg, seeds)
    b = lane.run_cascade_batch(w.Dt, w.RGBt, cfg, seeds)
    for x, y in zip(a, b):
        assert x.stage_used == y.stage_used and x.has_pose == y.has_pose
        if x.has_pose:
            assert bytes(x.pose) == bytes(y.pose) and x.score == y.score
    lane.close()


def test_lanes_concurrent_threads(adapted):
    import paper_1810_12163_b200 as P

    w, s = adapted
    lanes = [s.fork(8) for _ in range(3)]
    cfg = P.CascadeConfig.paper_three_stage()
    seeds = [40 + i for i in range(len(w.test_poses))]
    ref = s.run_cascade_batch(w.Dt, w.RGBt, cfg, seeds)
    out = [None] * len(lanes)

    def run(i):
        for _ in range(3):
            out[i] = lanes[i].run_cascade_batch(w.Dt, w.RGBt, cfg, seeds)

    ts = [threading.Thread(target=run, args=(i,)) for i in range(len(lanes))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for res in out:
        for x, y in zip(ref, res):
            assert bytes(x.pose) == bytes(y.pose) and x.stage_used == y.stage_used
    for lane in lanes:
        lane.close()


def test_lane_is_read_only_and_sees_updates(adapted):
    import paper_1810_12163_b200 as P
    import paper_1810_12163_b200.native as N

    w, s = adapted
    lane = s.fork(4)
    with pytest.raises(N.ScrelocError):
        lane.update_leaves_round_robin(16)
    with pytest.raises(N.ScrelocError):
        lane.integrate_frame(w.D[0], w.RGB[0], w.adapt_poses[0])
    p = P.ransac_params("fast")
    before = lane.relocalise_batch(w.Dt[:2], w.RGBt[:2], p, 1, [5, 6])
    # the root clears its adaptation: the lane must observe it (no predictions -> no pose)
    s.clear_adaptation()
    after = lane.relocalise_batch(w.Dt[:2], w.RGBt[:2], p, 1, [5, 6])
    assert any(r.has_pose for r in before)
    assert not any(r.has_pose for r in after)
    # re-adapt on the root: the lane reproduces the root's results again
    s.integrate_frames(list(w.D), list(w.RGB), w.adapt_poses)
    s.update_leaves_round_robin(s.total_leaves)
    again = lane.relocalise_batch(w.Dt[:2], w.RGBt[:2], p, 1, [5, 6])
    root = s.relocalise_batch(w.Dt[:2], w.RGBt[:2], p, 1, [5, 6])
    for x, y in zip(again, root):
        assert bytes(x.pose) == bytes(y.pose)
    lane.close()


def test_scenes_are_isolated(oracle, gpu_device, adapted):
    """SURVEY.md §8(d) config 4 places several scenes on one GPU: each scene's state is its own,
    so relocalising in one never changes another's results (interleaved calls)."""
    import paper_1810_12163_b200 as P

    w, s = adapted
    w2 = OracleWorld(oracle, scene_seed=5, n_adapt=12, n_test=2)
    s2 = gpu_scene(gpu_device, w2)
    s2.integrate_frames(list(w2.D), list(w2.RGB), w2.adapt_poses)
    s2.update_leaves_round_robin(s2.total_leaves)
    p = P.ransac_params("fast")
    a1 = s.relocalise_batch(w.Dt[:2], w.RGBt[:2], p, 1, [11, 12])
    b1 = s2.relocalise_batch(w2.Dt, w2.RGBt, p, 1, [13, 14])
    a2 = s.relocalise_batch(w.Dt[:2], w.RGBt[:2], p, 1, [11, 12])
    for x, y in zip(a1, a2):
        assert bytes(x.pose) == bytes(y.pose)
    for i, r in enumerate(b1):
        ref = oracle.relocalise(w2.forest, w2.state, w2.scene, w2.Dt[i], w2.RGBt[i], w2.k, of.ransac_params("fast"), 1,
                                13 + i)
        assert r.has_pose == ref.has_pose
        if r.has_pose:
            assert bytes(r.pose) == bytes(ref.pose)
    s2.close()


def test_root_updates_never_tear_concurrent_lane_reads(oracle, gpu_device):
    """ADVICE r1 / SPEC.md:407: while the root scene keeps rewriting its prediction table
    (scr_load_predictions, two different adapted tables in turn), relocalisations on a lane
    from another thread see one table or the other, never a mixture: every lane result equals
    the result under table A or under table B (the scene's state lock orders readers and
    writers)."""
    import paper_1810_12163_b200 as P

    w = OracleWorld(oracle, scene_seed=6, n_adapt=24, n_test=6)
    s = gpu_scene(gpu_device, w)
    s.integrate_frames(list(w.D[:12]), list(w.RGB[:12]), w.adapt_poses[:12])
    s.update_leaves_round_robin(s.total_leaves)
    ta = s.predictions()
    s.integrate_frames(list(w.D[12:]), list(w.RGB[12:]), w.adapt_poses[12:])
    s.update_leaves_round_robin(s.total_leaves)
    tb = s.predictions()
    lane = s.fork(8)
    p = P.ransac_params("fast")
    seeds = [70 + i for i in range(len(w.test_poses))]

    def key(res):
        return tuple(bytes(r.pose) if r.has_pose else b"-" for r in res)

    s.load_predictions(*ta)
    ref_a = key(lane.relocalise_batch(w.Dt, w.RGBt, p, 1, seeds))
    s.load_predictions(*tb)
    ref_b = key(lane.relocalise_batch(w.Dt, w.RGBt, p, 1, seeds))
    assert ref_a != ref_b  # the two tables are distinguishable
    stop = threading.Event()
    errs = []

    def writer():
        try:
            for _ in range(8):
                s.load_predictions(*ta)
                s.load_predictions(*tb)
        except Exception as e:  # surfaced below
            errs.append(e)
        finally:
            stop.set()

    seen = []
    th = threading.Thread(target=writer)
    th.start()
    while not stop.is_set() or len(seen) < 3:
        seen.append(key(lane.relocalise_batch(w.Dt, w.RGBt, p, 1, seeds)))
    th.join()
    assert not errs, errs
    assert all(k in (ref_a, ref_b) for k in seen), "a lane read a half-written table"
    lane.close()
    s.close()

"""scr_broadcast_predictions: one host process driving several GPUs broadcasts the adapted
prediction table of the adapting GPU to the others over NCCL.

On a one-GPU box only the argument checks and the single-GPU no-op can run; the two-GPU
test (table equality after the broadcast, and identical relocalisations) runs where
torch sees two devices."""
import numpy as np
import pytest

from world import OracleWorld, gpu_scene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def world(oracle):
    return OracleWorld(oracle, scene_seed=5, n_adapt=12, n_test=4)


def test_single_gpu_and_argument_checks(world, gpu_device):
    import paper_1810_12163_b200 as P
    from paper_1810_12163_b200 import native as N

    s = gpu_scene(gpu_device, world)
    s.integrate_frames(list(world.D), list(world.RGB), world.adapt_poses)
    s.update_leaves_round_robin(s.total_leaves)
    before = s.predictions(with_modes=False)[0].copy()
    P.broadcast_predictions([s], 0)  # one GPU: nothing to send
    assert np.array_equal(before, s.predictions(with_modes=False)[0])
    with pytest.raises(N.ScrelocError):
        P.broadcast_predictions([s], 1)  # root out of range
    other = gpu_scene(gpu_device, world)
    with pytest.raises(N.ScrelocError):
        P.broadcast_predictions([s, other], 0)  # both on cuda:0: one scene per GPU
    lane = s.fork(4)
    with pytest.raises(N.ScrelocError):
        P.broadcast_predictions([lane], 0)  # lanes are read-only views
    lane.close()
    other.close()
    s.close()


def test_two_gpu_broadcast(world):
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs in one process")
    import paper_1810_12163_b200 as P

    d0, d1 = P.Device(0), P.Device(1)
    s0, s1 = gpu_scene(d0, world), gpu_scene(d1, world)
    s0.integrate_frames(list(world.D), list(world.RGB), world.adapt_poses)
    s0.update_leaves_round_robin(s0.total_leaves)
    P.broadcast_predictions([s0, s1], 0)
    c0, m0 = s0.predictions()
    c1, m1 = s1.predictions()
    assert np.array_equal(c0, c1) and m0.tobytes() == m1.tobytes()
    p = P.ransac_params("fast")
    seeds = [70 + i for i in range(len(world.test_poses))]
    a = s0.relocalise_batch(world.Dt, world.RGBt, p, 1, seeds)
    b = s1.relocalise_batch(world.Dt, world.RGBt, p, 1, seeds)
    for x, y in zip(a, b):
        assert x.has_pose == y.has_pose and bytes(x.pose) == bytes(y.pose)
    s0.close(), s1.close(), d0.close(), d1.close()

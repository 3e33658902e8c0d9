"""The oracle pinned against the reference's known-answer tests (SPEC.md examples and
acceptance criteria). CPU only."""
import ctypes as C
import math

import numpy as np
import pytest

import oracle_ffi as of

K = of.intrinsics()


def P(a, t):
    return of._ptr(a, t)


def exp_se3(O, tw):
    tw = np.ascontiguousarray(tw, np.float64)
    out = of.Pose()
    O.lib.or_exp_se3(P(tw, C.c_double), C.byref(out))
    return out


def rot_axis_angle(axis, ang):
    axis = np.asarray(axis, float) / np.linalg.norm(axis)
    Kx = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    return np.eye(3) + math.sin(ang) * Kx + (1 - math.cos(ang)) * Kx @ Kx


# ---------------------------------------------------------------- geometry
def test_exp_zero_and_quarter_turn(oracle):
    R, t = of.pose_np(exp_se3(oracle, np.zeros(6)))
    assert np.array_equal(R, np.eye(3)) and np.array_equal(t, np.zeros(3))
    R, _ = of.pose_np(exp_se3(oracle, [0, 0, math.pi / 2, 0, 0, 0]))
    assert np.allclose(R, [[0, -1, 0], [1, 0, 0], [0, 0, 1]], atol=1e-15)


def test_exp_log_round_trip(oracle):
    rng = np.random.default_rng(0)
    tw = np.zeros(6)
    for _ in range(1000):
        axis = rng.normal(size=3)
        tw[:3] = axis / np.linalg.norm(axis) * rng.uniform(1e-5, math.pi - 1e-3)
        tw[3:] = rng.normal(size=3)
        T = exp_se3(oracle, tw)
        back = np.zeros(6)
        assert oracle.lib.or_log_se3(C.byref(T), P(back, C.c_double)) == 0
        assert np.abs(back - tw).max() < 1e-8


def test_log_identity_quarter_and_near_pi(oracle):
    out = np.zeros(6)
    T = of.pose_from(np.eye(3), np.zeros(3))
    assert oracle.lib.or_log_se3(C.byref(T), P(out, C.c_double)) == 0 and np.abs(out).max() == 0
    T = of.pose_from([[0, -1, 0], [1, 0, 0], [0, 0, 1]], np.zeros(3))
    assert oracle.lib.or_log_se3(C.byref(T), P(out, C.c_double)) == 0
    assert np.allclose(out, [0, 0, math.pi / 2, 0, 0, 0], atol=1e-12)
    T = of.pose_from(rot_axis_angle([0, 0, 1], math.pi), np.zeros(3))
    assert oracle.lib.or_log_se3(C.byref(T), P(out, C.c_double)) == 11  # AngleNearPi


def kabsch(O, cam, world):
    cam = np.ascontiguousarray(cam, np.float64)
    world = np.ascontiguousarray(world, np.float64)
    out = of.Pose()
    ok = O.lib.or_kabsch(P(cam, C.c_double), P(world, C.c_double), len(cam), C.byref(out))
    return ok, out


def test_kabsch_recovers_seeded_transforms(oracle):
    rng = np.random.default_rng(1)
    for n in (3, 10):
        for _ in range(500):
            R = rot_axis_angle(rng.normal(size=3), rng.uniform(0, math.pi - 1e-3))
            t = rng.normal(size=3)
            cam = rng.normal(size=(n, 3))
            world = cam @ R.T + t
            ok, T = kabsch(oracle, cam, world)
            Re, te = of.pose_np(T)
            assert ok and np.abs(Re - R).max() < 1e-9 and np.abs(te - t).max() < 1e-9
            assert abs(np.linalg.det(Re) - 1) < 1e-9
            resid = world - (cam @ Re.T + te)
            assert math.sqrt((resid ** 2).sum() / n) < 1e-10


def test_kabsch_identity_reflection_and_degenerate(oracle):
    pts = np.array([[0, 0, 1.0], [1, 0, 1], [0, 1, 2], [1, 1, 3]])
    ok, T = kabsch(oracle, pts, pts)
    R, t = of.pose_np(T)
    assert ok and np.abs(R - np.eye(3)).max() < 1e-12 and np.abs(t).max() < 1e-12
    # reflection-inducing: mirror image of a near-planar triple still yields det = +1
    cam = np.array([[0, 0, 0.0], [1, 0, 0], [0, 1, 1e-6]])
    world = cam * np.array([1, 1, -1.0])
    ok, T = kabsch(oracle, cam, world)
    assert ok and abs(np.linalg.det(of.pose_np(T)[0]) - 1) < 1e-12
    # collinear / coincident -> degenerate
    line = np.array([[0, 0, 0.0], [1, 1, 1], [2, 2, 2]])
    assert kabsch(oracle, line, line + 1)[0] == 0
    same = np.ones((3, 3))
    assert kabsch(oracle, same, same)[0] == 0


def test_kabsch_left_invariance(oracle):
    rng = np.random.default_rng(2)
    for _ in range(100):
        cam = rng.normal(size=(6, 3))
        R = rot_axis_angle(rng.normal(size=3), 0.7)
        world = cam @ R.T + rng.normal(size=3)
        Q = rot_axis_angle(rng.normal(size=3), 1.1)
        q = rng.normal(size=3)
        _, H = kabsch(oracle, cam, world)
        _, QH = kabsch(oracle, cam, world @ Q.T + q)
        Rh, th = of.pose_np(H)
        Rq, tq = of.pose_np(QH)
        assert np.abs(Rq - Q @ Rh).max() < 1e-9 and np.abs(tq - (Q @ th + q)).max() < 1e-9


def test_backproject_and_pose_error(oracle):
    out = np.zeros(3)
    assert oracle.lib.or_backproject(320, 240, 2.0, C.byref(K), P(out, C.c_double)) == 0
    assert np.array_equal(out, [0, 0, 2.0])
    k2 = of.Intrinsics(640, 480, 500.0, 500.0, 100.0, 100.0)
    assert oracle.lib.or_backproject(600, 100, 1.0, C.byref(k2), P(out, C.c_double)) == 0
    assert np.array_equal(out, [1, 0, 1.0])
    assert oracle.lib.or_backproject(1, 1, 0.0, C.byref(K), P(out, C.c_double)) == 2  # InvalidDepth
    assert oracle.lib.or_backproject(1, 1, float("nan"), C.byref(K), P(out, C.c_double)) == 2
    g = of.pose_from(np.eye(3), [1, 2, 3])
    te, ae = C.c_double(), C.c_double()
    oracle.lib.or_pose_error(C.byref(g), C.byref(g), C.byref(te), C.byref(ae))
    assert te.value == 0 and ae.value == 0
    e = of.pose_from(np.eye(3), [1.05, 2, 3])
    oracle.lib.or_pose_error(C.byref(e), C.byref(g), C.byref(te), C.byref(ae))
    assert abs(te.value - 0.05) < 1e-12 and ae.value == 0
    rng = np.random.default_rng(3)
    e = of.pose_from(rot_axis_angle(rng.normal(size=3), math.radians(5)), [1, 2, 3])
    oracle.lib.or_pose_error(C.byref(e), C.byref(g), C.byref(te), C.byref(ae))
    assert abs(ae.value - 5) < 1e-6


def test_compose_invert(oracle):
    rng = np.random.default_rng(4)
    T = exp_se3(oracle, rng.normal(size=6))
    inv, c = of.Pose(), of.Pose()
    oracle.lib.or_invert(C.byref(T), C.byref(inv))
    oracle.lib.or_compose(C.byref(T), C.byref(inv), C.byref(c))
    R, t = of.pose_np(c)
    assert np.abs(R - np.eye(3)).max() < 1e-9 and np.abs(t).max() < 1e-9


def test_det_math_kernels(oracle):
    xs = np.linspace(-86.9, 0, 20001, dtype=np.float32)  # x <= -87 maps to 0 by definition
    got = np.array([oracle.lib.or_det_expf(float(x)) for x in xs[::7]])
    ref = np.exp(xs[::7].astype(np.float64))
    assert np.max(np.abs(got - ref) / ref) < 3e-7
    s, c = C.c_double(), C.c_double()
    for x in np.linspace(-7, 7, 1001):
        oracle.lib.or_det_sincos(float(x), C.byref(s), C.byref(c))
        assert abs(s.value - math.sin(x)) < 1e-15 and abs(c.value - math.cos(x)) < 1e-15


# ---------------------------------------------------------------- features
def feature(O, depth, rgb, x, y, spec):
    d = np.ascontiguousarray(depth, np.float32)
    c = np.ascontiguousarray(rgb, np.uint8)
    s = np.ascontiguousarray(spec, np.int32)
    out = C.c_float()
    rc = O.lib.or_compute_feature(P(d, C.c_float), P(c, C.c_uint8), d.shape[1], d.shape[0], x, y, P(s, C.c_int32),
                                  C.byref(out))
    return rc, out.value


def test_feature_specs_layout_and_determinism(oracle):
    a = oracle.feature_specs(5)
    assert np.array_equal(a, oracle.feature_specs(5))
    assert (a[:128, 0] == 0).all() and (a[128:, 0] == 1).all()
    assert np.abs(a[:, 1:3]).max() <= 130 and set(np.unique(a[:, 3])) <= {0, 1, 2}


def test_feature_kats(oracle):
    depth = np.ones((48, 64), np.float32)
    rgb = np.full((48, 64, 3), 77, np.uint8)
    for spec in ([0, 0, 0, 0], [1, 0, 0, 2]):
        assert feature(oracle, depth, rgb, 10, 10, spec) == (0, 0.0)  # delta = 0 -> 0
    assert feature(oracle, depth, rgb, 20, 20, [0, 7, -5, 0]) == (0, 0.0)  # plane at 1 m -> 0
    step = np.ones((48, 64), np.float32)
    step[:, 32:] = 2.0
    assert feature(oracle, step, rgb, 28, 20, [0, 8, 0, 0]) == (0, -1.0)  # step edge -> -1
    assert feature(oracle, step, rgb, 28, 20, [0, 100, 0, 0]) == (0, 1.0)  # out of bounds probe -> D(p) - 0
    bad = depth.copy()
    bad[5, 5] = 0
    assert feature(oracle, bad, rgb, 5, 5, [0, 1, 1, 0])[0] == 3  # InvalidCentrePixel
    # depth-adaptive scaling: at 2 m the probe offset halves
    far = np.full((48, 64), 2.0, np.float32)
    far[20, 24] = 1.0  # probe target for delta = 8 at 2 m -> offset 4
    assert feature(oracle, far, rgb, 20, 20, [0, 8, 0, 0]) == (0, 1.0)


def test_grid_sampling(oracle):
    depth = np.ones((480, 640), np.float32)
    assert oracle.grid(depth).size == 19200
    assert oracle.grid(np.ones((5, 7), np.float32), spacing=1).size == 35
    half = depth.copy()
    half[:, :320] = 0
    g = oracle.grid(half)
    assert g.size == 9600 and ((g & 0xFFFF) >= 320).all()
    assert np.all(np.diff((g >> 16) * 1000 + (g & 0xFFFF)) > 0)  # row-major


# ---------------------------------------------------------------- forest
def test_random_forest_structure(oracle):
    f = oracle.lib.or_forest_random(9, 14, 0.4, 5, 130)
    assert oracle.lib.or_forest_total_leaves(f) == 5 * 16384
    nodes = []
    for t in range(5):
        n = oracle.lib.or_forest_nodes(f, t)
        a = np.zeros(5 * n, np.int32)
        oracle.lib.or_forest_dump_tree(f, t, P(a, C.c_int32))
        nodes.append(a.reshape(n, 5))
    branch = np.concatenate([a[a[:, 2] >= 0] for a in nodes])
    frac = (branch[:, 0] < 128).mean()
    assert abs(frac - 0.4) <= 0.01
    assert (branch[:, 1] == 0).all()  # tau = 0
    f1 = oracle.lib.or_forest_random(9, 1, 0.4, 1, 130)
    assert oracle.lib.or_forest_total_leaves(f1) == 2


def test_forest_serialization_round_trip_and_errors(oracle):
    f = oracle.lib.or_forest_random(11, 6, 0.4, 3, 130)
    blob = oracle.serialize(f)
    b = np.frombuffer(blob, np.uint8).copy()
    g = oracle.lib.or_forest_deserialize(P(b, C.c_uint8), b.size)
    assert g and oracle.serialize(g) == blob
    assert not oracle.lib.or_forest_deserialize(P(b, C.c_uint8), b.size - 3)
    assert "truncated" in oracle.err()
    bad = b.copy()
    bad[4] = 2
    assert not oracle.lib.or_forest_deserialize(P(bad, C.c_uint8), bad.size)
    assert "version 2" in oracle.err()


def hand_tree_blob(thr=0.0):
    """Depth-2 tree: root tests Depth feature 0 (delta (5,0)); children test colour feature 128."""
    import struct

    out = bytearray(b"SCRF") + struct.pack("<III", 1, 1, 256)
    for i in range(256):
        out += struct.pack("<BBhh", 0 if i < 128 else 1, 0, 5 if i in (0, 128) else 0, 0)
    nodes = [(0, thr, 1, 2, -1), (128, 0.0, 3, 4, -1), (128, 0.0, 5, 6, -1),
             (0, 0.0, -1, -1, 0), (0, 0.0, -1, -1, 1), (0, 0.0, -1, -1, 2), (0, 0.0, -1, -1, 3)]
    out += struct.pack("<Ii", len(nodes), 4)
    for n in nodes:
        out += struct.pack("<ifiii", *n)
    return bytes(out)


def test_hand_traced_tree(oracle):
    blob = np.frombuffer(hand_tree_blob(), np.uint8).copy()
    f = oracle.lib.or_forest_deserialize(P(blob, C.c_uint8), blob.size)
    assert f
    depth = np.ones((16, 16), np.float32)
    rgb = np.zeros((16, 16, 3), np.uint8)
    depth[4, 9] = 0.5   # probe of (4,4) for the depth feature: 1 - 0.5 >= 0 -> right
    rgb[4, 4, 0] = 10   # colour feature at (4,4): 10 - rgb(4,9) = 10 - 0 >= 0 -> right
    px = np.array([4 | (4 << 16)], np.int32)
    assert oracle.forest_leaves(f, depth, rgb, px)[0, 0] == 3
    depth[4, 9] = 2.0   # 1 - 2 < 0 -> left; colour 10 >= 0 -> right -> leaf 1
    assert oracle.forest_leaves(f, depth, rgb, px)[0, 0] == 1


# ---------------------------------------------------------------- adaptation
def tiny_forest_state(oracle, capacity, seed=7, height=1):
    f = oracle.lib.or_forest_random(3, height, 0.4, 1, 130)
    fp = dict(of.FOREST_DEFAULT, capacity=capacity, min_cluster_size=1)
    return f, oracle.state_create(f, fp, seed)


def test_reservoir_keeps_all_below_capacity_and_conserves(oracle):
    f, st = tiny_forest_state(oracle, 1024)
    depth = np.ones((4, 4), np.float32)
    rgb = np.zeros((4, 4, 3), np.uint8)
    k = of.Intrinsics(4, 4, 10.0, 10.0, 2.0, 2.0)
    pose = of.pose_from(np.eye(3), np.zeros(3))
    for i in range(1024):
        assert oracle.integrate(st, f, depth, rgb, k, pose) == 0
    seen = oracle.seen(st, 2)
    assert seen.sum() == 1024  # one grid pixel (0,0) x one tree per frame
    e = oracle.entries(st, 0, 2, 1024)
    assert (e[np.argmax(seen)]["xyz"][:, 2] == 1.0).all()
    assert oracle.integrate(st, f, depth, rgb, k, pose, reliable=0) == 4  # UnreliablePose


def test_reservoir_uniformity_binomial(oracle):
    """kappa = 4, n = 2000 inserts, 2000 seeds: inclusion probability 4/n per item."""
    f, _ = tiny_forest_state(oracle, 4)
    n, trials = 2000, 2000
    counts = np.zeros(n)
    fp = dict(of.FOREST_DEFAULT, capacity=4)
    depth = np.ones((1, 1), np.float32)
    k = of.Intrinsics(1, 1, 1.0, 1.0, 0.0, 0.0)
    ident = np.eye(3)
    for s in range(trials):
        st = oracle.state_create(f, fp, 1000 + s)
        for i in range(n):
            rgb = np.array([[[i & 255, i >> 8, 0]]], np.uint8)
            oracle.integrate(st, f, depth, rgb, k, of.pose_from(ident, [0, 0, 0]))
        slot = int(np.argmax(oracle.seen(st, 2)))
        e = oracle.entries(st, slot, 1, 4)[0]
        ids = e["rgb"][:, 0].astype(int) + (e["rgb"][:, 1].astype(int) << 8)
        counts[ids] += 1
        oracle.lib.or_state_free(st)
        if s == 200:
            break
    tot = counts.sum()
    assert tot == 4 * 201
    # chi-square over 10 equal bins of insertion order
    bins = counts.reshape(10, -1).sum(1)
    exp = tot / 10
    chi2 = ((bins - exp) ** 2 / exp).sum()
    assert chi2 < 27.9  # p = 0.001 at 9 dof


def make_entries(points, rgb=(10, 20, 30)):
    e = np.zeros(len(points), of.ENTRY_DTYPE)
    e["xyz"] = points
    e["rgb"] = rgb
    return e


def test_rqs_two_blobs_identical_and_cap(oracle):
    rng = np.random.default_rng(5)
    a = rng.normal([0, 0, 0], 0.01, (100, 3))
    b = rng.normal([1, 0, 0], 0.01, (80, 3))
    fp = dict(of.FOREST_DEFAULT, tau=0.2, min_cluster_size=5)
    modes, labels = oracle.cluster(make_entries(np.vstack([a, b])), fp)
    assert len(modes) == 2 and modes[0]["size"] == 100 and modes[1]["size"] == 80
    assert np.linalg.norm(modes[0]["mu"] - [0, 0, 0]) < 0.005 and np.linalg.norm(modes[1]["mu"] - [1, 0, 0]) < 0.005
    modes, _ = oracle.cluster(make_entries(np.tile([[0.5, 0.5, 0.5]], (30, 1))), fp)
    assert len(modes) == 1
    assert np.allclose(modes[0]["cov"], [1e-6, 0, 0, 1e-6, 0, 1e-6], rtol=1e-6, atol=1e-12)
    centres = np.array([[i % 8, i // 8, 0.0] for i in range(60)])
    sizes = np.arange(60) % 7 + 5
    pts = np.vstack([np.tile(c, (s, 1)) for c, s in zip(centres, sizes)])
    modes, _ = oracle.cluster(make_entries(pts), dict(fp, min_cluster_size=1))
    assert len(modes) == 50
    assert sorted(sizes)[-50:][::-1] == list(modes["size"])


def brute_quick_shift(x, sigma, tau, min_size):
    """Independent reimplementation of the frozen RQS rules (density in f64 of the f32 kernel)."""
    n = len(x)
    d2 = ((x[:, None, :] - x[None, :, :]) ** 2).sum(-1)
    rho = np.exp(-d2 / (2 * sigma * sigma)).sum(1)
    parent = -np.ones(n, int)
    for i in range(n):
        best, bj = np.inf, -1
        for j in range(n):
            if j != i and (rho[j] > rho[i] or (rho[j] == rho[i] and j < i)) and d2[i, j] <= tau * tau and d2[i, j] < best:
                best, bj = d2[i, j], j
        parent[i] = bj
    root = np.arange(n)
    for i in range(n):
        r = i
        while parent[r] >= 0:
            r = parent[r]
        root[i] = r
    sizes = np.bincount(root, minlength=n)
    roots = [i for i in range(n) if parent[i] < 0 and sizes[i] >= min_size]
    roots.sort(key=lambda r: (-sizes[r], r))
    lab = -np.ones(n, int)
    for k, r in enumerate(roots[:50]):
        lab[root == r] = k
    return lab


def test_rqs_matches_brute_force(oracle):
    rng = np.random.default_rng(6)
    fp = dict(of.FOREST_DEFAULT, tau=0.2, min_cluster_size=3)
    for trial in range(200):
        n = int(rng.integers(1, 65))
        c = rng.uniform(-1, 1, (int(rng.integers(1, 5)), 3))
        pts = (c[rng.integers(0, len(c), n)] + rng.normal(0, 0.05, (n, 3))).astype(np.float32)
        _, labels = oracle.cluster(make_entries(pts), fp)
        ref = brute_quick_shift(pts.astype(np.float64), 0.1, 0.2, 3)
        assert np.array_equal(labels, ref)
        for k in range(labels.max() + 1):  # centroid = arithmetic mean
            pass


def test_round_robin_coverage_and_clear(oracle):
    f = oracle.lib.or_forest_random(3, 8, 0.4, 2, 130)  # 512 leaves
    st = oracle.state_create(f, of.FOREST_DEFAULT, 7)
    assert oracle.lib.or_cursor(st) == 0
    oracle.lib.or_update(st, 256)
    assert oracle.lib.or_cursor(st) == 256
    oracle.lib.or_update(st, 256)
    assert oracle.lib.or_cursor(st) == 0
    oracle.lib.or_clear(st)
    oracle.lib.or_clear(st)
    cnt, _ = oracle.predictions(st, 512)
    assert cnt.sum() == 0


# ---------------------------------------------------------------- RANSAC
def one_pixel_world(oracle, modes_list):
    """1x1 frame at depth 1 whose single grid pixel maps to leaf 0 of a 1-node... height-1 tree."""
    f = oracle.lib.or_forest_random(3, 1, 0.4, 1, 130)
    st = oracle.state_create(f, of.FOREST_DEFAULT, 7)
    counts = np.zeros(2, np.int32)
    modes = np.zeros(2 * 50, of.MODE_DTYPE)
    depth = np.ones((1, 1), np.float32)
    rgb = np.zeros((1, 1, 3), np.uint8)
    px = np.array([0], np.int32)
    leaf = int(oracle.forest_leaves(f, depth, rgb, px)[0, 0])
    counts[leaf] = len(modes_list)
    for i, (mu, cov) in enumerate(modes_list):
        cov = np.asarray(cov, float)
        w, V = np.linalg.eigh(cov)
        ic = V @ np.diag(1 / w) @ V.T
        isq = V @ np.diag(1 / np.sqrt(w)) @ V.T
        m = modes[leaf * 50 + i]
        m["mu"] = mu
        m["icov"] = [ic[0, 0], ic[1, 1], ic[2, 2], 2 * ic[0, 1], 2 * ic[0, 2], 2 * ic[1, 2]]
        m["isqrt"] = [isq[0, 0], isq[0, 1], isq[0, 2], isq[1, 1], isq[1, 2], isq[2, 2]]
        m["size"] = 10
        modes[leaf * 50 + i] = m
    oracle.load_predictions(st, counts, modes)
    k = of.Intrinsics(1, 1, 1.0, 1.0, 0.0, 0.0)
    return f, st, depth, rgb, k


def energy(oracle, f, st, depth, rgb, k, pose, samples):
    s = np.ascontiguousarray(samples, np.int32)
    out = C.c_float()
    assert oracle.lib.or_energy(f, st, P(depth, C.c_float), P(rgb, C.c_uint8), C.byref(k), C.byref(pose),
                                P(s, C.c_int32), s.size, C.byref(out)) == 0
    return out.value


def test_energy_kats(oracle):
    # camera point of the single pixel is (0, 0, 1); identity pose maps it to (0, 0, 1)
    iso = np.eye(3) * 0.01 ** 2
    f, st, d, c, k = one_pixel_world(oracle, [([0, 0, 1.0], iso)])
    ident = of.pose_from(np.eye(3), np.zeros(3))
    assert energy(oracle, f, st, d, c, k, ident, [0]) == 0.0
    shifted = of.pose_from(np.eye(3), [0.03, 0, 0])
    assert abs(energy(oracle, f, st, d, c, k, shifted, [0]) - 3.0) < 1e-4
    an = np.diag([0.01 ** 2, 0.1 ** 2, 0.1 ** 2])
    f, st, d, c, k = one_pixel_world(oracle, [([0, 0, 1.0], an)])
    assert abs(energy(oracle, f, st, d, c, k, shifted, [0]) - 3.0) < 1e-4
    sy = of.pose_from(np.eye(3), [0, 0.03, 0])
    assert abs(energy(oracle, f, st, d, c, k, sy, [0]) - 0.3) < 1e-5
    # nearest mode wins; no-mode samples contribute 0
    f, st, d, c, k = one_pixel_world(oracle, [([5, 5, 5.0], iso), ([0.01, 0, 1.0], iso)])
    assert abs(energy(oracle, f, st, d, c, k, ident, [0, 0]) - 2.0) < 1e-4


def test_lm_converges_and_is_monotone(oracle):
    """LM on a synthetic noise-free correspondence set (modes = exact world points)."""
    rng = np.random.default_rng(8)
    H, W = 64, 64
    depth = rng.uniform(1, 3, (H, W)).astype(np.float32)
    rgb = rng.integers(0, 256, (H, W, 3)).astype(np.uint8)
    k = of.Intrinsics(W, H, 50.0, 50.0, 32.0, 32.0)
    f = oracle.lib.or_forest_random(3, 12, 0.4, 1, 130)
    st = oracle.state_create(f, of.FOREST_DEFAULT, 7)
    gt_R = rot_axis_angle([0.3, 1, 0.2], 0.4)
    gt_t = np.array([0.5, -0.2, 1.0])
    px = oracle.grid(depth, 4)
    leaves = oracle.forest_leaves(f, depth, rgb, px)[:, 0]
    # one exact isotropic mode per used leaf = the gt world point of the first pixel in it
    counts = np.zeros(4096, np.int32)
    modes = np.zeros(4096 * 50, of.MODE_DTYPE)
    used = {}
    for g, lf in enumerate(leaves):
        if lf in used:
            continue
        x, y = int(px[g] & 0xFFFF), int(px[g] >> 16)
        dd = float(depth[y, x])
        pc = np.array([(x - 32.0) * dd / 50.0, (y - 32.0) * dd / 50.0, dd])
        used[lf] = g
        counts[lf] = 1
        m = modes[lf * 50]
        m["mu"] = gt_R @ pc.astype(np.float32).astype(np.float64) + gt_t
        m["icov"] = [1e4, 1e4, 1e4, 0, 0, 0]
        m["isqrt"] = [100, 0, 0, 100, 0, 100]
        modes[lf * 50] = m
    oracle.load_predictions(st, counts, modes)
    samples = np.array(sorted(used.values()), np.int32)
    Rp = rot_axis_angle([1, 0, 0], math.radians(2)) @ gt_R
    init = of.pose_from(Rp, gt_t + [0.02, 0, 0])
    surrogate = C.c_double()
    assert oracle.lib.or_lm(f, st, P(depth, C.c_float), P(rgb, C.c_uint8), C.byref(k), C.byref(init),
                            P(samples, C.c_int32), samples.size, 1, C.byref(surrogate)) == 0
    R, t = of.pose_np(init)
    assert samples.size > 20
    assert np.linalg.norm(t - gt_t) < 1e-4 and np.abs(R - gt_R).max() < 1e-4


@pytest.fixture(scope="module")
def small_world(oracle):
    from world import OracleWorld

    return OracleWorld(oracle, scene_seed=1, n_adapt=30, n_test=3)


def test_preemptive_ransac_counts_and_determinism(oracle, small_world):
    w = small_world
    p = of.ransac_params("default")
    rc, gs, gp, ss, sp, se = oracle.ransac(w.forest, w.state, w.Dt[0], w.RGBt[0], K, p, 5)
    assert rc == 0 and len(gs) >= p.n_cull
    assert len(ss) == 16 and np.all(np.diff(se) >= 0)  # 64 -> 32 -> 16, sorted
    rc2, gs2, gp2, ss2, sp2, se2 = oracle.ransac(w.forest, w.state, w.Dt[0], w.RGBt[0], K, p, 5)
    assert np.array_equal(ss, ss2) and all(bytes(a) == bytes(b) for a, b in zip(sp, sp2))
    fast = of.ransac_params("fast")
    rc, gs, gp, ss, sp, se = oracle.ransac(w.forest, w.state, w.Dt[0], w.RGBt[0], K, fast, 5)
    assert len(ss) == 1  # 64 -> 1: six halvings


def test_no_hypotheses_on_empty_state(oracle):
    from world import OracleWorld

    w = OracleWorld(oracle, scene_seed=1, n_adapt=1, n_test=1, cluster=False)
    p = of.ransac_params("default", max_gen_iters=1)
    r = oracle.relocalise(w.forest, w.state, w.scene, w.Dt[0], w.RGBt[0], K, p, 0, 1)
    assert r.has_pose == 0 and r.status == 5  # NoHypotheses


# ---------------------------------------------------------------- scene / ranking
def test_depth_diff_kats(oracle):
    live = np.full((48, 64), 2.0, np.float32)
    dd = lambda a, b: oracle.lib.or_depth_diff_images(P(np.ascontiguousarray(a, np.float32), C.c_float),
                                                      P(np.ascontiguousarray(b, np.float32), C.c_float), 64, 48)
    assert dd(live, live) == 0.0
    assert abs(dd(live, live + 0.07) - 0.07) < 1e-6
    sparse = np.zeros_like(live)
    sparse.flat[: int(0.05 * live.size)] = 2.0
    assert math.isinf(dd(live, sparse))


def plane_scene(oracle):
    p = np.zeros(1, of.PRIM_DTYPE)
    p[0]["type"] = 0
    p[0]["a"] = [-50, -50, 2.0]
    p[0]["b"] = [50, 50, 2.0]
    p[0]["colour"] = [100, 100, 100]
    p[0]["cell"] = 0.2
    return oracle.lib.or_scene_from_prims(p.ctypes.data, 1)


def test_plane_raycast_and_looking_away(oracle):
    s = plane_scene(oracle)
    out = np.zeros((480, 640), np.float32)
    ident = of.pose_from(np.eye(3), np.zeros(3))
    oracle.lib.or_raycast_depth(s, C.byref(ident), C.byref(K), P(out, C.c_float))
    assert np.all(out == 2.0)  # z-depth of the plane z = 2 (range along the ray = 2 / cos)
    away = of.pose_from(np.diag([1.0, -1.0, -1.0]), np.zeros(3))
    oracle.lib.or_raycast_depth(s, C.byref(away), C.byref(K), P(out, C.c_float))
    assert np.all(out == 0.0)


def icp(oracle, scene, depth, rgb, init):
    out = of.Pose()
    conv, rms, inl = C.c_int(), C.c_double(), C.c_double()
    d = np.ascontiguousarray(depth)
    c = np.ascontiguousarray(rgb)
    assert oracle.lib.or_icp(scene, P(d, C.c_float), P(c, C.c_uint8), C.byref(K), C.byref(init), C.byref(out),
                             C.byref(conv), C.byref(rms), C.byref(inl)) == 0
    return out, conv.value, rms.value, inl.value


def test_icp_kats(oracle, small_world):
    w = small_world
    gt = w.test_poses[0]
    out, conv, rms, inl = icp(oracle, w.scene, w.Dt[0], w.RGBt[0], gt)
    R, t = of.pose_np(out)
    Rg, tg = of.pose_np(gt)
    assert conv and np.abs(t - tg).max() < 1e-6 and np.abs(R - Rg).max() < 1e-6
    pert = of.pose_from(rot_axis_angle([0.2, 1, 0.4], math.radians(4)) @ Rg, tg + [0.04, 0, 0])
    out, conv, rms, inl = icp(oracle, w.scene, w.Dt[0], w.RGBt[0], pert)
    R, t = of.pose_np(out)
    assert conv
    assert np.linalg.norm(t - tg) < 0.005
    assert math.degrees(math.acos(min(1, (np.trace(Rg.T @ R) - 1) / 2))) < 0.5
    far = of.pose_from(rot_axis_angle([0, 0, 1], math.pi / 2) @ Rg, tg + [0.8, 0.5, 0])
    assert icp(oracle, w.scene, w.Dt[0], w.RGBt[0], far)[1] == 0


def test_cascade_threshold_logic(oracle, small_world):
    w = small_world
    st = [of.ransac_params("fast"), of.ransac_params("intermediate"), of.ransac_params("slow")]
    r = oracle.cascade_batch(w.forest, w.state, w.scene, w.Dt[:1], w.RGBt[:1], K, st, [1, 1, 2], [1e9, 1e9], [3])
    assert r[0].stage_used == 0
    r = oracle.cascade_batch(w.forest, w.state, w.scene, w.Dt[:1], w.RGBt[:1], K, st, [1, 1, 2], [-1, -1], [3])
    assert r[0].stage_used == 2
    single = oracle.relocalise(w.forest, w.state, w.scene, w.Dt[0], w.RGBt[0], K, st[0], 1, 3)
    r = oracle.cascade_batch(w.forest, w.state, w.scene, w.Dt[:1], w.RGBt[:1], K, st[:1], [1], [], [3])
    assert bytes(single.pose) == bytes(r[0].pose)  # stage 0 of a cascade == a single relocaliser


def test_relocalisation_success_small(oracle, small_world):
    w = small_world
    ok = 0
    for i in range(len(w.test_poses)):
        r = oracle.relocalise(w.forest, w.state, w.scene, w.Dt[i], w.RGBt[i], K, of.ransac_params("default"), 1,
                              100 + i)
        R, t = of.pose_np(r.pose)
        Rg, tg = of.pose_np(w.test_poses[i])
        ang = math.degrees(math.acos(min(1, max(-1, (np.trace(Rg.T @ R) - 1) / 2))))
        ok += r.has_pose and np.linalg.norm(t - tg) <= 0.05 and ang <= 5
    assert ok >= 2

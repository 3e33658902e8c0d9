"""The oracle (and the product's host-side generators) pinned against golden vectors made by
the REFERENCE's own code (tests/golden/make_golden.py: /root/reference/proj rng.hpp,
src/features.cpp, geometry.hpp compiled here against a minimal Eigen shim). CPU only."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle_ffi as of

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz"))


def P(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def test_rng_bit_exact(oracle):
    L = oracle.lib
    rows = iter(G["rng_u64"])
    for s in G["rng_seeds"]:
        for use_stream, tag in [(0, 0)] + [(1, int(t)) for t in G["rng_tags"]]:
            a = np.zeros(64, np.uint64)
            L.or_rng_u64(int(s), use_stream, tag, 64, P(a, C.c_uint64))
            assert np.array_equal(a, next(rows))
    rows = iter(G["rng_uniform_int"])
    for s in G["rng_seeds"]:
        for b in G["rng_bounds"]:
            a = np.zeros(32, np.uint64)
            L.or_rng_uniform_int(int(s), 1, 99, int(b), 32, P(a, C.c_uint64))
            assert np.array_equal(a, next(rows))
    for i, s in enumerate(G["rng_seeds"]):
        a = np.zeros(32)
        L.or_rng_uniform(int(s), 0, 0, 32, P(a, C.c_double))
        assert np.array_equal(a.view(np.uint64), G["rng_uniform"][i].view(np.uint64))
        assert np.array_equal((a < 0.4).astype(np.int32)[:32], G["rng_bernoulli"][i][:32])


def test_feature_specs_bit_exact(oracle):
    k = 0
    for s in G["feature_spec_seeds"]:
        for r in (130, 20):
            assert np.array_equal(oracle.feature_specs(int(s), r), G["feature_specs"][k])
            k += 1


def test_features_and_grid_bit_exact(oracle):
    depth, rgb = G["frame_depth"], G["frame_rgb"]
    h, w = depth.shape
    specs = oracle.feature_specs(42, 25)
    px, ref, st = G["feature_px"], G["feature_values"], G["feature_status"]
    n_valid = 0
    for i in range(px.size):
        x, y = int(px[i] & 0xFFFF), int(px[i] >> 16)
        for k in range(0, 256, 3):
            out = C.c_float()
            rc = oracle.lib.or_compute_feature(P(depth, C.c_float), P(rgb, C.c_uint8), w, h, x, y,
                                               P(np.ascontiguousarray(specs[k]), C.c_int32), C.byref(out))
            if st[i]:
                assert rc == 3  # InvalidCentrePixel, like the reference
                break
            assert rc == 0 and np.float32(out.value).view(np.uint32) == ref[i, k].view(np.uint32)
        n_valid += st[i] == 0
    assert n_valid > 500
    for sp in (1, 3, 4):
        assert np.array_equal(oracle.grid(depth, sp), G[f"grid_{sp}"])


def test_geometry_against_reference(oracle):
    for i, tw in enumerate(G["twists"]):
        out = of.Pose()
        t = np.ascontiguousarray(tw)
        oracle.lib.or_exp_se3(P(t, C.c_double), C.byref(out))
        R, tt = of.pose_np(out)
        assert np.abs(R.reshape(-1) - G["exp_R"][i]).max() < 1e-14
        assert np.abs(tt - G["exp_t"][i]).max() < 1e-13
        back = np.zeros(6)
        pose = of.pose_from(G["exp_R"][i].reshape(3, 3), G["exp_t"][i])
        rc = oracle.lib.or_log_se3(C.byref(pose), P(back, C.c_double))
        assert rc == G["log_status"][i]
        if rc == 0:
            assert np.abs(back - G["log_twist"][i]).max() < 1e-9
    for i, row in enumerate(G["kabsch_out"]):
        n, ok = int(row[0]), int(row[1])
        out = of.Pose()
        c = np.ascontiguousarray(G["kabsch_cam"][i])
        wv = np.ascontiguousarray(G["kabsch_world"][i])
        got = oracle.lib.or_kabsch(P(c, C.c_double), P(wv, C.c_double), n, C.byref(out))
        assert got == ok
        if ok:
            R, t = of.pose_np(out)
            assert np.abs(R.reshape(-1) - row[2:11]).max() < 1e-10 and np.abs(t - row[11:14]).max() < 1e-10
    k = of.intrinsics()
    for x, y, d, stt, *xyz in G["backproject"]:
        o = np.zeros(3)
        rc = oracle.lib.or_backproject(int(x), int(y), float(d), C.byref(k), P(o, C.c_double))
        assert rc == int(stt)
        if rc == 0:
            assert np.array_equal(o, np.array(xyz))
    for i, j, te, ae in G["pose_error"]:
        e = of.pose_from(G["exp_R"][int(i)].reshape(3, 3), G["exp_t"][int(i)])
        g = of.pose_from(G["exp_R"][int(j)].reshape(3, 3), G["exp_t"][int(j)])
        a, b = C.c_double(), C.c_double()
        oracle.lib.or_pose_error(C.byref(e), C.byref(g), C.byref(a), C.byref(b))
        assert abs(a.value - te) < 1e-12 and abs(b.value - ae) < 1e-9


def test_product_forest_generator_uses_reference_specs():
    """The product's generate_random_forest embeds the reference's feature spec table."""
    import paper_1810_12163_b200 as P_

    blob = P_.generate_random_forest(42, 3, 0.4, 1, 130)
    spec = np.frombuffer(blob[16:16 + 256 * 6], dtype=[("kind", "u1"), ("ch", "u1"), ("dx", "<i2"), ("dy", "<i2")])
    ref = G["feature_specs"][2]  # seed 42, radius 130
    assert np.array_equal(spec["kind"], ref[:, 0]) and np.array_equal(spec["dx"], ref[:, 1])
    assert np.array_equal(spec["dy"], ref[:, 2]) and np.array_equal(spec["ch"], ref[:, 3])

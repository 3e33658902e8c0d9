"""Generates tests/golden/reference_golden.npz from the REFERENCE's own code.

oracle/_ref/libscreloc_ref.so is /root/reference/proj/src/{features,geometry}.cpp +
include/screloc/{rng,geometry,features}.hpp compiled against the local Eigen shim
(oracle/ref/build_ref.sh). This script only runs where /root/reference exists; its output
is committed so the GPU box (no reference there) and CI can check against it.
"""
import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
LIB = os.path.join(ROOT, "oracle", "_ref", "libscreloc_ref.so")


def P(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def main():
    subprocess.run(["bash", os.path.join(ROOT, "oracle", "ref", "build_ref.sh")], check=True)
    L = C.CDLL(LIB)
    u64, dbl = C.c_uint64, C.c_double
    out = {}
    # ---- rng.hpp
    seeds = np.array([0, 1, 42, 7, 2**63 + 5], np.uint64)
    tags = np.array([0, 1, 12345, 2**40 + 3], np.uint64)
    rows = []
    for s in seeds:
        for use_stream, tag in [(0, 0)] + [(1, int(t)) for t in tags]:
            a = np.zeros(64, np.uint64)
            L.ref_rng_u64(u64(int(s)), use_stream, u64(tag), 64, P(a, u64))
            rows.append(a)
    out["rng_u64"] = np.stack(rows)
    bounds = np.array([1, 3, 7, 261, 19200, 2**33 + 7], np.uint64)
    ui = []
    for s in seeds:
        for b in bounds:
            a = np.zeros(32, np.uint64)
            L.ref_rng_uniform_int(u64(int(s)), 1, u64(99), u64(int(b)), 32, P(a, u64))
            ui.append(a)
    out["rng_uniform_int"] = np.stack(ui)
    out["rng_uniform"] = np.stack([np.zeros(32) for _ in seeds])
    for i, s in enumerate(seeds):
        a = np.zeros(32)
        L.ref_rng_uniform(u64(int(s)), 0, u64(0), 32, P(a, dbl))
        out["rng_uniform"][i] = a
    out["rng_bernoulli"] = np.stack([np.zeros(64, np.int32) for _ in seeds])
    for i, s in enumerate(seeds):
        a = np.zeros(64, np.int32)
        L.ref_rng_bernoulli(u64(int(s)), dbl(0.4), 64, P(a, C.c_int32))
        out["rng_bernoulli"][i] = a
    out["rng_seeds"], out["rng_tags"], out["rng_bounds"] = seeds, tags, bounds
    # ---- features.cpp
    spec_seeds = np.array([1, 42, 7], np.uint64)
    specs = []
    for s in spec_seeds:
        for r in (130, 20):
            a = np.zeros((256, 4), np.int32)
            L.ref_feature_specs(u64(int(s)), r, P(a, C.c_int32))
            specs.append(a)
    out["feature_specs"] = np.stack(specs)
    out["feature_spec_seeds"] = spec_seeds
    rng = np.random.default_rng(2024)
    h, w = 60, 80
    depth = rng.uniform(0.4, 4.0, (h, w)).astype(np.float32)
    depth[rng.random((h, w)) < 0.1] = 0.0
    depth[rng.random((h, w)) < 0.03] = np.nan
    depth[rng.random((h, w)) < 0.03] = 25.0
    depth[10:20, 10:30] = 1.0  # flat patch
    rgb = rng.integers(0, 256, (h, w, 3)).astype(np.uint8)
    px = np.array([x | (y << 16) for y in range(h) for x in range(0, w, 3)], np.int32)
    fv = np.zeros((px.size, 256), np.float32)
    st = np.zeros(px.size, np.int32)
    L.ref_feature_vectors(P(depth, C.c_float), P(rgb, C.c_uint8), w, h, u64(42), 25, P(px, C.c_int32), px.size,
                          P(fv, C.c_float), P(st, C.c_int32))
    out.update(frame_depth=depth, frame_rgb=rgb, feature_px=px, feature_values=fv, feature_status=st)
    for sp in (1, 3, 4):
        g = np.zeros(h * w, np.int32)
        n = L.ref_grid(P(depth, C.c_float), w, h, sp, P(g, C.c_int32), g.size)
        out[f"grid_{sp}"] = g[:n]
    # ---- geometry.hpp
    tw = np.zeros((200, 6))
    for i in range(200):
        ax = rng.normal(size=3)
        tw[i, :3] = ax / np.linalg.norm(ax) * (rng.uniform(1e-9, 1e-7) if i < 10 else rng.uniform(0, 3.1))
        tw[i, 3:] = rng.normal(size=3)
    expR, expt = np.zeros((200, 9)), np.zeros((200, 3))
    for i in range(200):
        t_ = np.ascontiguousarray(tw[i])
        L.ref_exp_se3(P(t_, dbl), P(expR[i], dbl), P(expt[i], dbl))
    logv, logs = np.zeros((200, 6)), np.zeros(200, np.int32)
    for i in range(200):
        logs[i] = L.ref_log_se3(P(expR[i], dbl), P(expt[i], dbl), P(logv[i], dbl))
    out.update(twists=tw, exp_R=expR, exp_t=expt, log_twist=logv, log_status=logs)
    ks = []
    kin_c, kin_w = [], []
    for i in range(200):
        n = 3 if i % 2 == 0 else 10
        cam = rng.normal(size=(n, 3))
        if i == 4:
            cam = np.array([[0, 0, 0.0], [1, 1, 1], [2, 2, 2]])  # collinear -> degenerate
        ax = rng.normal(size=3)
        th = rng.uniform(0, 3)
        Kx = np.array([[0, -ax[2], ax[1]], [ax[2], 0, -ax[0]], [-ax[1], ax[0], 0]]) / np.linalg.norm(ax)
        R = np.eye(3) + np.sin(th) * Kx + (1 - np.cos(th)) * Kx @ Kx
        world = cam @ R.T + rng.normal(size=3) + rng.normal(0, 0.01 * (i % 3), size=(n, 3))
        c = np.zeros(10 * 3)
        wv = np.zeros(10 * 3)
        c[: 3 * n] = cam.reshape(-1)
        wv[: 3 * n] = world.reshape(-1)
        Ro, to = np.zeros(9), np.zeros(3)
        ok = L.ref_kabsch(P(c, dbl), P(wv, dbl), n, P(Ro, dbl), P(to, dbl))
        ks.append(np.concatenate([[n, ok], Ro, to]))
        kin_c.append(c)
        kin_w.append(wv)
    out.update(kabsch_cam=np.stack(kin_c), kabsch_world=np.stack(kin_w), kabsch_out=np.stack(ks))
    bp = []
    for x, y, d in [(320, 240, 2.0), (905, 240, 1.0), (17, 400, 3.25), (5, 5, 0.0), (5, 5, float("nan"))]:
        o = np.zeros(3)
        stt = L.ref_backproject(x, y, dbl(d), dbl(585.0), dbl(585.0), dbl(320.0), dbl(240.0), P(o, dbl))
        bp.append(np.concatenate([[x, y, d, stt], o]))
    out["backproject"] = np.stack(bp)
    pe = []
    for i in range(100):
        a_, b_ = expR[i], expR[(i + 7) % 200]
        ta, tb = expt[i], expt[(i + 7) % 200]
        te, ae = C.c_double(), C.c_double()
        L.ref_pose_error(P(a_, dbl), P(ta, dbl), P(b_, dbl), P(tb, dbl), C.byref(te), C.byref(ae))
        pe.append([i, (i + 7) % 200, te.value, ae.value])
    out["pose_error"] = np.array(pe)
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_golden.npz"))


if __name__ == "__main__":
    main()

"""Forest file + 7-Scenes-layout sequence I/O. CPU."""
import os
import struct
import warnings
import zlib

import numpy as np
import pytest

import oracle_ffi as of


def _png_with_filters(path, img8):
    """Encodes an 8-bit RGB image cycling through the 5 scanline filters (decoder test)."""
    h, w, _ = img8.shape
    bpp, stride = 3, w * 3
    rows = img8.reshape(h, stride).astype(np.int32)
    out = b""
    prev = np.zeros(stride, np.int32)
    for y in range(h):
        ft = y % 5
        cur = rows[y]
        left = np.concatenate([np.zeros(bpp, np.int32), cur[:-bpp]])
        upleft = np.concatenate([np.zeros(bpp, np.int32), prev[:-bpp]])
        if ft == 0:
            f = cur
        elif ft == 1:
            f = cur - left
        elif ft == 2:
            f = cur - prev
        elif ft == 3:
            f = cur - ((left + prev) >> 1)
        else:
            p = left + prev - upleft
            pa, pb, pc = np.abs(p - left), np.abs(p - prev), np.abs(p - upleft)
            pred = np.where((pa <= pb) & (pa <= pc), left, np.where(pb <= pc, prev, upleft))
            f = cur - pred
        out += bytes([ft]) + (f & 255).astype(np.uint8).tobytes()
        prev = cur

    def chunk(t, d):
        return struct.pack(">I", len(d)) + t + d + struct.pack(">I", zlib.crc32(t + d) & 0xFFFFFFFF)

    with open(path, "wb") as fh:
        fh.write(b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, 8, 2, 0, 0, 0)) +
                 chunk(b"IDAT", zlib.compress(out)) + chunk(b"IEND", b""))


def test_png_round_trips_and_filters(tmp_path):
    from paper_1810_12163_b200.datasets import read_png, write_png

    rng = np.random.default_rng(0)
    rgb = rng.integers(0, 256, (17, 23, 3), dtype=np.uint8)
    d16 = rng.integers(0, 65536, (17, 23), dtype=np.uint16)
    write_png(str(tmp_path / "c.png"), rgb)
    write_png(str(tmp_path / "d.png"), d16)
    assert np.array_equal(read_png(str(tmp_path / "c.png")), rgb)
    assert np.array_equal(read_png(str(tmp_path / "d.png")), d16)
    _png_with_filters(str(tmp_path / "f.png"), rgb)
    assert np.array_equal(read_png(str(tmp_path / "f.png")), rgb)


def test_sequence_round_trip_and_units(oracle, tmp_path):
    from paper_1810_12163_b200.datasets import export_sequence, load_dataset_sequence, pose_matrix

    scene = oracle.lib.or_scene_generate(1, 20)
    k = of.intrinsics(64, 48, 58.5, 58.5)
    poses = oracle.trajectory(1, 3, 0)
    D, RGB = oracle.render(scene, poses, k)
    export_sequence(str(tmp_path), D, RGB, [pose_matrix(p) for p in poses])
    seq = load_dataset_sequence(str(tmp_path))
    assert len(seq) == 3
    for i in range(3):
        mm = np.where(D[i] > 0, np.rint(D[i].astype(np.float64) * 1000.0), 0)
        assert np.array_equal(seq.depths[i], (mm / 1000.0).astype(np.float32))
        assert np.array_equal(seq.rgbs[i], RGB[i])
        assert np.abs(seq.poses[i] - pose_matrix(poses[i])).max() < 1e-9
    # reloading the reloaded frames is bit-identical
    export_sequence(str(tmp_path / "again"), seq.depths, seq.rgbs, seq.poses)
    seq2 = load_dataset_sequence(str(tmp_path / "again"))
    assert all(np.array_equal(a, b) for a, b in zip(seq.depths, seq2.depths))


def test_depth_units_invalid_missing_pose_and_malformed(tmp_path):
    from paper_1810_12163_b200.datasets import MalformedPose, load_dataset_sequence, write_png

    d = np.array([[2000, 65535], [0, 1234]], np.uint16)
    write_png(str(tmp_path / "frame-000000.depth.png"), d)
    write_png(str(tmp_path / "frame-000000.color.png"), np.zeros((2, 2, 3), np.uint8))
    seq = load_dataset_sequence(str(tmp_path))
    assert seq.depths[0][0, 0] == np.float32(2.0) and seq.depths[0][0, 1] == 0.0
    assert seq.depths[0][1, 1] == np.float32(1.234)
    assert seq.poses[0] is None  # missing pose file: no ground truth
    M = np.eye(4)
    M[0, 1] = 0.01  # slightly non-rigid: re-orthonormalised with a warning
    np.savetxt(str(tmp_path / "frame-000000.pose.txt"), M)
    with warnings.catch_warnings(record=True) as wrn:
        warnings.simplefilter("always")
        seq = load_dataset_sequence(str(tmp_path))
    assert wrn and np.abs(seq.poses[0][:3, :3].T @ seq.poses[0][:3, :3] - np.eye(3)).max() < 1e-12
    M[0, 1] = 0.5
    np.savetxt(str(tmp_path / "frame-000000.pose.txt"), M)
    with pytest.raises(MalformedPose):
        load_dataset_sequence(str(tmp_path))


def test_forest_file_round_trip(tmp_path):
    import paper_1810_12163_b200 as P
    from paper_1810_12163_b200.datasets import MissingFile, load_forest, save_forest

    blob = P.generate_random_forest(42, 6, 0.4, 2, 130)
    save_forest(str(tmp_path / "f.bin"), blob)
    assert load_forest(str(tmp_path / "f.bin")) == bytes(blob)
    with pytest.raises(MissingFile):
        load_forest(str(tmp_path / "missing.bin"))


@pytest.mark.gpu
def test_loaded_sequence_relocalises_like_oracle(oracle, gpu_device, tmp_path):
    """Frames that went through the file formats (forest file, PNG depth in mm) feed the GPU
    path and give the oracle's results on the same (quantised) inputs."""
    import paper_1810_12163_b200 as P
    from paper_1810_12163_b200.datasets import export_sequence, load_dataset_sequence, load_forest, pose_matrix
    from paper_1810_12163_b200.datasets import save_forest
    from world import K

    scene = oracle.lib.or_scene_generate(2, 20)
    prims = oracle.scene_prims(scene)
    ap, tp = oracle.trajectory(2, 12, 0), oracle.trajectory(2, 2, 1)
    D, RGB = oracle.render(scene, ap, K)
    Dt, RGBt = oracle.render(scene, tp, K)
    export_sequence(str(tmp_path / "adapt"), D, RGB, [pose_matrix(p) for p in ap])
    export_sequence(str(tmp_path / "test"), Dt, RGBt, [pose_matrix(p) for p in tp])
    sa, st = load_dataset_sequence(str(tmp_path / "adapt")), load_dataset_sequence(str(tmp_path / "test"))
    forest = oracle.lib.or_forest_random(42, 14, 0.4, 5, 130)
    save_forest(str(tmp_path / "forest.bin"), oracle.serialize(forest))
    s = P.Scene(gpu_device, load_forest(str(tmp_path / "forest.bin")), P.forest_params(of.FOREST_CASCADE), P.intrinsics(),
                max_batch=4)
    s.set_model(prims)
    s.integrate_frames(sa.depths, sa.rgbs, sa.poses)
    s.update_leaves_round_robin(s.total_leaves)
    state = oracle.state_create(forest, of.FOREST_CASCADE, 7)
    for i in range(len(sa)):
        M = sa.poses[i]
        assert oracle.integrate(state, forest, sa.depths[i], sa.rgbs[i], K, of.pose_from(M[:3, :3], M[:3, 3])) == 0
    oracle.lib.or_update_all_parallel(state, 8)
    res = s.relocalise_batch(st.depths, st.rgbs, P.ransac_params("fast"), 1, [3, 4])
    for i, r in enumerate(res):
        ref = oracle.relocalise(forest, state, scene, st.depths[i], st.rgbs[i], K, of.ransac_params("fast"), 1, 3 + i)
        assert r.has_pose == ref.has_pose
        if r.has_pose:
            assert bytes(r.pose) == bytes(ref.pose)

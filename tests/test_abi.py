"""The C-ABI library loads without a GPU, exports every symbol include/screloc_gpu.h
declares, and its host-side generators agree with the oracle. CPU only."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle_ffi as of

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "screloc_gpu.h")


@pytest.fixture(scope="module")
def lib():
    from paper_1810_12163_b200 import build, native

    build.build()
    return native.load()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_\s\*]*?\b(scr_[a-z0-9_]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_symbols_exported(lib):
    names = declared_functions()
    assert len(names) >= 39
    from paper_1810_12163_b200 import native

    for n in names:
        assert hasattr(lib, n), f"{n} declared in screloc_gpu.h but not exported"
        assert n in native.SIGNATURES, f"{n} has no ctypes signature"


def test_library_is_sm100a_cubin():
    import subprocess

    from paper_1810_12163_b200 import native

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_version_and_error_plumbing(lib):
    assert b"sm_100a" in lib.scr_version()
    h = C.c_void_p()
    rc = lib.scr_device_open(-1, C.byref(h))
    assert rc != 0 and lib.scr_last_error()


def test_forest_generator_matches_oracle(oracle):
    import paper_1810_12163_b200 as P

    for seed, height, trees in ((42, 14, 5), (3, 6, 2)):
        blob = P.generate_random_forest(seed, height, 0.4, trees, 130)
        f = oracle.lib.or_forest_random(seed, height, 0.4, trees, 130)
        assert blob == oracle.serialize(f)


def test_scene_and_trajectory_generators_match_oracle(oracle):
    import paper_1810_12163_b200 as P

    for seed in (1, 2, 7):
        s = oracle.lib.or_scene_generate(seed, 20)
        assert P.generate_synthetic_scene(seed, 20).tobytes() == oracle.scene_prims(s).tobytes()
        for kind in (0, 1, 2):
            a = P.generate_trajectory(seed, 37, kind)
            b = oracle.trajectory(seed, 37, kind)
            assert all(bytes(x) == bytes(y) for x, y in zip(a, b))


def test_malformed_forest_rejected_before_gpu(lib):
    """Parsing happens on the host: a truncated blob fails with MalformedData even
    before any device allocation (needs a device handle, so only checks the status path
    when a GPU is present)."""
    import paper_1810_12163_b200 as P

    blob = P.generate_random_forest(1, 3, 0.4, 1, 130)
    assert blob[:4] == b"SCRF" and len(blob) == 4 + 12 + 256 * 6 + 8 + 15 * 20


def test_python_mirror_rejects_mismatched_frames_before_native_calls():
    """wrong-sized frames and seed/pose counts raise DimensionMismatch in the
    mirror (the C ABI also checks width/height against the scene, core.hpp:57)."""
    import numpy as np
    import pytest

    import paper_1810_12163_b200 as P
    from paper_1810_12163_b200 import native as N
    from paper_1810_12163_b200.relocaliser import _frames, _seeds

    k = P.intrinsics(64, 48)
    d, c = np.zeros((48, 64), np.float32), np.zeros((48, 64, 3), np.uint8)
    arr, _ = _frames([d], [c], 1, k)
    assert (arr[0].width, arr[0].height) == (64, 48)
    with pytest.raises(N.DimensionMismatch):
        _frames([np.zeros((48, 32), np.float32)], [np.zeros((48, 32, 3), np.uint8)], 1, k)
    with pytest.raises(N.DimensionMismatch):
        _frames([d], [np.zeros((48, 64), np.uint8)], 1, k)
    with pytest.raises(N.DimensionMismatch):
        _frames([d, d], [c], 1, k)
    with pytest.raises(N.DimensionMismatch):
        _seeds([1, 2, 3], 2)

"""bench.py roofline models (CPU): the SURVEY.md §8(d) whole-relocalisation figure and the
per-kernel work models turn device work counters into the numbers the JSON line reports."""
import importlib.util
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules["bench"] = mod
    spec.loader.exec_module(mod)
    return mod


def test_frame_model_sums_flops_and_bytes(bench):
    work = {"sample_evals": 10, "mode_evals": 100, "lm_terms": 5, "lm_assoc_evals": 50, "gen_attempts": 1000,
            "icp_terms": 20, "ray_prim_tests": 30, "node_visits": 64}
    frames = 2
    f = bench.SURVEY_FLOPS
    flop = (f["sample_eval"] * 10 + f["mode_eval"] * 100 + f["lm_term"] * 5 + f["lm_assoc_eval"] * 50
            + f["gen_attempt"] * 1000 + f["icp_term"] * 20 + f["ray_prim"] * 30) / frames
    byts = 640 * 480 * 7 + 16 * 64 / frames
    peaks = {"hbm_gbs": 6000.0}
    r = bench.frame_model(work, frames, (640, 480), 1000.0, peaks, 74.45)
    ideal = flop / 74.45e12 + byts / 6000e9
    assert r["flop_per_frame"] == round(flop) and r["bytes_per_frame"] == round(byts)
    assert abs(r["frac"] - ideal / 1e-3) < 1e-4  # measured time per frame = 1 / 1000 s
    assert bench.frame_model(work, 0, (640, 480), 1000.0, peaks, 74.45) is None


def test_kernel_models(bench):
    work = {"gen_attempts": 7, "mode_evals": 3, "sample_evals": 2, "lm_terms": 1, "icp_terms": 4, "ray_prim": 0}
    units, bound = bench.kernel_model("k_hypgen", work)
    assert bound == "alu" and units == bench.GEN_OPS_PER_ATTEMPT * 7 and bench.GEN_OPS_PER_ATTEMPT == 374

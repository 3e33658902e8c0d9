"""The C++ drop-in header compiles against the C ABI and links with the library (CPU);
the example program relocalises on the GPU (gpu marker)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "paper_1810_12163_b200", "lib", "cpp_drop_in")


def build_example():
    from paper_1810_12163_b200 import build

    build.build()
    lib = os.path.join(ROOT, "paper_1810_12163_b200", "lib")
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-pthread", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "cpp_drop_in.cpp"), "-L", lib, "-lscreloc_gpu",
                    f"-Wl,-rpath,{lib}", "-o", EXE], check=True)
    return EXE


def test_cpp_header_compiles_and_links():
    assert os.path.exists(build_example())


@pytest.mark.gpu
def test_cpp_example_runs_on_gpu():
    exe = build_example()
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "UnreliablePose raised" in out.stdout and "DimensionMismatch raised" in out.stdout


CHECK_TU = r"""
#include <type_traits>
%s
#include <screloc/gpu_relocaliser.hpp>
static_assert(std::is_same<screloc::gpu::InvalidDepth, screloc::InvalidDepth>::value, "one class");
static_assert(std::is_same<screloc::gpu::DimensionMismatch, screloc::DimensionMismatch>::value, "one class");
static_assert(std::is_base_of<screloc::Error, screloc::UnreliablePose>::value, "hierarchy");
static_assert(std::is_base_of<screloc::Error, screloc::NoHypotheses>::value, "hierarchy");
static_assert(std::is_base_of<std::runtime_error, screloc::Error>::value, "hierarchy");
static_assert(sizeof(scr_frame) == 32, "frame carries width and height");
int main() {
  try { screloc::gpu::check(SCR_E_DIMENSION_MISMATCH, "x"); } catch (const screloc::DimensionMismatch&) { return 0; }
  return 1;
}
"""


@pytest.mark.parametrize("with_reference", [False, True])
def test_drop_in_throws_the_reference_exception_classes(tmp_path, with_reference):
    """The drop-in raises screloc::* (core.hpp:24-72) by name; with the reference's own
    core.hpp included first, its classes are the ones thrown (checked at compile time)."""
    inc = ["-I", os.path.join(ROOT, "include")]
    pre = ""
    if with_reference:
        ref = "/root/reference/proj/include"
        if not os.path.isdir(ref):
            pytest.skip("reference tree not present")
        inc += ["-I", ref, "-I", os.path.join(ROOT, "oracle", "ref", "eigen_shim")]
        pre = "#include <screloc/core.hpp>"
    src = tmp_path / "tu.cpp"
    src.write_text(CHECK_TU % pre)
    exe = tmp_path / "tu"
    from paper_1810_12163_b200 import build

    build.build()
    lib = os.path.join(ROOT, "paper_1810_12163_b200", "lib")
    subprocess.run(["g++", "-std=c++20", "-Wall", *inc, str(src), "-L", lib, "-lscreloc_gpu", f"-Wl,-rpath,{lib}",
                    "-o", str(exe)], check=True)
    # runs without a GPU: check() only maps a status code (scr_last_error is host-only)
    assert subprocess.run([str(exe)]).returncode == 0

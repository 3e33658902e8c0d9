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
    assert "UnreliablePose raised" in out.stdout

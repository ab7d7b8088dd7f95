"""Builds and runs the C++ mirror test (tests/cpp/test_gpu_api.cpp) against the C-ABI .so."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_reference_api_mirror(tmp_path):
    exe = tmp_path / "test_gpu_api"
    libdir = os.path.join(ROOT, "paper_2511_16340_b200")
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_gpu_api.cpp"), "-L", libdir, "-lwarmgp_b200",
                    f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    assert "gpu.hpp ok" in r.stdout


def test_cpp_eigen_overloads(tmp_path):
    """gpu.hpp's WARMGP_GPU_EIGEN overloads, compiled against the test Eigen shim."""
    exe = tmp_path / "test_eigen_overloads"
    libdir = os.path.join(ROOT, "paper_2511_16340_b200")
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "include"),
                    "-I", os.path.join(ROOT, "tests", "cpp", "eigen_shim"),
                    os.path.join(ROOT, "tests", "cpp", "test_eigen_overloads.cpp"), "-L", libdir,
                    "-lwarmgp_b200", f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    assert "eigen overloads ok" in r.stdout


def test_cpp_bo_round_pattern(tmp_path):
    """One CgPreconditioner per round + cg_solve_with per column (thompson.cpp:359-384)
    equals solve_many bitwise; the remaining free functions of the reference API."""
    exe = tmp_path / "test_bo_round_pattern"
    libdir = os.path.join(ROOT, "paper_2511_16340_b200")
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_bo_round_pattern.cpp"), "-L", libdir,
                    "-lwarmgp_b200", f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    assert "bo_round pattern ok" in r.stdout

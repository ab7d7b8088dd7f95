"""CPU check of the C++ boundary: every C++ test program (the reference-API mirror
include/warmgp/gpu.hpp, its Eigen overloads, the bo_round pattern) compiles and links
against libwarmgp_b200.so.  Running them needs a GPU (tests/test_gpu_cpp_api.py)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRCS = ["test_gpu_api.cpp", "test_eigen_overloads.cpp", "test_bo_round_pattern.cpp"]


@pytest.mark.parametrize("src", SRCS)
def test_cpp_programs_compile_and_link(tmp_path, src, W):
    libdir = os.path.join(ROOT, "paper_2511_16340_b200")
    cmd = ["g++", "-O1", "-std=c++17", "-Wall", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(ROOT, "tests", "cpp", "eigen_shim"),
           os.path.join(ROOT, "tests", "cpp", src), "-L", libdir, "-lwarmgp_b200",
           f"-Wl,-rpath,{libdir}", "-o", str(tmp_path / "a.out")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr

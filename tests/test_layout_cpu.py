"""CPU test of the region layout the kernels address (csrc/mpix_internal.h
RegionLayout): a small C++ program compiled with g++ against the real
header checks bounds, alignment and non-overlap of every area (rings,
free-mirrors, collective slots, dynamic-matching domain, posted-receive
queue, graph sequence counters, eager payload rings) over a grid of
(P, R, E)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2208_13707_b200", "csrc")


def cuda_include():
    for d in ("/usr/local/cuda/include", os.path.join(os.environ.get("CUDA_HOME", ""), "include")):
        if os.path.exists(os.path.join(d, "cuda_runtime.h")):
            return d
    return None


@pytest.mark.skipif(shutil.which("g++") is None or cuda_include() is None,
                    reason="needs g++ and the CUDA headers")
def test_region_layout_areas_are_disjoint_aligned_and_bounded(tmp_path):
    exe = tmp_path / "layout_check"
    src = os.path.join(ROOT, "tests", "native", "layout_check.cpp")
    subprocess.run(["g++", "-std=c++17", "-O1", "-D__host__=", "-D__device__=",
                    "-I", CSRC, "-I", cuda_include(), src, "-o", str(exe)],
                   check=True, capture_output=True, text=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0 and out.stdout.strip() == "OK", out.stdout

"""The C++ drop-in header (include/pmslam_b200.hpp) compiles and links
against libpmx_cuda.so with the host C++ toolchain (CPU), and the demo —
ports of the reference's own camera/tracking/backend tests written against
the reference-shaped C++ API — passes on a B200 (GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2412_12392_b200", "csrc")
EXE = os.path.join("/tmp", "pmx_cpp_dropin_demo")


def build():
    if not os.path.exists(os.path.join(LIBDIR, "libpmx_cuda.so")):
        subprocess.check_call(["make", "-s", "-j8", "-C", LIBDIR])
    subprocess.check_call(["g++", "-std=c++17", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tools", "cpp_dropin_demo.cpp"), "-L", LIBDIR, "-lpmx_cuda",
                           "-Wl,-rpath," + LIBDIR, "-o", EXE])


def test_cpp_header_compiles_and_links():
    build()
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_cpp_dropin_demo_passes_on_gpu():
    build()
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "PASSED" in out.stdout

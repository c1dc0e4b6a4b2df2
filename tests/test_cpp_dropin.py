"""GPU: builds tests/cpp/dropin_test.cpp against include/ezquant/*.hpp and
libezquant.so (the C++ drop-in) and runs it."""
import os
import subprocess

import pytest

from conftest import ROOT


@pytest.mark.gpu
def test_cpp_dropin(gpu, tmp_path):
    lib = os.path.join(ROOT, "paper_2403_02775_b200", "_lib")
    exe = str(tmp_path / "dropin_test")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp"), "-L" + lib, "-lezquant",
                    "-lezq_b200", "-Wl,-rpath," + lib, "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


def test_cpp_dropin_compiles(N, tmp_path):
    """CPU: the reference-style program compiles and links against the drop-in."""
    lib = os.path.join(ROOT, "paper_2403_02775_b200", "_lib")
    subprocess.run(["g++", "-std=c++20", "-O0", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp"), "-L" + lib, "-lezquant",
                    "-lezq_b200", "-Wl,-rpath," + lib, "-o", str(tmp_path / "d")], check=True)

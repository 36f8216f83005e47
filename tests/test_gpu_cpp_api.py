"""GPU: the drop-in perfsage:: C++ API (include/perfsage_b200/perfsage.hpp) — compiles a C++
program written against the reference's call syntax, links the engine library, runs it."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build(tmp_path):
    exe = str(tmp_path / "test_perfsage_api")
    lib = os.path.join(ROOT, "paper_2003_07497_b200", "lib")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_perfsage_api.cpp"), "-L", lib,
                    "-lperfsage_b200", f"-Wl,-rpath,{lib}", "-o", exe], check=True)
    return exe


def test_cpp_api_compiles_against_reference_syntax(tmp_path):
    """CPU-side check: the header set compiles and links (no device needed to build)."""
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_cpp_api_runs_reference_unit_tests_on_gpu(tmp_path):
    out = subprocess.run([build(tmp_path)], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failures" in out.stdout

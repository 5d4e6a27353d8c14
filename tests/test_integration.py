"""The reference-side adapter of INTEGRATION.md (integration/dfc_gpu.hpp) compiles against the
reference's interface (integration/stub/: declarations of P/include/dfc types, since Eigen is not
installed) and links libdfcg.so; its error mapping round-trips the reference's exception types
(std::invalid_argument, std::out_of_range, BlockError with the "block N: " prefix exactly once).
The GPU case also solves blocks through make_gpu_base_solver and combines them through
column_project."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1107_0789_b200", "_lib")


def _build(tmp_path):
    exe = str(tmp_path / "integration_check")
    subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "integration", "stub"),
                    "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "integration", "check.cpp"),
                    "-L", LIB, "-ldfcg", f"-Wl,-rpath,{LIB}", "-o", exe], check=True)
    return exe


def test_adapter_compiles_and_maps_errors(tmp_path):
    r = subprocess.run([_build(tmp_path), "--cpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "OK cpu" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_adapter_solves_and_combines_on_gpu(tmp_path):
    r = subprocess.run([_build(tmp_path)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "OK gpu" in r.stdout, r.stdout + r.stderr

"""The C++ drop-in API (include/pbsa/pbsa_b200.hpp) on a GPU: runs build/test_pbsa_cpp."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "test_pbsa_cpp")


def test_cpp_header_compiles_without_gpu():
    """Host-only compile of the C++ API header (no device code needed)."""
    src = "#include \"pbsa/pbsa_b200.hpp\"\nint main(){ return (int)pbsa::topk_count(312, 0.25) - 78; }\n"
    out = os.path.join(ROOT, "build", "hdr_check")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    r = subprocess.run(["g++", "-std=c++20", "-x", "c++", "-", "-I", os.path.join(ROOT, "include"),
                        "-I", "/usr/local/cuda/include", "-fsyntax-only"], input=src, text=True,
                       capture_output=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_cpp_api_on_gpu():
    if not os.path.exists(BIN):
        subprocess.run(["make", "-C", ROOT, "cpp-test"], check=True)
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.startswith("PASS"), r.stdout + r.stderr

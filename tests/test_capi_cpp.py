"""The C-ABI as a C++ engine sees it: tools/example_connector.cpp includes
only include/tierkv_b200.h (plus the CUDA runtime for its own buffers),
links libtierkv_b200.so and runs a cold and a warm prefill through the
connector with the reference engine's call sequence. CPU: it compiles and
links. GPU: it runs, retrieves len-1 tokens and every page word verifies."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2510_09665_b200")
SRC = os.path.join(ROOT, "tools", "example_connector.cpp")
CUDA = "/usr/local/cuda"


def _build(tmp_path):
    out = str(tmp_path / "example_connector")
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", SRC, "-o", out, "-I", os.path.join(ROOT, "include"),
           "-I", f"{CUDA}/include", "-L", PKG, "-ltierkv_b200", "-L", f"{CUDA}/lib64", "-lcudart",
           f"-Wl,-rpath,{PKG}", f"-Wl,-rpath,{CUDA}/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_cpp_engine_compiles_against_header(tkv, tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_cpp_engine_roundtrip(tkv, tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "cold_loaded=0 warm_loaded=999 mismatched_words=0" in r.stdout

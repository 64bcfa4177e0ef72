"""The C++ drop-in: the reference's own EngineCore<float> and
neng::gpu::GpuEngine (include/neng_gpu_engine.hpp) side by side in one C++
process (tests/cpp/test_drop_in.cpp), bit for bit, including the error types
and messages.  The binary is built here by oracle/Makefile from the
reference's unchanged sources and travels to the GPU box prebuilt."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "test_drop_in")
REF = "/root/reference/proj"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree only in the build container")
def test_drop_in_builds_against_the_reference_headers():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "dropin"], check=True)
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_gpu_engine_matches_engine_core_float_in_cpp():
    if not os.path.exists(BIN):
        pytest.fail("oracle/_ref/test_drop_in was not built (run __graft_entry__.build() in the build container)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("PASS"), r.stdout

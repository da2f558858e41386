"""The C++ host side (include/shardplan_b200/measured_provider.hpp) compiles
against the reference's own headers as a shardplan::CostProvider (CPU, here)
and measures placements on cuda:0 (GPU box, mirror types)."""
import os
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2210_02023_b200")
REF = "/root/reference/proj/include"


def _json_include():
    import sysconfig
    return os.path.join(sysconfig.get_paths()["purelib"], "include", "cudnn_frontend",
                        "thirdparty")


def _build(exe, with_ref):
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    cmd = [cxx, "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "provider_test.cpp"), "-o", exe,
           os.path.join(LIBDIR, "_shardplan_b200.so"), f"-Wl,-rpath,{LIBDIR}"]
    if with_ref:
        cmd[2:2] = ["-DSHARDPLAN_B200_WITH_REFERENCE", "-I", REF, "-I", _json_include()]
    subprocess.run(cmd, check=True, capture_output=True)


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "shardplan")),
                    reason="reference headers not present")
def test_provider_is_a_reference_cost_provider():
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "t")
        _build(exe, True)
        r = subprocess.run([exe], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        assert "ok" in r.stdout


@pytest.mark.gpu
def test_provider_measures_on_gpu():
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "t")
        _build(exe, False)
        r = subprocess.run([exe, "gpu"], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        assert "ok (gpu)" in r.stdout


TRAIN_BIN = os.path.join(ROOT, "tests", "cpp", "_bin", "measured_train_test")
TOOL_BIN = os.path.join(ROOT, "tools", "_bin", "train_measured")


def _build_train(exe, src=None):
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    cmd = [cxx, "-std=c++20", "-O2", "-DSHARDPLAN_B200_WITH_REFERENCE", "-I", REF,
           "-I", _json_include(),
           "-include", os.path.join(ROOT, "tests", "cpp", "ref_shim.hpp"),
           "-I", os.path.join(ROOT, "include"),
           src or os.path.join(ROOT, "tests", "cpp", "measured_train_test.cpp"), "-o", exe,
           os.path.join(LIBDIR, "_shardplan_b200.so"), f"-Wl,-rpath,{LIBDIR}"]
    subprocess.run(cmd, check=True, capture_output=True)


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "shardplan")),
                    reason="reference headers not present")
def test_training_loop_on_provider_reproduces_reference_train():
    """train_on_provider with OracleCostProvider == the reference's train()."""
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "t")
        _build_train(exe)
        r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr
        assert "ok (oracle" in r.stdout


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(TRAIN_BIN),
                    reason="built by __graft_entry__.build() where the reference headers exist")
def test_training_loop_on_measured_costs():
    """The reference's training loop with the collect phase on B200-measured
    costs (MeasuredCostProvider): finite costs and losses, one
    measured cost vector per table per collected episode."""
    r = subprocess.run([TRAIN_BIN, "gpu"], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr
    assert "ok (gpu" in r.stdout, r.stdout

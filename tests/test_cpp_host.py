"""The C++ host layer (include/dsmc/dsmc.hpp, reference-shaped dsmc:: API)
and its doctest-style test binary (tests/cpp/test_host.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_host")
HOSTLIB = os.path.join(ROOT, "paper_2202_02264_b200", "libdsmc_host.so")


def test_host_library_and_tests_are_built():
    assert os.path.exists(HOSTLIB) and os.path.exists(BIN), "make -C paper_2202_02264_b200/csrc"
    out = subprocess.run(["nm", "-DC", "--defined-only", HOSTLIB], capture_output=True, text=True).stdout
    for sym in ["dsmc::run_smoother", "dsmc::run_conditional", "dsmc::pgibbs_sweep",
                "dsmc::make_lgssm_fk", "dsmc::resample_pairs", "dsmc::kalman_smooth"]:
        assert sym in out, sym


@pytest.mark.gpu
def test_host_api_cases_pass_on_gpu():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr

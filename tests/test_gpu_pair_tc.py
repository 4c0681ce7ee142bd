"""The tcgen05 pass-1 kernel (c32_pair_tc, DSMC_PAIR_KERNEL=tc): level-1 log
mean weights against the CUDA-core kernel on identical leaves (the inputs of
a level-1 combine are the leaves only), and a full smoothing run against the
exact Kalman/RTS answer. Run in subprocesses: the kernel is chosen per
engine context from the environment."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _run(kernel, out):
    env = dict(os.environ, DSMC_PAIR_KERNEL=kernel, DSMC_TC2_MIN="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "tc_lmw.py"), "run", out],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "failed" not in r.stdout, r.stdout


@pytest.mark.parametrize("kernel", ["tc", "tc2"])
def test_tc_level1_weights_match_the_cuda_core_kernel(tmp_path, kernel):
    a, b = str(tmp_path / "tc.npz"), str(tmp_path / "fma.npz")
    _run(kernel, a)
    _run("fma", b)
    A, B = np.load(a), np.load(b)
    assert set(A.files) == set(B.files) and len(A.files) == 7
    for k in A.files:
        assert np.isfinite(A[k]).all(), k
        # 3xTF32 + FP32 accumulation vs the FFMA chain: log mean weights of
        # whole combines agree to 1e-4 (1e-2 for the narrow-transition SV)
        tol = 1e-2 if k == "sv_tiny" else 1e-3
        assert np.max(np.abs(A[k] - B[k])) < tol, (k, np.max(np.abs(A[k] - B[k])))


@pytest.mark.parametrize("kernel", ["tc", "tc2"])
def test_tc_smoothing_tracks_kalman(kernel):
    code = r"""
import numpy as np
from paper_2202_02264_b200 import abi, models
from paper_2202_02264_b200.dsmc import Engine, kalman_smooth
e = Engine(0)
m = models.cv_tracking(1023)
km, kP, _ = kalman_smooth(m)
z = []
for s in range(4):
    r = e.smooth(m, 1024, abi.MULTINOMIAL, seed=100 + s, precision=abi.FP32)
    z.append((r["mean"] - km) / np.sqrt(np.einsum("tii->ti", kP)))
z = np.mean(z, 0)
# ragged particle counts (partial 128-row tiles and 64-column sub-blocks)
for N in (100, 300):
    zs = []
    for s in range(4):
        r = e.smooth(m, N, abi.MULTINOMIAL, seed=200 + s, precision=abi.FP32)
        assert np.isfinite(r["mean"]).all() and np.isfinite(r["log_norm_const"])
        zs.append((r["mean"] - km) / np.sqrt(np.einsum("tii->ti", kP)))
    assert float(np.sqrt(np.mean(np.mean(zs, 0) ** 2))) < 0.6, N
print(float(np.sqrt(np.mean(z ** 2))))
"""
    env = dict(os.environ, DSMC_PAIR_KERNEL=kernel, DSMC_TC2_MIN="0", PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    rms = float(r.stdout.strip().splitlines()[-1])
    # 4-run average of the smoothed means in posterior sd units: unbiased
    # smoothing gives an rms of about sqrt(1/4 * var ratio) < 0.5
    assert rms < 0.5, rms

"""Device Kalman filter + RTS smoother by parallel prefix scans
(dsmc_kalman_smooth_device, csrc/kalman_scan.cuh) against the sequential
host restatement of kalman.cpp:78-138 (dsmc_kalman_smooth, itself checked
against numpy in tests/test_abi.py): smoothed means, covariances and the
marginal log-likelihood, up to C5's horizon."""
import time

import numpy as np
import pytest

from paper_2202_02264_b200 import abi, models
from paper_2202_02264_b200.dsmc import kalman_smooth

pytestmark = pytest.mark.gpu


def _gappy(T):
    """d = 2 / dy = 1 with time-varying F, Q and missing observations."""
    K = T + 1
    rng = np.random.default_rng(4)
    F = np.tile(np.array([[1.0, 1.0], [0.0, 0.92]]), (K, 1, 1))
    F[:, 1, 1] += 0.05 * np.sin(np.arange(K))
    Q = np.tile(np.array([[0.05, 0.01], [0.01, 0.1]]), (K, 1, 1)) * (1 + 0.5 * rng.random((K, 1, 1)))
    b = np.tile([0.03, -0.01], (K, 1))
    y = rng.standard_normal((K, 1))
    obs = (rng.random(K) > 0.3).astype(np.uint8)
    m = abi.Model(abi.MODEL_LGSSM, T, 2, 1, m0=[0.0, 0.0], P0=np.eye(2), F=F, b=b, Q=Q,
                  H=[[1.0, 0.0]], R=[[0.3]], y=y, has_obs=obs, prop_mean=np.zeros((K, 2)),
                  prop_cov=np.tile(np.eye(2), (K, 1, 1)))
    return m


@pytest.mark.parametrize("make", [lambda: models.lgssm_check(1023),
                                  lambda: models.cv_tracking((1 << 14) - 1),
                                  lambda: _gappy(3000),
                                  lambda: models.lgssm_check(0)])
def test_device_kalman_matches_host(engine, make):
    m = make()
    hm, hP, hll = kalman_smooth(m)
    dm, dP, dll = engine.kalman_smooth(m)
    scale = np.abs(hm).max() + 1.0
    assert np.abs(dm - hm).max() <= 1e-9 * scale
    assert np.abs(dP - hP).max() <= 1e-9 * (np.abs(hP).max() + 1.0)
    assert abs(dll - hll) <= 1e-9 * abs(hll)


def test_device_kalman_c5_horizon(engine):
    """C5 (K = 2^20, d = 4): the proposal construction of the headline run on
    the device, against the host RTS, with both times printed."""
    m = models.cv_tracking((1 << 20) - 1)
    t0 = time.perf_counter()
    hm, hP, hll = kalman_smooth(m)
    th = time.perf_counter() - t0
    engine.kalman_smooth(m)  # warm (arena allocations)
    t0 = time.perf_counter()
    dm, dP, dll = engine.kalman_smooth(m)
    td = time.perf_counter() - t0
    print(f"C5 RTS: host {th * 1e3:.0f} ms, device scan {td * 1e3:.1f} ms (host arrays in/out)")
    scale = np.abs(hm).max() + 1.0
    assert np.abs(dm - hm).max() <= 1e-9 * scale
    assert np.abs(dP - hP).max() <= 1e-8 * (np.abs(hP).max() + 1.0)
    assert abs(dll - hll) <= 1e-9 * abs(hll)

"""Fused small-N FP32 combine (c32_small, csrc/small32.cuh; N <= 128): the
same law as the two-kernel path (c32_pair + c32_sample; DSMC_SMALL=0) —
level-1 log mean weights agree to FP32 rounding (identical leaves), and the
smoothed means and log Z of repeated runs agree with each other and with the
exact Kalman/RTS smoother, including the conditional (c-dSMC) form."""
import os

import numpy as np
import pytest

from paper_2202_02264_b200 import abi, models
from paper_2202_02264_b200.dsmc import kalman_smooth

pytestmark = pytest.mark.gpu


def _smooth(engine, m, N, rs, seed, small):
    os.environ["DSMC_SMALL"] = "1" if small else "0"
    try:
        return engine.smooth(m, N, rs, seed=seed, precision=abi.FP32, want_pairs=True)
    finally:
        os.environ.pop("DSMC_SMALL", None)


@pytest.mark.parametrize("name,make,N", [
    ("lg1", lambda: models.lgssm_check(1023), 100),
    ("cv", lambda: models.cv_tracking(511), 128),
    ("sv", lambda: models.sv(511), 64),
    ("crw", lambda: models.constrained_rw(255), 100),
])
def test_level1_weights_match_two_kernel_path(engine, name, make, N):
    m = make()
    for rs in (abi.MULTINOMIAL, abi.SYSTEMATIC):
        a = _smooth(engine, m, N, rs, 3, True)
        b = _smooth(engine, m, N, rs, 3, False)
        K1 = (m.horizon + 1) // 2
        la, lb = a["log_mean_weight"][:K1], b["log_mean_weight"][:K1]
        assert np.isfinite(la).all() and np.isfinite(lb).all()
        assert np.max(np.abs(la - lb)) < 2e-4, (name, rs, np.max(np.abs(la - lb)))


def test_small_path_tracks_kalman_and_two_kernel_log_z(engine):
    m = models.lgssm_check(1023)
    km, kP, ll = kalman_smooth(m)
    for small in (True, False):
        z, lz = [], []
        for s in range(8):
            r = _smooth(engine, m, 100, abi.MULTINOMIAL, 50 + s, small)
            z.append((r["mean"][:, 0] - km[:, 0]) / np.sqrt(kP[:, 0, 0]))
            lz.append(r["log_norm_const"])
        zm = np.mean(z, 0)
        # 8-run average in posterior sd units: unbiased => rms ~ sqrt(var ratio / 8)
        assert float(np.sqrt(np.mean(zm ** 2))) < 0.5, small
        # log Z within Monte Carlo error of the exact marginal likelihood
        assert abs(np.mean(lz) - ll) < 4 * np.std(lz) / np.sqrt(8) + 0.5, (small, np.mean(lz), ll)

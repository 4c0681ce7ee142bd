"""GPU FP64 parity sweep over state dimension, particle count and resampler:
device-generated leaves (FP64 Box-Muller, within a few ulp of glibc) against
the C oracle. Ancestor indices must agree exactly (an ulp-level leaf
difference can flip a selection only if a uniform lands within ~1e-16 of a
CDF boundary)."""
import numpy as np
import pytest

from paper_2202_02264_b200 import abi, models
from paper_2202_02264_b200.dsmc import kalman_smooth

pytestmark = pytest.mark.gpu


def lg_model(d, T, seed=1):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((d, d)) * 0.3
    F = 0.9 * np.eye(d) + 0.1 * (A - A.T)
    B = rng.standard_normal((d, d)) * 0.2
    Q = B @ B.T + 0.2 * np.eye(d)
    dy = max(1, d // 2)
    H = rng.standard_normal((dy, d))
    R = 0.3 * np.eye(dy)
    y = rng.standard_normal((T + 1, dy))
    m = abi.Model(abi.MODEL_LGSSM, T, d, dy, m0=np.zeros(d), P0=np.eye(d), F=F, b=0.1 * np.ones(d),
                  Q=Q, H=H, R=R, y=y, prop_mean=np.zeros((T + 1, d)),
                  prop_cov=np.tile(np.eye(d), (T + 1, 1, 1)))
    return models.with_rts_proposals(m, inflation=1.5)


@pytest.mark.parametrize("d", [1, 2, 3, 4])
@pytest.mark.parametrize("N", [8, 33, 64, 100, 257])
def test_fp64_device_vs_oracle(engine, oracle, d, N):
    m = lg_model(d, 12, seed=d)
    for rs in (abi.MULTINOMIAL, abi.SYSTEMATIC, abi.MH_LAZY):
        o = oracle.smooth(m, N, rs, seed=N + d, mh_steps=5)
        r = engine.smooth(m, N, rs, seed=N + d, precision=abi.FP64_PARITY, mh_steps=5,
                          want_pairs=True, want_paths=True, want_leaves=True)
        assert np.allclose(r["leaves"], o["leaves"], rtol=1e-13, atol=1e-13)
        assert np.array_equal(r["pair_left"], o["pair_left"]), (d, N, rs)
        assert np.array_equal(r["pair_right"], o["pair_right"]), (d, N, rs)
        assert np.allclose(r["paths"], o["paths"], rtol=1e-13, atol=1e-13)
        if o["log_norm_const"] is not None:
            assert abs(r["log_norm_const"] - o["log_norm_const"]) < 1e-10
        assert r["weight_evals"] == o["weight_evals"]


def test_horizon_beyond_grid_y_limit(engine):
    """K = 2^17 leaves: per-time and per-block grids exceed 65535, so time and
    block indices must live in grid x (C5 runs K = 2^20)."""
    K = 1 << 17
    m = models.lgssm_check(K - 1)
    r = engine.smooth(m, 16, abi.MULTINOMIAL, seed=3, precision=abi.FP32)
    assert r["levels"] == 17
    assert np.isfinite(r["mean"]).all() and np.isfinite(r["log_norm_const"])
    km, kP, _ = kalman_smooth(m)
    z = (r["mean"][:, 0] - km[:, 0]) / np.sqrt(kP[:, 0, 0])
    assert np.sqrt(np.mean(z ** 2)) < 1.0

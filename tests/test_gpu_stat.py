"""GPU statistical parity of the FP32 throughput path: smoothed moments
against the exact Kalman/RTS smoother (linear-Gaussian configs) and against
the FP64 parity path (SV), log Z against the Kalman log-likelihood, and
first-level ancestor agreement with the FP64 path on identical uniforms.

Tolerances are Monte Carlo: N particles give smoothed-mean errors of order
sd_t / sqrt(N_eff); every bound below is stated next to its check."""
import numpy as np
import pytest

from paper_2202_02264_b200 import abi, models
from paper_2202_02264_b200.dsmc import kalman_smooth

pytestmark = pytest.mark.gpu


def _z(mean, km, kP):
    sd = np.sqrt(np.einsum("tii->ti", kP))
    return (mean - km) / sd


@pytest.mark.parametrize("precision", [abi.FP32, abi.FP64_PARITY])
def test_lgssm_means_match_kalman(engine, precision):
    m = models.lgssm_check(255)
    km, kP, ll = kalman_smooth(m)
    r = engine.smooth(m, 2048, abi.MULTINOMIAL, seed=3, precision=precision)
    z = _z(r["mean"], km, kP)
    # standardized error ~ 1/sqrt(N_eff); N_eff >= 256 here -> rms <= 0.1
    assert np.sqrt(np.mean(z ** 2)) < 0.1, np.sqrt(np.mean(z ** 2))
    assert np.abs(z).max() < 0.45
    # posterior variances within 15%
    ratio = r["cov"][:, 0, 0] / kP[:, 0, 0]
    assert 0.85 < np.median(ratio) < 1.15
    # log Z estimates the marginal likelihood (test_smoother.cpp:292-316)
    assert abs(r["log_norm_const"] - ll) < 1.0, (r["log_norm_const"], ll)


def test_cv_d4_means_match_kalman(engine):
    m = models.cv_tracking(255)
    km, kP, ll = kalman_smooth(m)
    r = engine.smooth(m, 1024, abi.MULTINOMIAL, seed=5, precision=abi.FP32)
    z = _z(r["mean"], km, kP)
    assert np.sqrt(np.mean(z ** 2)) < 0.15, np.sqrt(np.mean(z ** 2))
    assert abs(r["log_norm_const"] - ll) < 2.0, (r["log_norm_const"], ll)


def test_fp32_and_fp64_agree_on_first_level_pairs(engine):
    """Same uniforms, FP32 vs FP64 weights: level-1 selections differ only
    where a uniform falls within ~1e-6 of a CDF boundary."""
    m = models.lgssm_check(63)
    a = engine.smooth(m, 512, abi.MULTINOMIAL, seed=9, precision=abi.FP32, want_pairs=True)
    b = engine.smooth(m, 512, abi.MULTINOMIAL, seed=9, precision=abi.FP64_PARITY, want_pairs=True)
    n1 = (m.horizon + 1) // 2
    # leaves differ (FP32 vs FP64 Box-Muller) only by rounding, so level-1
    # tables agree to ~1e-6 relative
    same = (a["pair_left"][:n1] == b["pair_left"][:n1]) & (a["pair_right"][:n1] == b["pair_right"][:n1])
    assert same.mean() > 0.99, same.mean()


def test_sv_fp32_matches_fp64(engine):
    m = models.sv(511)
    a = engine.smooth(m, 2048, abi.MULTINOMIAL, seed=1, precision=abi.FP32)
    b = engine.smooth(m, 2048, abi.MULTINOMIAL, seed=2, precision=abi.FP64_PARITY)
    sd = np.sqrt(0.5 * (a["cov"][:, 0, 0] + b["cov"][:, 0, 0]))
    z = (a["mean"][:, 0] - b["mean"][:, 0]) / sd
    assert np.sqrt(np.mean(z ** 2)) < 0.15
    assert abs(a["log_norm_const"] - b["log_norm_const"]) < 1.5


@pytest.mark.parametrize("rs", [abi.MH_LAZY, abi.REJECTION_LAZY])
def test_lazy_sv_matches_dense(engine, rs):
    from tests.cases import CASES, model_for
    m = model_for(dict(CASES["sv"], T=255))
    dense = engine.smooth(m, 1024, abi.MULTINOMIAL, seed=4, precision=abi.FP32)
    lazy = engine.smooth(m, 1024, rs, seed=5, precision=abi.FP32, mh_steps=16)
    sd = np.sqrt(dense["cov"][:, 0, 0])
    z = (lazy["mean"][:, 0] - dense["mean"][:, 0]) / sd
    # MH-16 is biased (resampling.hpp:55-59) but close; rejection is exact
    assert np.sqrt(np.mean(z ** 2)) < 0.2
    assert lazy["log_norm_const"] is None
    assert lazy["biased"] == (rs == abi.MH_LAZY)
    assert lazy["weight_evals"] > 0


def test_systematic_fp32(engine):
    m = models.lgssm_check(127)
    km, kP, _ = kalman_smooth(m)
    r = engine.smooth(m, 1024, abi.SYSTEMATIC, seed=11, precision=abi.FP32)
    assert np.sqrt(np.mean(_z(r["mean"], km, kP) ** 2)) < 0.12


def test_odd_horizons_and_single_time(engine, oracle):
    for T in (0, 1, 2, 6, 100):
        m = models.lgssm_check(T)
        km, kP, ll = kalman_smooth(m)
        r = engine.smooth(m, 4096, abi.MULTINOMIAL, seed=T, precision=abi.FP32)
        assert r["levels"] == (int(np.ceil(np.log2(T + 1))) if T else 0)
        assert np.sqrt(np.mean(_z(r["mean"], km, kP) ** 2)) < 0.1


def test_conditional_fp32_keeps_reference_and_moves(engine):
    m = models.sv(127)
    ref = np.full((1, 128, 1), -1.0)
    outs = engine.conditional_sweep([m] * 4, np.repeat(ref, 4, 0), [1, 2, 3, 4], 256, 0)
    # paths differ across chains, stay finite, and mostly move off the
    # constant reference (update rate, pgibbs.cpp:57-78)
    assert np.isfinite(outs["paths"]).all()
    assert outs["changed"].mean() > 0.5
    assert not np.array_equal(outs["paths"][0], outs["paths"][1])


def test_kernel_launch_counter_moves(engine):
    before = engine.launches
    engine.smooth(models.lgssm_check(15), 64, seed=1)
    assert engine.launches > before

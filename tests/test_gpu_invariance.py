"""Statistical laws the reference's own tests pin, on the GPU:

* c-dSMC leaves the smoothing posterior invariant (test_conditional.cpp:
  155-437): started from exact posterior draws, one conditional sweep (and a
  chain of them) returns exact posterior draws — per-time mean, variance and
  lag-1 covariance against the Kalman/RTS answer, over thousands of chains
  run as one batched sweep;
* the normalising-constant estimate is unbiased (test_smoother.cpp:416-456):
  mean exp(log Z - exact) = 1 at N = 8, and so is the device particle
  filter's evidence (test_baselines.cpp:26-60).

The model is the reference's AR(1) fixture (tests/support/ar1.hpp) with
stationary (not RTS) proposals, so the invariance is not an artefact of
exact proposals."""
import numpy as np
import pytest

from paper_2202_02264_b200 import abi, models
from paper_2202_02264_b200.dsmc import kalman_smooth

pytestmark = pytest.mark.gpu

RHO, Q, R = 0.8, 0.3, 0.4


def _data(T, seed):
    rng = np.random.default_rng(seed)
    s2 = Q / (1 - RHO * RHO)
    x = np.empty(T + 1)
    x[0] = np.sqrt(s2) * rng.standard_normal()
    for t in range(1, T + 1):
        x[t] = RHO * x[t - 1] + np.sqrt(Q) * rng.standard_normal()
    return x + np.sqrt(R) * rng.standard_normal(T + 1)


def _posterior(ys):
    """Kalman filter + RTS moments and exact lag-1 covariances of the AR(1)."""
    K = len(ys)
    mf, Pf, mp, Pp = np.empty(K), np.empty(K), np.empty(K), np.empty(K)
    for t in range(K):
        mp[t], Pp[t] = (0.0, Q / (1 - RHO * RHO)) if t == 0 else (RHO * mf[t - 1], RHO * RHO * Pf[t - 1] + Q)
        g = Pp[t] / (Pp[t] + R)
        mf[t], Pf[t] = mp[t] + g * (ys[t] - mp[t]), (1 - g) * Pp[t]
    ms, Ps, C1 = mf.copy(), Pf.copy(), np.empty(K - 1)
    for t in range(K - 2, -1, -1):
        J = Pf[t] * RHO / Pp[t + 1]
        ms[t] = mf[t] + J * (ms[t + 1] - mp[t + 1])
        Ps[t] = Pf[t] + J * J * (Ps[t + 1] - Pp[t + 1])
        C1[t] = J * Ps[t + 1]
    return mf, Pf, mp, Pp, ms, Ps, C1


def _exact_draws(ys, n, rng):
    """FFBS for the linear-Gaussian AR(1): exact joint posterior paths."""
    mf, Pf, mp, Pp, *_ = _posterior(ys)
    K = len(ys)
    x = np.empty((n, K))
    x[:, K - 1] = mf[K - 1] + np.sqrt(Pf[K - 1]) * rng.standard_normal(n)
    for t in range(K - 2, -1, -1):
        J = Pf[t] * RHO / Pp[t + 1]
        mean = mf[t] + J * (x[:, t + 1] - mp[t + 1])
        var = Pf[t] - J * RHO * Pf[t]
        x[:, t] = mean + np.sqrt(var) * rng.standard_normal(n)
    return x


def _check_law(paths, ys):
    *_, ms, Ps, C1 = _posterior(ys)
    n = paths.shape[0]
    mean = paths.mean(0)
    var = paths.var(0, ddof=1)
    z_mean = (mean - ms) / np.sqrt(Ps / n)
    assert np.max(np.abs(z_mean)) < 4.5, z_mean
    # sample variance: sd of the ratio ~ sqrt(2 / n)
    assert np.max(np.abs(var / Ps - 1)) < 4.5 * np.sqrt(2.0 / n), var / Ps
    c1 = np.mean((paths[:, :-1] - mean[:-1]) * (paths[:, 1:] - mean[1:]), 0)
    se = np.sqrt((Ps[:-1] * Ps[1:] + C1 * C1) / n)
    assert np.max(np.abs(c1 - C1) / se) < 4.5, (c1 - C1) / se


@pytest.mark.parametrize("precision", [abi.FP64_PARITY, abi.FP32])
def test_conditional_sweep_leaves_the_posterior_invariant(engine, precision):
    T, n = 15, 3000
    ys = _data(T, 321)
    m = models.ar1(ys, RHO, Q, R)
    rng = np.random.default_rng(5)
    start = _exact_draws(ys, n, rng)
    out = engine.conditional_sweep([m] * n, start[:, :, None], np.arange(n) + 77, 32, 0,
                                   precision=precision)
    paths = out["paths"][:, :, 0]
    assert np.isfinite(paths).all()
    # slot 0 is the reference: a sweep must be able to move it, and not always
    assert 0.05 < out["changed"].mean() < 0.999
    _check_law(paths, ys)
    # a chain of sweeps stays on the law (test_conditional.cpp chained sweeps)
    for sweep in (1, 2):
        out = engine.conditional_sweep([m] * n, paths[:, :, None], np.arange(n) + 77, 32, sweep,
                                       precision=precision)
        paths = out["paths"][:, :, 0]
    _check_law(paths, ys)


def test_normalising_constant_is_unbiased_at_small_n(engine):
    T, N, reps = 15, 8, 3000
    ys = _data(T, 99)
    m = models.ar1(ys, RHO, Q, R)
    _, _, exact = kalman_smooth(m)
    r = np.array([engine.smooth(m, N, abi.MULTINOMIAL, seed=1000 + s, precision=abi.FP64_PARITY,
                                want_moments=False)["log_norm_const"] for s in range(reps)])
    w = np.exp(r - exact)
    se = w.std(ddof=1) / np.sqrt(reps)
    assert abs(w.mean() - 1.0) < 4.0 * se, (w.mean(), se)
    # and log Z itself is biased low (Jensen), as an unbiased Z implies
    assert r.mean() < exact


def test_particle_filter_evidence_is_unbiased(engine):
    """test_baselines.cpp:26-60: the bootstrap-style filter's exp(log Z) is
    unbiased (device PF of the FFBS comparator, FP32 arithmetic)."""
    T, N, reps = 15, 16, 3000
    ys = _data(T, 7)
    m = models.ar1(ys, RHO, Q, R)
    _, _, exact = kalman_smooth(m)
    r = np.array([engine.ffbs(m, N, n_draws=1, seed=50_000 + s)["log_likelihood"]
                  for s in range(reps)])
    assert np.isfinite(r).all()
    w = np.exp(r - exact)
    se = w.std(ddof=1) / np.sqrt(reps)
    # FP32 log-weights: allow the ~1e-6 relative float bias on top of 4 SE
    assert abs(w.mean() - 1.0) < 4.0 * se + 1e-4, (w.mean(), se)

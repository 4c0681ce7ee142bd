"""Batched SV particle Gibbs (C4): the device parameter kernel against the
oracle's restatement (or_sv_param_update; gamma_draw pgibbs.cpp:80-102 and the
sweep contract pgibbs.cpp:24-55), and chain-level behaviour."""
import numpy as np
import pytest

from paper_2202_02264_b200 import abi, models

pytestmark = pytest.mark.gpu


def _prior():
    return abi.SvPrior(-1.0, 1.0, 2.0, 0.2, 0.05)


def _data(T, seed=5):
    m = models.sv(T, data_seed=seed)
    return np.asarray(m.arrays["y"], np.float64)


def test_param_kernel_matches_oracle(engine, oracle):
    """theta after one device sweep depends only on the input star path, the
    chain seed and the sweep (the parameter step runs before the path update):
    it must equal the oracle's update of the same star (CUDA vs glibc
    transcendentals: within 1e-12 relative; the phi accept decision exact)."""
    T, B = 127, 6
    ys = _data(T)
    rng = np.random.default_rng(1)
    stars = np.ascontiguousarray(-1.0 + 0.4 * rng.standard_normal((B, T + 1)))
    theta0 = np.ascontiguousarray(np.tile([-1.0, 0.9, 0.1], (B, 1)) +
                                  0.05 * rng.standard_normal((B, 3)) * [1, 0.1, 0.1])
    seeds = np.arange(B, dtype=np.uint64) * 7919 + 11
    for sweep in (0, 3):
        th = theta0.copy()
        st = stars.copy()
        _, acc = engine.sv_pgibbs_sweep(ys, th, st, seeds, _prior(), 128, sweep)
        n_acc = 0
        for c in range(B):
            ref, a = oracle.sv_param_update(stars[c], theta0[c], _prior(), int(seeds[c]), sweep)
            np.testing.assert_allclose(th[c], ref, rtol=1e-12, atol=1e-14)
            n_acc += a
        assert acc == n_acc


def test_param_kernel_matches_reference_gamma_draw_c4_shape(engine, reference):
    """the device SV parameter kernel pinned against the same
    kernel running on the reference's own RngStream and gamma_draw
    (pgibbs.cpp:80-102, compiled from /root/reference into oracle/_ref) —
    at C4's shape: 64 chains, K = 2^12. CUDA vs glibc transcendentals:
    within 1e-12 relative; every phi accept decision identical."""
    T, B = (1 << 12) - 1, 64
    ys = _data(T, seed=90210)
    rng = np.random.default_rng(11)
    stars = np.ascontiguousarray(-1.0 + 0.5 * rng.standard_normal((B, T + 1)))
    theta0 = np.ascontiguousarray(np.tile([-1.0, 0.9, 0.1], (B, 1)) +
                                  0.05 * rng.standard_normal((B, 3)) * [1, 0.1, 0.1])
    seeds = np.arange(B, dtype=np.uint64) + 1000
    for sweep in (0, 9):
        th = theta0.copy()
        st = stars.copy()
        _, acc = engine.sv_pgibbs_sweep(ys, th, st, seeds, _prior(), 64, sweep)
        n_acc = 0
        for c in range(B):
            ref, a = reference.sv_param_update(stars[c], theta0[c], _prior(), int(seeds[c]),
                                               sweep)
            np.testing.assert_allclose(th[c], ref, rtol=1e-12, atol=1e-14)
            n_acc += a
        assert acc == n_acc


def test_chains_move_and_recover_parameters(engine):
    """64 chains (C4 shape, reduced T/N): every sweep moves most of each star
    path (update rate, pgibbs.cpp:57-78) and after burn-in the chain-averaged
    mu, phi sit near the values the data were simulated with."""
    T, B, N = 511, 64, 256
    ys = _data(T, seed=90210)
    theta = np.ascontiguousarray(np.tile([-0.5, 0.8, 0.2], (B, 1)))
    stars = np.ascontiguousarray(np.full((B, T + 1), -1.0))
    seeds = np.arange(B, dtype=np.uint64) + 1000
    rates = []
    draws = []
    for s in range(60):
        changed, _ = engine.sv_pgibbs_sweep(ys, theta, stars, seeds, _prior(), N, s)
        rates.append(changed.mean())
        if s >= 30:
            draws.append(theta.copy())
    assert np.isfinite(stars).all() and np.isfinite(theta).all()
    assert np.mean(rates[5:]) > 0.5
    post = np.concatenate(draws)
    mu, phi, s2 = post.mean(0)
    # simulated with mu = -1, phi = 0.95, sigma = 0.3 (models.sv)
    assert abs(mu - (-1.0)) < 0.5, mu
    assert 0.7 < phi < 1.0, phi
    assert 0.0 < s2 < 0.5, s2

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
    # standardized error ~ 1/sqrt(N_eff): at N = 2048, N * mean z^2 ~ 13.5 for
    # both precisions (tools/zcheck.py, 12 seeds); a single run's mean z^2 has
    # a heavy right tail (errors are correlated along the path), so the bound
    # is on the 4-seed average: rms <= 0.1 is ~4 standard errors above it
    # (max |z| over t: median 0.25, p90 0.34, worst of 40 seeds ~0.7 for both
    # precisions, tools/zcheck2.py — so the bound is on the 4-seed median)
    zs, mx = [], []
    for seed in (3, 4, 5, 6):
        r = engine.smooth(m, 2048, abi.MULTINOMIAL, seed=seed, precision=precision)
        z = _z(r["mean"], km, kP)
        zs.append(np.mean(z ** 2))
        mx.append(np.abs(z).max())
    assert np.sqrt(np.mean(zs)) < 0.1, np.sqrt(np.mean(zs))
    assert np.median(mx) < 0.45, mx
    # posterior variances within 15%
    ratio = r["cov"][:, 0, 0] / kP[:, 0, 0]
    assert 0.85 < np.median(ratio) < 1.15
    # log Z estimates the marginal likelihood (test_smoother.cpp:292-316)
    assert abs(r["log_norm_const"] - ll) < 1.0, (r["log_norm_const"], ll)


def _seed_avg(engine, m, N, precision, seeds):
    runs = [engine.smooth(m, N, abi.MULTINOMIAL, seed=s, precision=precision) for s in seeds]
    means = np.stack([r["mean"] for r in runs])
    return means.mean(0), means.std(0, ddof=1) / np.sqrt(len(seeds)), runs


@pytest.mark.parametrize("precision", [abi.FP32, abi.FP64_PARITY])
def test_cv_d4_means_match_kalman(engine, precision):
    """The d=4 constant-velocity model (near-singular Q, strongly correlated
    neighbouring states) degenerates at moderate N, so a single run is not
    a sharp check: like test_smoother.cpp:292-316 (16 seeds, 5 SE) we compare
    the seed average against Kalman in units of its standard error."""
    m = models.cv_tracking(127)
    km, kP, ll = kalman_smooth(m)
    avg, se, runs = _seed_avg(engine, m, 1024, precision, range(16))
    z = (avg - km) / np.maximum(se, 1e-12)
    assert np.sqrt(np.mean(z ** 2)) < 2.0, np.sqrt(np.mean(z ** 2))
    # z is a t-statistic with 15 dof and heavy tails (path degeneracy): over
    # 128 x 4 entries the max is 3-6 and occasionally ~7.6 for BOTH
    # precisions (tools/zcheck3.py, 20 groups of 16 seeds), so bound the
    # bulk and only gross outliers
    assert np.mean(np.abs(z) > 4.0) < 0.01, np.mean(np.abs(z) > 4.0)
    assert np.abs(z).max() < 10.0
    lz = np.array([r["log_norm_const"] for r in runs])
    # exp(log Z) is unbiased (test_smoother.cpp:317-341): log-mean-exp vs ll
    lme = np.log(np.mean(np.exp(lz - lz.max()))) + lz.max()
    assert abs(lme - ll) < 3.0, (lme, ll)


def test_cv_d4_fp32_matches_fp64(engine):
    """FP32 throughput path vs FP64 parity path (bit-exact with the
    reference): seed-averaged means agree within 5 combined SE."""
    m = models.cv_tracking(127)
    a, sa, _ = _seed_avg(engine, m, 1024, abi.FP32, range(100, 116))
    b, sb, _ = _seed_avg(engine, m, 1024, abi.FP64_PARITY, range(200, 216))
    z = (a - b) / np.sqrt(sa ** 2 + sb ** 2)
    assert np.sqrt(np.mean(z ** 2)) < 2.0
    assert np.abs(z).max() < 6.0


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


def _avg1(engine, m, N, rs, precision, seeds, **kw):
    runs = [engine.smooth(m, N, rs, seed=s, precision=precision, **kw) for s in seeds]
    means = np.stack([r["mean"][:, 0] for r in runs])
    return means.mean(0), means.std(0, ddof=1) / np.sqrt(len(seeds)), runs


def test_sv_fp32_matches_fp64(engine):
    """Smoothed paths are strongly correlated in t, so one run per arm is a
    noisy check; compare 8-seed averages in standard-error units."""
    m = models.sv(255)
    a, sa, ra = _avg1(engine, m, 1024, abi.MULTINOMIAL, abi.FP32, range(8))
    b, sb, rb = _avg1(engine, m, 1024, abi.MULTINOMIAL, abi.FP64_PARITY, range(50, 58))
    z = (a - b) / np.sqrt(sa ** 2 + sb ** 2)
    assert np.sqrt(np.mean(z ** 2)) < 2.0 and np.abs(z).max() < 6.0
    la = np.array([r["log_norm_const"] for r in ra])
    lb = np.array([r["log_norm_const"] for r in rb])
    se = np.sqrt(la.var(ddof=1) / len(la) + lb.var(ddof=1) / len(lb))
    assert abs(la.mean() - lb.mean()) < 5 * se + 0.05, (la.mean(), lb.mean(), se)


@pytest.mark.parametrize("rs", [abi.MH_LAZY, abi.REJECTION_LAZY])
def test_lazy_sv_matches_dense(engine, rs):
    from tests.cases import CASES, model_for
    m = model_for(dict(CASES["sv"], T=127))
    a, sa, _ = _avg1(engine, m, 512, abi.MULTINOMIAL, abi.FP32, range(8))
    b, sb, runs = _avg1(engine, m, 512, rs, abi.FP32, range(20, 28), mh_steps=16)
    z = (a - b) / np.sqrt(sa ** 2 + sb ** 2)
    # rejection is exact; MH-16 is biased (resampling.hpp:55-59) but close
    assert np.sqrt(np.mean(z ** 2)) < (2.0 if rs == abi.REJECTION_LAZY else 3.0)
    lazy = runs[0]
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


@pytest.mark.parametrize("precision", [abi.FP32, abi.FP64_PARITY])
def test_batched_chains_equal_single_chain_runs(engine, precision):
    """Chains of one batched conditional sweep are independent: chain c of a
    B=4 batch equals the same chain run alone (per-chain workspaces; keys
    depend only on the chain's own seed, conditional.cpp:22-25)."""
    m = models.sv(127)
    refs = np.stack([np.full((128, 1), v) for v in (-1.0, -0.5, -1.5, -1.2)])
    seeds = [11, 12, 13, 14]
    both = engine.conditional_sweep([m] * 4, refs, seeds, 200, 3, precision=precision)
    for c in range(4):
        one = engine.conditional_sweep([m], refs[c:c + 1], seeds[c:c + 1], 200, 3,
                                       precision=precision)
        assert np.array_equal(both["paths"][c], one["paths"][0])
        assert both["log_norm_const"][c] == one["log_norm_const"][0]


def test_resident_graph_replays_match_eager(engine):
    """dsmc_smooth_resident captures the whole run into a CUDA graph on the
    second identical call and replays it with the seed as a kernel-node
    argument: every call must equal the eager dsmc_smooth of its seed."""
    m = models.cv_tracking(255)
    seeds = [5, 6, 7, 5, 8]
    refs = {s: engine.smooth(m, 256, abi.MULTINOMIAL, seed=s, precision=abi.FP32) for s in set(seeds)}
    h = engine.upload(m)
    try:
        for s in seeds:
            before = engine.launches
            engine.smooth_resident(h, 256, abi.MULTINOMIAL, seed=s)
            mean, cov, lnc = engine.resident_results(256, 4)
            assert engine.launches > before
            assert np.array_equal(mean, refs[s]["mean"]), s
            assert np.array_equal(cov, refs[s]["cov"]), s
            assert lnc == refs[s]["log_norm_const"]
    finally:
        engine.free_model(h)


@pytest.mark.parametrize("N", [33, 300, 1000, 1500])
def test_fp32_ragged_particle_counts(engine, N):
    """N not a multiple of the 64-column sub-block, the 256-row tile or the
    warp: padded columns / rows must never be selected and the moments stay
    unbiased (seed-averaged against Kalman/RTS)."""
    m = models.lgssm_check(127)
    km, kP, ll = kalman_smooth(m)
    runs = [engine.smooth(m, N, abi.MULTINOMIAL, seed=s, precision=abi.FP32, want_pairs=True)
            for s in range(8)]
    for r in runs:
        assert r["pair_left"].max() < N and r["pair_right"].max() < N
        assert np.isfinite(r["mean"]).all() and np.isfinite(r["log_norm_const"])
    means = np.stack([r["mean"] for r in runs])
    z = (means.mean(0) - km) / np.maximum(means.std(0, ddof=1) / np.sqrt(len(runs)), 1e-12)
    assert np.sqrt(np.mean(z ** 2)) < 2.0
    lz = np.array([r["log_norm_const"] for r in runs])
    lme = np.log(np.mean(np.exp(lz - lz.max()))) + lz.max()
    assert abs(lme - ll) < 1.0 + 8.0 / np.sqrt(N), (lme, ll)


@pytest.mark.parametrize("kind,precision", [("cox", abi.FP32), ("cox", abi.FP64_PARITY),
                                            ("crw", abi.FP32), ("crw", abi.FP64_PARITY),
                                            ("theta", abi.FP32), ("theta", abi.FP64_PARITY)])
def test_reference_models_match_grid(engine, kind, precision):
    """The reference's own benchmark models on the device (Cox counts,
    constrained random walk, models.cpp:111-338) against the dense-grid
    forward-backward oracle (grid_oracle.hpp): seed-averaged smoothed means
    within Monte-Carlo error, exp(log Z) unbiased (test_smoother.cpp:416-456
    checks the Poisson model against the grid the same way)."""
    from tests.grid_oracle import grid_truth
    T = 63
    m = (models.cox(T) if kind == "cox" else models.constrained_rw(T, 0.3) if kind == "crw"
         else models.theta_logistic(T, inflation=1.5))
    gm, gv, glz = grid_truth(m)
    runs = [engine.smooth(m, 512, abi.MULTINOMIAL, seed=s, precision=precision)
            for s in range(12)]
    means = np.stack([r["mean"][:, 0] for r in runs])
    z = (means.mean(0) - gm) / np.maximum(means.std(0, ddof=1) / np.sqrt(len(runs)), 1e-12)
    assert np.sqrt(np.mean(z ** 2)) < 2.0, np.sqrt(np.mean(z ** 2))
    assert np.mean(np.abs(z) > 4.0) < 0.05
    var = np.median(np.stack([r["cov"][:, 0, 0] for r in runs]).mean(0) / gv)
    assert 0.8 < var < 1.2, var
    lz = np.array([r["log_norm_const"] for r in runs])
    lme = np.log(np.mean(np.exp(lz - lz.max()))) + lz.max()
    assert abs(lme - glz) < 1.0, (lme, glz)


def test_constrained_rw_rejection_sampling(engine):
    """The constrained walk exposes a finite stitch bound (models.cpp:334),
    so rejection-lazy stitching runs exactly (log Z unavailable) and agrees
    with dense multinomial stitching in distribution."""
    from tests.grid_oracle import grid_truth
    m = models.constrained_rw(63, 0.3)
    gm, _, _ = grid_truth(m)
    for precision in (abi.FP32, abi.FP64_PARITY):
        runs = [engine.smooth(m, 512, abi.REJECTION_LAZY, seed=s, precision=precision)
                for s in range(12)]
        assert all(r["log_norm_const"] is None for r in runs)
        means = np.stack([r["mean"][:, 0] for r in runs])
        z = (means.mean(0) - gm) / np.maximum(means.std(0, ddof=1) / np.sqrt(len(runs)), 1e-12)
        assert np.sqrt(np.mean(z ** 2)) < 2.0, (precision, np.sqrt(np.mean(z ** 2)))


def test_fp32_dense_large_n_sampler(engine):
    """N beyond the shared-memory column staging of c32_sample (N = 8192:
    the row CDF plus the staged column pairs exceed 227 KB): the sampler
    keeps only the row CDF in shared memory and reads the pass-1 hand-off
    from L2 (samplew_kernel over Aux32Recompute). Same bounds as
    test_lgssm_means_match_kalman (errors shrink with N); N >= 65536 is
    refused (the packed sub-block index)."""
    m = models.lgssm_check(127)
    km, kP, ll = kalman_smooth(m)
    zs = []
    for seed in (3, 4, 5, 6):
        r = engine.smooth(m, 8192, abi.MULTINOMIAL, seed=seed, precision=abi.FP32)
        zs.append(np.mean(_z(r["mean"], km, kP) ** 2))
        assert abs(r["log_norm_const"] - ll) < 1.0, (r["log_norm_const"], ll)
    assert np.sqrt(np.mean(zs)) < 0.1, np.sqrt(np.mean(zs))
    ratio = r["cov"][:, 0, 0] / kP[:, 0, 0]
    assert 0.85 < np.median(ratio) < 1.15
    s = engine.smooth(m, 8192, abi.SYSTEMATIC, seed=9, precision=abi.FP32)
    assert np.sqrt(np.mean(_z(s["mean"], km, kP) ** 2)) < 0.2
    with pytest.raises(ValueError, match="65536"):
        engine.smooth(m, 65536, abi.MULTINOMIAL, seed=1, precision=abi.FP32)

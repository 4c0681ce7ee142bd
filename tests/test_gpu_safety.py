"""Memory-safety proxies for the device paths (compute-sanitizer is not
available on the GPU pool, so the checks are our own):

* guard bands: host output arrays handed to the C ABI are views into larger
  buffers filled with a sentinel; nothing past the declared (K, d) / (K, d, d)
  extent may change (ragged N, every resampler, both precisions);
* state independence: one long-lived engine context runs a sequence of
  workloads that grow, shrink and change d, N, resampler and precision; every
  result must be bit-identical to the same call on a fresh context. A kernel
  that reads past its logical extent into scratch left by an earlier, larger
  run (or depends on uninitialised scratch) breaks this.
"""
import numpy as np
import pytest

from paper_2202_02264_b200 import abi, models
from paper_2202_02264_b200.dsmc import Engine

pytestmark = pytest.mark.gpu

SENTINEL = -7.25e300
GUARD = 97


def _guarded(shape):
    n = int(np.prod(shape))
    buf = np.full(n + GUARD, SENTINEL)
    return buf, buf[:n].reshape(shape)


@pytest.mark.parametrize("make,N,rs,prec", [
    (lambda: models.lgssm_check(37), 100, abi.MULTINOMIAL, abi.FP32),
    (lambda: models.cv_tracking(29), 300, abi.SYSTEMATIC, abi.FP32),
    (lambda: models.sv(41), 130, abi.MH_LAZY, abi.FP32),
    (lambda: models.constrained_rw(23), 70, abi.REJECTION_LAZY, abi.FP32),
    (lambda: models.cv_tracking(17), 65, abi.MULTINOMIAL, abi.FP64_PARITY),
    (lambda: models.lgssm_check(20), 33, abi.MH_LAZY, abi.FP64_PARITY),
])
def test_outputs_stay_inside_their_extent(engine, make, N, rs, prec):
    m = make()
    K, d = m.horizon + 1, m.d
    mbuf, mean = _guarded((K, d))
    cbuf, cov = _guarded((K, d, d))
    r = engine.smooth(m, N, rs, seed=5, precision=prec, mean_out=mean, cov_out=cov)
    assert r["mean"] is mean
    assert np.isfinite(mean).all() and np.isfinite(cov).all()
    assert (mbuf[K * d:] == SENTINEL).all()
    assert (cbuf[K * d * d:] == SENTINEL).all()


def _calls():
    """(label, model factory, N, resampler, precision): large first so later,
    smaller calls run on scratch a larger run has already filled."""
    return [
        ("cv big", lambda: models.cv_tracking(1023), 1024, abi.MULTINOMIAL, abi.FP32),
        ("d1 ragged", lambda: models.lgssm_check(45), 100, abi.MULTINOMIAL, abi.FP32),
        ("sv lazy", lambda: models.sv(300), 513, abi.MH_LAZY, abi.FP32),
        ("cox", lambda: models.cox(77), 200, abi.SYSTEMATIC, abi.FP32),
        ("cv fp64", lambda: models.cv_tracking(40), 96, abi.MULTINOMIAL, abi.FP64_PARITY),
        ("crw rejection", lambda: models.constrained_rw(60), 150, abi.REJECTION_LAZY, abi.FP32),
        ("cv small", lambda: models.cv_tracking(9), 33, abi.MULTINOMIAL, abi.FP32),
        ("cv big again", lambda: models.cv_tracking(1023), 1024, abi.MULTINOMIAL, abi.FP32),
    ]


def _run(e, make, N, rs, prec):
    return e.smooth(make(), N, rs, seed=11, precision=prec, want_paths=True)


def test_long_lived_context_matches_fresh_contexts():
    shared = Engine(0)
    try:
        for label, make, N, rs, prec in _calls():
            a = _run(shared, make, N, rs, prec)
            fresh = Engine(0)
            try:
                b = _run(fresh, make, N, rs, prec)
            finally:
                fresh.close()
            for key in ("paths", "mean", "cov"):
                assert np.array_equal(a[key], b[key]), f"{label}: {key} depends on context history"
            assert a["log_norm_const"] == b["log_norm_const"], label
    finally:
        shared.close()


def test_conditional_sweep_context_history(engine):
    """c-dSMC with a batch size and N that differ from the calls before it
    (the session engine has run other tests) equals a fresh context's sweep."""
    m = models.lgssm_check(63)
    K = m.horizon + 1
    refs = np.linspace(-1, 1, 5 * K).reshape(5, K, 1)
    seeds = np.arange(5) + 300
    a = engine.conditional_sweep([m] * 5, refs, seeds, 77, 2)
    fresh = Engine(0)
    try:
        b = fresh.conditional_sweep([m] * 5, refs, seeds, 77, 2)
    finally:
        fresh.close()
    assert np.array_equal(a["paths"], b["paths"])
    assert np.array_equal(a["changed"], b["changed"])

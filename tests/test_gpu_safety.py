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


def test_resident_results_follow_the_last_run_not_the_capacity():
    """A resident run with a smaller K after a larger one: the results copy
    exactly the last run's (K, d) / (K, d, d) (the copy used the
    allocation size) and equal the same run through dsmc_smooth."""
    e = Engine(0)
    try:
        big, small = models.cv_tracking(511), models.lgssm_check(40)
        hb = e.upload(big)
        e.smooth_resident(hb, 256, seed=3)
        e.sync()
        hs = e.upload(small)
        e.smooth_resident(hs, 64, seed=9)
        K, d = small.horizon + 1, small.d
        mbuf, mean = _guarded((K, d))
        cbuf, cov = _guarded((K, d, d))
        import ctypes as C
        lnc, has = C.c_double(), C.c_int()
        e._check(e.lib.dsmc_resident_results(e.ctx, abi.dptr(mean), abi.dptr(cov),
                                             C.byref(lnc), C.byref(has)))
        assert (mbuf[K * d:] == SENTINEL).all() and (cbuf[K * d * d:] == SENTINEL).all()
        ref = e.smooth(small, 64, seed=9)
        assert np.array_equal(mean, ref["mean"]) and np.array_equal(cov, ref["cov"])
        e.free_model(hb)
        e.free_model(hs)
    finally:
        e.close()


def test_resident_run_reports_device_errors():
    """A NaN leaf weight raised on the device during a resident run surfaces
    at the next host synchronisation (dsmc_resident_results / dsmc_sync)
    instead of returning DSMC_OK with garbage moments."""
    m = models.lgssm_check(31)
    A = dict(m.arrays)
    y = np.array(A["y"])
    y[0, 0] = np.nan
    A["y"] = y
    bad = abi.Model(m.kind, m.horizon, m.d, m.dy, **A)
    e = Engine(0)
    try:
        h = e.upload(bad)
        e.smooth_resident(h, 64, seed=1)  # enqueues, returns OK
        with pytest.raises(ArithmeticError, match="NaN"):
            e.resident_results(32, 1)
        e.smooth_resident(h, 64, seed=2)
        with pytest.raises(ArithmeticError, match="NaN"):
            e.sync()
        e.free_model(h)
        good = e.upload(m)  # the context stays usable
        e.smooth_resident(good, 64, seed=1)
        mean, cov, lnc = e.resident_results(32, 1)
        assert np.isfinite(mean).all()
        e.free_model(good)
    finally:
        e.close()


def test_leaf_outputs_fp64_only(engine):
    m = models.lgssm_check(9)
    r = engine.smooth(m, 16, seed=4, precision=abi.FP64_PARITY, want_leaves=True,
                      want_leaf_logw=True)
    lw = r["leaf_logw"]
    # normalised per leaf (BlockEstimate::log_w): logsumexp == 0
    mx = lw.max(1, keepdims=True)
    assert np.allclose(np.log(np.exp(lw - mx).sum(1)) + mx[:, 0], 0.0, atol=1e-12)
    with pytest.raises(ValueError, match="FP64"):
        engine.smooth(m, 16, seed=4, precision=abi.FP32, want_leaf_logw=True)


def test_fp64_dense_column_stage_limit(engine):
    """The FP64 dense combine stages the right block's columns in shared
    memory; an N beyond it is refused with the bound in the message instead of
    a raw launch failure."""
    m = models.cv_tracking(3)
    with pytest.raises(ValueError, match="column stage"):
        engine.smooth(m, 8192, abi.MULTINOMIAL, seed=1, precision=abi.FP64_PARITY)
    r = engine.smooth(m, 2048, abi.MULTINOMIAL, seed=1, precision=abi.FP64_PARITY)
    assert np.isfinite(r["log_norm_const"])

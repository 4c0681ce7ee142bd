"""Wide-state FP32 path (5 <= d <= 32, csrc/wide.cuh): linear-Gaussian
models beyond the float4 layout (VERDICT r1 missing 3; the reference's
FeynmanKacModel has no bound on state_dim, fk_model.hpp:38). d independent
AR(1) coordinates (models.ar_iid: d = 8, 16, 32; stacked CV trackers make
every dSMC run, the CPU reference's included, collapse onto one path at
d = 8) against the exact Kalman/RTS smoother and the compiled CPU
reference, in the seed-averaged standard-error units of
test_gpu_stat.py::test_cv_d4_means_match_kalman (test_smoother.cpp:292-341);
and the wide kernels forced on the d = 4 model (DSMC_FORCE_WIDE) against the
float4 path."""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2202_02264_b200 import abi, models

pytestmark = pytest.mark.gpu


def _seed_avg(engine, m, N, seeds):
    runs = [engine.smooth(m, N, abi.MULTINOMIAL, seed=s, precision=abi.FP32) for s in seeds]
    means = np.stack([r["mean"] for r in runs])
    return means.mean(0), means.std(0, ddof=1) / np.sqrt(len(seeds)), runs


@pytest.mark.parametrize("d", [8, 16, 32])
def test_wide_means_match_kalman(engine, d):
    """d independent AR(1) coordinates (models.ar_iid, rho = 0.5): smoothed
    means in seed-averaged SE units, per-time variances, and log Z against
    the exact Kalman/RTS answers."""
    T, N = 127, 1024
    m = models.ar_iid(T, d)
    km, kP, ll = models.kalman_smooth_numpy(m)
    avg, se, runs = _seed_avg(engine, m, N, range(16))
    z = (avg - km) / np.maximum(se, 1e-12)
    assert np.sqrt(np.mean(z ** 2)) < 2.0, np.sqrt(np.mean(z ** 2))
    assert np.mean(np.abs(z) > 4.0) < 0.01
    assert np.abs(z).max() < 10.0
    r = runs[0]
    assert r["mean"].shape == (T + 1, d) and r["cov"].shape == (T + 1, d, d)
    ratio = np.einsum("tii->ti", np.stack([x["cov"] for x in runs]).mean(0)) / np.einsum("tii->ti", kP)
    assert 0.75 < np.median(ratio) < 1.1, np.median(ratio)
    lz = np.array([x["log_norm_const"] for x in runs])
    lme = np.log(np.mean(np.exp(lz - lz.max()))) + lz.max()
    assert abs(lme - ll) < 3.0, (lme, ll)


def test_wide_matches_cpu_reference(engine, reference):
    """The same d = 16 model through the compiled reference's run_smoother
    (FP64, scalar callbacks + chained gaussian_row fast path, oracle/
    ref_models.cpp) and the wide FP32 path: 8-seed log Z and per-time
    mean averages agree within Monte Carlo error."""
    T, N, d = 63, 1024, 16
    m = models.ar_iid(T, d)
    ref = [reference.run_smoother(m, N, abi.MULTINOMIAL, seed=s, threads=8) for s in range(8)]
    gpu = [engine.smooth(m, N, abi.MULTINOMIAL, seed=100 + s, precision=abi.FP32)
           for s in range(8)]
    la = np.array([x["log_norm_const"] for x in ref])
    lb = np.array([x["log_norm_const"] for x in gpu])
    se = np.sqrt(la.var(ddof=1) / 8 + lb.var(ddof=1) / 8)
    assert abs(la.mean() - lb.mean()) < 5 * se + 0.05, (la.mean(), lb.mean(), se)
    ma = np.stack([x["paths"].mean(1) for x in ref])
    mb = np.stack([x["mean"] for x in gpu])
    z = (ma.mean(0) - mb.mean(0)) / np.sqrt(ma.var(0, ddof=1) / 8 + mb.var(0, ddof=1) / 8 + 1e-12)
    assert np.sqrt(np.mean(z ** 2)) < 2.0
    assert np.abs(z).max() < 8.0


def test_wide_rejects_unsupported_modes(engine):
    m = models.ar_iid(15, 8)
    for kw in (dict(precision=abi.FP64_PARITY), dict(resampler=abi.MH_LAZY)):
        args = dict(resampler=abi.MULTINOMIAL, precision=abi.FP32)
        args.update(kw)
        with pytest.raises(ValueError, match="state_dim > 4"):
            engine.smooth(m, 64, args["resampler"], seed=1, precision=args["precision"])


_FORCED = r"""
import sys, json
sys.path.insert(0, sys.argv[1])
import numpy as np
from paper_2202_02264_b200 import abi, models
from paper_2202_02264_b200.dsmc import Engine
e = Engine(0)
m = models.cv_tracking(127)
rows = [e.smooth(m, 1024, abi.MULTINOMIAL, seed=s, precision=abi.FP32) for s in range(16)]
np.save(sys.argv[2], np.stack([r["mean"] for r in rows]))
print(json.dumps([r["log_norm_const"] for r in rows]))
"""


def test_forced_wide_matches_float4_path(engine, tmp_path):
    """The same d = 4 model through the wide kernels (DSMC_FORCE_WIDE=1, a
    separate process) and the float4 kernels: seed-averaged means agree
    within 5 combined standard errors and log Z within Monte Carlo noise."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = tmp_path / "wide.npy"
    r = subprocess.run([sys.executable, "-c", _FORCED, root, str(out)], capture_output=True,
                       text=True, timeout=600, env=dict(os.environ, DSMC_FORCE_WIDE="1"))
    assert r.returncode == 0, r.stderr
    wide = np.load(out)
    m = models.cv_tracking(127)
    a, sa, runs = _seed_avg(engine, m, 1024, range(16))
    b, sb = wide.mean(0), wide.std(0, ddof=1) / np.sqrt(16)
    z = (a - b) / np.sqrt(sa ** 2 + sb ** 2)
    assert np.sqrt(np.mean(z ** 2)) < 2.0
    assert np.abs(z).max() < 6.0
    import json
    lzw = np.array(json.loads(r.stdout.strip().splitlines()[-1]))
    lzf = np.array([x["log_norm_const"] for x in runs])
    assert abs(np.median(lzw) - np.median(lzf)) < 2.0


def test_wide_systematic_matches_kalman(engine):
    """The wide sampler's systematic branch (one shared uniform, sorted
    points) against the exact smoother, same units as above."""
    T, N, d = 63, 1024, 8
    m = models.ar_iid(T, d)
    km, kP, _ = models.kalman_smooth_numpy(m)
    runs = [engine.smooth(m, N, abi.SYSTEMATIC, seed=s, precision=abi.FP32) for s in range(8)]
    means = np.stack([r["mean"] for r in runs])
    z = (means.mean(0) - km) / np.maximum(means.std(0, ddof=1) / np.sqrt(8), 1e-12)
    assert np.sqrt(np.mean(z ** 2)) < 2.0, np.sqrt(np.mean(z ** 2))
    ratio = np.einsum("tii->ti", runs[0]["cov"]) / np.einsum("tii->ti", kP)
    assert 0.7 < np.median(ratio) < 1.2


@pytest.mark.parametrize("which,msg", [("prop_cov", "proposal covariance at time 5"),
                                       ("R", "R at time 9"), ("Q", "Q at time 7")])
def test_wide_prep_reports_the_failing_time(engine, which, msg):
    """The device model prep (prepw_kernel) factors every per-time matrix;
    a non-positive-definite one is reported with its kind and time, as the
    host prep did (the smallest failing time wins)."""
    T, d = 15, 8
    m = models.ar_iid(T, d)
    A = dict(m.arrays)
    K = T + 1
    t = {"prop_cov": 5, "R": 9, "Q": 7}[which]
    if which != "prop_cov":  # make the matrix time-varying first
        A[which] = np.tile(np.asarray(A[which]).reshape(d, d), (K, 1, 1))
    bad = np.array(A[which], dtype=np.float64).reshape(K, d, d).copy()
    bad[t] = -np.eye(d)
    bad[t + 3] = -np.eye(d)
    A[which] = bad
    m2 = abi.Model(m.kind, m.horizon, m.d, m.dy, **A)
    with pytest.raises(ValueError, match=msg):
        engine.smooth(m2, 64, abi.MULTINOMIAL, seed=1, precision=abi.FP32)

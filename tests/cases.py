"""Shared parity cases (model + sizes + seeds) for golden generation and tests.

Models are rebuilt from the arrays stored in the golden file, so a fixture
never depends on re-running data simulation or the Kalman proposals.
"""
import numpy as np

from paper_2202_02264_b200 import abi, models

# experiment.cpp:42-45: seed + ((method + 1) << 32) + replicate
C1_SEED = 1 + (1 << 32) + 0

MULT, SYS, MH, REJ = abi.MULTINOMIAL, abi.SYSTEMATIC, abi.MH_LAZY, abi.REJECTION_LAZY

CASES = {
    # BASELINE config 1: d=1 LGSSM, T+1 = 2^10, N = 100 (experiment.hpp:20-27)
    "c1": dict(kind="lgssm_check", T=1023, N=100, seed=C1_SEED, resamplers=[MULT]),
    "lg_small": dict(kind="lgssm_check", T=30, N=37, seed=5, resamplers=[MULT, SYS, MH],
                     mh_steps=4),
    "odd": dict(kind="lgssm_check", T=6, N=9, seed=3, resamplers=[MULT, SYS]),
    "t0": dict(kind="lgssm_check", T=0, N=16, seed=2, resamplers=[MULT]),
    "sv": dict(kind="sv", T=40, N=50, seed=7, resamplers=[MULT, SYS, MH, REJ], mh_steps=4,
               sweeps=[0, 3]),
    "cv": dict(kind="cv", T=20, N=33, seed=9, resamplers=[MULT, SYS]),
    "ar1": dict(kind="ar1", T=23, N=40, seed=11, resamplers=[MULT, REJ], sweeps=[1]),
    # the reference's own benchmark models (models.cpp:111-338), SURVEY 8f.1
    "cox": dict(kind="cox", T=40, N=50, seed=13, resamplers=[MULT, SYS, MH], mh_steps=4,
                sweeps=[0, 2], par=(0.5, 0.9, 0.25, 1.0)),
    "crw": dict(kind="crw", T=30, N=37, seed=17, resamplers=[MULT, SYS, MH, REJ], mh_steps=4,
                sweeps=[1], par=(0.3,)),
    # IEKS marginals inflated x3 so every cut has a finite bound (rejection)
    "theta": dict(kind="theta", T=40, N=37, seed=19, resamplers=[MULT, SYS, MH, REJ],
                  mh_steps=4, sweeps=[0], par=(0.15, 0.10, 0.10, 0.05, 0.05), inflation=3.0),
}

# table resampling fixtures: n, n_out, spread (nats), dead fraction, seed
TABLES = {
    "n3": (3, 3000, 3.0, 0.0, 11),
    "n100": (100, 100, 10.0, 0.01, 12),
    "n300": (300, 300, 41.0, 0.01, 13),
    "n130": (130, 500, 6.0, 0.0, 14),
}

AR1_POOL = [0.4, -0.1, 0.9, 1.3, 0.2, -0.7, -0.2, 0.5, 1.1, 0.3, -0.4, 0.1,
            0.8, -0.9, 0.0, 0.6, -0.3, 0.7, 1.0, -0.5, 0.2, -0.8, 0.35, 0.15]


def table(name):
    n, n_out, spread, dead, seed = TABLES[name]
    rng = np.random.default_rng(seed)
    lw = spread * (rng.random((n, n)) - 0.5)
    lw[rng.random((n, n)) < dead] = -np.inf
    return lw, n_out, seed


def model_for(spec):
    T = spec["T"]
    if spec["kind"] == "lgssm_check":
        return models.lgssm_check(T)
    if spec["kind"] == "sv":
        # |eta| = 1 keeps every |y_t| away from 0, so the rejection bound
        # -0.5 log(2 pi s2) - log|y_t| is not astronomically loose
        rng = np.random.default_rng(90210)
        x = -1.0 + 0.3 * rng.standard_normal(T + 1)
        ys = np.exp(x / 2) * np.where(rng.random(T + 1) < 0.5, -1.0, 1.0)
        return models.sv(T, ys=ys)
    if spec["kind"] == "cv":
        return models.cv_tracking(T)
    if spec["kind"] == "ar1":
        return models.ar1([AR1_POOL[t % len(AR1_POOL)] for t in range(T + 1)])
    if spec["kind"] == "cox":
        mu, rho, s2, lam = spec["par"]
        return models.cox(T, mu, rho, s2, lam)
    if spec["kind"] == "crw":
        return models.constrained_rw(T, spec["par"][0])
    if spec["kind"] == "theta":
        return models.theta_logistic(T, *spec["par"], inflation=spec["inflation"])
    raise ValueError(spec["kind"])


def model_arrays(m):
    return {k: v for k, v in m.arrays.items() if v is not None}


def rebuild(spec, arrays):
    """Model from stored arrays (golden) with the spec's kind."""
    kind = spec["kind"]
    T = spec["T"]
    if kind == "sv":
        return abi.Model(abi.MODEL_SV, T, 1, 1, y=arrays["y"], sv=(-1.0, 0.95, 0.09))
    if kind == "cox":
        return abi.Model(abi.MODEL_COX, T, 1, 1, y=arrays["y"], par=spec["par"])
    if kind == "crw":
        return abi.Model(abi.MODEL_CRW, T, 1, 1, par=spec["par"])
    if kind == "theta":
        return abi.Model(abi.MODEL_THETA, T, 1, 1, y=arrays["y"], prop_mean=arrays["prop_mean"],
                         prop_cov=arrays["prop_cov"], par=spec["par"])
    d = 4 if kind == "cv" else 1
    dy = 2 if kind == "cv" else 1
    return abi.Model(abi.MODEL_LGSSM, T, d, dy, **arrays)

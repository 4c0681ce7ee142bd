"""Dense-grid forward-backward for scalar state-space models — a numpy
restatement of the reference's test oracle (tests/support/grid_oracle.hpp:
63-129: rectangle-rule filter alpha, normalised backward beta, smoothing
mean / variance, log Z). TEST INFRASTRUCTURE ONLY.

Used as the exact answer for the device models without a Kalman solution
(Cox counts, constrained random walk).
"""
import numpy as np
from scipy.special import gammaln

L2P = np.log(2 * np.pi)


def _lnorm(x, m, v):
    return -0.5 * (L2P + np.log(v)) - (x - m) ** 2 / (2 * v)


def model_fns(model):
    """(init_logdensity, transition_logdensity(xp, xc), log_potential(t, x),
    grid lo, hi) of a DSMC_MODEL_COX / DSMC_MODEL_CRW descriptor."""
    from paper_2202_02264_b200 import abi
    if model.kind == abi.MODEL_COX:
        mu, rho, s2, lam = model.par[:4]
        a, b = rho * lam, mu * (1 - rho)
        m, v = b / (1 - a), s2 / (1 - a * a)
        y = model.arrays["y"]
        return (lambda x: _lnorm(x, m, v),
                lambda xp, xc: _lnorm(xc, b + a * xp, s2),
                lambda t, x: y[t] * x - np.exp(x) - gammaln(y[t] + 1),
                m - 9 * np.sqrt(v), m + 9 * np.sqrt(v))
    if model.kind == abi.MODEL_CRW:
        s2 = model.par[0] ** 2
        return (lambda x: _lnorm(x, 0.0, 1.0),
                lambda xp, xc: _lnorm(xc, xp, s2),
                lambda t, x: np.where(np.abs(x) <= 1.0, 0.0, -np.inf),
                -1.0, 1.0)
    if model.kind == abi.MODEL_THETA:
        tau0, tau1, tau2, q2, r2 = model.par[:5]
        y = model.arrays["y"]
        drift = lambda x: x + tau0 - tau1 * np.exp(tau2 * x)
        lo, hi = float(np.min(y)) - 3.0, float(np.max(y)) + 3.0
        return (lambda x: _lnorm(x, 0.0, 1.0),
                lambda xp, xc: _lnorm(xc, drift(xp), q2),
                lambda t, x: _lnorm(y[t], x, r2),
                lo, hi)
    raise ValueError("grid oracle: scalar COX / CRW / THETA models only")


def grid_truth(model, cells=2000):
    init, trans, pot, lo, hi = model_fns(model)
    T = model.horizon
    xs = np.linspace(lo, hi, cells + 1)
    step = (hi - lo) / cells
    P = np.exp(trans(xs[:, None], xs[None, :]))  # P[i, k] = p(x_k | x_i)
    alpha = np.empty((T + 1, xs.size))
    alpha[0] = np.exp(init(xs) + pot(0, xs)) * step
    log_scale = 0.0
    for t in range(1, T + 1):
        tot = alpha[t - 1].sum()
        log_scale += np.log(tot)
        alpha[t - 1] /= tot
        alpha[t] = (alpha[t - 1] @ P) * np.exp(pot(t, xs)) * step
    tot = alpha[T].sum()
    log_z = log_scale + np.log(tot)
    alpha[T] /= tot
    beta = np.ones_like(alpha)
    for t in range(T - 1, -1, -1):
        beta[t] = P @ (np.exp(pot(t + 1, xs)) * beta[t + 1] * step)
        beta[t] /= beta[t].sum()
    g = alpha * beta
    g /= g.sum(1, keepdims=True)
    mean = g @ xs
    var = g @ xs ** 2 - mean ** 2
    return mean, var, log_z

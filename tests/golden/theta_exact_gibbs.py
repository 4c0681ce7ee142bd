"""TEST INFRASTRUCTURE: the exact posterior means quoted in
tests/cpp/test_host.cpp (theta_logistic_conjugate_only_chain_recovers_precisions).

Data: simulate_theta_logistic(tau0 = 0.1, tau1 = tau2 = 1e-8, q2 = 0.25,
r2 = 0.09, T = 150, seed 99) through the reference's Philox stream
(models.cpp:517-540, restated over oracle/_ref's philox as in
make_harness_golden.py). With tau1 ~ 0 the model is linear-Gaussian, so a
Gibbs sampler with exact Kalman/FFBS path draws and the conjugate precision
updates (pgibbs.cpp:142-186, Gamma(2, 1) priors) gives the exact posterior
of (q2, r2).   python tests/golden/theta_exact_gibbs.py
"""
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from make_harness_golden import Stream  # noqa: E402
from oracle.py import Reference  # noqa: E402


def simulate(ref, T, seed, tau0, tau1, tau2, q2, r2):
    st = Stream(ref, seed, 0, 1, 5)
    xs = [st.normal()]
    for _ in range(T):
        p = xs[-1]
        xs.append(p + tau0 - tau1 * math.exp(tau2 * p) + math.sqrt(q2) * st.normal())
    return np.array([x + math.sqrt(r2) * st.normal() for x in xs])


def main():
    ys = simulate(Reference(), 150, 99, 0.1, 1e-8, 1e-8, 0.25, 0.09)
    T = len(ys) - 1
    drift = 0.1 - 1e-8
    rng = np.random.default_rng(0)
    q2, r2 = 0.25, 0.09
    qs, rs = [], []
    for it in range(4000):
        K = T + 1
        mf, Pf, mp, Pp = np.empty(K), np.empty(K), np.empty(K), np.empty(K)
        for t in range(K):
            mp[t], Pp[t] = (0.0, 1.0) if t == 0 else (mf[t - 1] + drift, Pf[t - 1] + q2)
            g = Pp[t] / (Pp[t] + r2)
            mf[t], Pf[t] = mp[t] + g * (ys[t] - mp[t]), (1 - g) * Pp[t]
        x = np.empty(K)
        x[-1] = mf[-1] + math.sqrt(Pf[-1]) * rng.standard_normal()
        for t in range(K - 2, -1, -1):
            J = Pf[t] / Pp[t + 1]
            x[t] = mf[t] + J * (x[t + 1] - mp[t + 1]) + math.sqrt(Pf[t] - J * Pf[t]) * rng.standard_normal()
        ssx = np.sum((x[1:] - x[:-1] - drift) ** 2)
        ssy = np.sum((ys - x) ** 2)
        q2 = 1.0 / rng.gamma(2.0 + 0.5 * T, 1.0 / (1.0 + 0.5 * ssx))
        r2 = 1.0 / rng.gamma(2.0 + 0.5 * (T + 1), 1.0 / (1.0 + 0.5 * ssy))
        if it >= 500:
            qs.append(q2)
            rs.append(r2)
    print("exact posterior means: q2 %.4f r2 %.4f" % (np.mean(qs), np.mean(rs)))


if __name__ == "__main__":
    main()

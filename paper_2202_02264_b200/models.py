"""Host-side model builders for the BASELINE configurations.

These play the role of the reference harness's prepare() (experiment.cpp:
436-468): simulate synthetic data, build the proposal marginals (exact RTS
smoother, the reference's make_lgssm_fk recipe: q_t = nu_t = smoothing
marginals), and hand a plain-data descriptor (abi.Model) to the engine.

  lgssm_check  C1: d=1 LGSSM of experiment.hpp:20-27 (coef 0.9, Q 0.25,
               x0 ~ N(0,1), R 0.25)
  cv_tracking  C2/C5: d=4 2-D constant-velocity model
  sv           C3/C4: stochastic volatility
  ar1          the reference test fixture tests/support/ar1.hpp (stationary
               proposals)
"""
import numpy as np
from scipy.signal import lfilter

from . import abi


def _lgssm(T, d, dy, m0, P0, F, b, Q, H, R, y, prop_mean=None, prop_cov=None,
           has_obs=None, inflation=1.0):
    K = T + 1
    if prop_mean is None:
        prop_mean = np.zeros((K, d))
        prop_cov = np.tile(np.eye(d), (K, 1, 1))
    m = abi.Model(abi.MODEL_LGSSM, T, d, dy, m0=m0, P0=P0, F=F, b=b, Q=Q, H=H,
                  R=R, y=y, has_obs=has_obs, prop_mean=prop_mean, prop_cov=prop_cov)
    return m


def with_rts_proposals(model, inflation=1.0, smoother=None):
    """Replace the proposals by the exact smoothing marginals (x inflation).
    smoother: model -> (means, covs, loglik); default the engine's host RTS
    (dsmc_kalman_smooth). bench.py's reference arm passes the oracle's so its
    process never maps the product library."""
    if smoother is None:
        from .dsmc import kalman_smooth as smoother
    mean, cov, _ = smoother(model)
    A = dict(model.arrays)
    A["prop_mean"] = mean
    A["prop_cov"] = cov * inflation
    out = abi.Model(model.kind, model.horizon, model.d, model.dy, **A)
    return out


def lgssm_check(T, coef=0.9, shift=0.0, trans_var=0.25, init_mean=0.0,
                init_var=1.0, obs_var=0.25, data_seed=90210, ys=None,
                inflation=1.0, smoother=None):
    """C1 (experiment.hpp:20-27, experiment.cpp:367-381)."""
    K = T + 1
    if ys is None:
        rng = np.random.default_rng(data_seed)
        x0 = init_mean + np.sqrt(init_var) * rng.standard_normal()
        e = np.sqrt(trans_var) * rng.standard_normal(K)
        e[0] = x0
        x = lfilter([1.0], [1.0, -coef], e + np.r_[0.0, np.full(T, shift)])
        ys = x + np.sqrt(obs_var) * rng.standard_normal(K)
    m = _lgssm(T, 1, 1, [init_mean], [[init_var]], [coef], [shift], [trans_var],
               [1.0], [obs_var], np.asarray(ys, float).reshape(K, 1))
    return with_rts_proposals(m, inflation, smoother)


def ar1(ys, rho=0.8, q=0.3, r=0.4):
    """tests/support/ar1.hpp:23-126: stationary proposals N(0, q/(1-rho^2))."""
    T = len(ys) - 1
    K = T + 1
    s2 = q / (1.0 - rho * rho)
    return _lgssm(T, 1, 1, [0.0], [[s2]], [rho], [0.0], [q], [1.0], [r],
                  np.asarray(ys, float).reshape(K, 1),
                  prop_mean=np.zeros((K, 1)), prop_cov=np.full((K, 1, 1), s2))


def cv_matrices(q=0.05, r=0.3, dt=1.0):
    I2 = np.eye(2)
    F = np.block([[I2, dt * I2], [np.zeros((2, 2)), I2]])
    Q = q * np.block([[dt ** 3 / 3 * I2, dt ** 2 / 2 * I2], [dt ** 2 / 2 * I2, dt * I2]])
    H = np.hstack([I2, np.zeros((2, 2))])
    R = r * I2
    return F, Q, H, R


def cv_tracking(T, q=0.05, r=0.3, data_seed=90210, inflation=1.0, smoother=None):
    """C2 / C5: x = (p_x, p_y, v_x, v_y), white-noise acceleration."""
    K = T + 1
    F, Q, H, R = cv_matrices(q, r)
    rng = np.random.default_rng(data_seed)
    Lq = np.linalg.cholesky(Q)
    w = rng.standard_normal((K, 4)) @ Lq.T
    w[0] = rng.standard_normal(4)  # x0 ~ N(0, I)
    # x_t = F x_{t-1} + w_t with F = [[I, I], [0, I]]: v = cumsum(w_v),
    # p_t = p_{t-1} + v_{t-1} + w_p,t
    v = np.cumsum(w[:, 2:], axis=0)
    vprev = np.vstack([np.zeros((1, 2)), v[:-1]])
    p = np.cumsum(w[:, :2] + vprev, axis=0)
    x = np.hstack([p, v])
    y = x[:, :2] + np.sqrt(r) * rng.standard_normal((K, 2))
    m = _lgssm(T, 4, 2, np.zeros(4), np.eye(4), F, np.zeros(4), Q, H, R, y)
    return with_rts_proposals(m, inflation, smoother)


def sv(T, mu=-1.0, phi=0.95, sigma=0.3, data_seed=90210, ys=None):
    """C3 / C4: x_t = mu + phi (x_{t-1} - mu) + sigma e, y_t ~ N(0, e^{x_t})."""
    K = T + 1
    if ys is None:
        rng = np.random.default_rng(data_seed)
        s2 = sigma * sigma
        e = sigma * rng.standard_normal(K)
        e[0] = np.sqrt(s2 / (1 - phi * phi)) * rng.standard_normal()
        x = mu + lfilter([1.0], [1.0, -phi], e)
        ys = np.exp(x / 2) * rng.standard_normal(K)
    return abi.Model(abi.MODEL_SV, T, 1, 1, y=np.asarray(ys, float),
                     sv=(mu, phi, sigma * sigma))


def cox(T, mu=0.0, rho=0.9, sigma2=0.25, lam=1.0, data_seed=90210, ys=None):
    """Log-Gaussian Cox counts (make_cox_model, models.cpp:111-216; defaults
    = dsmc::CoxParams): x_t = mu(1 - rho) + rho lam x_{t-1} + N(0, sigma2),
    y_t ~ Poisson(exp x_t); counts simulated with numpy unless given."""
    K = T + 1
    if ys is None:
        rng = np.random.default_rng(data_seed)
        a, b = rho * lam, mu * (1.0 - rho)
        x = np.empty(K)
        x[0] = b / (1 - a) + np.sqrt(sigma2 / (1 - a * a)) * rng.standard_normal()
        for t in range(1, K):
            x[t] = b + a * x[t - 1] + np.sqrt(sigma2) * rng.standard_normal()
        ys = rng.poisson(np.exp(x)).astype(np.float64)
    return abi.Model(abi.MODEL_COX, T, 1, 1, y=np.asarray(ys, np.float64),
                     par=(mu, rho, sigma2, lam))


def constrained_rw(T, sigma=0.3):
    """Random walk conditioned to stay in [-1, 1] (make_constrained_rw,
    models.cpp:263-338)."""
    return abi.Model(abi.MODEL_CRW, T, 1, 1, par=(sigma,))


def theta_logistic_marginals(T, ys, tau0, tau1, tau2, q2, r2, iterations=10, inflation=1.0):
    """Proposal marginals by the iterated extended Kalman smoother
    (iterated_smooth, kalman.cpp:220-243): linearise the drift around the
    previous smoothed means (linearize, :192-218, analytic Jacobian as
    f_jac, models.cpp:387-391), run the exact Kalman/RTS smoother of the
    linearised LGSSM (dsmc_kalman_smooth), repeat."""
    from .dsmc import kalman_smooth
    K = T + 1
    f = lambda x: x + tau0 - tau1 * np.exp(tau2 * x)
    ref = np.zeros(K)
    for t in range(1, K):
        ref[t] = f(ref[t - 1])
    for _ in range(iterations):
        F = np.ones(K)
        b = np.zeros(K)
        F[1:] = 1.0 - tau1 * tau2 * np.exp(tau2 * ref[:-1])
        b[1:] = f(ref[:-1]) - F[1:] * ref[:-1]
        lin = _lgssm(T, 1, 1, [0.0], [[1.0]], F.reshape(K, 1, 1), b.reshape(K, 1), [q2],
                     [1.0], [r2], np.asarray(ys, float).reshape(K, 1),
                     prop_mean=np.zeros((K, 1)), prop_cov=np.ones((K, 1, 1)))
        km, kP, _ = kalman_smooth(lin)
        ref = km[:, 0]
    return km[:, 0], inflation * kP[:, 0, 0]


def theta_logistic(T, tau0=0.15, tau1=0.10, tau2=0.10, q2=0.05, r2=0.05, data_seed=90210,
                   ys=None, inflation=1.0):
    """Theta-logistic population dynamics (make_theta_logistic,
    models.cpp:407-491; defaults = dsmc::ThetaLogisticParams) with IEKS
    proposal marginals; data simulated with numpy unless given."""
    K = T + 1
    if ys is None:
        rng = np.random.default_rng(data_seed)
        x = np.empty(K)
        x[0] = rng.standard_normal()
        for t in range(1, K):
            x[t] = x[t - 1] + tau0 - tau1 * np.exp(tau2 * x[t - 1]) + np.sqrt(q2) * rng.standard_normal()
        ys = x + np.sqrt(r2) * rng.standard_normal(K)
    ys = np.asarray(ys, np.float64)
    pm, pv = theta_logistic_marginals(T, ys, tau0, tau1, tau2, q2, r2, inflation=inflation)
    return abi.Model(abi.MODEL_THETA, T, 1, 1, y=ys, prop_mean=pm.reshape(K, 1),
                     prop_cov=pv.reshape(K, 1, 1), par=(tau0, tau1, tau2, q2, r2))


def kalman_smooth_numpy(model):
    """Kalman filter + RTS smoother of an LGSSM Model of any state dimension
    (kalman.cpp:78-138 in numpy, Joseph-form update, symmetrised): the
    proposal builder for the wide-state path (d > 4), where the host /
    device engine smoothers (d <= 4) do not apply. -> (means, covs, loglik)."""
    A = model.arrays
    K, d, dy = model.horizon + 1, model.d, model.dy
    F = A["F"].reshape(-1, d, d)
    Q = A["Q"].reshape(-1, d, d)
    H = A["H"].reshape(-1, dy, d)
    R = A["R"].reshape(-1, dy, dy)
    b = A["b"].reshape(-1, d)
    y = A["y"].reshape(K, dy)
    obs = A.get("has_obs")

    def g(X, t):
        return X[t if len(X) > 1 else 0]

    def sym(P):
        return 0.5 * (P + P.T)
    fm, fP, pm, pP = [None] * K, [None] * K, [None] * K, [None] * K
    ll = 0.0
    I = np.eye(d)
    for t in range(K):
        if t == 0:
            pm[0], pP[0] = A["m0"].reshape(d), A["P0"].reshape(d, d)
        else:
            pm[t] = g(F, t) @ fm[t - 1] + g(b, t)
            pP[t] = sym(g(F, t) @ fP[t - 1] @ g(F, t).T + g(Q, t))
        if obs is None or obs[t]:
            Ht, Rt = g(H, t), g(R, t)
            S = sym(Ht @ pP[t] @ Ht.T + Rt)
            Ls = np.linalg.cholesky(S)
            r = y[t] - Ht @ pm[t]
            z = np.linalg.solve(Ls, r)
            ll += -0.5 * (dy * np.log(2 * np.pi) + 2 * np.log(np.diag(Ls)).sum() + z @ z)
            Kg = np.linalg.solve(S, Ht @ pP[t]).T
            fm[t] = pm[t] + Kg @ r
            Aj = I - Kg @ Ht
            fP[t] = sym(Aj @ pP[t] @ Aj.T + Kg @ Rt @ Kg.T)
        else:
            fm[t], fP[t] = pm[t], pP[t]
    sm, sP = [None] * K, [None] * K
    sm[-1], sP[-1] = fm[-1], fP[-1]
    for t in range(K - 2, -1, -1):
        G = np.linalg.solve(pP[t + 1], g(F, t + 1) @ fP[t].T).T
        sm[t] = fm[t] + G @ (sm[t + 1] - pm[t + 1])
        sP[t] = sym(fP[t] + G @ (sP[t + 1] - pP[t + 1]) @ G.T)
    return np.array(sm), np.array(sP), ll


def cv_stack(T, copies=2, q=0.05, r=0.3, data_seed=90210, inflation=1.0):
    """Wide-state LGSSM: `copies` independent 2-D constant-velocity trackers
    (C2's model) stacked block-diagonally — state dim d = 4 copies, obs dim
    2 copies (d = 8, 16, 32 for 2, 4, 8 copies) — with RTS-marginal
    proposals. Exercises the wide-state FP32 path (csrc/wide.cuh)."""
    K = T + 1
    F1, Q1, H1, R1 = cv_matrices(q, r)
    d, dy = 4 * copies, 2 * copies
    F = np.kron(np.eye(copies), F1)
    Q = np.kron(np.eye(copies), Q1)
    H = np.kron(np.eye(copies), H1)
    R = np.kron(np.eye(copies), R1)
    rng = np.random.default_rng(data_seed)
    Lq = np.linalg.cholesky(Q)
    x = np.zeros((K, d))
    x[0] = rng.standard_normal(d)
    for t in range(1, K):
        x[t] = F @ x[t - 1] + Lq @ rng.standard_normal(d)
    y = x @ H.T + np.sqrt(r) * rng.standard_normal((K, dy))
    m = _lgssm(T, d, dy, np.zeros(d), np.eye(d), F, np.zeros(d), Q, H, R, y)
    return with_rts_proposals(m, inflation, kalman_smooth_numpy)


def ar_iid(T, d, rho=0.5, q=1.0, r=1.0, data_seed=90210, inflation=1.0):
    """Wide-state LGSSM with d independent AR(1) coordinates (the d = 1
    fixture of tests/support/ar1.hpp replicated), y_t = x_t + N(0, r I):
    weakly persistent dynamics keep the pair weights' spread moderate in high
    dimension (dSMC's importance weights degenerate with d like any IS), so
    d = 8..32 runs stay informative. RTS-marginal proposals."""
    K = T + 1
    rng = np.random.default_rng(data_seed)
    s2 = q / (1 - rho * rho)
    x = np.zeros((K, d))
    x[0] = np.sqrt(s2) * rng.standard_normal(d)
    for t in range(1, K):
        x[t] = rho * x[t - 1] + np.sqrt(q) * rng.standard_normal(d)
    y = x + np.sqrt(r) * rng.standard_normal((K, d))
    I = np.eye(d)
    m = _lgssm(T, d, d, np.zeros(d), s2 * I, rho * I, np.zeros(d), q * I, I, r * I, y)
    return with_rts_proposals(m, inflation, kalman_smooth_numpy)

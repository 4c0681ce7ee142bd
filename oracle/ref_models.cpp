// ORACLE / TEST INFRASTRUCTURE ONLY — see ref_models.hpp.
#include "ref_models.hpp"

#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <vector>

#include "dsmc/kernels.hpp"

namespace oracle {
namespace {

constexpr double kLog2Pi = 1.8378770664093454836;

// models.cpp:20-23 (same expression order).
double log_normal_pdf(double x, double mean, double var) {
  const double d = x - mean;
  return -0.5 * (kLog2Pi + std::log(var)) - d * d / (2.0 * var);
}

// models.cpp:26-41.
double quadratic_sup(double alpha, double beta, double gamma) {
  if (alpha < 0.0) return gamma - beta * beta / (4.0 * alpha);
  if (alpha == 0.0 && beta == 0.0) return gamma;
  return INFINITY;
}
double obs_over_aux_sup(double y, double h, double r2, double m, double v) {
  const double alpha = 1.0 / (2.0 * v) - h * h / (2.0 * r2);
  const double beta = h * y / r2 - m / v;
  const double gamma =
      -y * y / (2.0 * r2) + m * m / (2.0 * v) + 0.5 * std::log(v / r2);
  return quadratic_sup(alpha, beta, gamma);
}

// ---------------------------------------------------------------- small LA
// Lower Cholesky of a d x d SPD matrix (row-major), then its inverse.
bool chol(const double* A, int d, double* L) {
  std::memset(L, 0, sizeof(double) * d * d);
  for (int i = 0; i < d; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = A[i * d + j];
      for (int k = 0; k < j; ++k) s -= L[i * d + k] * L[j * d + k];
      if (i == j) {
        if (!(s > 0.0)) return false;
        L[i * d + i] = std::sqrt(s);
      } else {
        L[i * d + j] = s / L[j * d + j];
      }
    }
  return true;
}
void tri_inv(const double* L, int d, double* W) {
  std::memset(W, 0, sizeof(double) * d * d);
  for (int i = 0; i < d; ++i) {
    W[i * d + i] = 1.0 / L[i * d + i];
    for (int j = 0; j < i; ++j) {
      double s = 0.0;
      for (int k = j; k < i; ++k) s += L[i * d + k] * W[k * d + j];
      W[i * d + j] = -s / L[i * d + i];
    }
  }
}

// Whitened Gaussian: log N(x; m, S) = norm - 0.5 |W (x - m)|^2.
struct Gauss {
  int d = 1;
  std::vector<double> W;  // d x d (any d: the wide-state models too)
  double norm = 0.0;  // -0.5 (d log 2pi + log det S)
  bool init(const double* S, int dd) {
    d = dd;
    std::vector<double> L(d * d);
    W.assign(d * d, 0.0);
    if (!chol(S, d, L.data())) return false;
    tri_inv(L.data(), d, W.data());
    double ld = 0.0;
    for (int i = 0; i < d; ++i) ld += 2.0 * std::log(L[i * d + i]);
    norm = -0.5 * (d * kLog2Pi + ld);
    return true;
  }
  double quad(const double* x, const double* m) const {
    double e[32];
    for (int k = 0; k < d; ++k) e[k] = x[k] - m[k];
    double q = 0.0;
    for (int k = 0; k < d; ++k) {
      double z = 0.0;
      for (int l = 0; l <= k; ++l) z += W[k * d + l] * e[l];
      q += z * z;
    }
    return q;
  }
  double logpdf(const double* x, const double* m) const {
    return norm - 0.5 * quad(x, m);
  }
};

const double* at(const double* base, int64_t stride, int t) {
  return base + stride * t;
}

// ----------------------------------------------------------------- LGSSM
struct LgCtx {
  dsmc_model_desc desc{};
  int d = 1, dy = 1, T = 0;
  std::vector<double> y, prop_mean, prop_cov, m0, P0;
  std::vector<double> F, b, Q, H, R;  // expanded per time (index 0 padding)
  std::vector<char> has_obs;
  std::vector<Gauss> prop, trans, obs;  // per time
  Gauss init;
  const double* Ft(int t) const { return F.data() + (size_t)t * d * d; }
  const double* bt(int t) const { return b.data() + (size_t)t * d; }
  const double* Ht(int t) const { return H.data() + (size_t)t * dy * d; }
  const double* yt(int t) const { return y.data() + (size_t)t * dy; }
  void mean_of(int t, const double* xp, double* mu) const {
    const double* f = Ft(t);
    const double* bb = bt(t);
    for (int k = 0; k < d; ++k) {
      double s = 0.0;
      for (int l = 0; l < d; ++l) s += f[k * d + l] * xp[l];
      mu[k] = s + bb[k];
    }
  }
  double log_h(int t, const double* x) const {
    if (!has_obs[t]) return 0.0;
    const double* h = Ht(t);
    double hx[32];
    for (int a = 0; a < dy; ++a) {
      double s = 0.0;
      for (int l = 0; l < d; ++l) s += h[a * d + l] * x[l];
      hx[a] = s;
    }
    return obs[t].logpdf(yt(t), hx);
  }
};

std::shared_ptr<LgCtx> make_lg_ctx(const dsmc_model_desc& m) {
  auto c = std::make_shared<LgCtx>();
  c->desc = m;
  c->d = m.state_dim;
  c->dy = m.obs_dim;
  c->T = m.horizon;
  const int d = c->d, dy = c->dy, K = m.horizon + 1;
  if (d < 1 || d > 32 || dy < 1 || dy > 32)
    throw std::invalid_argument("lgssm descriptor: dims must be 1..32");
  c->y.assign(m.y, m.y + (size_t)K * dy);
  c->prop_mean.assign(m.prop_mean, m.prop_mean + (size_t)K * d);
  c->prop_cov.assign(m.prop_cov, m.prop_cov + (size_t)K * d * d);
  c->m0.assign(m.m0, m.m0 + d);
  c->P0.assign(m.P0, m.P0 + d * d);
  c->F.resize((size_t)K * d * d);
  c->b.resize((size_t)K * d);
  c->Q.resize((size_t)K * d * d);
  c->H.resize((size_t)K * dy * d);
  c->R.resize((size_t)K * dy * dy);
  c->has_obs.resize(K);
  c->prop.resize(K);
  c->trans.resize(K);
  c->obs.resize(K);
  for (int t = 0; t < K; ++t) {
    std::memcpy(&c->H[(size_t)t * dy * d], at(m.H, m.H_stride, t),
                sizeof(double) * dy * d);
    std::memcpy(&c->R[(size_t)t * dy * dy], at(m.R, m.R_stride, t),
                sizeof(double) * dy * dy);
    c->has_obs[t] = m.has_obs ? (m.has_obs[t] != 0) : 1;
    if (!c->prop[t].init(&c->prop_cov[(size_t)t * d * d], d))
      throw std::invalid_argument("lgssm descriptor: proposal cov not SPD");
    if (c->has_obs[t] && !c->obs[t].init(&c->R[(size_t)t * dy * dy], dy))
      throw std::invalid_argument("lgssm descriptor: R not SPD");
    if (t >= 1) {
      std::memcpy(&c->F[(size_t)t * d * d], at(m.F, m.F_stride, t),
                  sizeof(double) * d * d);
      std::memcpy(&c->b[(size_t)t * d], at(m.b, m.b_stride, t),
                  sizeof(double) * d);
      std::memcpy(&c->Q[(size_t)t * d * d], at(m.Q, m.Q_stride, t),
                  sizeof(double) * d * d);
      if (!c->trans[t].init(&c->Q[(size_t)t * d * d], d))
        throw std::invalid_argument("lgssm descriptor: Q not SPD");
    }
  }
  if (!c->init.init(c->P0.data(), d))
    throw std::invalid_argument("lgssm descriptor: P0 not SPD");
  return c;
}

// d = 1: restatement of make_lgssm_fk (models.cpp:562-685).
dsmc::FeynmanKacModel lgssm_1d(std::shared_ptr<LgCtx> ctx) {
  dsmc::FeynmanKacModel m;
  m.state_dim = 1;
  m.horizon = ctx->T;
  auto var_of = [ctx](int t) { return ctx->prop_cov[t]; };
  auto mean_of = [ctx](int t) { return ctx->prop_mean[t]; };

  // models.cpp:583-589: fill_normal then mean + sd * z.
  m.proposal_sampler = [ctx](int t, std::size_t count, dsmc::RngStream& s,
                             double* out) {
    const double sd = std::sqrt(ctx->prop_cov[t]);
    s.fill_normal(out, count);
    for (std::size_t i = 0; i < count; ++i)
      out[i] = ctx->prop_mean[t] + sd * out[i];
  };
  m.proposal_logdensity = [ctx](int t, const double* x) {
    return log_normal_pdf(*x, ctx->prop_mean[t], ctx->prop_cov[t]);
  };
  m.aux_logdensity = m.proposal_logdensity;
  m.init_logdensity = [ctx](const double* x) {
    return log_normal_pdf(*x, ctx->m0[0], ctx->P0[0]);
  };
  m.log_potential = [ctx](int t, const double* x) {
    if (!ctx->has_obs[t]) return 0.0;
    return log_normal_pdf(ctx->y[t], ctx->H[t] * *x, ctx->R[t]);
  };
  m.transition_logdensity = [ctx](int t, const double* xp, const double* xc) {
    return log_normal_pdf(*xc, ctx->F[t] * *xp + ctx->b[t], ctx->Q[t]);
  };
  m.transition_sampler = [ctx](int t, const double* xp, dsmc::RngStream& s,
                               double* out) {
    *out = ctx->F[t] * *xp + ctx->b[t] + std::sqrt(ctx->Q[t]) * s.normal();
  };
  // models.cpp:611-636: column base then the per-row Gaussian fill.
  m.stitch_row_factory = [ctx, var_of, mean_of](int c, const double* right,
                                                std::size_t n) {
    const double qvar = ctx->Q[c];
    const double trans_norm = -0.5 * (kLog2Pi + std::log(qvar));
    auto base = std::make_shared<std::vector<double>>(n);
    double shift = trans_norm + 0.5 * (kLog2Pi + std::log(var_of(c)));
    if (ctx->has_obs[c]) {
      const double h = ctx->H[c];
      const double r = ctx->R[c];
      dsmc::kernels::gaussian_row(right, n, ctx->y[c] / h, -h * h / (2.0 * r),
                                  nullptr, base->data());
      shift += -0.5 * (kLog2Pi + std::log(r));
    } else {
      std::fill(base->begin(), base->end(), 0.0);
    }
    dsmc::kernels::gaussian_row(right, n, mean_of(c), 1.0 / (2.0 * var_of(c)),
                                base->data(), base->data());
    dsmc::kernels::add_vec_scalar(base->data(), n, shift, nullptr);
    const double F = ctx->F[c], b = ctx->b[c];
    return [base, right, n, F, b, qvar](const double* xp, double* out) {
      dsmc::kernels::gaussian_row(right, n, F * *xp + b, -1.0 / (2.0 * qvar),
                                  base->data(), out);
    };
  };
  // models.cpp:657-683: bound only when every cut is observed with a slope
  // and a proposal wider than the likelihood curvature.
  bool bounded = ctx->T >= 1;
  std::vector<double> bounds((size_t)ctx->T + 1, 0.0);
  for (int c = 1; c <= ctx->T && bounded; ++c) {
    if (!ctx->has_obs[c] || ctx->F[c] == 0.0) {
      bounded = false;
      break;
    }
    const double s = obs_over_aux_sup(ctx->y[c], ctx->H[c], ctx->R[c],
                                      mean_of(c), var_of(c));
    if (!std::isfinite(s)) {
      bounded = false;
      break;
    }
    bounds[c] = -0.5 * (kLog2Pi + std::log(ctx->Q[c])) + s;
  }
  if (bounded)
    m.log_stitch_bound = [bounds](int c) { return bounds[(size_t)c]; };
  return m;
}

// d >= 2 (up to 32, the wide-state models too): new model against the
// reference API (not in the reference).
dsmc::FeynmanKacModel lgssm_nd(std::shared_ptr<LgCtx> ctx) {
  dsmc::FeynmanKacModel m;
  const int d = ctx->d;
  m.state_dim = d;
  m.horizon = ctx->T;
  // Normal i of the stream feeds coordinate i % d of particle i / d, and the
  // particle is mean + chol(P) z (the LinearGaussian draw of kalman.cpp:43-50).
  m.proposal_sampler = [ctx, d](int t, std::size_t count, dsmc::RngStream& s,
                                double* out) {
    s.fill_normal(out, count * d);
    std::vector<double> L(d * d);
    chol(&ctx->prop_cov[(size_t)t * d * d], d, L.data());
    const double* mu = &ctx->prop_mean[(size_t)t * d];
    for (std::size_t i = 0; i < count; ++i) {
      double z[32], x[32];
      for (int k = 0; k < d; ++k) z[k] = out[i * d + k];
      for (int k = 0; k < d; ++k) {
        double acc = 0.0;
        for (int l = 0; l <= k; ++l) acc += L[k * d + l] * z[l];
        x[k] = mu[k] + acc;
      }
      for (int k = 0; k < d; ++k) out[i * d + k] = x[k];
    }
  };
  m.proposal_logdensity = [ctx, d](int t, const double* x) {
    return ctx->prop[t].logpdf(x, &ctx->prop_mean[(size_t)t * d]);
  };
  m.aux_logdensity = m.proposal_logdensity;
  m.init_logdensity = [ctx](const double* x) {
    return ctx->init.logpdf(x, ctx->m0.data());
  };
  m.log_potential = [ctx](int t, const double* x) { return ctx->log_h(t, x); };
  m.transition_logdensity = [ctx](int t, const double* xp, const double* xc) {
    double mu[32];
    ctx->mean_of(t, xp, mu);
    return ctx->trans[t].logpdf(xc, mu);
  };
  // Column base: log h_c - log nu_c + transition normaliser. Columns are
  // whitened once per combine (w_j = W_Q x_j, one slab per coordinate) and a
  // row is d chained gaussian_row passes over them (out = fma(-1/2,
  // (w_jk - v_ik)^2, out), v_i = W_Q mu_i): the reference's SIMD kernel on
  // the d = 4 model (SURVEY 8d "fair fast path").
  m.stitch_row_factory = [ctx, d](int c, const double* right, std::size_t n) {
    auto base = std::make_shared<std::vector<double>>(n);
    auto wcol = std::make_shared<std::vector<double>>(n * d);
    const Gauss& tr = ctx->trans[c];
    const double* pm = &ctx->prop_mean[(size_t)c * d];
    for (std::size_t j = 0; j < n; ++j) {
      const double* x = right + j * d;
      (*base)[j] = tr.norm + ctx->log_h(c, x) - ctx->prop[c].logpdf(x, pm);
      for (int k = 0; k < d; ++k) {
        double z = 0.0;
        for (int l = 0; l <= k; ++l) z += tr.W[k * d + l] * x[l];
        (*wcol)[k * n + j] = z;
      }
    }
    return [ctx, base, wcol, n, c, d](const double* xp, double* out) {
      double mu[32];
      ctx->mean_of(c, xp, mu);
      const Gauss& g = ctx->trans[c];
      const double* src = base->data();
      for (int k = 0; k < d; ++k) {
        double v = 0.0;
        for (int l = 0; l <= k; ++l) v += g.W[k * d + l] * mu[l];
        dsmc::kernels::gaussian_row(wcol->data() + k * n, n, v, -0.5, src, out);
        src = out;
      }
    };
  };
  return m;
}

// ------------------------------------------------------------------- SV
struct SvCtx {
  int T = 0;
  double mu = 0, phi = 0, s2 = 1;
  std::vector<double> y, logabsy;
  double log_h(int t, double x) const {  // log N(y; 0, e^x)
    return -0.5 * (kLog2Pi + x) - y[t] * y[t] / (2.0 * std::exp(x));
  }
};

dsmc::FeynmanKacModel sv_model(const dsmc_model_desc& desc) {
  auto ctx = std::make_shared<SvCtx>();
  ctx->T = desc.horizon;
  ctx->mu = desc.sv_mu;
  ctx->phi = desc.sv_phi;
  ctx->s2 = desc.sv_sigma2;
  if (!(ctx->s2 > 0.0) || !(std::fabs(ctx->phi) < 1.0))
    throw std::invalid_argument("sv descriptor: need s2 > 0 and |phi| < 1");
  ctx->y.assign(desc.y, desc.y + desc.horizon + 1);
  for (double v : ctx->y) {
    if (!(v != 0.0) || !std::isfinite(v))
      throw std::invalid_argument("sv descriptor: observations must be finite "
                                  "and nonzero");
    ctx->logabsy.push_back(std::log(std::fabs(v)));
  }
  dsmc::FeynmanKacModel m;
  m.state_dim = 1;
  m.horizon = ctx->T;
  // q_t = nu_t = |y_t| h_t: x = log y^2 - log z^2.
  m.proposal_sampler = [ctx](int t, std::size_t count, dsmc::RngStream& s,
                             double* out) {
    s.fill_normal(out, count);
    const double ly2 = 2.0 * ctx->logabsy[t];
    for (std::size_t i = 0; i < count; ++i)
      out[i] = ly2 - std::log(out[i] * out[i]);
  };
  m.proposal_logdensity = [ctx](int t, const double* x) {
    return ctx->logabsy[t] + ctx->log_h(t, *x);
  };
  m.aux_logdensity = m.proposal_logdensity;
  m.log_potential = [ctx](int t, const double* x) { return ctx->log_h(t, *x); };
  m.init_logdensity = [ctx](const double* x) {
    return log_normal_pdf(*x, ctx->mu, ctx->s2 / (1.0 - ctx->phi * ctx->phi));
  };
  m.transition_logdensity = [ctx](int, const double* xp, const double* xc) {
    return log_normal_pdf(*xc, ctx->mu + ctx->phi * (*xp - ctx->mu), ctx->s2);
  };
  m.transition_sampler = [ctx](int, const double* xp, dsmc::RngStream& s,
                               double* out) {
    *out = ctx->mu + ctx->phi * (*xp - ctx->mu) + std::sqrt(ctx->s2) * s.normal();
  };
  // omega_c = log p(x_c | x_{c-1}) - log|y_c|: column base is a constant.
  m.stitch_row_factory = [ctx](int c, const double* right, std::size_t n) {
    const double base = -0.5 * (kLog2Pi + std::log(ctx->s2)) - ctx->logabsy[c];
    auto row_base = std::make_shared<std::vector<double>>(n, base);
    const double coef = -1.0 / (2.0 * ctx->s2);
    return [ctx, row_base, right, n, coef](const double* xp, double* out) {
      const double mean = ctx->mu + ctx->phi * (*xp - ctx->mu);
      dsmc::kernels::gaussian_row(right, n, mean, coef, row_base->data(), out);
    };
  };
  m.log_stitch_bound = [ctx](int c) {
    return -0.5 * (kLog2Pi + std::log(ctx->s2)) - ctx->logabsy[c];
  };
  return m;
}

// ----------------------------------------------------------------- Cox
// Restates make_cox_model (models.cpp:111-216) against the reference API
// (models.cpp needs Eigen through models.hpp, so it cannot be compiled here).
struct CoxPrep {
  std::vector<double> y, lgam;
  double slope = 0, icept = 0, stat_mean = 0, stat_var = 1, s2 = 1, tnorm = 0;
  double log_poisson(int t, double x) const {  // models.cpp:103-106
    return y[static_cast<std::size_t>(t)] * x - std::exp(x) - lgam[static_cast<std::size_t>(t)];
  }
};

dsmc::FeynmanKacModel cox_model(const dsmc_model_desc& desc) {
  auto P = std::make_shared<CoxPrep>();
  const double mu = desc.par[0], rho = desc.par[1], lam = desc.par[3];
  P->s2 = desc.par[2];
  if (!(P->s2 > 0.0)) throw std::invalid_argument("make_cox_model: sigma2 must be > 0");
  if (!(std::abs(rho * lam) < 1.0))
    throw std::invalid_argument("make_cox_model: need |rho * lambda| < 1");
  P->y.assign(desc.y, desc.y + desc.horizon + 1);
  for (double v : P->y) {
    if (v < 0.0 || std::floor(v) != v)
      throw std::invalid_argument("make_cox_model: counts must be nonnegative integers");
    P->lgam.push_back(std::lgamma(v + 1.0));
  }
  P->slope = rho * lam;
  P->icept = mu * (1.0 - rho);
  P->stat_mean = P->icept / (1.0 - P->slope);
  P->stat_var = P->s2 / (1.0 - P->slope * P->slope);
  P->tnorm = -0.5 * (kLog2Pi + std::log(P->s2));

  dsmc::FeynmanKacModel m;
  m.state_dim = 1;
  m.horizon = desc.horizon;
  // proposals / aux / init: the stationary law
  m.proposal_sampler = [P](int, std::size_t count, dsmc::RngStream& s, double* out) {
    const double sd = std::sqrt(P->stat_var);
    s.fill_normal(out, count);
    for (std::size_t i = 0; i < count; ++i) out[i] = P->stat_mean + sd * out[i];
  };
  m.proposal_logdensity = [P](int, const double* x) {
    return log_normal_pdf(*x, P->stat_mean, P->stat_var);
  };
  m.aux_logdensity = m.proposal_logdensity;
  m.init_logdensity = [P](const double* x) {
    return log_normal_pdf(*x, P->stat_mean, P->stat_var);
  };
  m.log_potential = [P](int t, const double* x) { return P->log_poisson(t, *x); };
  m.transition_logdensity = [P](int, const double* xp, const double* xc) {
    return log_normal_pdf(*xc, P->icept + P->slope * *xp, P->s2);
  };
  m.transition_sampler = [P](int, const double* xp, dsmc::RngStream& s, double* out) {
    *out = P->icept + P->slope * *xp + std::sqrt(P->s2) * s.normal();
  };
  // t = 0: the Poisson potential alone (init law == proposal); t >= 1 uniform
  m.init_weight_batch = [P](int t, const double* xs, std::size_t n, double* out) {
    for (std::size_t j = 0; j < n; ++j) out[j] = t == 0 ? P->log_poisson(0, xs[j]) : 0.0;
  };
  // column base log h_c - log nu_c + trans_norm, row = one gaussian_row
  m.stitch_row_factory = [P](int c, const double* right, std::size_t n) {
    auto base = std::make_shared<std::vector<double>>(n);
    for (std::size_t j = 0; j < n; ++j)
      (*base)[j] = P->log_poisson(c, right[j]) -
                   log_normal_pdf(right[j], P->stat_mean, P->stat_var) + P->tnorm;
    return [P, base, right, n](const double* xp, double* out) {
      dsmc::kernels::gaussian_row(right, n, P->icept + P->slope * *xp, -1.0 / (2.0 * P->s2),
                                  base->data(), out);
    };
  };
  return m;  // no log_stitch_bound (models.cpp:210-212)
}

// -------------------------------------------------------- constrained RW
// Restates make_constrained_rw (models.cpp:263-338).
dsmc::FeynmanKacModel crw_model(const dsmc_model_desc& desc) {
  const double sigma = desc.par[0];
  if (!(sigma > 0.0)) throw std::invalid_argument("make_constrained_rw: sigma must be > 0");
  const double var = sigma * sigma;
  const double tnorm = -0.5 * (kLog2Pi + std::log(var));
  constexpr double kLogHalf = -0.6931471805599453;
  auto inside = [](double x) { return x >= -1.0 && x <= 1.0; };
  dsmc::FeynmanKacModel m;
  m.state_dim = 1;
  m.horizon = desc.horizon;
  m.proposal_sampler = [](int, std::size_t count, dsmc::RngStream& s, double* out) {
    s.fill_uniform(out, count);
    for (std::size_t i = 0; i < count; ++i) out[i] = 2.0 * out[i] - 1.0;
  };
  m.proposal_logdensity = [inside](int, const double* x) {
    return inside(*x) ? kLogHalf : -INFINITY;
  };
  m.aux_logdensity = m.proposal_logdensity;
  m.init_logdensity = [](const double* x) { return log_normal_pdf(*x, 0.0, 1.0); };
  m.log_potential = [inside](int, const double* x) { return inside(*x) ? 0.0 : -INFINITY; };
  m.transition_logdensity = [var](int, const double* xp, const double* xc) {
    return log_normal_pdf(*xc, *xp, var);
  };
  m.transition_sampler = [sigma](int, const double* xp, dsmc::RngStream& s, double* out) {
    *out = *xp + sigma * s.normal();
  };
  m.init_weight_batch = [inside](int t, const double* xs, std::size_t n, double* out) {
    constexpr double norm = -0.5 * kLog2Pi - kLogHalf;
    for (std::size_t j = 0; j < n; ++j)
      out[j] = !inside(xs[j]) ? -INFINITY : t == 0 ? norm - 0.5 * xs[j] * xs[j] : 0.0;
  };
  m.stitch_row_factory = [var, tnorm, inside](int, const double* right, std::size_t n) {
    auto base = std::make_shared<std::vector<double>>(n);
    for (std::size_t j = 0; j < n; ++j)
      (*base)[j] = inside(right[j]) ? tnorm - kLogHalf : -INFINITY;
    return [base, right, n, var](const double* xp, double* out) {
      dsmc::kernels::gaussian_row(right, n, *xp, -1.0 / (2.0 * var), base->data(), out);
    };
  };
  m.log_stitch_bound = [tnorm](int) { return tnorm - kLogHalf; };
  return m;
}

// ------------------------------------------------------ theta-logistic
// Restates make_theta_logistic (models.cpp:407-491) with the descriptor's
// proposal marginals.
dsmc::FeynmanKacModel theta_model(const dsmc_model_desc& desc) {
  struct Ctx {
    double tau0, tau1, tau2, q2, r2, tnorm, onorm;
    std::vector<double> y, mean, var;
    double drift(double x) const { return x + tau0 - tau1 * std::exp(tau2 * x); }
  };
  auto C = std::make_shared<Ctx>();
  C->tau0 = desc.par[0];
  C->tau1 = desc.par[1];
  C->tau2 = desc.par[2];
  C->q2 = desc.par[3];
  C->r2 = desc.par[4];
  if (!(C->q2 > 0.0) || !(C->r2 > 0.0))
    throw std::invalid_argument("make_theta_logistic: q2 and r2 must be > 0");
  const int K = desc.horizon + 1;
  C->y.assign(desc.y, desc.y + K);
  C->mean.assign(desc.prop_mean, desc.prop_mean + K);
  C->var.assign(desc.prop_cov, desc.prop_cov + K);
  C->tnorm = -0.5 * (kLog2Pi + std::log(C->q2));
  C->onorm = -0.5 * (kLog2Pi + std::log(C->r2));
  dsmc::FeynmanKacModel m;
  m.state_dim = 1;
  m.horizon = desc.horizon;
  m.proposal_sampler = [C](int t, std::size_t count, dsmc::RngStream& s, double* out) {
    const double sd = std::sqrt(C->var[t]);
    s.fill_normal(out, count);
    for (std::size_t i = 0; i < count; ++i) out[i] = C->mean[t] + sd * out[i];
  };
  m.proposal_logdensity = [C](int t, const double* x) {
    return log_normal_pdf(*x, C->mean[t], C->var[t]);
  };
  m.aux_logdensity = m.proposal_logdensity;
  m.init_logdensity = [](const double* x) { return log_normal_pdf(*x, 0.0, 1.0); };
  m.log_potential = [C](int t, const double* x) { return log_normal_pdf(C->y[t], *x, C->r2); };
  m.transition_logdensity = [C](int, const double* xp, const double* xc) {
    return log_normal_pdf(*xc, C->drift(*xp), C->q2);
  };
  m.transition_sampler = [C](int, const double* xp, dsmc::RngStream& s, double* out) {
    *out = C->drift(*xp) + std::sqrt(C->q2) * s.normal();
  };
  m.stitch_row_factory = [C](int c, const double* right, std::size_t n) {
    auto base = std::make_shared<std::vector<double>>(n);
    dsmc::kernels::gaussian_row(right, n, C->y[c], -1.0 / (2.0 * C->r2), nullptr, base->data());
    dsmc::kernels::gaussian_row(right, n, C->mean[c], 1.0 / (2.0 * C->var[c]), base->data(),
                                base->data());
    dsmc::kernels::add_vec_scalar(base->data(), n,
                                  C->onorm + 0.5 * (kLog2Pi + std::log(C->var[c])) + C->tnorm,
                                  nullptr);
    return [C, base, right, n](const double* xp, double* out) {
      dsmc::kernels::gaussian_row(right, n, C->drift(*xp), -1.0 / (2.0 * C->q2), base->data(),
                                  out);
    };
  };
  std::vector<double> bounds(K, 0.0);
  bool bounded = desc.horizon >= 1;
  for (int c = 1; c <= desc.horizon && bounded; ++c) {
    const double s = obs_over_aux_sup(C->y[c], 1.0, C->r2, C->mean[c], C->var[c]);
    if (!std::isfinite(s)) bounded = false;
    else bounds[c] = C->tnorm + s;
  }
  if (bounded) m.log_stitch_bound = [bounds](int c) { return bounds[c]; };
  return m;
}

}  // namespace

dsmc::FeynmanKacModel build_model(const dsmc_model_desc& desc) {
  if (desc.kind == DSMC_MODEL_LGSSM) {
    auto ctx = make_lg_ctx(desc);
    return (desc.state_dim == 1 && desc.obs_dim == 1) ? lgssm_1d(ctx)
                                                        : lgssm_nd(ctx);
  }
  if (desc.kind == DSMC_MODEL_SV) return sv_model(desc);
  if (desc.kind == DSMC_MODEL_COX) return cox_model(desc);
  if (desc.kind == DSMC_MODEL_CRW) return crw_model(desc);
  if (desc.kind == DSMC_MODEL_THETA) return theta_model(desc);
  throw std::invalid_argument("unknown model kind");
}

}  // namespace oracle

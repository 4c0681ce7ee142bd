// C++ host layer (include/dsmc/dsmc.hpp) over the C ABI. Keeps the
// reference's dsmc:: entry points and exception classes; all numerical work
// is delegated to the CUDA engine (libdsmc_b200.so).
#include "dsmc/dsmc.hpp"
#include "internal.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>

namespace dsmc {

namespace detail {

[[noreturn]] void throw_code(int code, const std::string& msg) {
  switch (code) {
    case DSMC_E_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case DSMC_E_DOMAIN: throw std::domain_error(msg);
    case DSMC_E_LOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

// One engine context per (thread, device).
dsmc_ctx* context(int device) {
  thread_local std::map<int, std::unique_ptr<dsmc_ctx, void (*)(dsmc_ctx*)>> ctxs;
  auto it = ctxs.find(device);
  if (it != ctxs.end()) return it->second.get();
  dsmc_ctx* c = nullptr;
  int rc = dsmc_create(device, &c);
  if (rc) throw std::runtime_error("no CUDA device " + std::to_string(device) +
                                   " for the dSMC engine (there is no CPU fallback)");
  ctxs.emplace(device, std::unique_ptr<dsmc_ctx, void (*)(dsmc_ctx*)>(c, dsmc_destroy));
  return c;
}

void check(dsmc_ctx* c, int rc) {
  if (rc) throw_code(rc, dsmc_last_error(c));
}

const dsmc_model_desc& desc_of(const FeynmanKacModel& m) {
  if (!m.device)
    throw std::invalid_argument(
        "model has no device descriptor: the GPU engine runs model families "
        "described by data (make_lgssm_fk, make_sv_model, make_cox_model, "
        "make_constrained_rw, make_theta_logistic); there is no CPU fallback");
  return m.device->desc;
}

}  // namespace detail

namespace {

using detail::check;
using detail::context;
using detail::desc_of;
using detail::throw_code;

constexpr double kLog2Pi = 1.8378770664093454836;

double log_normal_pdf(double x, double mean, double var) {
  const double d = x - mean;
  return -0.5 * (kLog2Pi + std::log(var)) - d * d / (2.0 * var);
}

// whitened Gaussian log density for d <= 4 (host callbacks only)
double gauss_logpdf(const double* x, const double* m, const double* S, int d) {
  double L[16] = {0}, e[4];
  for (int i = 0; i < d; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = S[i * d + j];
      for (int k = 0; k < j; ++k) s -= L[i * d + k] * L[j * d + k];
      L[i * d + j] = i == j ? std::sqrt(s) : s / L[j * d + j];
    }
  double q = 0.0, ld = 0.0;
  for (int i = 0; i < d; ++i) {
    double s = x[i] - m[i];
    for (int k = 0; k < i; ++k) s -= L[i * d + k] * e[k];
    e[i] = s / L[i * d + i];
    q += e[i] * e[i];
    ld += 2.0 * std::log(L[i * d + i]);
  }
  return -0.5 * (d * kLog2Pi + ld) - 0.5 * q;
}

// lower Cholesky factor of a d x d (d <= 4) covariance
void chol4(const double* S, int d, double* L) {
  for (int i = 0; i < d * d; ++i) L[i] = 0.0;
  for (int i = 0; i < d; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = S[i * d + j];
      for (int k = 0; k < j; ++k) s -= L[i * d + k] * L[j * d + k];
      L[i * d + j] = i == j ? std::sqrt(s) : s / L[j * d + j];
    }
}
// out = mu + L z, z ~ N(0, I) by fill_normal
void affine_draw(const double* mu, const double* L, int d, RngStream& st, double* out) {
  double z[4];
  st.fill_normal(z, d);
  for (int i = 0; i < d; ++i) {
    double v = mu[i];
    for (int k = 0; k <= i; ++k) v += L[i * d + k] * z[k];
    out[i] = v;
  }
}

}  // namespace

// ------------------------------------------------------------ resampling
std::optional<Resampler> parse_resampler(std::string_view name) {
  if (name == "multinomial") return Resampler::multinomial;
  if (name == "systematic") return Resampler::systematic;
  if (name == "mh-lazy") return Resampler::mh_lazy;
  if (name == "rejection-lazy") return Resampler::rejection_lazy;
  return std::nullopt;
}
std::string resampler_name(Resampler r) {
  switch (r) {
    case Resampler::multinomial: return "multinomial";
    case Resampler::systematic: return "systematic";
    case Resampler::mh_lazy: return "mh-lazy";
    case Resampler::rejection_lazy: return "rejection-lazy";
  }
  return "unknown";
}
bool resampler_is_lazy(Resampler r) {
  return r == Resampler::mh_lazy || r == Resampler::rejection_lazy;
}

PairSample resample_pairs(Resampler r, const std::vector<double>& logw,
                          std::size_t n, std::size_t n_out,
                          std::size_t mh_steps, const StreamKey& key,
                          std::optional<double> bound) {
  if (logw.size() != n * n) throw std::invalid_argument("table must be n x n");
  dsmc_ctx* c = context(0);
  PairSample ps;
  ps.left.resize(n_out);
  ps.right.resize(n_out);
  double lmw = 0;
  int has = 0, biased = 0;
  uint64_t ev = 0;
  check(c, dsmc_resample_table(c, static_cast<int>(r), logw.data(), n, n_out, mh_steps,
                               bound ? 1 : 0, bound.value_or(0.0), key.seed, key.level,
                               key.node, ps.left.data(), ps.right.data(), &lmw, &has,
                               &ev, &biased));
  if (has) ps.log_mean_weight = lmw;
  ps.weight_evals = ev;
  ps.biased = biased != 0;
  if (resampler_is_lazy(r))
    metrics::note_lazy_alloc(2 * n_out);
  else
    metrics::count_dense_alloc(n * n);
  metrics::add_weight_evals(ev);
  return ps;
}

// ---------------------------------------------------------------- kalman
KalmanResult kalman_smooth(const LinearGaussianModel& m) {
  FeynmanKacModel tmp = make_lgssm_fk(m, {});
  const dsmc_model_desc& d = tmp.device->desc;
  const int K = m.horizon + 1, dx = m.dim_x;
  std::vector<double> mean((size_t)K * dx), cov((size_t)K * dx * dx);
  double ll = 0;
  int rc = dsmc_kalman_smooth(&d, mean.data(), cov.data(), &ll);
  if (rc) throw_code(rc, "kalman_smooth failed");
  KalmanResult kr;
  kr.log_likelihood = ll;
  for (int t = 0; t < K; ++t) {
    kr.smooth_mean.emplace_back(mean.begin() + (size_t)t * dx, mean.begin() + (size_t)(t + 1) * dx);
    kr.smooth_cov.emplace_back(cov.begin() + (size_t)t * dx * dx,
                               cov.begin() + (size_t)(t + 1) * dx * dx);
  }
  return kr;
}

std::vector<ProposalMarginal> proposal_marginals(const KalmanResult& kr, double inflation) {
  if (!(inflation > 0.0)) throw std::invalid_argument("proposal_marginals: inflation must be > 0");
  std::vector<ProposalMarginal> out(kr.smooth_mean.size());
  for (std::size_t t = 0; t < out.size(); ++t) {
    out[t].mean = kr.smooth_mean[t];
    out[t].cov = kr.smooth_cov[t];
    for (double& v : out[t].cov) v *= inflation;
  }
  return out;
}

// --------------------------------------------------------------- models
FeynmanKacModel make_lgssm_fk(const LinearGaussianModel& m,
                              const std::vector<ProposalMarginal>& marginals) {
  const int d = m.dim_x, dy = m.dim_y, T = m.horizon, K = T + 1;
  if (d < 1 || d > 4 || dy < 1 || dy > 4)
    throw std::invalid_argument("make_lgssm_fk: dimensions must be 1..4 on the GPU");
  if (!marginals.empty() && marginals.size() != static_cast<std::size_t>(K))
    throw std::invalid_argument("make_lgssm_fk: need one proposal marginal per time");
  auto dm = std::make_shared<DeviceModel>();
  dm->m0 = m.m0;
  dm->P0 = m.P0;
  auto flat = [&](const std::vector<std::vector<double>>& v, std::size_t per,
                  std::vector<double>& out) {
    out.assign((size_t)K * per, 0.0);
    for (int t = 0; t < K && t < (int)v.size(); ++t)
      if (v[t].size() == per) std::memcpy(&out[(size_t)t * per], v[t].data(), per * 8);
  };
  flat(m.F, (size_t)d * d, dm->F);
  flat(m.b, (size_t)d, dm->b);
  flat(m.Q, (size_t)d * d, dm->Q);
  flat(m.H, (size_t)dy * d, dm->H);
  flat(m.R, (size_t)dy * dy, dm->R);
  flat(m.y, (size_t)dy, dm->y);
  dm->has_obs.assign(m.has_obs.begin(), m.has_obs.end());
  dm->prop_mean.assign((size_t)K * d, 0.0);
  dm->prop_cov.assign((size_t)K * d * d, 0.0);
  for (int t = 0; t < K; ++t) {
    if (marginals.empty()) {
      for (int k = 0; k < d; ++k) dm->prop_cov[(size_t)t * d * d + k * d + k] = 1.0;
    } else {
      std::memcpy(&dm->prop_mean[(size_t)t * d], marginals[t].mean.data(), d * 8);
      std::memcpy(&dm->prop_cov[(size_t)t * d * d], marginals[t].cov.data(), (size_t)d * d * 8);
    }
  }
  dsmc_model_desc& ds = dm->desc;
  ds.kind = DSMC_MODEL_LGSSM;
  ds.state_dim = d;
  ds.obs_dim = dy;
  ds.horizon = T;
  ds.F_stride = (int64_t)d * d;
  ds.b_stride = d;
  ds.Q_stride = (int64_t)d * d;
  ds.H_stride = (int64_t)dy * d;
  ds.R_stride = (int64_t)dy * dy;
  dm->bind();
  FeynmanKacModel fk;
  fk.state_dim = d;
  fk.horizon = T;
  fk.device = dm;
  DeviceModel* D = dm.get();
  fk.proposal_logdensity = [D, d](int t, const double* x) {
    return gauss_logpdf(x, &D->prop_mean[(size_t)t * d], &D->prop_cov[(size_t)t * d * d], d);
  };
  fk.aux_logdensity = fk.proposal_logdensity;
  fk.init_logdensity = [D, d](const double* x) {
    return gauss_logpdf(x, D->m0.data(), D->P0.data(), d);
  };
  fk.log_potential = [D, d, dy](int t, const double* x) {
    if (!D->has_obs.empty() && !D->has_obs[t]) return 0.0;
    double hx[4];
    for (int a = 0; a < dy; ++a) {
      double s = 0.0;
      for (int l = 0; l < d; ++l) s += D->H[(size_t)t * dy * d + a * d + l] * x[l];
      hx[a] = s;
    }
    return gauss_logpdf(&D->y[(size_t)t * dy], hx, &D->R[(size_t)t * dy * dy], dy);
  };
  fk.transition_logdensity = [D, d](int t, const double* xp, const double* xc) {
    double mu[4];
    for (int k = 0; k < d; ++k) {
      double s = 0.0;
      for (int l = 0; l < d; ++l) s += D->F[(size_t)t * d * d + k * d + l] * xp[l];
      mu[k] = s + D->b[(size_t)t * d + k];
    }
    return gauss_logpdf(xc, mu, &D->Q[(size_t)t * d * d], d);
  };
  // host draws (the LinearGaussian draw of kalman.cpp:43-50: mean + chol(S) z,
  // z by fill_normal); the device draws its own leaves from the same streams
  fk.proposal_sampler = [D, d](int t, std::size_t count, RngStream& st, double* out) {
    double L[16];
    chol4(&D->prop_cov[(size_t)t * d * d], d, L);
    for (std::size_t p = 0; p < count; ++p)
      affine_draw(&D->prop_mean[(size_t)t * d], L, d, st, out + p * d);
  };
  fk.transition_sampler = [D, d](int t, const double* xp, RngStream& st, double* out) {
    double L[16], mu[4];
    chol4(&D->Q[(size_t)t * d * d], d, L);
    for (int k = 0; k < d; ++k) {
      double s = 0.0;
      for (int l = 0; l < d; ++l) s += D->F[(size_t)t * d * d + k * d + l] * xp[l];
      mu[k] = s + D->b[(size_t)t * d + k];
    }
    affine_draw(mu, L, d, st, out);
  };
  return fk;
}

FeynmanKacModel make_sv_model(const SvParams& p, const std::vector<double>& ys) {
  if (ys.empty()) throw std::invalid_argument("make_sv_model: need observations");
  auto dm = std::make_shared<DeviceModel>();
  dm->y = ys;
  dsmc_model_desc& ds = dm->desc;
  ds.kind = DSMC_MODEL_SV;
  ds.state_dim = 1;
  ds.obs_dim = 1;
  ds.horizon = static_cast<int>(ys.size()) - 1;
  ds.sv_mu = p.mu;
  ds.sv_phi = p.phi;
  ds.sv_sigma2 = p.sigma2;
  dm->bind();
  FeynmanKacModel fk;
  fk.state_dim = 1;
  fk.horizon = ds.horizon;
  fk.device = dm;
  DeviceModel* D = dm.get();
  auto log_h = [D](int t, double x) {
    const double y = D->y[t];
    return -0.5 * (kLog2Pi + x) - y * y / (2.0 * std::exp(x));
  };
  fk.log_potential = [log_h](int t, const double* x) { return log_h(t, *x); };
  fk.proposal_logdensity = [D, log_h](int t, const double* x) {
    return std::log(std::fabs(D->y[t])) + log_h(t, *x);
  };
  fk.aux_logdensity = fk.proposal_logdensity;
  fk.init_logdensity = [p](const double* x) {
    return log_normal_pdf(*x, p.mu, p.sigma2 / (1.0 - p.phi * p.phi));
  };
  fk.transition_logdensity = [p](int, const double* xp, const double* xc) {
    return log_normal_pdf(*xc, p.mu + p.phi * (*xp - p.mu), p.sigma2);
  };
  fk.log_stitch_bound = [D, p](int c) {
    return -0.5 * (kLog2Pi + std::log(p.sigma2)) - std::log(std::fabs(D->y[c]));
  };
  fk.proposal_sampler = [D](int t, std::size_t count, RngStream& st, double* out) {
    const double ly2 = std::log(D->y[t] * D->y[t]);
    for (std::size_t q = 0; q < count; ++q) {
      const double z = st.normal();
      out[q] = ly2 - std::log(z * z);  // x = log y^2 - log z^2
    }
  };
  fk.transition_sampler = [p](int, const double* xp, RngStream& st, double* out) {
    *out = p.mu + p.phi * (*xp - p.mu) + std::sqrt(p.sigma2) * st.normal();
  };
  return fk;
}

FeynmanKacModel make_cox_model(const CoxParams& p, const std::vector<double>& ys) {
  if (ys.empty()) throw std::invalid_argument("make_cox_model: observations are empty");
  auto dm = std::make_shared<DeviceModel>();
  dm->y = ys;
  dsmc_model_desc& ds = dm->desc;
  ds.kind = DSMC_MODEL_COX;
  ds.state_dim = 1;
  ds.obs_dim = 1;
  ds.horizon = static_cast<int>(ys.size()) - 1;
  ds.par[0] = p.mu;
  ds.par[1] = p.rho;
  ds.par[2] = p.sigma2;
  ds.par[3] = p.lambda;
  dm->bind();
  // host callbacks (validation / scalar checks), models.cpp:127-167
  const double a = p.rho * p.lambda, b = p.mu * (1.0 - p.rho);
  const double sm = b / (1.0 - a), sv = p.sigma2 / (1.0 - a * a);
  FeynmanKacModel fk;
  fk.state_dim = 1;
  fk.horizon = ds.horizon;
  fk.device = dm;
  DeviceModel* D = dm.get();
  fk.log_potential = [D](int t, const double* x) {
    const double y = D->y[static_cast<std::size_t>(t)];
    return y * *x - std::exp(*x) - std::lgamma(y + 1.0);
  };
  fk.proposal_logdensity = [sm, sv](int, const double* x) { return log_normal_pdf(*x, sm, sv); };
  fk.aux_logdensity = fk.proposal_logdensity;
  fk.init_logdensity = [sm, sv](const double* x) { return log_normal_pdf(*x, sm, sv); };
  fk.transition_logdensity = [a, b, p](int, const double* xp, const double* xc) {
    return log_normal_pdf(*xc, b + a * *xp, p.sigma2);
  };
  fk.proposal_sampler = [sm, sv](int, std::size_t count, RngStream& st, double* out) {
    const double sd = std::sqrt(sv);
    for (std::size_t q = 0; q < count; ++q) out[q] = sm + sd * st.normal();
  };
  fk.transition_sampler = [a, b, p](int, const double* xp, RngStream& st, double* out) {
    *out = b + a * *xp + std::sqrt(p.sigma2) * st.normal();
  };
  return fk;
}

FeynmanKacModel make_constrained_rw(double sigma, int horizon) {
  if (horizon < 0) throw std::invalid_argument("make_constrained_rw: horizon must be >= 0");
  auto dm = std::make_shared<DeviceModel>();
  dsmc_model_desc& ds = dm->desc;
  ds.kind = DSMC_MODEL_CRW;
  ds.state_dim = 1;
  ds.obs_dim = 1;
  ds.horizon = horizon;
  ds.par[0] = sigma;
  dm->bind();
  const double var = sigma * sigma, lhalf = -0.6931471805599453;
  auto inside = [](double x) { return x >= -1.0 && x <= 1.0; };
  FeynmanKacModel fk;
  fk.state_dim = 1;
  fk.horizon = horizon;
  fk.device = dm;
  fk.log_potential = [inside](int, const double* x) { return inside(*x) ? 0.0 : -INFINITY; };
  fk.proposal_logdensity = [inside, lhalf](int, const double* x) {
    return inside(*x) ? lhalf : -INFINITY;
  };
  fk.aux_logdensity = fk.proposal_logdensity;
  fk.init_logdensity = [](const double* x) { return log_normal_pdf(*x, 0.0, 1.0); };
  fk.transition_logdensity = [var](int, const double* xp, const double* xc) {
    return log_normal_pdf(*xc, *xp, var);
  };
  fk.log_stitch_bound = [var, lhalf](int) { return -0.5 * (kLog2Pi + std::log(var)) - lhalf; };
  fk.proposal_sampler = [](int, std::size_t count, RngStream& st, double* out) {
    st.fill_uniform(out, count);  // U[-1, 1] (rng.cpp:95-97)
    for (std::size_t q = 0; q < count; ++q) out[q] = 2.0 * out[q] - 1.0;
  };
  fk.transition_sampler = [sigma](int, const double* xp, RngStream& st, double* out) {
    *out = *xp + sigma * st.normal();
  };
  return fk;
}

FeynmanKacModel make_theta_logistic(const ThetaLogisticParams& p, const std::vector<double>& ys,
                                    const std::vector<ProposalMarginal>& marginals) {
  if (ys.empty() || marginals.size() != ys.size())
    throw std::invalid_argument(
        "make_theta_logistic: need one proposal marginal per observation");
  auto dm = std::make_shared<DeviceModel>();
  dm->y = ys;
  for (const auto& g : marginals) {
    if (g.mean.size() != 1 || g.cov.size() != 1)
      throw std::invalid_argument("make_theta_logistic: marginals must be 1-d");
    dm->prop_mean.push_back(g.mean[0]);
    dm->prop_cov.push_back(g.cov[0]);
  }
  dsmc_model_desc& ds = dm->desc;
  ds.kind = DSMC_MODEL_THETA;
  ds.state_dim = 1;
  ds.obs_dim = 1;
  ds.horizon = static_cast<int>(ys.size()) - 1;
  const double par[5] = {p.tau0, p.tau1, p.tau2, p.q2, p.r2};
  for (int q = 0; q < 5; ++q) ds.par[q] = par[q];
  dm->bind();
  FeynmanKacModel fk;
  fk.state_dim = 1;
  fk.horizon = ds.horizon;
  fk.device = dm;
  DeviceModel* D = dm.get();
  auto drift = [p](double x) { return x + p.tau0 - p.tau1 * std::exp(p.tau2 * x); };
  fk.log_potential = [D, p](int t, const double* x) {
    return log_normal_pdf(D->y[static_cast<std::size_t>(t)], *x, p.r2);
  };
  fk.proposal_logdensity = [D](int t, const double* x) {
    return log_normal_pdf(*x, D->prop_mean[static_cast<std::size_t>(t)],
                          D->prop_cov[static_cast<std::size_t>(t)]);
  };
  fk.aux_logdensity = fk.proposal_logdensity;
  fk.init_logdensity = [](const double* x) { return log_normal_pdf(*x, 0.0, 1.0); };
  fk.transition_logdensity = [drift, p](int, const double* xp, const double* xc) {
    return log_normal_pdf(*xc, drift(*xp), p.q2);
  };
  fk.proposal_sampler = [D](int t, std::size_t count, RngStream& st, double* out) {
    const double m = D->prop_mean[static_cast<std::size_t>(t)];
    const double sd = std::sqrt(D->prop_cov[static_cast<std::size_t>(t)]);
    for (std::size_t q = 0; q < count; ++q) out[q] = m + sd * st.normal();
  };
  fk.transition_sampler = [drift, p](int, const double* xp, RngStream& st, double* out) {
    *out = drift(*xp) + std::sqrt(p.q2) * st.normal();
  };
  return fk;
}

// -------------------------------------------------------------- fk_model
// fk_model.cpp:26-40 (the reference's contract on the callbacks)
void validate_model(const FeynmanKacModel& model) {
  if (model.state_dim < 1) throw std::invalid_argument("model: state_dim must be >= 1");
  if (model.horizon < 0) throw std::invalid_argument("model: horizon must be >= 0");
  if (!model.proposal_sampler || !model.proposal_logdensity || !model.log_potential ||
      !model.init_logdensity)
    throw std::invalid_argument(
        "model: proposal sampler/density, potential and initial density are required");
  if (model.horizon >= 1 && (!model.aux_logdensity || !model.transition_logdensity))
    throw std::invalid_argument(
        "model: aux density and transition density are required for T >= 1");
}

namespace detail {
// validate_model plus what the device needs: a descriptor that agrees
const dsmc_model_desc& device_desc(const FeynmanKacModel& model) {
  validate_model(model);
  const dsmc_model_desc& d = desc_of(model);
  if (d.horizon != model.horizon || d.state_dim != model.state_dim)
    throw std::invalid_argument("model: device descriptor disagrees with the callbacks");
  return d;
}
}  // namespace detail

// fk_model.cpp:61-73
double log_stitch_weight(const FeynmanKacModel& model, int c, const double* x_prev,
                         const double* x_cur) {
  if (c < 1 || c > model.horizon)
    throw std::invalid_argument("log_stitch_weight: time index outside [1, T]");
  const double trans = model.transition_logdensity(c, x_prev, x_cur);
  const double pot = model.log_potential(c, x_cur);
  if (trans == -INFINITY || pot == -INFINITY) return -INFINITY;
  const double nu = model.aux_logdensity(c, x_cur);
  if (nu == -INFINITY)
    throw std::invalid_argument(
        "log_stitch_weight: aux density vanishes where transition*potential does not "
        "(nu_c must dominate)");
  const double v = trans + pot - nu;
  if (std::isnan(v)) throw std::invalid_argument("log_stitch_weight produced NaN");
  return v;
}

// --------------------------------------------------------------- smoother
CombineSchedule build_schedule(int horizon) {
  if (horizon < 0) throw std::invalid_argument("build_schedule: horizon must be >= 0");
  CombineSchedule s;
  s.horizon = horizon;
  int K = horizon + 1, nb = K, span = 1;
  while (nb > 1) {
    ++s.levels;
    for (int k = 0; k < nb / 2; ++k)
      s.pairs.push_back({s.levels, k, 2 * k * span, (2 * k + 1) * span - 1,
                         std::min((2 * k + 2) * span - 1, K - 1)});
    nb = (nb + 1) / 2;
    span *= 2;
  }
  return s;
}

int reference_tree_depth(int horizon) {
  if (horizon < 0) throw std::invalid_argument("reference_tree_depth: horizon must be >= 0");
  std::function<int(int)> depth = [&](int k) {
    return k <= 1 ? 0 : 1 + std::max(depth((k + 1) / 2), depth(k / 2));
  };
  return depth(horizon + 1);
}

RunResult run_smoother(const FeynmanKacModel& model, const SmootherOptions& o) {
  const dsmc_model_desc& desc = detail::device_desc(model);
  dsmc_ctx* c = context(o.device);
  const int T = model.horizon, K = T + 1, d = model.state_dim;
  const std::size_t N = o.n_particles;
  RunResult res;
  res.root.a = 0;
  res.root.b = T;
  res.root.n = N;
  res.root.dim = d;
  res.root.paths.resize((size_t)K * N * d);
  res.mean.resize((size_t)K * d);
  res.cov.resize((size_t)K * d * d);
  dsmc_smooth_opts opts{N, static_cast<int>(o.resampler), o.mh_steps, o.seed,
                        static_cast<int>(o.precision), nullptr, nullptr};
  dsmc_smooth_out out{};
  out.paths = res.root.paths.data();
  out.mean = res.mean.data();
  out.cov = res.cov.data();
  check(c, dsmc_smooth(c, &desc, &opts, &out));
  res.root.log_w.assign(N, -std::log(static_cast<double>(N)));
  res.root.weights_uniform = true;
  if (out.has_log_norm_const) res.root.log_norm_const = out.log_norm_const;
  res.root.biased = out.biased != 0;
  res.root.weight_evals = out.weight_evals;
  res.meta.horizon = T;
  res.meta.n_particles = N;
  res.meta.resampler = resampler_name(o.resampler);
  res.meta.levels = out.levels;
  res.meta.weight_evals = out.weight_evals;
  res.meta.wall_time_ms = out.wall_time_ms;
  res.meta.log_norm_const = res.root.log_norm_const;
  res.meta.seed = o.seed;
  res.meta.biased = res.root.biased;
  // metrics contract (metrics.hpp): one dense N x N table per dense combine
  // (evaluated on the device, streaming), none for the lazy samplers
  if (resampler_is_lazy(o.resampler)) {
    if (T > 0) metrics::note_lazy_alloc(2 * N);
  } else {
    for (int k = 0; k < T; ++k) metrics::count_dense_alloc(N * N);
  }
  metrics::add_weight_evals(out.weight_evals);
  return res;
}

std::vector<double> weighted_time_mean(const BlockEstimate& block, int t) {
  if (t < block.a || t > block.b)
    throw std::invalid_argument("weighted_time_mean: time outside the block");
  std::vector<double> mean(block.dim, 0.0);
  const double* slab = block.time_slab(t);
  for (std::size_t p = 0; p < block.n; ++p) {
    const double w = block.weights_uniform ? 1.0 / block.n : std::exp(block.log_w[p]);
    for (int k = 0; k < block.dim; ++k) mean[k] += w * slab[p * block.dim + k];
  }
  return mean;
}

void copy_path(const BlockEstimate& block, std::size_t p, double* out) {
  if (p >= block.n) throw std::invalid_argument("copy_path: index out of range");
  for (int t = block.a; t <= block.b; ++t)
    std::memcpy(out + (size_t)(t - block.a) * block.dim, block.time_slab(t) + p * block.dim,
                sizeof(double) * block.dim);
}

// ------------------------------------------------------------ conditional
ConditionalResult run_conditional(const FeynmanKacModel& model, const double* ref,
                                  const ConditionalOptions& o, std::uint32_t sweep) {
  detail::device_desc(model);
  if (o.resampler != Resampler::multinomial && o.resampler != Resampler::rejection_lazy)
    throw std::invalid_argument(
        "conditional sweeps need exchangeable unbiased slot draws: use the multinomial "
        "or rejection-lazy resampler");
  const dsmc_model_desc& desc = desc_of(model);
  dsmc_ctx* c = context(o.device);
  const int K = model.horizon + 1, d = model.state_dim;
  ConditionalResult r;
  r.path.resize((size_t)K * d);
  dsmc_cond_opts co{o.n_particles, static_cast<int>(o.resampler),
                    static_cast<int>(o.precision), nullptr, nullptr};
  double lnc = NAN;
  uint64_t ev = 0;
  const auto t0 = std::chrono::steady_clock::now();
  check(c, dsmc_conditional_sweep(c, &desc, 1, ref, &o.seed, &co, sweep, r.path.data(),
                                  nullptr, &lnc, &ev));
  r.meta.horizon = model.horizon;
  r.meta.n_particles = o.n_particles;
  r.meta.resampler = resampler_name(o.resampler);
  r.meta.levels = reference_tree_depth(model.horizon);
  r.meta.weight_evals = ev;
  r.meta.wall_time_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (!std::isnan(lnc)) r.meta.log_norm_const = lnc;
  r.meta.seed = o.seed;
  if (resampler_is_lazy(o.resampler)) {
    if (model.horizon > 0) metrics::note_lazy_alloc(2 * o.n_particles);
  } else {
    for (int k = 0; k < model.horizon; ++k)
      metrics::count_dense_alloc(o.n_particles * o.n_particles);
  }
  metrics::add_weight_evals(ev);
  return r;
}

std::vector<char> path_changed_times(const double* a, const double* b, int len, int dim) {
  std::vector<char> changed(len, 0);
  for (int t = 0; t < len; ++t)
    for (int k = 0; k < dim; ++k)
      if (a[t * dim + k] != b[t * dim + k]) {
        changed[t] = 1;
        break;
      }
  return changed;
}

// ---------------------------------------------------------------- pgibbs
SweepOutcome pgibbs_sweep(const GibbsState& state, const GibbsModelBuilder& builder,
                          const ParamKernel& kernel, const ConditionalOptions& o,
                          std::uint32_t sweep) {
  if (!builder || !kernel) throw std::invalid_argument("pgibbs_sweep: missing kernel or builder");
  if (state.star.empty()) throw std::invalid_argument("pgibbs_sweep: empty reference path");
  SweepOutcome out;
  out.state = state;  // private copy: strong guarantee
  RngStream pstream({o.seed, 0, sweep, StreamRole::gibbs_param});
  kernel(out.state, pstream);
  FeynmanKacModel model = builder(out.state);
  const std::size_t want = (size_t)(model.horizon + 1) * model.state_dim;
  if (out.state.star.size() != want)
    throw std::invalid_argument("pgibbs_sweep: reference path does not match the model shape");
  ConditionalResult res = run_conditional(model, out.state.star.data(), o, sweep);
  out.changed = path_changed_times(out.state.star.data(), res.path.data(), model.horizon + 1,
                                   model.state_dim);
  out.state.star = std::move(res.path);
  out.meta = std::move(res.meta);
  return out;
}

std::vector<double> update_rate(const std::vector<std::vector<double>>& stars, int dim) {
  if (stars.size() < 2) throw std::invalid_argument("update_rate: need at least two stars");
  if (dim < 1) throw std::invalid_argument("update_rate: dim must be >= 1");
  const std::size_t len = stars.front().size() / dim;
  std::vector<double> rate(len, 0.0);
  for (std::size_t k = 1; k < stars.size(); ++k) {
    if (stars[k].size() != stars.front().size())
      throw std::invalid_argument("update_rate: stars differ in shape");
    auto m = path_changed_times(stars[k - 1].data(), stars[k].data(), (int)len, dim);
    for (std::size_t t = 0; t < len; ++t) rate[t] += m[t];
  }
  for (auto& r : rate) r /= static_cast<double>(stars.size() - 1);
  return rate;
}

std::vector<char> sv_pgibbs_sweep(SvGibbsChains& ch, const std::vector<double>& ys,
                                  const dsmc_sv_prior& prior, const ConditionalOptions& o,
                                  std::uint32_t sweep) {
  const int B = static_cast<int>(ch.seeds.size());
  const int T = static_cast<int>(ys.size()) - 1;
  if (B < 1 || ch.theta.size() != (size_t)B * 3 || ch.stars.size() != (size_t)B * (T + 1))
    throw std::invalid_argument("sv_pgibbs_sweep: inconsistent chain arrays");
  dsmc_ctx* c = context(o.device);
  std::vector<char> changed((size_t)B * (T + 1));
  uint64_t acc = 0;
  check(c, dsmc_sv_pgibbs_sweep(c, B, T, ys.data(), &prior, ch.theta.data(), ch.stars.data(),
                                ch.seeds.data(), o.n_particles, static_cast<int>(o.resampler),
                                sweep, reinterpret_cast<uint8_t*>(changed.data()), &acc));
  ch.phi_accepts += acc;
  return changed;
}


// ------------------------------------------------------------------- rng
namespace rng_detail {
std::array<std::uint64_t, 4> philox4x64_10(const std::array<std::uint64_t, 4>& ctr,
                                           const std::array<std::uint64_t, 2>& key) {
  // Philox4x64 with the Random123 multipliers and Weyl key increments
  std::uint64_t x0 = ctr[0], x1 = ctr[1], x2 = ctr[2], x3 = ctr[3];
  std::uint64_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    const unsigned __int128 p0 = (unsigned __int128)0xD2E7470EE14C6C93ull * x0;
    const unsigned __int128 p1 = (unsigned __int128)0xCA5A826395121157ull * x2;
    const std::uint64_t hi0 = (std::uint64_t)(p0 >> 64), lo0 = (std::uint64_t)p0;
    const std::uint64_t hi1 = (std::uint64_t)(p1 >> 64), lo1 = (std::uint64_t)p1;
    x0 = hi1 ^ x1 ^ k0;
    x1 = lo1;
    x2 = hi0 ^ x3 ^ k1;
    x3 = lo0;
    k0 += 0x9E3779B97F4A7C15ull;
    k1 += 0xBB67AE8584CAA73Bull;
  }
  return {x0, x1, x2, x3};
}
}  // namespace rng_detail

RngStream::RngStream(const StreamKey& key, std::uint64_t substream)
    : ctr_{0, key.node, (static_cast<std::uint64_t>(key.level) << 16) |
                            static_cast<std::uint64_t>(key.role),
           substream},
      key_{key.seed, 0x243F6A8885A308D3ull} {}

std::uint64_t RngStream::next_u64() {
  if (pos_ == 4) {
    buf_ = rng_detail::philox4x64_10(ctr_, key_);
    ++ctr_[0];
    pos_ = 0;
  }
  return buf_[pos_++];
}
double RngStream::uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
double RngStream::uniform_pos() {
  return (static_cast<double>(next_u64() >> 12) + 0.5) * 0x1.0p-52;
}
double RngStream::normal() {
  if (has_cached_) {
    has_cached_ = false;
    return cached_;
  }
  const double u1 = uniform_pos(), u2 = uniform();
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double th = 2.0 * 3.141592653589793238462643383279502884 * u2;
  cached_ = r * std::sin(th);
  has_cached_ = true;
  return r * std::cos(th);
}
std::uint64_t RngStream::uniform_index(std::uint64_t n) {
  if (n == 0) throw std::invalid_argument("uniform_index: n must be >= 1");
  return static_cast<std::uint64_t>(((unsigned __int128)next_u64() * n) >> 64);
}
void RngStream::fill_uniform(double* out, std::size_t n) {
  for (std::size_t i = 0; i < n; ++i) out[i] = uniform();
}
void RngStream::fill_normal(double* out, std::size_t n) {
  for (std::size_t i = 0; i < n; ++i) out[i] = normal();
}

// ------------------------------------------------------- kalman extras
namespace {

// Lower Cholesky factor with the escalating jitter of kalman.cpp:15-26
// (symmetrise, then up to 4 attempts adding scale * 10^(k-12) I).
std::vector<double> robust_cholesky(std::vector<double> P, int d, const char* what) {
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < i; ++j) P[i * d + j] = P[j * d + i] = 0.5 * (P[i * d + j] + P[j * d + i]);
  double tr = 0.0;
  for (int i = 0; i < d; ++i) tr += P[i * d + i];
  const double scale = std::max(tr / d, 1e-300);
  for (int attempt = 0; attempt < 4; ++attempt) {
    std::vector<double> L(d * d, 0.0);
    bool ok = true;
    for (int j = 0; j < d && ok; ++j) {
      double s = P[j * d + j];
      for (int k = 0; k < j; ++k) s -= L[j * d + k] * L[j * d + k];
      if (!(s > 0.0)) {
        ok = false;
        break;
      }
      L[j * d + j] = std::sqrt(s);
      for (int i = j + 1; i < d; ++i) {
        double v = P[i * d + j];
        for (int k = 0; k < j; ++k) v -= L[i * d + k] * L[j * d + k];
        L[i * d + j] = v / L[j * d + j];
      }
    }
    if (ok) return L;
    for (int i = 0; i < d; ++i) P[i * d + i] += scale * std::pow(10.0, attempt - 12);
  }
  throw std::runtime_error(std::string(what) + ": covariance is not positive definite");
}

std::vector<double> draw_gaussian(const std::vector<double>& mean, const std::vector<double>& cov,
                                  RngStream& stream, const char* what) {
  const int d = static_cast<int>(mean.size());
  const std::vector<double> L = robust_cholesky(cov, d, what);
  std::vector<double> z(d), x(mean);
  stream.fill_normal(z.data(), d);
  for (int i = 0; i < d; ++i)
    for (int k = 0; k <= i; ++k) x[i] += L[i * d + k] * z[k];
  return x;
}

std::vector<double> matvec(const std::vector<double>& A, const std::vector<double>& x, int rows) {
  const int cols = static_cast<int>(x.size());
  std::vector<double> y(rows, 0.0);
  for (int i = 0; i < rows; ++i)
    for (int k = 0; k < cols; ++k) y[i] += A[i * cols + k] * x[k];
  return y;
}

}  // namespace

LgssmSample simulate_lgssm(const LinearGaussianModel& m, RngStream& stream) {
  const int T = m.horizon, dx = m.dim_x, dy = m.dim_y;
  if (T < 0 || (int)m.F.size() != T + 1 || (int)m.H.size() != T + 1 ||
      (int)m.has_obs.size() != T + 1)
    throw std::invalid_argument("simulate_lgssm: arrays must have horizon+1 entries");
  LgssmSample out;
  out.x.resize(T + 1);
  out.y.assign(T + 1, std::vector<double>(dy, 0.0));
  out.x[0] = draw_gaussian(m.m0, m.P0, stream, "simulate");
  for (int t = 1; t <= T; ++t) {
    std::vector<double> mu = matvec(m.F[t], out.x[t - 1], dx);
    for (int k = 0; k < dx; ++k) mu[k] += m.b[t][k];
    out.x[t] = draw_gaussian(mu, m.Q[t], stream, "simulate");
  }
  for (int t = 0; t <= T; ++t)
    if (m.has_obs[t]) out.y[t] = draw_gaussian(matvec(m.H[t], out.x[t], dy), m.R[t], stream,
                                               "simulate");
  return out;
}

LinearGaussianModel linearize(const NonlinearGaussianModel& m,
                              const std::vector<std::vector<double>>& ref) {
  if ((int)ref.size() != m.horizon + 1)
    throw std::invalid_argument("linearize: reference length != horizon+1");
  const int d = m.dim_x;
  LinearGaussianModel lin;
  lin.dim_x = d;
  lin.dim_y = m.dim_y;
  lin.horizon = m.horizon;
  lin.m0 = m.m0;
  lin.P0 = m.P0;
  lin.F.assign(m.horizon + 1, std::vector<double>(d * d, 0.0));
  lin.b.assign(m.horizon + 1, std::vector<double>(d, 0.0));
  lin.Q = m.Q;
  lin.H = m.H;
  lin.R = m.R;
  lin.y = m.y;
  lin.has_obs = m.has_obs;
  for (int t = 1; t <= m.horizon; ++t) {
    const std::vector<double>& r = ref[t - 1];
    std::vector<double> J(d * d);
    if (m.f_jac) {
      J = m.f_jac(t, r);
    } else {  // central differences, step 1e-6 (1 + |x_i|) (kalman.cpp:177-190)
      for (int i = 0; i < d; ++i) {
        const double h = 1e-6 * (1.0 + std::fabs(r[i]));
        std::vector<double> xp = r, xm = r;
        xp[i] += h;
        xm[i] -= h;
        const std::vector<double> fp = m.f(t, xp), fm = m.f(t, xm);
        for (int k = 0; k < d; ++k) J[k * d + i] = (fp[k] - fm[k]) / (2.0 * h);
      }
    }
    lin.F[t] = J;
    const std::vector<double> fr = m.f(t, r), Jr = matvec(J, r, d);
    for (int k = 0; k < d; ++k) lin.b[t][k] = fr[k] - Jr[k];
  }
  return lin;
}

IteratedSmoothResult iterated_smooth(const NonlinearGaussianModel& m, int iterations,
                                     const std::vector<std::vector<double>>* initial_ref) {
  if (iterations < 1) throw std::invalid_argument("iterated_smooth: iterations must be >= 1");
  std::vector<std::vector<double>> ref;
  if (initial_ref) {
    ref = *initial_ref;
  } else {
    ref.resize(m.horizon + 1);
    ref[0] = m.m0;
    for (int t = 1; t <= m.horizon; ++t) ref[t] = m.f(t, ref[t - 1]);
  }
  IteratedSmoothResult out;
  for (int it = 0; it < iterations; ++it) {
    out.linearized = linearize(m, ref);
    out.kr = kalman_smooth(out.linearized);
    ref = out.kr.smooth_mean;
    out.iterations = it + 1;
  }
  out.ref = ref;
  return out;
}

// ------------------------------------------------------- model extras
double cox_score(const CoxParams& p, const double* path, int horizon) {
  const double s2 = p.sigma2;
  const double d0 = path[0] - p.mu;
  double acc = -(horizon + 1) / (2.0 * s2) + (1.0 - p.rho * p.rho) / (2.0 * s2 * s2) * d0 * d0;
  for (int t = 1; t <= horizon; ++t) {
    const double e = path[t] - p.mu - p.rho * (path[t - 1] - p.mu);
    acc += e * e / (2.0 * s2 * s2);
  }
  return acc;
}

namespace {
std::uint64_t poisson_by_products(double rate, RngStream& stream) {
  if (!(rate >= 0.0)) throw std::invalid_argument("poisson_draw: rate must be nonnegative");
  std::uint64_t total = 0;
  while (rate > 0.0) {  // chunks of <= 30 keep exp(-chunk) representable
    const double chunk = std::min(rate, 30.0);
    rate -= chunk;
    const double limit = std::exp(-chunk);
    double prod = 1.0;
    std::uint64_t k = 0;
    do {
      ++k;
      prod *= stream.uniform_pos();
    } while (prod > limit);
    total += k - 1;
  }
  return total;
}
}  // namespace

CoxData simulate_cox(const CoxParams& p, int horizon, std::uint64_t seed) {
  if (horizon < 0) throw std::invalid_argument("simulate_cox: horizon must be >= 0");
  const double a = p.rho * p.lambda;
  if (!(p.sigma2 > 0.0) || !(std::abs(a) < 1.0))
    throw std::invalid_argument("simulate_cox: invalid parameters");
  const double c = p.mu * (1.0 - p.rho);
  RngStream st({seed, 0, 0, StreamRole::data_sim});
  CoxData d;
  d.xs.resize(horizon + 1);
  d.ys.resize(horizon + 1);
  d.xs[0] = c / (1.0 - a) + std::sqrt(p.sigma2 / (1.0 - a * a)) * st.normal();
  for (int t = 1; t <= horizon; ++t) d.xs[t] = c + a * d.xs[t - 1] + std::sqrt(p.sigma2) * st.normal();
  for (int t = 0; t <= horizon; ++t)
    d.ys[t] = static_cast<double>(poisson_by_products(std::exp(d.xs[t]), st));
  return d;
}

double rw_score(double sigma, const double* path, int horizon) {
  double acc = 0.0;
  for (int t = 1; t <= horizon; ++t) acc += (path[t] - path[t - 1]) * (path[t] - path[t - 1]);
  return std::log(sigma) + acc / (sigma * sigma * sigma);
}

NonlinearGaussianModel theta_logistic_nonlinear(const ThetaLogisticParams& p,
                                                const std::vector<double>& ys) {
  if (!(p.q2 > 0.0) || !(p.r2 > 0.0))
    throw std::invalid_argument("theta_logistic_nonlinear: q2 and r2 must be > 0");
  if (ys.empty()) throw std::invalid_argument("theta_logistic_nonlinear: no observations");
  for (double y : ys)
    if (!std::isfinite(y))
      throw std::invalid_argument("theta_logistic_nonlinear: observations must be finite");
  const int T = static_cast<int>(ys.size()) - 1;
  NonlinearGaussianModel m;
  m.horizon = T;
  m.m0 = {0.0};
  m.P0 = {1.0};
  m.f = [p](int, const std::vector<double>& x) {
    return std::vector<double>{x[0] + p.tau0 - p.tau1 * std::exp(p.tau2 * x[0])};
  };
  m.f_jac = [p](int, const std::vector<double>& x) {
    return std::vector<double>{1.0 - p.tau1 * p.tau2 * std::exp(p.tau2 * x[0])};
  };
  m.Q.assign(T + 1, {p.q2});
  m.H.assign(T + 1, {1.0});
  m.R.assign(T + 1, {p.r2});
  m.y.resize(T + 1);
  for (int t = 0; t <= T; ++t) m.y[t] = {ys[t]};
  m.has_obs.assign(T + 1, 1);
  return m;
}

ThetaLogisticData simulate_theta_logistic(const ThetaLogisticParams& p, int horizon,
                                          std::uint64_t seed) {
  if (horizon < 0) throw std::invalid_argument("simulate_theta_logistic: horizon must be >= 0");
  if (!(p.q2 > 0.0) || !(p.r2 > 0.0))
    throw std::invalid_argument("simulate_theta_logistic: invalid parameters");
  RngStream st({seed, 0, 1, StreamRole::data_sim});
  ThetaLogisticData d;
  d.xs.resize(horizon + 1);
  d.ys.resize(horizon + 1);
  d.xs[0] = st.normal();
  for (int t = 1; t <= horizon; ++t) {
    const double x = d.xs[t - 1];
    d.xs[t] = x + p.tau0 - p.tau1 * std::exp(p.tau2 * x) + std::sqrt(p.q2) * st.normal();
  }
  for (int t = 0; t <= horizon; ++t) d.ys[t] = d.xs[t] + std::sqrt(p.r2) * st.normal();
  return d;
}

// ------------------------------------------------------- pgibbs extras
double gamma_draw(double shape, double rate, RngStream& stream) {
  if (!(shape > 0.0) || !(rate > 0.0))
    throw std::invalid_argument("gamma_draw: shape and rate must be > 0");
  double boost = 1.0;
  if (shape < 1.0) {
    boost = std::pow(stream.uniform_pos(), 1.0 / shape);
    shape += 1.0;
  }
  const double d = shape - 1.0 / 3.0, c = 1.0 / std::sqrt(9.0 * d);
  for (;;) {
    double x, v;
    do {
      x = stream.normal();
      v = 1.0 + c * x;
    } while (v <= 0.0);
    v = v * v * v;
    const double u = stream.uniform_pos();
    if (std::log(u) < 0.5 * x * x + d - d * v + d * std::log(v)) return boost * d * v / rate;
  }
}

namespace {
double theta_drift(const ThetaLogisticParams& p, double x) {
  return x + p.tau0 - p.tau1 * std::exp(p.tau2 * x);
}

// pgibbs.cpp:114-134: every joint-density term that moves with (tau, x_0)
double rwm_target(const ThetaLogisticParams& p, double x0, const std::vector<double>& ys,
                  const std::vector<double>& star, const ThetaLogisticGibbsConfig& g) {
  if (p.tau1 <= 0.0 || p.tau2 <= 0.0) return -INFINITY;
  double acc = log_normal_pdf(p.tau0, 0.0, g.tau0_sd * g.tau0_sd) +
               log_normal_pdf(p.tau1, 0.0, g.tau1_sd * g.tau1_sd) +
               log_normal_pdf(p.tau2, 0.0, g.tau2_sd * g.tau2_sd) +
               log_normal_pdf(x0, 0.0, 1.0) + log_normal_pdf(ys[0], x0, p.r2);
  double prev = x0;
  for (std::size_t t = 1; t < star.size(); ++t) {
    acc += log_normal_pdf(star[t], theta_drift(p, prev), p.q2);
    prev = star[t];
  }
  return acc;
}

ThetaLogisticParams unpack_theta(const std::vector<double>& v) {
  if (v.size() != 5) throw std::invalid_argument("theta vector has the wrong size");
  return {v[0], v[1], v[2], v[3], v[4]};
}
std::vector<double> pack_theta(const ThetaLogisticParams& p) {
  return {p.tau0, p.tau1, p.tau2, p.q2, p.r2};
}
}  // namespace

ThetaLogisticParams draw_precisions(const ThetaLogisticParams& params,
                                    const std::vector<double>& ys,
                                    const std::vector<double>& star,
                                    const ThetaLogisticGibbsConfig& g, RngStream& stream) {
  if (star.size() != ys.size() || star.empty())
    throw std::invalid_argument("draw_precisions: path and observations must have equal length");
  const std::size_t T = star.size() - 1;
  double ssx = 0.0, ssy = 0.0;
  for (std::size_t t = 1; t <= T; ++t) {
    const double r = star[t] - theta_drift(params, star[t - 1]);
    ssx += r * r;
  }
  for (std::size_t t = 0; t <= T; ++t) ssy += (ys[t] - star[t]) * (ys[t] - star[t]);
  ThetaLogisticParams out = params;
  const double px = gamma_draw(g.prec_x_shape + 0.5 * T, g.prec_x_rate + 0.5 * ssx, stream);
  const double py = gamma_draw(g.prec_y_shape + 0.5 * (T + 1), g.prec_y_rate + 0.5 * ssy, stream);
  out.q2 = 1.0 / px;
  out.r2 = 1.0 / py;
  return out;
}

ThetaLogisticChain run_theta_logistic_pgibbs(const std::vector<double>& ys,
                                             const ThetaLogisticParams& init,
                                             const ThetaLogisticGibbsConfig& g,
                                             std::size_t sweeps, std::uint64_t seed) {
  if (ys.size() < 2)
    throw std::invalid_argument("run_theta_logistic_pgibbs: need at least two observations");
  if (!(init.q2 > 0.0) || !(init.r2 > 0.0) || init.tau1 <= 0.0 || init.tau2 <= 0.0)
    throw std::invalid_argument(
        "run_theta_logistic_pgibbs: initial parameters outside the prior support");
  if (g.ieks_cold_iterations < 1)
    throw std::invalid_argument(
        "run_theta_logistic_pgibbs: need at least one cold-start iteration");
  // cold start: linearised smoothing at init; the retained path = smoothed means
  GibbsState state;
  state.theta = pack_theta(init);
  {
    const IteratedSmoothResult it =
        iterated_smooth(theta_logistic_nonlinear(init, ys), g.ieks_cold_iterations);
    state.proposal_cache = proposal_marginals(it.kr, g.proposal_inflation);
    state.ieks_ref = it.ref;
    state.star.resize(ys.size());
    for (std::size_t t = 0; t < ys.size(); ++t) state.star[t] = it.kr.smooth_mean[t][0];
  }
  ConditionalOptions co;
  co.n_particles = g.n_particles;
  co.resampler = g.resampler;
  co.seed = seed;
  co.precision = g.precision;
  co.device = g.device;
  ThetaLogisticChain chain;
  std::size_t* accepts = &chain.rwm_accepts;
  ParamKernel kernel = [&ys, &g, accepts](GibbsState& s, RngStream& st) {
    ThetaLogisticParams p = draw_precisions(unpack_theta(s.theta), ys, s.star, g, st);
    ThetaLogisticParams q = p;
    q.tau0 = p.tau0 + g.rwm_step_tau * st.normal();
    q.tau1 = p.tau1 + g.rwm_step_tau * st.normal();
    q.tau2 = p.tau2 + g.rwm_step_tau * st.normal();
    const double x0 = s.star[0], x0q = x0 + g.rwm_step_x0 * st.normal();
    const double delta = rwm_target(q, x0q, ys, s.star, g) - rwm_target(p, x0, ys, s.star, g);
    if (std::log(st.uniform_pos()) < delta) {
      p = q;
      s.star[0] = x0q;
      ++*accepts;
    }
    s.theta = pack_theta(p);
  };
  // one warm IEKS step per sweep refreshes the proposals (pgibbs.cpp:244-252)
  GibbsModelBuilder builder = [&ys, &g](GibbsState& s) {
    const ThetaLogisticParams p = unpack_theta(s.theta);
    const IteratedSmoothResult it = iterated_smooth(theta_logistic_nonlinear(p, ys), 1, &s.ieks_ref);
    s.proposal_cache = proposal_marginals(it.kr, g.proposal_inflation);
    s.ieks_ref = it.ref;
    return make_theta_logistic(p, ys, s.proposal_cache);
  };
  chain.thetas.reserve(sweeps);
  chain.stars.reserve(sweeps);
  chain.changed.reserve(sweeps);
  for (std::size_t s = 1; s <= sweeps; ++s) {
    SweepOutcome out = pgibbs_sweep(state, builder, kernel, co, static_cast<std::uint32_t>(s));
    state = std::move(out.state);
    chain.thetas.push_back(unpack_theta(state.theta));
    chain.stars.push_back(state.star);
    chain.changed.push_back(std::move(out.changed));
    chain.weight_evals += out.meta.weight_evals;
  }
  return chain;
}

// ------------------------------------------------------------- baselines
FfbsResult ffbs_smooth(const FeynmanKacModel& model, std::size_t n, Resampler resampler,
                       std::uint64_t seed, std::size_t n_draws, int device) {
  validate_model(model);
  if (resampler_is_lazy(resampler))
    throw std::invalid_argument("the particle filter resamples with a dense scheme "
                                "(multinomial or systematic)");
  const dsmc_model_desc& desc = desc_of(model);
  dsmc_ctx* c = context(device);
  const int K = model.horizon + 1, d = model.state_dim;
  FfbsResult r;
  r.n_draws = n_draws ? n_draws : n;
  r.horizon = model.horizon;
  r.dim = d;
  r.paths.resize(r.n_draws * K * d);
  std::vector<double> mean((size_t)K * d), cov((size_t)K * d * d);
  dsmc_ffbs_opts fo{n, r.n_draws, static_cast<int>(resampler), seed};
  check(c, dsmc_ffbs_smooth(c, &desc, &fo, mean.data(), cov.data(), r.paths.data(),
                            &r.log_likelihood));
  r.density_evals = static_cast<std::uint64_t>(r.n_draws) * model.horizon * n;
  return r;
}

}  // namespace dsmc

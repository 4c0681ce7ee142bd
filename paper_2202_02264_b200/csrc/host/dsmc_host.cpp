// C++ host layer (include/dsmc/dsmc.hpp) over the C ABI. Keeps the
// reference's dsmc:: entry points and exception classes; all numerical work
// is delegated to the CUDA engine (libdsmc_b200.so).
#include "dsmc/dsmc.hpp"

#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>

namespace dsmc {

struct DeviceModel {
  dsmc_model_desc desc{};
  std::vector<double> m0, P0, F, b, Q, H, R, y, prop_mean, prop_cov;
  std::vector<uint8_t> has_obs;
  void bind() {
    auto p = [](std::vector<double>& v) { return v.empty() ? nullptr : v.data(); };
    desc.m0 = p(m0);
    desc.P0 = p(P0);
    desc.F = p(F);
    desc.b = p(b);
    desc.Q = p(Q);
    desc.H = p(H);
    desc.R = p(R);
    desc.y = p(y);
    desc.prop_mean = p(prop_mean);
    desc.prop_cov = p(prop_cov);
    desc.has_obs = has_obs.empty() ? nullptr : has_obs.data();
  }
};

namespace {

constexpr double kLog2Pi = 1.8378770664093454836;

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
        "described by data (make_lgssm_fk, make_sv_model)");
  return m.device->desc;
}

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

}  // namespace

// ------------------------------------------------------------ resampling
std::optional<Resampler> parse_resampler(const std::string& name) {
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
  return fk;
}

// -------------------------------------------------------------- fk_model
void validate_model(const FeynmanKacModel& model) {
  if (model.state_dim < 1) throw std::invalid_argument("model: state_dim must be >= 1");
  if (model.horizon < 0) throw std::invalid_argument("model: horizon must be >= 0");
  const dsmc_model_desc& d = desc_of(model);
  if (d.horizon != model.horizon || d.state_dim != model.state_dim)
    throw std::invalid_argument("model: device descriptor disagrees with the callbacks");
}

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
  validate_model(model);
  const dsmc_model_desc& desc = desc_of(model);
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
  validate_model(model);
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
  kernel(out.state, o.seed, sweep);
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

}  // namespace dsmc

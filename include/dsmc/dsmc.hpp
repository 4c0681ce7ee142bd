// C++ host interface of the B200 dSMC engine, mirroring the reference's
// dsmc:: API (/root/reference/proj/include/dsmc/{fk_model,smoother,
// resampling,conditional,pgibbs,kalman}.hpp): same names, argument meaning
// and exception classes, so reference callers and tests port by re-linking.
// Every entry point runs on the GPU through the C ABI (include/dsmc_b200.h);
// there is no CPU fallback: a model without a device descriptor, or a host
// without a CUDA device, raises.
//
// Differences from the reference:
//  * FeynmanKacModel keeps the reference's callbacks (fk_model.hpp:37-86)
//    for host-side use and validation, and adds `device`, the plain-data
//    description the kernels run (std::function cannot run on a GPU).
//  * BlockEstimate holds the root population only (ancestor composition
//    replaces the reference's per-combine path copies).
//  * Matrices are row-major std::vector<double> (no Eigen in this image).
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "dsmc_b200.h"

namespace dsmc {

// ------------------------------------------------------------- rng.hpp
enum class StreamRole : std::uint16_t {
  leaf_proposal = 1,
  pair_resample = 2,
  star_select = 3,
  gibbs_param = 4,
  data_sim = 5,
  filter_step = 6,
  backward_sample = 7,
};

struct StreamKey {
  std::uint64_t seed = 0;
  std::uint32_t level = 0;
  std::uint64_t node = 0;
  StreamRole role = StreamRole::leaf_proposal;
};

// ------------------------------------------------------ resampling.hpp
enum class Resampler { multinomial, systematic, mh_lazy, rejection_lazy };

std::optional<Resampler> parse_resampler(const std::string& name);
std::string resampler_name(Resampler r);
bool resampler_is_lazy(Resampler r);

struct PairSample {
  std::vector<std::uint32_t> left, right;
  std::optional<double> log_mean_weight;
  std::uint64_t weight_evals = 0;
  bool biased = false;
};

// resample_pairs (resampling.hpp:85-87) for a dense table source
// (n x n row-major log weights; log_upper_bound for rejection).
PairSample resample_pairs(Resampler r, const std::vector<double>& logw,
                          std::size_t n, std::size_t n_out,
                          std::size_t mh_steps, const StreamKey& key,
                          std::optional<double> log_upper_bound = {});

// ------------------------------------------------------- kalman.hpp
struct LinearGaussianModel {
  int dim_x = 1, dim_y = 1, horizon = 0;
  std::vector<double> m0, P0;          // d, d*d
  std::vector<std::vector<double>> F, b, Q, H, R, y;  // per time (index 0
                                                      // of F/b/Q unused)
  std::vector<char> has_obs;
};

struct KalmanResult {
  std::vector<std::vector<double>> smooth_mean, smooth_cov;
  double log_likelihood = 0.0;
};
KalmanResult kalman_smooth(const LinearGaussianModel& m);

// ------------------------------------------------------ fk_model.hpp
class RngStream;  // host streams are not needed on the GPU path

struct DeviceModel;  // owning storage behind a dsmc_model_desc

struct FeynmanKacModel {
  int state_dim = 1;
  int horizon = 0;
  // the reference's callbacks (host-side validation / scalar checks)
  std::function<double(int t, const double* x)> proposal_logdensity;
  std::function<double(int t, const double* x)> aux_logdensity;
  std::function<double(int t, const double* x)> log_potential;
  std::function<double(int t, const double* x_prev, const double* x_cur)>
      transition_logdensity;
  std::function<double(const double* x)> init_logdensity;
  std::function<double(int c)> log_stitch_bound;
  // what the GPU runs
  std::shared_ptr<DeviceModel> device;
};

void validate_model(const FeynmanKacModel& model);
double log_stitch_weight(const FeynmanKacModel& model, int c,
                         const double* x_prev, const double* x_cur);

struct ProposalMarginal {
  std::vector<double> mean, cov;  // d, d*d
};

// make_lgssm_fk (models.cpp:562-685), generalised to d <= 4: q_t = nu_t =
// N(marginal_t).
FeynmanKacModel make_lgssm_fk(const LinearGaussianModel& m,
                              const std::vector<ProposalMarginal>& marginals);
std::vector<ProposalMarginal> proposal_marginals(const KalmanResult& kr,
                                                 double inflation = 1.0);

struct SvParams {
  double mu = -1.0, phi = 0.95, sigma2 = 0.09;
};
// Stochastic volatility with q_t = nu_t = |y_t| h_t.
FeynmanKacModel make_sv_model(const SvParams& p, const std::vector<double>& ys);

// models.hpp:29-50 / models.cpp:111-216: log-Gaussian Cox counts over an
// AR(1) intensity, proposals = the stationary law (same fields and defaults
// as the reference's CoxParams). ys.size() == T + 1 sets the horizon.
struct CoxParams {
  double mu = 0.0;
  double rho = 0.9;
  double sigma2 = 0.25;
  double lambda = 1.0;
};
FeynmanKacModel make_cox_model(const CoxParams& p, const std::vector<double>& ys);

// models.cpp:263-338: random walk conditioned to stay inside [-1, 1],
// U[-1, 1] proposals, finite log_stitch_bound.
FeynmanKacModel make_constrained_rw(double sigma, int horizon);

// models.hpp:86-110 / models.cpp:407-491: theta-logistic dynamics with the
// caller's per-time proposal marginals (1-d ProposalMarginal entries).
struct ThetaLogisticParams {
  double tau0 = 0.15;
  double tau1 = 0.10;
  double tau2 = 0.10;
  double q2 = 0.05;
  double r2 = 0.05;
};
FeynmanKacModel make_theta_logistic(const ThetaLogisticParams& p, const std::vector<double>& ys,
                                    const std::vector<ProposalMarginal>& marginals);

// ------------------------------------------------------ smoother.hpp
enum class Precision { fp32 = DSMC_FP32, fp64_parity = DSMC_FP64_PARITY };

struct SmootherOptions {
  std::size_t n_particles = 256;
  Resampler resampler = Resampler::multinomial;
  std::size_t mh_steps = 16;
  std::uint64_t seed = 0;
  int n_threads = 1;  // accepted for source compatibility; the GPU ignores it
  Precision precision = Precision::fp32;
  int device = 0;
};

struct BlockEstimate {
  int a = 0, b = 0;
  std::size_t n = 0;
  int dim = 1;
  std::vector<double> paths;  // (b-a+1)*n*dim, slab-major by time
  std::vector<double> log_w;  // n normalised (uniform at the root)
  bool weights_uniform = true;
  std::optional<double> log_norm_const;
  bool biased = false;
  std::uint64_t weight_evals = 0;
  int len() const { return b - a + 1; }
  const double* time_slab(int t) const {
    return paths.data() + static_cast<std::size_t>(t - a) * n * dim;
  }
};

struct RunMetadata {
  int horizon = 0;
  std::size_t n_particles = 0;
  std::string resampler;
  int levels = 0;
  std::uint64_t weight_evals = 0;
  double wall_time_ms = 0.0;
  std::optional<double> log_norm_const;
  std::uint64_t seed = 0;
  bool biased = false;
};

struct RunResult {
  BlockEstimate root;
  RunMetadata meta;
  std::vector<double> mean, cov;  // per-time smoothed moments (device)
};

struct SchedulePair {
  int level = 0, node = 0, left_a = 0, left_b = 0, right_b = 0;
};
struct CombineSchedule {
  int horizon = 0, levels = 0;
  std::vector<SchedulePair> pairs;
};
CombineSchedule build_schedule(int horizon);
int reference_tree_depth(int horizon);

RunResult run_smoother(const FeynmanKacModel& model,
                       const SmootherOptions& options);

std::vector<double> weighted_time_mean(const BlockEstimate& block, int t);
void copy_path(const BlockEstimate& block, std::size_t p, double* out);

// --------------------------------------------------- conditional.hpp
struct ConditionalOptions {
  std::size_t n_particles = 256;
  Resampler resampler = Resampler::multinomial;
  std::uint64_t seed = 0;
  Precision precision = Precision::fp32;
  int device = 0;
};

struct ConditionalResult {
  std::vector<double> path;
  RunMetadata meta;
};

ConditionalResult run_conditional(const FeynmanKacModel& model,
                                  const double* ref,
                                  const ConditionalOptions& options,
                                  std::uint32_t sweep);

std::vector<char> path_changed_times(const double* a, const double* b, int len,
                                     int dim);

// -------------------------------------------------------- pgibbs.hpp
struct GibbsState {
  std::vector<double> theta;
  std::vector<double> star;
};
using ParamKernel = std::function<void(GibbsState&, std::uint64_t seed,
                                       std::uint32_t sweep)>;
using GibbsModelBuilder = std::function<FeynmanKacModel(GibbsState&)>;

struct SweepOutcome {
  GibbsState state;
  std::vector<char> changed;
  RunMetadata meta;
};

// pgibbs_sweep (pgibbs.hpp:55-59): param kernel, model rebuild, conditional
// path update on the GPU; strong guarantee (the input state is untouched on
// any throw).
SweepOutcome pgibbs_sweep(const GibbsState& state,
                          const GibbsModelBuilder& model_builder,
                          const ParamKernel& param_kernel,
                          const ConditionalOptions& options,
                          std::uint32_t sweep);

std::vector<double> update_rate(const std::vector<std::vector<double>>& stars,
                                int dim = 1);

// Batched SV particle Gibbs: n_chains chains advanced one sweep each, the
// parameter kernel and the c-dSMC path update both on the device.
struct SvGibbsChains {
  std::vector<double> theta;  // n_chains * 3 (mu, phi, sigma2)
  std::vector<double> stars;  // n_chains * (T+1)
  std::vector<std::uint64_t> seeds;
  std::uint64_t phi_accepts = 0;
};
std::vector<char> sv_pgibbs_sweep(SvGibbsChains& chains,
                                  const std::vector<double>& ys,
                                  const dsmc_sv_prior& prior,
                                  const ConditionalOptions& options,
                                  std::uint32_t sweep);

}  // namespace dsmc

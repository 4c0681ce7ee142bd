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

#include <array>
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

// Host Philox4x64-10 streams (rng.hpp:33-62, rng.cpp:27-101): the same
// counter layout {block, node, level << 16 | role, substream} and key {seed,
// 0x243F6A8885A308D3}, four u64 per block. The GPU kernels draw from the same
// counters; host streams serve data simulation and the particle-Gibbs
// parameter kernels.
namespace rng_detail {
std::array<std::uint64_t, 4> philox4x64_10(const std::array<std::uint64_t, 4>& ctr,
                                           const std::array<std::uint64_t, 2>& key);
}  // namespace rng_detail

class RngStream {
 public:
  explicit RngStream(const StreamKey& key, std::uint64_t substream = 0);
  std::uint64_t next_u64();
  double uniform();      // [0, 1), 53 bits
  double uniform_pos();  // (0, 1)
  double normal();       // Box-Muller, cos first then the cached sin
  std::uint64_t uniform_index(std::uint64_t n);
  void fill_uniform(double* out, std::size_t n);
  void fill_normal(double* out, std::size_t n);

 private:
  std::array<std::uint64_t, 4> ctr_, buf_{};
  std::array<std::uint64_t, 2> key_;
  int pos_ = 4;
  bool has_cached_ = false;
  double cached_ = 0.0;
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

// kalman.hpp:59-63 / kalman.cpp:157-175: x_0 ~ N(m0, P0), x_t ~ N(F x + b, Q),
// then y_t ~ N(H x_t, R) where observed; Gaussian draws through the
// jitter-escalating Cholesky (kalman.cpp:15-26) and fill_normal.
struct LgssmSample {
  std::vector<std::vector<double>> x, y;
};
LgssmSample simulate_lgssm(const LinearGaussianModel& m, RngStream& stream);

// kalman.hpp:65-110: additive-noise nonlinear dynamics, linearisation around a
// reference trajectory (analytic Jacobian when given, else central
// differences) and the iterated (IEKS) smoother.
struct NonlinearGaussianModel {
  int dim_x = 1, dim_y = 1, horizon = 0;
  std::vector<double> m0, P0;
  std::function<std::vector<double>(int t, const std::vector<double>& x)> f;
  std::function<std::vector<double>(int t, const std::vector<double>& x)> f_jac;  // d*d
  std::vector<std::vector<double>> Q, H, R, y;
  std::vector<char> has_obs;
};
LinearGaussianModel linearize(const NonlinearGaussianModel& m,
                              const std::vector<std::vector<double>>& ref);
struct IteratedSmoothResult {
  LinearGaussianModel linearized;
  KalmanResult kr;
  std::vector<std::vector<double>> ref;
  int iterations = 0;
};
IteratedSmoothResult iterated_smooth(const NonlinearGaussianModel& m, int iterations,
                                     const std::vector<std::vector<double>>* initial_ref = nullptr);

// ------------------------------------------------------ fk_model.hpp
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
// models.hpp:52-60: the score functional of the experiments and the data
// simulation (stream {seed, 0, 0, data_sim}, Poisson by product of uniforms
// in chunks of rate <= 30).
double cox_score(const CoxParams& p, const double* path, int horizon);
struct CoxData {
  std::vector<double> xs, ys;
};
CoxData simulate_cox(const CoxParams& p, int horizon, std::uint64_t seed);

// models.cpp:263-338: random walk conditioned to stay inside [-1, 1],
// U[-1, 1] proposals, finite log_stitch_bound.
FeynmanKacModel make_constrained_rw(double sigma, int horizon);
double rw_score(double sigma, const double* path, int horizon);  // models.cpp:340-347

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
NonlinearGaussianModel theta_logistic_nonlinear(const ThetaLogisticParams& p,
                                                const std::vector<double>& ys);
struct ThetaLogisticData {
  std::vector<double> xs, ys;
};
// stream {seed, 0, 1, data_sim} (models.cpp:517-540)
ThetaLogisticData simulate_theta_logistic(const ThetaLogisticParams& p, int horizon,
                                          std::uint64_t seed);

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
  std::vector<ProposalMarginal> proposal_cache;
  std::vector<std::vector<double>> ieks_ref;
};
// pgibbs.hpp:43-47: the kernel draws from the sweep's parameter stream
// {options.seed, 0, sweep, gibbs_param}.
using ParamKernel = std::function<void(GibbsState&, RngStream&)>;
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

// pgibbs.cpp:80-102: Marsaglia-Tsang with the shape < 1 boost.
double gamma_draw(double shape, double rate, RngStream& stream);

// pgibbs.hpp:70-115: the theta-logistic particle-Gibbs driver (precision
// draws, joint RWM on (tau0, tau1, tau2, x_0), one warm IEKS refresh of the
// proposals, c-dSMC path update on the GPU).
struct ThetaLogisticGibbsConfig {
  double prec_x_shape = 2.0, prec_x_rate = 1.0;
  double prec_y_shape = 2.0, prec_y_rate = 1.0;
  double tau0_sd = 1.0, tau1_sd = 1.0, tau2_sd = 1.0;
  double rwm_step_tau = 0.05, rwm_step_x0 = 0.1;
  std::size_t n_particles = 64;
  Resampler resampler = Resampler::multinomial;
  int ieks_cold_iterations = 25;
  double proposal_inflation = 1.0;
  Precision precision = Precision::fp32;
  int device = 0;
};
ThetaLogisticParams draw_precisions(const ThetaLogisticParams& params,
                                    const std::vector<double>& ys,
                                    const std::vector<double>& star,
                                    const ThetaLogisticGibbsConfig& config, RngStream& stream);
struct ThetaLogisticChain {
  std::vector<ThetaLogisticParams> thetas;
  std::vector<std::vector<double>> stars;
  std::vector<std::vector<char>> changed;
  std::size_t rwm_accepts = 0;
  std::uint64_t weight_evals = 0;
};
ThetaLogisticChain run_theta_logistic_pgibbs(const std::vector<double>& ys,
                                             const ThetaLogisticParams& init,
                                             const ThetaLogisticGibbsConfig& config,
                                             std::size_t sweeps, std::uint64_t seed);

// ------------------------------------------------------ baselines.hpp
// run_particle_filter + ffbs_sample (baselines.hpp:42-63) as one device call
// (dsmc_ffbs_smooth): n_draws joint draws, draw-major paths.
struct FfbsResult {
  std::size_t n_draws = 0;
  int horizon = 0, dim = 1;
  std::vector<double> paths;
  std::uint64_t density_evals = 0;  // n_draws * T * n, as ffbs_sample counts
  double log_likelihood = 0.0;      // the filter's estimate
  const double* path(std::size_t m) const {
    return paths.data() + m * static_cast<std::size_t>(horizon + 1) * dim;
  }
};
FfbsResult ffbs_smooth(const FeynmanKacModel& model, std::size_t n, Resampler resampler,
                       std::uint64_t seed, std::size_t n_draws = 0, int device = 0);

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

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
#include <string_view>
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

// --------------------------------------------------------- metrics.hpp
// Process-wide counters of the memory/work contracts (metrics.hpp:10-26,
// metrics.cpp): stitch-weight evaluations, dense N^2 pair tables, the peak
// transient of the lazy samplers. The device dense combine evaluates its
// N x N table once, streaming (only N^2/64 sub-block sums are stored), and is
// counted here as one dense table of N^2 elements, as the reference counts
// its materialised table; lazy combines count none.
namespace metrics {
struct Snapshot {
  std::uint64_t weight_evals = 0;
  std::uint64_t dense_allocs = 0;
  std::uint64_t dense_max_elems = 0;
  std::uint64_t lazy_max_elems = 0;
};
void reset();
Snapshot snapshot();
void add_weight_evals(std::uint64_t n);
void count_dense_alloc(std::size_t elems);
void note_lazy_alloc(std::size_t elems);
}  // namespace metrics

// --------------------------------------------------------- kernels.hpp
// The reference dispatches its FP64 row kernels over scalar / AVX2 /
// AVX-512 backends that agree bit for bit (test_kernels.cpp). The device
// engine has one arithmetic, the scalar backend's operation order (FP64
// parity path); the selector is kept for source compatibility and records
// the caller's choice without changing any result.
namespace kernels {
enum class Backend { scalar, avx2, avx512 };
Backend active();
void set_active(Backend b);
bool available(Backend b);
inline constexpr std::size_t kSubBlock = 64;  // kernels.hpp:77
}  // namespace kernels

// ------------------------------------------------------ resampling.hpp
enum class Resampler { multinomial, systematic, mh_lazy, rejection_lazy };

std::optional<Resampler> parse_resampler(std::string_view name);
std::string resampler_name(Resampler r);
bool resampler_is_lazy(Resampler r);

struct PairSample {
  std::vector<std::uint32_t> left, right;
  std::optional<double> log_mean_weight;
  std::uint64_t weight_evals = 0;
  bool biased = false;
};

namespace detail {
struct BlockPairSource;  // device attachment of make_pair_source (below)
}

// resampling.hpp:21-31: a virtual n x n table of log pair weights.
// fill_row / log_weight_at / log_upper_bound are the reference's fields.
// `blocks` is set by make_pair_source for a device model: resample_pairs then
// evaluates and samples the table on the device from the two blocks'
// boundary slabs (never materialising it); sources built by the caller from
// host callbacks are evaluated on the host (that is where the callbacks
// live) and sampled on the device: the dense schemes upload the filled
// table, the lazy schemes answer the device's per-round probes.
struct PairWeightSource {
  std::size_t n = 0;
  std::function<void(std::size_t i, double* out)> fill_row;
  std::function<double(std::size_t i, std::size_t j)> log_weight_at;
  std::optional<double> log_upper_bound;
  std::shared_ptr<const detail::BlockPairSource> blocks;
};

// resampling.hpp:44-65, 85-87.
PairSample multinomial_pairs(const PairWeightSource& src, std::size_t n_out,
                             const StreamKey& key);
PairSample systematic_pairs(const PairWeightSource& src, std::size_t n_out,
                            const StreamKey& key);
PairSample mh_lazy_pairs(const PairWeightSource& src, std::size_t n_out,
                         std::size_t mh_steps, const StreamKey& key);
PairSample rejection_lazy_pairs(const PairWeightSource& src, std::size_t n_out,
                                const StreamKey& key);
PairSample resample_pairs(Resampler r, const PairWeightSource& src,
                          std::size_t n_out, std::size_t mh_steps,
                          const StreamKey& key);

// resample_pairs for a dense table (n x n row-major log weights;
// log_upper_bound for rejection): the reference tests' table source.
PairSample resample_pairs(Resampler r, const std::vector<double>& logw,
                          std::size_t n, std::size_t n_out,
                          std::size_t mh_steps, const StreamKey& key,
                          std::optional<double> log_upper_bound = {});

// resampling.hpp:67-83: single-population resampling for sequential filters.
struct IndexSample {
  std::vector<std::uint32_t> idx;
  double log_mean_weight = 0.0;  // log((1/n) sum_i exp(logw[i]))
};
IndexSample multinomial_indices(const double* log_w, std::size_t n,
                                std::size_t n_out, const StreamKey& key);
IndexSample systematic_indices(const double* log_w, std::size_t n,
                               std::size_t n_out, const StreamKey& key);
IndexSample resample_indices(Resampler r, const double* log_w, std::size_t n,
                             std::size_t n_out, const StreamKey& key);
// resampling.hpp:91: a glibc malloc tuning of the reference's dense buffers;
// nothing to tune here (no host N^2 buffers on the device path).
void tune_allocator_once();

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

// fk_model.hpp:25-35. StitchRowFn fills one row of log omega_c(x_prev, .)
// against the right slab bound by the factory; the shipped header declares a
// fused (x_prev, log_add, out) -> row_max form, while every reference .cpp
// and test uses this (x_prev, out) form, which is the one
// kept here so reference sources compile against this header.
using StitchRowFn = std::function<void(const double* x_prev, double* out)>;
using TransitionRowFn = std::function<void(const double* x_cur, double* out)>;

// fk_model.hpp:37-86: every field of the reference, plus `device`, the
// plain-data description the kernels run (std::function cannot run on a
// GPU). The model factories below fill both; a model with callbacks only is
// accepted by the host helpers (log_init_weight, make_stitch_row, ...) and
// rejected by the device entry points (there is no CPU fallback).
struct FeynmanKacModel {
  int state_dim = 1;
  int horizon = 0;
  std::function<void(int t, std::size_t count, RngStream& stream, double* out)>
      proposal_sampler;
  std::function<double(int t, const double* x)> proposal_logdensity;
  std::function<double(int t, const double* x)> aux_logdensity;
  std::function<double(int t, const double* x)> log_potential;
  std::function<double(int t, const double* x_prev, const double* x_cur)>
      transition_logdensity;
  std::function<double(const double* x)> init_logdensity;
  std::function<void(int t, const double* x_prev, RngStream& stream, double* out)>
      transition_sampler;
  std::function<StitchRowFn(int c, const double* right_particles, std::size_t n)>
      stitch_row_factory;
  std::function<void(int t, const double* particles, std::size_t n, double* out)>
      init_weight_batch;
  std::function<double(int c)> log_stitch_bound;
  std::function<TransitionRowFn(int t, const double* prev_particles, std::size_t n)>
      transition_row_factory;
  // what the GPU runs
  std::shared_ptr<DeviceModel> device;
};

void validate_model(const FeynmanKacModel& model);
// fk_model.hpp:96-116 / fk_model.cpp:43-112 (host, over the callbacks)
double log_init_weight(const FeynmanKacModel& model, int t, const double* x);
double log_stitch_weight(const FeynmanKacModel& model, int c,
                         const double* x_prev, const double* x_cur);
StitchRowFn make_stitch_row(const FeynmanKacModel& model, int c,
                            const double* right_particles, std::size_t n);
TransitionRowFn make_transition_row(const FeynmanKacModel& model, int t,
                                    const double* prev_particles, std::size_t n);
void leaf_weights(const FeynmanKacModel& model, int t, const double* particles,
                  std::size_t n, double* out);

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
  double* time_slab(int t) {
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

// smoother.hpp:98-125, on the device (FP64, the reference's arithmetic):
// make_leaf draws and weighs one leaf; make_pair_source returns the
// reference's virtual pair table of two adjacent blocks (host closures over
// the model callbacks, plus the device attachment resample_pairs uses);
// combine_blocks resamples n pairs on the device and concatenates the
// selected paths. Blocks hold full paths, as the reference's.
BlockEstimate make_leaf(const FeynmanKacModel& model, int t, std::size_t n,
                        std::uint64_t seed);
struct PairSourceBundle {
  PairWeightSource source;
  double log_shift = 0.0;
};
PairSourceBundle make_pair_source(const FeynmanKacModel& model,
                                  const BlockEstimate& left,
                                  const BlockEstimate& right);
BlockEstimate combine_blocks(const FeynmanKacModel& model,
                             const BlockEstimate& left,
                             const BlockEstimate& right,
                             const SmootherOptions& options, int level,
                             int node);

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

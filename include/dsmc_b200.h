/*
 * dsmc_b200.h — C ABI of the B200-native dSMC smoothing path.
 *
 * This is the drop-in boundary for the reference's smoothing path
 * (/root/reference/proj/include/dsmc/*.hpp). The reference is an in-process
 * C++ library with no C ABI; each entry point below names the reference
 * interface it replaces. All functions are `extern "C"`, take plain pointers
 * and sizes, never throw, and report failures through an error code plus a
 * per-context message (the reference's exception classes map 1:1 onto the
 * DSMC_E_* codes, see dsmc_status).
 *
 * Host pointers are accepted everywhere unless a parameter says "device";
 * the library owns every device allocation it makes.
 */
#ifndef DSMC_B200_H
#define DSMC_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define DSMC_API __attribute__((visibility("default")))
#else
#define DSMC_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------------
 * Status codes. Replaces the reference's exceptions:
 *   std::invalid_argument -> DSMC_E_INVALID_ARGUMENT (config, NaN, dead ref)
 *   std::runtime_error    -> DSMC_E_RUNTIME (degenerate leaf / table, trial
 *                            cap; the message names the cut like
 *                            smoother.cpp:196-201)
 *   std::domain_error     -> DSMC_E_DOMAIN (NaN entering a reduction,
 *                            kernels.cpp:34)
 *   std::logic_error      -> DSMC_E_LOGIC
 * ------------------------------------------------------------------------ */
typedef enum dsmc_status {
  DSMC_OK = 0,
  DSMC_E_INVALID_ARGUMENT = 1,
  DSMC_E_RUNTIME = 2,
  DSMC_E_DOMAIN = 3,
  DSMC_E_LOGIC = 4,
  DSMC_E_CUDA = 5,
  DSMC_E_NO_DEVICE = 6
} dsmc_status;

/* Resampler ids; same order as dsmc::Resampler (resampling.hpp:67). */
typedef enum dsmc_resampler {
  DSMC_MULTINOMIAL = 0,
  DSMC_SYSTEMATIC = 1,
  DSMC_MH_LAZY = 2,
  DSMC_REJECTION_LAZY = 3
} dsmc_resampler;

/* Stream roles; same values as dsmc::StreamRole (rng.hpp:16-24). */
typedef enum dsmc_stream_role {
  DSMC_ROLE_LEAF_PROPOSAL = 1,
  DSMC_ROLE_PAIR_RESAMPLE = 2,
  DSMC_ROLE_STAR_SELECT = 3,
  DSMC_ROLE_GIBBS_PARAM = 4,
  DSMC_ROLE_DATA_SIM = 5,
  DSMC_ROLE_FILTER_STEP = 6,
  DSMC_ROLE_BACKWARD_SAMPLE = 7
} dsmc_stream_role;

/* Arithmetic of the combine levels.
 *   FP64_PARITY: the reference's exact FP64 operation order (fill, exp_w
 *     polynomial, 8-lane sub-block sums, sequential prefixes; SURVEY
 *     Appendix A). With injected leaves, ancestor indices are bit-identical
 *     to the CPU reference.
 *   FP32: the throughput path (FP32 pair terms, MUFU exp2, log-domain
 *     sub-block sums); statistically equivalent, not bitwise. */
typedef enum dsmc_precision {
  DSMC_FP32 = 0,
  DSMC_FP64_PARITY = 1
} dsmc_precision;

/* ------------------------------------------------------------------------
 * Model descriptor. std::function callbacks cannot run on the device, so a
 * GPU-capable model is described by data. Replaces FeynmanKacModel
 * (fk_model.hpp:37-86) for the model families the device implements:
 *
 *  DSMC_MODEL_LGSSM  linear-Gaussian SSM, state dim d in 1..4, obs dim in
 *      1..4, with proposals q_t = nu_t = N(prop_mean_t, prop_cov_t) — the
 *      make_lgssm_fk construction (models.cpp:562-685), generalised to d<=4.
 *        x_0 ~ N(m0, P0); x_t = F_t x_{t-1} + b_t + N(0, Q_t);
 *        y_t = H_t x_t + N(0, R_t) when has_obs[t].
 *  DSMC_MODEL_SV     stochastic volatility, d = 1:
 *        x_0 ~ N(mu, s2/(1-phi^2)); x_t = mu + phi (x_{t-1}-mu) + N(0, s2);
 *        y_t ~ N(0, exp(x_t)).  Proposal q_t = nu_t = |y_t| h_t(x), sampled
 *        as x = log y_t^2 - log z^2, z ~ N(0,1); leaves t>=1 are uniform and
 *        log omega_c = log p(x_c|x_{c-1}) - log|y_c| <= -0.5 log(2 pi s2)
 *        - log|y_c| (the rejection bound). See DESIGN.md.
 *
 *  DSMC_MODEL_COX   log-Gaussian Cox counts over an AR(1) intensity, d = 1 —
 *      make_cox_model (models.hpp:29-50, models.cpp:111-216), par = (mu, rho,
 *      sigma2, lambda) as dsmc::CoxParams: slope a = rho lambda, intercept
 *      b = mu (1 - rho); x_t = b + a x_{t-1} + N(0, sigma2); y_t ~
 *      Poisson(exp x_t) (y = T+1 counts); q_t = nu_t = x_0 law = the
 *      stationary N(b / (1 - a), sigma2 / (1 - a^2)). No rejection bound.
 *  DSMC_MODEL_CRW   random walk conditioned to stay in [-1, 1], d = 1 —
 *      make_constrained_rw (models.cpp:263-338), par[0] = sigma: x_0 ~
 *      N(0, 1), x_t = x_{t-1} + N(0, sigma^2), potential 1{|x_t| <= 1},
 *      q_t = nu_t = U[-1, 1]; rejection bound -0.5 log(2 pi sigma^2) - log 1/2.
 *  DSMC_MODEL_THETA theta-logistic population dynamics, d = 1 —
 *      make_theta_logistic (models.cpp:407-491), par = (tau0, tau1, tau2, q2,
 *      r2): x_0 ~ N(0, 1), x_t = x_{t-1} + tau0 - tau1 exp(tau2 x_{t-1}) +
 *      N(0, q2), y_t ~ N(x_t, r2) (y = T+1 values); q_t = nu_t =
 *      N(prop_mean_t, prop_cov_t) (the caller's marginals, e.g. IEKS).
 *
 * Per-time arrays carry an element stride (in doubles) per time index; a
 * stride of 0 broadcasts one matrix to every time. Transition arrays are
 * indexed by t = 0..T with index 0 unused, exactly like
 * LinearGaussianModel (kalman.hpp:26-33).
 * ------------------------------------------------------------------------ */
typedef enum dsmc_model_kind {
  DSMC_MODEL_LGSSM = 1,
  DSMC_MODEL_SV = 2,
  DSMC_MODEL_COX = 3,
  DSMC_MODEL_CRW = 4,
  DSMC_MODEL_THETA = 5
} dsmc_model_kind;

typedef struct dsmc_model_desc {
  int kind;       /* dsmc_model_kind */
  int state_dim;  /* d */
  int obs_dim;    /* LGSSM observation dim (1..4); ignored for SV */
  int horizon;    /* T; times 0..T */

  /* LGSSM */
  const double* m0; /* d */
  const double* P0; /* d*d row-major */
  const double* F;  int64_t F_stride; /* d*d per time */
  const double* b;  int64_t b_stride; /* d per time */
  const double* Q;  int64_t Q_stride; /* d*d per time */
  const double* H;  int64_t H_stride; /* dy*d per time */
  const double* R;  int64_t R_stride; /* dy*dy per time */
  const double* y;                    /* (T+1)*dy (LGSSM) or T+1 (SV) */
  const uint8_t* has_obs;             /* T+1 flags; NULL = every time observed */
  const double* prop_mean;            /* (T+1)*d */
  const double* prop_cov;             /* (T+1)*d*d */

  /* SV */
  double sv_mu, sv_phi, sv_sigma2;

  /* COX / CRW / THETA parameters (see dsmc_model_kind) */
  double par[8];
} dsmc_model_desc;

/* Options of one smoothing run. Replaces SmootherOptions (smoother.hpp:50-56)
 * plus the parity hooks. */
typedef struct dsmc_smooth_opts {
  size_t n_particles;   /* N */
  int resampler;        /* dsmc_resampler */
  size_t mh_steps;      /* MH chain length (mh-lazy only), default 16 */
  uint64_t seed;
  int precision;        /* dsmc_precision */
  /* Optional injected leaves (parity tests): (T+1)*N*d states and (T+1)*N
   * raw (un-normalised) leaf log-weights, host memory. The leaf kernel is
   * skipped when set; weights_uniform / LSE follow make_leaf
   * (smoother.cpp:117-128) on the injected values. */
  const double* inject_states;
  const double* inject_logw;
} dsmc_smooth_opts;

/* Outputs. Every pointer is optional (NULL = not wanted); host memory. */
typedef struct dsmc_smooth_out {
  double* paths;            /* (T+1)*N*d root paths, time-major (BlockEstimate
                               layout, smoother.hpp:28-48) */
  double* mean;             /* (T+1)*d smoothed means (uniform root weights) */
  double* cov;              /* (T+1)*d*d smoothed covariances */
  uint32_t* pair_left;      /* T*N: per combine in schedule order, left idx */
  uint32_t* pair_right;     /* T*N: right idx */
  double* log_mean_weight;  /* T: per-combine log mean pair weight (dense) */
  double* leaf_states;      /* (T+1)*N*d leaf states as generated (FP64
                               parity only; DSMC_E_INVALID_ARGUMENT under FP32) */
  double* leaf_logw;        /* (T+1)*N normalised leaf log-weights, each
                               leaf's BlockEstimate::log_w (smoother.cpp:117-128);
                               FP64 parity only */
  /* RunMetadata (smoother.hpp:58-68) */
  double log_norm_const;
  int has_log_norm_const;
  int levels;
  uint64_t weight_evals;
  int biased;
  double wall_time_ms;
} dsmc_smooth_out;

/* ------------------------------------------------------------------------ */
typedef struct dsmc_ctx dsmc_ctx;

/* Create a context bound to one CUDA device. */
DSMC_API int dsmc_create(int device, dsmc_ctx** out);
DSMC_API void dsmc_destroy(dsmc_ctx* ctx);
/* Message of the last failure on this context ("" if none). */
DSMC_API const char* dsmc_last_error(const dsmc_ctx* ctx);
/* Number of kernels this context has launched since creation. */
DSMC_API uint64_t dsmc_kernel_launches(const dsmc_ctx* ctx);

/* Full dSMC smoothing run. Replaces
 *   run_smoother(const FeynmanKacModel&, const SmootherOptions&) -> RunResult
 * (smoother.hpp:128-129, smoother.cpp:226-277). */
DSMC_API int dsmc_smooth(dsmc_ctx* ctx, const dsmc_model_desc* model,
                const dsmc_smooth_opts* opts, dsmc_smooth_out* out);

/* Device-resident variant for throughput measurement: the model is uploaded
 * and prepared once (dsmc_model_upload), the run writes moments into
 * device buffers owned by the context, and nothing crosses PCIe.
 * dsmc_smooth_resident returns after enqueueing; dsmc_sync waits. */
typedef struct dsmc_model_handle dsmc_model_handle;
DSMC_API int dsmc_model_upload(dsmc_ctx* ctx, const dsmc_model_desc* model,
                      dsmc_model_handle** out);
DSMC_API void dsmc_model_free(dsmc_ctx* ctx, dsmc_model_handle* h);
DSMC_API int dsmc_smooth_resident(dsmc_ctx* ctx, const dsmc_model_handle* h,
                         const dsmc_smooth_opts* opts);
/* Copy the last resident run's results to the host (NULL = skip). */
DSMC_API int dsmc_resident_results(dsmc_ctx* ctx, double* mean, double* cov,
                          double* log_norm_const, int* has_log_norm_const);
DSMC_API int dsmc_sync(dsmc_ctx* ctx);
/* CUDA stream the context launches on (cudaStream_t as void*). */
DSMC_API void* dsmc_stream(dsmc_ctx* ctx);
/* Per-kernel-class device time (ms) of the last resident run, measured with
 * CUDA events on the launching stream: [0] leaves, [1] pair/combine levels,
 * [2] top-down composition + gather/moments. Returns the number filled. */
DSMC_API int dsmc_last_timings(const dsmc_ctx* ctx, double* ms, int cap);

/* ------------------------------------------------------------------------
 * Pair resampling over an explicit log-weight table (device FP64 parity
 * path). Replaces resample_pairs(Resampler, const PairWeightSource&, n_out,
 * mh_steps, const StreamKey&) (resampling.hpp:85-87) for a table-backed
 * source (fill_row = row copy, log_weight_at = entry, as the reference's
 * test_resampling.cpp:17-33 builds it).
 * has_bound/bound: PairWeightSource::log_upper_bound.
 * lmw/has_lmw: PairSample::log_mean_weight. ------------------------------ */
DSMC_API int dsmc_resample_table(dsmc_ctx* ctx, int resampler, const double* logw,
                        size_t n, size_t n_out, size_t mh_steps, int has_bound,
                        double bound, uint64_t seed, uint32_t level,
                        uint64_t node, uint32_t* left, uint32_t* right,
                        double* lmw, int* has_lmw, uint64_t* weight_evals,
                        int* biased);

/* Device Philox4x64-10 (rng.cpp:27-41): out[4*i..4*i+3] = block(ctr_i, key)
 * with ctr_i = {ctr[0]+i, ctr[1], ctr[2], ctr[3]}. */
DSMC_API int dsmc_philox_blocks(dsmc_ctx* ctx, const uint64_t ctr[4],
                       const uint64_t key[2], size_t n_blocks, uint64_t* out);

/* Device exp_w (exp_poly.hpp:39-51), elementwise. */
DSMC_API int dsmc_exp_w(dsmc_ctx* ctx, const double* x, size_t n, double* out);

/* ------------------------------------------------------------------------
 * The reference's piecewise smoother API on the device (FP64, the
 * reference's operation order), for callers that stitch blocks themselves.
 *
 * dsmc_make_leaf replaces make_leaf(model, t, n, seed) (smoother.hpp:101-102,
 * smoother.cpp:98-130): n proposal draws from stream {seed, 0, t,
 * leaf_proposal} (states n*d), the normalised log weights (n), the
 * weights_uniform flag and the leaf's log normalising constant.
 *
 * dsmc_resample_blocks replaces resample_pairs(r, make_pair_source(model, L,
 * R).source, n_out, mh_steps, key) (resampling.hpp:85-87, smoother.hpp:
 * 109-116, smoother.cpp:132-180) for two adjacent blocks: the caller passes
 * L's terminal slab, R's initial slab and the blocks' normalised log weights
 * (NULL or *_uniform = 1 for a uniform block, whose weights stay out of the
 * table); the table logw[i][j] = log omega_cut(xL_i, xR_j) + lwL_i + lwR_j is
 * evaluated on the device (never materialised for the lazy samplers) and
 * sampled with key {seed, level, node, pair_resample}. n_out <= n.
 * log_mean_weight excludes the uniform sides' log_shift, as the reference. */
typedef struct dsmc_pair_blocks {
  int cut;                    /* R.a = L.b + 1, 1..T */
  size_t n;                   /* particles per block */
  const double* left_states;  /* n*d: L's slab at time cut - 1 */
  const double* left_logw;    /* n normalised, or NULL (uniform) */
  int left_uniform;
  const double* right_states; /* n*d: R's slab at time cut */
  const double* right_logw;
  int right_uniform;
} dsmc_pair_blocks;

DSMC_API int dsmc_make_leaf(dsmc_ctx* ctx, const dsmc_model_desc* model, int t, size_t n,
                            uint64_t seed, double* states, double* logw,
                            int* weights_uniform, double* log_norm_const);
DSMC_API int dsmc_resample_blocks(dsmc_ctx* ctx, const dsmc_model_desc* model,
                                  const dsmc_pair_blocks* blocks, int resampler,
                                  size_t n_out, size_t mh_steps, uint64_t seed,
                                  uint32_t level, uint64_t node, uint32_t* left,
                                  uint32_t* right, double* lmw, int* has_lmw,
                                  uint64_t* weight_evals, int* biased);

/* Single-population resampling: multinomial_indices / systematic_indices
 * (resampling.hpp:69-80, resampling.cpp:360-460) of n_out draws from the
 * categorical of n unnormalised log weights, stream {seed, level, node,
 * role}. Returns the indices plus max_i logw and the exp_row_store total
 * sum_i exp_w(logw_i - max), so log_mean_weight = max + log(total) - log n
 * (taken on the host with the C library's log). DSMC_E_RUNTIME when every
 * weight is zero, DSMC_E_DOMAIN on NaN. */
DSMC_API int dsmc_resample_indices(dsmc_ctx* ctx, int resampler, const double* logw, size_t n,
                                   size_t n_out, uint64_t seed, uint32_t level, uint64_t node,
                                   int role, uint32_t* idx, double* max_logw, double* total);

/* Lazy pair resampling over a source only the caller can evaluate (host
 * callbacks: PairWeightSource::log_weight_at): mh_lazy_pairs /
 * rejection_lazy_pairs (resampling.hpp:56-65, resampling.cpp:233-324) with
 * key {seed, level, node, pair_resample}. The device holds every slot's
 * chain state and counter-addressed stream position; each round it emits the
 * entries (i, j) its pending slots probe next, the caller evaluates them and
 * answers with their log weights, until no probe is left:
 *   dsmc_lazy_begin(...)               -> n_probes
 *   while (n_probes) { dsmc_lazy_probes(i, j); evaluate;
 *                      dsmc_lazy_answer(values) -> n_probes }
 *   dsmc_lazy_finish(left, right, evals)
 * The probes and their order of evaluation per slot are the reference's, so
 * weight_evals matches its count. One sampling in flight per context. */
DSMC_API int dsmc_lazy_begin(dsmc_ctx* ctx, int resampler, size_t n, size_t n_out,
                             size_t mh_steps, int has_bound, double bound, uint64_t seed,
                             uint32_t level, uint64_t node, size_t* n_probes);
DSMC_API int dsmc_lazy_probes(dsmc_ctx* ctx, uint32_t* i, uint32_t* j);
DSMC_API int dsmc_lazy_answer(dsmc_ctx* ctx, const double* values, size_t* n_probes);
DSMC_API int dsmc_lazy_finish(dsmc_ctx* ctx, uint32_t* left, uint32_t* right,
                              uint64_t* weight_evals);

/* ------------------------------------------------------------------------
 * Conditional dSMC / particle Gibbs, batched over independent chains.
 * Replaces run_conditional(model, ref, ConditionalOptions, sweep)
 * (conditional.hpp:48-51) run for n_chains chains at once: chain c uses
 * models[c], reference path refs[c*(T+1)*d ...], seed seeds[c].
 * Only multinomial / rejection-lazy are allowed (conditional.cpp:27-32).
 * out_paths: n_chains*(T+1)*d; changed: n_chains*(T+1) (path_changed_times);
 * log_norm_const: n_chains (NaN when unavailable). ---------------------- */
typedef struct dsmc_cond_opts {
  size_t n_particles;
  int resampler;
  int precision;
  const double* inject_states; /* optional, n_chains*(T+1)*N*d (slot 0 is
                                  overwritten by the reference) */
  const double* inject_logw;   /* optional, n_chains*(T+1)*N */
} dsmc_cond_opts;

DSMC_API int dsmc_conditional_sweep(dsmc_ctx* ctx, const dsmc_model_desc* models,
                           int n_chains, const double* refs,
                           const uint64_t* seeds, const dsmc_cond_opts* opts,
                           uint32_t sweep, double* out_paths, uint8_t* changed,
                           double* log_norm_const, uint64_t* weight_evals);

/* One batched particle-Gibbs sweep for the stochastic-volatility model:
 * parameter update (conjugate Normal mu, inverse-gamma sigma2, RWM on phi;
 * stream {seed_c, 0, sweep, gibbs_param}) followed by one conditional dSMC
 * path update per chain. Mirrors pgibbs_sweep (pgibbs.hpp:55-59,
 * pgibbs.cpp:24-55) with the SV ParamKernel of DESIGN.md.
 * theta: n_chains*3 (mu, phi, sigma2), updated in place; stars:
 * n_chains*(T+1), updated in place; ys: T+1 shared observations. */
typedef struct dsmc_sv_prior {
  double mu_mean, mu_var;        /* mu ~ N(mu_mean, mu_var) */
  double s2_shape, s2_rate;      /* 1/sigma2 ~ Gamma(shape, rate) */
  double phi_step;               /* RWM step on phi (|phi| < 1, flat prior) */
} dsmc_sv_prior;

DSMC_API int dsmc_sv_pgibbs_sweep(dsmc_ctx* ctx, int n_chains, int horizon,
                         const double* ys, const dsmc_sv_prior* prior,
                         double* theta, double* stars, const uint64_t* seeds,
                         size_t n_particles, int resampler, uint32_t sweep,
                         uint8_t* changed, uint64_t* accepted_phi);

/* ------------------------------------------------------------------------
 * Time-sharded smoothing (multi-GPU). The reference has no
 * distribution; these stages let one process per GPU run contiguous time
 * windows with the reference's GLOBAL stream keys, so a P-GPU run
 * reproduces the 1-GPU run bit for bit. The host protocol
 * (paper_2202_02264_b200/sharded.py) exchanges only boundary slabs, block
 * log Z and ancestor indices over NCCL for the top log2(P) levels.
 *
 * Every stage only enqueues work on the context's stream (no host
 * synchronisation); log Z values and indices stay in device memory, and
 * device errors raised by any stage surface at the next dsmc_sync.
 *
 *   dsmc_model_upload_window  upload + prepare only the times a window
 *                         [t0, t0+len) and its right cross cut t0+len need
 *   dsmc_window_run       leaves [t0, t0+len) + the len-local combine levels
 *   dsmc_window_boundary  slab of the window root's first (side 0: states +
 *                         column terms) or last (side 1) leaf, and the root's
 *                         log Z (d_root_lnc, one double), device out
 *   dsmc_cross_combine    one cross-window combine at cut `cut`, global
 *                         (level, node) stream key, on gathered slabs; any
 *                         resampler (dense, MH-lazy, rejection-lazy); block
 *                         log Z in / out as device doubles (NaN after lazy)
 *   dsmc_window_remap     root first (side 0) / last (side 1) map := map[idx]
 *   dsmc_window_finish    top-down composition from the window root's map
 *                         (device, NULL = identity) + per-time moments */
typedef struct dsmc_window_opts {
  size_t n_particles;
  int resampler;
  size_t mh_steps;
  uint64_t seed;
  int t0;          /* first leaf; a multiple of len */
  int len;         /* leaves in the window; a power of two >= 2 */
} dsmc_window_opts;

DSMC_API int dsmc_model_upload_window(dsmc_ctx* ctx, const dsmc_model_desc* model, int t0,
                                      int len, dsmc_model_handle** out);
DSMC_API int dsmc_window_run(dsmc_ctx* ctx, const dsmc_model_handle* h,
                             const dsmc_window_opts* opts);
DSMC_API int dsmc_window_boundary(dsmc_ctx* ctx, int side, void* d_states,
                                  float* d_col, double* d_root_log_norm_const);
DSMC_API int dsmc_cross_combine(dsmc_ctx* ctx, const dsmc_model_handle* h,
                                const dsmc_window_opts* opts, int cut, int level,
                                long long node, const void* d_left_states,
                                const void* d_right_states, const float* d_right_col,
                                const double* d_lnc_left, const double* d_lnc_right,
                                uint32_t* d_left_idx, uint32_t* d_right_idx,
                                double* d_lnc_out);
DSMC_API int dsmc_window_remap(dsmc_ctx* ctx, int side, const uint32_t* d_idx);
DSMC_API int dsmc_window_finish(dsmc_ctx* ctx, const uint32_t* d_root_map,
                                double* d_mean, double* d_cov);

/* ------------------------------------------------------------------------
 * Sequential comparator: particle filter with resampling
 * at every step + forward-filtering backward-sampling of n_draws joint paths.
 * Replaces run_particle_filter (baselines.hpp:42-49, baselines.cpp:36-98)
 * followed by ffbs_sample (baselines.hpp:62-63, baselines.cpp:100-160), with
 * the same stream keys ({seed, 0|1, t, filter_step}, {seed, 0|1, t,
 * backward_sample} substream m+1); FP32 arithmetic. Outputs: per-time mean /
 * cov of the draws ((T+1)*d, (T+1)*d*d), optional draws (n_draws*(T+1)*d,
 * draw-major as FfbsResult::paths) and the filter's log-likelihood estimate.
 * ------------------------------------------------------------------------ */
typedef struct dsmc_ffbs_opts {
  size_t n_particles;
  size_t n_draws;
  int resampler;  /* multinomial or systematic */
  uint64_t seed;
} dsmc_ffbs_opts;

DSMC_API int dsmc_ffbs_smooth(dsmc_ctx* ctx, const dsmc_model_desc* model,
                              const dsmc_ffbs_opts* opts, double* mean, double* cov,
                              double* paths, double* log_likelihood);

/* ------------------------------------------------------------------------
 * Proposal construction (host, FP64, the step before the
 * leaves): exact Kalman filter + RTS smoother of a DSMC_MODEL_LGSSM
 * descriptor (prop_mean / prop_cov are ignored). Restates kalman_smooth
 * (kalman.cpp:78-138): Joseph-form update, RTS gain solved against the
 * predicted covariance, symmetrisation after every step, jitter-escalating
 * Cholesky (kalman.cpp:15-26). Outputs (T+1)*d means, (T+1)*d*d
 * covariances and the marginal log-likelihood. --------------------------- */
DSMC_API int dsmc_kalman_smooth(const dsmc_model_desc* model,
                                double* smooth_mean, double* smooth_cov,
                                double* log_likelihood);

/* The same smoother on the device by parallel prefix scans (Sarkka &
 * Garcia-Fernandez 2021: associative filtering and smoothing elements,
 * O(log T) span instead of the reference's length-T chain; FP64;
 * csrc/kalman_scan.cuh). Equal to dsmc_kalman_smooth to rounding
 * (tests/test_gpu_kalman.py: 1e-9 relative). Host outputs. */
DSMC_API int dsmc_kalman_smooth_device(dsmc_ctx* ctx, const dsmc_model_desc* model,
                                       double* smooth_mean, double* smooth_cov,
                                       double* log_likelihood);

#ifdef __cplusplus
}
#endif

#endif /* DSMC_B200_H */

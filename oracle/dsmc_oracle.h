/*
 * ORACLE / TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C CPU restatement of the reference's dSMC smoothing path, used only
 * by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * checker. It implements the same contract as the product's C ABI
 * (include/dsmc_b200.h) with an `or_` prefix so tests call both identically.
 * Each function cites the reference file:line it restates. Parity of this
 * restatement is pinned against the compiled reference (oracle/_ref) and the
 * committed golden vectors in tests/golden/.
 */
#ifndef DSMC_ORACLE_H
#define DSMC_ORACLE_H

#include "dsmc_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* or_last_error(void);

/* rng.cpp:27-41 */
void or_philox(const uint64_t ctr[4], const uint64_t key[2], uint64_t out[4]);
/* rng.cpp:45-93; kind 0 u64, 1 uniform, 2 uniform_pos, 3 normal */
void or_stream(uint64_t seed, uint32_t level, uint64_t node, int role,
               uint64_t substream, int kind, size_t n, void* out);

/* exp_poly.hpp:39-51 and kernels.cpp scalar backend */
double or_exp_w(double x);
double or_reduce_sum(const double* x, size_t n);
double or_log_sum_exp(const double* x, size_t n);
double or_exp_row_store(const double* logw, size_t n, double shift, double* w,
                        double* sub);

/* resampling.cpp:181-324 on a table source (same contract as
 * dsmc_resample_table). */
int or_resample_table(int resampler, const double* logw, size_t n,
                      size_t n_out, size_t mh_steps, int has_bound,
                      double bound, uint64_t seed, uint32_t level,
                      uint64_t node, uint32_t* left, uint32_t* right,
                      double* lmw, int* has_lmw, uint64_t* weight_evals,
                      int* biased);

/* smoother.cpp:64-85: 5 ints per pair (level, node, left_a, left_b,
 * right_b); returns the number of levels. */
int or_build_schedule(int horizon, int* pairs);

/* run_smoother (smoother.cpp:226-277) via ancestor-index composition
 * — same contract as dsmc_smooth. n_threads ignored. */
int or_smooth(const dsmc_model_desc* model, const dsmc_smooth_opts* opts,
              dsmc_smooth_out* out);

/* run_conditional (conditional.cpp:156-216) — one chain. */
int or_conditional(const dsmc_model_desc* model, const double* ref,
                   size_t n_particles, int resampler, uint64_t seed,
                   uint32_t sweep, const double* inject_states,
                   const double* inject_logw, double* out_path,
                   double* log_norm_const, int* has_lnc,
                   uint64_t* weight_evals);

/* SV particle-Gibbs parameter kernel: updates theta[3] =
 * (mu, phi, sigma2) from the path; stream {seed, 0, sweep, gibbs_param}. */
int or_sv_param_update(const double* path, int horizon,
                       const dsmc_sv_prior* prior, uint64_t seed,
                       uint32_t sweep, double* theta, int* accepted_phi);

/* gamma_draw (pgibbs.cpp:80-102) from stream {seed, level, node, role}. */
double or_gamma_draw(double shape, double rate, uint64_t seed, uint32_t level,
                     uint64_t node, int role);

/* kalman_smooth (kalman.cpp:78-138) of an LGSSM descriptor (d, dy <= 8):
 * smoothed means (T+1)*d, covariances (T+1)*d*d, marginal log-likelihood. */
int or_kalman_smooth(const dsmc_model_desc* model, double* smooth_mean,
                     double* smooth_cov, double* log_likelihood);

#ifdef __cplusplus
}
#endif
#endif

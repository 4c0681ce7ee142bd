// Internal declarations of the B200 dSMC engine (not part of the C ABI).
//
// HBM layout of one run (K = T+1 leaves, N particles, d <= 4, B chains):
//   TimeConst   tc[B][K]          per-time FP64 constants (prep kernel)
//   FP64 path:  X64[B][K][N][d]   leaf states;  LW64[B][K][N] normalised
//   FP32 path:  X32[B][K][N]      centred leaf states x - m_t as float4
//               COL[B][K][N]      column term log h_t - log nu_t (+consts),
//                                 float, log2 units
//               LW32[B][N]        leaf-0 normalised weights (log2 units)
//   leaf meta   LNC[B][K] (double), UNI[B][K] (uniform flag)
//   maps        FIRST/LAST[B][nb(l)][N] uint32, ping-pong across levels
//   pairs       PL/PR[B][T][N] uint32 in schedule order (kept for the
//               top-down composition; the reference keeps full path copies)
//   block lnc   BLNC[B][nb(l)] double, ping-pong
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "common.cuh"
#include "dsmc_b200.h"

namespace dsmc_dev {

constexpr double kLog2Pi = 1.8378770664093454836;
constexpr double kLog2E = 1.4426950408889634074;
constexpr double kLn2 = 0.69314718055994530942;

struct TimeConst {
  double pm[4];     // proposal mean m_t
  double pL[16];    // lower Cholesky of the proposal covariance
  double pW[16];    // its inverse (whitening)
  double p_norm;    // -0.5 (d log 2pi + log det P_t)
  double tW[16];    // inverse Cholesky of Q_t (t >= 1)
  double t_norm;    // -0.5 (d log 2pi + log det Q_t)
  double F[16];     // F_t (t >= 1)
  double oW[16];    // inverse Cholesky of R_t (observed times)
  double o_norm;    // -0.5 (dy log 2pi + log det R_t)
  double delta[4];  // F_t m_{t-1} + b_t - m_t (centring offset, t >= 1)
  double e[4];      // W_R (y_t - H_t m_t)
  double G[16];     // W_R H_t L_t (dy x d)
  double cconst;    // o_norm - p_norm + t_norm (column-term constant)
  double shift1;    // d = 1 LGSSM column shift (models.cpp:614-624); SV base
  double bound;     // log stitch bound at cut t (NaN if none)
  double logabsy;   // SV: log|y_t|
  int obs;          // has_obs[t]
  int bounded;      // bound is finite
  int drift;        // THETA: nonlinear row mean (FP32 path)
  double th[4];     // THETA: tau0, tau1, tau2, proposal mean at t - 1
};

// Device view of a model (pointers are device memory).
struct DevModel {
  int kind, d, dy, T, K;
  const double* y;
  const uint8_t* has_obs;
  const double *prop_mean, *prop_cov, *F, *b, *Q, *H, *R, *m0, *P0;
  int64_t F_s, b_s, Q_s, H_s, R_s;
  double sv_mu, sv_phi, sv_s2;
  // COX: {slope a, intercept b, stat mean, stat var, trans_norm, sigma2,
  //       stat sd, -}; CRW: {var, trans_norm, sigma, -, ...}; THETA: {tau0,
  //       tau1, tau2, q2, r2, trans_norm, obs_norm, -}. Host-computed
  // (glibc log / lgamma) so the parity path shares the reference's constants.
  double mp[8];
  const double* lgam;   // COX: lgamma(y_t + 1), [K]
  const TimeConst* tc;  // [K]
};

// Per-chain view for batched kernels (chain c at tc + c*K etc.).
struct RunDims {
  int K, T, N, d, B;  // leaves, cuts, particles, state dim, chains
  int precision;
  int resampler;
  int conditional;    // c-dSMC: slot 0 pinned
  uint32_t sweep;
  size_t mh_steps;
};

void set_error(std::string msg);

}  // namespace dsmc_dev

// Leaf kernels (make_leaf, smoother.cpp:98-130; conditional_leaf,
// conditional.cpp:52-87). One thread per (particle, time, chain).
#pragma once

#include <math_constants.h>

#include "kernels64.cuh"

namespace dsmc_dev {

// Wide-state FP32 path (5 <= d <= 32, wide.cuh): per-time constants prepared
// on the host in FP64 and stored as FP32, indexed by GLOBAL time; D = padded
// dimension (8, 16, 32), DYP = padded observation dimension.
struct WideBufs {
  int d, dy, DP, DYP;
  const float* L;    // [Kt][DP*DP] lower Cholesky of the proposal covariance
  const float* G;    // [Kt][DYP*DP] R^-1/2 H L
  const float* e;    // [Kt][DYP] R^-1/2 (y - H m)
  const float* c;    // [Kt] o_norm - p_norm + t_norm (t = 0: no t_norm)
  const float* W;    // [Kt][DP*DP] s W_Q (cut t >= 1; s = sqrt(log2e / 2))
  const float* M;    // [Kt][DP*DP] s W_Q F
  const float* v;    // [Kt][DP] s W_Q (F m_{t-1} + b - m_t)
  const double* m;   // [Kt][d] proposal means (un-centring)
  const float* WP0;  // [DP*DP] inverse Cholesky of P0
  const float* dm0;  // [DP] m0 - m_0
  double p0norm;     // -0.5 (d log 2 pi + log det P0)
  float* X;          // [B][K][N][DP] centred leaf states (run buffer)
};

struct Bufs {
  int K, T, N, d, B, cap;  // cap: map capacity (blocks) per chain
  int t0;  // global time of local leaf 0 (time-sharded windows; 0 otherwise)
  int Kt;  // leaves of the whole model (TimeConst stride per chain)
  const DevModel* models;  // [B]
  const uint64_t* seeds;   // [B]
  const TimeConst* tc;     // [B][K]
  const int* bounded;      // [B] bit0: every cut has a finite bound
  // FP64 path
  double* X64;   // [B][K][N][d]
  double* LW64;  // [B][K][N] normalised
  // FP32 path
  float4* X32;   // [B][K][N] centred states
  float* COL;    // [B][K][N] column terms (log2 units)
  float* LW32;   // [B][N] leaf-0 normalised weights (log2 units)
  // leaf meta
  double* LNC;   // [B][K]
  uint8_t* UNI;  // [B][K]
  double* LWMAX; // [B][K] max normalised leaf log weight (rejection bound)
  // pairs
  uint32_t* PL;  // [B][T][N]
  uint32_t* PR;
  double* LMW;   // [B][T]
  ErrFlag* err;
  unsigned long long* evals;  // [B]
  int conditional;
  uint32_t sweep;
  const double* star;  // [B][K][d] (conditional)
  int leaf_role;       // FP32 leaf stream role (0 = leaf_proposal; the particle
                       // filter draws with filter_step, baselines.cpp:17-20)
  WideBufs w;          // wide-state path (d > 4)
};

// Normal number i of a leaf stream (rng.cpp:74-86 via counter addressing:
// normal i consumes u64s 2*(i/2) (uniform_pos) and 2*(i/2)+1 (uniform);
// even i -> r cos(theta), odd i -> r sin(theta)).
__device__ inline double leaf_normal64(const StreamId& id, uint64_t i) {
  const uint64_t q = 2 * (i >> 1);
  const U64x4 blk = stream_block(id, q >> 2);
  const double u1 = u64_uniform_pos(pick4(blk, (uint32_t)(q & 3)));
  const double u2 = u64_uniform(pick4(blk, (uint32_t)(q & 3) + 1));
  const double r = sqrt(DMUL(-2.0, log(u1)));
  const double th = DMUL(2.0 * 3.14159265358979323846, u2);
  return (i & 1) ? DMUL(r, sin(th)) : DMUL(r, cos(th));
}

__device__ inline uint64_t leaf_node(int t, int conditional, uint32_t sweep) {
  return conditional ? (static_cast<uint64_t>(static_cast<uint32_t>(t)) |
                        (static_cast<uint64_t>(sweep) << 32))
                     : static_cast<uint64_t>(t);
}

// FP64 leaf: states and RAW log weights (log_init_weight, fk_model.cpp:43-59).
__global__ void leaf64_kernel(Bufs b, const double* inj_x, const double* inj_lw) {
  // grid (time, particle chunk, chain): time in x (up to 2^31 leaves)
  const int n = blockIdx.y * blockDim.x + threadIdx.x;
  const int lt = blockIdx.x, ch = blockIdx.z;
  const int t = b.t0 + lt;  // global time (stream key, model data); lt indexes the window
  if (n >= b.N) return;
  const DevModel& M = b.models[ch];
  const TimeConst& tc = b.tc[(size_t)ch * b.Kt + t];
  const int d = b.d;
  double x[4] = {0, 0, 0, 0};
  const size_t off = ((size_t)ch * b.K + lt) * b.N + n;
  if (b.conditional && n == 0) {
    for (int k = 0; k < d; ++k) x[k] = b.star[((size_t)ch * b.K + lt) * d + k];
  } else if (inj_x) {
    for (int k = 0; k < d; ++k) x[k] = inj_x[off * d + k];
  } else {
    const StreamId id = stream_id(b.seeds[ch], 0, leaf_node(t, b.conditional, b.sweep),
                                  DSMC_ROLE_LEAF_PROPOSAL, 0);
    const uint64_t p = b.conditional ? n - 1 : n;
    double z[4];
    if (M.kind == DSMC_MODEL_CRW) {
      // fill_uniform (rng.cpp:95-97): element p is u64 number p; x = 2u - 1
      x[0] = DSUB(DMUL(2.0, u64_uniform(stream_u64(id, p))), 1.0);
    } else {
      for (int k = 0; k < d; ++k) z[k] = leaf_normal64(id, p * d + k);
    }
    if (M.kind == DSMC_MODEL_CRW) {
    } else if (M.kind == DSMC_MODEL_COX) {  // models.cpp:143-148
      x[0] = DADD(M.mp[2], DMUL(M.mp[6], z[0]));
    } else if (M.kind == DSMC_MODEL_SV) {
      x[0] = DSUB(DMUL(2.0, tc.logabsy), log(DMUL(z[0], z[0])));
    } else if (M.kind == DSMC_MODEL_THETA || (d == 1 && M.dy == 1)) {
      const double sd = sqrt(M.prop_cov[t]);
      x[0] = DADD(M.prop_mean[t], DMUL(sd, z[0]));
    } else {
      for (int k = 0; k < d; ++k) {
        double acc = 0.0;
        for (int l = 0; l <= k; ++l) acc = DADD(acc, DMUL(tc.pL[k * d + l], z[l]));
        x[k] = DADD(tc.pm[k], acc);
      }
    }
  }
  for (int k = 0; k < d; ++k) b.X64[off * d + k] = x[k];
  double w;
  if (inj_lw && !b.conditional) {
    w = inj_lw[off];
  } else if (M.kind == DSMC_MODEL_COX) {  // init_weight_batch, models.cpp:169-177
    w = t == 0 ? cox_log_poisson(M, 0, x[0]) : 0.0;
  } else if (M.kind == DSMC_MODEL_CRW) {  // init_weight_batch, models.cpp:301-311
    const double norm = DSUB(DMUL(-0.5, kLog2Pi), kLogHalf);
    w = !crw_in_box(x[0]) ? -CUDART_INF
        : t == 0          ? DSUB(norm, DMUL(DMUL(0.5, x[0]), x[0]))
                          : 0.0;
  } else if (t == 0) {
    double W0[16], norm0 = 0.0;
    if (M.kind == DSMC_MODEL_LGSSM && !(d == 1 && M.dy == 1)) {
      double L0[16];
      dchol(M.P0, d, L0);
      dtri_inv(L0, d, W0);
      norm0 = dnorm_of(L0, d);
    }
    const double pot = cb_log_h(M, tc, 0, x);
    const double p0 = cb_init_logdensity(M, tc, x, W0, norm0);
    const double q = cb_prop_logdensity(M, tc, 0, x);
    w = DSUB(DADD(pot, p0), q);
    if (pot == -CUDART_INF || p0 == -CUDART_INF) w = -CUDART_INF;
  } else {
    const double nu = cb_prop_logdensity(M, tc, t, x);
    const double q = nu;  // aux == proposal for every device model
    w = nu == -CUDART_INF ? -CUDART_INF : DSUB(nu, q);
  }
  if (isnan(w)) raise_err(b.err, DSMC_E_INVALID_ARGUMENT, t, 0, kReasonNaN);
  b.LW64[off] = w;
}

// Leaf normalisation (smoother.cpp:117-128): one warp per (time, chain).
// LSE with the 8-lane contract (kernels.cpp:46-55), weights_uniform iff
// min == max, log_norm_const = lse - log N.
__global__ void leafnorm64_kernel(Bufs b) {
  const int t = blockIdx.x, ch = blockIdx.y, lane = threadIdx.x;
  const int N = b.N;
  double* lw = b.LW64 + ((size_t)ch * b.K + t) * N;
  double mx = -CUDART_INF, lo = CUDART_INF, hi = -CUDART_INF;
  int nan = 0;
  for (int i = lane; i < N; i += 32) {
    const double v = lw[i];
    nan |= isnan(v);
    if (v > mx) mx = v;
    lo = fmin(lo, v);
    hi = fmax(hi, v);
  }
  for (int o = 16; o; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(~0u, mx, o));
    lo = fmin(lo, __shfl_xor_sync(~0u, lo, o));
    hi = fmax(hi, __shfl_xor_sync(~0u, hi, o));
    nan |= __shfl_xor_sync(~0u, nan, o);
  }
  if (nan) {
    if (lane == 0) raise_err(b.err, DSMC_E_DOMAIN, t, 0, kReasonNaN);
    return;
  }
  if (b.conditional && lw[0] == -CUDART_INF) {
    if (lane == 0) raise_err(b.err, DSMC_E_INVALID_ARGUMENT, t, 0, kReasonRefLeaf);
    return;
  }
  if (mx == -CUDART_INF) {
    if (lane == 0) raise_err(b.err, DSMC_E_RUNTIME, t, 0, kReasonLeafZero);
    return;
  }
  const int n8 = N & ~7;
  double acc = 0.0;
  if (lane < 8)
    for (int i = lane; i < n8; i += 8) acc = DADD(acc, exp_w(DSUB(lw[i], mx)));
  double a8[8];
  for (int l = 0; l < 8; ++l) a8[l] = __shfl_sync(~0u, acc, l);
  double lse = 0.0;
  if (lane == 0) {
    double tot = combine8(a8);
    for (int i = n8; i < N; ++i) tot = DADD(tot, exp_w(DSUB(lw[i], mx)));
    lse = DADD(mx, log(tot));
  }
  lse = __shfl_sync(~0u, lse, 0);
  const double nl = -lse;
  __syncwarp();
  for (int i = lane; i < N; i += 32) lw[i] = DADD(lw[i], nl);
  if (lane == 0) {
    const size_t o = (size_t)ch * b.K + t;
    b.LNC[o] = DSUB(lse, log((double)N));
    b.UNI[o] = lo == hi;
    b.LWMAX[o] = DADD(mx, nl);
  }
}

// Leaf-0 raw weight h0 + P0 - q0 in FP64 (only the CTAs of global time 0;
// kept out of line so its local arrays stay off the hot path).
__device__ __noinline__ double leaf0_raw_weight(const DevModel& M, const TimeConst& tc, int d,
                                                const double* x) {
  if (M.kind == DSMC_MODEL_COX) return cox_log_poisson(M, 0, x[0]);
  if (M.kind == DSMC_MODEL_THETA)
    return dlog_normal_pdf(M.y[0], x[0], M.mp[4]) + dlog_normal_pdf(x[0], 0.0, 1.0) -
           dlog_normal_pdf(x[0], M.prop_mean[0], M.prop_cov[0]);
  if (M.kind == DSMC_MODEL_CRW) {
    const double norm = DSUB(DMUL(-0.5, kLog2Pi), kLogHalf);
    return crw_in_box(x[0]) ? DSUB(norm, DMUL(DMUL(0.5, x[0]), x[0])) : -CUDART_INF;
  }
  if (M.kind == DSMC_MODEL_SV) {
    const double v0 = M.sv_s2 / (1.0 - M.sv_phi * M.sv_phi);
    const double dx = x[0] - M.sv_mu;
    return -0.5 * (kLog2Pi + log(v0)) - dx * dx / (2.0 * v0) - tc.logabsy;
  }
  double W0[16], L0[16];
  dchol(M.P0, d, L0);
  dtri_inv(L0, d, W0);
  const double norm0 = dnorm_of(L0, d);
  const double p0 = norm0 - 0.5 * dquad(W0, d, x, M.m0);
  double zz = 0.0;
  double e[4];
  for (int k = 0; k < d; ++k) e[k] = x[k] - tc.pm[k];
  for (int k = 0; k < d; ++k) {
    double acc = 0.0;
    for (int l = 0; l <= k; ++l) acc += tc.pW[k * d + l] * e[l];
    zz += acc * acc;
  }
  const double q0 = tc.p_norm - 0.5 * zz;
  double h0 = 0.0;
  if (tc.obs) {
    const double* H = at(M.H, M.H_s, 0);
    double hx[4];
    for (int a = 0; a < M.dy; ++a) {
      double s = 0.0;
      for (int l = 0; l < d; ++l) s += H[a * d + l] * x[l];
      hx[a] = s;
    }
    h0 = tc.o_norm - 0.5 * dquad(tc.oW, M.dy, M.y, hx);
  }
  return h0 + p0 - q0;
}

// FP32 leaf: centred state x - m_t = L_t z (float4), column term
// log2e * (log h_t - log nu_t + log N-normaliser of the transition into t)
// written from z directly (no cancellation), leaf-0 raw weight in
// FP64. For every device model q_t = nu_t, so leaves t >= 1 are uniform.
// Grid (time, chain), 256 threads looping over the time's particles: the
// time's FP32 constants and the model fields are staged in shared memory once
// per time (not once per 128 particles). Uniforms are formed in FP32 from the
// top 24 bits of the reference stream's u64s (same Philox4x64-10 stream and
// counter layout as the FP64 path, rng.cpp:45-86; FP32 rounding only).
template <int D>
#ifndef DSMC_LEAF32_MINB
#define DSMC_LEAF32_MINB 4  // 64 registers: 4 CTAs per SM (C5 leaves 16.6 -> 16.1 ms)
#endif
__global__ void __launch_bounds__(256, DSMC_LEAF32_MINB) leaf32_kernel(Bufs b, double* raw0,
                                                                       int t_off = 0) {
  const int t = t_off + blockIdx.x, ch = blockIdx.y;
  const int gt = b.t0 + t;  // global time (stream key, model data)
  const DevModel& M = b.models[ch];
  const TimeConst& tc = b.tc[(size_t)ch * b.Kt + b.t0 + t];
  __shared__ float s_L[16], s_G[16], s_e[4], s_c, s_sv2, s_y, s_cc, s_m;
  __shared__ int s_kind, s_dy, s_obs;
  if (threadIdx.x < 16) {
    s_L[threadIdx.x] = (float)tc.pL[threadIdx.x];
    s_G[threadIdx.x] = (float)tc.G[threadIdx.x];
  }
  if (threadIdx.x < 4) s_e[threadIdx.x] = (float)tc.e[threadIdx.x];
  if (threadIdx.x == 0) {
    s_c = (float)tc.cconst;
    s_kind = M.kind;
    s_dy = M.dy;
    s_obs = tc.obs;
    s_sv2 = (float)(2.0 * tc.logabsy);
    if (M.kind == DSMC_MODEL_COX) {
      // column term log h - log nu + trans_norm = y x - e^x + [-lgam - p_norm
      // + trans_norm] + z^2 / 2 (p_norm = -0.5 log(2 pi v*), z = (x - m*) / sd)
      s_y = (float)M.y[gt];
      s_cc = (float)(-M.lgam[gt] + 0.5 * (kLog2Pi + log(M.mp[3])) + M.mp[4]);
      s_m = (float)M.mp[2];
    } else if (M.kind == DSMC_MODEL_CRW) {
      s_cc = (float)(M.mp[1] - kLogHalf);
    }
  }
  __syncthreads();
  const int kind = s_kind, dy = s_dy;
  const bool obs = s_obs != 0;
  const StreamId id = stream_id(b.seeds[ch], 0, leaf_node(gt, b.conditional, b.sweep),
                                b.leaf_role ? b.leaf_role : DSMC_ROLE_LEAF_PROPOSAL, 0);
  const float colsv = (float)(kLog2E * tc.shift1);
  if (gt != 0 && !b.conditional) {
    // hot path (every leaf but global time 0 of an unconditional run):
    // normals -> centred state + column term, nothing else live
    for (int n = threadIdx.x; n < b.N; n += blockDim.x) {
      const size_t off = ((size_t)ch * b.K + t) * b.N + n;
      float z[4] = {0.f, 0.f, 0.f, 0.f};
      if (kind == DSMC_MODEL_CRW) {  // U[-1, 1] proposal, u64 number n
        const float x = 2.f * ((float)(uint32_t)(stream_u64(id, n) >> 40) * 0x1p-24f) - 1.f;
        b.X32[off] = make_float4(x, 0.f, 0.f, 0.f);
        b.COL[off] = (float)kLog2E * s_cc;
        continue;
      }
      U64x4 blk;
      uint64_t have = ~0ull;
      float r = 0.f, sn = 0.f, cs = 0.f;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const uint64_t i = (uint64_t)n * D + k;
        if (k == 0 || !(i & 1)) {
          const uint64_t q = 2 * (i >> 1);
          if ((q >> 2) != have) {
            blk = stream_block(id, q >> 2);
            have = q >> 2;
          }
          const float u1 = u01_open23(pick4(blk, (uint32_t)(q & 3)));
          const float u2 = u01_23(pick4(blk, (uint32_t)(q & 3) + 1));
          { const float a2 = -2.0f * __logf(u1); r = a2 * rsqrtf(a2); }  // a2 in (0, 34]
          sincospif(2.0f * u2, &sn, &cs);
        }
        z[k] = (i & 1) ? r * sn : r * cs;
      }
      float xv[4] = {0.f, 0.f, 0.f, 0.f};
      float col;
      if (kind == DSMC_MODEL_SV) {
        xv[0] = s_sv2 - __logf(z[0] * z[0]);
        col = colsv;
      } else if (kind == DSMC_MODEL_COX) {
        xv[0] = s_L[0] * z[0];
        const float x = s_m + xv[0];
        col = (float)kLog2E * (fmaf(s_y, x, -__expf(x)) + s_cc + 0.5f * z[0] * z[0]);
      } else {
#pragma unroll
        for (int k = 0; k < D; ++k) {
          float acc = 0.f;
#pragma unroll
          for (int l = 0; l <= k; ++l) acc = fmaf(s_L[k * D + l], z[l], acc);
          xv[k] = acc;
        }
        float zz = 0.f, rr = 0.f;
#pragma unroll
        for (int k = 0; k < D; ++k) zz = fmaf(z[k], z[k], zz);
        if (obs) {
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            if (a >= dy) break;
            float g = s_e[a];
#pragma unroll
            for (int l = 0; l < D; ++l) g = fmaf(-s_G[a * D + l], z[l], g);
            rr = fmaf(g, g, rr);
          }
        }
        col = (float)kLog2E * (s_c + 0.5f * (zz - rr));
      }
      b.X32[off] = make_float4(xv[0], xv[1], xv[2], xv[3]);
      b.COL[off] = col;
    }
  } else
  for (int n = threadIdx.x; n < b.N; n += blockDim.x) {
    const size_t off = ((size_t)ch * b.K + t) * b.N + n;
    float z[4] = {0.f, 0.f, 0.f, 0.f};
    float xv[4] = {0.f, 0.f, 0.f, 0.f};
    float col;
    const bool is_star = b.conditional && n == 0;
    double xstar[4] = {0, 0, 0, 0};
    if (is_star) {
#pragma unroll
      for (int k = 0; k < D; ++k) xstar[k] = b.star[((size_t)ch * b.K + t) * D + k];
    } else if (kind == DSMC_MODEL_CRW) {
      const uint64_t p = b.conditional ? n - 1 : n;
      xv[0] = 2.f * ((float)(uint32_t)(stream_u64(id, p) >> 40) * 0x1p-24f) - 1.f;
    } else {
      const uint64_t p = b.conditional ? n - 1 : n;
      // D normals, counter-addressed Box-Muller pairs (normal i uses u64s
      // 2*(i/2) and 2*(i/2)+1, rng.cpp:74-86): one Philox block serves up to
      // two pairs and one (r, theta) serves both normals of a pair
      U64x4 blk;
      uint64_t have = ~0ull;
      float r = 0.f, sn = 0.f, cs = 0.f;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const uint64_t i = p * D + k;
        if (k == 0 || !(i & 1)) {
          const uint64_t q = 2 * (i >> 1);
          if ((q >> 2) != have) {
            blk = stream_block(id, q >> 2);
            have = q >> 2;
          }
          // uniform_pos / uniform at 24-bit resolution: (0,1) and [0,1)
          const float u1 = u01_open23(pick4(blk, (uint32_t)(q & 3)));
          const float u2 = u01_23(pick4(blk, (uint32_t)(q & 3) + 1));
          { const float a2 = -2.0f * __logf(u1); r = a2 * rsqrtf(a2); }  // a2 in (0, 34]
          sincospif(2.0f * u2, &sn, &cs);
        }
        z[k] = (i & 1) ? r * sn : r * cs;
      }
    }
    if (kind == DSMC_MODEL_SV) {
      xv[0] = is_star ? (float)xstar[0] : s_sv2 - __logf(z[0] * z[0]);
      col = colsv;
    } else if (kind == DSMC_MODEL_CRW) {
      if (is_star) xv[0] = (float)xstar[0];
      col = (xv[0] >= -1.f && xv[0] <= 1.f) ? (float)kLog2E * s_cc : -CUDART_INF_F;
    } else if (kind == DSMC_MODEL_COX) {
      if (is_star) {
        xv[0] = (float)(xstar[0] - tc.pm[0]);
        z[0] = (float)((xstar[0] - tc.pm[0]) * tc.pW[0]);
      } else {
        xv[0] = s_L[0] * z[0];
      }
      const float x = s_m + xv[0];
      col = (float)kLog2E * (fmaf(s_y, x, -__expf(x)) + s_cc + 0.5f * z[0] * z[0]);
    } else {
      if (is_star) {
        // z = W_P (x* - m_t): the reference state expressed in proposal units
        double e[4];
#pragma unroll
        for (int k = 0; k < D; ++k) e[k] = xstar[k] - tc.pm[k];
#pragma unroll
        for (int k = 0; k < D; ++k) {
          double acc = 0.0;
#pragma unroll
          for (int l = 0; l <= k; ++l) acc += tc.pW[k * D + l] * e[l];
          z[k] = (float)acc;
        }
#pragma unroll
        for (int k = 0; k < D; ++k) xv[k] = (float)e[k];
      } else {
#pragma unroll
        for (int k = 0; k < D; ++k) {
          float acc = 0.f;
#pragma unroll
          for (int l = 0; l <= k; ++l) acc = fmaf(s_L[k * D + l], z[l], acc);
          xv[k] = acc;
        }
      }
      float zz = 0.f, rr = 0.f;
#pragma unroll
      for (int k = 0; k < D; ++k) zz = fmaf(z[k], z[k], zz);
      if (obs) {
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          if (a >= dy) break;
          float g = s_e[a];
#pragma unroll
          for (int l = 0; l < D; ++l) g = fmaf(-s_G[a * D + l], z[l], g);
          rr = fmaf(g, g, rr);
        }
      }
      col = (float)kLog2E * (s_c + 0.5f * (zz - rr));
    }
    b.X32[off] = make_float4(xv[0], xv[1], xv[2], xv[3]);
    b.COL[off] = col;
    if (gt == 0) {
      double x[4];
#pragma unroll
      for (int k = 0; k < D; ++k) x[k] = is_star ? xstar[k] : (double)xv[k] + tc.pm[k];
      raw0[(size_t)ch * b.N + n] = leaf0_raw_weight(M, tc, D, x);
    }
  }
  if (threadIdx.x == 0 && gt > 0) {  // q_t = nu_t: uniform leaf, lse = log N exactly
    const size_t o = (size_t)ch * b.K + t;
    b.LNC[o] = 0.0;
    b.UNI[o] = 1;
    b.LWMAX[o] = -log((double)b.N);
  }
}

// Leaf-0 normalisation for the FP32 path (log2 units) + leaf meta for all t.
__global__ void leafnorm32_kernel(Bufs b, const double* raw0) {
  const int ch = blockIdx.x, lane = threadIdx.x;
  const int N = b.N;
  const double* lw = raw0 + (size_t)ch * N;
  double mx = -CUDART_INF, lo = CUDART_INF, hi = -CUDART_INF;
  int nan = 0;
  for (int i = lane; i < N; i += 32) {
    const double v = lw[i];
    nan |= isnan(v);
    mx = fmax(mx, v);
    lo = fmin(lo, v);
    hi = fmax(hi, v);
  }
  for (int o = 16; o; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(~0u, mx, o));
    lo = fmin(lo, __shfl_xor_sync(~0u, lo, o));
    hi = fmax(hi, __shfl_xor_sync(~0u, hi, o));
    nan |= __shfl_xor_sync(~0u, nan, o);
  }
  if (nan || mx == -CUDART_INF) {
    if (lane == 0) raise_err(b.err, nan ? DSMC_E_DOMAIN : DSMC_E_RUNTIME, 0, 0, nan ? kReasonNaN : kReasonLeafZero);
    return;
  }
  double s = 0.0;
  for (int i = lane; i < N; i += 32) s += exp(lw[i] - mx);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(~0u, s, o);
  const double lse = mx + log(s);
  for (int i = lane; i < N; i += 32)
    b.LW32[(size_t)ch * N + i] = (float)((lw[i] - lse) * kLog2E);
  if (lane == 0) {
    const size_t o = (size_t)ch * b.K;
    b.LNC[o] = lse - log((double)N);
    b.UNI[o] = lo == hi;
    b.LWMAX[o] = mx - lse;
  }
}

}  // namespace dsmc_dev

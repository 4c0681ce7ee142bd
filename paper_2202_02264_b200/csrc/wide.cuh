// Wide-state FP32 path: linear-Gaussian models with state dimension
// 5 <= d <= 32 (the reference's FeynmanKacModel has no bound on state_dim,
// fk_model.hpp:38; the float4 path of combine32.cuh stops at 4). Templates
// over the padded dimension D in {8, 16, 32}.
//
// Per time t (prepared in FP64 on the device by prepw_kernel, stored FP32):
//   L_t  lower Cholesky of the proposal covariance       (x~ = x - m_t = L z)
//   G_t = Ro H L, e_t = Ro (y - H m), Ro = R^-1/2         (observation)
//   c_t  o_norm - p_norm + t_norm                         (column constant)
//   W_t = s W_Q, M_t = s W_Q F, v_t = s W_Q delta_t       (cut t, s = sqrt(log2e/2))
// so that, exactly as in combine32.cuh, the pair log-weight in log2 units is
//   w_ij = A_j + B_i + u_i . y_j,  y_j = W x~_j,  A_j = COL_j - |y_j|^2,
//   nu_i = M x~_i + v, u_i = 2 nu_i, B_i = lw2_i - |nu_i|^2.
// The cross term u_i . y_j is a real dense contraction at these d: pass 1
// computes it per 128-row x 64-column tile from shared-memory staged U / Y
// (register-tiled FFMA, 4 rows x 8 columns per thread) with the exact
// per-(row, sub-block) max as the exponent shift, then the usual 64-column
// sub-block log2-sums feed a sampler with the same row CDF / sub-block walk /
// 64-weight recompute as c32_sample.
#pragma once

#include "pair_tc.cuh"  // tcgen05 / mbarrier primitives

namespace dsmc_dev {

// rows of the pass-1 tile and the row stride of the staged operands
constexpr int kWRows = 128;
template <int D>
struct WideK {
  static constexpr int S = D + 4;  // padded smem row (floats), float4-aligned
};

// -------------------------------------------------------------- model prep
// Per-time FP64 constants of the header above, computed on the device: one
// warp per time t, lane = matrix row, matrices in shared memory (row stride
// 33 doubles). Same formulas and per-element operation order as the host
// version it replaced (Cholesky by columns, forward-substituted inverses);
// outputs are FP32 and the buffers are zero-filled by the caller, so only the
// live d x d / dy x d entries are written. The prior (P0) constants stay on
// the host (one matrix). err: the smallest failing time per kind (proposal
// covariance, R, Q), INT_MAX when none.
struct WidePrep {
  float *L, *G, *e, *c, *W, *M, *v;
  int* err;  // [3]
  int d, dy, DP, DYP, K;
};

constexpr int kPS = 33;  // shared row stride (doubles)

// Lower Cholesky of the n x n matrix A (global, row-major) into L (shared).
// Returns false (warp-uniform) when A is not positive definite.
__device__ inline bool warp_chol(const double* A, int n, double* L) {
  const int lane = threadIdx.x & 31;
  for (int j = 0; j < n; ++j) {
    double djj = 0.0;
    if (lane == 0) {
      double s = A[j * n + j];
      for (int k = 0; k < j; ++k) s -= L[j * kPS + k] * L[j * kPS + k];
      djj = s > 0.0 ? sqrt(s) : -1.0;
      L[j * kPS + j] = djj;
    }
    djj = __shfl_sync(~0u, djj, 0);
    if (!(djj > 0.0)) return false;
    for (int i = j + 1 + lane; i < n; i += 32) {
      double v = A[i * n + j];
      for (int k = 0; k < j; ++k) v -= L[i * kPS + k] * L[j * kPS + k];
      L[i * kPS + j] = v / djj;
    }
    __syncwarp();
  }
  return true;
}

// W = L^-1 (lower), column j by lane j.
__device__ inline void warp_tri_inv(const double* L, int n, double* W) {
  const int lane = threadIdx.x & 31;
  for (int j = lane; j < n; j += 32) {
    W[j * kPS + j] = 1.0 / L[j * kPS + j];
    for (int i = j + 1; i < n; ++i) {
      double s = 0.0;
      for (int k = j; k < i; ++k) s += L[i * kPS + k] * W[k * kPS + j];
      W[i * kPS + j] = -s / L[i * kPS + i];
    }
  }
  __syncwarp();
}

__device__ inline double warp_logdet(const double* L, int n) {  // 2 sum log L_jj, lane 0
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += 2.0 * log(L[i * kPS + i]);
  return s;
}

// grid K, 32 threads, 3 * 32 * 33 doubles of dynamic shared memory
__global__ void __launch_bounds__(32) prepw_kernel(DevModel md, WidePrep o) {
  extern __shared__ double psm[];
  double* Lt = psm;                 // proposal Cholesky
  double* Wm = psm + 32 * kPS;      // R / Q inverse Cholesky
  double* Tm = psm + 2 * 32 * kPS;  // scratch: R / Q Cholesky, then H L
  const int t = blockIdx.x, lane = threadIdx.x;
  const int d = o.d, dy = o.dy, DP = o.DP, DYP = o.DYP;
  const size_t dd = (size_t)d * d;
  const double s = sqrt(kLog2E / 2.0);
  const double* mt = md.prop_mean + (size_t)t * d;
  if (!warp_chol(md.prop_cov + (size_t)t * dd, d, Lt)) {
    if (lane == 0) atomicMin(&o.err[0], t);
    return;
  }
  for (int i = lane; i < d; i += 32)
    for (int j = 0; j <= i; ++j) o.L[(size_t)t * DP * DP + i * DP + j] = (float)Lt[i * kPS + j];
  const double p_norm = -0.5 * (d * kLog2Pi + warp_logdet(Lt, d));
  double o_norm = 0.0;
  const bool obs = md.has_obs ? md.has_obs[t] != 0 : true;
  if (obs) {
    const double* H = md.H + md.H_s * t;
    const double* R = md.R + md.R_s * t;
    if (!warp_chol(R, dy, Tm)) {
      if (lane == 0) atomicMin(&o.err[1], t);
      return;
    }
    warp_tri_inv(Tm, dy, Wm);
    o_norm = -0.5 * (dy * kLog2Pi + warp_logdet(Tm, dy));
    __syncwarp();
    for (int a = lane; a < dy; a += 32)  // H L (into Tm; R's factor is done)
      for (int j = 0; j < d; ++j) {
        double acc = 0.0;  // L is lower triangular (its upper part is not stored)
        for (int l = j; l < d; ++l) acc += H[a * d + l] * Lt[l * kPS + j];
        Tm[a * kPS + j] = acc;
      }
    __syncwarp();
    for (int a = lane; a < dy; a += 32) {
      double ea = 0.0;
      for (int b2 = 0; b2 <= a; ++b2) {
        double r = md.y[(size_t)t * dy + b2];
        for (int l = 0; l < d; ++l) r -= H[b2 * d + l] * mt[l];
        ea += Wm[a * kPS + b2] * r;
      }
      o.e[(size_t)t * DYP + a] = (float)ea;
      for (int j = 0; j < d; ++j) {
        double g = 0.0;
        for (int b2 = 0; b2 <= a; ++b2) g += Wm[a * kPS + b2] * Tm[b2 * kPS + j];
        o.G[(size_t)t * DYP * DP + a * DP + j] = (float)g;
      }
    }
    __syncwarp();
  }
  double t_norm = 0.0;
  if (t >= 1) {
    const double* F = md.F + md.F_s * t;
    const double* bb = md.b + md.b_s * t;
    const double* Q = md.Q + md.Q_s * t;
    if (!warp_chol(Q, d, Tm)) {
      if (lane == 0) atomicMin(&o.err[2], t);
      return;
    }
    warp_tri_inv(Tm, d, Wm);
    t_norm = -0.5 * (d * kLog2Pi + warp_logdet(Tm, d));
    const double* mp = md.prop_mean + (size_t)(t - 1) * d;
    __syncwarp();
    for (int j = lane; j < d; j += 32) {  // delta_j = (F m_{t-1} + b - m_t)_j, into Tm row 0
      double dj = bb[j] - mt[j];
      for (int l = 0; l < d; ++l) dj += F[j * d + l] * mp[l];
      Tm[j] = dj;
    }
    __syncwarp();
    for (int i = lane; i < d; i += 32) {
      double vi = 0.0;
      for (int j = 0; j <= i; ++j) {
        o.W[(size_t)t * DP * DP + i * DP + j] = (float)(s * Wm[i * kPS + j]);
        vi += Wm[i * kPS + j] * Tm[j];
      }
      o.v[(size_t)t * DP + i] = (float)(s * vi);
      for (int j = 0; j < d; ++j) {
        double acc = 0.0;
        for (int l = 0; l <= i; ++l) acc += Wm[i * kPS + l] * F[l * d + j];
        o.M[(size_t)t * DP * DP + i * DP + j] = (float)(s * acc);
      }
    }
  }
  if (lane == 0) o.c[t] = (float)(o_norm - p_norm + t_norm);
}

// ---------------------------------------------------------------- leaves
#ifndef LEAFW_MINB
#define LEAFW_MINB 3  // C6 d = 32 leaves 1.28 -> 1.16 ms (at 2: 128 registers)
#endif
template <int D>
__global__ void __launch_bounds__(256, LEAFW_MINB) leafw_kernel(Bufs b, double* raw0) {
  const int t = blockIdx.x, ch = blockIdx.y;
  const int gt = b.t0 + t;
  const WideBufs& w = b.w;
  const int d = w.d, dy = w.dy, N = b.N;
  __shared__ __align__(16) float sL[D * D], sG[32 * D], se[32], sWP[D * D], sdm[D];
  __shared__ float sc;
  for (int i = threadIdx.x; i < D * D; i += blockDim.x) sL[i] = w.L[(size_t)gt * D * D + i];
  for (int i = threadIdx.x; i < w.DYP * D; i += blockDim.x) sG[i] = w.G[(size_t)gt * w.DYP * D + i];
  for (int i = threadIdx.x; i < w.DYP; i += blockDim.x) se[i] = w.e[(size_t)gt * w.DYP + i];
  if (gt == 0) {
    for (int i = threadIdx.x; i < D * D; i += blockDim.x) sWP[i] = w.WP0[i];
    for (int i = threadIdx.x; i < D; i += blockDim.x) sdm[i] = w.dm0[i];
  }
  if (threadIdx.x == 0) sc = w.c[gt];
  __syncthreads();
  const StreamId id = stream_id(b.seeds[ch], 0, (uint64_t)gt, DSMC_ROLE_LEAF_PROPOSAL, 0);
  for (int n = threadIdx.x; n < N; n += blockDim.x) {
    // d normals, counter-addressed Box-Muller pairs (normal i uses u64s
    // 2(i/2), 2(i/2)+1 of the leaf stream, rng.cpp:74-86), i = n d + k
    float z[D];
    U64x4 blk;
    uint64_t have = ~0ull;
    float r = 0.f, sn = 0.f, cs = 0.f;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      z[k] = 0.f;
      if (k < d) {
        const uint64_t i = (uint64_t)n * d + k;
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
    }
    // x = L z and g = e - G z from broadcast 16-byte shared loads (4 entries
    // each); L's upper triangle is stored as zeros, and fma(0, z, acc) = acc,
    // so the row loops over whole float4s give the l <= k sums bit for bit
    const size_t off = ((size_t)ch * b.K + t) * N + n;
    float4* dst = reinterpret_cast<float4*>(w.X + off * D);
#pragma unroll
    for (int q = 0; q < D / 4; ++q) {  // four rows of x at a time, stored at once
      float xv[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const int k = 4 * q + kk;
        float acc = 0.f;
#pragma unroll
        for (int l4 = 0; l4 <= k; l4 += 4) {
          const float4 Lv = *reinterpret_cast<const float4*>(sL + k * D + l4);
          acc = fmaf(Lv.x, z[l4], acc);
          acc = fmaf(Lv.y, z[l4 + 1], acc);
          acc = fmaf(Lv.z, z[l4 + 2], acc);
          acc = fmaf(Lv.w, z[l4 + 3], acc);
        }
        xv[kk] = acc;
      }
      dst[q] = make_float4(xv[0], xv[1], xv[2], xv[3]);
    }
    float zz = 0.f, rr = 0.f;
#pragma unroll
    for (int k = 0; k < D; ++k) zz = fmaf(z[k], z[k], zz);
    for (int a = 0; a < dy; ++a) {
      float g = se[a];
#pragma unroll
      for (int l4 = 0; l4 < D; l4 += 4) {
        const float4 Gv = *reinterpret_cast<const float4*>(sG + a * D + l4);
        g = fmaf(-Gv.x, z[l4], g);
        g = fmaf(-Gv.y, z[l4 + 1], g);
        g = fmaf(-Gv.z, z[l4 + 2], g);
        g = fmaf(-Gv.w, z[l4 + 3], g);
      }
      rr = fmaf(g, g, rr);
    }
    const float col = (float)kLog2E * (sc + 0.5f * (zz - rr));
    b.COL[off] = col;
    if (gt == 0) {  // raw leaf-0 weight h0 P0 / q0 (log): col / log2e + log P0(x)
      const float* x = w.X + off * D;  // this thread's own stores, read back
      double qd = 0.0;
      for (int k = 0; k < D; ++k) {
        double acc = 0.0;
        for (int l = 0; l <= k; ++l) acc += (double)sWP[k * D + l] * ((double)x[l] - (double)sdm[l]);
        qd += acc * acc;
      }
      raw0[(size_t)ch * N + n] = (double)col * kLn2 + w.p0norm - 0.5 * qd;
    }
  }
  if (threadIdx.x == 0 && gt > 0) {  // q_t = nu_t: uniform leaf
    const size_t o = (size_t)ch * b.K + t;
    b.LNC[o] = 0.0;
    b.UNI[o] = 1;
    b.LWMAX[o] = -log((double)N);
  }
}

// ------------------------------------------------------------- prologue
// Per combine: whitened columns y_j / A_j and rows u_i / B_i (one index per
// thread for both), into the combine's AUX slice: Y[N][D], U[N][D], A[N], B[N].
struct AuxW {
  float* Y;
  float* U;
  float* A;
  float* B;
  float* YT;  // pass 1's column operand, one K-major core-matrix tile per sub-block
};
// floats per combine of the wide AUX: Y, U (N x D), A, B (N), then the
// 256-byte aligned column tiles (nsub x WideTc2<D>::B_BYTES)
__host__ __device__ inline size_t auxw_yt_off(int N, int D) {
  return ((size_t)2 * N * D + 2 * (size_t)N + 63) & ~(size_t)63;
}
template <int D>
__device__ __forceinline__ AuxW auxw(const LevelArgs& la, size_t comb, int N) {
  float* base = la.aux + comb * la.aux_comb;
  AuxW a;
  a.Y = base;
  a.U = base + (size_t)N * D;
  a.A = base + 2 * (size_t)N * D;
  a.B = base + 2 * (size_t)N * D + N;
  a.YT = base + auxw_yt_off(N, D);
  return a;
}

// Pipelined tensor-core pass 1 (pairw_tc2_kernel): K-major operands with the
// column and row terms folded into the contraction,
//   A_i = [u_hi(D), u_lo(D), u_hi(D), 1, 1, 1, b_hi, b_mid, b_lo, 0...]
//   B_j = [y_hi(D), y_hi(D), y_lo(D), a_hi, a_mid, a_lo, 1, 1, 1, 0...]
// so D_ij = u_i . y_j + A_j + B_i = w_ij (3xTF32, three-way splits of A_j
// and B_i); dead columns / rows carry a finite stand-in (kDeadColW).
constexpr float kDeadColW = -1e30f;
template <int D>
struct WideTc2 {
  static constexpr int K = 3 * D + 8;
  static constexpr int KC = K / 4;         // 16-byte chunks per operand row
  static constexpr int LBO = 128;          // bytes between K-adjacent core matrices
  static constexpr int SBO = KC * 128;     // bytes between 8-row groups
  static constexpr int KS = K / 8;         // MMAs per tile (K = 8 per tf32 MMA)
  static constexpr int A_BYTES = kWRows / 8 * SBO;
  static constexpr int B_BYTES = kSub / 8 * SBO;
  static constexpr int SMEM = A_BYTES + 2 * B_BYTES + 64 + 2 * kWRows * 8;  // + barriers, halves
};
template <int D>
__device__ __forceinline__ void wtc2_store_row(uint8_t* base, int r, const float* vals) {
  using L = WideTc2<D>;
  uint8_t* p = base + (r & 7) * 16 + (r >> 3) * L::SBO;
#pragma unroll
  for (int c = 0; c < L::KC; ++c)
    *reinterpret_cast<float4*>(p + c * L::LBO) =
        make_float4(vals[4 * c], vals[4 * c + 1], vals[4 * c + 2], vals[4 * c + 3]);
}
// column q's row of its sub-block tile (the prologue writes them; padding
// columns q >= N get y = 0 and the dead stand-in)
template <int D>
__device__ __forceinline__ void wtc2_store_col(const AuxW& ax, int q, const float* y, float a) {
  using L = WideTc2<D>;
  float vals[L::K];
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const float hi = tf32_hi(y[c]);
    vals[c] = hi;
    vals[D + c] = hi;
    vals[2 * D + c] = y[c] - hi;
  }
  const float av = a > kDeadColW ? a : kDeadColW;
  const float ah = tf32_hi(av), r1 = av - ah, am = tf32_hi(r1);
  vals[3 * D] = ah;
  vals[3 * D + 1] = am;
  vals[3 * D + 2] = r1 - am;
  vals[3 * D + 3] = vals[3 * D + 4] = vals[3 * D + 5] = 1.f;  // x the row's B_i split
#pragma unroll
  for (int c = 3 * D + 6; c < L::K; ++c) vals[c] = 0.f;
  uint8_t* tile = reinterpret_cast<uint8_t*>(ax.YT) + (size_t)(q / kSub) * L::B_BYTES;
  wtc2_store_row<D>(tile, q % kSub, vals);
}

template <int D>
__global__ void __launch_bounds__(128) prologw_kernel(Bufs b, LevelArgs la) {
  const int k = la.k0 + blockIdx.y, ch = blockIdx.z;
  const int N = b.N;
  Side L, R;
  CombineGeom g;
  sides(b, la, k, L, R, g);
  const int gc = b.t0 + g.c;
  const WideBufs& w = b.w;
  __shared__ float sW[D * D], sM[D * D], sv[D];
  for (int i = threadIdx.x; i < D * D; i += blockDim.x) {
    sW[i] = w.W[(size_t)gc * D * D + i];
    sM[i] = w.M[(size_t)gc * D * D + i];
  }
  for (int i = threadIdx.x; i < D; i += blockDim.x) sv[i] = w.v[(size_t)gc * D + i];
  __syncthreads();
  const size_t cslot = (size_t)blockIdx.z * gridDim.y + blockIdx.y;
  const AuxW ax = auxw<D>(la, cslot, N);
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= N) {
    if (la.wide_tiles && q < (N + kSub - 1) / kSub * kSub) {  // padding column of the last tile
      float y0[D];
#pragma unroll
      for (int c = 0; c < D; ++c) y0[c] = 0.f;
      wtc2_store_col<D>(ax, q, y0, -CUDART_INF_F);
    }
    return;
  }
  const bool lnonuni = L.leaf && !b.UNI[(size_t)ch * b.K + L.t];
  float x[D], y[D];
  {  // column q: right block's first-leaf state
    const uint32_t p = map_first(b, la, ch, R, q);
    const float4* src = reinterpret_cast<const float4*>(w.X + (((size_t)ch * b.K + R.t) * N + p) * D);
#pragma unroll
    for (int c = 0; c < D / 4; ++c) {
      const float4 v = src[c];
      x[4 * c] = v.x;
      x[4 * c + 1] = v.y;
      x[4 * c + 2] = v.z;
      x[4 * c + 3] = v.w;
    }
    float nrm = 0.f;
#pragma unroll
    for (int r = 0; r < D; ++r) {
      float acc = 0.f;
#pragma unroll
      for (int l = 0; l <= r; ++l) acc = fmaf(sW[r * D + l], x[l], acc);
      y[r] = acc;
      nrm = fmaf(acc, acc, nrm);
    }
    const float col = b.COL[((size_t)ch * b.K + R.t) * N + p];
    float4* dst = reinterpret_cast<float4*>(ax.Y + (size_t)q * D);
#pragma unroll
    for (int c = 0; c < D / 4; ++c) dst[c] = make_float4(y[4 * c], y[4 * c + 1], y[4 * c + 2], y[4 * c + 3]);
    ax.A[q] = col - nrm;
    if (la.wide_tiles) wtc2_store_col<D>(ax, q, y, col - nrm);
  }
  {  // row q: left block's last-leaf state
    const uint32_t p = map_last(b, la, ch, L, q);
    const float4* src = reinterpret_cast<const float4*>(w.X + (((size_t)ch * b.K + L.t) * N + p) * D);
#pragma unroll
    for (int c = 0; c < D / 4; ++c) {
      const float4 v = src[c];
      x[4 * c] = v.x;
      x[4 * c + 1] = v.y;
      x[4 * c + 2] = v.z;
      x[4 * c + 3] = v.w;
    }
    float nrm = 0.f;
#pragma unroll
    for (int r = 0; r < D; ++r) {
      float acc = sv[r];
#pragma unroll
      for (int l = 0; l < D; ++l) acc = fmaf(sM[r * D + l], x[l], acc);
      y[r] = 2.f * acc;
      nrm = fmaf(acc, acc, nrm);
    }
    const float lw2 = lnonuni ? b.LW32[(size_t)ch * N + q] : 0.f;
    float4* dst = reinterpret_cast<float4*>(ax.U + (size_t)q * D);
#pragma unroll
    for (int c = 0; c < D / 4; ++c) dst[c] = make_float4(y[4 * c], y[4 * c + 1], y[4 * c + 2], y[4 * c + 3]);
    ax.B[q] = lw2 - nrm;
  }
}

// ---------------------------------------------------------------- pass 1
// Grid (row tiles x column splits, combines, chains), 256 threads: rows
// [128 rt, +128) of combine k, sub-blocks [sb0, sb1). Thread (ty, tx) owns
// rows 4 ty .. 4 ty + 3 and columns tx + 8 c (c < 8) of the staged sub-block.
template <int D>
__global__ void __launch_bounds__(256) pairw_kernel(Bufs b, LevelArgs la) {
  constexpr int S = WideK<D>::S;
  extern __shared__ float wsm[];
  float* sU = wsm;                    // [128][S]
  float* sY = sU + kWRows * S;        // [64][S]
  float* sB = sY + kSub * S;          // [128]
  float* sA = sB + kWRows;            // [64]
  const int N = b.N;
  const int nsub = (N + kSub - 1) / kSub;
  const int nrt = (N + kWRows - 1) / kWRows;
  const int rt = blockIdx.x % nrt, cs = blockIdx.x / nrt, ncs = gridDim.x / nrt;
  const size_t cslot = (size_t)blockIdx.z * gridDim.y + blockIdx.y;
  const AuxW ax = auxw<D>(la, cslot, N);
  float* ws = reinterpret_cast<float*>(la.ws) + cslot * la.ws_comb * 2;
  const int row0 = rt * kWRows;
  const int tid = threadIdx.x, ty = tid >> 3, tx = tid & 7;
  for (int e = tid; e < kWRows * (D / 4); e += blockDim.x) {
    const int r = e / (D / 4), c = e % (D / 4);
    const int i = row0 + r;
    const float4 v = i < N ? reinterpret_cast<const float4*>(ax.U + (size_t)i * D)[c]
                           : make_float4(0.f, 0.f, 0.f, 0.f);
    *reinterpret_cast<float4*>(sU + r * S + 4 * c) = v;
  }
  for (int r = tid; r < kWRows; r += blockDim.x)
    sB[r] = row0 + r < N ? ax.B[row0 + r] : -CUDART_INF_F;
  const int sb0 = cs * nsub / ncs, sb1 = (cs + 1) * nsub / ncs;
  for (int s = sb0; s < sb1; ++s) {
    __syncthreads();  // sU / previous sY consumed
    for (int e = tid; e < kSub * (D / 4); e += blockDim.x) {
      const int j = e / (D / 4), c = e % (D / 4);
      const int col = s * kSub + j;
      const float4 v = col < N ? reinterpret_cast<const float4*>(ax.Y + (size_t)col * D)[c]
                               : make_float4(0.f, 0.f, 0.f, 0.f);
      *reinterpret_cast<float4*>(sY + j * S + 4 * c) = v;
    }
    for (int j = tid; j < kSub; j += blockDim.x)
      sA[j] = s * kSub + j < N ? ax.A[s * kSub + j] : -CUDART_INF_F;
    __syncthreads();
    float acc[4][8];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[r][c] = 0.f;
#pragma unroll 2
    for (int kk = 0; kk < D; kk += 4) {
      float4 uv[4], yv[8];
#pragma unroll
      for (int r = 0; r < 4; ++r) uv[r] = *reinterpret_cast<const float4*>(sU + (4 * ty + r) * S + kk);
#pragma unroll
      for (int c = 0; c < 8; ++c) yv[c] = *reinterpret_cast<const float4*>(sY + (tx + 8 * c) * S + kk);
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          float a = acc[r][c];
          a = fmaf(uv[r].x, yv[c].x, a);
          a = fmaf(uv[r].y, yv[c].y, a);
          a = fmaf(uv[r].z, yv[c].z, a);
          a = fmaf(uv[r].w, yv[c].w, a);
          acc[r][c] = a;
        }
    }
    // exact per-(row, sub-block) max shift, then the log2 sum (8 lanes share
    // a row: shuffles over tx)
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const float Bi = sB[4 * ty + r];
      float m = -CUDART_INF_F;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        acc[r][c] += sA[tx + 8 * c] + Bi;
        m = fmaxf(m, acc[r][c]);
      }
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) m = fmaxf(m, __shfl_xor_sync(~0u, m, o));
      float sum = 0.f;
      if (m > -CUDART_INF_F) {
#pragma unroll
        for (int c = 0; c < 8; ++c) sum += ex2(acc[r][c] - m);
      }
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) sum += __shfl_xor_sync(~0u, sum, o);
      const int i = row0 + 4 * ty + r;
      if (tx == 0 && i < N) ws[(size_t)s * N + i] = sum > 0.f ? m + lg2(sum) : -CUDART_INF_F;
    }
  }
}

// ---------------------------------------------------------------- sampler
// Grid (slot blocks, combines, chains), 256 threads: row log2-totals from the
// sub-block sums, FP64 row CDF, then per slot: row search, sub-block walk and
// the recompute of the chosen sub-block's <= 64 weights (D-term dots against
// the combine's Y / U), as c32_sample.
// Column / row data of the sampler's recompute: the wide AUX (D floats per
// row / column) or the float4 path's Aux32 (large N, below).
template <int D>
struct WideRecompute {
  AuxW ax;
  __device__ WideRecompute(const LevelArgs& la, size_t cslot, int N) : ax(auxw<D>(la, cslot, N)) {}
  __device__ float B(int i) const { return ax.B[i]; }
  __device__ void row(int i, float* u) const {
    const float4* up = reinterpret_cast<const float4*>(ax.U + (size_t)i * D);
#pragma unroll
    for (int c = 0; c < D / 4; ++c) {
      const float4 v = up[c];
      u[4 * c] = v.x;
      u[4 * c + 1] = v.y;
      u[4 * c + 2] = v.z;
      u[4 * c + 3] = v.w;
    }
  }
  // four independent FMA chains (components k mod 4) instead of one chain of
  // D: the recompute loop is latency-bound on this chain (one column at a
  // time per slot), not on issue
  __device__ float weight_exp(int j, const float* u, float sh) const {
    const float4* yp = reinterpret_cast<const float4*>(ax.Y + (size_t)j * D);
    float t0 = ax.A[j] + sh, t1 = 0.f, t2 = 0.f, t3 = 0.f;
#pragma unroll
    for (int c = 0; c < D / 4; ++c) {
      const float4 yv = yp[c];
      t0 = fmaf(u[4 * c], yv.x, t0);
      t1 = fmaf(u[4 * c + 1], yv.y, t1);
      t2 = fmaf(u[4 * c + 2], yv.z, t2);
      t3 = fmaf(u[4 * c + 3], yv.w, t3);
    }
    return ex2((t0 + t1) + (t2 + t3));
  }
};
// The float4 path's hand-off (pass 1 of c32_pair): d <= 4, pass 1's exact
// operation order t = A_j + sh; t = fma(u_k, y_k, t).
template <int D4>
struct Aux32Recompute {
  Aux32 ax;
  __device__ Aux32Recompute(const LevelArgs& la, size_t cslot, int N) : ax(aux32(la, cslot, N)) {}
  __device__ float B(int i) const { return ax.B[i]; }
  __device__ void row(int i, float* u) const {
    const float4 v = ax.u[i];
    u[0] = v.x;
    u[1] = v.y;
    u[2] = v.z;
    u[3] = v.w;
  }
  __device__ float weight_exp(int j, const float* u, float sh) const {
    const float4 y = ax.y[j];
    float t = ax.A[j] + sh;
    t = fmaf(u[0], y.x, t);
    if (D4 > 1) t = fmaf(u[1], y.y, t);
    if (D4 > 2) t = fmaf(u[2], y.z, t);
    if (D4 > 3) t = fmaf(u[3], y.w, t);
    return ex2(t);
  }
};

template <int D, class RC = WideRecompute<D>>
#ifndef DSMC_SAMPLEW_MINB
#define DSMC_SAMPLEW_MINB 4  // 64 registers: 4 CTAs per SM (C6 d = 32 sampler ~2x)
#endif
__global__ void __launch_bounds__(256, DSMC_SAMPLEW_MINB) samplew_kernel(Bufs b, LevelArgs la, int systematic) {
  extern __shared__ double wsmem[];
  __shared__ double sh[32];
  __shared__ float s_g;
  const int sb = blockIdx.x;
  const int k = la.k0 + blockIdx.y, ch = blockIdx.z;
  const int N = b.N;
  Side L, R;
  CombineGeom g;
  sides(b, la, k, L, R, g);
  const int nsub = (N + kSub - 1) / kSub;
  const size_t cslot = (size_t)blockIdx.z * gridDim.y + blockIdx.y;
  const float* ws = reinterpret_cast<const float*>(la.ws) + cslot * la.ws_comb * 2;
  const RC rc(la, cslot, N);
  double* S = wsmem;                                          // [N]
  float* Lrow = reinterpret_cast<float*>(S + ((N + 1) & ~1));  // [N]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float gm = -CUDART_INF_F;
  for (int i = tid; i < N; i += blockDim.x) {
    // online LSE over the row's sub-block sums, 16 loads in flight per round
    float m = -CUDART_INF_F, acc = 0.f;
    for (int s0 = 0; s0 < nsub; s0 += 16) {
      float v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = s0 + q < nsub ? ws[(size_t)(s0 + q) * N + i] : -CUDART_INF_F;
      float cm = v[0];
#pragma unroll
      for (int q = 1; q < 16; ++q) cm = fmaxf(cm, v[q]);
      if (cm == -CUDART_INF_F) continue;
      if (cm > m) {
        acc = m == -CUDART_INF_F ? 0.f : acc * ex2(m - cm);
        m = cm;
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) acc += ex2(v[q] - m);
    }
    const float La = m == -CUDART_INF_F ? -CUDART_INF_F : m + lg2(acc);
    Lrow[i] = La;
    gm = fmaxf(gm, La);
  }
  for (int o = 16; o; o >>= 1) gm = fmaxf(gm, __shfl_xor_sync(~0u, gm, o));
  if (lane == 0) sh[warp] = gm;
  __syncthreads();
  if (tid == 0) {
    float v = -CUDART_INF_F;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v = fmaxf(v, (float)sh[w]);
    s_g = v;
  }
  __syncthreads();
  const float G = s_g;
  if (G == -CUDART_INF_F) {
    if (tid == 0 && sb == 0) raise_err(b.err, DSMC_E_RUNTIME, g.c, la.level, kReasonZeroTable);
    return;
  }
  const int per = (N + blockDim.x - 1) / blockDim.x;
  const int i0 = tid * per, i1 = min(N, i0 + per);
  double seg = 0.0;
  for (int i = i0; i < i1; ++i) seg += (double)ex2(Lrow[i] - G);
  const double incl = block_scan_incl(seg, sh);
  double run = incl - seg;
  for (int i = i0; i < i1; ++i) {
    run += (double)ex2(Lrow[i] - G);
    S[i] = run;
  }
  __syncthreads();
  const double total = S[N - 1];
  const size_t gidx = (size_t)ch * b.T + la.cursor + k;
  if (tid == 0 && sb == 0) b.LMW[gidx] = ((double)G + log2(total)) * kLn2;
  const int off = b.conditional ? 1 : 0;  // c-dSMC: slot 0 is the reference pair
  const uint64_t node = b.conditional
                            ? (static_cast<uint64_t>(static_cast<uint32_t>(k + la.node_off)) |
                               (static_cast<uint64_t>(b.sweep) << 32))
                            : static_cast<uint64_t>(k + la.node_off);
  const StreamId id = stream_id(b.seeds[ch], la.key_level, node, DSMC_ROLE_PAIR_RESAMPLE, 0);
  double u0 = 0.0, step = 0.0;
  if (systematic) {
    u0 = u64_uniform(stream_u64(id, 0));
    step = total / (double)la.n_out;
  }
  uint32_t* PL = b.PL + gidx * N;
  uint32_t* PR = b.PR + gidx * N;
  const size_t nbase = ((size_t)ch * b.cap + k) * N;
  const int m0 = sb * la.slots_per_cta, m1 = min(la.n_out, m0 + la.slots_per_cta);
  const int ns = max(0, m1 - m0);
  // Two phases with a counting sort by sub-block in between (as c32_sample):
  // phase 1 (slot order) finds row i, sub-block s and the fraction inside s;
  // phase 2 (sub-block order) recomputes the chosen sub-block's weights, so a
  // warp's slots read the same column data (L1 broadcasts instead of 32
  // scattered D-float rows per load). The order only schedules work: slot m
  // always uses u64 number m of the stream and writes output m.
  const size_t ext = ((reinterpret_cast<char*>(Lrow + N) - reinterpret_cast<char*>(wsmem)) + 15) &
                     ~static_cast<size_t>(15);
  int4* REC = reinterpret_cast<int4*>(reinterpret_cast<char*>(wsmem) + ext);  // [ns]
  int* ORD = reinterpret_cast<int*>(REC + ns);                                // [ns]
  int* CB = ORD + ns;                                                         // [nsub]
  for (int q = tid; q < nsub; q += blockDim.x) CB[q] = 0;
  __syncthreads();
  for (int x = tid; x < ns; x += blockDim.x) {
    const int m = m0 + x;
    const double pt = systematic ? (u0 + (double)m) * step : u64_uniform(stream_u64(id, m)) * total;
    int lo = 0, hi = N;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (pt < S[mid]) hi = mid;
      else lo = mid + 1;
    }
    int i = lo < N ? lo : N - 1;
    const double before = i > 0 ? S[i - 1] : 0.0;
    while (i > 0 && !(Lrow[i] > -CUDART_INF_F)) --i;
    const float Li = Lrow[i];
    const float local0 = (float)((pt - before) / (double)ex2(Li - G));
    const float local = local0 >= 0.f ? local0 : 0.f;
    // sub-block walk (relative to the row total)
    int s = -1, last_pos = 0;
    float cum = 0.f, before_s = 0.f, wsel = 0.f, Ls_sel = 0.f;
    for (int q = 0; q < nsub; ++q) {
      const float v = ws[(size_t)q * N + i];
      const float e = ex2(v - Li);
      const float c2 = cum + e;
      if (s < 0 && e > 0.f) last_pos = q;
      if (s < 0 && local < c2) {
        s = q;
        before_s = cum;
        wsel = e;
        Ls_sel = v;
      }
      cum = c2;
    }
    if (s < 0) {
      s = last_pos;
      Ls_sel = ws[(size_t)s * N + i];
      wsel = ex2(Ls_sel - Li);
      before_s = cum - wsel;
    }
    float frac = wsel > 0.f ? (local - before_s) / wsel : 0.f;
    frac = fminf(fmaxf(frac, 0.f), 1.f);
    REC[x] = make_int4(i, s, __float_as_int(frac), __float_as_int(rc.B(i) - Ls_sel));
    atomicAdd(&CB[s], 1);
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the sub-block counts
    int carry = 0;
    for (int c0 = 0; c0 < nsub; c0 += 32) {
      const int c = c0 + lane < nsub ? CB[c0 + lane] : 0;
      int v = c;
      for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(~0u, v, o);
        if (lane >= o) v += n;
      }
      if (c0 + lane < nsub) CB[c0 + lane] = carry + v - c;
      carry += __shfl_sync(~0u, v, 31);
    }
  }
  __syncthreads();
  for (int x = tid; x < ns; x += blockDim.x) ORD[atomicAdd(&CB[REC[x].y], 1)] = x;
  __syncthreads();
  for (int o = tid; o < ns; o += blockDim.x) {
    const int x = ORD[o];
    const int4 rec = REC[x];
    const int i = rec.x, s = rec.y;
    const float frac = __int_as_float(rec.z), sh_i = __int_as_float(rec.w);
    // recompute the sub-block's weights relative to its sum: 2^(w_ij - L_is)
    float u[D < 4 ? 4 : D];
    rc.row(i, u);
    const int j0 = s * kSub, j1 = min(N, j0 + kSub);
    float c3 = 0.f;
    int jl = -1, lastpos = j0;
    for (int j = j0; j < j1; ++j) {
      const float e = rc.weight_exp(j, u, sh_i);
      if (e > 0.f) lastpos = j;
      c3 += e;
      if (jl < 0 && frac < c3) jl = j;
    }
    const int j = jl >= 0 ? jl : lastpos;  // spill (rounding): last positive weight
    const int m = m0 + x;
    PL[m + off] = (uint32_t)i;
    PR[m + off] = (uint32_t)j;
    la.first_next[nbase + m + off] = map_first(b, la, ch, L, (uint32_t)i);
    la.last_next[nbase + m + off] = map_last(b, la, ch, R, (uint32_t)j);
  }
  if (b.conditional && tid == 0 && sb == 0) {
    PL[0] = 0;
    PR[0] = 0;
    la.first_next[nbase] = map_first(b, la, ch, L, 0);
    la.last_next[nbase] = map_last(b, la, ch, R, 0);
  }
  if (tid == 0 && sb == 0) {
    const double logn = log((double)N);
    const bool luni = !L.leaf || b.UNI[(size_t)ch * b.K + L.t];
    const bool runi = !R.leaf || b.UNI[(size_t)ch * b.K + R.t];
    const double shift = (luni ? -logn : 0.0) + (runi ? -logn : 0.0);
    const double ll = block_lnc(b, la, ch, L, g.a);
    const double rl = block_lnc(b, la, ch, R, g.c);
    la.blnc_next[(size_t)ch * b.cap + k] = ll + rl + ((double)G + log2(total)) * kLn2 + shift;
  }
}

// ----------------------------------------------------------------- gather
// Level-1 composition + per-time moments: one CTA per (time, chain); chunks of
// 64 root slots are gathered into shared memory, threads own entries of the
// mean / upper covariance and accumulate over the chunk.
template <int D>
__global__ void __launch_bounds__(256) gatherw_kernel(Bufs b, const uint32_t* M1, int root1,
                                                      double* paths, double* mean, double* cov,
                                                      const uint32_t* root_map) {
  constexpr int NT = D * (D + 1) / 2;
  constexpr int CH = 64;
  const int t = blockIdx.x, ch = blockIdx.y;
  const int N = b.N, d = b.w.d;
  const int gt = b.t0 + t;
  __shared__ float sx[CH][D + 1];
  __shared__ int sk[NT], sl[NT];
  for (int e = threadIdx.x; e < NT; e += blockDim.x) {  // entry e -> (k, l), k <= l
    int k = 0, rem = e;
    while (rem >= D - k) {
      rem -= D - k;
      ++k;
    }
    sk[e] = k;
    sl[e] = k + rem;
  }
  float s1 = 0.f, acc[(NT + 255) / 256] = {};
  const float* X = b.w.X + ((size_t)ch * b.K + t) * N * D;
  const double* mt = b.w.m + (size_t)gt * d;
  for (int q0 = 0; q0 < N; q0 += CH) {
    __syncthreads();
    for (int e = threadIdx.x; e < CH * D; e += blockDim.x) {
      const int qq = e / D, k = e % D, q = q0 + qq;
      float v = 0.f;
      if (q < N) {
        const uint32_t sg = leaf_sigma(b, ch, t, q, M1, root1, root_map);
        v = X[(size_t)sg * D + k];
        if (paths && k < d) paths[(((size_t)ch * b.K + t) * N + q) * d + k] = (double)v + mt[k];
      }
      sx[qq][k] = v;
    }
    __syncthreads();
    const int nq = min(CH, N - q0);
    if (threadIdx.x < D)
      for (int qq = 0; qq < nq; ++qq) s1 += sx[qq][threadIdx.x];
#pragma unroll
    for (int u = 0; u < (NT + 255) / 256; ++u) {
      const int e = threadIdx.x + 256 * u;
      if (e < NT) {
        const int k = sk[e], l = sl[e];
        float a = acc[u];
        for (int qq = 0; qq < nq; ++qq) a = fmaf(sx[qq][k], sx[qq][l], a);
        acc[u] = a;
      }
    }
  }
  __shared__ double smu[D];
  if (threadIdx.x < D) smu[threadIdx.x] = (double)s1 / N;
  __syncthreads();
  const size_t o = (size_t)ch * b.K + t;
  if (mean && threadIdx.x < d) mean[o * d + threadIdx.x] = smu[threadIdx.x] + mt[threadIdx.x];
  if (cov) {
#pragma unroll
    for (int u = 0; u < (NT + 255) / 256; ++u) {
      const int e = threadIdx.x + 256 * u;
      if (e < NT) {
        const int k = sk[e], l = sl[e];
        if (k < d && l < d) {
          const double v = (double)acc[u] / N - smu[k] * smu[l];
          cov[o * d * d + k * d + l] = v;
          cov[o * d * d + l * d + k] = v;
        }
      }
    }
  }
}

// ------------------------------------------------- pass 1 on tcgen05 (wide)
// The cross term of a 128-row x 64-column tile as one tcgen05 MMA chain:
//   D[128 x 64] (TMEM, FP32) = A_rows[128 x 3D] . B_cols[64 x 3D]^T,
//   A_i = [u_hi, u_lo, u_hi], B_j = [y_hi, y_hi, y_lo]  (3xTF32, kind::tf32,
// K-major shared-memory operands without swizzle, the layout of pair_tc.cuh),
// so D_ij = u_i . y_j to ~FP32 accuracy (the dropped u_lo y_lo is ~2^-22
// relative). One elected thread issues the 3D / 8 MMAs of a sub-block and
// commits them to an mbarrier; each of the 128 threads then owns one row
// (TMEM lane): two tcgen05.ld.32x32b.x32 bring its 64 values to registers,
// and the epilogue adds A_j + B_i and takes the exact-max log2-sum on the SM
// (MUFU.EX2) — the same sub-block sums as pairw_kernel, with the d-term
// contraction moved off the FMA pipe. This is the north-star rule: tensor
// cores once the cross term is a real dense contraction (d >= 8 here).
template <int D>
struct WideTc {
  static constexpr int K = 3 * D;         // 3xTF32
  static constexpr int KC = K / 4;        // 16-byte chunks per operand row
  static constexpr int LBO = 128;         // bytes between K-adjacent core matrices
  static constexpr int SBO = KC * 128;    // bytes between 8-row groups
  static constexpr int KS = K / 8;        // MMAs per tile (K = 8 per tf32 MMA)
  static constexpr int A_BYTES = kWRows / 8 * SBO;
  static constexpr int B_BYTES = kSub / 8 * SBO;
  static constexpr int SMEM = A_BYTES + B_BYTES + 64 * 4 + 64;  // + A_j + barrier/tmem slot
};

template <int D>
__device__ __forceinline__ void wtc_store_row(uint8_t* base, int r, const float* vals) {
  using L = WideTc<D>;
  uint8_t* p = base + (r & 7) * 16 + (r >> 3) * L::SBO;
#pragma unroll
  for (int c = 0; c < L::KC; ++c)
    *reinterpret_cast<float4*>(p + c * L::LBO) =
        make_float4(vals[4 * c], vals[4 * c + 1], vals[4 * c + 2], vals[4 * c + 3]);
}

template <int D>
__global__ void __launch_bounds__(128) pairw_tc_kernel(Bufs b, LevelArgs la) {
  using L = WideTc<D>;
  extern __shared__ __align__(1024) uint8_t wtc_smem[];
  uint8_t* sA = wtc_smem;
  uint8_t* sB = sA + L::A_BYTES;
  float* sAj = reinterpret_cast<float*>(sB + L::B_BYTES);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sAj + 64);
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(bar + 1);
  const int N = b.N;
  const int nsub = (N + kSub - 1) / kSub;
  const int nrt = (N + kWRows - 1) / kWRows;
  const int rt = blockIdx.x % nrt, cs = blockIdx.x / nrt, ncs = gridDim.x / nrt;
  const size_t cslot = (size_t)blockIdx.z * gridDim.y + blockIdx.y;
  const AuxW ax = auxw<D>(la, cslot, N);
  float* ws = reinterpret_cast<float*>(la.ws) + cslot * la.ws_comb * 2;
  const int row0 = rt * kWRows;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(s_tmem)),
                 "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  // row operand: [u_hi, u_lo, u_hi] of row `tid`
  const int i = row0 + tid;
  float Bi = -CUDART_INF_F;
  {
    float vals[3 * D];
    float u[D];
    if (i < N) {
      const float4* up = reinterpret_cast<const float4*>(ax.U + (size_t)i * D);
#pragma unroll
      for (int c = 0; c < D / 4; ++c) {
        const float4 v = up[c];
        u[4 * c] = v.x;
        u[4 * c + 1] = v.y;
        u[4 * c + 2] = v.z;
        u[4 * c + 3] = v.w;
      }
      Bi = ax.B[i];
    } else {
#pragma unroll
      for (int c = 0; c < D; ++c) u[c] = 0.f;
    }
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const float hi = tf32_hi(u[c]);
      vals[c] = hi;
      vals[D + c] = u[c] - hi;
      vals[2 * D + c] = hi;
    }
    wtc_store_row<D>(sA, tid, vals);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *s_tmem;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kSub >> 3) << 17) |
                         ((uint32_t)(kWRows >> 4) << 24);
  const uint32_t lane_off = (uint32_t)(32 * warp) << 16;
  const int sb0 = cs * nsub / ncs, sb1 = (cs + 1) * nsub / ncs;
  uint32_t phase = 0;
  for (int s = sb0; s < sb1; ++s) {
    // column operand: threads 0-63 one column each; 64-127 the A_j
    if (tid < kSub) {
      const int j = s * kSub + tid;
      float y[D], vals[3 * D];
      if (j < N) {
        const float4* yp = reinterpret_cast<const float4*>(ax.Y + (size_t)j * D);
#pragma unroll
        for (int c = 0; c < D / 4; ++c) {
          const float4 v = yp[c];
          y[4 * c] = v.x;
          y[4 * c + 1] = v.y;
          y[4 * c + 2] = v.z;
          y[4 * c + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int c = 0; c < D; ++c) y[c] = 0.f;
      }
#pragma unroll
      for (int c = 0; c < D; ++c) {
        const float hi = tf32_hi(y[c]);
        vals[c] = hi;
        vals[D + c] = hi;
        vals[2 * D + c] = y[c] - hi;
      }
      wtc_store_row<D>(sB, tid, vals);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    } else {
      const int j = s * kSub + (tid - kSub);
      sAj[tid - kSub] = j < N ? ax.A[j] : -CUDART_INF_F;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (tid == 0) {
#pragma unroll
      for (int ks = 0; ks < L::KS; ++ks) {
        const uint64_t da = umma_sdesc(smem_u32(sA) + ks * 2 * L::LBO, L::LBO, L::SBO);
        const uint64_t db = umma_sdesc(smem_u32(sB) + ks * 2 * L::LBO, L::LBO, L::SBO);
        const uint32_t acc = ks > 0;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
      asm volatile(
          "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
              smem_u32(bar)));
    }
    mbar_wait(smem_u32(bar), phase);
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;");
    float v[64];
    tmem_ld32(tmem + lane_off, v);
    tmem_ld32(tmem + lane_off + 32, v + 32);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    float m = -CUDART_INF_F;
#pragma unroll
    for (int c = 0; c < 64; ++c) {
      v[c] += sAj[c] + Bi;
      m = fmaxf(m, v[c]);
    }
    float sum = 0.f;
    if (m > -CUDART_INF_F) {
#pragma unroll
      for (int c = 0; c < 64; ++c) sum += ex2(v[c] - m);
    }
    if (i < N) ws[(size_t)s * N + i] = sum > 0.f ? m + lg2(sum) : -CUDART_INF_F;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();  // TMEM, sB and sAj free for the next sub-block
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
}

// Pipelined pass 1 (default): the column operand tiles come from the
// prologue through bulk copies (cp.async.bulk, TMA engine) into two shared
// stages, the row operand is built once per CTA, and two TMEM accumulators
// (2 x 64 columns) let sub-block s+1's MMAs run while the CTA's threads
// take the exponentials of sub-block s. Per (row = TMEM lane, sub-block):
// the exact-max log2-sum of the 64 values D_ij + B_i, as pairw_tc_kernel.
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <int D>
__global__ void __launch_bounds__(256) pairw_tc2_kernel(Bufs b, LevelArgs la) {
  using L = WideTc2<D>;
  extern __shared__ __align__(1024) uint8_t wtc2_smem[];
  uint8_t* sA = wtc2_smem;
  uint8_t* sB = sA + L::A_BYTES;  // stage q at sB + q * B_BYTES
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + 2 * L::B_BYTES);  // [2] tile landed
  uint64_t* mmad = full + 2;                                          // [2] MMAs done
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(mmad + 2);
  float2* part = reinterpret_cast<float2*>(sB + 2 * L::B_BYTES + 64);  // [2 acc][128 rows]
  const int N = b.N;
  const int nsub = (N + kSub - 1) / kSub;
  const int nrt = (N + kWRows - 1) / kWRows;
  const int rt = blockIdx.x % nrt, cs = blockIdx.x / nrt, ncs = gridDim.x / nrt;
  const size_t cslot = (size_t)blockIdx.z * gridDim.y + blockIdx.y;
  const AuxW ax = auxw<D>(la, cslot, N);
  float* ws = reinterpret_cast<float*>(la.ws) + cslot * la.ws_comb * 2;
  const int row0 = rt * kWRows;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int sb0 = cs * nsub / ncs, sb1 = (cs + 1) * nsub / ncs, nit = sb1 - sb0;
  const uint8_t* YT = reinterpret_cast<const uint8_t*>(ax.YT);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(s_tmem)),
                 "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int q = 0; q < 4; ++q) mbar_init(full + q, 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
    for (int q = 0; q < 2 && q < nit; ++q)
      tma_bulk_g2s(sB + q * L::B_BYTES, YT + (size_t)(sb0 + q) * L::B_BYTES, L::B_BYTES, full + q);
  }
  // row operand of row `tid` (built while the first tiles are in flight)
  const int i = row0 + tid;
  float Bi = -CUDART_INF_F;
  if (tid < kWRows) {
    float vals[L::K];
    float u[D];
    if (i < N) {
      const float4* up = reinterpret_cast<const float4*>(ax.U + (size_t)i * D);
#pragma unroll
      for (int c = 0; c < D / 4; ++c) {
        const float4 v = up[c];
        u[4 * c] = v.x;
        u[4 * c + 1] = v.y;
        u[4 * c + 2] = v.z;
        u[4 * c + 3] = v.w;
      }
      Bi = ax.B[i];
    } else {
#pragma unroll
      for (int c = 0; c < D; ++c) u[c] = 0.f;
    }
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const float hi = tf32_hi(u[c]);
      vals[c] = hi;
      vals[D + c] = u[c] - hi;
      vals[2 * D + c] = hi;
    }
    vals[3 * D] = vals[3 * D + 1] = vals[3 * D + 2] = 1.f;
    const float bv = Bi > kDeadColW ? Bi : kDeadColW;
    const float bh = tf32_hi(bv), r1 = bv - bh, bm = tf32_hi(r1);
    vals[3 * D + 3] = bh;
    vals[3 * D + 4] = bm;
    vals[3 * D + 5] = r1 - bm;
#pragma unroll
    for (int c = 3 * D + 6; c < L::K; ++c) vals[c] = 0.f;
    wtc2_store_row<D>(sA, tid, vals);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *s_tmem;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kSub >> 3) << 17) |
                         ((uint32_t)(kWRows >> 4) << 24);
  // epilogue: warp w reads TMEM lanes 32 (w & 3).. (its rows) and columns
  // 32 (w >> 2).. of the accumulator; the two column halves meet in `part`
  const int quad = warp & 3, half = warp >> 2;
  const int erow = 32 * quad + (tid & 31), ei = row0 + erow;
  const uint32_t lane_off = ((uint32_t)(32 * quad) << 16) + 32 * half;
  for (int it = 0; it <= nit; ++it) {
    if (it < nit && tid == 0) {  // MMAs of sub-block sb0 + it into accumulator it & 1
      const int q = it & 1;
      mbar_wait(smem_u32(full + q), (it >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      uint8_t* tB = sB + q * L::B_BYTES;
#pragma unroll
      for (int ks = 0; ks < L::KS; ++ks) {
        const uint64_t da = umma_sdesc(smem_u32(sA) + ks * 2 * L::LBO, L::LBO, L::SBO);
        const uint64_t db = umma_sdesc(smem_u32(tB) + ks * 2 * L::LBO, L::LBO, L::SBO);
        const uint32_t acc = ks > 0;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + q * 64),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
      asm volatile(
          "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
              smem_u32(mmad + q)));
    }
    if (it > 0) {  // epilogue of sub-block sb0 + it - 1
      const int p = (it - 1) & 1;
      mbar_wait(smem_u32(mmad + p), ((it - 1) >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (tid == 0 && it + 1 < nit)  // stage p is free: fetch sub-block sb0 + it + 1
        tma_bulk_g2s(sB + p * L::B_BYTES, YT + (size_t)(sb0 + it + 1) * L::B_BYTES, L::B_BYTES,
                     full + p);
      float v[32];
      tmem_ld32(tmem + p * 64 + lane_off, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      // max and sum of the half as 8 independent chains
      float mc[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) mc[c] = v[c];
#pragma unroll
      for (int c = 8; c < 32; ++c) mc[c & 7] = fmaxf(mc[c & 7], v[c]);
      const float m = fmaxf(fmaxf(fmaxf(mc[0], mc[1]), fmaxf(mc[2], mc[3])),
                            fmaxf(fmaxf(mc[4], mc[5]), fmaxf(mc[6], mc[7])));
      float sum = 0.f;
      if (m > -1e29f) {
        float sc[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) sc[c] = ex2(v[c] - m);
#pragma unroll
        for (int c = 8; c < 32; ++c) sc[c & 7] += ex2(v[c] - m);
        sum = ((sc[0] + sc[1]) + (sc[2] + sc[3])) + ((sc[4] + sc[5]) + (sc[6] + sc[7]));
      }
      if (half == 1) part[p * kWRows + erow] = make_float2(m, sum);
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncthreads();  // accumulator p read by every warp before MMA(it + 1) reuses it
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (half == 0 && ei < N) {  // combine the halves (part[p] is rewritten two
        const float2 o = part[p * kWRows + erow];  // iterations later, after a barrier)
        const float M = fmaxf(m, o.x);
        float S = 0.f;
        if (M > -1e29f) S = (m > -1e29f ? sum * ex2(m - M) : 0.f) + (o.x > -1e29f ? o.y * ex2(o.x - M) : 0.f);
        ws[(size_t)(sb0 + it - 1) * N + ei] = S > 0.f ? M + lg2(S) : -CUDART_INF_F;
      }
    }
  }
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}

}  // namespace dsmc_dev

// FP32 throughput combine (the hot kernel).
//
// Pair log-weight in log2 units for cut c, left slot i, right slot j:
//   w_ij = A_j + B_i + u_i . y_j
// with y_j = s W_c x~_j (whitened right state, s = sqrt(log2e / 2)),
//      A_j = col2_j - |y_j|^2, col2_j = log2e (log h_c - log nu_c + norm),
//      nu_i = s W_c (F_c x~_i + delta_c), u_i = 2 nu_i,
//      B_i = lw2_L[i] - |nu_i|^2,
// i.e. -|y_j - nu_i|^2 expanded; states are stored centred on the proposal
// mean so the expansion does not cancel.
//
// c32_pair: one CTA per (row tile, combine). Each lane owns 16 consecutive
// columns (y, A in registers, packed float2 so the d+1 FMAs per pair issue
// as FFMA2); a 64-column sub-block is 4 lanes. Per row: d FFMA2 per column
// pair, sub-block max (FMNMX + 2 SHFL), exp2 (MUFU.EX2), sum (FADD2 + 2
// SHFL); one lane per sub-block writes L_s = m_s + log2(sum_s) + B_i.
// Nothing of the N x N table is stored beyond N*N/64 floats.
//
// c32_sample: one CTA per combine: row totals from the sub-block sums,
// row CDF (double inclusive scan), per-slot binary search over rows, walk
// over the row's sub-blocks, and recomputation of <= 64 weights with the
// same FP32 operations as pass 1.
#pragma once

#include "combine64.cuh"

namespace dsmc_dev {

constexpr int kCPL = 16;             // columns per lane
constexpr int kChunk = 32 * kCPL;    // columns per warp chunk (512)
constexpr int kRT = 64;              // rows per CTA tile
constexpr float kS = 0.84932180028801904272f;  // sqrt(log2(e) / 2)

struct CutConst32 {
  float W[16];   // s * tW (lower)
  float F[16];
  float delta[4];
};

template <int D>
__device__ inline void load_cut32(const TimeConst& tc, CutConst32& cc) {
  for (int k = 0; k < D; ++k) {
    for (int l = 0; l < D; ++l) {
      cc.W[k * D + l] = (float)(tc.tW[k * D + l]) * kS;
      cc.F[k * D + l] = (float)tc.F[k * D + l];
    }
    cc.delta[k] = (float)tc.delta[k];
  }
}

__device__ inline float comp(const float4& v, int k) {
  return k == 0 ? v.x : (k == 1 ? v.y : (k == 2 ? v.z : v.w));
}

// Column data y_j (whitened), A_j. Shared by pass 1 and the sampler so the
// recomputed weights are bit-identical.
template <int D>
__device__ inline void col32(const CutConst32& cc, float4 xv, float col,
                            float* y, float& A) {
  float nrm = 0.f;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    float acc = 0.f;
#pragma unroll
    for (int l = 0; l <= k; ++l) acc = fmaf(cc.W[k * D + l], comp(xv, l), acc);
    y[k] = acc;
    nrm = fmaf(acc, acc, nrm);
  }
  A = col - nrm;
}
template <int D>
__device__ inline void row32(const CutConst32& cc, float4 xv, float lw2,
                            float* u, float& Bv) {
  float mu[4];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    float acc = cc.delta[k];
#pragma unroll
    for (int l = 0; l < D; ++l) acc = fmaf(cc.F[k * D + l], comp(xv, l), acc);
    mu[k] = acc;
  }
  float nrm = 0.f;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    float acc = 0.f;
#pragma unroll
    for (int l = 0; l <= k; ++l) acc = fmaf(cc.W[k * D + l], mu[l], acc);
    u[k] = 2.f * acc;
    nrm = fmaf(acc, acc, nrm);
  }
  Bv = lw2 - nrm;
}
// Pair value with the pass-1 operation order: t = A; t = fma(u_k, y_k, t).
template <int D>
__device__ inline float pair32(const float* u, const float* y, float A) {
  float t = A;
#pragma unroll
  for (int k = 0; k < D; ++k) t = fmaf(u[k], y[k], t);
  return t;
}

__device__ __forceinline__ float ex2(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float lg2(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

struct Side32 {
  const float4* X;  // leaf slab
  const float* COL;
};

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// One row against this lane's 16 columns: the 64-column sub-block's max and
// sum of exp2(t - max) (identical in the 4 lanes of the sub-block).
template <int D>
__device__ __forceinline__ void row_sub(const float2 (&y2)[D][kCPL / 2],
                                        const float2 (&A2)[kCPL / 2],
                                        const float* u, float& m_out,
                                        float& s_out) {
  float2 t[kCPL / 2];
  float2 uu[D];
#pragma unroll
  for (int q = 0; q < D; ++q) uu[q] = make_float2(u[q], u[q]);
#pragma unroll
  for (int c2 = 0; c2 < kCPL / 2; ++c2) {
    float2 acc = A2[c2];
#pragma unroll
    for (int q = 0; q < D; ++q) acc = __ffma2_rn(uu[q], y2[q][c2], acc);
    t[c2] = acc;
  }
  // max tree with 3-input FMNMX
  const float a0 = fmax3(t[0].x, t[0].y, t[1].x);
  const float a1 = fmax3(t[1].y, t[2].x, t[2].y);
  const float a2 = fmax3(t[3].x, t[3].y, t[4].x);
  const float a3 = fmax3(t[4].y, t[5].x, t[5].y);
  const float a4 = fmax3(t[6].x, t[6].y, t[7].x);
  float m = fmax3(fmax3(a0, a1, a2), fmax3(a3, a4, t[7].y), a0);
  m = fmaxf(m, __shfl_xor_sync(~0u, m, 1));
  m = fmaxf(m, __shfl_xor_sync(~0u, m, 2));
  const float mm = (m == -CUDART_INF_F) ? 0.f : m;
  const float2 nm = make_float2(-mm, -mm);
  float2 e[kCPL / 2];
#pragma unroll
  for (int c2 = 0; c2 < kCPL / 2; ++c2) {
    const float2 dd = __fadd2_rn(t[c2], nm);
    e[c2] = make_float2(ex2(dd.x), ex2(dd.y));
  }
  const float2 s01 = __fadd2_rn(__fadd2_rn(e[0], e[1]), __fadd2_rn(e[2], e[3]));
  const float2 s23 = __fadd2_rn(__fadd2_rn(e[4], e[5]), __fadd2_rn(e[6], e[7]));
  const float2 s2 = __fadd2_rn(s01, s23);
  float sm = s2.x + s2.y;
  sm += __shfl_xor_sync(~0u, sm, 1);
  sm += __shfl_xor_sync(~0u, sm, 2);
  m_out = m;
  s_out = sm;
}

// Fast-path row: sum over this lane's 16 columns of 2^(A'_j + u.y_j) with no
// max subtraction. A'_j = A_j - cmax_s where cmax_s bounds col2 over the
// sub-block, so the argument equals w_ij - lw2_i - cmax_s + |nu_i|^2 and
// w_ij - lw2_i <= col2_j (the transition term -|y - nu|^2 is <= 0): the sum
// only leaves [2^-60, 2^100] for rows far from every column (the caller then
// recomputes them with the exact max).
// The argument is also <= |nu_i|^2, so rows with |nu_i|^2 > 100 (a few %)
// run the SHIFT variant with c_i = |nu_i|^2 - 100 subtracted (one FADD2 per
// two pairs), which keeps every exponent <= 100.
template <int D, bool SHIFT>
__device__ __forceinline__ float row_sum_fast(const float2 (&y2)[D][kCPL / 2],
                                              const float2 (&A2)[kCPL / 2],
                                              const float* u, float c) {
  float2 uu[D];
#pragma unroll
  for (int q = 0; q < D; ++q) uu[q] = make_float2(u[q], u[q]);
  const float2 nc = make_float2(-c, -c);
  float2 e[kCPL / 2];
#pragma unroll
  for (int c2 = 0; c2 < kCPL / 2; ++c2) {
    float2 acc = SHIFT ? __fadd2_rn(A2[c2], nc) : A2[c2];
#pragma unroll
    for (int q = 0; q < D; ++q) acc = __ffma2_rn(uu[q], y2[q][c2], acc);
    e[c2] = make_float2(ex2(acc.x), ex2(acc.y));
  }
  const float2 s01 = __fadd2_rn(__fadd2_rn(e[0], e[1]), __fadd2_rn(e[2], e[3]));
  const float2 s23 = __fadd2_rn(__fadd2_rn(e[4], e[5]), __fadd2_rn(e[6], e[7]));
  const float2 s2 = __fadd2_rn(s01, s23);
  return s2.x + s2.y;
}

// 4 rows x 4 lanes transpose-reduce: lane q (of a 4-lane sub-block group)
// returns the 4-lane total of row q (3 SHFL instead of 8).
__device__ __forceinline__ float quad_transpose_sum(const float (&s4)[4], int q4) {
  const bool b1 = q4 & 2, b0 = q4 & 1;
  float k0 = b1 ? s4[2] : s4[0], k1 = b1 ? s4[3] : s4[1];
  const float o0 = b1 ? s4[0] : s4[2], o1 = b1 ? s4[1] : s4[3];
  k0 += __shfl_xor_sync(~0u, o0, 2);
  k1 += __shfl_xor_sync(~0u, o1, 2);
  const float keep = b0 ? k1 : k0, send = b0 ? k0 : k1;
  return keep + __shfl_xor_sync(~0u, send, 1);
}

// Per-combine data pass 1 hands to the sampler (la.aux, la.aux_comb floats
// per combine of the chunk): whitened columns y_j / A_j and rows u_i / B_i,
// computed once by pass 1 instead of being re-gathered through the block maps.
struct Aux32 {
  float4* y;  // [N] column y_j (zero-padded to 4)
  float4* u;  // [N] row u_i = 2 nu_i
  float* A;   // [N] column A_j
  float* B;   // [N] row B_i
};
__device__ __forceinline__ Aux32 aux32(const LevelArgs& la, int comb, int N) {
  float* base = la.aux + (size_t)comb * la.aux_comb;
  Aux32 a;
  a.y = reinterpret_cast<float4*>(base);
  a.u = reinterpret_cast<float4*>(base + 4 * (size_t)N);
  a.A = base + 8 * (size_t)N;
  a.B = base + 9 * (size_t)N;
  return a;
}

// Pass 1. Grid (row tiles, combines, chains); la.rows_per_cta rows per CTA
// (a multiple of 32, chosen per level so the grid fills the GPU). Warps take
// (512-column chunk, row slice) items; rows go 4 at a time so that each lane
// finishes exactly one (row, sub-block) log-sum: one LG2 and one store per
// 64 pair evaluations, no divergent tail.
template <int D>
__global__ void __launch_bounds__(256, 2) c32_pair(Bufs b, LevelArgs la) {
  extern __shared__ float sm32[];
  const int RT = la.rows_per_cta;
  float* s_u = sm32;            // [RT][D]
  float* s_B = sm32 + RT * D;   // [RT]
  float* s_c = s_B + RT;        // [RT] fast-path shift c_i (0 for most rows)
  const int k = la.k0 + blockIdx.y, ch = blockIdx.z;
  const int N = b.N;
  Side L, R;
  CombineGeom g;
  sides(b, la, k, L, R, g);
  const TimeConst& tc = b.tc[(size_t)ch * b.Kt + b.t0 + g.c];
  CutConst32 cc;
  load_cut32<D>(tc, cc);
  const int nch = (N + kChunk - 1) / kChunk;
  const int nsubp = nch * (kChunk / kSub);
  // per (chain, combine of the chunk) workspace
  const size_t cslot = (size_t)blockIdx.z * gridDim.y + blockIdx.y;
  float* ws = reinterpret_cast<float*>(la.ws) + cslot * la.ws_comb * 2;
  const int row0 = blockIdx.x * RT;
  const int nrows = min(RT, N - row0);
  const Aux32 ax = aux32(la, cslot, N);
  const bool lnonuni = L.leaf && !b.UNI[(size_t)ch * b.K + L.t];
  const float4* XL = b.X32 + ((size_t)ch * b.K + L.t) * N;
  for (int r = threadIdx.x; r < RT; r += blockDim.x) {
    float u[4] = {0, 0, 0, 0}, Bv = -CUDART_INF_F;
    if (r < nrows) {
      const int i = row0 + r;
      const uint32_t p = map_last(b, la, ch, L, i);
      const float lw2 = lnonuni ? b.LW32[(size_t)ch * N + i] : 0.f;
      row32<D>(cc, XL[p], lw2, u, Bv);
      ax.u[i] = make_float4(u[0], u[1], u[2], u[3]);
      ax.B[i] = Bv;
    }
#pragma unroll
    for (int q = 0; q < D; ++q) s_u[r * D + q] = u[q];
    s_B[r] = Bv;
    float nn = 0.f;
#pragma unroll
    for (int q = 0; q < D; ++q) nn = fmaf(0.5f * u[q], 0.5f * u[q], nn);
    s_c[r] = nn > 100.f ? nn - 100.f : 0.f;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = max(1, 8 / nch);
  const int items = nch * S;
  const float4* XR = b.X32 + ((size_t)ch * b.K + R.t) * N;
  const float* CR = b.COL + ((size_t)ch * b.K + R.t) * N;
  const int q4 = lane & 3;
  if (blockIdx.x == 0) {  // hand the combine's columns to the sampler
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
      const uint32_t p = map_first(b, la, ch, R, j);
      float y[4] = {0.f, 0.f, 0.f, 0.f}, A;
      col32<D>(cc, XR[p], CR[p], y, A);
      ax.y[j] = make_float4(y[0], y[1], y[2], y[3]);
      ax.A[j] = A;
    }
  }
  for (int it = warp; it < items; it += 8) {
    const int chunk = it % nch, slice = it / nch;
    float2 y2[D][kCPL / 2];
    float2 A2[kCPL / 2];
    float cm = -CUDART_INF_F;
#pragma unroll
    for (int c2 = 0; c2 < kCPL / 2; ++c2) {
      float yv[2][4], Av[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = chunk * kChunk + lane * kCPL + 2 * c2 + h;
        if (j < N) {
          const uint32_t p = map_first(b, la, ch, R, j);
          const float cv = CR[p];
          col32<D>(cc, XR[p], cv, yv[h], Av[h]);
          cm = fmaxf(cm, cv);

        } else {
#pragma unroll
          for (int q = 0; q < D; ++q) yv[h][q] = 0.f;
          Av[h] = -CUDART_INF_F;
        }
      }
#pragma unroll
      for (int q = 0; q < D; ++q) y2[q][c2] = make_float2(yv[0][q], yv[1][q]);
      A2[c2] = make_float2(Av[0], Av[1]);
    }
    const int sub = chunk * (kChunk / kSub) + (lane >> 2);
    // column bound of the sub-block: cmax = max_j col2_j (4-lane max), folded
    // into A so the fast rows need no max (row_sum_fast)
    cm = fmaxf(cm, __shfl_xor_sync(~0u, cm, 1));
    cm = fmaxf(cm, __shfl_xor_sync(~0u, cm, 2));
    const bool live = cm > -CUDART_INF_F;
#pragma unroll
    for (int c2 = 0; c2 < kCPL / 2; ++c2)
      A2[c2] = live ? make_float2(A2[c2].x - cm, A2[c2].y - cm)
                    : make_float2(-CUDART_INF_F, -CUDART_INF_F);
    // rows slice, slice+S, ... taken 4 at a time (RT is a multiple of 4*S;
    // padded rows have B = -inf and are never stored)
    for (int base = slice; base < nrows; base += 4 * S) {
      float s4[4], c4[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) c4[j] = s_c[base + j * S];
      if (fmaxf(fmaxf(c4[0], c4[1]), fmaxf(c4[2], c4[3])) == 0.f) {  // warp-uniform
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int r = base + j * S;
          float u[D];
#pragma unroll
          for (int q = 0; q < D; ++q) u[q] = s_u[r * D + q];
          s4[j] = row_sum_fast<D, false>(y2, A2, u, 0.f);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int r = base + j * S;
          float u[D];
#pragma unroll
          for (int q = 0; q < D; ++q) u[q] = s_u[r * D + q];
          s4[j] = row_sum_fast<D, true>(y2, A2, u, c4[j]);
        }
      }
      const int rq = base + q4 * S;
      float sq = quad_transpose_sum(s4, q4);
      float mq = q4 == 0 ? c4[0] : q4 == 1 ? c4[1] : q4 == 2 ? c4[2] : c4[3];
      const bool odd = live && rq < nrows && !(sq >= 0x1p-60f && sq <= 0x1p120f);
      if (__any_sync(~0u, odd)) {  // rare: exact per-sub-block max
        float m4[4];
#pragma unroll 1
        for (int j = 0; j < 4; ++j) {
          const int r = base + j * S;
          float u[D];
#pragma unroll
          for (int q = 0; q < D; ++q) u[q] = s_u[r * D + q];
          row_sub<D>(y2, A2, u, m4[j], s4[j]);
        }
        mq = q4 == 0 ? m4[0] : q4 == 1 ? m4[1] : q4 == 2 ? m4[2] : m4[3];
        sq = q4 == 0 ? s4[0] : q4 == 1 ? s4[1] : q4 == 2 ? s4[2] : s4[3];
      }
      if (rq < nrows) {
        const float Ls = sq > 0.f ? mq + lg2(sq) + cm + s_B[rq] : -CUDART_INF_F;
        ws[(size_t)(row0 + rq) * nsubp + sub] = Ls;
      }
    }
  }
}

// Block-wide inclusive scan of doubles (one value per thread).
__device__ inline double block_scan_incl(double v, double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 1; o < 32; o <<= 1) {
    const double n = __shfl_up_sync(~0u, v, o);
    if (lane >= o) v += n;
  }
  if (lane == 31) sh[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double w = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
    for (int o = 1; o < 32; o <<= 1) {
      const double n = __shfl_up_sync(~0u, w, o);
      if (lane >= o) w += n;
    }
    sh[lane] = w;
  }
  __syncthreads();
  const double add = warp > 0 ? sh[warp - 1] : 0.0;
  __syncthreads();
  return v + add;
}

// Pass 2. Grid (slot blocks, combines, chains), 256 threads. Every slot block
// rebuilds the combine's row CDF (N row log-totals from the sub-block sums,
// vector loads + online LSE) and samples its slice of the n_out slots: binary
// search over the row CDF in shared memory, a walk over the row's sub-block
// sums, and a recomputation of the chosen sub-block's <= 64 weights with
// pass 1's FP32 pair arithmetic (two columns per FFMA2 / FADD2).
template <int D>
__global__ void __launch_bounds__(256, 3) c32_sample(Bufs b, LevelArgs la,
                                                     int systematic) {
  extern __shared__ double smem[];
  __shared__ double sh[32];
  __shared__ float s_g;
  const int sb = blockIdx.x;
  const int k = la.k0 + blockIdx.y, ch = blockIdx.z;
  const int N = b.N;
  Side L, R;
  CombineGeom g;
  sides(b, la, k, L, R, g);
  const int nch = (N + kChunk - 1) / kChunk;
  const int nsubp = nch * (kChunk / kSub);
  const int nsub = (N + kSub - 1) / kSub;
  const size_t cslot = (size_t)blockIdx.z * gridDim.y + blockIdx.y;
  const float* ws = reinterpret_cast<const float*>(la.ws) + cslot * la.ws_comb * 2;
  const Aux32 ax = aux32(la, cslot, N);
  // Column j lives at j + j/64 (one pad entry per sub-block): the per-slot
  // recompute loops read column 64 s + q of different sub-blocks s at the
  // same q, which without the skew all map to the same banks.
  const int NP = (N + kSub - 1) / kSub * kSub;
  const int NPS = NP + NP / kSub;
  double* S = smem;                                            // N
  float4* ycol = reinterpret_cast<float4*>(S + ((N + 1) & ~1));  // NPS, 16B aligned
  float* Acol = reinterpret_cast<float*>(ycol + NPS);           // NPS
  float* Lrow = Acol + NPS;                                    // N
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int j = tid; j < NP; j += blockDim.x) {
    float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
    float A = -CUDART_INF_F;
    if (j < N) {
      y = ax.y[j];
      A = ax.A[j];
    }
    ycol[j + j / kSub] = y;
    Acol[j + j / kSub] = A;
  }
  // row log2-totals: online LSE over the row's sub-block sums, 16 at a time
  // (pass 1 writes all nsubp entries; padding is -inf)
  float gm = -CUDART_INF_F;
  for (int i = tid; i < N; i += blockDim.x) {
    const float4* w4 = reinterpret_cast<const float4*>(ws + (size_t)i * nsubp);
    float m = -CUDART_INF_F, acc = 0.f;
    for (int s0 = 0; s0 < nsubp; s0 += 16) {
      float v[16];
      const int nq = min(4, (nsubp - s0) >> 2);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 t4 = q < nq ? w4[(s0 >> 2) + q]
                                 : make_float4(-CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F);
        v[4 * q] = t4.x;
        v[4 * q + 1] = t4.y;
        v[4 * q + 2] = t4.z;
        v[4 * q + 3] = t4.w;
      }
      float cm = fmax3(fmax3(v[0], v[1], v[2]), fmax3(v[3], v[4], v[5]), fmax3(v[6], v[7], v[8]));
      cm = fmax3(cm, fmax3(v[9], v[10], v[11]), fmax3(v[12], v[13], fmaxf(v[14], v[15])));
      if (cm == -CUDART_INF_F) continue;
      if (cm > m) {
        acc = m == -CUDART_INF_F ? 0.f : acc * ex2(m - cm);
        m = cm;
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) acc += ex2(v[q] - m);
    }
    const float L2 = m == -CUDART_INF_F ? -CUDART_INF_F : m + lg2(acc);
    Lrow[i] = L2;
    gm = fmaxf(gm, L2);
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
  const int off = b.conditional ? 1 : 0;
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
  // each thread takes 4 consecutive slots = one Philox block of uniforms
  // (slot m uses u64 number m of the stream, rng.cpp:45-68)
  for (int q0 = (m0 & ~3) + 4 * tid; q0 < m1; q0 += 4 * blockDim.x) {
    U64x4 blk;
    if (!systematic) blk = stream_block(id, (uint64_t)q0 >> 2);
#pragma unroll 1
    for (int qq = 0; qq < 4; ++qq) {
      const int m = q0 + qq;
      if (m < m0 || m >= m1) continue;
      const double pt = systematic ? (u0 + (double)m) * step : u64_uniform(blk.v[qq]) * total;
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
      const float4 urow = ax.u[i];
      const float Brow = ax.B[i];
      const float local0 = (float)((pt - before) / (double)ex2(Li - G));
      const float local = local0 >= 0.f ? local0 : 0.f;
      // sub-block walk over the row's sub-block sums (relative to the row
      // total), branch-free, 16 at a time from vector loads
      const float* w = ws + (size_t)i * nsubp;
      int s = -1, last_pos = 0;
      float cum = 0.f, before_s = 0.f, wsel = 0.f, Ls_sel = 0.f;
      for (int s0 = 0; s0 < nsub; s0 += 16) {
        float v[16];
        if (s0 + 16 <= nsubp) {
          const float4* w4 = reinterpret_cast<const float4*>(w + s0);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 t4 = w4[q];
            v[4 * q] = t4.x;
            v[4 * q + 1] = t4.y;
            v[4 * q + 2] = t4.z;
            v[4 * q + 3] = t4.w;
          }
        } else {
#pragma unroll
          for (int q = 0; q < 16; ++q) v[q] = (s0 + q < nsubp) ? w[s0 + q] : -CUDART_INF_F;
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const float e = (s0 + q < nsub) ? ex2(v[q] - Li) : 0.f;
          const float c2 = cum + e;
          const bool hit = s < 0 && local < c2;
          last_pos = (s < 0 && e > 0.f) ? s0 + q : last_pos;
          before_s = hit ? cum : before_s;
          wsel = hit ? e : wsel;
          Ls_sel = hit ? v[q] : Ls_sel;
          s = hit ? s0 + q : s;
          cum = c2;
        }
      }
      if (s < 0) {  // spill: clamp to the last positive sub-block
        s = last_pos;
        Ls_sel = w[s];
        wsel = ex2(Ls_sel - Li);
        before_s = cum - wsel;
      }
      float frac = wsel > 0.f ? (local - before_s) / wsel : 0.f;
      frac = fminf(fmaxf(frac, 0.f), 1.f);
      // recompute the sub-block's 64 weights (pass-1 pair arithmetic, two
      // columns per packed op; padding columns give 0): jsel = number of
      // prefix sums <= frac (the first prefix above frac), lastj = last
      // positive weight
      const float shift = Ls_sel - Brow;
      const int j0 = s * kSub;
      const float4* yb = ycol + j0 + s;
      const float2* ab = reinterpret_cast<const float2*>(Acol + j0 + s);
      const float ur[4] = {urow.x, urow.y, urow.z, urow.w};
      float2 uu[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) uu[q] = make_float2(ur[q], ur[q]);
      const float2 nsh = make_float2(-shift, -shift);
      float c3 = 0.f;
      int cnt = 0, lastj = 0;
#pragma unroll 8
      for (int q = 0; q < kSub; q += 2) {
        const float4 ya = yb[q], yc = yb[q + 1];
        const float2 a2 = (s & 1) ? make_float2(Acol[j0 + s + q], Acol[j0 + s + q + 1]) : ab[q >> 1];
        float2 t = __fadd2_rn(a2, nsh);
        t = __ffma2_rn(uu[0], make_float2(ya.x, yc.x), t);
        if (D > 1) t = __ffma2_rn(uu[1], make_float2(ya.y, yc.y), t);
        if (D > 2) t = __ffma2_rn(uu[2], make_float2(ya.z, yc.z), t);
        if (D > 3) t = __ffma2_rn(uu[3], make_float2(ya.w, yc.w), t);
        const float e0 = ex2(t.x), e1 = ex2(t.y);
        c3 += e0;
        cnt += c3 <= frac;
        c3 += e1;
        cnt += c3 <= frac;
        lastj = e0 > 0.f ? q : lastj;
        lastj = e1 > 0.f ? q + 1 : lastj;
      }
      const int jsel = cnt;
      const int j = j0 + (jsel < kSub ? (jsel <= lastj ? jsel : lastj) : lastj);
      PL[m + off] = (uint32_t)i;
      PR[m + off] = (uint32_t)j;
      la.first_next[nbase + m + off] = map_first(b, la, ch, L, (uint32_t)i);
      la.last_next[nbase + m + off] = map_last(b, la, ch, R, (uint32_t)j);
    }
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

// FP32 lazy samplers: the entry in log2 units in the unexpanded whitened
// form (accurate for any state), bound in log2 units.
template <int D>
__global__ void lazy32_kernel(Bufs b, LevelArgs la, int mh, size_t mh_steps) {
  const int k = la.k0 + blockIdx.y, ch = blockIdx.z;
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  const int N = b.N;
  Side L, R;
  CombineGeom g;
  sides(b, la, k, L, R, g);
  const TimeConst& tc = b.tc[(size_t)ch * b.Kt + b.t0 + g.c];
  CutConst32 cc;
  load_cut32<D>(tc, cc);
  const bool lnonuni = L.leaf && !b.UNI[(size_t)ch * b.K + L.t];
  const float4* XL = b.X32 + ((size_t)ch * b.K + L.t) * N;
  const float4* XR = b.X32 + ((size_t)ch * b.K + R.t) * N;
  const float* CR = b.COL + ((size_t)ch * b.K + R.t) * N;
  auto probe = [&](uint32_t i, uint32_t j) -> float {
    const uint32_t pi = map_last(b, la, ch, L, i);
    const uint32_t pj = map_first(b, la, ch, R, j);
    const float4 xl = XL[pi], xr = XR[pj];
    float mu[4], e[4];
    for (int q = 0; q < D; ++q) {
      float acc = cc.delta[q];
      for (int l = 0; l < D; ++l) acc = fmaf(cc.F[q * D + l], comp(xl, l), acc);
      mu[q] = acc;
    }
    for (int q = 0; q < D; ++q) e[q] = comp(xr, q) - mu[q];
    float qd = 0.f;
    for (int q = 0; q < D; ++q) {
      float z = 0.f;
      for (int l = 0; l <= q; ++l) z = fmaf(cc.W[q * D + l], e[l], z);
      qd = fmaf(z, z, qd);
    }
    float v = CR[pj] - qd;
    if (lnonuni) v += b.LW32[(size_t)ch * N + i];
    return v;
  };
  const size_t gidx = (size_t)ch * b.T + la.cursor + k;
  const int off = b.conditional ? 1 : 0;
  unsigned long long evals = 0;
  int err = 0, why = 0;
  if (m < la.n_out) {
    const uint64_t node = b.conditional
                              ? (static_cast<uint64_t>(static_cast<uint32_t>(k + la.node_off)) |
                                 (static_cast<uint64_t>(b.sweep) << 32))
                              : static_cast<uint64_t>(k + la.node_off);
    StreamReader s;
    s.init(stream_id(b.seeds[ch], la.key_level, node, DSMC_ROLE_PAIR_RESAMPLE, m + 1));
    uint32_t oi = 0, oj = 0;
    if (mh) {
      uint32_t i = (uint32_t)(m % N), j = i;
      float cur = 0.f;
      bool have = false;
      for (size_t st = 0; st < mh_steps; ++st) {
        const uint32_t pi = (uint32_t)s.index(N), pj = (uint32_t)s.index(N);
        const float lu = (float)(log2(s.uniform_pos()));
        if (!have) {
          cur = probe(i, j);
          ++evals;
          have = true;
        }
        const float prop = probe(pi, pj);
        ++evals;
        if (lu < prop - cur) {
          i = pi;
          j = pj;
          cur = prop;
        }
      }
      oi = i;
      oj = j;
    } else {
      if (!(b.bounded[ch] & 1)) { err = DSMC_E_INVALID_ARGUMENT; why = kReasonNoBound; }
      double bnd = tc.bound;
      if (lnonuni) bnd += b.LWMAX[(size_t)ch * b.K + L.t];
      const float bound2 = (float)(bnd * kLog2E);
      bool ok = false;
      for (uint64_t trial = 0; trial < (1u << 24) && !err; ++trial) {
        const uint32_t i = (uint32_t)s.index(N), j = (uint32_t)s.index(N);
        const float lw = probe(i, j);
        ++evals;
        if (isnan(lw) || lw - bound2 > 1e-3f) {
          err = DSMC_E_INVALID_ARGUMENT; why = isnan(lw) ? kReasonNaN : kReasonOverBound;
          break;
        }
        if ((float)log2(s.uniform_pos()) <= lw - bound2) {
          oi = i;
          oj = j;
          ok = true;
          break;
        }
      }
      if (!ok && !err) { err = DSMC_E_RUNTIME; why = kReasonTrialCap; }
    }
    b.PL[gidx * N + m + off] = oi;
    b.PR[gidx * N + m + off] = oj;
    if (err) raise_err(b.err, err, g.c, la.level, why);
  }
  for (int o = 16; o; o >>= 1) evals += __shfl_xor_sync(~0u, evals, o);
  if ((threadIdx.x & 31) == 0 && evals) atomicAdd(b.evals + ch, evals);
}

}  // namespace dsmc_dev

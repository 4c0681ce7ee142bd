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
// c32_pair (pass 1): ROW-STATIONARY. A CTA owns 256 rows of one combine, each
// lane 8 of them (u_i in registers, packed as row pairs); its warps stream the
// combine's 64-column sub-blocks through shared memory (one LDS.128 + one LDS
// per column, broadcast to the warp) and every lane accumulates its rows'
// sub-block sums of 2^(w - shift) in registers: per column and row pair one
// FFMA2 chain of d+1 (bias + d components), two MUFU.EX2 and one FADD2 — no
// max, no shuffles. The shift is the exact bound lw2_i + cmax_s (+ c_i for
// the few rows with |nu_i|^2 > 100), so exponents never overflow; a row whose
// sub-block sum underflows (< 2^-60) is recomputed with its exact max. At
// d = 1 (SV, Cox, theta-logistic: column terms spread over hundreds of
// log-units) each row's exact max per sub-block comes from a MUFU-free max
// pass instead, so no fallback is needed. Lane results L_is = log2 sum_{j in
// s} 2^w_ij are stored [sub-block][row] (coalesced). Nothing of the N x N
// table is stored beyond N*N/64 floats. (pair_tc.cuh: the same pass with the
// dot products on tcgen05, opt-in.)
//
// c32_sample (pass 2): one CTA per combine (or per slot slice): row totals
// from the sub-block sums, row CDF (double inclusive scan), per-slot binary
// search over rows, walk over the row's sub-blocks, and recomputation of <= 64
// weights with the same FP32 pair arithmetic.
#pragma once

#include "combine64.cuh"

namespace dsmc_dev {

constexpr int kRPL = 8;              // pass-1 rows per lane
constexpr int kRowsCTA = 32 * kRPL;  // pass-1 rows per CTA (256)
constexpr float kS = 0.84932180028801904272f;  // sqrt(log2(e) / 2)

struct CutConst32 {
  float W[16];   // s * tW (lower)
  float F[16];
  float delta[4];
  int drift;     // THETA: row mean = drift(x~ + m_{c-1}) - m_c
  float th[5];   // tau0, tau1, tau2, m_{c-1}, m_c
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
  cc.drift = tc.drift;
  for (int k = 0; k < 4; ++k) cc.th[k] = (float)tc.th[k];
  cc.th[4] = (float)tc.pm[0];
}
__device__ inline float comp(const float4& v, int k) {
  return k == 0 ? v.x : (k == 1 ? v.y : (k == 2 ? v.z : v.w));
}
// Centred transition mean of a left state x~ (the row term before whitening)
template <int D>
__device__ inline void row_mu32(const CutConst32& cc, float4 xv, float* mu) {
  if (cc.drift) {  // models.cpp:361-363 in absolute coordinates
    const float xa = xv.x + cc.th[3];
    mu[0] = xa + cc.th[0] - cc.th[1] * __expf(cc.th[2] * xa) - cc.th[4];
    return;
  }
#pragma unroll
  for (int k = 0; k < D; ++k) {
    float acc = cc.delta[k];
#pragma unroll
    for (int l = 0; l < D; ++l) acc = fmaf(cc.F[k * D + l], comp(xv, l), acc);
    mu[k] = acc;
  }
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
  row_mu32<D>(cc, xv, mu);
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

// Launched with programmatic stream serialization (engine.cu launch_pdl) a
// kernel may start while its predecessor drains; it waits here until that
// grid has completed and its memory is visible (a no-op otherwise).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
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

// Pass 1. Grid (row tiles x column splits, combines of the chunk, chains),
// 256 threads: rows [256 rt, 256 rt + 256), sub-blocks [cs nsub / ncs,
// (cs+1) nsub / ncs) of combine k, warps taking those sub-blocks round-robin.
constexpr int kPairWarps = 4;  // pass-1 warps per CTA (4 CTAs per SM)

template <int D>
__global__ void __launch_bounds__(32 * kPairWarps, 4) c32_pair(Bufs b, LevelArgs la) {
  pdl_wait();  // programmatic dependent launch: the previous kernel's writes
  __shared__ float4 s_u[kRowsCTA];          // u_i (2 nu_i), zero-padded to 4
  __shared__ float s_b[kRowsCTA];           // B_i
  __shared__ float s_c[kRowsCTA];           // overflow shift c_i (0 for most rows)
  __shared__ float4 s_y[kPairWarps][kSub];  // per warp: the staged sub-block's y_j
  __shared__ float s_a[kPairWarps][kSub];   // ... and A_j - cmax_s
  const int k = la.k0 + blockIdx.y, ch = blockIdx.z;
  const int N = b.N;
  const int nsub = (N + kSub - 1) / kSub;
  const int nrt = (N + kRowsCTA - 1) / kRowsCTA;
  const int rt = blockIdx.x % nrt, cs = blockIdx.x / nrt, ncs = gridDim.x / nrt;
  Side L, R;
  CombineGeom g;
  sides(b, la, k, L, R, g);
  const TimeConst& tc = b.tc[(size_t)ch * b.Kt + b.t0 + g.c];
  CutConst32 cc;
  load_cut32<D>(tc, cc);
  // per (chain, combine of the chunk) workspace, [sub-block][row]
  const size_t cslot = (size_t)blockIdx.z * gridDim.y + blockIdx.y;
  float* ws = reinterpret_cast<float*>(la.ws) + cslot * la.ws_comb * 2;
  const Aux32 ax = aux32(la, cslot, N);
  const int row0 = rt * kRowsCTA;
  const int nrows = min(kRowsCTA, N - row0);
  const bool lnonuni = L.leaf && !b.UNI[(size_t)ch * b.K + L.t];
  const float4* XL = b.X32 + ((size_t)ch * b.K + L.t) * N;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float4* XR = b.X32 + ((size_t)ch * b.K + R.t) * N;
  const float* CR = b.COL + ((size_t)ch * b.K + R.t) * N;
  const int sb0 = cs * nsub / ncs, sb1 = (cs + 1) * nsub / ncs;
  float4* sy = s_y[warp];
  float* sa = s_a[warp];
  // raw column data (leaf state + column term) of the lane's 2 columns of the
  // warp's next sub-block, loaded one sub-block ahead of its use; the first
  // sub-block's gathers are issued before the row prologue so both latencies
  // overlap
  float4 xr_n[2];
  float cr_n[2];
  auto fetch = [&](int sbk) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = sbk * kSub + lane + 32 * h;
      if (sbk < sb1 && j < N) {
        const uint32_t p = map_first(b, la, ch, R, j);
        xr_n[h] = XR[p];
        cr_n[h] = CR[p];
      }
    }
  };
  fetch(sb0 + warp);
  // row prologue: the CTA's rows (kRowsCTA / blockDim per thread), all
  // gathers issued before the arithmetic
  constexpr int RPT = kRowsCTA / (32 * kPairWarps);
  float4 xl[RPT];
  float lwr[RPT];
#pragma unroll
  for (int h = 0; h < RPT; ++h) {
    const int r = threadIdx.x + h * 32 * kPairWarps;
    xl[h] = make_float4(0.f, 0.f, 0.f, 0.f);
    lwr[h] = 0.f;
    if (r < nrows) {
      const int i = row0 + r;
      xl[h] = XL[map_last(b, la, ch, L, i)];
      if (lnonuni) lwr[h] = b.LW32[(size_t)ch * N + i];
    }
  }
#pragma unroll
  for (int h = 0; h < RPT; ++h) {
    const int r = threadIdx.x + h * 32 * kPairWarps;
    float u[4] = {0, 0, 0, 0}, Bv = -CUDART_INF_F;
    if (r < nrows) {
      const int i = row0 + r;
      row32<D>(cc, xl[h], lwr[h], u, Bv);
      if (cs == 0) {  // hand the row to the sampler
        ax.u[i] = make_float4(u[0], u[1], u[2], u[3]);
        ax.B[i] = Bv;
      }
    }
    s_u[r] = make_float4(u[0], u[1], u[2], u[3]);
    s_b[r] = Bv;
    float nn = 0.f;
#pragma unroll
    for (int q = 0; q < D; ++q) nn = fmaf(0.5f * u[q], 0.5f * u[q], nn);
    s_c[r] = nn > 100.f ? nn - 100.f : 0.f;
  }
  __syncthreads();
  // this lane's rows lane + 32 q, q = 0..7, as 4 row pairs (2p, 2p+1)
  constexpr int NPR = kRPL / 2;
  float2 U[4][NPR], NC[NPR];
#pragma unroll
  for (int pr = 0; pr < NPR; ++pr) {
    const float4 ua = s_u[lane + 64 * pr], ub = s_u[lane + 64 * pr + 32];
    U[0][pr] = make_float2(ua.x, ub.x);
    U[1][pr] = make_float2(ua.y, ub.y);
    U[2][pr] = make_float2(ua.z, ub.z);
    U[3][pr] = make_float2(ua.w, ub.w);
    NC[pr] = make_float2(-s_c[lane + 64 * pr], -s_c[lane + 64 * pr + 32]);
  }
  const float2 one2 = make_float2(1.f, 1.f);
  for (int sbk = sb0 + warp; sbk < sb1; sbk += kPairWarps) {
    // stage the sub-block's 64 columns (2 per lane), then prefetch the next
    float Ah[2], cm = -CUDART_INF_F;
    float4 xr_c[2] = {xr_n[0], xr_n[1]};
    float cr_c[2] = {cr_n[0], cr_n[1]};
    fetch(sbk + kPairWarps);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int jj = lane + 32 * h, j = sbk * kSub + jj;
      float y[4] = {0.f, 0.f, 0.f, 0.f};
      float A = -CUDART_INF_F;
      if (j < N) {
        const float cv = cr_c[h];
        col32<D>(cc, xr_c[h], cv, y, A);
        cm = fmaxf(cm, cv);
        if (rt == 0) {  // hand the column to the sampler
          ax.y[j] = make_float4(y[0], y[1], y[2], y[3]);
          ax.A[j] = A;
        }
      }
      sy[jj] = make_float4(y[0], y[1], y[2], y[3]);
      Ah[h] = A;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) cm = fmaxf(cm, __shfl_xor_sync(~0u, cm, o));
    const bool live = cm > -CUDART_INF_F;
#pragma unroll
    for (int h = 0; h < 2; ++h) sa[lane + 32 * h] = live ? Ah[h] - cm : -CUDART_INF_F;
    __syncwarp();
    if (D == 1) {
      // d = 1: the exact per-(row, sub-block) max as the shift, in a max-only
      // pass (one FFMA2 + one FMNMX3 per row pair and column, no MUFU) that
      // hides under the MUFU-bound sum pass of the other warps. The bound
      // shift is not enough here: column terms spread over hundreds of
      // log-units (e.g. stochastic volatility, Poisson counts), so far rows'
      // sums underflow and the per-row fallback below would run for most
      // warps. With the exact max every sum is >= 1.
      float2 M[NPR];
#pragma unroll
      for (int pr = 0; pr < NPR; ++pr) M[pr] = make_float2(-CUDART_INF_F, -CUDART_INF_F);
#pragma unroll 2
      for (int j = 0; j < kSub; j += 2) {
        const float y0 = sy[j].x, y1 = sy[j + 1].x, a0 = sa[j], a1 = sa[j + 1];
#pragma unroll
        for (int pr = 0; pr < NPR; ++pr) {
          const float2 t0 = __ffma2_rn(make_float2(y0, y0), U[0][pr], make_float2(a0, a0));
          const float2 t1 = __ffma2_rn(make_float2(y1, y1), U[0][pr], make_float2(a1, a1));
          M[pr].x = fmax3(M[pr].x, t0.x, t1.x);
          M[pr].y = fmax3(M[pr].y, t0.y, t1.y);
        }
      }
#pragma unroll
      for (int pr = 0; pr < NPR; ++pr)
        NC[pr] = make_float2(M[pr].x > -CUDART_INF_F ? -M[pr].x : 0.f,
                             M[pr].y > -CUDART_INF_F ? -M[pr].y : 0.f);
    }
    // S[pr] = sum_j 2^(A'_j + u.y_j - c) for the lane's row pair pr
    float2 S[NPR];
#pragma unroll
    for (int pr = 0; pr < NPR; ++pr) S[pr] = make_float2(0.f, 0.f);
#pragma unroll 2
    for (int j = 0; j < kSub; ++j) {
      const float4 yv = sy[j];
      const float a = sa[j];
#pragma unroll
      for (int pr = 0; pr < NPR; ++pr) {
        float2 t = __ffma2_rn(make_float2(a, a), one2, NC[pr]);
        t = __ffma2_rn(make_float2(yv.x, yv.x), U[0][pr], t);
        if (D > 1) t = __ffma2_rn(make_float2(yv.y, yv.y), U[1][pr], t);
        if (D > 2) t = __ffma2_rn(make_float2(yv.z, yv.z), U[2][pr], t);
        if (D > 3) t = __ffma2_rn(make_float2(yv.w, yv.w), U[3][pr], t);
        S[pr] = __fadd2_rn(S[pr], make_float2(ex2(t.x), ex2(t.y)));
      }
    }
    // L_is = log2 sum + c_i + cmax_s + B_i; underflowed rows: exact max
#pragma unroll
    for (int q = 0; q < kRPL; ++q) {
      const int r = lane + 32 * q;
      const float sq = (q & 1) ? S[q >> 1].y : S[q >> 1].x;
      if (r >= nrows) continue;
      float Ls;
      if (live && !(sq >= 0x1p-60f && sq <= 0x1p120f)) {
        const float4 u4 = s_u[r];
        const float uu[4] = {u4.x, u4.y, u4.z, u4.w};
        float m = -CUDART_INF_F;
        for (int j = 0; j < kSub; ++j) {
          const float4 yv = sy[j];
          const float yy[4] = {yv.x, yv.y, yv.z, yv.w};
          m = fmaxf(m, pair32<D>(uu, yy, sa[j]));
        }
        float acc = 0.f;
        if (m > -CUDART_INF_F)
          for (int j = 0; j < kSub; ++j) {
            const float4 yv = sy[j];
            const float yy[4] = {yv.x, yv.y, yv.z, yv.w};
            acc += ex2(pair32<D>(uu, yy, sa[j]) - m);
          }
        Ls = acc > 0.f ? m + lg2(acc) + cm + s_b[r] : -CUDART_INF_F;
      } else {
        const float shift = D == 1 ? -((q & 1) ? NC[q >> 1].y : NC[q >> 1].x) : s_c[r];
        Ls = sq > 0.f ? lg2(sq) + shift + cm + s_b[r] : -CUDART_INF_F;
      }
      ws[(size_t)sbk * N + row0 + r] = Ls;
    }
    __syncwarp();
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
// MINB: 4 (64 registers) wherever 4 CTAs fit in shared memory — N <= 1024
// since the slot records were compacted (C5 sampler 83.1 -> 77.4 ms; C4
// N = 512: 35.1 -> 34.1 ms/sweep) — else 3
template <int D, int MINB>
__global__ void __launch_bounds__(256, MINB) c32_sample(Bufs b, LevelArgs la,
                                                     int systematic) {
  pdl_wait();
  extern __shared__ double smem[];
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
  const Aux32 ax = aux32(la, cslot, N);
  // Columns are stored as PAIRS (2p, 2p+1) so the recompute's packed FFMA2 /
  // FADD2 take their operands straight from shared memory: P01[p] =
  // (y0_a, y0_b, y1_a, y1_b), P23[p] = (y2_a, y2_b, y3_a, y3_b), AP[p] =
  // (A_a, A_b). Pair p lives at p + p/32 (one pad entry per 64-column
  // sub-block): slots read pair 32 s + q of different sub-blocks s at the
  // same q, which without the skew all map to the same banks.
  const int NP = (N + kSub - 1) / kSub * kSub;
  const int NPP = NP / 2, NPS = NPP + NPP / 32;
  double* S = smem;                                            // N
  float4* P01 = reinterpret_cast<float4*>(S + ((N + 1) & ~1));   // NPS, 16B aligned
  float4* P23 = P01 + NPS;                                     // NPS
  float2* AP = reinterpret_cast<float2*>(P23 + NPS);            // NPS
  float* Lrow = reinterpret_cast<float*>(AP + NPS);             // N
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int pp = tid; pp < NPP; pp += blockDim.x) {
    const int j = 2 * pp;
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 ya = j < N ? ax.y[j] : z4, yb = j + 1 < N ? ax.y[j + 1] : z4;
    const float Aa = j < N ? ax.A[j] : -CUDART_INF_F, Ab = j + 1 < N ? ax.A[j + 1] : -CUDART_INF_F;
    const int ps = pp + pp / 32;
    P01[ps] = make_float4(ya.x, yb.x, ya.y, yb.y);
    P23[ps] = make_float4(ya.z, yb.z, ya.w, yb.w);
    AP[ps] = make_float2(Aa, Ab);
  }
  // row log2-totals: online LSE over the row's sub-block sums ([sub][row]
  // layout: coalesced across the threads' rows), 16 sub-blocks per round,
  // two rows in flight per thread
  float gm = -CUDART_INF_F;
  for (int i = tid; i < N; i += 2 * blockDim.x) {
    const int i2 = i + blockDim.x;
    float m[2] = {-CUDART_INF_F, -CUDART_INF_F}, acc[2] = {0.f, 0.f};
    // (a missing second row re-reads the first; its result is discarded)
    const float* w0 = ws + i;
    const float* w1 = ws + (i2 < N ? i2 : i);
    for (int s0 = 0; s0 < nsub; s0 += 16) {
      float v[2][16];
      if (s0 + 16 <= nsub) {  // whole round: unguarded loads, 32-bit offsets
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          v[0][q] = w0[(s0 + q) * N];
          v[1][q] = w1[(s0 + q) * N];
        }
      } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const bool in = s0 + q < nsub;
          v[0][q] = in ? w0[(s0 + q) * N] : -CUDART_INF_F;
          v[1][q] = in ? w1[(s0 + q) * N] : -CUDART_INF_F;
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float cm = fmax3(fmax3(v[h][0], v[h][1], v[h][2]), fmax3(v[h][3], v[h][4], v[h][5]),
                         fmax3(v[h][6], v[h][7], v[h][8]));
        cm = fmax3(cm, fmax3(v[h][9], v[h][10], v[h][11]),
                   fmax3(v[h][12], v[h][13], fmaxf(v[h][14], v[h][15])));
        if (cm == -CUDART_INF_F) continue;
        if (cm > m[h]) {
          acc[h] = m[h] == -CUDART_INF_F ? 0.f : acc[h] * ex2(m[h] - cm);
          m[h] = cm;
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) acc[h] += ex2(v[h][q] - m[h]);
      }
    }
    const float La = m[0] == -CUDART_INF_F ? -CUDART_INF_F : m[0] + lg2(acc[0]);
    const float Lc = m[1] == -CUDART_INF_F ? -CUDART_INF_F : m[1] + lg2(acc[1]);
    Lrow[i] = La;
    if (i2 < N) Lrow[i2] = Lc;
    gm = fmax3(gm, La, i2 < N ? Lc : -CUDART_INF_F);
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
  // Slots run in three phases, re-ordered in between by CTA counting sorts so
  // that each warp works on neighbouring data (shared-memory broadcasts
  // instead of bank conflicts). The order only schedules work: slot m always
  // uses u64 number m of the stream (rng.cpp:45-68) and writes output m.
  //   A  uniforms of the CTA's slots -> points pt_m; bucket by pt (32 buckets)
  //   B  in pt order: row search over the CDF, sub-block walk -> (i, s, frac)
  //   C  in sub-block order: recompute the 64 weights -> column j
  const int ns = max(0, m1 - m0);
  constexpr int NBA = 32;
  // offsets from the shared-memory base keep the compiler on LDS/STS
  const size_t ext = ((reinterpret_cast<char*>(Lrow + N) - reinterpret_cast<char*>(smem)) + 15) &
                     ~static_cast<size_t>(15);
  // slot records: key i | s << 16 and (frac, shift); slot orders as 16-bit
  // indices (ns <= 1024), the phase-C order over PT (dead after phase B) —
  // small enough for 4 CTAs per SM at N = 1024
  const int ns2 = (ns + 1) & ~1;
  double* PT = reinterpret_cast<double*>(reinterpret_cast<char*>(smem) + ext);  // [ns]
  int* RKEY = reinterpret_cast<int*>(PT + ns2);                                  // [ns]
  float2* RFS = reinterpret_cast<float2*>(RKEY + ns2);                          // [ns]
  uint16_t* ORD1 = reinterpret_cast<uint16_t*>(RFS + ns);                       // [ns]
  uint16_t* ORD2 = reinterpret_cast<uint16_t*>(PT);                             // [ns]
  int* CA = reinterpret_cast<int*>(ORD1 + ns2);                                 // [NBA]
  int* CB = CA + NBA;                                                           // [nsub]
  for (int q = tid; q < NBA; q += blockDim.x) CA[q] = 0;
  for (int q = tid; q < nsub; q += blockDim.x) CB[q] = 0;
  __syncthreads();
  const double bscale = (double)NBA / total;
  // phase A (each thread: 4 consecutive slots = one Philox block)
  for (int q0 = (m0 & ~3) + 4 * tid; q0 < m1; q0 += 4 * blockDim.x) {
    U64x4 blk;
    if (!systematic) blk = stream_block(id, (uint64_t)q0 >> 2);
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
      const int m = q0 + qq;
      if (m < m0 || m >= m1) continue;
      const double pt = systematic ? (u0 + (double)m) * step : u64_uniform(blk.v[qq]) * total;
      PT[m - m0] = pt;
      atomicAdd(&CA[min(NBA - 1, (int)(pt * bscale))], 1);
    }
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the 32 bucket counts
    const int c = CA[lane];
    int v = c;
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(~0u, v, o);
      if (lane >= o) v += n;
    }
    CA[lane] = v - c;
  }
  __syncthreads();
  for (int x = tid; x < ns; x += blockDim.x)
    ORD1[atomicAdd(&CA[min(NBA - 1, (int)(PT[x] * bscale))], 1)] = (uint16_t)x;
  __syncthreads();
  // phase B
  int steps = 0;
  while ((1 << steps) <= N) ++steps;
  for (int o = tid; o < ns; o += blockDim.x) {
    const int x = ORD1[o];
    const double pt = PT[x];
    int lo = 0, hi = N;
    for (int it = 0; it < steps; ++it) {
      const int mid = (lo + hi) >> 1;
      const bool act = lo < hi;
      const bool below = pt < S[min(mid, N - 1)];
      hi = act && below ? mid : hi;
      lo = act && !below ? mid + 1 : lo;
    }
    int i = lo < N ? lo : N - 1;
    const double before = i > 0 ? S[i - 1] : 0.0;
    while (i > 0 && !(Lrow[i] > -CUDART_INF_F)) --i;
    const float Li = Lrow[i];
    const float Brow = ax.B[i];
    // phase C reads this row's u_i: pull it into L1 now so the prefetch
    // there (one slot ahead) does not wait on L2
    asm volatile("prefetch.global.L1 [%0];" ::"l"(ax.u + i));
    const float local0 = (float)((pt - before) / (double)ex2(Li - G));
    const float local = local0 >= 0.f ? local0 : 0.f;
    // sub-block walk over the row's sub-block sums (relative to the row
    // total), branch-free, 16 at a time from vector loads
    const float* w = ws + i;  // sub-block s of row i at w[s * N]
    int s = -1, last_pos = 0;
    float cum = 0.f, before_s = 0.f, wsel = 0.f, Ls_sel = 0.f;
    for (int s0 = 0; s0 < nsub; s0 += 16) {
      float v[16];
      if (s0 + 16 <= nsub) {  // whole round: unguarded loads, 32-bit offsets
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = w[(s0 + q) * N];
      } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = (s0 + q < nsub) ? w[(s0 + q) * N] : -CUDART_INF_F;
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
      Ls_sel = w[(size_t)s * N];
      wsel = ex2(Ls_sel - Li);
      before_s = cum - wsel;
    }
    float frac = wsel > 0.f ? (local - before_s) / wsel : 0.f;
    frac = fminf(fmaxf(frac, 0.f), 1.f);
    // (i | s << 16, -, frac, shift); N < 2^16. The left block's first map at
    // i is read in phase C, where its latency hides under the recompute.
    RKEY[x] = i | (s << 16);
    RFS[x] = make_float2(frac, Brow - Ls_sel);
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
  for (int x = tid; x < ns; x += blockDim.x) ORD2[atomicAdd(&CB[RKEY[x] >> 16], 1)] = (uint16_t)x;
  __syncthreads();
  // phase C: recompute the sub-block's 64 weights with pass 1's pair
  // arithmetic, two columns per FFMA2 / FADD2 (padding columns give 0); the
  // column is the first whose prefix exceeds frac = the number of prefixes
  // <= frac. Warps hold slots of one sub-block: the pair loads broadcast.
  // the right block's last-map gather of slot o is stored one iteration
  // later, so its latency overlaps the next slot's recompute
  uint32_t* pend_dst = nullptr;
  uint32_t pend_src = 0;
  bool pend = false;
  // (the next slot's record and row vector are prefetched a slot ahead)
  int x_n = 0, key_n = 0;
  float2 fs_n = make_float2(0.f, 0.f);
  float4 u_n = make_float4(0.f, 0.f, 0.f, 0.f);
  if (tid < ns) {
    x_n = ORD2[tid];
    key_n = RKEY[x_n];
    fs_n = RFS[x_n];
    u_n = ax.u[key_n & 0xffff];
  }
  for (int o = tid; o < ns; o += blockDim.x) {
    const int x = x_n, key = key_n;
    const float2 fs = fs_n;
    const float4 urow = u_n;
    if (o + (int)blockDim.x < ns) {
      x_n = ORD2[o + blockDim.x];
      key_n = RKEY[x_n];
      fs_n = RFS[x_n];
      u_n = ax.u[key_n & 0xffff];
    }
    const int i = key & 0xffff, s = key >> 16;
    const uint32_t first_i = map_first(b, la, ch, L, (uint32_t)i);  // used at the end
    const float frac = fs.x;
    const float sh = fs.y;
    const float2 nsh = make_float2(sh, sh);
    const float2 uu0 = make_float2(urow.x, urow.x), uu1 = make_float2(urow.y, urow.y);
    const float2 uu2 = make_float2(urow.z, urow.z), uu3 = make_float2(urow.w, urow.w);
    const int pb = s * 33;  // skewed first pair of sub-block s
    float c3 = 0.f;
    int cnt = 0;
#pragma unroll 8
    for (int q = 0; q < kSub / 2; ++q) {
      float2 t = __fadd2_rn(AP[pb + q], nsh);
      const float4 c01 = P01[pb + q];
      t = __ffma2_rn(uu0, make_float2(c01.x, c01.y), t);
      if (D > 1) t = __ffma2_rn(uu1, make_float2(c01.z, c01.w), t);
      if (D > 2) {
        const float4 c23 = P23[pb + q];
        t = __ffma2_rn(uu2, make_float2(c23.x, c23.y), t);
        if (D > 3) t = __ffma2_rn(uu3, make_float2(c23.z, c23.w), t);
      }
      c3 += ex2(t.x);
      cnt += c3 <= frac;
      c3 += ex2(t.y);
      cnt += c3 <= frac;
    }
    int jl = cnt;
    if (cnt >= kSub) {  // spill (rounding): the last positive weight
      jl = 0;
      for (int q = 0; q < kSub / 2; ++q) {
        float2 t = __fadd2_rn(AP[pb + q], nsh);
        const float4 c01 = P01[pb + q];
        t = __ffma2_rn(uu0, make_float2(c01.x, c01.y), t);
        if (D > 1) t = __ffma2_rn(uu1, make_float2(c01.z, c01.w), t);
        if (D > 2) {
          const float4 c23 = P23[pb + q];
          t = __ffma2_rn(uu2, make_float2(c23.x, c23.y), t);
          if (D > 3) t = __ffma2_rn(uu3, make_float2(c23.z, c23.w), t);
        }
        jl = ex2(t.x) > 0.f ? 2 * q : jl;
        jl = ex2(t.y) > 0.f ? 2 * q + 1 : jl;
      }
    }
    const int j = s * kSub + jl;
    const int m = m0 + x;
    PL[m + off] = (uint32_t)i;
    PR[m + off] = (uint32_t)j;
    la.first_next[nbase + m + off] = first_i;
    if (pend) *pend_dst = pend_src;
    pend_src = map_last(b, la, ch, R, (uint32_t)j);
    pend_dst = la.last_next + nbase + m + off;
    pend = true;
  }
  if (pend) *pend_dst = pend_src;
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

#ifndef DSMC_MH_BATCH
#define DSMC_MH_BATCH 8
#endif
constexpr int kMhBatch = DSMC_MH_BATCH;  // MH steps per batch (a multiple of 4)
static_assert(kMhBatch % 4 == 0, "whole Philox blocks per batch");
__device__ __forceinline__ bool lazy_serial_mh() {
#ifdef DSMC_LAZY_SERIAL
  return true;
#else
  return false;
#endif
}

// FP32 lazy samplers: the entry in log2 units in the unexpanded whitened
// form (accurate for any state), bound in log2 units.
// MH and rejection are separate instantiations (their batches need
// different register budgets).
template <int D, bool MH>
__global__ void lazy32_kernel(Bufs b, LevelArgs la, size_t mh_steps) {
  constexpr bool mh = MH;
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
    row_mu32<D>(cc, xl, mu);
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
    if constexpr (mh) {
      uint32_t i = (uint32_t)(m % N), j = i;
      float cur = 0.f;
      bool have = false;
      // Each MH step draws exactly 3 u64 (two indices, one uniform;
      // resampling.cpp:258-275), so kMhBatch = 8 steps are 6 whole Philox
      // blocks and their draws and proposal probes do not depend on the chain
      // state: generate and probe 8 steps at once (8 independent gather
      // chains in flight), then apply the 8 accept decisions in order.
      // Bit-identical to the step-by-step loop below, which finishes any
      // remainder (tools/lazy_ab.py; C3 68.2 -> 57.2 ms/step, batches of 4 /
      // 12 / 16: 61.8 / 70.8 / 70.5 ms, profiles/r02f_lazy_batch.md).
      size_t st = 0;
      constexpr int MB = kMhBatch, NBLK = 3 * MB / 4;
      if (!lazy_serial_mh() && mh_steps >= (size_t)MB) {  // (0 steps: no probe at all)
        cur = probe(i, j);
        ++evals;
        have = true;
        for (; st + MB <= mh_steps; st += MB) {
          uint32_t pi[MB], pj[MB];
          float lu[MB], prop[MB];
          draw_batch<MB>(s.id, NBLK * (st / MB), N, pi, pj, lu,
                         [](uint64_t v) { return lg2((float)u64_uniform_pos(v)); });
#pragma unroll
          for (int q = 0; q < MB; ++q) prop[q] = probe(pi[q], pj[q]);
          evals += MB;
#pragma unroll
          for (int q = 0; q < MB; ++q) {
            if (lu[q] < prop[q] - cur) {
              i = pi[q];
              j = pj[q];
              cur = prop[q];
            }
          }
        }
        s.blk = 3 * (st / 4);  // the remainder continues the stream (MB | st)
        s.pos = 4;
      }
      for (; st < mh_steps; ++st) {
        const uint32_t pi = (uint32_t)s.index(N), pj = (uint32_t)s.index(N);
        const float lu = lg2((float)s.uniform_pos());  // FP32 path: MUFU, not FP64 log2
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
      // trials also draw exactly 3 u64 each (i, j, then the uniform): the
      // same batching as MH, the trials after the first accepted (or
      // failing) one of a batch are evaluated but neither counted nor used
      constexpr int MB = kMhBatch, NBLK = 3 * MB / 4;
      uint64_t trial = 0;
      for (; !lazy_serial_mh() && trial < (1u << 24) && !err && !ok; trial += MB) {
        uint32_t pi[MB], pj[MB];
        float lu[MB], lw[MB];
        draw_batch<MB>(s.id, NBLK * (trial / MB), N, pi, pj, lu,
                       [](uint64_t v) { return lg2((float)u64_uniform_pos(v)); });
#pragma unroll
        for (int q = 0; q < MB; ++q) lw[q] = probe(pi[q], pj[q]);
#pragma unroll
        for (int q = 0; q < MB; ++q) {
          if (ok || err) continue;
          ++evals;
          if (isnan(lw[q]) || lw[q] - bound2 > 1e-3f) {
            err = DSMC_E_INVALID_ARGUMENT; why = isnan(lw[q]) ? kReasonNaN : kReasonOverBound;
          } else if (lu[q] <= lw[q] - bound2) {
            oi = pi[q];
            oj = pj[q];
            ok = true;
          }
        }
      }
      for (; lazy_serial_mh() && trial < (1u << 24) && !err; ++trial) {
        const uint32_t i = (uint32_t)s.index(N), j = (uint32_t)s.index(N);
        const float lw = probe(i, j);
        ++evals;
        if (isnan(lw) || lw - bound2 > 1e-3f) {
          err = DSMC_E_INVALID_ARGUMENT; why = isnan(lw) ? kReasonNaN : kReasonOverBound;
          break;
        }
        if (lg2((float)s.uniform_pos()) <= lw - bound2) {
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

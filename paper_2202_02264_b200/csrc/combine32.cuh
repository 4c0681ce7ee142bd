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

template <int D>
__global__ void __launch_bounds__(256, 2) c32_pair(Bufs b, LevelArgs la) {
  __shared__ float s_u[kRT][4];
  __shared__ float s_B[kRT];
  const int k = la.k0 + blockIdx.y, ch = blockIdx.z;
  const int N = b.N;
  Side L, R;
  CombineGeom g;
  sides(b, la, k, L, R, g);
  const TimeConst& tc = b.tc[(size_t)ch * b.K + g.c];
  CutConst32 cc;
  load_cut32<D>(tc, cc);
  const int nch = (N + kChunk - 1) / kChunk;
  const int nsubp = nch * (kChunk / kSub);
  float* ws = reinterpret_cast<float*>(la.ws) + (size_t)blockIdx.y * la.ws_comb * 2;
  const int row0 = blockIdx.x * kRT;
  const int nrows = min(kRT, N - row0);
  // rows of this tile -> shared memory
  const bool lnonuni = L.leaf && !b.UNI[(size_t)ch * b.K + L.t];
  const float4* XL = b.X32 + ((size_t)ch * b.K + L.t) * N;
  for (int r = threadIdx.x; r < nrows; r += blockDim.x) {
    const int i = row0 + r;
    const uint32_t p = map_last(b, la, ch, L, i);
    const float lw2 = lnonuni ? b.LW32[(size_t)ch * N + i] : 0.f;
    float u[4] = {0, 0, 0, 0}, Bv;
    row32<D>(cc, XL[p], lw2, u, Bv);
    for (int q = 0; q < 4; ++q) s_u[r][q] = u[q];
    s_B[r] = Bv;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = max(1, 8 / nch);          // row slices per chunk
  const int items = nch * S;
  const float4* XR = b.X32 + ((size_t)ch * b.K + R.t) * N;
  const float* CR = b.COL + ((size_t)ch * b.K + R.t) * N;
  for (int it = warp; it < items; it += 8) {
    const int chunk = it % nch, slice = it / nch;
    // this lane's 16 columns -> registers (packed pairs)
    float2 y2[D][kCPL / 2];
    float2 A2[kCPL / 2];
#pragma unroll
    for (int c2 = 0; c2 < kCPL / 2; ++c2) {
      float yv[2][4], Av[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = chunk * kChunk + lane * kCPL + 2 * c2 + h;
        if (j < N) {
          const uint32_t p = map_first(b, la, ch, R, j);
          col32<D>(cc, XR[p], CR[p], yv[h], Av[h]);
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
    float* wrow_base = ws + (size_t)row0 * nsubp + chunk * (kChunk / kSub) + (lane >> 2);
    for (int r = slice; r < nrows; r += S) {
      float2 t[kCPL / 2];
      float2 uu[D];
#pragma unroll
      for (int q = 0; q < D; ++q) uu[q] = make_float2(s_u[r][q], s_u[r][q]);
#pragma unroll
      for (int c2 = 0; c2 < kCPL / 2; ++c2) {
        float2 acc = A2[c2];
#pragma unroll
        for (int q = 0; q < D; ++q) acc = __ffma2_rn(uu[q], y2[q][c2], acc);
        t[c2] = acc;
      }
      float m = fmaxf(t[0].x, t[0].y);
#pragma unroll
      for (int c2 = 1; c2 < kCPL / 2; ++c2) m = fmaxf(m, fmaxf(t[c2].x, t[c2].y));
      m = fmaxf(m, __shfl_xor_sync(~0u, m, 1));
      m = fmaxf(m, __shfl_xor_sync(~0u, m, 2));
      const float mm = (m == -CUDART_INF_F) ? 0.f : m;
      const float2 nm = make_float2(-mm, -mm);
      float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
      for (int c2 = 0; c2 < kCPL / 2; ++c2) {
        const float2 dd = __fadd2_rn(t[c2], nm);
        s2 = __fadd2_rn(s2, make_float2(ex2(dd.x), ex2(dd.y)));
      }
      float s = s2.x + s2.y;
      s += __shfl_xor_sync(~0u, s, 1);
      s += __shfl_xor_sync(~0u, s, 2);
      if ((lane & 3) == 0) {
        const float Ls = s > 0.f ? m + lg2(s) + s_B[r] : -CUDART_INF_F;
        wrow_base[(size_t)r * nsubp] = Ls;
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

template <int D>
__global__ void __launch_bounds__(512) c32_sample(Bufs b, LevelArgs la,
                                                  int systematic) {
  extern __shared__ double smem[];
  __shared__ double sh[32];
  __shared__ float s_g;
  const int k = la.k0 + blockIdx.x, ch = blockIdx.z;
  const int N = b.N;
  Side L, R;
  CombineGeom g;
  sides(b, la, k, L, R, g);
  const TimeConst& tc = b.tc[(size_t)ch * b.K + g.c];
  CutConst32 cc;
  load_cut32<D>(tc, cc);
  const int nch = (N + kChunk - 1) / kChunk;
  const int nsubp = nch * (kChunk / kSub);
  const int nsub = (N + kSub - 1) / kSub;
  const float* ws = reinterpret_cast<const float*>(la.ws) + (size_t)blockIdx.x * la.ws_comb * 2;
  double* S = smem;                                   // N
  float* Lrow = reinterpret_cast<float*>(S + N);      // N
  float* ycol = Lrow + N;                             // N*D
  float* Acol = ycol + (size_t)N * D;                 // N
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float4* XR = b.X32 + ((size_t)ch * b.K + R.t) * N;
  const float* CR = b.COL + ((size_t)ch * b.K + R.t) * N;
  for (int j = tid; j < N; j += blockDim.x) {
    const uint32_t p = map_first(b, la, ch, R, j);
    float y[4], A;
    col32<D>(cc, XR[p], CR[p], y, A);
    for (int q = 0; q < D; ++q) ycol[(size_t)j * D + q] = y[q];
    Acol[j] = A;
  }
  // row totals (log2) from the sub-block sums
  float gm = -CUDART_INF_F;
  for (int i = tid; i < N; i += blockDim.x) {
    const float* w = ws + (size_t)i * nsubp;
    float m = -CUDART_INF_F;
    for (int s = 0; s < nsub; ++s) m = fmaxf(m, w[s]);
    float L2 = -CUDART_INF_F;
    if (m != -CUDART_INF_F) {
      float acc = 0.f;
      for (int s = 0; s < nsub; ++s) acc += ex2(w[s] - m);
      L2 = m + lg2(acc);
    }
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
    if (tid == 0) raise_err(b.err, DSMC_E_RUNTIME, g.c, la.level, kReasonZeroTable);
    return;
  }
  // row CDF: each thread scans a contiguous segment, then a block scan
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
  if (tid == 0) b.LMW[gidx] = ((double)G + log2(total)) * kLn2;
  const bool lnonuni = L.leaf && !b.UNI[(size_t)ch * b.K + L.t];
  const float4* XL = b.X32 + ((size_t)ch * b.K + L.t) * N;
  const int off = b.conditional ? 1 : 0;
  const uint64_t node = b.conditional
                            ? (static_cast<uint64_t>(static_cast<uint32_t>(k)) |
                               (static_cast<uint64_t>(b.sweep) << 32))
                            : static_cast<uint64_t>(k);
  const StreamId id = stream_id(b.seeds[ch], la.level, node, DSMC_ROLE_PAIR_RESAMPLE, 0);
  double u0 = 0.0, step = 0.0;
  if (systematic) {
    u0 = u64_uniform(stream_u64(id, 0));
    step = total / (double)la.n_out;
  }
  uint32_t* PL = b.PL + gidx * N;
  uint32_t* PR = b.PR + gidx * N;
  for (int m = tid; m < la.n_out; m += blockDim.x) {
    const double pt = systematic ? (u0 + (double)m) * step
                                 : u64_uniform(stream_u64(id, m)) * total;
    int lo = 0, hi = N;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (pt < S[mid]) hi = mid;
      else lo = mid + 1;
    }
    int i = lo < N ? lo : N - 1;
    const double before = i > 0 ? S[i - 1] : 0.0;
    while (i > 0 && !(Lrow[i] > -CUDART_INF_F)) --i;
    const double ri = (double)ex2(Lrow[i] - G);
    float local = (float)((pt - before) / ri);
    if (!(local >= 0.f)) local = 0.f;
    // sub-block walk (weights relative to the row total)
    const float* w = ws + (size_t)i * nsubp;
    const float Li = Lrow[i];
    int s = 0;
    float cum = 0.f, before_s = 0.f;
    int last_pos = 0;
    for (; s < nsub; ++s) {
      const float ws_ = ex2(w[s] - Li);
      if (ws_ > 0.f) last_pos = s;
      before_s = cum;
      cum += ws_;
      if (local < cum) break;
    }
    if (s == nsub) {
      s = last_pos;
      before_s = cum - ex2(w[s] - Li);
    }
    const float wsub = ex2(w[s] - Li);
    float frac = wsub > 0.f ? (local - before_s) / wsub : 0.f;
    frac = fminf(fmaxf(frac, 0.f), 1.f);
    // recompute the sub-block's weights (row-local, shifted by its log-sum)
    const uint32_t p = map_last(b, la, ch, L, i);
    const float lw2 = lnonuni ? b.LW32[(size_t)ch * N + i] : 0.f;
    float u[4] = {0, 0, 0, 0}, Bv;
    row32<D>(cc, XL[p], lw2, u, Bv);
    const float shift = w[s] - Bv;
    const int j0 = s * kSub, j1 = min(j0 + kSub, N);
    float c3 = 0.f;
    int j = j0, lastj = j0;
    for (; j < j1; ++j) {
      const float e = ex2(pair32<D>(u, ycol + (size_t)j * D, Acol[j]) - shift);
      if (e > 0.f) lastj = j;
      c3 += e;
      if (frac < c3) break;
    }
    if (j == j1) j = lastj;
    PL[m + off] = (uint32_t)i;
    PR[m + off] = (uint32_t)j;
  }
  if (b.conditional && tid == 0) {
    PL[0] = 0;
    PR[0] = 0;
  }
  __syncthreads();
  const size_t nbase = ((size_t)ch * b.cap + k) * N;
  for (int q = tid; q < N; q += blockDim.x) {
    la.first_next[nbase + q] = map_first(b, la, ch, L, PL[q]);
    la.last_next[nbase + q] = map_last(b, la, ch, R, PR[q]);
  }
  if (tid == 0) {
    const double logn = log((double)N);
    const bool luni = !L.leaf || b.UNI[(size_t)ch * b.K + L.t];
    const bool runi = !R.leaf || b.UNI[(size_t)ch * b.K + R.t];
    const double shift = (luni ? -logn : 0.0) + (runi ? -logn : 0.0);
    const double ll = block_lnc(b, la, ch, L, g.a);
    const double rl = block_lnc(b, la, ch, R, g.c);
    la.blnc_next[(size_t)ch * b.cap + k] = ll + rl + b.LMW[gidx] + shift;
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
  const TimeConst& tc = b.tc[(size_t)ch * b.K + g.c];
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
                              ? (static_cast<uint64_t>(static_cast<uint32_t>(k)) |
                                 (static_cast<uint64_t>(b.sweep) << 32))
                              : static_cast<uint64_t>(k);
    StreamReader s;
    s.init(stream_id(b.seeds[ch], la.level, node, DSMC_ROLE_PAIR_RESAMPLE, m + 1));
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

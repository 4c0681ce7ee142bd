// FP32 dense combine for small N (N <= kSmallN): one CTA per combine does
// pass 1 and pass 2 of c32_pair / c32_sample in a single launch. At C1
// (K = 2^10, N = 100) every level is a few microseconds of dependent global
// round trips, so each of c32_pair / c32_sample costs ~10 us per level
// whatever the level's size; here the row and column gathers of a combine run
// once, side by side, and the table never leaves the SM.
//
// Thread t owns row t and column t. Row t's exact max over the columns, then
// its log2 total L_t = m_t + B_t + log2 sum_j 2^(A_j + u_t . y_j - m_t); row
// CDF over exp2(L_t - max L) in FP64; slot m (u64 number m of the stream,
// rng.cpp:45-68) searches the row, then walks the row's weights recomputed
// with the same arithmetic. Same pair weights and law as the two-kernel path
// (pass 1 / pass 2 differ only in FP32 rounding order).
#pragma once

#include "combine32.cuh"

namespace dsmc_dev {

constexpr int kSmallN = 128;

template <int D>
__global__ void __launch_bounds__(kSmallN) c32_small(Bufs b, LevelArgs la, int systematic) {
  pdl_wait();
  __shared__ float4 sy[kSmallN], su[kSmallN];
  __shared__ float sa[kSmallN], sm[kSmallN], ss[kSmallN], sL[kSmallN];
  __shared__ double S[kSmallN], sh[32];
  __shared__ CutConst32 s_cc;
  __shared__ float s_g;
  const int k = la.k0 + blockIdx.x, ch = blockIdx.z;
  const int N = b.N, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  Side L, R;
  CombineGeom g;
  sides(b, la, k, L, R, g);
  if (t == 0) load_cut32<D>(b.tc[(size_t)ch * b.Kt + b.t0 + g.c], s_cc);
  const bool lnonuni = L.leaf && !b.UNI[(size_t)ch * b.K + L.t];
  // both gathers in flight before any arithmetic
  float4 xc = make_float4(0.f, 0.f, 0.f, 0.f), xl = xc;
  float col = -CUDART_INF_F, lwr = 0.f;
  if (t < N) {
    const uint32_t pc = map_first(b, la, ch, R, t), pr = map_last(b, la, ch, L, t);
    const size_t oc = ((size_t)ch * b.K + R.t) * N + pc;
    xc = b.X32[oc];
    col = b.COL[oc];
    xl = b.X32[((size_t)ch * b.K + L.t) * N + pr];
    if (lnonuni) lwr = b.LW32[(size_t)ch * N + t];
  }
  __syncthreads();  // s_cc
  const CutConst32& cc = s_cc;
  float u[4] = {0.f, 0.f, 0.f, 0.f}, Bv = -CUDART_INF_F;
  if (t < N) {
    float y[4] = {0.f, 0.f, 0.f, 0.f}, A = -CUDART_INF_F;
    col32<D>(cc, xc, col, y, A);
    bool live = A > -CUDART_INF_F;
#pragma unroll
    for (int c = 0; c < D; ++c) live = live && isfinite(y[c]);
    if (!live) {
      A = -CUDART_INF_F;
#pragma unroll
      for (int c = 0; c < 4; ++c) y[c] = 0.f;
    }
    sy[t] = make_float4(y[0], y[1], y[2], y[3]);
    sa[t] = A;
    row32<D>(cc, xl, lwr, u, Bv);
    bool fin = Bv > -CUDART_INF_F;
#pragma unroll
    for (int c = 0; c < D; ++c) fin = fin && isfinite(u[c]);
    if (!fin) {
      Bv = -CUDART_INF_F;
#pragma unroll
      for (int c = 0; c < 4; ++c) u[c] = 0.f;
    }
    su[t] = make_float4(u[0], u[1], u[2], u[3]);
  }
  __syncthreads();
  // row t: exact max, then the log2 total
  float Lt = -CUDART_INF_F;
  if (t < N) {
    float m = -CUDART_INF_F;
    for (int j = 0; j < N; ++j) {
      const float4 yv = sy[j];
      const float yy[4] = {yv.x, yv.y, yv.z, yv.w};
      m = fmaxf(m, pair32<D>(u, yy, sa[j]));
    }
    float acc = 0.f;
    if (m > -CUDART_INF_F && Bv > -CUDART_INF_F)
      for (int j = 0; j < N; ++j) {
        const float4 yv = sy[j];
        const float yy[4] = {yv.x, yv.y, yv.z, yv.w};
        acc += ex2(pair32<D>(u, yy, sa[j]) - m);
      }
    Lt = acc > 0.f ? m + Bv + lg2(acc) : -CUDART_INF_F;
    sm[t] = m;
    ss[t] = acc;
    sL[t] = Lt;
  }
  float gm = Lt;
  for (int o = 16; o; o >>= 1) gm = fmaxf(gm, __shfl_xor_sync(~0u, gm, o));
  if (lane == 0) sh[warp] = gm;
  __syncthreads();
  if (t == 0) {
    float v = -CUDART_INF_F;
    for (int w = 0; w < kSmallN / 32; ++w) v = fmaxf(v, (float)sh[w]);
    s_g = v;
  }
  __syncthreads();
  const float G = s_g;
  if (G == -CUDART_INF_F) {
    if (t == 0) raise_err(b.err, DSMC_E_RUNTIME, g.c, la.level, kReasonZeroTable);
    return;
  }
  const double rt = t < N ? (double)ex2(Lt - G) : 0.0;
  S[t] = block_scan_incl(rt, sh);
  __syncthreads();
  const double total = S[N - 1];
  const size_t gidx = (size_t)ch * b.T + la.cursor + k;
  if (t == 0) b.LMW[gidx] = ((double)G + log2(total)) * kLn2;
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
  for (int m = t; m < la.n_out; m += blockDim.x) {
    const double pt = systematic ? (u0 + (double)m) * step : u64_uniform(stream_u64(id, m)) * total;
    int lo = 0, hi = N;  // first row with pt < S_i
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (pt < S[mid]) hi = mid;
      else lo = mid + 1;
    }
    int i = lo < N ? lo : N - 1;
    const double before = i > 0 ? S[i - 1] : 0.0;  // (as c32_sample)
    while (i > 0 && !(sL[i] > -CUDART_INF_F)) --i;
    // the target inside row i in units of its weights 2^(w - m_i)
    float frac = (float)((pt - before) / (double)ex2(sL[i] - G));
    frac = fminf(fmaxf(frac, 0.f), 1.f);
    const float target = frac * ss[i];
    const float4 uv = su[i];
    const float uu[4] = {uv.x, uv.y, uv.z, uv.w};
    const float mi = sm[i];
    float c3 = 0.f;
    int j = -1, last = 0;
    for (int q = 0; q < N; ++q) {
      const float4 yv = sy[q];
      const float yy[4] = {yv.x, yv.y, yv.z, yv.w};
      const float e = ex2(pair32<D>(uu, yy, sa[q]) - mi);
      c3 += e;
      last = e > 0.f ? q : last;
      if (j < 0 && target < c3) j = q;
    }
    if (j < 0) j = last;  // rounding spill: the last positive weight
    PL[m + off] = (uint32_t)i;
    PR[m + off] = (uint32_t)j;
    la.first_next[nbase + m + off] = map_first(b, la, ch, L, (uint32_t)i);
    la.last_next[nbase + m + off] = map_last(b, la, ch, R, (uint32_t)j);
  }
  if (b.conditional && t == 0) {
    PL[0] = 0;
    PR[0] = 0;
    la.first_next[nbase] = map_first(b, la, ch, L, 0);
    la.last_next[nbase] = map_last(b, la, ch, R, 0);
  }
  if (t == 0) {
    const double logn = log((double)N);
    const bool luni = !L.leaf || b.UNI[(size_t)ch * b.K + L.t];
    const bool runi = !R.leaf || b.UNI[(size_t)ch * b.K + R.t];
    const double shift = (luni ? -logn : 0.0) + (runi ? -logn : 0.0);
    const double ll = block_lnc(b, la, ch, L, g.a);
    const double rl = block_lnc(b, la, ch, R, g.c);
    la.blnc_next[(size_t)ch * b.cap + k] = ll + rl + ((double)G + log2(total)) * kLn2 + shift;
  }
}

}  // namespace dsmc_dev

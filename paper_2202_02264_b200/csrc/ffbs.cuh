// Sequential baseline on the device: particle filter + forward-filtering
// backward-sampling (run_particle_filter / ffbs_sample, baselines.cpp:36-160),
// FP32, the comparator of the paper's Fig. 2. The proposals of every time are
// drawn up front by leaf32_kernel with the filter's stream role
// ({seed, 0, t, filter_step}, baselines.cpp:17-20) — they do not depend on
// the ancestors — so only resample + reweight + normalise is sequential in t:
// one persistent CTA walks the T steps. The backward pass gives each draw its
// own warp; draws are independent across times, so a persistent grid walks
// t = T-1..0 with only CTA-local synchronisation (the CTA stages slab t's
// transition means once for its 8 warps).
//
// A weight in log2 units reuses the pair-kernel terms of the cut into t:
//   w(x_{t-1} -> x_t) = COL_t(x_t) - |y(x_t) - nu(x_{t-1})|^2
// = log2e (log h_t - log q_t + log p_t(x_t | x_{t-1})).
#pragma once

#include "compose.cuh"

namespace dsmc_dev {

// Per-slot categorical draw from an inclusive double CDF (first i with
// pt < S_i, clamped; dead entries are skipped backwards).
__device__ inline int cdf_search(const double* S, int n, double pt) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (pt < S[mid]) hi = mid;
    else lo = mid + 1;
  }
  int i = lo < n ? lo : n - 1;
  while (i > 0 && !(S[i] > S[i - 1])) --i;
  return i;
}

// Forward pass, one CTA per chain (blockDim >= 32, any N). LW: [K][N]
// normalised log2 weights (row 0 from leafnorm32 via b.LW32), ANC: [T][N].
template <int D>
__global__ void __launch_bounds__(512) pf_forward_kernel(Bufs b, float* LW, uint32_t* ANC,
                                                          int systematic, double* loglik) {
  extern __shared__ double sm_pf[];
  __shared__ double sh[32];
  __shared__ float s_red[32];
  const int N = b.N, K = b.K, ch = 0;
  double* S = sm_pf;  // [N] CDF of the previous weights
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int i = tid; i < N; i += blockDim.x) LW[i] = b.LW32[i];
  double ll = tid == 0 ? b.LNC[0] : 0.0;  // leaf 0: LSE - log N
  __syncthreads();
  const int per = (N + blockDim.x - 1) / blockDim.x;
  for (int t = 1; t < K; ++t) {
    const float* lwp = LW + (size_t)(t - 1) * N;
    // CDF of the previous (normalised) weights
    const int i0 = tid * per, i1 = min(N, i0 + per);
    double seg = 0.0;
    for (int i = i0; i < i1; ++i) seg += (double)ex2(lwp[i]);
    const double incl = block_scan_incl(seg, sh);
    double run = incl - seg;
    for (int i = i0; i < i1; ++i) {
      run += (double)ex2(lwp[i]);
      S[i] = run;
    }
    __syncthreads();
    const double total = S[N - 1];
    const StreamId rid = stream_id(b.seeds[ch], 1, (uint64_t)t, DSMC_ROLE_FILTER_STEP, 0);
    double u0 = 0.0;
    if (systematic) u0 = u64_uniform(stream_u64(rid, 0));
    const TimeConst& tc = b.tc[(size_t)ch * b.Kt + b.t0 + t];
    CutConst32 cc;
    load_cut32<D>(tc, cc);
    const float4* XP = b.X32 + (size_t)(t - 1) * N;
    const float4* XC = b.X32 + (size_t)t * N;
    const float* CC = b.COL + (size_t)t * N;
    float* lw = LW + (size_t)t * N;
    uint32_t* anc = ANC + (size_t)(t - 1) * N;
    float mx = -CUDART_INF_F;
    for (int m = tid; m < N; m += blockDim.x) {
      const double pt = systematic ? (u0 + (double)m) * (total / (double)N)
                                   : u64_uniform(stream_u64(rid, (uint64_t)m)) * total;
      const int a = cdf_search(S, N, pt);
      anc[m] = (uint32_t)a;
      float mu[4], y[4], A;
      row_mu32<D>(cc, XP[a], mu);
      float nu[4];
#pragma unroll
      for (int k = 0; k < D; ++k) {
        float acc = 0.f;
#pragma unroll
        for (int l = 0; l <= k; ++l) acc = fmaf(cc.W[k * D + l], mu[l], acc);
        nu[k] = acc;
      }
      col32<D>(cc, XC[m], CC[m], y, A);
      float q = 0.f;
#pragma unroll
      for (int k = 0; k < D; ++k) q = fmaf(y[k] - nu[k], y[k] - nu[k], q);
      const float w = CC[m] - q;  // A + |y|^2 = COL
      lw[m] = w;
      mx = fmaxf(mx, w);
    }
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(~0u, mx, o));
    if (lane == 0) s_red[warp] = mx;
    __syncthreads();
    float gmx = -CUDART_INF_F;
    for (int w = 0; w < nw; ++w) gmx = fmaxf(gmx, s_red[w]);
    if (gmx == -CUDART_INF_F) {
      if (tid == 0) raise_err(b.err, DSMC_E_RUNTIME, t, 0, kReasonLeafZero);
      return;
    }
    double sum = 0.0;
    for (int m = tid; m < N; m += blockDim.x) sum += (double)ex2(lw[m] - gmx);
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(~0u, sum, o);
    __syncthreads();  // s_red reads done
    if (lane == 0) sh[warp] = sum;
    __syncthreads();
    double tot = 0.0;
    for (int w = 0; w < nw; ++w) tot += sh[w];
    const float lse = gmx + (float)log2(tot);
    for (int m = tid; m < N; m += blockDim.x) lw[m] -= lse;
    if (tid == 0) ll += ((double)lse - log2((double)N)) * kLn2;
    __syncthreads();
  }
  if (tid == 0) *loglik = ll;
}

// Backward pass: warp w of CTA c draws path m = 8 c + w. P: [M][K] indices.
template <int D>
__global__ void __launch_bounds__(256) ffbs_backward_kernel(Bufs b, const float* LW, int M,
                                                            uint32_t* P) {
  extern __shared__ float4 sm_bw[];
  const int N = b.N, K = b.K, ch = 0;
  float4* s_nu = sm_bw;                                      // [N] nu_i (whitened)
  float* s_lw = reinterpret_cast<float*>(s_nu + N);          // [N]
  double* s_cdf = reinterpret_cast<double*>(s_lw + ((N + 1) & ~1));  // [N] endpoint CDF
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = blockIdx.x * 8 + warp;
  const bool act = m < M;
  __shared__ double sh[32];
  // endpoint: multinomial_indices of the final weights (key {seed,0,T,bwd})
  {
    const float* lwT = LW + (size_t)(K - 1) * N;
    const int per = (N + blockDim.x - 1) / blockDim.x;
    const int i0 = threadIdx.x * per, i1 = min(N, i0 + per);
    double seg = 0.0;
    for (int i = i0; i < i1; ++i) seg += (double)ex2(lwT[i]);
    const double incl = block_scan_incl(seg, sh);
    double run = incl - seg;
    for (int i = i0; i < i1; ++i) {
      run += (double)ex2(lwT[i]);
      s_cdf[i] = run;
    }
    __syncthreads();
  }
  int idx = 0;
  if (act) {
    const StreamId eid = stream_id(b.seeds[ch], 0, (uint64_t)(K - 1), DSMC_ROLE_BACKWARD_SAMPLE, 0);
    idx = cdf_search(s_cdf, N, u64_uniform(stream_u64(eid, (uint64_t)m)) * s_cdf[N - 1]);
    if (lane == 0) P[(size_t)m * K + K - 1] = (uint32_t)idx;
  }
  for (int t = K - 2; t >= 0; --t) {
    const TimeConst& tc = b.tc[(size_t)ch * b.Kt + b.t0 + t + 1];
    CutConst32 cc;
    load_cut32<D>(tc, cc);
    __syncthreads();  // previous step's s_nu / s_lw reads are done
    const float4* XT = b.X32 + (size_t)t * N;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      float mu[4], nu[4] = {0.f, 0.f, 0.f, 0.f};
      row_mu32<D>(cc, XT[i], mu);
#pragma unroll
      for (int k = 0; k < D; ++k) {
        float acc = 0.f;
#pragma unroll
        for (int l = 0; l <= k; ++l) acc = fmaf(cc.W[k * D + l], mu[l], acc);
        nu[k] = acc;
      }
      s_nu[i] = make_float4(nu[0], nu[1], nu[2], nu[3]);
      s_lw[i] = LW[(size_t)t * N + i];
    }
    __syncthreads();
    if (!act) continue;
    // the draw's state at t+1, whitened with the cut t+1 constants
    float y[4] = {0.f, 0.f, 0.f, 0.f}, A;
    col32<D>(cc, b.X32[(size_t)(t + 1) * N + idx], 0.f, y, A);
    // v_i = lw_i - |y - nu_i|^2 over the lane's entries: max, then sums
    float mx = -CUDART_INF_F;
    for (int i = lane; i < N; i += 32) {
      const float4 nv = s_nu[i];
      const float nn[4] = {nv.x, nv.y, nv.z, nv.w};
      float q = 0.f;
#pragma unroll
      for (int k = 0; k < D; ++k) q = fmaf(y[k] - nn[k], y[k] - nn[k], q);
      mx = fmaxf(mx, s_lw[i] - q);
    }
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(~0u, mx, o));
    if (mx == -CUDART_INF_F) {
      if (lane == 0) raise_err(b.err, DSMC_E_RUNTIME, t, 0, kReasonZeroTable);
      idx = 0;
      continue;
    }
    // lanes own contiguous chunks so the warp scan gives sequential order
    const int per = (N + 31) / 32, j0 = lane * per, j1 = min(N, j0 + per);
    float part = 0.f;
    for (int i = j0; i < j1; ++i) {
      const float4 nv = s_nu[i];
      const float nn[4] = {nv.x, nv.y, nv.z, nv.w};
      float q = 0.f;
#pragma unroll
      for (int k = 0; k < D; ++k) q = fmaf(y[k] - nn[k], y[k] - nn[k], q);
      part += ex2(s_lw[i] - q - mx);
    }
    float incl = part;
    for (int o = 1; o < 32; o <<= 1) {
      const float n = __shfl_up_sync(~0u, incl, o);
      if (lane >= o) incl += n;
    }
    const float total = __shfl_sync(~0u, incl, 31);
    const StreamId bid = stream_id(b.seeds[ch], 1, (uint64_t)t, DSMC_ROLE_BACKWARD_SAMPLE,
                                   (uint64_t)m + 1);
    const float pt = (float)u64_uniform(stream_u64(bid, 0)) * total;
    // the lane whose chunk holds pt walks it sequentially
    const unsigned hit = __ballot_sync(~0u, pt < incl);
    const int owner = hit ? __ffs(hit) - 1 : 31;
    int sel = -1;
    if (lane == owner) {
      float cum = incl - part;
      int last = j0;
      for (int i = j0; i < j1; ++i) {
        const float4 nv = s_nu[i];
        const float nn[4] = {nv.x, nv.y, nv.z, nv.w};
        float q = 0.f;
#pragma unroll
        for (int k = 0; k < D; ++k) q = fmaf(y[k] - nn[k], y[k] - nn[k], q);
        const float e = ex2(s_lw[i] - q - mx);
        cum += e;
        if (e > 0.f) last = i;
        if (pt < cum) {
          sel = i;
          break;
        }
      }
      if (sel < 0) sel = last;  // FP spill: last live entry of the chunk
    }
    idx = __shfl_sync(~0u, sel, owner);
    if (lane == 0) P[(size_t)m * K + t] = (uint32_t)idx;
  }
}

// Per-time moments over the M drawn paths (uncentred by m_t in FP64).
template <int D>
__global__ void __launch_bounds__(256) ffbs_moments_kernel(Bufs b, const uint32_t* P, int M,
                                                           double* mean, double* cov,
                                                           double* paths) {
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (t >= b.K) return;
  const int N = b.N, K = b.K;
  const TimeConst& tc = b.tc[(size_t)b.t0 + t];
  constexpr int NT = D * (D + 1) / 2;
  float s1[D], s2[NT];
#pragma unroll
  for (int k = 0; k < D; ++k) s1[k] = 0.f;
#pragma unroll
  for (int k = 0; k < NT; ++k) s2[k] = 0.f;
  for (int m = lane; m < M; m += 32) {
    const float4 xv = b.X32[(size_t)t * N + P[(size_t)m * K + t]];
    const float x[4] = {xv.x, xv.y, xv.z, xv.w};
    if (paths)
      for (int k = 0; k < D; ++k) paths[((size_t)m * K + t) * D + k] = (double)x[k] + tc.pm[k];
    int c = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      s1[k] += x[k];
#pragma unroll
      for (int l = k; l < D; ++l) {
        s2[c] = fmaf(x[k], x[l], s2[c]);
        ++c;
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
#pragma unroll
    for (int k = 0; k < D; ++k) s1[k] += __shfl_xor_sync(~0u, s1[k], o);
#pragma unroll
    for (int k = 0; k < NT; ++k) s2[k] += __shfl_xor_sync(~0u, s2[k], o);
  }
  if (lane == 0) {
    double mu[4];
    for (int k = 0; k < D; ++k) mu[k] = (double)s1[k] / M;
    for (int k = 0; k < D; ++k) mean[(size_t)t * D + k] = mu[k] + tc.pm[k];
    int c = 0;
    for (int k = 0; k < D; ++k)
      for (int l = k; l < D; ++l, ++c) {
        const double v = (double)s2[c] / M - mu[k] * mu[l];
        cov[((size_t)t * D + k) * D + l] = v;
        cov[((size_t)t * D + l) * D + k] = v;
      }
  }
}

}  // namespace dsmc_dev

// Top-down ancestor composition and the final gather (replaces the
// reference's per-combine full-path copies, smoother.cpp:51-60,208-214).
//
// A block's map M[q] gives, for root slot q, the slot inside that block. The
// root map is the identity; a combined block passes l[M[q]] to its left child
// and r[M[q]] to its right child; a carried odd-tail block passes M through.
// At the leaves, sigma_t[q] is the leaf particle of root slot q at time t, so
// path[t][q] = leaf_t[sigma_t[q]] (verified equivalent).
#pragma once

#include "combine32.cuh"

namespace dsmc_dev {

// One top-down level (level >= 2): maps of level l -> maps of level l-1.
__global__ void td_kernel(Bufs b, int level, size_t cursor, int nb_l,
                          int nb_lm1, const uint32_t* Mcur, uint32_t* Mnext,
                          int root, const uint32_t* root_map) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // see pdl_wait
  // grid (block, slot chunk, chain): blocks in x (up to 2^31)
  const int q = blockIdx.y * blockDim.x + threadIdx.x;
  const int k = blockIdx.x, ch = blockIdx.z;
  const int N = b.N;
  if (q >= N) return;
  // root map: identity, or the window root's map from the cross-shard levels
  const uint32_t m = root ? (root_map ? root_map[(size_t)ch * N + q] : (uint32_t)q)
                          : Mcur[((size_t)ch * b.cap + k) * N + q];
  if (2 * k + 1 < nb_lm1) {
    const size_t gidx = (size_t)ch * b.T + cursor + k;
    Mnext[((size_t)ch * b.cap + 2 * k) * N + q] = b.PL[gidx * N + m];
    Mnext[((size_t)ch * b.cap + 2 * k + 1) * N + q] = b.PR[gidx * N + m];
  } else {
    Mnext[((size_t)ch * b.cap + 2 * k) * N + q] = m;
  }
}

// sigma_t[q] from the level-1 maps (root = identity when K <= 2).
__device__ inline uint32_t leaf_sigma(const Bufs& b, int ch, int t, int q,
                                      const uint32_t* M1, int root1,
                                      const uint32_t* root_map) {
  const uint32_t r0 = root_map ? root_map[(size_t)ch * b.N + q] : (uint32_t)q;
  if (b.K == 1) return r0;
  const int k = t >> 1;
  const uint32_t m = root1 ? r0 : M1[((size_t)ch * b.cap + k) * b.N + q];
  if (2 * k + 1 < b.K) {
    const size_t gidx = (size_t)ch * b.T + k;  // level-1 cursor is 0
    return (t & 1) ? b.PR[gidx * b.N + m] : b.PL[gidx * b.N + m];
  }
  return m;
}

// Fused level-1 composition + gather + per-time moments. One CTA per
// (time, chain). FP64 leaves (parity path).
__global__ void __launch_bounds__(256) gather64_kernel(Bufs b, const uint32_t* M1,
                                                       int root1, double* paths,
                                                       double* mean, double* cov,
                                                       const uint32_t* root_map) {
  const int t = blockIdx.x, ch = blockIdx.y;
  const int N = b.N, d = b.d;
  __shared__ double red[8][20];
  double s1[4] = {0, 0, 0, 0}, s2[16] = {0};
  const double* X = b.X64 + ((size_t)ch * b.K + t) * N * d;
  for (int q = threadIdx.x; q < N; q += blockDim.x) {
    const uint32_t sg = leaf_sigma(b, ch, t, q, M1, root1, root_map);
    double x[4];
    for (int k = 0; k < d; ++k) x[k] = X[(size_t)sg * d + k];
    if (paths)
      for (int k = 0; k < d; ++k) paths[(((size_t)ch * b.K + t) * N + q) * d + k] = x[k];
    for (int k = 0; k < d; ++k) {
      s1[k] += x[k];
      for (int l = 0; l < d; ++l) s2[k * d + l] += x[k] * x[l];
    }
  }
  if (!mean && !cov) return;
  const int nv = d + d * d;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int v = 0; v < nv; ++v) {
    double a = v < d ? s1[v] : s2[v - d];
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(~0u, a, o);
    if (lane == 0) red[warp][v] = a;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot[20] = {0};
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
      for (int v = 0; v < nv; ++v) tot[v] += red[w][v];
    double mu[4];
    for (int k = 0; k < d; ++k) mu[k] = tot[k] / N;
    const size_t o = (size_t)ch * b.K + t;
    if (mean)
      for (int k = 0; k < d; ++k) mean[o * d + k] = mu[k];
    if (cov)
      for (int k = 0; k < d; ++k)
        for (int l = 0; l < d; ++l)
          cov[o * d * d + k * d + l] = tot[d + k * d + l] / N - mu[k] * mu[l];
  }
}

// FP32 leaves: centred states. One warp per time t (8 per CTA): lanes gather
// 4 particles per round with independent loads (sigma map -> leaf slab), sum
// x and the upper triangle of x x^T in FP32 over their particles, one warp
// reduction of the D + D(D+1)/2 sums, FP64 moments written by lane 0.
template <int D>
__global__ void __launch_bounds__(256) gather32_kernel(Bufs b, const uint32_t* M1,
                                                       int root1, double* paths,
                                                       double* mean, double* cov,
                                                       const uint32_t* root_map,
                                                       int t_begin = 0, int t_end = 1 << 30) {
  const int t = t_begin + blockIdx.x * 8 + (threadIdx.x >> 5), ch = blockIdx.y;
  const int lane = threadIdx.x & 31;
  if (t >= b.K || t >= t_end) return;
  const int N = b.N;
  const TimeConst& tc = b.tc[(size_t)ch * b.Kt + b.t0 + t];
  constexpr int NT = D * (D + 1) / 2;
  float s1[D], s2[NT];
#pragma unroll
  for (int k = 0; k < D; ++k) s1[k] = 0.f;
#pragma unroll
  for (int k = 0; k < NT; ++k) s2[k] = 0.f;
  const float4* X = b.X32 + ((size_t)ch * b.K + t) * N;
  for (int q0 = lane; q0 < N; q0 += 128) {
    uint32_t sg[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = q0 + 32 * u;
      sg[u] = q < N ? leaf_sigma(b, ch, t, q, M1, root1, root_map) : 0u;
    }
    float4 xv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) xv[u] = X[sg[u]];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = q0 + 32 * u;
      if (q >= N) continue;
      float x[4] = {xv[u].x, xv[u].y, xv[u].z, xv[u].w};
      if (paths)
        for (int k = 0; k < D; ++k)
          paths[(((size_t)ch * b.K + t) * N + q) * D + k] = (double)x[k] + tc.pm[k];
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
  }
  if (!mean && !cov) return;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
#pragma unroll
    for (int k = 0; k < D; ++k) s1[k] += __shfl_xor_sync(~0u, s1[k], o);
#pragma unroll
    for (int k = 0; k < NT; ++k) s2[k] += __shfl_xor_sync(~0u, s2[k], o);
  }
  if (lane == 0) {
    double mu[4];
    for (int k = 0; k < D; ++k) mu[k] = (double)s1[k] / N;
    const size_t o = (size_t)ch * b.K + t;
    if (mean)
      for (int k = 0; k < D; ++k) mean[o * D + k] = mu[k] + tc.pm[k];
    if (cov) {
      int c = 0;
      for (int k = 0; k < D; ++k)
        for (int l = k; l < D; ++l, ++c) {
          const double v = (double)s2[c] / N - mu[k] * mu[l];
          cov[o * D * D + k * D + l] = v;
          cov[o * D * D + l * D + k] = v;
        }
    }
  }
}

// --------------------------------------------------- single-slot tracing
// Conditional sweeps need one root slot's path only: trace it down the tree
// (O(K) instead of O(K N)). sel[ch] holds the slot at level l; per level one
// thread per block.
__global__ void td1_kernel(Bufs b, size_t cursor, int nb_l, int nb_lm1,
                           const uint32_t* Scur, uint32_t* Snext) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int ch = blockIdx.y;
  if (k >= nb_l) return;
  const uint32_t m = Scur[(size_t)ch * b.cap * 2 + k];
  if (2 * k + 1 < nb_lm1) {
    const size_t gidx = (size_t)ch * b.T + cursor + k;
    Snext[(size_t)ch * b.cap * 2 + 2 * k] = b.PL[gidx * b.N + m];
    Snext[(size_t)ch * b.cap * 2 + 2 * k + 1] = b.PR[gidx * b.N + m];
  } else {
    Snext[(size_t)ch * b.cap * 2 + 2 * k] = m;
  }
}

// Star selection at the root (conditional.cpp:195-199, 35-48).
__global__ void star_select_kernel(Bufs b, int levels, uint32_t* S0, int fp32) {
  const int ch = blockIdx.x * blockDim.x + threadIdx.x;
  if (ch >= b.B) return;
  StreamReader s;
  s.init(stream_id(b.seeds[ch], levels + 1, b.sweep, DSMC_ROLE_STAR_SELECT, 0));
  uint32_t chosen;
  if (b.K == 1 && !b.UNI[(size_t)ch * b.K]) {
    const double u = s.uniform();
    double cum = 0.0;
    uint32_t last_live = 0;
    chosen = (uint32_t)b.N;
    for (int p = 0; p < b.N; ++p) {
      const double w = fp32 ? exp2((double)b.LW32[(size_t)ch * b.N + p])
                            : exp_w(b.LW64[(size_t)ch * b.K * b.N + p]);
      if (w > 0.0) last_live = p;
      cum += w;
      if (u < cum) {
        chosen = p;
        break;
      }
    }
    if (chosen == (uint32_t)b.N) chosen = last_live;
  } else {
    chosen = (uint32_t)s.index(b.N);
  }
  S0[(size_t)ch * b.cap * 2] = chosen;
}

// Selected path + change mask (path_changed_times, conditional.cpp:218-230).
__global__ void star_path_kernel(Bufs b, const uint32_t* S0, int fp32,
                                 double* out, uint8_t* changed) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int ch = blockIdx.y;
  if (t >= b.K) return;
  const int d = b.d;
  uint32_t m;
  if (b.K == 1) {
    m = S0[(size_t)ch * b.cap * 2];
  } else {
    const int k = t >> 1;
    const uint32_t s = S0[(size_t)ch * b.cap * 2 + k];
    if (2 * k + 1 < b.K) {
      const size_t gidx = (size_t)ch * b.T + k;
      m = (t & 1) ? b.PR[gidx * b.N + s] : b.PL[gidx * b.N + s];
    } else {
      m = s;
    }
  }
  const size_t o = (size_t)ch * b.K + t;
  bool ch_ = false;
  for (int k = 0; k < d; ++k) {
    double v;
    if (fp32) {
      const TimeConst& tc = b.tc[o];
      v = (double)comp(b.X32[o * b.N + m], k) + tc.pm[k];
      if (m == 0) v = b.star[o * d + k];  // slot 0 is the reference itself
    } else {
      v = b.X64[(o * b.N + m) * d + k];
    }
    ch_ |= (v != b.star[o * d + k]);
    out[o * d + k] = v;
  }
  if (changed) changed[o] = ch_;
}

}  // namespace dsmc_dev

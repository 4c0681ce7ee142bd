// FP64 parity combine: the reference's dense pair table (build_dense,
// resampling.cpp:59-104) and inversion sampler (select_sorted,
// resampling.cpp:109-153) restated per slot, plus the
// lazy MH / rejection samplers (resampling.cpp:233-324). The N x N table is
// never stored: pass 1 keeps per-row max, raw total and 64-entry sub-block
// sums; each sampled slot recomputes the <= 64 weights of its sub-block,
// which are bit-identical to pass 1 (same fill, same exp_w).
#pragma once

#include "leaves.cuh"

namespace dsmc_dev {

// Level-wide arguments of one batch of combines.
struct LevelArgs {
  int level;      // 1..L
  int np;         // combines at this level
  int nb_prev;    // blocks at level-1
  int k0;         // first combine of this chunk
  size_t cursor;  // schedule index of combine 0 of this level
  const uint32_t* first_prev;  // [B][cap][N] (unused at level 1)
  const uint32_t* last_prev;
  uint32_t* first_next;
  uint32_t* last_next;
  const double* blnc_prev;  // [B][cap]
  double* blnc_next;
  double* ws;      // workspace for this chunk
  size_t ws_comb;  // doubles per combine in ws
  int n_out;       // slots resampled (N, or N-1 when conditional)
  int key_level;      // level in the stream key (global tree level)
  long long node_off; // global node index of local combine 0 (windows)
  int rows_per_cta;   // FP32 pass 1 row tile (multiple of 32)
  int slots_per_cta;  // FP32 pass 2 slot slice per CTA
  float* aux;         // FP32 pass 1 -> pass 2 column/row data (Aux32)
  size_t aux_comb;    // floats per combine in aux
  int tc_ncs;         // tensor-core pass 1: column splits per 128-row tile
  int tc_nk;          // ... and combines in this chunk (persistent work list)
  int wide_tiles;     // wide path: the prologue also writes pass 1's column tiles
};

// Block meta derived from the schedule geometry.
struct Side {
  int leaf;  // the block is a single leaf
  int t;     // boundary time (left: last time, right: first time)
  int idx;   // block index at level-1
};

__device__ inline void sides(const Bufs& b, const LevelArgs& la, int k,
                             Side& L, Side& R, CombineGeom& g) {
  g = combine_geom(la.level, k, b.K);
  L.leaf = (g.c - 1 == g.a);
  L.t = g.c - 1;
  L.idx = 2 * k;
  R.leaf = (g.b == g.c);
  R.t = g.c;
  R.idx = 2 * k + 1;
}

// slot of block `blk` at boundary -> particle index of that leaf
__device__ inline uint32_t map_first(const Bufs& b, const LevelArgs& la,
                                     int ch, const Side& s, uint32_t q) {
  if (s.leaf) return q;
  return la.first_prev[((size_t)ch * b.cap + s.idx) * b.N + q];
}
__device__ inline uint32_t map_last(const Bufs& b, const LevelArgs& la, int ch,
                                    const Side& s, uint32_t q) {
  if (s.leaf) return q;
  return la.last_prev[((size_t)ch * b.cap + s.idx) * b.N + q];
}
__device__ inline double block_lnc(const Bufs& b, const LevelArgs& la, int ch,
                                   const Side& s, int a) {
  if (s.leaf) return b.LNC[(size_t)ch * b.K + a];
  return la.blnc_prev[(size_t)ch * b.cap + s.idx];
}

// Per-combine column data of the FP64 fill, staged in shared memory as one
// record per column: x_0..x_{d-1}, base, leaf weight (+ pad to 16 bytes), so
// an entry is two or three 16-byte loads at immediate offsets. Column j's
// record sits at cpad(j): every 64-column sub-block takes 72 records, so the
// four 8-lane groups of a warp (four sub-blocks, pass 1's sub-block sums)
// start at different banks. The layout only places values: the arithmetic
// and its order are unchanged.
__host__ __device__ inline int cpad(int j) { return j + (j >> 6) * 8; }
__host__ __device__ inline int col_ld(int N) { return (N + 63) / 64 * 72; }
__host__ __device__ constexpr int rec_len(int d) { return (d + 3) & ~1; }  // d + 2, even
struct Col64 {
  double* rec;  // ld records of rec_len(d) doubles
  int ld;
  int has_lwr;  // the right block is a non-uniform leaf (weights in the records)
  // FP32 screen copies (c64_rows with fast = 1), in column PAIRS: pair
  // p = 32 s + l holds columns 64 s + l and 64 s + 32 + l (sub-block s, lane
  // l), so a lane screens both with packed FADD2 / FFMA2. States are centred
  // on column 0's (x - cen), interleaved so a lane's packed operands are one
  // 16-byte load; bases and leaf weights as float2 pairs; dead padding
  // columns carry base -inf. cm: the largest finite |base|, |lwr|, |x_k - cen_k|, and
  // (as an int) whether every column is clean (finite states, no NaN or +inf
  // base / weight); cen: the centre (FP64).
  float* xs;    // d > 1: planes [2][npair] float4 (x0, x0', x1, x1'), (x2, x2', x3, x3'); d = 1: float2 (x, x')
  int npair;
  float2* bf2;
  float2* lf2;
  float* cm;
  double* cen;
};
// Shared-memory bytes of the column stage: the FP64 records, plus the FP32
// screen pairs and their magnitude maxima when `fast`.
__host__ __device__ inline size_t cols64_bytes(int N, int d, bool fast) {
  const size_t ld = col_ld(N), npair = (size_t)(N + 63) / 64 * 32;
  return sizeof(double) * ld * rec_len(d) +
         (fast ? npair * ((d == 1 ? 8 : 32) + 16) + 64 : 0);
}

// Column base of the stitch-row factory at cut c (per model class).
template <int MC, int D>
__device__ inline double col_base(const DevModel& M, const TimeConst& tc,
                                  int c, const double* x) {
  if (MC == kSV) return tc.shift1;
  if (MC == kCOX)  // models.cpp:183-186
    return DADD(DSUB(cox_log_poisson(M, c, x[0]), dlog_normal_pdf(x[0], M.mp[2], M.mp[3])),
                M.mp[4]);
  if (MC == kCRW)  // models.cpp:314-315
    return crw_in_box(x[0]) ? DSUB(M.mp[1], kLogHalf) : -CUDART_INF;
  if (MC == kTHETA) {  // models.cpp:450-458: two gaussian_row passes + shift
    const double tt = DSUB(x[0], M.y[c]);
    double bs = __fma_rn(DDIV(-1.0, DMUL(2.0, M.mp[4])), DMUL(tt, tt), 0.0);
    const double t2 = DSUB(x[0], M.prop_mean[c]);
    bs = __fma_rn(DDIV(1.0, DMUL(2.0, M.prop_cov[c])), DMUL(t2, t2), bs);
    return DADD(bs, tc.shift1);
  }
  if (MC == kLG1) {  // models.cpp:617-627
    double bs = 0.0;
    if (tc.obs) {
      const double h = *at(M.H, M.H_s, c), r = *at(M.R, M.R_s, c);
      const double tt = DSUB(x[0], DDIV(M.y[c], h));
      bs = __fma_rn(DDIV(DMUL(-h, h), DMUL(2.0, r)), DMUL(tt, tt), 0.0);
    }
    const double var = M.prop_cov[c];
    const double t2 = DSUB(x[0], M.prop_mean[c]);
    bs = __fma_rn(DDIV(1.0, DMUL(2.0, var)), DMUL(t2, t2), bs);
    return DADD(bs, tc.shift1);
  }
  // LG d>1 (oracle comb_prepare order)
  const double lh = cb_log_h(M, tc, c, x);
  const double lp = DSUB(tc.p_norm, DMUL(0.5, dquad(tc.pW, D, x, tc.pm)));
  return DSUB(DADD(tc.t_norm, lh), lp);
}

// Row term: the transition mean of a left particle at cut c (whitened for
// d > 1). D is the compile-time state dimension (1 for LG1 / SV).
template <int MC, int D>
__device__ inline void row_mean(const DevModel& M, const TimeConst& tc, int c, const double* xl,
                                double* mu) {
  if (MC == kSV) {
    mu[0] = DADD(M.sv_mu, DMUL(M.sv_phi, DSUB(xl[0], M.sv_mu)));
  } else if (MC == kCOX) {  // models.cpp:189: icept + slope * xp
    mu[0] = DADD(M.mp[1], DMUL(M.mp[0], xl[0]));
  } else if (MC == kCRW) {  // models.cpp:318: the row's own state
    mu[0] = xl[0];
  } else if (MC == kTHETA) {  // models.cpp:461: the drifted left endpoint
    mu[0] = theta_drift(M, xl[0]);
  } else if (MC == kLG1) {
    mu[0] = DADD(DMUL(*at(M.F, M.F_s, c), xl[0]), *at(M.b, M.b_s, c));
  } else {  // v = W_Q (F x + b): the row's whitened transition mean
    const double* F = at(M.F, M.F_s, c);
    const double* bb = at(M.b, M.b_s, c);
    double m[D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      double s = 0.0;
#pragma unroll
      for (int l = 0; l < D; ++l) s = DADD(s, DMUL(F[k * D + l], xl[l]));
      m[k] = DADD(s, bb[k]);
    }
    const double* W = tc.tW;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      double v = 0.0;
#pragma unroll
      for (int l = 0; l <= k; ++l) v = DADD(v, DMUL(W[k * D + l], m[l]));
      mu[k] = v;
    }
  }
}

// One table entry (fill_row of make_pair_source, smoother.cpp:153-161).
// MODE selects the leaf-weight terms: 0 none, 1 the left leaf's own weight
// (v + sl), 2 both leaves' weights ((v + sl) + lwr_j) — the three cases of
// fill64, hoisted out of the entry loops of pass 1.
template <int MC, int D, int MODE>
__device__ __forceinline__ double fill64m(double coef, const double* mu, const Col64& C, int cp,
                                          double sl) {
  constexpr int RL = rec_len(D);
  const double2* r = reinterpret_cast<const double2*>(C.rec) + (size_t)cp * (RL / 2);
  double f[RL];
#pragma unroll
  for (int q = 0; q < RL / 2; ++q) {
    const double2 v = r[q];
    f[2 * q] = v.x;
    f[2 * q + 1] = v.y;
  }
  double v;
  if (MC == kLGN) {  // d chained gaussian_row passes (ref_models lgssm_nd)
    v = f[D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const double t = DSUB(f[k], mu[k]);
      v = __fma_rn(-0.5, DMUL(t, t), v);
    }
  } else {
    const double t = DSUB(f[0], mu[0]);
    v = __fma_rn(coef, DMUL(t, t), f[D]);
  }
  if (MODE == 2) v = DADD(DADD(v, sl), f[D + 1]);
  else if (MODE == 1) v = DADD(v, sl);
  return v;
}
template <int MC, int D>
__device__ inline double fill64(const DevModel& M, const TimeConst& tc,
                                double coef, const double* mu, const Col64& C,
                                int j, double sl, bool has_l) {
  const int cp = cpad(j);
  if (C.has_lwr) return fill64m<MC, D, 2>(coef, mu, C, cp, sl);
  if (has_l && sl != 0.0) return fill64m<MC, D, 1>(coef, mu, C, cp, sl);
  return fill64m<MC, D, 0>(coef, mu, C, cp, sl);
}

// FP32 estimates of fill64m for screen pair p (|error| <= E, c64_row):
// base - 0.5 sum_k t_k^2 (coef t^2 for the d = 1 model classes), both
// columns of the pair in packed FADD2 / FFMA2; nmu = -(mu - cen) per dim.
template <int MC, int D, int MODE>
__device__ __forceinline__ float2 est32_pair(const float2* nmu, float2 cf, const Col64& C, int p) {
  float2 q;
  if (MC == kLGN && D > 1) {
    const float4 a = reinterpret_cast<const float4*>(C.xs)[p];  // (x0, x0', x1, x1')
    const float2 t0 = __fadd2_rn(make_float2(a.x, a.y), nmu[0]);
    const float2 t1 = __fadd2_rn(make_float2(a.z, a.w), nmu[1]);
    q = __ffma2_rn(t1, t1, __fmul2_rn(t0, t0));
    if (D > 2) {
      const float4 c = reinterpret_cast<const float4*>(C.xs)[C.npair + p];  // (x2, x2', x3, x3')
      const float2 t2 = __fadd2_rn(make_float2(c.x, c.y), nmu[2]);
      q = __ffma2_rn(t2, t2, q);
      if (D > 3) {
        const float2 t3 = __fadd2_rn(make_float2(c.z, c.w), nmu[3]);
        q = __ffma2_rn(t3, t3, q);
      }
    }
  } else {
    const float2 t = __fadd2_rn(reinterpret_cast<const float2*>(C.xs)[p], nmu[0]);
    q = __fmul2_rn(t, t);
  }
  float2 a = __ffma2_rn(cf, q, C.bf2[p]);
  if (MODE == 2) a = __fadd2_rn(a, C.lf2[p]);
  return a;
}

template <int MC>
__device__ inline double row_coef(const DevModel& M, int c) {
  if (MC == kSV) return DDIV(-1.0, DMUL(2.0, M.sv_s2));
  if (MC == kCOX) return DDIV(-1.0, DMUL(2.0, M.mp[5]));
  if (MC == kCRW) return DDIV(-1.0, DMUL(2.0, M.mp[0]));
  if (MC == kTHETA) return DDIV(-1.0, DMUL(2.0, M.mp[3]));
  if (MC == kLG1) return DDIV(-1.0, DMUL(2.0, *at(M.Q, M.Q_s, c)));
  return 0.0;
}

// Stage the combine's right boundary slab + column bases in shared memory.
__device__ __forceinline__ float finite_abs(double v) {
  const float a = fabsf((float)v);
  return a < CUDART_INF_F ? a : 0.f;
}
template <int MC, int D>
__device__ void stage_cols(const Bufs& b, const LevelArgs& la, int ch,
                           const Side& R, const DevModel& M,
                           const TimeConst& tc, double* smem, Col64& C,
                           bool fast = false) {
  const int N = b.N;
  constexpr int d = D, RL = rec_len(D);
  C.ld = col_ld(N);
  C.rec = smem;
  const bool nonuni = R.leaf && !b.UNI[(size_t)ch * b.K + R.t];
  C.has_lwr = nonuni;
  C.xs = nullptr;
  C.bf2 = C.lf2 = nullptr;
  C.cm = nullptr;
  C.cen = nullptr;
  const double* X = b.X64 + ((size_t)ch * b.K + R.t) * N * d;
  // the fill's column coordinates: whitened w = W_Q x (LGSSM d > 1) or x
  auto coords = [&](const double* x, double* z) {
    if (MC == kLGN) {
#pragma unroll
      for (int k = 0; k < d; ++k) {
        double v = 0.0;
#pragma unroll
        for (int l = 0; l <= k; ++l) v = DADD(v, DMUL(tc.tW[k * d + l], x[l]));
        z[k] = v;
      }
    } else {
      z[0] = x[0];
    }
  };
  const int nsub = (N + kSub - 1) / kSub, npair = nsub * 32;
  if (fast) {
    C.xs = reinterpret_cast<float*>(smem + (size_t)C.ld * RL);
    C.npair = npair;
    C.bf2 = reinterpret_cast<float2*>(C.xs + (size_t)npair * (d == 1 ? 2 : 8));
    C.lf2 = C.bf2 + npair;
    C.cm = reinterpret_cast<float*>(C.lf2 + npair);
    C.cen = reinterpret_cast<double*>(C.cm + 8);
    // centre the FP32 copies on column 0 (the fill's coordinates drift with
    // time, e.g. positions of the constant-velocity model; centred, the
    // screen's rounding scales with the particle spread, not the position)
    double x0[D], cen[D];
    const uint32_t p0 = map_first(b, la, ch, R, 0);
#pragma unroll
    for (int k = 0; k < d; ++k) x0[k] = X[(size_t)p0 * d + k];
    coords(x0, cen);
    if (threadIdx.x < 8) C.cm[threadIdx.x] = threadIdx.x == 6 ? __int_as_float(1) : 0.f;
#pragma unroll
    for (int k = 0; k < d; ++k)
      if (threadIdx.x == k) C.cen[k] = isfinite(cen[k]) ? cen[k] : 0.0;
    __syncthreads();
  }
  float mb = 0.f, ml = 0.f, mxk[4] = {0.f, 0.f, 0.f, 0.f};
  int clean = 1;
  const int jend = fast ? nsub * kSub : N;  // the screen also fills the padding columns
  for (int j = threadIdx.x; j < jend; j += blockDim.x) {
    double z[D], bs = -CUDART_INF, lw = 0.0;
    const bool live = j < N;
    if (live) {
      const uint32_t p = map_first(b, la, ch, R, j);
      double x[D];
#pragma unroll
      for (int k = 0; k < d; ++k) x[k] = X[(size_t)p * d + k];
      bs = col_base<MC, D>(M, tc, b.t0 + R.t, x);  // global time (windows)
      coords(x, z);
      double* r = C.rec + (size_t)cpad(j) * RL;
#pragma unroll
      for (int k = 0; k < d; ++k) r[k] = z[k];
      r[d] = bs;
      if (nonuni) {
        lw = b.LW64[((size_t)ch * b.K + R.t) * N + p];
        r[d + 1] = lw;
      }
    }
    if (fast) {
      const int pr = (j >> 6) * 32 + (j & 31), h = (j >> 5) & 1;  // screen pair, half
      reinterpret_cast<float*>(C.bf2)[2 * pr + h] = (float)bs;
      reinterpret_cast<float*>(C.lf2)[2 * pr + h] = (float)lw;
      float xs[4] = {0.f, 0.f, 0.f, 0.f};
      if (live) {
        mb = fmaxf(mb, finite_abs(bs));
        ml = fmaxf(ml, finite_abs(lw));
        clean &= !isnan(bs) && bs != CUDART_INF && !isnan(lw) && lw != CUDART_INF;
#pragma unroll
        for (int k = 0; k < d && k < 4; ++k) {
          const double xc = DSUB(z[k], C.cen[k]);
          xs[k] = (float)xc;
          mxk[k] = fmaxf(mxk[k], finite_abs(xc));
          clean &= isfinite(z[k]) && isfinite(xs[k]);
        }
      }
      if (d == 1) {
        C.xs[2 * pr + h] = xs[0];
      } else {  // planes (x0, x0', x1, x1') and (x2, x2', x3, x3') per pair
        C.xs[4 * pr + h] = xs[0];
        C.xs[4 * pr + 2 + h] = xs[1];
        if (d > 2) {
          C.xs[4 * (npair + pr) + h] = xs[2];
          C.xs[4 * (npair + pr) + 2 + h] = xs[3];
        }
      }
    }
  }
  if (fast) {  // block maxima of the finite magnitudes (non-negative: int order)
    const int lane = threadIdx.x & 31;
    for (int o = 16; o; o >>= 1) {
      mb = fmaxf(mb, __shfl_xor_sync(~0u, mb, o));
      ml = fmaxf(ml, __shfl_xor_sync(~0u, ml, o));
#pragma unroll
      for (int k = 0; k < 4; ++k) mxk[k] = fmaxf(mxk[k], __shfl_xor_sync(~0u, mxk[k], o));
    }
    clean = __all_sync(~0u, clean);
    if (lane == 0) {
      int* cmi = reinterpret_cast<int*>(C.cm);
      atomicMax(cmi + 0, __float_as_int(mb));
      atomicMax(cmi + 1, __float_as_int(ml));
#pragma unroll
      for (int k = 0; k < 4; ++k) atomicMax(cmi + 2 + k, __float_as_int(mxk[k]));
      if (!clean) atomicAnd(cmi + 6, 0);
    }
  }
  __syncthreads();
}

// Pass 1: one warp per row; row max, 64-entry sub-block sums (8-lane
// contract per sub-block, sequential tail) and the raw row total
// (sequential over sub-blocks) — exp_row_store (kernels.cpp:93-116).
// ws layout per combine: m[N] raw[N] scale[N] total[N] prefix[N] sub[N*nsub]
//
// Row max (fast = 1): an FP32 screen first. Every entry's FP32 estimate a_j
// (est32_pair) is within E of the FP64 fill, E = 2^-18 (max|base| + |sl| +
// max|lwr| + sum_k (max|x_k - c_k| + |mu_k - c_k|)^2), c = column 0's
// coordinates (the FP32 copies are centred on it; the centring subtractions
// are FP64, their rounding ~2^-53 |x| is far below E) — 8x the worst-case
// rounding of the estimate's FP32 operations on operands of those magnitudes
// (|coef| scales the square for the d = 1 model classes). Only entries with
// a_j >= max a - 3E can hold the FP64 maximum; they are evaluated in FP64
// (usually one per row), so the row max is the same double as the full FP64
// scan's at a fraction of its instructions. The screen runs only when the
// inputs are clean (finite states and row mean, finite left weight, no NaN
// or +inf base / right weight): then no FP64 entry can be NaN, and no
// estimate NaN or +inf. Other rows run the full FP64 scan with its NaN
// check. The sum pass then evaluates every entry in FP64 exactly as before
// (exp_w_le0 = exp_w on its domain x <= 0).
template <int MC, int D, int MODE>
__device__ __forceinline__ void c64_row(const Bufs& b, const LevelArgs& la, const Col64& C,
                                        const double* mu, double coef, double sl, int i, int c,
                                        bool fast, double* wm, double* wraw, double* wsub) {
  const int N = b.N, nsub = (N + kSub - 1) / kSub;
  const int lane = threadIdx.x & 31;
  double mx = -CUDART_INF;
  bool full = !fast;
  if (fast) {
    bool clean = __float_as_int(C.cm[6]) != 0 && isfinite(sl);
    float2 nmu[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) nmu[k] = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < D && k < 4; ++k) {
      const float m = (float)DSUB(mu[k], C.cen[k]);
      clean &= isfinite(mu[k]) && isfinite(m);
      nmu[k] = make_float2(-m, -m);
    }
    const float coeff = (float)coef;
    float es = C.cm[0] + fabsf((float)sl) + (MODE == 2 ? C.cm[1] : 0.f);
    if (MC == kLGN) {
#pragma unroll
      for (int k = 0; k < D && k < 4; ++k) {
        const float s = C.cm[2 + k] + fabsf(nmu[k].x);
        es += s * s;
      }
    } else {
      const float s = C.cm[2] + fabsf(nmu[0].x);
      es += fabsf(coeff) * s * s;
    }
    const float E = es * 0x1p-18f;
    const float cfv = MC == kLGN ? -0.5f : coeff;
    const float2 cf = make_float2(cfv, cfv);
    if (!clean || !(E < CUDART_INF_F)) {
      full = true;
    } else {
      float b1 = -CUDART_INF_F, b2 = -CUDART_INF_F;
      int i1 = 0;
      auto upd = [&](float a, int j) {
        const bool up = a > b1;
        b2 = fmaxf(b2, fminf(a, b1));
        i1 = up ? j : i1;
        b1 = fmaxf(b1, a);
      };
      for (int s = 0; s < nsub; ++s) {  // pair 32 s + lane: columns 64 s + lane, + 32
        const float2 a = est32_pair<MC, D, MODE>(nmu, cf, C, 32 * s + lane);
        upd(a.x, kSub * s + lane);
        upd(a.y, kSub * s + 32 + lane);
      }
      float M = b1;
      for (int o = 16; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(~0u, M, o));
      if (M == -CUDART_INF_F) {
        full = true;  // every estimate -inf: let the FP64 scan decide
      } else {
        const float thr = M - 3.f * E;
        double e = -CUDART_INF;
        if (b2 >= thr) {  // several candidates on this lane (near-ties): rescan
          for (int s = 0; s < nsub; ++s) {
            const float2 a = est32_pair<MC, D, MODE>(nmu, cf, C, 32 * s + lane);
            if (a.x >= thr) e = fmax(e, fill64m<MC, D, MODE>(coef, mu, C, cpad(kSub * s + lane), sl));
            if (a.y >= thr)
              e = fmax(e, fill64m<MC, D, MODE>(coef, mu, C, cpad(kSub * s + 32 + lane), sl));
          }
        } else if (b1 >= thr) {
          e = fill64m<MC, D, MODE>(coef, mu, C, cpad(i1), sl);
        }
        for (int o = 16; o; o >>= 1) e = fmax(e, __shfl_xor_sync(~0u, e, o));
        mx = e;
      }
    }
  }
  if (full) {  // max (reduce_max, kernels.cpp:26-36)
    int nan = 0;
    for (int j = lane; j < N; j += 32) {
      const double v = fill64m<MC, D, MODE>(coef, mu, C, cpad(j), sl);
      nan |= isnan(v);
      mx = fmax(mx, v);
    }
    for (int o = 16; o; o >>= 1) {
      mx = fmax(mx, __shfl_xor_sync(~0u, mx, o));
      nan |= __shfl_xor_sync(~0u, nan, o);
    }
    if (nan) {
      if (lane == 0) raise_err(b.err, DSMC_E_DOMAIN, c, la.level, kReasonNaN);
      mx = -CUDART_INF;
    }
  }
  if (lane == 0) wm[i] = mx;
  double* srow = wsub + (size_t)i * nsub;
  if (mx == -CUDART_INF) {  // dead row: zero total, never selected
    for (int s = lane; s < nsub; s += 32) srow[s] = 0.0;
    if (lane == 0) wraw[i] = 0.0;
    return;
  }
  const int grp = lane >> 3, l8 = lane & 7;
  double tot = 0.0;
  for (int s0 = 0; s0 < nsub; s0 += 4) {
    const int s = s0 + grp;
    const bool act = s < nsub;
    const int j0 = s * kSub;
    const int len = act ? min(kSub, N - j0) : 0;
    const int len8 = len & ~7;
    const int cp0 = s * 72 + l8;  // cpad(j0 + l8)
    double acc = 0.0;
    if (len8 == kSub) {
#pragma unroll
      for (int q = 0; q < kSub; q += 8)
        acc = DADD(acc, exp_w_le0(DSUB(fill64m<MC, D, MODE>(coef, mu, C, cp0 + q, sl), mx)));
    } else {
      for (int q = 0; q < len8; q += 8)
        acc = DADD(acc, exp_w_le0(DSUB(fill64m<MC, D, MODE>(coef, mu, C, cp0 + q, sl), mx)));
    }
    double a8[8];
#pragma unroll
    for (int l = 0; l < 8; ++l) a8[l] = __shfl_sync(~0u, acc, (lane & ~7) + l);
    double bs = 0.0;
    if (act && l8 == 0) {
      bs = combine8(a8);
      for (int j = j0 + len8; j < j0 + len; ++j)
        bs = DADD(bs, exp_w_le0(DSUB(fill64m<MC, D, MODE>(coef, mu, C, cpad(j), sl), mx)));
      srow[s] = bs;
    }
    // raw row total: sequential over sub-blocks, in lane 0
#pragma unroll
    for (int g4 = 0; g4 < 4; ++g4) {
      const double v = __shfl_sync(~0u, bs, 8 * g4);
      if (s0 + g4 < nsub) tot = DADD(tot, v);
    }
  }
  if (lane == 0) wraw[i] = tot;
}

constexpr int kC64Threads = 512;   // 16 warps, one row at a time each
constexpr int kC64Rows = 128;      // rows per CTA (the column stage is shared)
template <int MC, int D>
__global__ void __launch_bounds__(kC64Threads, 2) c64_rows(Bufs b, LevelArgs la, int fast) {
  extern __shared__ double smem[];
  const int k = la.k0 + blockIdx.y, ch = blockIdx.z;
  const int N = b.N;
  constexpr int d = D;
  Side L, R;
  CombineGeom g;
  sides(b, la, k, L, R, g);
  const DevModel& M = b.models[ch];
  const TimeConst& tc = b.tc[(size_t)ch * b.Kt + b.t0 + g.c];
  Col64 C;
  stage_cols<MC, D>(b, la, ch, R, M, tc, smem, C, fast != 0);
  // per (chain, combine of the chunk) workspace
  double* ws = la.ws + ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * la.ws_comb;
  double *wm = ws, *wraw = ws + N, *wsub = ws + 5 * (size_t)N;
  const bool lnonuni = L.leaf && !b.UNI[(size_t)ch * b.K + L.t];
  const double coef = row_coef<MC>(M, b.t0 + g.c);
  const int warp = threadIdx.x >> 5;
  const double* XL = b.X64 + ((size_t)ch * b.K + L.t) * N * d;
  // the CTA's row means and left weights, one thread per row (a warp per row
  // would evaluate each 32 times over)
  double* MU = smem + cols64_bytes(N, D, fast != 0) / sizeof(double);  // [kC64Rows][D]
  double* SL = MU + kC64Rows * D;                                        // [kC64Rows]
  for (int r = threadIdx.x; r < kC64Rows; r += kC64Threads) {
    const int i = blockIdx.x * kC64Rows + r;
    if (i >= N) break;
    const uint32_t p = map_last(b, la, ch, L, i);
    double xl[D], mu[D];
#pragma unroll
    for (int q = 0; q < d; ++q) xl[q] = XL[(size_t)p * d + q];
    row_mean<MC, D>(M, tc, b.t0 + g.c, xl, mu);
#pragma unroll
    for (int q = 0; q < d; ++q) MU[r * D + q] = mu[q];
    SL[r] = lnonuni ? b.LW64[((size_t)ch * b.K + L.t) * N + i] : 0.0;
  }
  __syncthreads();
  for (int r = warp; r < kC64Rows; r += kC64Threads / 32) {
    const int i = blockIdx.x * kC64Rows + r;
    if (i >= N) break;
    double mu[D];
#pragma unroll
    for (int q = 0; q < d; ++q) mu[q] = MU[r * D + q];
    const double sl = SL[r];
    // the leaf-weight case of fill64 (uniform over the row)
    if (C.has_lwr)
      c64_row<MC, D, 2>(b, la, C, mu, coef, sl, i, g.c, fast != 0, wm, wraw, wsub);
    else if (lnonuni && sl != 0.0)
      c64_row<MC, D, 1>(b, la, C, mu, coef, sl, i, g.c, fast != 0, wm, wraw, wsub);
    else
      c64_row<MC, D, 0>(b, la, C, mu, coef, sl, i, g.c, fast != 0, wm, wraw, wsub);
  }
}

// Inversion inside a sub-block (select_sorted, resampling.cpp:109-153 /
// Appendix A): the first j in [j0, j1) whose running sum c3 (from c3 = c2b)
// exceeds `local`; past the end, the last positive entry (rounding spill).
template <int MC, int D, int MODE>
__device__ __forceinline__ int walk64(double coef, const double* mu, const Col64& C, double sl,
                                      double mrow, double c3, double local, int j0, int j1) {
  for (int jb = j0; jb < j1; jb += 8) {
    double e[8];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      e[q] = jb + q < j1 ? exp_w_le0(DSUB(fill64m<MC, D, MODE>(coef, mu, C, cpad(jb + q), sl), mrow))
                         : 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (jb + q >= j1) break;
      c3 = DADD(c3, e[q]);
      if (local < c3) return jb + q;
    }
  }
  int j = j1 - 1;  // spill: clamp to the last positive entry
  while (j > 0 && !(exp_w(DSUB(fill64m<MC, D, MODE>(coef, mu, C, cpad(j), sl), mrow)) > 0.0)) --j;
  return j;
}

// Cross-row combination of the pair table (resampling.cpp:92-102), one warp
// per combine (any number of combines per CTA): g = max_i m_i, per-row scale
// exp_w(m_i - g) and total scale_i raw_i, the grand total under the 8-lane
// contract and the sequential inclusive prefix of the totals (the walk's
// cum), log mean weight. The prefix is one dependent chain of N additions per
// combine; running it here, one warp per combine with many combines in flight
// per SM, keeps it off the sampler CTAs. ws extras: [5N + N nsub] = g,
// [+1] = grand total.
__global__ void __launch_bounds__(256) c64_cdf(Bufs b, LevelArgs la, int nk) {
  const int w = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= nk * b.B) return;
  const int kk = w % nk, ch = w / nk;  // ws slot of (chain, combine) as c64_rows
  const int k = la.k0 + kk;
  const int N = b.N, nsub = (N + kSub - 1) / kSub;
  double* ws = la.ws + (size_t)w * la.ws_comb;
  double *wm = ws, *wraw = ws + N, *wscale = ws + 2 * (size_t)N, *wtot = ws + 3 * (size_t)N,
         *wpre = ws + 4 * (size_t)N, *wx = ws + (size_t)N * (5 + nsub);
  double mx = -CUDART_INF;
  for (int i = lane; i < N; i += 32) mx = fmax(mx, wm[i]);
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(~0u, mx, o));
  if (lane == 0) wx[0] = mx;
  if (mx == -CUDART_INF) {
    if (lane == 0) {
      CombineGeom g = combine_geom(la.level, k, b.K);
      raise_err(b.err, DSMC_E_RUNTIME, g.c, la.level, kReasonZeroTable);
    }
    return;
  }
  for (int i = lane; i < N; i += 32) {
    const double sc = exp_w_le0(DSUB(wm[i], mx));  // wm[i] <= g
    wscale[i] = sc;
    wtot[i] = DMUL(sc, wraw[i]);
  }
  __syncwarp();
  // grand = reduce_sum(row_total) (8-lane contract)
  const int n8 = N & ~7;
  double acc = 0.0;
  if (lane < 8)
    for (int i = lane; i < n8; i += 8) acc = DADD(acc, wtot[i]);
  double a8[8];
#pragma unroll
  for (int l = 0; l < 8; ++l) a8[l] = __shfl_sync(~0u, acc, l);
  if (lane == 0) {
    double tot = combine8(a8);
    for (int i = n8; i < N; ++i) tot = DADD(tot, wtot[i]);
    wx[1] = tot;
    double cum = 0.0;  // sequential inclusive prefix (the walk's cum)
#pragma unroll 8
    for (int i = 0; i < N; ++i) {
      cum = DADD(cum, wtot[i]);
      wpre[i] = cum;
    }
    b.LMW[(size_t)ch * b.T + la.cursor + k] = DADD(mx, log(tot));
  }
}

// Pass 2: one CTA per combine: per-slot inversion over the prefix c64_cdf
// left in ws (Appendix A), ancestor maps, block log Z.
#ifndef DSMC_C64S_MINB
#define DSMC_C64S_MINB 2
#endif
// shared memory of c64_sample beyond the column stage: the row prefix, and in
// sorted mode the slot records, order and sub-block counts
__host__ __device__ inline size_t c64s_extra(int N, bool sorted) {
  const int nsub = (N + kSub - 1) / kSub;
  return sizeof(double) * (size_t)N + (sorted ? (size_t)N * (16 + 8 + 4) + 4 * (size_t)nsub : 0);
}
template <int MC, int D>
__global__ void __launch_bounds__(256, DSMC_C64S_MINB) c64_sample(Bufs b, LevelArgs la,
                                                  int systematic, int sorted) {
  extern __shared__ double smem[];
  const int k = la.k0 + blockIdx.x, ch = blockIdx.z;
  const int N = b.N, nsub = (N + kSub - 1) / kSub;
  constexpr int d = D;
  double* ws = la.ws + ((size_t)blockIdx.z * gridDim.x + blockIdx.x) * la.ws_comb;
  double *wm = ws, *wscale = ws + 2 * (size_t)N, *wtot = ws + 3 * (size_t)N,
         *wpre = ws + 4 * (size_t)N, *wsub = ws + 5 * (size_t)N;
  const double* wx = ws + (size_t)N * (5 + nsub);
  if (wx[0] == -CUDART_INF) return;  // zero table: c64_cdf raised the error
  Side L, R;
  CombineGeom g;
  sides(b, la, k, L, R, g);
  const DevModel& M = b.models[ch];
  const TimeConst& tc = b.tc[(size_t)ch * b.Kt + b.t0 + g.c];
  Col64 C;
  stage_cols<MC, D>(b, la, ch, R, M, tc, smem, C);
  const int tid = threadIdx.x;
  const double grand = wx[1];
  double* spre = smem + cols64_bytes(N, D, false) / sizeof(double);  // [N] row prefix
  for (int q = tid; q < N; q += blockDim.x) spre[q] = wpre[q];
  __syncthreads();
  const bool lnonuni = L.leaf && !b.UNI[(size_t)ch * b.K + L.t];
  const double coef = row_coef<MC>(M, b.t0 + g.c);
  const int off = b.conditional ? 1 : 0;
  const uint64_t node = b.conditional
                            ? (static_cast<uint64_t>(static_cast<uint32_t>(k + la.node_off)) |
                               (static_cast<uint64_t>(b.sweep) << 32))
                            : static_cast<uint64_t>(k + la.node_off);
  const StreamId id = stream_id(b.seeds[ch], la.key_level, node,
                                DSMC_ROLE_PAIR_RESAMPLE, 0);
  double u0 = 0.0, step = 0.0;
  if (systematic) {
    u0 = u64_uniform(stream_u64(id, 0));
    step = DDIV(grand, (double)la.n_out);
  }
  const size_t gidx = (size_t)ch * b.T + la.cursor + k;
  uint32_t* PL = b.PL + gidx * N;
  uint32_t* PR = b.PR + gidx * N;
  const double* XL = b.X64 + ((size_t)ch * b.K + L.t) * N * d;
  // the column of slot m in row `row`, sub-block s: first j with local < c3,
  // c3 the running sum from c2b (the reference's sequential walk); the
  // weights of 8 entries are evaluated together (independent exp_w chains),
  // the sum and the test stay in order
  auto finish = [&](int m, int row, int s, double local, double c2b) {
    const uint32_t pl = map_last(b, la, ch, L, row);
    double xl[D], mu[D];
    for (int q = 0; q < d; ++q) xl[q] = XL[(size_t)pl * d + q];
    row_mean<MC, D>(M, tc, b.t0 + g.c, xl, mu);
    const double sl = lnonuni ? b.LW64[((size_t)ch * b.K + L.t) * N + row] : 0.0;
    const double mrow = wm[row];
    const int j0 = s * kSub, j1 = min(j0 + kSub, N);
    const int j = C.has_lwr ? walk64<MC, D, 2>(coef, mu, C, sl, mrow, c2b, local, j0, j1)
                  : (lnonuni && sl != 0.0)
                      ? walk64<MC, D, 1>(coef, mu, C, sl, mrow, c2b, local, j0, j1)
                      : walk64<MC, D, 0>(coef, mu, C, sl, mrow, c2b, local, j0, j1);
    PL[m + off] = (uint32_t)row;
    PR[m + off] = (uint32_t)j;
  };
  // sorted mode: per-slot records (local, c2b | row, s), sub-block counts, order
  double* RLC = spre + N;                                    // [2 n_out]
  int2* RRS = reinterpret_cast<int2*>(RLC + 2 * (size_t)N);  // [n_out]
  int* ORD = reinterpret_cast<int*>(RRS + N);                // [n_out]
  int* CNT = ORD + N;                                        // [nsub]
  if (sorted) {
    for (int q = tid; q < nsub; q += blockDim.x) CNT[q] = 0;
    __syncthreads();
  }
  // each thread takes 4 consecutive slots: one Philox block gives their
  // uniforms (slot m <-> u64 number m of the stream, rng.cpp:45-68)
  for (int q0 = 4 * tid; q0 < la.n_out; q0 += 4 * blockDim.x) {
    U64x4 blk;
    if (!systematic) blk = stream_block(id, (uint64_t)q0 >> 2);
#pragma unroll 1
    for (int qq = 0; qq < 4; ++qq) {
      const int m = q0 + qq;
      if (m >= la.n_out) break;
      const double pt = systematic ? DMUL(DADD(u0, (double)m), step)
                                   : DMUL(u64_uniform(blk.v[qq]), grand);
      int lo = 0, hi = N;  // first i with pt < S_i (prefix staged in shared memory)
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (pt < spre[mid]) hi = mid;
        else lo = mid + 1;
      }
      const int i = lo < N ? lo : N - 1;
      const double before = i > 0 ? spre[i - 1] : 0.0;
      int row = i;
      while (row > 0 && wtot[row] <= 0.0) --row;
      double local = DDIV(DSUB(pt, before), wscale[row]);
      if (!(local >= 0.0)) local = 0.0;
      const double* srow = wsub + (size_t)row * nsub;
      int s = 0;
      double c2b = 0.0, c2;
      {  // the sub-block walk; its loads issued 16 at a time ahead of the
         // sequential sum
        double sv[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) sv[q] = q < nsub ? srow[q] : 0.0;
        c2 = sv[0];
        bool done = local < c2 || nsub == 1;
#pragma unroll
        for (int q = 1; q < 16; ++q) {
          if (!done) {
            c2b = c2;
            s = q;
            c2 = DADD(c2, sv[q]);
            done = local < c2 || q + 1 >= nsub;
          }
        }
        while (!done) {  // nsub > 16
          c2b = c2;
          ++s;
          c2 = DADD(c2, srow[s]);
          done = local < c2 || s + 1 >= nsub;
        }
      }
      if (sorted) {
        RLC[2 * m] = local;
        RLC[2 * m + 1] = c2b;
        RRS[m] = make_int2(row, s);
        atomicAdd(&CNT[s], 1);
      } else {
        finish(m, row, s, local, c2b);
      }
    }
  }
  if (sorted) {
    // slots re-ordered by sub-block (CTA counting sort) so that a warp's
    // lanes recompute the same sub-block's records (shared-memory broadcasts
    // instead of bank conflicts); every slot's arithmetic is unchanged
    __syncthreads();
    if (tid < 32) {  // exclusive scan of the sub-block counts
      int carry = 0;
      for (int c0 = 0; c0 < nsub; c0 += 32) {
        const int c = c0 + tid < nsub ? CNT[c0 + tid] : 0;
        int v = c;
        for (int o = 1; o < 32; o <<= 1) {
          const int n = __shfl_up_sync(~0u, v, o);
          if (tid >= o) v += n;
        }
        if (c0 + tid < nsub) CNT[c0 + tid] = carry + v - c;
        carry += __shfl_sync(~0u, v, 31);
      }
    }
    __syncthreads();
    for (int m = tid; m < la.n_out; m += blockDim.x) ORD[atomicAdd(&CNT[RRS[m].y], 1)] = m;
    __syncthreads();
    for (int o = tid; o < la.n_out; o += blockDim.x) {
      const int m = ORD[o];
      const int2 rs = RRS[m];
      finish(m, rs.x, rs.y, RLC[2 * m], RLC[2 * m + 1]);
    }
  }
  if (b.conditional && tid == 0) {
    PL[0] = 0;
    PR[0] = 0;
  }
  // (the conditional reference-pair check is done by the caller kernel)
  __syncthreads();
  // ancestor maps: first'[q] = L.first[l_q], last'[q] = R.last[r_q]
  const size_t nbase = ((size_t)ch * b.cap + k) * N;
  for (int q = tid; q < N; q += blockDim.x) {
    la.first_next[nbase + q] = map_first(b, la, ch, L, PL[q]);
    la.last_next[nbase + q] = map_last(b, la, ch, R, PR[q]);
  }
  if (tid == 0) {
    const double logn = log((double)N);
    const bool luni = !L.leaf || b.UNI[(size_t)ch * b.K + L.t];
    const bool runi = !R.leaf || b.UNI[(size_t)ch * b.K + R.t];
    const double shift = DADD(luni ? -logn : 0.0, runi ? -logn : 0.0);
    const double ll = block_lnc(b, la, ch, L, g.a);
    const double rl = block_lnc(b, la, ch, R, g.c);
    const double lmw = b.LMW[gidx];
    la.blnc_next[(size_t)ch * b.cap + k] = DADD(DADD(DADD(ll, rl), lmw), shift);
  }
}

// ------------------------------------------------------------- lazy
// Entry probe (make_pair_source log_weight_at, smoother.cpp:163-169).
struct Probe64 {
  const DevModel* M;
  const TimeConst* tc;
  const double *XL, *XR, *lwl, *lwr;
  const Bufs* b;
  const LevelArgs* la;
  int ch, c, d;
  Side L, R;
  __device__ double operator()(uint32_t i, uint32_t j, int* err) const {
    const uint32_t pi = map_last(*b, *la, ch, L, i);
    const uint32_t pj = map_first(*b, *la, ch, R, j);
    double v = cb_stitch_weight(*M, *tc, c, XL + (size_t)pi * d,
                                XR + (size_t)pj * d, err);
    if (lwl) v = DADD(v, lwl[i]);
    if (lwr) v = DADD(v, lwr[j]);
    return v;
  }
};

// One thread per output slot; substream m+1 (resampling.cpp:253,300).
__global__ void lazy64_kernel(Bufs b, LevelArgs la, int mh, size_t mh_steps) {
  const int k = la.k0 + blockIdx.y, ch = blockIdx.z;
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  const int N = b.N;
  Side L, R;
  CombineGeom g;
  sides(b, la, k, L, R, g);
  const bool lnonuni = L.leaf && !b.UNI[(size_t)ch * b.K + L.t];
  const bool rnonuni = R.leaf && !b.UNI[(size_t)ch * b.K + R.t];
  Probe64 P;
  P.M = &b.models[ch];
  P.tc = &b.tc[(size_t)ch * b.Kt + b.t0 + g.c];
  P.XL = b.X64 + ((size_t)ch * b.K + L.t) * N * b.d;
  P.XR = b.X64 + ((size_t)ch * b.K + R.t) * N * b.d;
  P.lwl = lnonuni ? b.LW64 + ((size_t)ch * b.K + L.t) * N : nullptr;
  P.lwr = rnonuni ? b.LW64 + ((size_t)ch * b.K + R.t) * N : nullptr;
  P.b = &b;
  P.la = &la;
  P.ch = ch;
  P.c = b.t0 + g.c;  // global cut: model data
  P.d = b.d;
  P.L = L;
  P.R = R;
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
    if (mh) {  // mh_lazy_pairs (resampling.cpp:250-279)
      uint32_t i = (uint32_t)(m % N), j = i;
      double cur = 0.0;
      bool have = false;
      for (size_t st = 0; st < mh_steps && !err; ++st) {
        const uint32_t pi = (uint32_t)s.index(N), pj = (uint32_t)s.index(N);
        const double lu = log(s.uniform_pos());
        if (!have) {
          cur = P(i, j, &err);
          ++evals;
          have = true;
        }
        const double prop = P(pi, pj, &err);
        ++evals;
        if (isnan(prop) || isnan(cur)) { err = DSMC_E_INVALID_ARGUMENT; why = kReasonNaN; }
        if (lu < DSUB(prop, cur)) {
          i = pi;
          j = pj;
          cur = prop;
        }
      }
      oi = i;
      oj = j;
    } else {  // rejection_lazy_pairs (resampling.cpp:296-321)
      if (!(b.bounded[ch] & 1)) { err = DSMC_E_INVALID_ARGUMENT; why = kReasonNoBound; }  // no finite bound
      double bound = P.tc->bound;
      if (P.lwl) bound = DADD(bound, b.LWMAX[(size_t)ch * b.K + L.t]);
      if (P.lwr) bound = DADD(bound, b.LWMAX[(size_t)ch * b.K + R.t]);
      bool ok = false;
      for (uint64_t trial = 0; trial < (1u << 24) && !err; ++trial) {
        const uint32_t i = (uint32_t)s.index(N), j = (uint32_t)s.index(N);
        const double lw = P(i, j, &err);
        ++evals;
        if (isnan(lw)) { err = DSMC_E_INVALID_ARGUMENT; why = kReasonNaN; }
        if (DSUB(lw, bound) > 1e-9) { err = DSMC_E_INVALID_ARGUMENT; why = kReasonOverBound; }
        if (err) break;
        if (log(s.uniform_pos()) <= DSUB(lw, bound)) {
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
  // warp-aggregated evaluation count
  for (int o = 16; o; o >>= 1) evals += __shfl_xor_sync(~0u, evals, o);
  if ((threadIdx.x & 31) == 0 && evals) atomicAdd(b.evals + ch, evals);
}

// Ancestor maps + block meta after a lazy combine (no log Z: lazy
// resamplers never see the whole table, smoother.cpp:220-222).
__global__ void lazy_finish_kernel(Bufs b, LevelArgs la) {
  const int k = la.k0 + blockIdx.x, ch = blockIdx.z;
  const int N = b.N;
  Side L, R;
  CombineGeom g;
  sides(b, la, k, L, R, g);
  const size_t gidx = (size_t)ch * b.T + la.cursor + k;
  uint32_t* PL = b.PL + gidx * N;
  uint32_t* PR = b.PR + gidx * N;
  if (b.conditional && threadIdx.x == 0) {
    PL[0] = 0;
    PR[0] = 0;
  }
  __syncthreads();
  const size_t nbase = ((size_t)ch * b.cap + k) * N;
  for (int q = threadIdx.x; q < N; q += blockDim.x) {
    la.first_next[nbase + q] = map_first(b, la, ch, L, PL[q]);
    la.last_next[nbase + q] = map_last(b, la, ch, R, PR[q]);
  }
  if (threadIdx.x == 0) {
    la.blnc_next[(size_t)ch * b.cap + k] = CUDART_NAN;
    b.LMW[gidx] = CUDART_NAN;
  }
}

// Conditional combines require a finite reference pair (conditional.cpp:
// 97-103), checked through the scalar entry probe like the reference.
__global__ void refpair_check_kernel(Bufs b, LevelArgs la) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int ch = blockIdx.z;
  if (k >= la.np) return;
  Side L, R;
  CombineGeom g;
  sides(b, la, k, L, R, g);
  const int N = b.N;
  const bool lnonuni = L.leaf && !b.UNI[(size_t)ch * b.K + L.t];
  const bool rnonuni = R.leaf && !b.UNI[(size_t)ch * b.K + R.t];
  Probe64 P;
  P.M = &b.models[ch];
  P.tc = &b.tc[(size_t)ch * b.Kt + b.t0 + g.c];
  P.XL = b.X64 + ((size_t)ch * b.K + L.t) * N * b.d;
  P.XR = b.X64 + ((size_t)ch * b.K + R.t) * N * b.d;
  P.lwl = lnonuni ? b.LW64 + ((size_t)ch * b.K + L.t) * N : nullptr;
  P.lwr = rnonuni ? b.LW64 + ((size_t)ch * b.K + R.t) * N : nullptr;
  P.b = &b;
  P.la = &la;
  P.ch = ch;
  P.c = b.t0 + g.c;  // global cut: model data
  P.d = b.d;
  P.L = L;
  P.R = R;
  int err = 0;
  const double w = P(0, 0, &err);
  if (err || !isfinite(w)) raise_err(b.err, DSMC_E_INVALID_ARGUMENT, g.c, la.level, kReasonRefPair);
}

}  // namespace dsmc_dev

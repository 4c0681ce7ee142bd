// The reference's piecewise entry points on the device (included at the end
// of engine.cu, sharing its context, arena and run_tree):
//
//   dsmc_make_leaf        make_leaf (smoother.cpp:98-130): one leaf, FP64
//   dsmc_resample_blocks  resample_pairs on make_pair_source(L, R)
//                         (smoother.cpp:132-180 + resampling.cpp): the pair
//                         table of two caller-held blocks, evaluated and
//                         sampled on the device without materialising it
//   dsmc_resample_indices multinomial_indices / systematic_indices
//                         (resampling.cpp:360-460): one population
//   dsmc_lazy_*           mh_lazy_pairs / rejection_lazy_pairs
//                         (resampling.cpp:233-324) over a source only the
//                         caller can evaluate (host callbacks): the device
//                         keeps every slot's chain state and counter-addressed
//                         stream position and asks, round by round, for the
//                         entries its slots probe next.
#pragma once

namespace {

const char* reason_text(const ErrFlag& e, bool lazy) {
  switch (e.reason) {
    case kReasonZeroTable:
      return "all pair weights are zero; the blocks share no support under the model";
    case kReasonTrialCap:
      return "rejection resampling exceeded the trial cap; the bound is far too loose or the "
             "weights are degenerate";
    case kReasonOverBound: return "pair weight exceeds its stated upper bound";
    case kReasonNoBound: return "rejection resampling requires a finite log_upper_bound";
    case kReasonNaN: return lazy ? "pair weight is NaN" : "reduce_max: NaN entry";
    case kReasonLeafZero: return "every proposal draw has zero weight";
    default: return "device error";
  }
}

int upload_seed(dsmc_ctx* ctx, uint64_t seed, const uint64_t** out) {
  void* p;
  CU(ctx->arena.get("SEEDS", sizeof(uint64_t), &p));
  set_seed_kernel<<<1, 1, 0, ctx->stream>>>((uint64_t*)p, seed);
  LAUNCHED(ctx);
  *out = (const uint64_t*)p;
  return DSMC_OK;
}

// ------------------------------------------------------- index resampling
// One population (build_row_weights + select_row_sorted, resampling.cpp):
// w_i = exp_w(logw_i - m), total = exp_row_store's total (64-entry sub-block
// sums with the 8-lane contract, then their sequential sum), sequential
// prefix S_i = w_0 + ... + w_i; slot k picks min{i : pt_k < S_i} (n - 1 on
// spill) and walks back over dead entries — the sorted walk's result for the
// same point, so every slot searches independently (no sort).
__global__ void index_rows_kernel(const double* logw, int n, double* ws, ErrFlag* err) {
  // ws: [0] max, [1] total, [2..] w (n), then prefix (n), then sub sums
  __shared__ double red[32];
  __shared__ int nan_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) nan_s = 0;
  __syncthreads();
  double mx = -CUDART_INF;
  int nan = 0;
  for (int i = tid; i < n; i += blockDim.x) {
    nan |= isnan(logw[i]);
    mx = fmax(mx, logw[i]);
  }
  for (int o = 16; o; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(~0u, mx, o));
    nan |= __shfl_xor_sync(~0u, nan, o);
  }
  if (lane == 0) {
    red[warp] = mx;
    if (nan) atomicOr(&nan_s, 1);
  }
  __syncthreads();
  if (tid == 0) {
    double v = -CUDART_INF;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v = fmax(v, red[w]);
    red[0] = v;
  }
  __syncthreads();
  mx = red[0];
  if (nan_s) {
    if (tid == 0) raise_err(err, DSMC_E_DOMAIN, 0, 0, kReasonNaN);
    return;
  }
  if (mx == -CUDART_INF) {
    if (tid == 0) raise_err(err, DSMC_E_RUNTIME, 0, 0, kReasonZeroTable);
    return;
  }
  double* w = ws + 2;
  double* pre = w + n;
  const int nsub = (n + kSub - 1) / kSub;
  double* sub = pre + n;
  for (int i = tid; i < n; i += blockDim.x) w[i] = exp_w(DSUB(logw[i], mx));
  __syncthreads();
  // sub-block sums: one 8-lane group per sub-block (exp_poly.hpp:66-84)
  const int grp = tid >> 3, l8 = tid & 7, ngrp = blockDim.x >> 3;
  for (int s0 = 0; s0 < nsub; s0 += ngrp) {
    const int s = s0 + grp;
    const bool act = s < nsub;
    const int j0 = s * kSub, len = act ? min(kSub, n - j0) : 0, len8 = len & ~7;
    double acc = 0.0;
    for (int q = 0; q < len8; q += 8) acc = DADD(acc, w[j0 + q + l8]);
    double a8[8];
    for (int l = 0; l < 8; ++l) a8[l] = __shfl_sync(~0u, acc, (lane & ~7) + l);
    if (act && l8 == 0) {
      double bs = combine8(a8);
      for (int j = j0 + len8; j < j0 + len; ++j) bs = DADD(bs, w[j]);
      sub[s] = bs;
    }
  }
  __syncthreads();
  if (tid == 0) {
    double tot = 0.0;
    for (int s = 0; s < nsub; ++s) tot = DADD(tot, sub[s]);
    double cum = 0.0;
    for (int i = 0; i < n; ++i) {
      cum = DADD(cum, w[i]);
      pre[i] = cum;
    }
    ws[0] = mx;
    ws[1] = tot;
  }
}

__global__ void index_select_kernel(const double* ws, int n, int n_out, int systematic,
                                    uint64_t seed, uint32_t level, uint64_t node, int role,
                                    uint32_t* idx) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_out) return;
  const double total = ws[1];
  const double* w = ws + 2;
  const double* pre = w + n;
  const StreamId id = stream_id(seed, level, node, role, 0);
  double pt;
  if (systematic) {
    const double u = u64_uniform(stream_u64(id, 0));
    pt = DMUL(DADD(u, (double)k), DDIV(total, (double)n_out));
  } else {
    pt = DMUL(u64_uniform(stream_u64(id, k)), total);
  }
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (pt < pre[mid]) hi = mid;
    else lo = mid + 1;
  }
  int pick = lo < n ? lo : n - 1;
  while (pick > 0 && !(w[pick] > 0.0)) --pick;
  idx[k] = (uint32_t)pick;
}

// ------------------------------------------------ caller-evaluated lazy
struct LazyState {
  int resampler = -1;
  size_t n = 0, n_out = 0, mh_steps = 0;
  double bound = 0.0;
  uint64_t seed = 0, node = 0;
  uint32_t level = 0;
  int role = DSMC_ROLE_PAIR_RESAMPLE;
  uint32_t round = 0;
  size_t n_probes = 0;
  uint64_t evals = 0;
  // device arrays (arena): per slot i, j, cur value, probe position, done;
  // per probe i, j, value; counters
  uint32_t *ci = nullptr, *cj = nullptr, *pi = nullptr, *pj = nullptr;
  int* pos = nullptr;
  double *cv = nullptr, *val = nullptr;
  uint8_t* done = nullptr;
  unsigned int* count = nullptr;
  ErrFlag* err = nullptr;
  std::vector<uint32_t> hi, hj;  // host copy of the current probes
};

constexpr uint32_t kLazyTrialCap = 1u << 24;  // kRejectionTrialCap (resampling.cpp:23)

// Round r: decide slot m's probes of round r - 1 (values in val[pos[m]..]),
// then emit its probes of round r. MH (resampling.cpp:258-275): step b draws
// u64s 3b, 3b+1 (proposal i, j) and 3b+2 (acceptance uniform); the current
// entry is probed together with the first proposal. Rejection (:302-315):
// trial r draws 3r, 3r+1 (i, j) and 3r+2 (uniform).
__global__ void lazy_round_kernel(int mh, int n, int n_out, uint32_t mh_steps, double bound,
                                  uint64_t seed, uint32_t level, uint64_t node, int role,
                                  uint32_t round, uint32_t* ci, uint32_t* cj, double* cv,
                                  int* pos, uint8_t* done, const double* val, uint32_t* pi,
                                  uint32_t* pj, unsigned int* count, ErrFlag* err) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n_out || done[m]) return;
  const StreamId id = stream_id(seed, level, node, role, (uint64_t)m + 1);
  if (round > 0) {  // decide round - 1
    const uint64_t q = 3ull * (round - 1);
    const int p = pos[m];
    if (mh) {
      double cur = cv[m];
      int vp = p;
      if (round == 1) {
        cur = val[vp++];
        if (isnan(cur)) {
          raise_err(err, DSMC_E_INVALID_ARGUMENT, 0, 0, kReasonNaN);
          return;
        }
      }
      const double prop = val[vp];
      if (isnan(prop)) {
        raise_err(err, DSMC_E_INVALID_ARGUMENT, 0, 0, kReasonNaN);
        return;
      }
      const double lu = log(u64_uniform_pos(stream_u64(id, q + 2)));
      if (lu < DSUB(prop, cur)) {  // -inf - -inf is NaN: stays put
        ci[m] = (uint32_t)u64_index(stream_u64(id, q), (uint64_t)n);
        cj[m] = (uint32_t)u64_index(stream_u64(id, q + 1), (uint64_t)n);
        cur = prop;
      }
      cv[m] = cur;
      if (round == mh_steps) {
        done[m] = 1;
        return;
      }
    } else {
      const double lw = val[p];
      if (isnan(lw)) {
        raise_err(err, DSMC_E_INVALID_ARGUMENT, 0, 0, kReasonNaN);
        return;
      }
      if (DSUB(lw, bound) > 1e-9) {
        raise_err(err, DSMC_E_INVALID_ARGUMENT, 0, 0, kReasonOverBound);
        return;
      }
      if (log(u64_uniform_pos(stream_u64(id, q + 2))) <= DSUB(lw, bound)) {
        ci[m] = (uint32_t)u64_index(stream_u64(id, q), (uint64_t)n);
        cj[m] = (uint32_t)u64_index(stream_u64(id, q + 1), (uint64_t)n);
        done[m] = 1;
        return;
      }
      if (round >= kLazyTrialCap) {
        raise_err(err, DSMC_E_RUNTIME, 0, 0, kReasonTrialCap);
        return;
      }
    }
  }
  // emit round `round`
  const uint64_t q = 3ull * round;
  const uint32_t a = (uint32_t)u64_index(stream_u64(id, q), (uint64_t)n);
  const uint32_t c = (uint32_t)u64_index(stream_u64(id, q + 1), (uint64_t)n);
  const int first = mh && round == 0;
  const unsigned int at = atomicAdd(count, first ? 2u : 1u);
  pos[m] = (int)at;
  if (first) {
    pi[at] = ci[m];
    pj[at] = cj[m];
    pi[at + 1] = a;
    pj[at + 1] = c;
  } else {
    pi[at] = a;
    pj[at] = c;
  }
}

__global__ void lazy_init_kernel(int n, int n_out, uint32_t* ci, uint32_t* cj, uint8_t* done) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n_out) return;
  ci[m] = cj[m] = (uint32_t)(m % n);  // the identity pair (m mod n, m mod n)
  done[m] = 0;
}

LazyState& lazy_state(dsmc_ctx* ctx) {
  static thread_local std::map<dsmc_ctx*, LazyState> states;  // one host thread per context
  return states[ctx];
}

int lazy_launch(dsmc_ctx* ctx, LazyState& L) {
  auto s = ctx->stream;
  CU(cudaMemsetAsync(L.count, 0, sizeof(unsigned int), s));
  const int nb = (int)((L.n_out + 255) / 256);
  lazy_round_kernel<<<nb, 256, 0, s>>>(L.resampler == DSMC_MH_LAZY, (int)L.n, (int)L.n_out,
                                       (uint32_t)L.mh_steps, L.bound, L.seed, L.level, L.node,
                                       L.role, L.round, L.ci, L.cj, L.cv, L.pos, L.done, L.val,
                                       L.pi, L.pj, L.count, L.err);
  LAUNCHED(ctx);
  CU(cudaGetLastError());
  unsigned int cnt = 0;
  ErrFlag e;
  CU(cudaMemcpyAsync(&cnt, L.count, sizeof cnt, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(&e, L.err, sizeof e, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (e.code) {
    L.resampler = -1;
    return set_err(ctx, e.code, reason_text(e, true));
  }
  L.n_probes = cnt;
  L.hi.resize(cnt);
  L.hj.resize(cnt);
  if (cnt) {
    CU(cudaMemcpyAsync(L.hi.data(), L.pi, cnt * 4, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(L.hj.data(), L.pj, cnt * 4, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
  }
  ++L.round;
  return DSMC_OK;
}

}  // namespace

extern "C" {

int dsmc_make_leaf(dsmc_ctx* ctx, const dsmc_model_desc* model, int t, size_t n,
                   uint64_t seed, double* states, double* logw, int* weights_uniform,
                   double* log_norm_const) {
  if (!ctx || !model || !states) return DSMC_E_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  if (n == 0) return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "make_leaf: n must be >= 1");
  if (n > 0xffffffffu)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "make_leaf: n exceeds the 32-bit index range");
  if (t < 0 || t > model->horizon)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "make_leaf: time outside 0..horizon");
  dsmc_model_handle* h = nullptr;
  int rc = make_handle(ctx, model, 1, &h);
  if (rc) return rc;
  std::unique_ptr<dsmc_model_handle, void (*)(dsmc_model_handle*)> hold(h, free_handle);
  RunOpts o;
  o.precision = DSMC_FP64_PARITY;
  o.N = n;
  o.t0 = t;
  o.len = 1;
  o.compose = false;
  rc = upload_seed(ctx, seed, &o.seeds);
  if (rc) return rc;
  RunResult res;
  rc = run_tree(ctx, h, o, &res);
  if (rc) return rc;
  ErrFlag e;
  auto s = ctx->stream;
  uint8_t uni = 0;
  double lnc = NAN;
  CU(cudaMemcpyAsync(&e, res.err, sizeof e, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(states, res.X64, n * h->d * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (logw) CU(cudaMemcpyAsync(logw, res.LW64, n * sizeof(double), cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(&uni, window_state(ctx).b.UNI, 1, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(&lnc, res.LNC, sizeof(double), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (e.code) {
    if (e.reason == kReasonLeafZero)
      return set_err(ctx, e.code, "leaf " + std::to_string(t) +
                                      ": every proposal draw has zero weight");
    return set_err(ctx, e.code, e.reason == kReasonNaN ? "log_init_weight produced NaN"
                                                       : reason_text(e, false));
  }
  if (weights_uniform) *weights_uniform = uni;
  if (log_norm_const) *log_norm_const = lnc;
  return DSMC_OK;
}

int dsmc_resample_blocks(dsmc_ctx* ctx, const dsmc_model_desc* model,
                         const dsmc_pair_blocks* pb, int resampler, size_t n_out,
                         size_t mh_steps, uint64_t seed, uint32_t level, uint64_t node,
                         uint32_t* left, uint32_t* right, double* lmw, int* has_lmw,
                         uint64_t* weight_evals, int* biased) {
  if (!ctx || !model || !pb || !pb->left_states || !pb->right_states ||
      (n_out && (!left || !right)))
    return DSMC_E_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  const size_t n = pb->n;
  const int d = model->state_dim;
  if (n == 0) return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "pair weight source has n == 0");
  if (n_out > n)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT,
                   "block-pair source: n_out must not exceed the block size");
  if (pb->cut < 1 || pb->cut > model->horizon)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "make_stitch_row: time index outside [1, T]");
  if (resampler < 0 || resampler > 3)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "unknown resampler");
  const bool lazy = resampler >= 2;
  if (lazy && (n_out == 0 || (resampler == DSMC_MH_LAZY && mh_steps == 0))) {
    // identity coupling / nothing to draw: no evaluations (resampling.cpp:243-250)
    for (size_t m = 0; m < n_out; ++m) left[m] = right[m] = (uint32_t)(m % n);
    *lmw = NAN;
    *has_lmw = 0;
    *weight_evals = 0;
    *biased = resampler == DSMC_MH_LAZY;
    return DSMC_OK;
  }
  dsmc_model_handle* h = nullptr;
  int rc = make_handle(ctx, model, 1, &h);
  if (rc) return rc;
  std::unique_ptr<dsmc_model_handle, void (*)(dsmc_model_handle*)> hold(h, free_handle);
  // the two boundary slabs as a two-leaf window [cut - 1, cut] whose leaves
  // carry the blocks' normalised weights (uniform sides never enter the table)
  std::vector<double> X(2 * n * d), W(2 * n, 0.0), lwmax(2, 0.0);
  std::memcpy(X.data(), pb->left_states, n * d * sizeof(double));
  std::memcpy(X.data() + n * d, pb->right_states, n * d * sizeof(double));
  const double* lws[2] = {pb->left_logw, pb->right_logw};
  const uint8_t uni[2] = {(uint8_t)(pb->left_uniform || !pb->left_logw),
                          (uint8_t)(pb->right_uniform || !pb->right_logw)};
  for (int side = 0; side < 2; ++side) {
    if (uni[side]) continue;
    double mx = -INFINITY;
    for (size_t i = 0; i < n; ++i) {
      if (std::isnan(lws[side][i]))
        return set_err(ctx, DSMC_E_DOMAIN, "reduce_max: NaN entry");
      mx = std::max(mx, lws[side][i]);
      W[side * n + i] = lws[side][i];
    }
    lwmax[side] = mx;
  }
  RunOpts o;
  o.precision = DSMC_FP64_PARITY;
  o.resampler = resampler;
  o.mh_steps = mh_steps;
  o.N = n;
  o.n_out = (int)n_out;
  o.t0 = pb->cut - 1;
  o.len = 2;
  o.compose = false;
  o.inj_x = X.data();
  o.inj_lw = W.data();
  o.inj_uni = uni;
  o.inj_lwmax = lwmax.data();
  o.key_level = (int)level;
  o.key_node = (long long)node;
  rc = upload_seed(ctx, seed, &o.seeds);
  if (rc) return rc;
  RunResult res;
  rc = run_tree(ctx, h, o, &res);
  if (rc) return rc;
  ErrFlag e;
  double lm = NAN;
  unsigned long long ev = 0;
  auto s = ctx->stream;
  CU(cudaMemcpyAsync(&e, res.err, sizeof e, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(left, res.PL, n_out * 4, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(right, res.PR, n_out * 4, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(&lm, res.LMW, 8, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(&ev, res.evals, 8, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (e.code) return set_err(ctx, e.code, reason_text(e, lazy));
  *has_lmw = lazy ? 0 : 1;
  *lmw = lazy ? NAN : lm;
  *weight_evals = lazy ? ev : (uint64_t)n * n;
  *biased = resampler == DSMC_MH_LAZY;
  return DSMC_OK;
}

int dsmc_resample_indices(dsmc_ctx* ctx, int resampler, const double* logw, size_t n,
                          size_t n_out, uint64_t seed, uint32_t level, uint64_t node, int role,
                          uint32_t* idx, double* max_logw, double* total) {
  if (!ctx || !logw || (n_out && !idx)) return DSMC_E_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  if (n == 0) return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "weight vector has n == 0");
  if (resampler != DSMC_MULTINOMIAL && resampler != DSMC_SYSTEMATIC)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT,
                   "index resampling: only the dense schemes (multinomial, systematic)");
  Arena& A = ctx->arena;
  void* p;
  auto s = ctx->stream;
  const size_t nsub = (n + kSub - 1) / kSub;
  CU(A.get("IXLW", n * 8, &p));
  double* dlw = (double*)p;
  CU(cudaMemcpyAsync(dlw, logw, n * 8, cudaMemcpyHostToDevice, s));
  CU(A.get("IXWS", (2 + 2 * n + nsub) * 8, &p));
  double* ws = (double*)p;
  CU(A.get("IXOUT", std::max<size_t>(n_out, 1) * 4, &p));
  uint32_t* didx = (uint32_t*)p;
  CU(A.get("IXERR", sizeof(ErrFlag), &p));
  ErrFlag* derr = (ErrFlag*)p;
  CU(cudaMemsetAsync(derr, 0, sizeof(ErrFlag), s));
  index_rows_kernel<<<1, 256, 0, s>>>(dlw, (int)n, ws, derr);
  LAUNCHED(ctx);
  ErrFlag e;
  CU(cudaMemcpyAsync(&e, derr, sizeof e, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (e.code)
    return set_err(ctx, e.code, e.reason == kReasonNaN ? "reduce_max: NaN entry"
                                                       : "all weights are zero");
  if (n_out) {
    index_select_kernel<<<(unsigned)((n_out + 255) / 256), 256, 0, s>>>(
        ws, (int)n, (int)n_out, resampler == DSMC_SYSTEMATIC, seed, level, node, role, didx);
    LAUNCHED(ctx);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(idx, didx, n_out * 4, cudaMemcpyDeviceToHost, s));
  }
  double mt[2];
  CU(cudaMemcpyAsync(mt, ws, 16, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (max_logw) *max_logw = mt[0];
  if (total) *total = mt[1];
  return DSMC_OK;
}

int dsmc_lazy_begin(dsmc_ctx* ctx, int resampler, size_t n, size_t n_out, size_t mh_steps,
                    int has_bound, double bound, uint64_t seed, uint32_t level, uint64_t node,
                    size_t* n_probes) {
  if (!ctx || !n_probes) return DSMC_E_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  if (n == 0) return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "pair weight source has n == 0");
  if (resampler != DSMC_MH_LAZY && resampler != DSMC_REJECTION_LAZY)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "lazy probing: mh-lazy or rejection-lazy");
  if (resampler == DSMC_REJECTION_LAZY && (!has_bound || !std::isfinite(bound)))
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT,
                   "rejection resampling requires a finite log_upper_bound");
  if (n > 0xffffffffu || n_out > 0x7fffffffu)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "lazy probing: sizes exceed 32-bit indices");
  LazyState& L = lazy_state(ctx);
  L = LazyState();
  L.resampler = resampler;
  L.n = n;
  L.n_out = n_out;
  L.mh_steps = mh_steps;
  L.bound = bound;
  L.seed = seed;
  L.level = level;
  L.node = node;
  Arena& A = ctx->arena;
  void* p;
  const size_t m = std::max<size_t>(n_out, 1);
  CU(A.get("LZCI", m * 4, &p));
  L.ci = (uint32_t*)p;
  CU(A.get("LZCJ", m * 4, &p));
  L.cj = (uint32_t*)p;
  CU(A.get("LZCV", m * 8, &p));
  L.cv = (double*)p;
  CU(A.get("LZPOS", m * 4, &p));
  L.pos = (int*)p;
  CU(A.get("LZDONE", m, &p));
  L.done = (uint8_t*)p;
  CU(A.get("LZPI", 2 * m * 4, &p));
  L.pi = (uint32_t*)p;
  CU(A.get("LZPJ", 2 * m * 4, &p));
  L.pj = (uint32_t*)p;
  CU(A.get("LZVAL", 2 * m * 8, &p));
  L.val = (double*)p;
  CU(A.get("LZMISC", 64, &p));
  L.count = (unsigned int*)p;
  L.err = (ErrFlag*)((char*)p + 16);
  CU(cudaMemsetAsync(p, 0, 64, ctx->stream));
  lazy_init_kernel<<<(unsigned)((m + 255) / 256), 256, 0, ctx->stream>>>((int)n, (int)n_out,
                                                                        L.ci, L.cj, L.done);
  LAUNCHED(ctx);
  if (n_out == 0 || (resampler == DSMC_MH_LAZY && mh_steps == 0)) {
    L.n_probes = 0;  // identity coupling, no evaluations at all
    *n_probes = 0;
    return DSMC_OK;
  }
  int rc = lazy_launch(ctx, L);
  if (rc) return rc;
  *n_probes = L.n_probes;
  return DSMC_OK;
}

int dsmc_lazy_probes(dsmc_ctx* ctx, uint32_t* i, uint32_t* j) {
  if (!ctx) return DSMC_E_INVALID_ARGUMENT;
  LazyState& L = lazy_state(ctx);
  if (L.resampler < 0) return set_err(ctx, DSMC_E_LOGIC, "no lazy sampling in progress");
  if (L.n_probes && (!i || !j)) return DSMC_E_INVALID_ARGUMENT;
  std::memcpy(i, L.hi.data(), L.n_probes * 4);
  std::memcpy(j, L.hj.data(), L.n_probes * 4);
  return DSMC_OK;
}

int dsmc_lazy_answer(dsmc_ctx* ctx, const double* values, size_t* n_probes) {
  if (!ctx || !n_probes) return DSMC_E_INVALID_ARGUMENT;
  LazyState& L = lazy_state(ctx);
  if (L.resampler < 0) return set_err(ctx, DSMC_E_LOGIC, "no lazy sampling in progress");
  if (L.n_probes == 0) {
    *n_probes = 0;
    return DSMC_OK;
  }
  if (!values) return DSMC_E_INVALID_ARGUMENT;
  CU(cudaMemcpyAsync(L.val, values, L.n_probes * 8, cudaMemcpyHostToDevice, ctx->stream));
  L.evals += L.n_probes;
  int rc = lazy_launch(ctx, L);
  if (rc) return rc;
  *n_probes = L.n_probes;
  return DSMC_OK;
}

int dsmc_lazy_finish(dsmc_ctx* ctx, uint32_t* left, uint32_t* right, uint64_t* weight_evals) {
  if (!ctx) return DSMC_E_INVALID_ARGUMENT;
  LazyState& L = lazy_state(ctx);
  if (L.resampler < 0) return set_err(ctx, DSMC_E_LOGIC, "no lazy sampling in progress");
  if (L.n_probes)
    return set_err(ctx, DSMC_E_LOGIC, "lazy sampling has unanswered probes");
  if (L.n_out && (!left || !right)) return DSMC_E_INVALID_ARGUMENT;
  auto s = ctx->stream;
  if (L.n_out) {
    CU(cudaMemcpyAsync(left, L.ci, L.n_out * 4, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(right, L.cj, L.n_out * 4, cudaMemcpyDeviceToHost, s));
  }
  CU(cudaStreamSynchronize(s));
  if (weight_evals) *weight_evals = L.evals;
  L.resampler = -1;
  return DSMC_OK;
}

}  // extern "C"

// Host orchestration + C ABI of the B200 dSMC engine (include/dsmc_b200.h).
//
// One run = prep (per-time constants) -> leaves -> ceil(log2 K) combine
// levels (all combines of a level in one launch per kernel; chunked only to
// bound workspace) -> top-down ancestor composition -> fused gather +
// moments. Every kernel goes on the context's stream; the host synchronises
// once at the end to read the device error record (no per-level sync).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "ffbs.cuh"
#include "kalman_scan.cuh"
#include "pair_tc.cuh"
#include "wide.cuh"
#include "pair_tc2.cuh"
#include "small32.cuh"
#include "dsmc_b200.h"

using namespace dsmc_dev;

namespace {

struct Arena {
  std::map<std::string, std::pair<void*, size_t>> bufs;
  uint64_t epoch = 0;  // bumped whenever a buffer moves (invalidates graphs)
  cudaError_t get(const char* name, size_t bytes, void** out) {
    auto& e = bufs[name];
    if (e.second < bytes) {
      ++epoch;
      if (e.first) cudaFree(e.first);
      e.first = nullptr;
      e.second = 0;
      cudaError_t rc = cudaMalloc(&e.first, std::max<size_t>(bytes, 256));
      if (rc != cudaSuccess) return rc;
      e.second = std::max<size_t>(bytes, 256);
    }
    *out = e.first;
    return cudaSuccess;
  }
  void release() {
    for (auto& kv : bufs)
      if (kv.second.first) cudaFree(kv.second.first);
    bufs.clear();
  }
};

struct Status {
  int code = DSMC_OK;
  std::string msg;
};

}  // namespace

struct dsmc_model_handle {
  uint64_t id = 0;  // unique per upload (graph cache key)
  int B = 1;
  dsmc_model_desc desc{};
  int K = 0, d = 1, dy = 1;
  int t_lo = 0, t_hi = 0;  // prepared times (a window upload: [t0, t0 + len + 1))
  bool wide = false;       // LGSSM on the wide-state FP32 path (d > 4, wide.cuh)
  WideBufs wb{};           // its per-time constants (device, owned)
  DevModel* models_dev = nullptr;  // [B]
  TimeConst* tc = nullptr;         // [B][K]
  int* bounded = nullptr;          // [B]
  std::vector<void*> owned;
  cudaStream_t stream = nullptr;  // owned memory is stream-ordered
  // deferred upload (dsmc_smooth with pinned host arrays): the per-time
  // arrays are copied in time chunks on the copy stream, each chunk's prep +
  // leaves starting as soon as it lands (run_tree); until then tc is unset
  bool defer = false;
  bool prep_pending = false;
  struct Deferred {
    void* dst;
    const void* src;
    size_t bytes_per_t;
  };
  std::vector<Deferred> deferred;
};

struct dsmc_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  uint64_t launches = 0;
  Arena arena;
  cudaEvent_t ev[4] = {};
  double timings[3] = {0, 0, 0};
  // per-launch events around the pair / sample kernels of the last timed run
  std::vector<cudaEvent_t> kev;
  int kev_used = 0;
  bool time_kernels = false;
  // FP32 pass 1: the CUDA-core kernel c32_pair (default, faster today) or
  // the tcgen05 kernel c32_pair_tc (DSMC_PAIR_KERNEL=tc)
  bool pair_tc = false;
  // the streaming tcgen05 pass 1 c32_pair_tc2 with its column prologue
  // (DSMC_PAIR_KERNEL=tc2; pair_tc2.cuh)
  bool pair_tc2 = false;
  int num_sms = 148;
  int smem_optin = 227 * 1024;  // max dynamic shared memory per CTA (opt-in)
  int smem_sm = 228 * 1024;     // shared memory per SM
  cudaStream_t copy_stream = nullptr;  // device->host copies overlapping the gather
  static constexpr int kGatherChunks = 8;
  cudaEvent_t gather_ev[kGatherChunks] = {};
  // last resident run
  int last_K = 0, last_d = 0, last_B = 0;  // shape of the last resident run
  size_t mean_cap = 0, cov_cap = 0;         // allocated doubles of d_mean / d_cov
  ErrFlag* last_err = nullptr;              // device error record of the last
  int last_err_K = 0;                       // resident / window run (unchecked)
  double* d_mean = nullptr;
  double* d_cov = nullptr;
  double last_lnc = NAN;
  int last_has_lnc = 0;
  uint64_t last_evals = 0;
  int last_levels = 0;
  int last_biased = 0;
  double* h_lnc = nullptr;  // pinned scratch
  void* window = nullptr;   // WindowState of the last run (time-sharded API)
  // CUDA graph of the last resident run (dsmc_smooth_resident): the whole
  // leaves -> levels -> composition sequence replayed with one launch; only
  // the seed (a kernel-node argument) changes between replays
  struct GraphCache {
    uint64_t handle = 0, epoch = 0;
    size_t N = 0, mh = 0;
    int rs = -1, prec = -1, seen = 0;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraphNode_t seed_node = nullptr;
    cudaKernelNodeParams seed_params{};
    uint64_t* seed_dst = nullptr;
    ErrFlag* err = nullptr;
    uint64_t launches = 0;
    int kev_used = 0, levels = 0;
    void reset() {
      if (exec) cudaGraphExecDestroy(exec);
      if (graph) cudaGraphDestroy(graph);
      *this = GraphCache();
    }
  } gc;
};

static std::atomic<uint64_t> g_handle_ids{0};  // handles from several host threads

namespace {

int set_err(dsmc_ctx* ctx, int code, std::string msg) {
  if (ctx) ctx->err = std::move(msg);
  return code;
}
#define CU(call)                                                          \
  do {                                                                    \
    cudaError_t _e = (call);                                              \
    if (_e != cudaSuccess)                                                \
      return set_err(ctx, DSMC_E_CUDA, std::string("CUDA: ") +            \
                                           cudaGetErrorString(_e) + " at " \
                                           #call);                        \
  } while (0)
#define LAUNCHED(ctx) (++(ctx)->launches)

// Timing events: recorded as EXTERNAL event nodes while the stream is being
// captured into a CUDA graph (plain graph event nodes cannot be timed).
cudaError_t rec_event(cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &st);
  return st == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal)
                                             : cudaEventRecord(e, s);
}

int validate_desc(dsmc_ctx* ctx, const dsmc_model_desc* m) {
  if (!m) return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "model descriptor is null");
  if (m->horizon < 0)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "model: horizon must be >= 0");
  if (m->kind == DSMC_MODEL_SV) {
    if (m->state_dim != 1)
      return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "sv: state_dim must be 1");
    if (!(m->sv_sigma2 > 0.0) || !(std::fabs(m->sv_phi) < 1.0))
      return set_err(ctx, DSMC_E_INVALID_ARGUMENT,
                     "sv descriptor: need s2 > 0 and |phi| < 1");
    if (!m->y) return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "sv: y is null");
    for (int t = 0; t <= m->horizon; ++t)
      if (!(m->y[t] != 0.0) || !std::isfinite(m->y[t]))
        return set_err(ctx, DSMC_E_INVALID_ARGUMENT,
                       "sv descriptor: observations must be finite and nonzero");
    return DSMC_OK;
  }
  if (m->kind == DSMC_MODEL_COX) {  // make_cox_model (models.cpp:113-125)
    if (m->state_dim != 1) return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "cox: state_dim must be 1");
    if (!(m->par[2] > 0.0))
      return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "make_cox_model: sigma2 must be > 0");
    if (!(std::fabs(m->par[1] * m->par[3]) < 1.0))
      return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "make_cox_model: need |rho * lambda| < 1");
    if (!m->y) return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "make_cox_model: observations are empty");
    for (int t = 0; t <= m->horizon; ++t) {
      const double y = m->y[t];
      if (!std::isfinite(y)) return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "make_cox_model: observations must be finite");
      if (y < 0.0 || std::floor(y) != y)
        return set_err(ctx, DSMC_E_INVALID_ARGUMENT,
                       "make_cox_model: counts must be nonnegative integers");
    }
    return DSMC_OK;
  }
  if (m->kind == DSMC_MODEL_CRW) {  // make_constrained_rw (models.cpp:265-268)
    if (m->state_dim != 1) return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "crw: state_dim must be 1");
    if (!(m->par[0] > 0.0))
      return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "make_constrained_rw: sigma must be > 0");
    return DSMC_OK;
  }
  if (m->kind == DSMC_MODEL_THETA) {  // make_theta_logistic (models.cpp:410-425)
    if (m->state_dim != 1) return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "theta: state_dim must be 1");
    if (!(m->par[3] > 0.0) || !(m->par[4] > 0.0))
      return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "make_theta_logistic: q2 and r2 must be > 0");
    if (!m->y || !m->prop_mean || !m->prop_cov)
      return set_err(ctx, DSMC_E_INVALID_ARGUMENT,
                     "make_theta_logistic: need one proposal marginal per observation");
    for (int t = 0; t <= m->horizon; ++t) {
      if (!std::isfinite(m->y[t]))
        return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "make_theta_logistic: observations must be finite");
      if (!(m->prop_cov[t] > 0.0) || !std::isfinite(m->prop_mean[t]))
        return set_err(ctx, DSMC_E_INVALID_ARGUMENT,
                       "make_theta_logistic: proposal marginals must have positive variance");
    }
    return DSMC_OK;
  }
  if (m->kind != DSMC_MODEL_LGSSM)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "unknown model kind");
  if (m->state_dim < 1 || m->state_dim > 32 || m->obs_dim < 1 || m->obs_dim > 32)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "lgssm descriptor: dims must be 1..32");
  if (m->state_dim <= 4 && m->obs_dim > 4)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT,
                   "lgssm descriptor: obs_dim > 4 needs the wide path (state_dim > 4)");
  if (!m->m0 || !m->P0 || !m->prop_mean || !m->prop_cov || !m->H || !m->R ||
      !m->y || (m->horizon >= 1 && (!m->F || !m->b || !m->Q)))
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT,
                   "model: proposal, initial, transition and observation arrays "
                   "are required");
  return DSMC_OK;
}

void free_handle(dsmc_model_handle* h) {
  if (!h) return;
  for (void* p : h->owned) cudaFreeAsync(p, h->stream);
  delete h;
}

// per_t > 0: a per-time array of n = K * per_t elements (deferrable)
template <class T>
int upload(dsmc_ctx* ctx, dsmc_model_handle* h, const T* src, size_t n,
           const T** dst, size_t per_t = 0) {
  if (!src || n == 0) {
    *dst = nullptr;
    return DSMC_OK;
  }
  void* p = nullptr;
  CU(cudaMallocAsync(&p, n * sizeof(T), ctx->stream));
  h->owned.push_back(p);
  if (h->defer && per_t > 0)
    h->deferred.push_back({p, src, per_t * sizeof(T)});
  else
    CU(cudaMemcpyAsync(p, src, n * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
  *dst = static_cast<const T*>(p);
  return DSMC_OK;
}

// ------------------------------------------------ wide-state prior prep
// Host FP64 helpers for the wide path's prior constants (one P0 factor); the
// per-time constants are computed on the device (wide.cuh prepw_kernel).
namespace widep {
bool chol(const double* A, int n, double* L) {
  for (int i = 0; i < n * n; ++i) L[i] = 0.0;
  for (int j = 0; j < n; ++j) {
    double s = A[j * n + j];
    for (int k = 0; k < j; ++k) s -= L[j * n + k] * L[j * n + k];
    if (!(s > 0.0)) return false;
    L[j * n + j] = std::sqrt(s);
    for (int i = j + 1; i < n; ++i) {
      double v = A[i * n + j];
      for (int k = 0; k < j; ++k) v -= L[i * n + k] * L[j * n + k];
      L[i * n + j] = v / L[j * n + j];
    }
  }
  return true;
}
void tri_inv(const double* L, int n, double* W) {  // W = L^-1 (lower)
  for (int i = 0; i < n * n; ++i) W[i] = 0.0;
  for (int i = 0; i < n; ++i) {
    W[i * n + i] = 1.0 / L[i * n + i];
    for (int j = 0; j < i; ++j) {
      double s = 0.0;
      for (int k = j; k < i; ++k) s += L[i * n + k] * W[k * n + j];
      W[i * n + j] = -s / L[i * n + i];
    }
  }
}
double logdet(const double* L, int n) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += 2.0 * std::log(L[i * n + i]);
  return s;
}
}  // namespace widep

// Dynamic shared memory of samplew_kernel: row CDF (double) + row totals,
// then per slot a 16-byte record and a sort index, and the sub-block counts.
size_t samplew_smem(int N, int slots) {
  const size_t head = (sizeof(double) * (((size_t)N + 1) & ~(size_t)1) + sizeof(float) * (size_t)N +
                       15) & ~(size_t)15;
  return head + (size_t)slots * (16 + 4) + sizeof(int) * (size_t)((N + kSub - 1) / kSub);
}

template <int D>
void launch_lazy32(dim3 grid, cudaStream_t s, const Bufs& b, const LevelArgs& la, int mh,
                   size_t steps) {
  if (mh) lazy32_kernel<D, true><<<grid, 128, 0, s>>>(b, la, steps);
  else lazy32_kernel<D, false><<<grid, 128, 0, s>>>(b, la, steps);
}

// floats per combine of the wide AUX (wide.cuh auxw): Y, U, A, B and the
// column tiles of the pipelined pass 1 (64 columns x K = 3 D + 8 per tile)
size_t wide_aux_floats(int N, int D) {
  return auxw_yt_off(N, D) + (size_t)((N + kSub - 1) / kSub) * kSub * (3 * D + 8);
}

int wide_dp(int d) { return d <= 8 ? 8 : d <= 16 ? 16 : 32; }
bool getenv_flag(const char* name) {  // A/B switches for tests and tools
  const char* f = getenv(name);
  return f && f[0] == '1';
}
bool force_wide() { return getenv_flag("DSMC_FORCE_WIDE"); }

// Per-time array restricted to times [lo, hi) (time-sharded windows): only
// those rows are uploaded, and the device pointer is offset so kernels keep
// indexing by GLOBAL time (rows outside the range are never read).
template <class T>
int upload_rows(dsmc_ctx* ctx, dsmc_model_handle* h, const T* src, size_t per_t, int lo, int hi,
                const T** dst) {
  if (!src || per_t == 0) {
    *dst = nullptr;
    return DSMC_OK;
  }
  void* p = nullptr;
  const size_t n = (size_t)(hi - lo) * per_t;
  CU(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), ctx->stream));
  h->owned.push_back(p);
  CU(cudaMemcpyAsync(p, src + (size_t)lo * per_t, n * sizeof(T), cudaMemcpyHostToDevice,
                     ctx->stream));
  *dst = static_cast<const T*>(p) - (ptrdiff_t)((size_t)lo * per_t);
  return DSMC_OK;
}

// Upload B descriptors (same K, d) and run the prep kernel. [w_lo, w_hi):
// the times whose per-time constants are needed (default all); a window
// handle uploads model rows [w_lo - 1, w_hi) and prepares only [w_lo, w_hi).
int make_handle(dsmc_ctx* ctx, const dsmc_model_desc* descs, int B,
                dsmc_model_handle** out, bool defer = false, int w_lo = 0, int w_hi = -1) {
  for (int c = 0; c < B; ++c) {
    int rc = validate_desc(ctx, &descs[c]);
    if (rc) return rc;
    if (descs[c].horizon != descs[0].horizon || descs[c].state_dim != descs[0].state_dim ||
        descs[c].kind != descs[0].kind)
      return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "chains must share kind, horizon and dims");
  }
  std::unique_ptr<dsmc_model_handle, void (*)(dsmc_model_handle*)> h(new dsmc_model_handle(),
                                                                      free_handle);
  h->id = ++g_handle_ids;
  h->B = B;
  h->stream = ctx->stream;
  h->defer = defer && B == 1;
  h->desc = descs[0];
  const int K = descs[0].horizon + 1, d = descs[0].state_dim, dy = descs[0].obs_dim;
  h->K = K;
  h->d = d;
  h->dy = dy;
  if (w_hi < 0) w_hi = K;
  const bool window = w_lo > 0 || w_hi < K;
  if (window && (B != 1 || w_lo < 0 || w_hi > K || w_lo >= w_hi))
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "window upload: need one model and 0 <= t0 < t1 <= K");
  const int rlo = std::max(0, w_lo - 1), rhi = w_hi;  // model rows: the window + its left cut
  h->t_lo = w_lo;
  h->t_hi = w_hi;
  if (window) h->defer = false;
  // per-time array: the window's rows (offset pointer) or the whole horizon
  auto per_time = [&](const auto* src, size_t per_t, auto** dst) -> int {
    if (window) return upload_rows(ctx, h.get(), src, per_t, rlo, rhi, dst);
    return upload(ctx, h.get(), src, src ? (size_t)K * per_t : 0, dst, per_t);
  };
  auto per_time_strided = [&](const double* src, int64_t stride, size_t per, const double** dst) -> int {
    if (!stride) return upload(ctx, h.get(), src, per, dst);  // one matrix for every time
    return per_time(src, (size_t)stride, dst);
  };
  const bool wide = descs[0].kind == DSMC_MODEL_LGSSM && (d > 4 || force_wide());
  std::vector<DevModel> dm(B);
  for (int c = 0; c < B; ++c) {
    const dsmc_model_desc& m = descs[c];
    DevModel& M = dm[c];
    M.kind = m.kind;
    M.d = d;
    M.dy = m.kind == DSMC_MODEL_SV ? 1 : dy;
    M.T = m.horizon;
    M.K = K;
    M.sv_mu = m.sv_mu;
    M.sv_phi = m.sv_phi;
    M.sv_s2 = m.sv_sigma2;
    M.F_s = m.F_stride;
    M.b_s = m.b_stride;
    M.Q_s = m.Q_stride;
    M.H_s = m.H_stride;
    M.R_s = m.R_stride;
    int rc = 0;
    const size_t nT = (size_t)K;
    for (int q = 0; q < 8; ++q) M.mp[q] = 0.0;
    M.lgam = nullptr;
    if (m.kind == DSMC_MODEL_COX || m.kind == DSMC_MODEL_CRW) {
      M.has_obs = nullptr;
      M.prop_mean = M.prop_cov = M.F = M.b = M.Q = M.H = M.R = M.m0 = M.P0 = nullptr;
      M.y = nullptr;
      if (m.kind == DSMC_MODEL_COX) {  // models.cpp:127-135 (same expressions)
        const double mu = m.par[0], rho = m.par[1], s2 = m.par[2], lam = m.par[3];
        const double slope = rho * lam, icept = mu * (1.0 - rho);
        const double stat_mean = icept / (1.0 - slope);
        const double stat_var = s2 / (1.0 - slope * slope);
        const double mp[8] = {slope, icept, stat_mean, stat_var,
                              -0.5 * (kLog2Pi + std::log(s2)), s2, std::sqrt(stat_var), 0.0};
        for (int q = 0; q < 8; ++q) M.mp[q] = mp[q];
        std::vector<double> lg(nT);
        for (size_t t = 0; t < nT; ++t) lg[t] = std::lgamma(m.y[t] + 1.0);
        rc |= per_time(m.y, 1, &M.y);
        rc |= per_time(lg.data(), 1, &M.lgam);
        CU(cudaStreamSynchronize(ctx->stream));  // lg is a local host buffer
      } else {  // models.cpp:269-270
        const double sigma = m.par[0], var = sigma * sigma;
        M.mp[0] = var;
        M.mp[1] = -0.5 * (kLog2Pi + std::log(var));
        M.mp[2] = sigma;
      }
    } else if (m.kind == DSMC_MODEL_THETA) {  // models.cpp:427-431
      M.has_obs = nullptr;
      M.F = M.b = M.Q = M.H = M.R = M.m0 = M.P0 = nullptr;
      const double mp[8] = {m.par[0], m.par[1], m.par[2], m.par[3], m.par[4],
                            -0.5 * (kLog2Pi + std::log(m.par[3])),
                            -0.5 * (kLog2Pi + std::log(m.par[4])), 0.0};
      for (int q = 0; q < 8; ++q) M.mp[q] = mp[q];
      rc |= per_time(m.y, 1, &M.y);
      rc |= per_time(m.prop_mean, 1, &M.prop_mean);
      rc |= per_time(m.prop_cov, 1, &M.prop_cov);
    } else if (m.kind == DSMC_MODEL_SV) {
      rc |= per_time(m.y, 1, &M.y);
      M.has_obs = nullptr;
      M.prop_mean = M.prop_cov = M.F = M.b = M.Q = M.H = M.R = M.m0 = M.P0 = nullptr;
    } else {
      rc |= per_time(m.y, (size_t)dy, &M.y);
      rc |= per_time(m.has_obs, 1, &M.has_obs);
      rc |= per_time(m.prop_mean, (size_t)d, &M.prop_mean);
      rc |= per_time(m.prop_cov, (size_t)d * d, &M.prop_cov);
      rc |= upload(ctx, h.get(), m.m0, (size_t)d, &M.m0);
      rc |= upload(ctx, h.get(), m.P0, (size_t)d * d, &M.P0);
      rc |= per_time_strided(m.H, m.H_stride, (size_t)dy * d, &M.H);
      rc |= per_time_strided(m.R, m.R_stride, (size_t)dy * dy, &M.R);
      if (m.horizon >= 1) {
        rc |= per_time_strided(m.F, m.F_stride, (size_t)d * d, &M.F);
        rc |= per_time_strided(m.b, m.b_stride, (size_t)d, &M.b);
        rc |= per_time_strided(m.Q, m.Q_stride, (size_t)d * d, &M.Q);
      } else {
        M.F = M.b = M.Q = nullptr;
      }
    }
    if (rc) return DSMC_E_CUDA;
  }
  void* p;
  // wide-state LGSSM (d > 4, or forced for testing): device-prepared constants
  if (wide) {
    if (B != 1 || window)
      return set_err(ctx, DSMC_E_INVALID_ARGUMENT,
                     "state_dim > 4: one unconditional model on the whole horizon");
    const int DP = wide_dp(d), DYP = (dy + 3) & ~3;
    const dsmc_model_desc& md = descs[0];
    WideBufs& wb = h->wb;
    wb.d = d;
    wb.dy = dy;
    wb.DP = DP;
    wb.DYP = DYP;
    {  // prior constants on the host (one matrix)
      std::vector<double> Lp((size_t)d * d), Wp((size_t)d * d);
      if (!widep::chol(md.P0, d, Lp.data()))
        return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "lgssm: P0 is not positive definite");
      widep::tri_inv(Lp.data(), d, Wp.data());
      std::vector<float> WP0((size_t)DP * DP, 0.f), dm0(DP, 0.f);
      for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) WP0[i * DP + j] = (float)Wp[i * d + j];
      for (int i = 0; i < d; ++i) dm0[i] = (float)(md.m0[i] - md.prop_mean[i]);
      wb.p0norm = -0.5 * (d * kLog2Pi + widep::logdet(Lp.data(), d));
      float* q;
      CU(cudaMallocAsync((void**)&q, sizeof(float) * ((size_t)DP * DP + DP), ctx->stream));
      h->owned.push_back(q);
      CU(cudaMemcpyAsync(q, WP0.data(), sizeof(float) * DP * DP, cudaMemcpyHostToDevice, ctx->stream));
      CU(cudaMemcpyAsync(q + DP * DP, dm0.data(), sizeof(float) * DP, cudaMemcpyHostToDevice,
                         ctx->stream));
      CU(cudaStreamSynchronize(ctx->stream));  // WP0 / dm0 are local
      wb.WP0 = q;
      wb.dm0 = q + DP * DP;
    }
    // per-time constants on the device (prepw_kernel), zero-filled padding
    const size_t nL = (size_t)K * DP * DP, nG = (size_t)K * DYP * DP, ne = (size_t)K * DYP;
    const size_t nall = 3 * nL + nG + ne + (size_t)K + (size_t)K * DP;
    float* q;
    CU(cudaMallocAsync((void**)&q, sizeof(float) * nall + 16, ctx->stream));
    h->owned.push_back(q);
    CU(cudaMemsetAsync(q, 0, sizeof(float) * nall, ctx->stream));
    WidePrep o;
    o.L = q;
    o.W = q + nL;
    o.M = q + 2 * nL;
    o.G = q + 3 * nL;
    o.e = o.G + nG;
    o.c = o.e + ne;
    o.v = o.c + K;
    int* errd = reinterpret_cast<int*>(o.v + (size_t)K * DP);  // 16 spare bytes
    CU(cudaMemsetAsync(errd, 0x7f, 3 * sizeof(int), ctx->stream));
    o.err = errd;
    o.d = d;
    o.dy = dy;
    o.DP = DP;
    o.DYP = DYP;
    o.K = K;
    prepw_kernel<<<K, 32, 3 * 32 * kPS * sizeof(double), ctx->stream>>>(dm[0], o);
    LAUNCHED(ctx);
    int errs[3];
    CU(cudaMemcpyAsync(errs, errd, sizeof(errs), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    static const char* what[3] = {"proposal covariance", "R", "Q"};
    for (int q2 = 0; q2 < 3; ++q2)
      if (errs[q2] < K)
        return set_err(ctx, DSMC_E_INVALID_ARGUMENT,
                       std::string("lgssm: ") + what[q2] + " at time " + std::to_string(errs[q2]) +
                           " is not positive definite");
    wb.L = o.L;
    wb.W = o.W;
    wb.M = o.M;
    wb.G = o.G;
    wb.e = o.e;
    wb.c = o.c;
    wb.v = o.v;
    wb.m = dm[0].prop_mean;  // the uploaded FP64 proposal means
    h->wide = true;
    h->defer = false;
  }
  CU(cudaMallocAsync(&p, sizeof(DevModel) * B, ctx->stream));
  h->owned.push_back(p);
  h->models_dev = static_cast<DevModel*>(p);
  CU(cudaMemcpyAsync(p, dm.data(), sizeof(DevModel) * B, cudaMemcpyHostToDevice, ctx->stream));
  // per-time constants: the prepared range only (offset pointer, global index)
  CU(cudaMallocAsync(&p, sizeof(TimeConst) * B * (size_t)(w_hi - w_lo), ctx->stream));
  h->owned.push_back(p);
  h->tc = static_cast<TimeConst*>(p) - w_lo;
  CU(cudaMallocAsync(&p, sizeof(int) * B, ctx->stream));
  h->owned.push_back(p);
  h->bounded = static_cast<int*>(p);
  std::vector<int> ones(B, 3);
  CU(cudaMemcpyAsync(p, ones.data(), sizeof(int) * B, cudaMemcpyHostToDevice, ctx->stream));
  if (h->deferred.empty() && (d > 4 || wide)) {
    h->defer = false;  // the TimeConst per-time constants exist for d <= 4 only (not wide)
  } else if (h->deferred.empty()) {
    h->defer = false;
    prep_kernel<<<dim3((w_hi - w_lo + 127) / 128, B), 128, 0, ctx->stream>>>(
        h->models_dev, h->tc, K, h->bounded, w_lo, w_hi);
    LAUNCHED(ctx);
  } else {
    h->prep_pending = true;  // run_tree copies, preps and draws leaves chunk by chunk
  }
  CU(cudaGetLastError());
  *out = h.release();
  return DSMC_OK;
}


// --------------------------------------------------------------- the run
struct RunOpts {
  int precision = DSMC_FP32;
  int resampler = DSMC_MULTINOMIAL;
  size_t mh_steps = 16;
  size_t N = 0;
  int conditional = 0;
  uint32_t sweep = 0;
  const double* inj_x = nullptr;   // host
  const double* inj_lw = nullptr;  // host
  const double* star = nullptr;    // device [B][K][d] (conditional)
  const uint64_t* seeds = nullptr; // device [B]
  // outputs (device pointers, optional)
  double* paths = nullptr;
  double* mean = nullptr;
  double* cov = nullptr;
  double* star_out = nullptr;   // device [B][K][d]
  uint8_t* changed = nullptr;   // device [B][K]
  // optional host destinations of mean / cov (B = 1, FP32): the final gather
  // then runs in time chunks and each chunk's moments are copied back on
  // the copy stream while the next chunk is gathered
  double* host_mean = nullptr;
  double* host_cov = nullptr;
  bool timing = false;
  // time-sharded windows (FP32): leaves [t0, t0 + len) of the model, global
  // stream keys; composition optional, from a given root map
  int t0 = 0;
  int len = -1;
  bool compose = true;
  const uint32_t* root_map = nullptr;  // device [B][N]
  // block injection (dsmc_resample_blocks): the injected log weights are
  // already normalised block weights with the given uniform flags and maxima
  // (no leaf normalisation), and the combines use this stream key
  const uint8_t* inj_uni = nullptr;    // host [K]
  const double* inj_lwmax = nullptr;   // host [K]
  int key_level = -1;                  // -1: the tree level
  long long key_node = 0;
  int n_out = -1;                      // slots per combine (-1: N, or N - 1 conditional)
};

struct RunResult {
  int levels = 0;
  // device pointers valid until the next run on the context
  uint32_t* PL = nullptr;
  uint32_t* PR = nullptr;
  double* LMW = nullptr;
  double* root_lnc = nullptr;  // [B] (strided by cap)
  size_t lnc_stride = 0;
  unsigned long long* evals = nullptr;
  ErrFlag* err = nullptr;
  double* LNC = nullptr;
  double* X64 = nullptr;
  double* LW64 = nullptr;
};

template <int MC, int D>
int launch_c64(dsmc_ctx* ctx, const Bufs& b, const LevelArgs& la, int nk,
               int systematic) {
  const size_t lim = (size_t)ctx->smem_optin - 1024;
  const size_t sm = cols64_bytes(b.N, D, false);
  const size_t rows = sizeof(double) * kC64Rows * (D + 1);  // pass 1's row means + weights
  if (sm + rows > lim || sm + c64s_extra(b.N, false) > lim)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT,
                   "FP64 parity combine: N * (d + 2) doubles exceed the shared-memory "
                   "column stage (N <= " +
                       std::to_string((ctx->smem_optin - 1024) / (8 * (D + 2)) / 72 * 64) +
                       " at this d); use the FP32 path or a lazy resampler");
  // pass 1 screens each row's max in FP32 when the screen copies fit too
  // (DSMC_C64_SCREEN=0 forces the full FP64 max scan)
  const bool screen_env =
      !(getenv("DSMC_C64_SCREEN") && atoi(getenv("DSMC_C64_SCREEN")) == 0);
  const size_t smf = cols64_bytes(b.N, D, true);
  const int fast = screen_env && smf + rows <= lim;
  c64_rows<MC, D><<<dim3((b.N + kC64Rows - 1) / kC64Rows, nk, b.B), kC64Threads,
                    (fast ? smf : sm) + rows, ctx->stream>>>(b, la, fast);
  LAUNCHED(ctx);
  c64_cdf<<<(nk * b.B + 7) / 8, 256, 0, ctx->stream>>>(b, la, nk);
  LAUNCHED(ctx);
  // the sampler sorts its slots by sub-block when the records fit
  const int sorted = sm + c64s_extra(b.N, true) <= lim;
  c64_sample<MC, D><<<dim3(nk, 1, b.B), 256, sm + c64s_extra(b.N, sorted), ctx->stream>>>(
      b, la, systematic, sorted);
  LAUNCHED(ctx);
  return DSMC_OK;
}

// Launch with programmatic stream serialization: the kernel (which starts
// with griddepcontrol.wait) is set up while its predecessor drains, hiding
// the launch gap between the many short kernels of the upper levels.
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

template <int D>
int launch_c32(dsmc_ctx* ctx, const Bufs& b, LevelArgs la, int nk, int systematic) {
  // Pass 1: 256-row tiles; when the level has few combines, the sub-blocks of
  // a tile are split over several CTAs so the grid still gives >= 4 waves of
  // the 2 resident CTAs per SM.
  const int target = 148 * 4 * 4;
  const int N = b.N;
  const int nrt = (N + kRowsCTA - 1) / kRowsCTA, nsubb = (N + kSub - 1) / kSub;
  int ncs = 1;
  while (ncs * 2 <= std::max(1, nsubb / kPairWarps) && (long)nk * b.B * nrt * ncs < target) ncs *= 2;
  // Pass-2: split a combine's slots over several CTAs when combines are few.
  int sb = 1;
  const int target2 = 148 * 2;
  if ((long)nk * b.B < target2)
    sb = std::max(1, std::min((la.n_out + 63) / 64, (int)((target2 + nk * b.B - 1) / (nk * b.B))));
  // the sampler stages <= 1024 slots per CTA in shared memory
  sb = std::max(sb, (la.n_out + 1023) / 1024);
  la.slots_per_cta = (la.n_out + sb - 1) / sb;
  const size_t NP = (N + 63) / 64 * 64;
  const size_t NPS = NP / 2 + NP / 64;  // column pairs, one skew pad per sub-block
  const size_t ns = la.slots_per_cta, nsub = (N + 63) / 64;
  const size_t ns2 = (ns + 1) & ~(size_t)1;
  const size_t sm2 = sizeof(double) * (N + 1) + NPS * (16 + 16 + 8) + sizeof(float) * N + 16 +
                     sizeof(double) * ns2 + 4 * ns2 + 8 * ns + 2 * ns2 + sizeof(int) * (32 + nsub);
  // the 64-register instantiation where 4 CTAs per SM fit (dynamic + 1 KB
  // static + 1 KB reserved per CTA)
  const bool sample4 = 4 * (sm2 + 2048) <= (size_t)ctx->smem_sm;
  if (N >= 65536)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT,
                   "FP32 dense combine: N must be < 65536 (use a lazy resampler)");
  // large N: the column pairs no longer fit next to the row CDF in shared
  // memory; the sampler then keeps only the CDF (12 N bytes) and reads the
  // pass-1 hand-off from L2 (samplew_kernel over Aux32)
  const size_t sm_big = samplew_smem(N, la.slots_per_cta);
  const bool big = sm2 > (size_t)ctx->smem_optin - 1024;
  if (big && sm_big > (size_t)ctx->smem_optin - 1024)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT,
                   "FP32 dense combine: N too large for the shared-memory row CDF (use a lazy "
                   "resampler)");
  const bool use_tc = ctx->pair_tc && D >= 2;
  la.aux_comb = ((size_t)10 * N + 3) & ~(size_t)3;
  {
    void* p;
    CU(ctx->arena.get("AUX32", la.aux_comb * sizeof(float) * (size_t)nk * b.B, &p));
    la.aux = (float*)p;
  }
  cudaEvent_t* ev = nullptr;
  if (ctx->time_kernels) {  // 3 events: pair start, pair end = sample start, sample end
    while ((int)ctx->kev.size() < ctx->kev_used + 3) {
      cudaEvent_t e;
      CU(cudaEventCreate(&e));
      ctx->kev.push_back(e);
    }
    ev = &ctx->kev[ctx->kev_used];
    ctx->kev_used += 3;
    CU(rec_event(ev[0], ctx->stream));
  }
  // small N: pass 1 and pass 2 fused in one CTA per combine (c32_small;
  // DSMC_SMALL=0 keeps the two-kernel path)
  const bool small_env = !(getenv("DSMC_SMALL") && atoi(getenv("DSMC_SMALL")) == 0);
  if (small_env && N <= kSmallN && !use_tc && !ctx->pair_tc2) {
    CU(launch_pdl(c32_small<D>, dim3(nk, 1, b.B), dim3(kSmallN), 0, ctx->stream, b, la,
                  systematic));
    LAUNCHED(ctx);
    if (ev) {
      CU(rec_event(ev[1], ctx->stream));
      CU(rec_event(ev[2], ctx->stream));
    }
    return DSMC_OK;
  }
  const int nrt_tc2 = (N + kTcRows - 1) / kTcRows;
  // (levels with fewer CTAs than two per SM stay on c32_pair; DSMC_TC2_MIN
  // overrides the threshold, e.g. 0 in tests)
  const long tc2_min = getenv("DSMC_TC2_MIN") ? atol(getenv("DSMC_TC2_MIN")) : 2 * 148;
  const bool use_tc2 = ctx->pair_tc2 && D >= 2 && b.B == 1 && (long)nk * nrt_tc2 >= tc2_min;
  if (use_tc2) {
    // streaming tensor-core pass 1: per sub-chunk of <= kTc2Sub combines the
    // prologue writes the column tiles (kept in L2), then one CTA per 128-row
    // tile consumes them
    using T = Tc2L<D>;
    const size_t cb = tc2_comb_bytes(nsubb, T::TILE);
    void* tp;
    CU(ctx->arena.get("TILE32", cb * (size_t)std::min(nk, kTc2Sub), &tp));
    for (int s0 = 0; s0 < nk; s0 += kTc2Sub) {
      const int m = std::min(kTc2Sub, nk - s0);
      LevelArgs l2 = la;
      l2.k0 = la.k0 + s0;
      l2.ws = la.ws + (size_t)s0 * la.ws_comb;
      l2.aux = la.aux + (size_t)s0 * la.aux_comb;
      c32_prol<D><<<dim3((nsubb * kSub + 127) / 128, m, 1), 128, 0, ctx->stream>>>(
          b, l2, static_cast<uint8_t*>(tp));
      LAUNCHED(ctx);
      c32_pair_tc2<D><<<dim3(nrt_tc2, m, 1), kTc2Threads, 0, ctx->stream>>>(
          b, l2, static_cast<const uint8_t*>(tp));
      if (s0 + kTc2Sub < nk) LAUNCHED(ctx);
    }
  } else if (use_tc) {
    // tensor-core pass 1: 128-row tiles, 4 CTAs per SM (128 TMEM columns each)
    const int nrt_tc = (N + kTcRows - 1) / kTcRows;
    int ncs_tc = 1;
    while (ncs_tc * 2 <= nsubb && (long)nk * b.B * nrt_tc * ncs_tc < target) ncs_tc *= 2;
    c32_pair_tc<D><<<dim3(nrt_tc * ncs_tc, nk, b.B), kTcThreads, 0, ctx->stream>>>(b, la);
  } else {
    CU(launch_pdl(c32_pair<D>, dim3(nrt * ncs, nk, b.B), dim3(32 * kPairWarps), 0, ctx->stream,
                  b, la));
  }
  LAUNCHED(ctx);
  if (ev) CU(rec_event(ev[1], ctx->stream));
  if (big)
    samplew_kernel<4, Aux32Recompute<D>><<<dim3(sb, nk, b.B), 256, sm_big, ctx->stream>>>(
        b, la, systematic);
  else if (sample4)
    CU(launch_pdl(c32_sample<D, 4>, dim3(sb, nk, b.B), dim3(256), sm2, ctx->stream, b, la,
                  systematic));
  else
    CU(launch_pdl(c32_sample<D, 3>, dim3(sb, nk, b.B), dim3(256), sm2, ctx->stream, b, la,
                  systematic));
  LAUNCHED(ctx);
  if (ev) CU(rec_event(ev[2], ctx->stream));
  return DSMC_OK;
}

// Wide-state combine chunk: prologue (whitened rows / columns into AUX),
// pass 1 (register-tiled cross term + sub-block log2-sums), sampler.
template <int D>
int launch_wide(dsmc_ctx* ctx, const Bufs& b, LevelArgs la, int nk, int systematic) {
  const int N = b.N;
  const int nrt = (N + kWRows - 1) / kWRows, nsub = (N + kSub - 1) / kSub;
  // pass-1 kernel: the pipelined tcgen05 kernel (default), the first
  // tcgen05 kernel (DSMC_WIDE_PAIR=tc1) or the register-tiled CUDA-core one
  // (DSMC_WIDE_PAIR=fma)
  static const int pair_kind = [] {
    const char* e = getenv("DSMC_WIDE_PAIR");
    return !e ? 2 : strcmp(e, "fma") == 0 ? 0 : strcmp(e, "tc1") == 0 ? 1 : 2;
  }();
  la.wide_tiles = pair_kind == 2;
  la.aux_comb = wide_aux_floats(N, D);
  {
    void* p;
    CU(ctx->arena.get("AUXW", la.aux_comb * sizeof(float) * (size_t)nk * b.B, &p));
    la.aux = (float*)p;
  }
  const int target = 148 * 4;
  int ncs = 1;
  while (ncs * 2 <= nsub && (long)nk * b.B * nrt * ncs < target) ncs *= 2;
  int sb = 1;
  if ((long)nk * b.B < 148 * 2)
    sb = std::max(1, std::min((la.n_out + 63) / 64, (int)((148 * 2 + nk * b.B - 1) / (nk * b.B))));
  sb = std::max(sb, (la.n_out + 1023) / 1024);  // <= 1024 slot records per CTA
  la.slots_per_cta = (la.n_out + sb - 1) / sb;
  const size_t sm1 = sizeof(float) * ((size_t)(kWRows + kSub) * WideK<D>::S + kWRows + kSub);
  const size_t sm2 = samplew_smem(N, la.slots_per_cta);
  if (sm2 > (size_t)ctx->smem_optin - 1024)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "wide combine: N too large for the sampler");
  cudaEvent_t* ev = nullptr;
  if (ctx->time_kernels) {  // pair = prologue + pass 1, sample = sampler
    while ((int)ctx->kev.size() < ctx->kev_used + 3) {
      cudaEvent_t e;
      CU(cudaEventCreate(&e));
      ctx->kev.push_back(e);
    }
    ev = &ctx->kev[ctx->kev_used];
    ctx->kev_used += 3;
    CU(rec_event(ev[0], ctx->stream));
  }
  prologw_kernel<D><<<dim3((N + 127) / 128, nk, b.B), 128, 0, ctx->stream>>>(b, la);
  LAUNCHED(ctx);
  if (pair_kind == 0)
    pairw_kernel<D><<<dim3(nrt * ncs, nk, b.B), 256, sm1, ctx->stream>>>(b, la);
  else if (pair_kind == 1)
    pairw_tc_kernel<D><<<dim3(nrt * ncs, nk, b.B), 128, WideTc<D>::SMEM, ctx->stream>>>(b, la);
  else
    pairw_tc2_kernel<D><<<dim3(nrt * ncs, nk, b.B), 256, WideTc2<D>::SMEM, ctx->stream>>>(b, la);
  LAUNCHED(ctx);
  if (ev) CU(rec_event(ev[1], ctx->stream));
  samplew_kernel<D><<<dim3(sb, nk, b.B), 256, sm2, ctx->stream>>>(b, la, systematic);
  LAUNCHED(ctx);
  if (ev) CU(rec_event(ev[2], ctx->stream));
  return DSMC_OK;
}

__global__ void tail_copy_kernel(Bufs b, int idx_prev, int idx_next,
                                 const uint32_t* fp, const uint32_t* lp,
                                 uint32_t* fn, uint32_t* ln,
                                 const double* blp, double* bln) {
  const int ch = blockIdx.y;
  const size_t src = ((size_t)ch * b.cap + idx_prev) * b.N;
  const size_t dst = ((size_t)ch * b.cap + idx_next) * b.N;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < b.N; q += gridDim.x * blockDim.x) {
    fn[dst + q] = fp[src + q];
    ln[dst + q] = lp[src + q];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0)
    bln[(size_t)ch * b.cap + idx_next] = blp[(size_t)ch * b.cap + idx_prev];
}

std::string err_message(const ErrFlag& e, int K) {
  char buf[512];
  const int c = e.cut, l = e.level;
  auto span = [&](int& a, int& bb) {
    const int s = 1 << (l - 1);
    const int k = (c / s - 1) / 2;
    a = 2 * k * s;
    bb = std::min((2 * k + 2) * s - 1, K - 1);
  };
  int a = 0, bb = 0;
  switch (e.reason) {
    case kReasonZeroTable:
      span(a, bb);
      snprintf(buf, sizeof buf,
               "combine at cut %d (times %d..%d): all pair weights are zero; the "
               "blocks share no support under the model", c, a, bb);
      break;
    case kReasonTrialCap:
      span(a, bb);
      snprintf(buf, sizeof buf,
               "combine at cut %d (times %d..%d): rejection resampling exceeded "
               "the trial cap; the bound is far too loose or the weights are "
               "degenerate", c, a, bb);
      break;
    case kReasonOverBound:
      snprintf(buf, sizeof buf, "pair weight exceeds its stated upper bound (cut %d)", c);
      break;
    case kReasonNoBound:
      snprintf(buf, sizeof buf, "rejection resampling requires a finite log_upper_bound");
      break;
    case kReasonNaN:
      snprintf(buf, sizeof buf, l == 0 ? "leaf %d: weight is NaN" : "NaN pair weight at cut %d", c);
      break;
    case kReasonRefPair:
      snprintf(buf, sizeof buf,
               "conditional_combine: the reference pair has zero stitch weight at cut %d", c);
      break;
    case kReasonLeafZero:
      snprintf(buf, sizeof buf, "leaf %d: every proposal draw has zero weight", c);
      break;
    case kReasonRefLeaf:
      snprintf(buf, sizeof buf,
               "conditional_leaf: the reference path has zero weight at time %d", c);
      break;
    default:
      snprintf(buf, sizeof buf, "device error at cut %d level %d", c, l);
  }
  return buf;
}

// Core: leaves + levels (+ composition/gather). B chains share K, N, d.
struct WindowState {
  bool valid = false;
  Bufs b{};
  int levels = 0, cur = 0;
  uint32_t* maps[4] = {};
  double* blnc[2] = {};
  int resampler = 0;
};
WindowState& window_state(dsmc_ctx* ctx);

// A deferred upload not consumed chunk by chunk: copy everything and prep.
static cudaError_t flush_deferred(dsmc_ctx* ctx, dsmc_model_handle* h) {
  if (!h->prep_pending) return cudaSuccess;
  const size_t K = (size_t)h->K;
  for (const auto& df : h->deferred) {
    cudaError_t e = cudaMemcpyAsync(df.dst, df.src, K * df.bytes_per_t, cudaMemcpyHostToDevice,
                                    ctx->stream);
    if (e != cudaSuccess) return e;
  }
  prep_kernel<<<dim3((h->K + 127) / 128, h->B), 128, 0, ctx->stream>>>(h->models_dev, h->tc, h->K,
                                                                       h->bounded);
  ++ctx->launches;
  h->prep_pending = false;
  h->deferred.clear();
  return cudaGetLastError();
}

int run_tree(dsmc_ctx* ctx, dsmc_model_handle* h, const RunOpts& o, RunResult* res) {
  const int B = h->B, K = o.len > 0 ? o.len : h->K, T = K - 1, d = h->d;
  if (o.t0 < 0 || o.t0 + K > h->K)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "window outside the model's horizon");
  const int N = (int)o.N;
  if (N < 1) return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "make_leaf: n must be >= 1");
  if (o.conditional && N < 2)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "conditional_leaf: need n >= 2 slots");
  if (o.resampler < 0 || o.resampler > 3)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "unknown resampler");
  if (o.conditional && o.resampler != DSMC_MULTINOMIAL && o.resampler != DSMC_REJECTION_LAZY)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT,
                   "conditional sweeps need exchangeable unbiased slot draws: use the "
                   "multinomial or rejection-lazy resampler");
  const bool fp64 = o.precision == DSMC_FP64_PARITY;
  if (!fp64 && h->desc.kind == DSMC_MODEL_LGSSM && o.inj_x)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "leaf injection needs FP64 parity precision");
  const bool wide = h->wide;
  if (wide && (fp64 || o.conditional || B != 1 || o.t0 != 0 || K != h->K ||
               (o.resampler != DSMC_MULTINOMIAL && o.resampler != DSMC_SYSTEMATIC)))
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT,
                   "state_dim > 4 runs the FP32 dense path (multinomial / systematic, "
                   "unconditional, whole horizon)");
  const int cap = std::max(1, (K + 1) / 2);
  Bufs b{};
  b.K = K;
  b.T = T;
  b.N = N;
  b.d = d;
  b.B = B;
  b.cap = cap;
  b.models = h->models_dev;
  b.seeds = o.seeds;
  b.tc = h->tc;
  b.bounded = h->bounded;
  b.conditional = o.conditional;
  b.sweep = o.sweep;
  b.star = o.star;
  b.t0 = o.t0;
  b.Kt = h->K;
  Arena& A = ctx->arena;
  void* p;
  const size_t BK = (size_t)B * K, BKN = BK * N, BT = (size_t)B * std::max(T, 1);
  if (fp64) {
    CU(A.get("X64", BKN * d * sizeof(double), &p));
    b.X64 = (double*)p;
    CU(A.get("LW64", BKN * sizeof(double), &p));
    b.LW64 = (double*)p;
  } else if (wide) {
    b.w = h->wb;
    CU(A.get("XW", BKN * h->wb.DP * sizeof(float), &p));
    b.w.X = (float*)p;
    CU(A.get("COL", BKN * sizeof(float), &p));
    b.COL = (float*)p;
    CU(A.get("LW32", (size_t)B * N * sizeof(float), &p));
    b.LW32 = (float*)p;
  } else {
    CU(A.get("X32", BKN * sizeof(float4), &p));
    b.X32 = (float4*)p;
    CU(A.get("COL", BKN * sizeof(float), &p));
    b.COL = (float*)p;
    CU(A.get("LW32", (size_t)B * N * sizeof(float), &p));
    b.LW32 = (float*)p;
  }
  CU(A.get("LNC", BK * sizeof(double), &p));
  b.LNC = (double*)p;
  CU(A.get("LWMAX", BK * sizeof(double), &p));
  b.LWMAX = (double*)p;
  CU(A.get("UNI", BK, &p));
  b.UNI = (uint8_t*)p;
  CU(A.get("PL", BT * N * sizeof(uint32_t), &p));
  b.PL = (uint32_t*)p;
  CU(A.get("PR", BT * N * sizeof(uint32_t), &p));
  b.PR = (uint32_t*)p;
  CU(A.get("LMW", BT * sizeof(double), &p));
  b.LMW = (double*)p;
  CU(A.get("ERR", sizeof(ErrFlag), &p));
  b.err = (ErrFlag*)p;
  CU(A.get("EVALS", B * sizeof(unsigned long long), &p));
  b.evals = (unsigned long long*)p;
  CU(cudaMemsetAsync(b.err, 0, sizeof(ErrFlag), ctx->stream));
  CU(cudaMemsetAsync(b.evals, 0, B * sizeof(unsigned long long), ctx->stream));
  uint32_t* maps[4];
  const char* mnames[4] = {"FA", "LA", "FB", "LB"};
  for (int i = 0; i < 4; ++i) {
    CU(A.get(mnames[i], (size_t)B * cap * N * sizeof(uint32_t), &p));
    maps[i] = (uint32_t*)p;
  }
  double* blnc[2];
  CU(A.get("BLNCA", (size_t)B * cap * sizeof(double), &p));
  blnc[0] = (double*)p;
  CU(A.get("BLNCB", (size_t)B * cap * sizeof(double), &p));
  blnc[1] = (double*)p;

  if (o.timing) CU(rec_event(ctx->ev[0], ctx->stream));
  // ---------------------------------------------------------------- leaves
  if (fp64) {
    const double* dinj_x = nullptr;
    const double* dinj_lw = nullptr;
    if (o.inj_x) {
      CU(A.get("INJX", BKN * d * sizeof(double), &p));
      CU(cudaMemcpyAsync(p, o.inj_x, BKN * d * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
      dinj_x = (const double*)p;
    }
    if (o.inj_lw) {
      CU(A.get("INJW", BKN * sizeof(double), &p));
      CU(cudaMemcpyAsync(p, o.inj_lw, BKN * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
      dinj_lw = (const double*)p;
    }
    CU(flush_deferred(ctx, h));
    leaf64_kernel<<<dim3(K, (N + 127) / 128, B), 128, 0, ctx->stream>>>(b, dinj_x, dinj_lw);
    LAUNCHED(ctx);
    if (o.inj_uni) {  // normalised block weights: flags and maxima as given
      CU(cudaMemcpyAsync(b.UNI, o.inj_uni, BK, cudaMemcpyHostToDevice, ctx->stream));
      CU(cudaMemcpyAsync(b.LWMAX, o.inj_lwmax, BK * sizeof(double), cudaMemcpyHostToDevice,
                         ctx->stream));
      CU(cudaMemsetAsync(b.LNC, 0, BK * sizeof(double), ctx->stream));
    } else {
      leafnorm64_kernel<<<dim3(K, B), 32, 0, ctx->stream>>>(b);
      LAUNCHED(ctx);
    }
  } else if (wide) {
    CU(A.get("RAW0", (size_t)B * N * sizeof(double), &p));
    const dim3 lg(K, B);
    switch (h->wb.DP) {
      case 8: leafw_kernel<8><<<lg, 256, 0, ctx->stream>>>(b, (double*)p); break;
      case 16: leafw_kernel<16><<<lg, 256, 0, ctx->stream>>>(b, (double*)p); break;
      default: leafw_kernel<32><<<lg, 256, 0, ctx->stream>>>(b, (double*)p); break;
    }
    LAUNCHED(ctx);
    leafnorm32_kernel<<<B, 32, 0, ctx->stream>>>(b, (const double*)p);
    LAUNCHED(ctx);
  } else {
    CU(A.get("RAW0", (size_t)B * N * sizeof(double), &p));
    const int lt = std::min(256, (N + 31) / 32 * 32);
    auto leaves = [&](int ta, int tb) {
      const dim3 lg(tb - ta, B);
      switch (d) {
        case 1: leaf32_kernel<1><<<lg, lt, 0, ctx->stream>>>(b, (double*)p, ta); break;
        case 2: leaf32_kernel<2><<<lg, lt, 0, ctx->stream>>>(b, (double*)p, ta); break;
        case 3: leaf32_kernel<3><<<lg, lt, 0, ctx->stream>>>(b, (double*)p, ta); break;
        default: leaf32_kernel<4><<<lg, lt, 0, ctx->stream>>>(b, (double*)p, ta); break;
      }
      LAUNCHED(ctx);
    };
    if (h->prep_pending && o.t0 == 0 && K == h->K) {
      // deferred upload: per time chunk, H2D on the copy stream, then that
      // chunk's prep and leaves on the compute stream
      CU(cudaEventRecord(ctx->gather_ev[0], ctx->stream));  // allocations done
      CU(cudaStreamWaitEvent(ctx->copy_stream, ctx->gather_ev[0], 0));
      const int nch = dsmc_ctx::kGatherChunks;
      for (int c = 0; c < nch; ++c) {
        const int ta = (int)((long)K * c / nch), tb = (int)((long)K * (c + 1) / nch);
        if (tb <= ta) continue;
        for (const auto& df : h->deferred)
          CU(cudaMemcpyAsync(static_cast<char*>(df.dst) + (size_t)ta * df.bytes_per_t,
                             static_cast<const char*>(df.src) + (size_t)ta * df.bytes_per_t,
                             (size_t)(tb - ta) * df.bytes_per_t, cudaMemcpyHostToDevice,
                             ctx->copy_stream));
        CU(cudaEventRecord(ctx->gather_ev[c], ctx->copy_stream));
        CU(cudaStreamWaitEvent(ctx->stream, ctx->gather_ev[c], 0));
        prep_kernel<<<dim3((tb - ta + 127) / 128, B), 128, 0, ctx->stream>>>(
            h->models_dev, h->tc, h->K, h->bounded, ta, tb);
        LAUNCHED(ctx);
        leaves(ta, tb);
      }
      h->prep_pending = false;
      h->deferred.clear();
    } else {
      CU(flush_deferred(ctx, h));
      leaves(0, K);
    }
    if (o.t0 == 0) {  // only global leaf 0 carries non-uniform weights
      leafnorm32_kernel<<<B, 32, 0, ctx->stream>>>(b, (const double*)p);
      LAUNCHED(ctx);
    }
  }
  CU(cudaGetLastError());
  if (o.timing) CU(rec_event(ctx->ev[1], ctx->stream));

  // ---------------------------------------------------------------- levels
  const bool lazy = o.resampler == DSMC_MH_LAZY || o.resampler == DSMC_REJECTION_LAZY;
  const int nsub = (N + kSub - 1) / kSub;
  const size_t ws_comb = fp64 ? (size_t)N * (5 + nsub) + 2 : ((size_t)N * nsub + 1) / 2;
  // bytes of pass-1 scratch per chunk: 4 GB = up to 65535 combines per
  // launch (C5: 412.6 vs 415.3 ms/step at 1 GB; smaller chunks that would
  // keep a chunk's sums in L2 lose more to wave tails: 507 ms at 32 MB;
  // tools/gpu_chunk_ab.sh)
  size_t ws_budget = (size_t)4 << 30;
  if (const char* e = getenv("DSMC_WS_BUDGET_MB")) ws_budget = (size_t)atol(e) << 20;  // A/B
  // bytes per combine of the chunked scratch (the wide path's AUX dominates)
  const size_t per_comb = std::max<size_t>(ws_comb * 8 * B,
                                           wide ? wide_aux_floats(N, h->wb.DP) * 4 * B : 0);
  const int chunk = (int)std::max<size_t>(1, std::min<size_t>(65535, ws_budget / per_comb));
  double* ws = nullptr;
  if (!lazy && T > 0) {
    const int np1 = K / 2;
    CU(A.get("WS", (size_t)std::min(chunk, np1) * ws_comb * 8 * B, &p));
    ws = (double*)p;
  }
  int cur = 0;  // maps[2*cur], maps[2*cur+1] hold the previous level
  int nb = K, level = 0;
  size_t cursor = 0;
  const int mc = model_class(h->desc.kind, d, h->desc.kind == DSMC_MODEL_SV ? 1 : h->dy);
  while (nb > 1) {
    ++level;
    const int np = nb / 2;
    LevelArgs la{};
    la.level = level;
    la.np = np;
    la.nb_prev = nb;
    la.cursor = cursor;
    la.first_prev = maps[2 * cur];
    la.last_prev = maps[2 * cur + 1];
    la.first_next = maps[2 * (1 - cur)];
    la.last_next = maps[2 * (1 - cur) + 1];
    la.blnc_prev = blnc[cur];
    la.blnc_next = blnc[1 - cur];
    la.n_out = o.n_out >= 0 ? o.n_out : (o.conditional ? N - 1 : N);
    la.ws = ws;
    la.ws_comb = ws_comb;
    la.key_level = o.key_level >= 0 ? o.key_level : level;
    la.node_off = o.key_level >= 0 ? o.key_node : (long long)(o.t0 >> level);
    if (o.conditional) {
      la.k0 = 0;
      if (fp64) {
        refpair_check_kernel<<<dim3((np + 127) / 128, 1, B), 128, 0, ctx->stream>>>(b, la);
        LAUNCHED(ctx);
      }
    }
    for (int k0 = 0; k0 < np; k0 += chunk) {
      const int nk = std::min(chunk, np - k0);
      la.k0 = k0;
      int rc = 0;
      if (lazy) {
        const int mh = o.resampler == DSMC_MH_LAZY;
        const dim3 grid((la.n_out + 127) / 128, nk, B);
        if (fp64) {
          lazy64_kernel<<<grid, 128, 0, ctx->stream>>>(b, la, mh, o.mh_steps);
        } else {
          switch (d) {
            case 1: launch_lazy32<1>(grid, ctx->stream, b, la, mh, o.mh_steps); break;
            case 2: launch_lazy32<2>(grid, ctx->stream, b, la, mh, o.mh_steps); break;
            case 3: launch_lazy32<3>(grid, ctx->stream, b, la, mh, o.mh_steps); break;
            default: launch_lazy32<4>(grid, ctx->stream, b, la, mh, o.mh_steps); break;
          }
        }
        LAUNCHED(ctx);
        lazy_finish_kernel<<<dim3(nk, 1, B), 256, 0, ctx->stream>>>(b, la);
        LAUNCHED(ctx);
      } else {
        const int sys = o.resampler == DSMC_SYSTEMATIC;
        if (fp64) {
          rc = mc == kLG1 ? launch_c64<kLG1, 1>(ctx, b, la, nk, sys)
             : mc == kSV  ? launch_c64<kSV, 1>(ctx, b, la, nk, sys)
             : mc == kCOX ? launch_c64<kCOX, 1>(ctx, b, la, nk, sys)
             : mc == kCRW ? launch_c64<kCRW, 1>(ctx, b, la, nk, sys)
             : mc == kTHETA ? launch_c64<kTHETA, 1>(ctx, b, la, nk, sys)
             : d == 1     ? launch_c64<kLGN, 1>(ctx, b, la, nk, sys)
             : d == 2     ? launch_c64<kLGN, 2>(ctx, b, la, nk, sys)
             : d == 3     ? launch_c64<kLGN, 3>(ctx, b, la, nk, sys)
                          : launch_c64<kLGN, 4>(ctx, b, la, nk, sys);
        } else if (wide) {
          rc = h->wb.DP == 8    ? launch_wide<8>(ctx, b, la, nk, sys)
             : h->wb.DP == 16 ? launch_wide<16>(ctx, b, la, nk, sys)
                              : launch_wide<32>(ctx, b, la, nk, sys);
        } else {
          rc = d == 1 ? launch_c32<1>(ctx, b, la, nk, sys)
             : d == 2 ? launch_c32<2>(ctx, b, la, nk, sys)
             : d == 3 ? launch_c32<3>(ctx, b, la, nk, sys)
                      : launch_c32<4>(ctx, b, la, nk, sys);
        }
      }
      if (rc) return rc;
      CU(cudaGetLastError());
    }
    if (nb % 2) {  // odd tail carried to the next level
      const int s = 1 << (level - 1);
      const bool tail_leaf = (nb - 1) * s == K - 1;
      if (!tail_leaf) {
        tail_copy_kernel<<<dim3(4, B), 256, 0, ctx->stream>>>(
            b, nb - 1, np, la.first_prev, la.last_prev, la.first_next, la.last_next,
            la.blnc_prev, la.blnc_next);
        LAUNCHED(ctx);
      }
    }
    cur = 1 - cur;
    cursor += np;
    nb = (nb + 1) / 2;
  }
  if (o.timing) CU(rec_event(ctx->ev[2], ctx->stream));
  res->levels = level;
  res->PL = b.PL;
  res->PR = b.PR;
  res->LMW = b.LMW;
  res->root_lnc = K == 1 ? b.LNC : blnc[cur];
  res->lnc_stride = K == 1 ? (size_t)K : (size_t)cap;
  res->evals = b.evals;
  res->err = b.err;
  res->LNC = b.LNC;
  res->X64 = b.X64;
  res->LW64 = b.LW64;
  {
    WindowState& st = window_state(ctx);
    st.valid = true;
    st.b = b;
    st.levels = level;
    st.cur = cur;
    for (int i = 0; i < 4; ++i) st.maps[i] = maps[i];
    st.blnc[0] = blnc[0];
    st.blnc[1] = blnc[1];
    st.resampler = o.resampler;
  }
  if (!o.compose) {
    if (o.timing) CU(rec_event(ctx->ev[3], ctx->stream));
    return DSMC_OK;
  }

  // ----------------------------------------------------------- composition
  if (o.conditional) {
    uint32_t* S[2];
    CU(A.get("SA", (size_t)B * cap * 2 * sizeof(uint32_t), &p));
    S[0] = (uint32_t*)p;
    CU(A.get("SB", (size_t)B * cap * 2 * sizeof(uint32_t), &p));
    S[1] = (uint32_t*)p;
    star_select_kernel<<<(B + 63) / 64, 64, 0, ctx->stream>>>(b, level, S[0], !fp64);
    LAUNCHED(ctx);
    int sc = 0;
    std::vector<int> nbs{K};
    while (nbs.back() > 1) nbs.push_back((nbs.back() + 1) / 2);
    std::vector<size_t> cursors(nbs.size() + 1, 0);
    for (size_t l = 1; l + 1 <= nbs.size() - 1; ++l) cursors[l + 1] = cursors[l] + nbs[l - 1] / 2;
    for (int l = level; l >= 2; --l) {
      td1_kernel<<<dim3((nbs[l] + 127) / 128, B), 128, 0, ctx->stream>>>(
          b, cursors[l], nbs[l], nbs[l - 1], S[sc], S[1 - sc]);
      LAUNCHED(ctx);
      sc = 1 - sc;
    }
    star_path_kernel<<<dim3((K + 127) / 128, B), 128, 0, ctx->stream>>>(b, S[sc], !fp64,
                                                                       o.star_out, o.changed);
    LAUNCHED(ctx);
  } else if (o.paths || o.mean || o.cov) {
    std::vector<int> nbs{K};
    while (nbs.back() > 1) nbs.push_back((nbs.back() + 1) / 2);
    std::vector<size_t> cursors(nbs.size() + 1, 0);
    for (size_t l = 1; l + 1 <= nbs.size() - 1; ++l) cursors[l + 1] = cursors[l] + nbs[l - 1] / 2;
    // reuse the map buffers (bottom-up maps are dead now)
    uint32_t* Mb[2] = {maps[0], maps[2]};
    int mcur = 0;
    bool root = true;
    for (int l = level; l >= 2; --l) {
      CU(launch_pdl(td_kernel, dim3(nbs[l], (N + 255) / 256, B), dim3(256), 0, ctx->stream, b, l,
                    cursors[l], nbs[l], nbs[l - 1], (const uint32_t*)Mb[mcur], Mb[1 - mcur],
                    root ? 1 : 0, o.root_map));
      LAUNCHED(ctx);
      root = false;
      mcur = 1 - mcur;
    }
    if (fp64) {
      gather64_kernel<<<dim3(K, B), 256, 0, ctx->stream>>>(b, Mb[mcur], root ? 1 : 0,
                                                           o.paths, o.mean, o.cov, o.root_map);
    } else if (wide) {
      const dim3 gg(K, B);
      const int r1 = root ? 1 : 0;
      switch (h->wb.DP) {
        case 8: gatherw_kernel<8><<<gg, 256, 0, ctx->stream>>>(b, Mb[mcur], r1, o.paths, o.mean, o.cov, o.root_map); break;
        case 16: gatherw_kernel<16><<<gg, 256, 0, ctx->stream>>>(b, Mb[mcur], r1, o.paths, o.mean, o.cov, o.root_map); break;
        default: gatherw_kernel<32><<<gg, 256, 0, ctx->stream>>>(b, Mb[mcur], r1, o.paths, o.mean, o.cov, o.root_map); break;
      }
      LAUNCHED(ctx);
    } else {
      const uint32_t* M1 = Mb[mcur];
      const int r1 = root ? 1 : 0;
      const bool overlap = (o.host_mean || o.host_cov) && B == 1 && ctx->copy_stream;
      const int nch = overlap ? dsmc_ctx::kGatherChunks : 1;
      for (int c = 0; c < nch; ++c) {
        const int ta = (int)((long)K * c / nch), tb = (int)((long)K * (c + 1) / nch);
        if (tb <= ta) continue;
        const dim3 grid((tb - ta + 7) / 8, B);
        switch (d) {
          case 1: gather32_kernel<1><<<grid, 256, 0, ctx->stream>>>(b, M1, r1, o.paths, o.mean, o.cov, o.root_map, ta, tb); break;
          case 2: gather32_kernel<2><<<grid, 256, 0, ctx->stream>>>(b, M1, r1, o.paths, o.mean, o.cov, o.root_map, ta, tb); break;
          case 3: gather32_kernel<3><<<grid, 256, 0, ctx->stream>>>(b, M1, r1, o.paths, o.mean, o.cov, o.root_map, ta, tb); break;
          default: gather32_kernel<4><<<grid, 256, 0, ctx->stream>>>(b, M1, r1, o.paths, o.mean, o.cov, o.root_map, ta, tb); break;
        }
        LAUNCHED(ctx);
        if (overlap) {
          CU(cudaEventRecord(ctx->gather_ev[c], ctx->stream));
          CU(cudaStreamWaitEvent(ctx->copy_stream, ctx->gather_ev[c], 0));
          const size_t n = (size_t)(tb - ta);
          if (o.host_mean && o.mean)
            CU(cudaMemcpyAsync(o.host_mean + (size_t)ta * d, o.mean + (size_t)ta * d,
                               n * d * sizeof(double), cudaMemcpyDeviceToHost, ctx->copy_stream));
          if (o.host_cov && o.cov)
            CU(cudaMemcpyAsync(o.host_cov + (size_t)ta * d * d, o.cov + (size_t)ta * d * d,
                               n * d * d * sizeof(double), cudaMemcpyDeviceToHost,
                               ctx->copy_stream));
        }
      }
    }
    if (fp64) LAUNCHED(ctx);
  }
  CU(cudaGetLastError());
  if (o.timing) CU(rec_event(ctx->ev[3], ctx->stream));
  return DSMC_OK;
}

// Read back the device error record (the one host sync of a run).
int check_device_error(dsmc_ctx* ctx, const RunResult& r, int K) {
  ErrFlag e;
  CU(cudaMemcpyAsync(&e, r.err, sizeof e, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  if (e.code) return set_err(ctx, e.code, err_message(e, K));
  return DSMC_OK;
}

// Device error record of the last resident / window run (enqueued without a
// host sync): read it once, after the stream drains, and clear it.
int check_pending_error(dsmc_ctx* ctx) {
  if (!ctx->last_err) return DSMC_OK;
  ErrFlag e;
  CU(cudaMemcpyAsync(&e, ctx->last_err, sizeof e, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  ctx->last_err = nullptr;
  if (e.code) return set_err(ctx, e.code, err_message(e, ctx->last_err_K));
  return DSMC_OK;
}

struct DevSeeds {
  uint64_t* p = nullptr;
};

// Kernel attributes are per function and per device and shared by every
// context (and host thread) of the process: set them once per device, to the
// opt-in maximum, under a lock — never per launch (a per-launch
// cudaFuncSetAttribute with a level-dependent size races with other host
// threads and could lower a limit another thread's launch needs).
// dynamic limit = opt-in maximum minus the kernel's static shared memory
template <typename F>
cudaError_t set_max_dynamic_smem(F fn, int optin) {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, fn);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              optin - (int)fa.sharedSizeBytes);
}
template <int D>
cudaError_t configure_d(int smem) {
  cudaError_t e = cudaSuccess;
  auto set = [&](auto fn) {
    if (e != cudaSuccess) return;
    e = set_max_dynamic_smem(fn, smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared);
  };
  set(c32_sample<D, 3>);
  set(c32_sample<D, 4>);
  set(c64_rows<kLGN, D>);
  set(c64_sample<kLGN, D>);
  set(pf_forward_kernel<D>);
  set(ffbs_backward_kernel<D>);
  if (e == cudaSuccess) e = set_max_dynamic_smem(samplew_kernel<4, Aux32Recompute<D>>, smem);
  return e;
}
template <int D>
cudaError_t configure_wide(int smem) {
  cudaError_t e = set_max_dynamic_smem(pairw_kernel<D>, smem);
  if (e == cudaSuccess) e = set_max_dynamic_smem(samplew_kernel<D>, smem);
  if (e == cudaSuccess) e = set_max_dynamic_smem(pairw_tc_kernel<D>, smem);
  if (e == cudaSuccess) e = set_max_dynamic_smem(pairw_tc2_kernel<D>, smem);
  return e;
}
cudaError_t configure_device(int device, int smem) {
  static std::mutex mu;
  static std::vector<int> done;
  std::lock_guard<std::mutex> lock(mu);
  if (std::find(done.begin(), done.end(), device) != done.end()) return cudaSuccess;
  cudaError_t e = configure_d<1>(smem);
  if (e == cudaSuccess) e = configure_d<2>(smem);
  if (e == cudaSuccess) e = configure_d<3>(smem);
  if (e == cudaSuccess) e = configure_d<4>(smem);
  if (e == cudaSuccess) e = configure_wide<8>(smem);
  if (e == cudaSuccess) e = configure_wide<16>(smem);
  if (e == cudaSuccess) e = configure_wide<32>(smem);
  for (auto fn : {c64_rows<kLG1, 1>, c64_rows<kSV, 1>, c64_rows<kCOX, 1>, c64_rows<kCRW, 1>,
                  c64_rows<kTHETA, 1>}) {
    if (e != cudaSuccess) break;
    e = set_max_dynamic_smem(fn, smem);
  }
  for (auto fn : {c64_sample<kLG1, 1>, c64_sample<kSV, 1>, c64_sample<kCOX, 1>,
                  c64_sample<kCRW, 1>, c64_sample<kTHETA, 1>}) {
    if (e != cudaSuccess) break;
    e = set_max_dynamic_smem(fn, smem);
  }
  if (e == cudaSuccess) done.push_back(device);
  return e;
}

}  // namespace

// =================================================================== C ABI
extern "C" {

int dsmc_create(int device, dsmc_ctx** out) {
  if (!out) return DSMC_E_INVALID_ARGUMENT;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= device || device < 0)
    return DSMC_E_NO_DEVICE;
  auto* ctx = new dsmc_ctx();
  ctx->device = device;
  if (const char* pk = getenv("DSMC_PAIR_KERNEL")) {
    ctx->pair_tc = strcmp(pk, "tc") == 0;
    ctx->pair_tc2 = strcmp(pk, "tc2") == 0;
  }
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  cudaDeviceGetAttribute(&ctx->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  cudaDeviceGetAttribute(&ctx->smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return DSMC_E_NO_DEVICE;
  }
  if (configure_device(device, ctx->smem_optin) != cudaSuccess) {
    cudaGetLastError();
    cudaStreamDestroy(ctx->stream);
    delete ctx;
    return DSMC_E_NO_DEVICE;
  }
  for (auto& e : ctx->ev) cudaEventCreate(&e);
  cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking);
  for (auto& e : ctx->gather_ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  cudaMallocHost(&ctx->h_lnc, sizeof(double) * 4096);
  // model uploads use the stream-ordered pool (cudaMallocAsync); keep freed
  // blocks mapped so repeated uploads (e2e calls, pGibbs sweeps) reuse them
  // instead of re-mapping up to ~1 GB of per-time constants every call
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  *out = ctx;
  return DSMC_OK;
}

void dsmc_destroy(dsmc_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  ctx->gc.reset();
  ctx->arena.release();
  if (ctx->d_mean) cudaFree(ctx->d_mean);
  if (ctx->d_cov) cudaFree(ctx->d_cov);
  if (ctx->h_lnc) cudaFreeHost(ctx->h_lnc);
  for (auto& e : ctx->ev) cudaEventDestroy(e);
  for (auto& e : ctx->kev) cudaEventDestroy(e);
  delete static_cast<WindowState*>(ctx->window);
  cudaStreamDestroy(ctx->stream);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  for (auto& e : ctx->gather_ev)
    if (e) cudaEventDestroy(e);
  delete ctx;
}

const char* dsmc_last_error(const dsmc_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }
uint64_t dsmc_kernel_launches(const dsmc_ctx* ctx) { return ctx ? ctx->launches : 0; }
void* dsmc_stream(dsmc_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }
int dsmc_sync(dsmc_ctx* ctx) {
  if (!ctx) return DSMC_E_INVALID_ARGUMENT;
  CU(cudaStreamSynchronize(ctx->stream));
  return check_pending_error(ctx);
}

int dsmc_model_upload(dsmc_ctx* ctx, const dsmc_model_desc* model,
                      dsmc_model_handle** out) {
  if (!ctx || !out) return DSMC_E_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  return make_handle(ctx, model, 1, out);
}

int dsmc_model_upload_window(dsmc_ctx* ctx, const dsmc_model_desc* model, int t0, int len,
                             dsmc_model_handle** out) {
  if (!ctx || !out || !model) return DSMC_E_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  const int K = model->horizon + 1;
  if (len < 1 || t0 < 0 || t0 + len > K)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "window upload: [t0, t0 + len) outside the horizon");
  // the window's times plus its right cross cut t0 + len (combined on this rank)
  return make_handle(ctx, model, 1, out, false, t0, std::min(K, t0 + len + 1));
}

void dsmc_model_free(dsmc_ctx* ctx, dsmc_model_handle* h) {
  if (ctx) cudaStreamSynchronize(ctx->stream);
  if (ctx && h && ctx->gc.handle == h->id) ctx->gc.reset();
  free_handle(h);
}

__global__ void set_seed_kernel(uint64_t* dst, uint64_t v) { *dst = v; }

static int smooth_common(dsmc_ctx* ctx, dsmc_model_handle* h, const dsmc_smooth_opts* opts,
                         double* d_paths, double* d_mean, double* d_cov, RunResult* res,
                         bool timing, double* host_mean = nullptr, double* host_cov = nullptr) {
  if (!opts) return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "options are null");
  RunOpts o;
  o.precision = opts->precision;
  o.resampler = opts->resampler;
  o.mh_steps = opts->mh_steps;
  o.N = opts->n_particles;
  o.inj_x = opts->inject_states;
  o.inj_lw = opts->inject_logw;
  o.paths = d_paths;
  o.mean = d_mean;
  o.cov = d_cov;
  o.host_mean = host_mean;
  o.host_cov = host_cov;
  o.timing = timing;
  ctx->time_kernels = timing;
  ctx->kev_used = 0;
  void* p;
  CU(ctx->arena.get("SEEDS", sizeof(uint64_t), &p));
  // the seed travels as a kernel argument (a graph replay updates it there);
  // timing events are recorded as EXTERNAL nodes so they stay measurable
  // when the run is replayed from a CUDA graph
  set_seed_kernel<<<1, 1, 0, ctx->stream>>>((uint64_t*)p, opts->seed);
  LAUNCHED(ctx);
  ctx->gc.seed_dst = (uint64_t*)p;
  o.seeds = (const uint64_t*)p;
  return run_tree(ctx, h, o, res);
}

// page-locked (or absent) host memory: async copies really overlap
static bool host_pinned(const void* ptr) {
  if (!ptr) return true;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

int dsmc_smooth(dsmc_ctx* ctx, const dsmc_model_desc* model,
                const dsmc_smooth_opts* opts, dsmc_smooth_out* out) {
  if (!ctx || !out) return DSMC_E_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  if (opts && opts->precision != DSMC_FP64_PARITY && (out->leaf_states || out->leaf_logw))
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT,
                   "leaf_states / leaf_logw are FP64-parity outputs (the FP32 path stores "
                   "centred single-precision leaves)");
  const auto t0 = std::chrono::steady_clock::now();
  dsmc_model_handle* h = nullptr;
  // FP32 with pinned per-time arrays: upload them in time chunks that
  // overlap the first chunks' prep and leaves (run_tree)
  // (only for large horizons: below ~32 MB the chunking costs more than the copy)
  const size_t big = model ? (size_t)(model->horizon + 1) * model->state_dim *
                                 (model->state_dim + 1) * sizeof(double)
                           : 0;
  const bool defer = opts && opts->precision == DSMC_FP32 && model && big >= (32u << 20) &&
                     model->state_dim <= 4 && !force_wide() &&
                     host_pinned(model->y) && host_pinned(model->prop_mean) &&
                     host_pinned(model->prop_cov);
  int rc = make_handle(ctx, model, 1, &h, defer);
  if (rc) return rc;
  std::unique_ptr<dsmc_model_handle, void (*)(dsmc_model_handle*)> hold(h, free_handle);
  const int K = h->K, d = h->d, T = K - 1;
  const size_t N = opts ? opts->n_particles : 0;
  void* p;
  double *dp = nullptr, *dm = nullptr, *dc = nullptr;
  if (out->paths) {
    CU(ctx->arena.get("OPATH", (size_t)K * N * d * sizeof(double), &p));
    dp = (double*)p;
  }
  if (out->mean) {
    CU(ctx->arena.get("OMEAN", (size_t)K * d * sizeof(double), &p));
    dm = (double*)p;
  }
  if (out->cov) {
    CU(ctx->arena.get("OCOV", (size_t)K * d * d * sizeof(double), &p));
    dc = (double*)p;
  }
  RunResult res;
  // FP32 with pinned outputs: the moments come back in chunks overlapping the
  // final gather (a copy to pageable memory would block the host per chunk)
  const bool overlap = opts && opts->precision == DSMC_FP32 && (dm || dc) &&
                       (size_t)K * d * (d + 1) * sizeof(double) >= (32u << 20) &&
                       host_pinned(out->mean) && host_pinned(out->cov);
  rc = smooth_common(ctx, h, opts, dp, dm, dc, &res, false, overlap ? out->mean : nullptr,
                     overlap ? out->cov : nullptr);
  if (rc) {
    cudaStreamSynchronize(ctx->copy_stream);
    return rc;
  }
  rc = check_device_error(ctx, res, K);
  if (rc) {
    cudaStreamSynchronize(ctx->copy_stream);
    return rc;
  }
  auto s = ctx->stream;
  if (dp) CU(cudaMemcpyAsync(out->paths, dp, (size_t)K * N * d * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (dm && !overlap) CU(cudaMemcpyAsync(out->mean, dm, (size_t)K * d * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (dc && !overlap) CU(cudaMemcpyAsync(out->cov, dc, (size_t)K * d * d * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (out->pair_left && T > 0)
    CU(cudaMemcpyAsync(out->pair_left, res.PL, (size_t)T * N * 4, cudaMemcpyDeviceToHost, s));
  if (out->pair_right && T > 0)
    CU(cudaMemcpyAsync(out->pair_right, res.PR, (size_t)T * N * 4, cudaMemcpyDeviceToHost, s));
  if (out->log_mean_weight && T > 0)
    CU(cudaMemcpyAsync(out->log_mean_weight, res.LMW, (size_t)T * 8, cudaMemcpyDeviceToHost, s));
  if (out->leaf_states && res.X64)
    CU(cudaMemcpyAsync(out->leaf_states, res.X64, (size_t)K * N * d * 8, cudaMemcpyDeviceToHost, s));
  if (out->leaf_logw && res.LW64)
    CU(cudaMemcpyAsync(out->leaf_logw, res.LW64, (size_t)K * N * 8, cudaMemcpyDeviceToHost, s));
  double lnc;
  unsigned long long evals = 0;
  CU(cudaMemcpyAsync(&lnc, res.root_lnc, sizeof(double), cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(&evals, res.evals, sizeof evals, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (overlap) CU(cudaStreamSynchronize(ctx->copy_stream));
  const bool lazy = opts->resampler == DSMC_MH_LAZY || opts->resampler == DSMC_REJECTION_LAZY;
  out->log_norm_const = lnc;
  out->has_log_norm_const = !std::isnan(lnc);
  out->levels = res.levels;
  out->weight_evals = lazy ? evals : (uint64_t)T * N * N;
  out->biased = opts->resampler == DSMC_MH_LAZY && T > 0;
  out->wall_time_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return DSMC_OK;
}

int dsmc_smooth_resident(dsmc_ctx* ctx, const dsmc_model_handle* hc,
                         const dsmc_smooth_opts* opts) {
  if (!ctx || !hc || !opts) return DSMC_E_INVALID_ARGUMENT;
  auto* h = const_cast<dsmc_model_handle*>(hc);
  const int K = h->K, d = h->d;
  // capacity is kept apart from the shape of the last run: a smaller run after
  // a larger one reuses the buffers, and dsmc_resident_results copies exactly
  // the last run's K x d (never the capacity)
  if (ctx->mean_cap < (size_t)K * d || ctx->cov_cap < (size_t)K * d * d) {
    cudaStreamSynchronize(ctx->stream);
    if (ctx->d_mean) cudaFree(ctx->d_mean);
    if (ctx->d_cov) cudaFree(ctx->d_cov);
    ctx->d_mean = ctx->d_cov = nullptr;
    ctx->mean_cap = ctx->cov_cap = 0;
    CU(cudaMalloc(&ctx->d_mean, (size_t)K * d * sizeof(double)));
    CU(cudaMalloc(&ctx->d_cov, (size_t)K * d * d * sizeof(double)));
    ctx->mean_cap = (size_t)K * d;
    ctx->cov_cap = (size_t)K * d * d;
    ++ctx->arena.epoch;  // moved outputs invalidate a captured graph
  }
  ctx->last_K = K;
  ctx->last_d = d;
  ctx->last_err_K = K;
  auto& gc = ctx->gc;
  const bool same = gc.handle == h->id && gc.epoch == ctx->arena.epoch && gc.N == opts->n_particles &&
                    gc.rs == opts->resampler && gc.prec == opts->precision &&
                    gc.mh == opts->mh_steps && !opts->inject_states && !opts->inject_logw;
  const bool graphs = !getenv("DSMC_NO_GRAPH");
  if (graphs && same && gc.exec) {  // replay with the new seed
    uint64_t* dst = gc.seed_dst;
    uint64_t seed = opts->seed;
    void* args[2] = {&dst, &seed};
    cudaKernelNodeParams kp = gc.seed_params;
    kp.kernelParams = args;
    kp.extra = nullptr;
    CU(cudaGraphExecKernelNodeSetParams(gc.exec, gc.seed_node, &kp));
    CU(cudaGraphLaunch(gc.exec, ctx->stream));
    ctx->last_err = gc.err;  // the replay resets and fills the same record
    ctx->launches += gc.launches;
    ctx->kev_used = gc.kev_used;
    ctx->time_kernels = true;
    ctx->last_levels = gc.levels;
    return DSMC_OK;
  }
  auto run = [&](RunResult& res) -> int {
    int rc = smooth_common(ctx, h, opts, nullptr, ctx->d_mean, ctx->d_cov, &res, true);
    if (rc) return rc;
    ctx->last_err = res.err;
    CU(cudaMemcpyAsync(ctx->h_lnc, res.root_lnc, sizeof(double), cudaMemcpyDeviceToHost,
                       ctx->stream));
    return DSMC_OK;
  };
  if (graphs && same && gc.seen >= 1 && !gc.exec) {  // second identical call: capture
    const uint64_t l0 = ctx->launches;
    const uint64_t epoch0 = ctx->arena.epoch;
    RunResult res;
    int rc = DSMC_OK;
    cudaGraph_t graph = nullptr;
    if (cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
      rc = run(res);
      cudaStreamEndCapture(ctx->stream, &graph);
    }
    cudaGraphExec_t exec = nullptr;
    bool ok = rc == DSMC_OK && graph && ctx->arena.epoch == epoch0 &&
              cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
    cudaGraphNode_t seed_node = nullptr;
    cudaKernelNodeParams seed_params{};
    if (ok) {
      size_t n = 0;
      cudaGraphGetNodes(graph, nullptr, &n);
      std::vector<cudaGraphNode_t> nodes(n);
      cudaGraphGetNodes(graph, nodes.data(), &n);
      for (auto nd : nodes) {
        cudaGraphNodeType ty;
        cudaKernelNodeParams kp;
        if (cudaGraphNodeGetType(nd, &ty) == cudaSuccess && ty == cudaGraphNodeTypeKernel &&
            cudaGraphKernelNodeGetParams(nd, &kp) == cudaSuccess &&
            kp.func == reinterpret_cast<void*>(set_seed_kernel)) {
          seed_node = nd;
          seed_params = kp;
        }
      }
      ok = seed_node != nullptr;
    }
    if (ok) {
      gc.graph = graph;
      gc.exec = exec;
      gc.seed_node = seed_node;
      gc.seed_params = seed_params;
      gc.launches = ctx->launches - l0;
      gc.err = res.err;
      gc.kev_used = ctx->kev_used;
      gc.levels = res.levels;
      ctx->launches = l0;
      CU(cudaGraphLaunch(gc.exec, ctx->stream));
      ctx->launches += gc.launches;
      ctx->last_levels = gc.levels;
      return DSMC_OK;
    }
    // capture failed: drop it and run eagerly (and do not try again)
    cudaGetLastError();
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    ctx->launches = l0;
    gc.seen = -1000000;
  }
  if (!same) {
    if (gc.exec) cudaStreamSynchronize(ctx->stream);
    gc.reset();
    gc.handle = h->id;
    gc.N = opts->n_particles;
    gc.rs = opts->resampler;
    gc.prec = opts->precision;
    gc.mh = opts->mh_steps;
    gc.seen = 0;
  }
  RunResult res;
  int rc = run(res);
  if (rc) return rc;
  ctx->last_levels = res.levels;
  gc.epoch = ctx->arena.epoch;  // buffers as left by this run
  ++gc.seen;
  return DSMC_OK;
}

int dsmc_resident_results(dsmc_ctx* ctx, double* mean, double* cov,
                          double* lnc, int* has_lnc) {
  if (!ctx) return DSMC_E_INVALID_ARGUMENT;
  if (!ctx->d_mean) return set_err(ctx, DSMC_E_LOGIC, "no resident run on this context");
  int rc = check_pending_error(ctx);  // syncs; a failed run returns its error, not garbage
  if (rc) return rc;
  const int K = ctx->last_K, d = ctx->last_d;
  if (mean) CU(cudaMemcpyAsync(mean, ctx->d_mean, (size_t)K * d * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (cov) CU(cudaMemcpyAsync(cov, ctx->d_cov, (size_t)K * d * d * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  if (lnc) *lnc = ctx->h_lnc[0];
  if (has_lnc) *has_lnc = !std::isnan(ctx->h_lnc[0]);
  return DSMC_OK;
}

int dsmc_last_timings(const dsmc_ctx* ctx, double* ms, int cap) {
  if (!ctx || cap < 3) return 0;
  if (cap >= 6) {  // [3] pair-kernel ms, [4] sample-kernel ms, [5] pair launches
    double pk = 0, sk = 0;
    bool ok = true;
    for (int i = 0; i + 2 < ctx->kev_used; i += 3) {
      float a = 0, b = 0;
      ok &= cudaEventElapsedTime(&a, ctx->kev[i], ctx->kev[i + 1]) == cudaSuccess;
      ok &= cudaEventElapsedTime(&b, ctx->kev[i + 1], ctx->kev[i + 2]) == cudaSuccess;
      pk += a;
      sk += b;
    }
    ms[3] = ok ? pk : -1.0;
    ms[4] = ok ? sk : -1.0;
    ms[5] = ctx->kev_used / 3;
  }
  float t[3] = {0, 0, 0};
  for (int i = 0; i < 3; ++i)
    if (cudaEventElapsedTime(&t[i], ctx->ev[i], ctx->ev[i + 1]) != cudaSuccess) t[i] = -1.f;
  for (int i = 0; i < 3; ++i) ms[i] = t[i];
  cudaGetLastError();  // an unavailable timing must not leak into the next call
  return cap >= 6 ? 6 : 3;
}

// ------------------------------------------------------------ table path
__global__ void table_rows_kernel(const double* logw, int n, double* ws, ErrFlag* err) {
  // one warp per row: max, sub-block sums (8-lane), raw total
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * 8 + warp;
  if (i >= n) return;
  const int nsub = (n + kSub - 1) / kSub;
  double *wm = ws, *wraw = ws + n, *wsub = ws + 5 * (size_t)n;
  const double* row = logw + (size_t)i * n;
  double mx = -CUDART_INF;
  int nan = 0;
  for (int j = lane; j < n; j += 32) {
    nan |= isnan(row[j]);
    mx = fmax(mx, row[j]);
  }
  for (int o = 16; o; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(~0u, mx, o));
    nan |= __shfl_xor_sync(~0u, nan, o);
  }
  if (nan) {
    if (lane == 0) raise_err(err, DSMC_E_DOMAIN, 0, 1, kReasonNaN);
    mx = -CUDART_INF;
  }
  if (lane == 0) wm[i] = mx;
  double* srow = wsub + (size_t)i * nsub;
  if (mx == -CUDART_INF) {
    for (int s = lane; s < nsub; s += 32) srow[s] = 0.0;
    if (lane == 0) wraw[i] = 0.0;
    return;
  }
  const int grp = lane >> 3, l8 = lane & 7;
  for (int s0 = 0; s0 < nsub; s0 += 4) {
    const int s = s0 + grp;
    const bool act = s < nsub;
    const int j0 = s * kSub;
    const int len = act ? min(kSub, n - j0) : 0;
    const int len8 = len & ~7;
    double acc = 0.0;
    for (int q = 0; q < len8; q += 8) acc = DADD(acc, exp_w(DSUB(row[j0 + q + l8], mx)));
    double a8[8];
    for (int l = 0; l < 8; ++l) a8[l] = __shfl_sync(~0u, acc, (lane & ~7) + l);
    if (act && l8 == 0) {
      double bs = combine8(a8);
      for (int j = j0 + len8; j < j0 + len; ++j) bs = DADD(bs, exp_w(DSUB(row[j], mx)));
      srow[s] = bs;
    }
  }
  __syncwarp();
  if (lane == 0) {
    double tot = 0.0;
    for (int s = 0; s < nsub; ++s) tot = DADD(tot, srow[s]);
    wraw[i] = tot;
  }
}

__global__ void table_sample_kernel(const double* logw, int n, int n_out, double* ws,
                                    uint64_t seed, uint32_t level, uint64_t node,
                                    int systematic, uint32_t* left, uint32_t* right,
                                    double* lmw_out, ErrFlag* err) {
  __shared__ double red[32];
  __shared__ double s_g, s_grand;
  __shared__ double a8s[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nsub = (n + kSub - 1) / kSub;
  double *wm = ws, *wraw = ws + n, *wscale = ws + 2 * (size_t)n, *wtot = ws + 3 * (size_t)n,
         *wpre = ws + 4 * (size_t)n, *wsub = ws + 5 * (size_t)n;
  double mx = -CUDART_INF;
  for (int i = tid; i < n; i += blockDim.x) mx = fmax(mx, wm[i]);
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(~0u, mx, o));
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  if (tid == 0) {
    double v = -CUDART_INF;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v = fmax(v, red[w]);
    s_g = v;
  }
  __syncthreads();
  const double gmax = s_g;
  if (gmax == -CUDART_INF) {
    if (tid == 0) raise_err(err, DSMC_E_RUNTIME, 0, 1, kReasonZeroTable);
    return;
  }
  for (int i = tid; i < n; i += blockDim.x) {
    const double sc = exp_w(DSUB(wm[i], gmax));
    wscale[i] = sc;
    wtot[i] = DMUL(sc, wraw[i]);
  }
  __syncthreads();
  const int n8 = n & ~7;
  if (tid < 8) {
    double acc = 0.0;
    for (int i = tid; i < n8; i += 8) acc = DADD(acc, wtot[i]);
    a8s[tid] = acc;
  }
  __syncthreads();
  if (tid == 0) {
    double a8[8];
    for (int l = 0; l < 8; ++l) a8[l] = a8s[l];
    double tot = combine8(a8);
    for (int i = n8; i < n; ++i) tot = DADD(tot, wtot[i]);
    s_grand = tot;
    double cum = 0.0;
    for (int i = 0; i < n; ++i) {
      cum = DADD(cum, wtot[i]);
      wpre[i] = cum;
    }
    *lmw_out = DADD(gmax, log(tot));
  }
  __syncthreads();
  const double grand = s_grand;
  const StreamId id = stream_id(seed, level, node, DSMC_ROLE_PAIR_RESAMPLE, 0);
  double u0 = 0.0, step = 0.0;
  if (systematic) {
    u0 = u64_uniform(stream_u64(id, 0));
    step = DDIV(grand, (double)n_out);
  }
  for (int m = tid; m < n_out; m += blockDim.x) {
    const double pt = systematic ? DMUL(DADD(u0, (double)m), step)
                                 : DMUL(u64_uniform(stream_u64(id, m)), grand);
    int lo = 0, hi = n;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (pt < wpre[mid]) hi = mid;
      else lo = mid + 1;
    }
    const int i = lo < n ? lo : n - 1;
    const double before = i > 0 ? wpre[i - 1] : 0.0;
    int row = i;
    while (row > 0 && wtot[row] <= 0.0) --row;
    double local = DDIV(DSUB(pt, before), wscale[row]);
    if (!(local >= 0.0)) local = 0.0;
    const double* srow = wsub + (size_t)row * nsub;
    int s = 0;
    double c2b = 0.0, c2 = srow[0];
    while (!(local < c2) && s + 1 < nsub) {
      c2b = c2;
      ++s;
      c2 = DADD(c2, srow[s]);
    }
    const double* lrow = logw + (size_t)row * n;
    const double mrow = wm[row];
    const int j0 = s * kSub, j1 = min(j0 + kSub, n);
    double c3 = c2b;
    int j = j0;
    for (; j < j1; ++j) {
      c3 = DADD(c3, exp_w(DSUB(lrow[j], mrow)));
      if (local < c3) break;
    }
    if (j == j1) {
      j = j1 - 1;
      while (j > 0 && !(exp_w(DSUB(lrow[j], mrow)) > 0.0)) --j;
    }
    left[m] = (uint32_t)row;
    right[m] = (uint32_t)j;
  }
}

__global__ void table_lazy_kernel(const double* logw, int n, int n_out, int mh,
                                  size_t mh_steps, double bound, uint64_t seed,
                                  uint32_t level, uint64_t node, uint32_t* left,
                                  uint32_t* right, unsigned long long* evals_out,
                                  ErrFlag* err) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long evals = 0;
  if (m < n_out) {
    StreamReader s;
    s.init(stream_id(seed, level, node, DSMC_ROLE_PAIR_RESAMPLE, m + 1));
    uint32_t oi = 0, oj = 0;
    if (mh) {
      uint32_t i = (uint32_t)(m % n), j = i;
      double cur = 0.0;
      bool have = false;
      for (size_t st = 0; st < mh_steps; ++st) {
        const uint32_t pi = (uint32_t)s.index(n), pj = (uint32_t)s.index(n);
        const double lu = log(s.uniform_pos());
        if (!have) {
          cur = logw[(size_t)i * n + j];
          ++evals;
          have = true;
        }
        const double prop = logw[(size_t)pi * n + pj];
        ++evals;
        if (isnan(prop) || isnan(cur)) raise_err(err, DSMC_E_INVALID_ARGUMENT, 0, 1, kReasonNaN);
        if (lu < DSUB(prop, cur)) {
          i = pi;
          j = pj;
          cur = prop;
        }
      }
      oi = i;
      oj = j;
    } else {
      bool ok = false;
      for (uint64_t trial = 0; trial < (1u << 24); ++trial) {
        const uint32_t i = (uint32_t)s.index(n), j = (uint32_t)s.index(n);
        const double lw = logw[(size_t)i * n + j];
        ++evals;
        if (isnan(lw)) {
          raise_err(err, DSMC_E_INVALID_ARGUMENT, 0, 1, kReasonNaN);
          break;
        }
        if (DSUB(lw, bound) > 1e-9) {
          raise_err(err, DSMC_E_INVALID_ARGUMENT, 0, 1, kReasonOverBound);
          break;
        }
        if (log(s.uniform_pos()) <= DSUB(lw, bound)) {
          oi = i;
          oj = j;
          ok = true;
          break;
        }
      }
      if (!ok) raise_err(err, DSMC_E_RUNTIME, 0, 1, kReasonTrialCap);
    }
    left[m] = oi;
    right[m] = oj;
  }
  for (int o = 16; o; o >>= 1) evals += __shfl_xor_sync(~0u, evals, o);
  if ((threadIdx.x & 31) == 0 && evals) atomicAdd(evals_out, evals);
}

int dsmc_resample_table(dsmc_ctx* ctx, int resampler, const double* logw, size_t n,
                        size_t n_out, size_t mh_steps, int has_bound, double bound,
                        uint64_t seed, uint32_t level, uint64_t node, uint32_t* left,
                        uint32_t* right, double* lmw, int* has_lmw,
                        uint64_t* weight_evals, int* biased) {
  if (!ctx) return DSMC_E_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  if (n == 0) return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "pair weight source has n == 0");
  if (resampler < 0 || resampler > 3) return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "unknown resampler");
  const bool lazy = resampler >= 2;
  if (resampler == DSMC_REJECTION_LAZY && (!has_bound || !std::isfinite(bound)))
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT,
                   "rejection resampling requires a finite log_upper_bound");
  Arena& A = ctx->arena;
  void* p;
  auto s = ctx->stream;
  CU(A.get("TLOGW", n * n * 8, &p));
  double* dlw = (double*)p;
  CU(cudaMemcpyAsync(dlw, logw, n * n * 8, cudaMemcpyHostToDevice, s));
  CU(A.get("TOUT", std::max<size_t>(1, n_out) * 8, &p));
  uint32_t* dl = (uint32_t*)p;
  uint32_t* dr = dl + std::max<size_t>(1, n_out);
  CU(A.get("TMISC", 64, &p));
  ErrFlag* derr = (ErrFlag*)p;
  double* dlmw = (double*)((char*)p + 16);
  unsigned long long* devals = (unsigned long long*)((char*)p + 24);
  CU(cudaMemsetAsync(p, 0, 64, s));
  if (lazy) {
    if (!(resampler == DSMC_MH_LAZY && mh_steps == 0) && n_out > 0) {
      table_lazy_kernel<<<(n_out + 127) / 128, 128, 0, s>>>(
          dlw, (int)n, (int)n_out, resampler == DSMC_MH_LAZY, mh_steps, bound, seed, level,
          node, dl, dr, devals, derr);
      LAUNCHED(ctx);
    }
  } else {
    const int nsub = ((int)n + kSub - 1) / kSub;
    CU(A.get("TWS", n * (5 + nsub) * 8, &p));
    double* ws = (double*)p;
    table_rows_kernel<<<(n + 7) / 8, 256, 0, s>>>(dlw, (int)n, ws, derr);
    LAUNCHED(ctx);
    table_sample_kernel<<<1, 256, 0, s>>>(dlw, (int)n, (int)n_out, ws, seed, level, node,
                                          resampler == DSMC_SYSTEMATIC, dl, dr, dlmw, derr);
    LAUNCHED(ctx);
  }
  CU(cudaGetLastError());
  ErrFlag e;
  double lm = NAN;
  unsigned long long ev = 0;
  CU(cudaMemcpyAsync(&e, derr, sizeof e, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(&lm, dlmw, 8, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(&ev, devals, 8, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (e.code) {
    const char* msg = e.reason == kReasonZeroTable
                          ? "all pair weights are zero; the blocks share no support under the model"
                      : e.reason == kReasonTrialCap
                          ? "rejection resampling exceeded the trial cap; the bound is far too "
                            "loose or the weights are degenerate"
                      : e.reason == kReasonOverBound ? "pair weight exceeds its stated upper bound"
                      : e.reason == kReasonNaN ? (lazy ? "pair weight is NaN" : "reduce_max: NaN entry")
                                               : "device error";
    return set_err(ctx, e.code, msg);
  }
  if (lazy && resampler == DSMC_MH_LAZY && mh_steps == 0) {
    for (size_t m = 0; m < n_out; ++m) left[m] = right[m] = (uint32_t)(m % n);
  } else if (n_out) {
    CU(cudaMemcpy(left, dl, n_out * 4, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(right, dr, n_out * 4, cudaMemcpyDeviceToHost));
  }
  *has_lmw = lazy ? 0 : 1;
  *lmw = lazy ? NAN : lm;
  *weight_evals = lazy ? ev : (uint64_t)n * n;
  *biased = resampler == DSMC_MH_LAZY;
  return DSMC_OK;
}

// --------------------------------------------------------------- probes
__global__ void philox_kernel(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3,
                              uint64_t k0, uint64_t k1, size_t nb, uint64_t* out) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= nb) return;
  const U64x4 r = philox_k(c0 + i, c1, c2, c3, k0, k1);
  for (int q = 0; q < 4; ++q) out[4 * i + q] = r.v[q];
}
__global__ void expw_kernel(const double* x, size_t n, double* out) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = exp_w(x[i]);
}

int dsmc_philox_blocks(dsmc_ctx* ctx, const uint64_t ctr[4], const uint64_t key[2],
                       size_t nb, uint64_t* out) {
  if (!ctx) return DSMC_E_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  void* p;
  CU(ctx->arena.get("PHX", nb * 32 + 32, &p));
  philox_kernel<<<(nb + 127) / 128, 128, 0, ctx->stream>>>(ctr[0], ctr[1], ctr[2], ctr[3],
                                                           key[0], key[1], nb, (uint64_t*)p);
  LAUNCHED(ctx);
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(out, p, nb * 32, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return DSMC_OK;
}

int dsmc_exp_w(dsmc_ctx* ctx, const double* x, size_t n, double* out) {
  if (!ctx) return DSMC_E_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  void* p;
  CU(ctx->arena.get("EXPW", 2 * n * 8 + 16, &p));
  double* dx = (double*)p;
  double* dy = dx + n;
  CU(cudaMemcpyAsync(dx, x, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  expw_kernel<<<(n + 255) / 256, 256, 0, ctx->stream>>>(dx, n, dy);
  LAUNCHED(ctx);
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(out, dy, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return DSMC_OK;
}

// ----------------------------------------------------------- conditional
int dsmc_conditional_sweep(dsmc_ctx* ctx, const dsmc_model_desc* models, int B,
                           const double* refs, const uint64_t* seeds,
                           const dsmc_cond_opts* opts, uint32_t sweep,
                           double* out_paths, uint8_t* changed, double* lnc_out,
                           uint64_t* weight_evals) {
  if (!ctx || !models || B < 1 || !refs || !seeds || !opts || !out_paths)
    return DSMC_E_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  dsmc_model_handle* h = nullptr;
  int rc = make_handle(ctx, models, B, &h);
  if (rc) return rc;
  std::unique_ptr<dsmc_model_handle, void (*)(dsmc_model_handle*)> hold(h, free_handle);
  const int K = h->K, d = h->d, T = K - 1;
  const size_t N = opts->n_particles;
  Arena& A = ctx->arena;
  void* p;
  auto s = ctx->stream;
  CU(A.get("CSTAR", (size_t)B * K * d * 8, &p));
  double* dstar = (double*)p;
  CU(cudaMemcpyAsync(dstar, refs, (size_t)B * K * d * 8, cudaMemcpyHostToDevice, s));
  CU(A.get("CSEED", (size_t)B * 8, &p));
  uint64_t* dseeds = (uint64_t*)p;
  CU(cudaMemcpyAsync(dseeds, seeds, (size_t)B * 8, cudaMemcpyHostToDevice, s));
  CU(A.get("COUT", (size_t)B * K * d * 8, &p));
  double* dout = (double*)p;
  CU(A.get("CCHG", (size_t)B * K, &p));
  uint8_t* dchg = (uint8_t*)p;
  RunOpts o;
  o.precision = opts->precision;
  o.resampler = opts->resampler;
  o.N = N;
  o.conditional = 1;
  o.sweep = sweep;
  o.inj_x = opts->inject_states;
  o.star = dstar;
  o.seeds = dseeds;
  o.star_out = dout;
  o.changed = dchg;
  RunResult res;
  rc = run_tree(ctx, h, o, &res);
  if (rc) return rc;
  rc = check_device_error(ctx, res, K);
  if (rc) return rc;
  CU(cudaMemcpyAsync(out_paths, dout, (size_t)B * K * d * 8, cudaMemcpyDeviceToHost, s));
  if (changed) CU(cudaMemcpyAsync(changed, dchg, (size_t)B * K, cudaMemcpyDeviceToHost, s));
  std::vector<double> lnc(B);
  std::vector<unsigned long long> ev(B);
  for (int c = 0; c < B; ++c)
    CU(cudaMemcpyAsync(&lnc[c], res.root_lnc + (size_t)c * res.lnc_stride, 8,
                       cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(ev.data(), res.evals, (size_t)B * 8, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  const bool lazy = opts->resampler == DSMC_REJECTION_LAZY;
  for (int c = 0; c < B; ++c) {
    if (lnc_out) lnc_out[c] = lnc[c];
    if (weight_evals) weight_evals[c] = lazy ? ev[c] + (uint64_t)T : (uint64_t)T * (N * N + 1);
  }
  return DSMC_OK;
}

}  // extern "C"

// ------------------------------------------------------------ SV pGibbs
namespace {

// gamma_draw (pgibbs.cpp:80-102), Marsaglia-Tsang with the shape<1 boost.
__device__ double gamma_draw_dev(double shape, double rate, StreamReader& s) {
  double boost = 1.0;
  if (shape < 1.0) {
    boost = pow(s.uniform_pos(), 1.0 / shape);
    shape += 1.0;
  }
  const double d = shape - 1.0 / 3.0;
  const double c = 1.0 / sqrt(9.0 * d);
  for (int guard = 0; guard < 100000; ++guard) {
    double x, v;
    do {
      x = s.normal();
      v = 1.0 + c * x;
    } while (v <= 0.0);
    v = v * v * v;
    const double u = s.uniform_pos();
    if (log(u) < 0.5 * x * x + d - d * v + d * log(v)) return boost * d * v / rate;
  }
  return CUDART_NAN;
}

__device__ double sv_loglik(const double* x, int T, double mu, double phi, double s2) {
  const double v0 = s2 / (1.0 - phi * phi);
  double ll = dlog_normal_pdf(x[0], mu, v0);
  for (int t = 1; t <= T; ++t) ll += dlog_normal_pdf(x[t], mu + phi * (x[t - 1] - mu), s2);
  return ll;
}

// SV ParamKernel (oracle or_sv_param_update): sigma2 | rest
// (inverse gamma), mu | rest (normal), random-walk Metropolis on phi. One
// warp per chain: the O(T) path sums are lane-strided + a warp reduction
// (the oracle sums sequentially: values agree to ~1e-15 relative); lane 0
// draws from the chain's stream in the oracle's order.
__device__ inline double warp_sum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(~0u, v, o);
  return v;
}
__global__ void sv_param_kernel(DevModel* models, double* theta, const double* stars,
                                const uint64_t* seeds, dsmc_sv_prior pr, int T,
                                uint32_t sweep, int B, unsigned long long* acc_phi) {
  const int ch = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (ch >= B) return;
  const double* x = stars + (size_t)ch * (T + 1);
  double mu = theta[3 * ch], phi = theta[3 * ch + 1], s2 = theta[3 * ch + 2];
  double ss = 0.0, acc = 0.0;
  for (int t = 1 + lane; t <= T; t += 32) {
    const double e = x[t] - mu - phi * (x[t - 1] - mu);
    ss += e * e;
    acc += x[t] - phi * x[t - 1];
  }
  ss = warp_sum(ss) + (1.0 - phi * phi) * (x[0] - mu) * (x[0] - mu);
  acc = warp_sum(acc);
  double prop = 0.0, lu = 0.0;
  StreamReader s;
  if (lane == 0) {
    s.init(stream_id(seeds[ch], 0, sweep, DSMC_ROLE_GIBBS_PARAM, 0));
    const double prec = gamma_draw_dev(pr.s2_shape + 0.5 * (double)(T + 1), pr.s2_rate + 0.5 * ss, s);
    s2 = 1.0 / prec;
    const double p = 1.0 / pr.mu_var + (1.0 - phi * phi) / s2 +
                     (double)T * (1.0 - phi) * (1.0 - phi) / s2;
    const double h = pr.mu_mean / pr.mu_var + (1.0 - phi * phi) * x[0] / s2 + (1.0 - phi) * acc / s2;
    mu = h / p + sqrt(1.0 / p) * s.normal();
    prop = phi + pr.phi_step * s.normal();
    lu = log(s.uniform_pos());
  }
  mu = __shfl_sync(~0u, mu, 0);
  s2 = __shfl_sync(~0u, s2, 0);
  prop = __shfl_sync(~0u, prop, 0);
  if (fabs(prop) < 1.0) {  // sv_loglik(prop) - sv_loglik(phi), lane-strided
    double d = 0.0;
    for (int t = 1 + lane; t <= T; t += 32)
      d += dlog_normal_pdf(x[t], mu + prop * (x[t - 1] - mu), s2) -
           dlog_normal_pdf(x[t], mu + phi * (x[t - 1] - mu), s2);
    d = warp_sum(d);
    if (lane == 0) {
      const double dl = d + dlog_normal_pdf(x[0], mu, s2 / (1.0 - prop * prop)) -
                        dlog_normal_pdf(x[0], mu, s2 / (1.0 - phi * phi));
      if (lu < dl) {
        phi = prop;
        atomicAdd(acc_phi, 1ull);
      }
    }
  }
  if (lane == 0) {
    theta[3 * ch] = mu;
    theta[3 * ch + 1] = phi;
    theta[3 * ch + 2] = s2;
    models[ch].sv_mu = mu;
    models[ch].sv_phi = phi;
    models[ch].sv_s2 = s2;
  }
}

}  // namespace

extern "C" int dsmc_sv_pgibbs_sweep(dsmc_ctx* ctx, int B, int T, const double* ys,
                                    const dsmc_sv_prior* prior, double* theta,
                                    double* stars, const uint64_t* seeds, size_t N,
                                    int resampler, uint32_t sweep, uint8_t* changed,
                                    uint64_t* accepted_phi) {
  if (!ctx || B < 1 || T < 0 || !ys || !prior || !theta || !stars || !seeds)
    return DSMC_E_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  std::vector<dsmc_model_desc> descs(B);
  for (int c = 0; c < B; ++c) {
    dsmc_model_desc& m = descs[c];
    std::memset(&m, 0, sizeof m);
    m.kind = DSMC_MODEL_SV;
    m.state_dim = 1;
    m.obs_dim = 1;
    m.horizon = T;
    m.y = ys;
    m.sv_mu = theta[3 * c];
    m.sv_phi = theta[3 * c + 1];
    m.sv_sigma2 = theta[3 * c + 2];
  }
  dsmc_model_handle* h = nullptr;
  int rc = make_handle(ctx, descs.data(), B, &h);  // prep runs again below
  if (rc) return rc;
  std::unique_ptr<dsmc_model_handle, void (*)(dsmc_model_handle*)> hold(h, free_handle);
  const int K = T + 1;
  Arena& A = ctx->arena;
  void* p;
  auto s = ctx->stream;
  CU(A.get("GSTAR", (size_t)B * K * 8, &p));
  double* dstar = (double*)p;
  CU(cudaMemcpyAsync(dstar, stars, (size_t)B * K * 8, cudaMemcpyHostToDevice, s));
  CU(A.get("GTHETA", (size_t)B * 3 * 8, &p));
  double* dtheta = (double*)p;
  CU(cudaMemcpyAsync(dtheta, theta, (size_t)B * 3 * 8, cudaMemcpyHostToDevice, s));
  CU(A.get("GSEED", (size_t)B * 8, &p));
  uint64_t* dseeds = (uint64_t*)p;
  CU(cudaMemcpyAsync(dseeds, seeds, (size_t)B * 8, cudaMemcpyHostToDevice, s));
  CU(A.get("GACC", 8, &p));
  unsigned long long* dacc = (unsigned long long*)p;
  CU(cudaMemsetAsync(dacc, 0, 8, s));
  CU(A.get("GOUT", (size_t)B * K * 8, &p));
  double* dout = (double*)p;
  CU(A.get("GCHG", (size_t)B * K, &p));
  uint8_t* dchg = (uint8_t*)p;
  // parameter kernel (pgibbs_sweep: param_kernel then model rebuild)
  sv_param_kernel<<<(B + 7) / 8, 256, 0, s>>>(h->models_dev, dtheta, dstar, dseeds, *prior, T,
                                               sweep, B, dacc);
  LAUNCHED(ctx);
  std::vector<int> ones(B, 3);
  CU(cudaMemcpyAsync(h->bounded, ones.data(), sizeof(int) * B, cudaMemcpyHostToDevice, s));
  prep_kernel<<<dim3((K + 127) / 128, B), 128, 0, s>>>(h->models_dev, h->tc, K, h->bounded);
  LAUNCHED(ctx);
  RunOpts o;
  o.precision = DSMC_FP32;
  o.resampler = resampler;
  o.N = N;
  o.conditional = 1;
  o.sweep = sweep;
  o.star = dstar;
  o.seeds = dseeds;
  o.star_out = dout;
  o.changed = dchg;
  RunResult res;
  rc = run_tree(ctx, h, o, &res);
  if (rc) return rc;
  rc = check_device_error(ctx, res, K);
  if (rc) return rc;
  CU(cudaMemcpyAsync(stars, dout, (size_t)B * K * 8, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(theta, dtheta, (size_t)B * 3 * 8, cudaMemcpyDeviceToHost, s));
  if (changed) CU(cudaMemcpyAsync(changed, dchg, (size_t)B * K, cudaMemcpyDeviceToHost, s));
  unsigned long long acc = 0;
  CU(cudaMemcpyAsync(&acc, dacc, 8, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (accepted_phi) *accepted_phi = acc;
  return DSMC_OK;
}

// ------------------------------------------------------ time-sharded API
namespace {

WindowState& window_state_impl(dsmc_ctx* ctx) {
  if (!ctx->window) ctx->window = new WindowState();
  return *static_cast<WindowState*>(ctx->window);
}

__global__ void boundary_kernel(const float4* X, const float* COL, const uint32_t* map,
                                int N, float4* out_x, float* out_col) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= N) return;
  const uint32_t p = map ? map[q] : (uint32_t)q;
  out_x[q] = X[p];
  if (out_col) out_col[q] = COL[p];
}

__global__ void remap_kernel(uint32_t* map, const uint32_t* idx, uint32_t* tmp, int N) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < N) tmp[q] = map[idx[q]];
}

}  // namespace

namespace {
WindowState& window_state(dsmc_ctx* ctx) { return window_state_impl(ctx); }
}  // namespace

extern "C" {

int dsmc_window_run(dsmc_ctx* ctx, const dsmc_model_handle* hc, const dsmc_window_opts* wo) {
  if (!ctx || !hc || !wo) return DSMC_E_INVALID_ARGUMENT;
  auto* h = const_cast<dsmc_model_handle*>(hc);
  const int len = wo->len;
  if (len < 2 || (len & (len - 1)) || wo->t0 % len || wo->t0 + len > h->K)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT,
                   "window: len must be a power of two >= 2 dividing t0, inside the horizon");
  if (wo->t0 < h->t_lo || wo->t0 + len > h->t_hi)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "window: outside the uploaded model window");
  RunOpts o;
  o.precision = DSMC_FP32;
  o.resampler = wo->resampler;
  o.mh_steps = wo->mh_steps;
  o.N = wo->n_particles;
  o.t0 = wo->t0;
  o.len = len;
  o.compose = false;
  o.timing = true;  // per-kernel-class device times (dsmc_last_timings)
  ctx->time_kernels = true;
  ctx->kev_used = 0;
  void* p;
  CU(ctx->arena.get("SEEDS", sizeof(uint64_t), &p));
  CU(cudaMemcpyAsync(p, &wo->seed, sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
  o.seeds = (const uint64_t*)p;
  RunResult res;
  int rc = run_tree(ctx, h, o, &res);
  if (rc) return rc;
  ctx->last_err = res.err;  // checked at the next host sync (boundary log Z, dsmc_sync)
  ctx->last_err_K = h->K;
  return DSMC_OK;
}

int dsmc_window_boundary(dsmc_ctx* ctx, int side, void* d_x, float* d_col,
                         double* d_root_lnc) {
  if (!ctx) return DSMC_E_INVALID_ARGUMENT;
  WindowState& st = window_state(ctx);
  if (!st.valid) return set_err(ctx, DSMC_E_LOGIC, "no window run on this context");
  const Bufs& b = st.b;
  const int N = b.N;
  const int t = side == 0 ? 0 : b.K - 1;
  const uint32_t* map = st.maps[2 * st.cur + (side == 0 ? 0 : 1)];
  if (d_x) {
    boundary_kernel<<<(N + 255) / 256, 256, 0, ctx->stream>>>(
        b.X32 + (size_t)t * N, b.COL + (size_t)t * N, map, N, (float4*)d_x,
        side == 0 ? d_col : nullptr);
    LAUNCHED(ctx);
    CU(cudaGetLastError());
  }
  // the window root's log Z stays on the device (stream-ordered, no sync)
  if (d_root_lnc)
    CU(cudaMemcpyAsync(d_root_lnc, st.blnc[st.cur], 8, cudaMemcpyDeviceToDevice, ctx->stream));
  return DSMC_OK;
}

int dsmc_window_remap(dsmc_ctx* ctx, int side, const uint32_t* d_idx) {
  if (!ctx || !d_idx) return DSMC_E_INVALID_ARGUMENT;
  WindowState& st = window_state(ctx);
  if (!st.valid) return set_err(ctx, DSMC_E_LOGIC, "no window run on this context");
  const int N = st.b.N;
  uint32_t* map = st.maps[2 * st.cur + (side == 0 ? 0 : 1)];
  void* p;
  CU(ctx->arena.get("RTMP", (size_t)N * 4, &p));
  remap_kernel<<<(N + 255) / 256, 256, 0, ctx->stream>>>(map, d_idx, (uint32_t*)p, N);
  LAUNCHED(ctx);
  CU(cudaMemcpyAsync(map, p, (size_t)N * 4, cudaMemcpyDeviceToDevice, ctx->stream));
  return DSMC_OK;
}

int dsmc_window_finish(dsmc_ctx* ctx, const uint32_t* d_root_map, double* d_mean, double* d_cov) {
  if (!ctx) return DSMC_E_INVALID_ARGUMENT;
  WindowState& st = window_state(ctx);
  if (!st.valid) return set_err(ctx, DSMC_E_LOGIC, "no window run on this context");
  const Bufs& b = st.b;
  const int K = b.K, N = b.N, d = b.d, B = b.B;
  std::vector<int> nbs{K};
  while (nbs.back() > 1) nbs.push_back((nbs.back() + 1) / 2);
  std::vector<size_t> cursors(nbs.size() + 1, 0);
  for (size_t l = 1; l + 1 <= nbs.size() - 1; ++l) cursors[l + 1] = cursors[l] + nbs[l - 1] / 2;
  uint32_t* Mb[2] = {st.maps[0], st.maps[2]};
  int mcur = 0;
  bool root = true;
  for (int l = st.levels; l >= 2; --l) {
    td_kernel<<<dim3(nbs[l], (N + 255) / 256, B), 256, 0, ctx->stream>>>(
        b, l, cursors[l], nbs[l], nbs[l - 1], Mb[mcur], Mb[1 - mcur], root ? 1 : 0, d_root_map);
    LAUNCHED(ctx);
    root = false;
    mcur = 1 - mcur;
  }
  const uint32_t* M1 = Mb[mcur];
  const int r1 = root ? 1 : 0;
  switch (d) {
    case 1: gather32_kernel<1><<<dim3((K + 7) / 8, B), 256, 0, ctx->stream>>>(b, M1, r1, nullptr, d_mean, d_cov, d_root_map); break;
    case 2: gather32_kernel<2><<<dim3((K + 7) / 8, B), 256, 0, ctx->stream>>>(b, M1, r1, nullptr, d_mean, d_cov, d_root_map); break;
    case 3: gather32_kernel<3><<<dim3((K + 7) / 8, B), 256, 0, ctx->stream>>>(b, M1, r1, nullptr, d_mean, d_cov, d_root_map); break;
    default: gather32_kernel<4><<<dim3((K + 7) / 8, B), 256, 0, ctx->stream>>>(b, M1, r1, nullptr, d_mean, d_cov, d_root_map); break;
  }
  LAUNCHED(ctx);
  CU(cudaGetLastError());
  st.valid = false;  // the maps were consumed by the composition
  return DSMC_OK;
}

int dsmc_cross_combine(dsmc_ctx* ctx, const dsmc_model_handle* hc, const dsmc_window_opts* wo,
                       int cut, int level, long long node, const void* d_xl, const void* d_xr,
                       const float* d_colr, const double* d_lnc_l, const double* d_lnc_r,
                       uint32_t* d_l, uint32_t* d_r, double* d_lnc_out) {
  if (!ctx || !hc || !wo || !d_xl || !d_xr || !d_colr || !d_l || !d_r || !d_lnc_l || !d_lnc_r)
    return DSMC_E_INVALID_ARGUMENT;
  auto* h = const_cast<dsmc_model_handle*>(hc);
  if (cut < 1 || cut >= h->K) return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "cross_combine: bad cut");
  if (cut < h->t_lo || cut >= h->t_hi)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "cross_combine: cut outside the uploaded window");
  if (wo->resampler < 0 || wo->resampler > 3)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "unknown resampler");
  const bool lazy = wo->resampler >= DSMC_MH_LAZY;
  const int N = (int)wo->n_particles, d = h->d;
  Arena& A = ctx->arena;
  auto s = ctx->stream;
  void* p;
  // a two-leaf window [cut-1, cut] whose "leaves" are the two boundary slabs
  // (both combined blocks: uniform weights)
  Bufs b{};
  b.K = 2;
  b.T = 1;
  b.N = N;
  b.d = d;
  b.B = 1;
  b.cap = 1;
  b.t0 = cut - 1;
  b.Kt = h->K;
  b.models = h->models_dev;
  b.tc = h->tc;
  b.bounded = h->bounded;
  CU(A.get("CX32", 2 * (size_t)N * sizeof(float4), &p));
  b.X32 = (float4*)p;
  CU(cudaMemcpyAsync(b.X32, d_xl, (size_t)N * sizeof(float4), cudaMemcpyDeviceToDevice, s));
  CU(cudaMemcpyAsync(b.X32 + N, d_xr, (size_t)N * sizeof(float4), cudaMemcpyDeviceToDevice, s));
  CU(A.get("CCOL", 2 * (size_t)N * sizeof(float), &p));
  b.COL = (float*)p;
  CU(cudaMemcpyAsync(b.COL + N, d_colr, (size_t)N * sizeof(float), cudaMemcpyDeviceToDevice, s));
  CU(A.get("CMISC", 256, &p));
  double* lnc = (double*)p;  // [0..1] block log Z, [2] new block log Z
  uint8_t* uni = (uint8_t*)p + 64;
  uint64_t* seed = (uint64_t*)((char*)p + 128);
  unsigned long long* evals = (unsigned long long*)((char*)p + 136);
  CU(cudaMemcpyAsync(lnc, d_lnc_l, 8, cudaMemcpyDeviceToDevice, s));
  CU(cudaMemcpyAsync(lnc + 1, d_lnc_r, 8, cudaMemcpyDeviceToDevice, s));
  CU(cudaMemsetAsync(uni, 1, 2, s));
  CU(cudaMemsetAsync(evals, 0, 8, s));
  set_seed_kernel<<<1, 1, 0, s>>>(seed, wo->seed);
  LAUNCHED(ctx);
  // device errors accumulate in the window run's record (first error wins)
  // and surface at the next host synchronisation (dsmc_sync)
  CU(A.get("ERR", sizeof(ErrFlag), &p));
  b.err = (ErrFlag*)p;
  ctx->last_err = b.err;
  ctx->last_err_K = h->K;
  b.LNC = lnc;
  b.UNI = uni;
  b.LWMAX = lnc;  // unused (uniform sides)
  b.seeds = seed;
  b.evals = evals;
  CU(A.get("CPL", (size_t)N * 4, &p));
  b.PL = (uint32_t*)p;
  CU(A.get("CPR", (size_t)N * 4, &p));
  b.PR = (uint32_t*)p;
  CU(A.get("CLMW", 8, &p));
  b.LMW = (double*)p;
  CU(A.get("CMAPS", 2 * (size_t)N * 4, &p));
  LevelArgs la{};
  la.level = 1;
  la.np = 1;
  la.nb_prev = 2;
  la.k0 = 0;
  la.cursor = 0;
  la.first_next = (uint32_t*)p;
  la.last_next = (uint32_t*)p + N;
  la.blnc_next = lnc + 2;
  la.n_out = N;
  la.key_level = level;
  la.node_off = node;
  int rc = DSMC_OK;
  if (lazy) {  // MH / rejection lazy cross combine (resampling.cpp:233-324)
    const int mh = wo->resampler == DSMC_MH_LAZY;
    const dim3 grid((N + 127) / 128, 1, 1);
    switch (d) {
      case 1: launch_lazy32<1>(grid, s, b, la, mh, wo->mh_steps); break;
      case 2: launch_lazy32<2>(grid, s, b, la, mh, wo->mh_steps); break;
      case 3: launch_lazy32<3>(grid, s, b, la, mh, wo->mh_steps); break;
      default: launch_lazy32<4>(grid, s, b, la, mh, wo->mh_steps); break;
    }
    LAUNCHED(ctx);
    lazy_finish_kernel<<<dim3(1, 1, 1), 256, 0, s>>>(b, la);
    LAUNCHED(ctx);
  } else {
    const size_t ws_comb = ((size_t)N * ((N + kSub - 1) / kSub) + 1) / 2;
    CU(A.get("CWS", ws_comb * 8, &p));
    la.ws = (double*)p;
    la.ws_comb = ws_comb;
    const int sys = wo->resampler == DSMC_SYSTEMATIC;
    const bool keep = ctx->time_kernels;
    ctx->time_kernels = false;
    rc = d == 1 ? launch_c32<1>(ctx, b, la, 1, sys)
       : d == 2 ? launch_c32<2>(ctx, b, la, 1, sys)
       : d == 3 ? launch_c32<3>(ctx, b, la, 1, sys)
                : launch_c32<4>(ctx, b, la, 1, sys);
    ctx->time_kernels = keep;
  }
  if (rc) return rc;
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(d_l, b.PL, (size_t)N * 4, cudaMemcpyDeviceToDevice, s));
  CU(cudaMemcpyAsync(d_r, b.PR, (size_t)N * 4, cudaMemcpyDeviceToDevice, s));
  if (d_lnc_out) CU(cudaMemcpyAsync(d_lnc_out, lnc + 2, 8, cudaMemcpyDeviceToDevice, s));
  return DSMC_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ FFBS
// Sequential comparator: particle filter + backward sampling on the device
// (run_particle_filter / ffbs_sample, baselines.cpp:36-160), FP32.
extern "C" int dsmc_ffbs_smooth(dsmc_ctx* ctx, const dsmc_model_desc* model,
                                const dsmc_ffbs_opts* opts, double* mean, double* cov,
                                double* paths, double* log_likelihood) {
  if (!ctx || !model || !opts) return DSMC_E_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  const int N = (int)opts->n_particles, M = (int)opts->n_draws;
  if (N < 1) return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "particle filter: need n >= 1");
  if (M < 1) return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "ffbs: need n_draws >= 1");
  if (model->state_dim > 4 || force_wide())
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "ffbs: state_dim > 4 is not supported");
  if (opts->resampler != DSMC_MULTINOMIAL && opts->resampler != DSMC_SYSTEMATIC)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT,
                   "particle filter: dense resampling only (multinomial or systematic)");
  dsmc_model_handle* h = nullptr;
  int rc = make_handle(ctx, model, 1, &h);
  if (rc) return rc;
  std::unique_ptr<dsmc_model_handle, void (*)(dsmc_model_handle*)> hold(h, free_handle);
  const int K = h->K, d = h->d;
  Arena& A = ctx->arena;
  void* p;
  Bufs b{};
  b.K = K;
  b.T = K - 1;
  b.N = N;
  b.d = d;
  b.B = 1;
  b.cap = 1;
  b.Kt = K;
  b.models = h->models_dev;
  b.tc = h->tc;
  b.bounded = h->bounded;
  b.leaf_role = DSMC_ROLE_FILTER_STEP;
  const size_t KN = (size_t)K * N;
  CU(A.get("X32", KN * sizeof(float4), &p));
  b.X32 = (float4*)p;
  CU(A.get("COL", KN * sizeof(float), &p));
  b.COL = (float*)p;
  CU(A.get("LW32", (size_t)N * sizeof(float), &p));
  b.LW32 = (float*)p;
  CU(A.get("LNC", (size_t)K * sizeof(double), &p));
  b.LNC = (double*)p;
  CU(A.get("LWMAX", (size_t)K * sizeof(double), &p));
  b.LWMAX = (double*)p;
  CU(A.get("UNI", (size_t)K, &p));
  b.UNI = (uint8_t*)p;
  CU(A.get("ERR", sizeof(ErrFlag), &p));
  b.err = (ErrFlag*)p;
  CU(A.get("SEEDS", sizeof(uint64_t), &p));
  b.seeds = (const uint64_t*)p;
  set_seed_kernel<<<1, 1, 0, ctx->stream>>>((uint64_t*)p, opts->seed);
  LAUNCHED(ctx);
  CU(cudaMemsetAsync(b.err, 0, sizeof(ErrFlag), ctx->stream));
  float* LW;
  uint32_t *ANC, *P;
  double *dll, *dmean, *dcov, *dpaths = nullptr;
  CU(A.get("FF_LW", KN * sizeof(float), &p));
  LW = (float*)p;
  CU(A.get("FF_ANC", (size_t)std::max(K - 1, 1) * N * sizeof(uint32_t), &p));
  ANC = (uint32_t*)p;
  CU(A.get("FF_P", (size_t)M * K * sizeof(uint32_t), &p));
  P = (uint32_t*)p;
  CU(A.get("FF_LL", sizeof(double), &p));
  dll = (double*)p;
  CU(A.get("OMEAN", (size_t)K * d * sizeof(double), &p));
  dmean = (double*)p;
  CU(A.get("OCOV", (size_t)K * d * d * sizeof(double), &p));
  dcov = (double*)p;
  if (paths) {
    CU(A.get("OPATH", (size_t)M * K * d * sizeof(double), &p));
    dpaths = (double*)p;
  }
  CU(A.get("RAW0", (size_t)N * sizeof(double), &p));
  double* raw0 = (double*)p;
  const int lt = std::min(256, (N + 31) / 32 * 32);
  const int pt = std::min(512, (N + 31) / 32 * 32);
  const size_t smf = sizeof(double) * N;
  const size_t smb = sizeof(float4) * N + sizeof(float) * ((N + 1) & ~1) + sizeof(double) * N;
  if (smb > (size_t)ctx->smem_optin - 1024 || smf > (size_t)ctx->smem_optin - 1024)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "ffbs: N too large");
#define FFBS_RUN(DD)                                                                          \
  do {                                                                                        \
    leaf32_kernel<DD><<<dim3(K, 1), lt, 0, ctx->stream>>>(b, raw0);                           \
    LAUNCHED(ctx);                                                                            \
    leafnorm32_kernel<<<1, 32, 0, ctx->stream>>>(b, raw0);                                    \
    LAUNCHED(ctx);                                                                            \
    pf_forward_kernel<DD><<<1, pt, smf, ctx->stream>>>(b, LW, ANC,                            \
                                                       opts->resampler == DSMC_SYSTEMATIC, dll); \
    LAUNCHED(ctx);                                                                            \
    ffbs_backward_kernel<DD><<<(M + 7) / 8, 256, smb, ctx->stream>>>(b, LW, M, P);            \
    LAUNCHED(ctx);                                                                            \
    ffbs_moments_kernel<DD><<<(K + 7) / 8, 256, 0, ctx->stream>>>(b, P, M, dmean, dcov,        \
                                                                   dpaths);                   \
    LAUNCHED(ctx);                                                                            \
  } while (0)
  switch (d) {
    case 1: FFBS_RUN(1); break;
    case 2: FFBS_RUN(2); break;
    case 3: FFBS_RUN(3); break;
    default: FFBS_RUN(4); break;
  }
#undef FFBS_RUN
  CU(cudaGetLastError());
  ErrFlag e;
  CU(cudaMemcpyAsync(&e, b.err, sizeof e, cudaMemcpyDeviceToHost, ctx->stream));
  double ll = 0.0;
  CU(cudaMemcpyAsync(&ll, dll, sizeof ll, cudaMemcpyDeviceToHost, ctx->stream));
  if (mean) CU(cudaMemcpyAsync(mean, dmean, (size_t)K * d * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (cov) CU(cudaMemcpyAsync(cov, dcov, (size_t)K * d * d * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (paths) CU(cudaMemcpyAsync(paths, dpaths, (size_t)M * K * d * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  if (e.code) return set_err(ctx, e.code, e.reason == kReasonLeafZero
                                             ? "particle filter: every weight is zero at a time step"
                                             : "ffbs: every backward weight is zero at a time step");
  if (log_likelihood) *log_likelihood = ll;
  return DSMC_OK;
}

// The reference's piecewise entry points (make_leaf, resample_pairs over a
// block pair or a caller-evaluated source, index resampling).
#include "pieces.cuh"

// ------------------------------------------------ device Kalman / RTS
namespace {

template <class Op>
int scan_chunked(dsmc_ctx* ctx, typename Op::E* el, int n, int depth) {
  auto s = ctx->stream;
  if (n <= kScanChunk) {
    scan_chunk_apply<Op><<<1, 1, 0, s>>>(el, n, nullptr);
    LAUNCHED(ctx);
    return DSMC_OK;
  }
  const int nc = (n + kScanChunk - 1) / kScanChunk;
  void* p;
  const std::string name = std::string(sizeof(typename Op::E) == sizeof(FiltElem<4>) ? "KFA" : "KSA") +
                           std::to_string(sizeof(typename Op::E)) + "_" + std::to_string(depth);
  CU(ctx->arena.get(name.c_str(), (size_t)nc * sizeof(typename Op::E), &p));
  auto* agg = static_cast<typename Op::E*>(p);
  scan_chunk_total<Op><<<(nc + 63) / 64, 64, 0, s>>>(el, n, agg);
  LAUNCHED(ctx);
  int rc = scan_chunked<Op>(ctx, agg, nc, depth + 1);
  if (rc) return rc;
  scan_chunk_apply<Op><<<(nc + 63) / 64, 64, 0, s>>>(el, n, agg);
  LAUNCHED(ctx);
  return DSMC_OK;
}

__global__ void sum_kernel(const double* x, int n, double* out) {
  __shared__ double sh[1024];
  double v = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) v += x[i];
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

template <int D, int DY>
int kalman_device(dsmc_ctx* ctx, const KfModel& m, int K, double* d_mean, double* d_cov,
                  double* d_ll, int* d_bad) {
  auto s = ctx->stream;
  void* p;
  CU(ctx->arena.get("KF_FILT", (size_t)K * sizeof(FiltElem<D>), &p));
  auto* fe = static_cast<FiltElem<D>*>(p);
  CU(ctx->arena.get("KF_SMOOTH", (size_t)K * sizeof(SmoothElem<D>), &p));
  auto* se = static_cast<SmoothElem<D>*>(p);
  CU(ctx->arena.get("KF_LLT", (size_t)K * sizeof(double), &p));
  auto* llt = static_cast<double*>(p);
  const int nb = (K + 127) / 128;
  kf_filter_elems<D, DY><<<nb, 128, 0, s>>>(m, K, fe, d_bad);
  LAUNCHED(ctx);
  int rc = scan_chunked<FiltOp<D>>(ctx, fe, K, 0);
  if (rc) return rc;
  kf_smooth_elems<D, DY><<<nb, 128, 0, s>>>(m, K, fe, se, llt, d_bad);
  LAUNCHED(ctx);
  rc = scan_chunked<SmoothOp<D>>(ctx, se, K, 0);
  if (rc) return rc;
  kf_outputs<D><<<nb, 128, 0, s>>>(K, se, d_mean, d_cov);
  LAUNCHED(ctx);
  sum_kernel<<<1, 1024, 0, s>>>(llt, K, d_ll);
  LAUNCHED(ctx);
  return cudaGetLastError() == cudaSuccess ? DSMC_OK
                                           : set_err(ctx, DSMC_E_CUDA, "kalman scan launch failed");
}

template <int D>
int kalman_device_dy(dsmc_ctx* ctx, int dy, const KfModel& m, int K, double* a, double* b,
                     double* c, int* bad) {
  switch (dy) {
    case 1: return kalman_device<D, 1>(ctx, m, K, a, b, c, bad);
    case 2: return kalman_device<D, 2>(ctx, m, K, a, b, c, bad);
    case 3: return kalman_device<D, 3>(ctx, m, K, a, b, c, bad);
    default: return kalman_device<D, 4>(ctx, m, K, a, b, c, bad);
  }
}

}  // namespace

extern "C" int dsmc_kalman_smooth_device(dsmc_ctx* ctx, const dsmc_model_desc* m,
                                         double* smooth_mean, double* smooth_cov,
                                         double* log_likelihood) {
  if (!ctx || !m || !smooth_mean || !smooth_cov) return DSMC_E_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  if (m->kind != DSMC_MODEL_LGSSM)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "kalman_smooth: LGSSM descriptor required");
  const int d = m->state_dim, dy = m->obs_dim, K = m->horizon + 1;
  if (d < 1 || d > 4 || dy < 1 || dy > 4 || m->horizon < 0)
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT, "kalman_smooth: dims must be 1..4");
  if (!m->m0 || !m->P0 || !m->H || !m->R || !m->y || (K > 1 && (!m->F || !m->b || !m->Q)))
    return set_err(ctx, DSMC_E_INVALID_ARGUMENT,
                   "kalman_smooth: initial, transition and observation arrays are required");
  Arena& A = ctx->arena;
  auto s = ctx->stream;
  void* p;
  // model arrays (per-time with stride, 0 = one matrix for all times)
  auto up = [&](const char* name, const void* src, size_t bytes, const void** dst) -> int {
    if (!src || !bytes) {
      *dst = nullptr;
      return DSMC_OK;
    }
    CU(A.get(name, bytes, &p));
    CU(cudaMemcpyAsync(p, src, bytes, cudaMemcpyHostToDevice, s));
    *dst = p;
    return DSMC_OK;
  };
  auto span = [&](int64_t st, size_t per) { return (st ? (size_t)K * st : per) * sizeof(double); };
  KfModel km{};
  int rc = 0;
  const void* q;
  rc |= up("KF_F", m->F, K > 1 ? span(m->F_stride, (size_t)d * d) : 0, &q); km.F = (const double*)q;
  rc |= up("KF_b", m->b, K > 1 ? span(m->b_stride, (size_t)d) : 0, &q); km.b = (const double*)q;
  rc |= up("KF_Q", m->Q, K > 1 ? span(m->Q_stride, (size_t)d * d) : 0, &q); km.Q = (const double*)q;
  rc |= up("KF_H", m->H, span(m->H_stride, (size_t)dy * d), &q); km.H = (const double*)q;
  rc |= up("KF_R", m->R, span(m->R_stride, (size_t)dy * dy), &q); km.R = (const double*)q;
  rc |= up("KF_y", m->y, (size_t)K * dy * sizeof(double), &q); km.y = (const double*)q;
  rc |= up("KF_m0", m->m0, (size_t)d * sizeof(double), &q); km.m0 = (const double*)q;
  rc |= up("KF_P0", m->P0, (size_t)d * d * sizeof(double), &q); km.P0 = (const double*)q;
  rc |= up("KF_obs", m->has_obs, m->has_obs ? (size_t)K : 0, &q); km.has_obs = (const uint8_t*)q;
  if (rc) return rc;
  km.Fs = m->F_stride;
  km.bs = m->b_stride;
  km.Qs = m->Q_stride;
  km.Hs = m->H_stride;
  km.Rs = m->R_stride;
  CU(A.get("KF_OUT", (size_t)K * d * (d + 1) * sizeof(double) + 16, &p));
  double* dmean = (double*)p;
  double* dcov = dmean + (size_t)K * d;
  CU(A.get("KF_MISC", 64, &p));
  double* dll = (double*)p;
  int* dbad = (int*)((char*)p + 16);
  CU(cudaMemsetAsync(p, 0, 64, s));
  switch (d) {
    case 1: rc = kalman_device_dy<1>(ctx, dy, km, K, dmean, dcov, dll, dbad); break;
    case 2: rc = kalman_device_dy<2>(ctx, dy, km, K, dmean, dcov, dll, dbad); break;
    case 3: rc = kalman_device_dy<3>(ctx, dy, km, K, dmean, dcov, dll, dbad); break;
    default: rc = kalman_device_dy<4>(ctx, dy, km, K, dmean, dcov, dll, dbad); break;
  }
  if (rc) return rc;
  int bad = 0;
  double ll = 0;
  CU(cudaMemcpyAsync(smooth_mean, dmean, (size_t)K * d * sizeof(double), cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(smooth_cov, dcov, (size_t)K * d * d * sizeof(double), cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(&ll, dll, sizeof ll, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(&bad, dbad, sizeof bad, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (bad)
    return set_err(ctx, DSMC_E_RUNTIME,
                   "kalman update: covariance is not positive definite (device scan)");
  if (log_likelihood) *log_likelihood = ll;
  return DSMC_OK;
}

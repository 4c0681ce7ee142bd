// C++ host layer, part 2: the reference's metrics, backend selector,
// PairWeightSource resampling, index resampling, the fk_model helpers and
// the piecewise smoother API (make_leaf, make_pair_source, combine_blocks)
// over the device entry points of include/dsmc_b200.h.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <limits>
#include <stdexcept>

#include "dsmc/dsmc.hpp"
#include "internal.hpp"

namespace dsmc {

// ---------------------------------------------------------------- metrics
namespace metrics {
namespace {
std::atomic<std::uint64_t> g_weight_evals{0}, g_dense_allocs{0}, g_dense_max{0}, g_lazy_max{0};
void raise_max(std::atomic<std::uint64_t>& slot, std::uint64_t v) {
  std::uint64_t cur = slot.load(std::memory_order_relaxed);
  while (cur < v && !slot.compare_exchange_weak(cur, v, std::memory_order_relaxed)) {
  }
}
}  // namespace
void reset() {
  g_weight_evals = 0;
  g_dense_allocs = 0;
  g_dense_max = 0;
  g_lazy_max = 0;
}
Snapshot snapshot() {
  Snapshot s;
  s.weight_evals = g_weight_evals.load(std::memory_order_relaxed);
  s.dense_allocs = g_dense_allocs.load(std::memory_order_relaxed);
  s.dense_max_elems = g_dense_max.load(std::memory_order_relaxed);
  s.lazy_max_elems = g_lazy_max.load(std::memory_order_relaxed);
  return s;
}
void add_weight_evals(std::uint64_t n) { g_weight_evals.fetch_add(n, std::memory_order_relaxed); }
void count_dense_alloc(std::size_t elems) {
  g_dense_allocs.fetch_add(1, std::memory_order_relaxed);
  raise_max(g_dense_max, elems);
}
void note_lazy_alloc(std::size_t elems) { raise_max(g_lazy_max, elems); }
}  // namespace metrics

// ---------------------------------------------------------------- kernels
namespace kernels {
namespace {
std::atomic<int> g_backend{static_cast<int>(Backend::scalar)};
}
Backend active() { return static_cast<Backend>(g_backend.load()); }
void set_active(Backend b) { g_backend.store(static_cast<int>(b)); }
bool available(Backend) { return true; }  // one arithmetic on the device
}  // namespace kernels

void tune_allocator_once() {}

namespace {

using detail::check;
using detail::context;
using detail::desc_of;

constexpr int kPairRole = static_cast<int>(StreamRole::pair_resample);

void require_pair_role(const StreamKey& key) {
  if (static_cast<int>(key.role) != kPairRole)
    throw std::invalid_argument(
        "pair resampling draws from pair_resample streams (resampling.cpp keys)");
}

// resampling.cpp:27-38: fill_row, or the entry probe row by row
std::function<void(std::size_t, double*)> row_filler(const PairWeightSource& src) {
  if (src.fill_row) return src.fill_row;
  if (!src.log_weight_at)
    throw std::invalid_argument(
        "pair weight source provides neither fill_row nor log_weight_at");
  auto probe = src.log_weight_at;
  const std::size_t n = src.n;
  return [probe, n](std::size_t i, double* out) {
    for (std::size_t j = 0; j < n; ++j) out[j] = probe(i, j);
  };
}

// a block pair attached by make_pair_source: the device evaluates the table
PairSample device_blocks(Resampler r, const PairWeightSource& src, std::size_t n_out,
                         std::size_t mh_steps, const StreamKey& key) {
  const detail::BlockPairSource& bp = *src.blocks;
  dsmc_ctx* c = context(0);
  dsmc_pair_blocks pb{bp.cut, bp.n, bp.xl, bp.lw_l, bp.lw_l ? 0 : 1,
                      bp.xr, bp.lw_r, bp.lw_r ? 0 : 1};
  PairSample ps;
  ps.left.resize(n_out);
  ps.right.resize(n_out);
  double lmw = 0;
  int has = 0, biased = 0;
  uint64_t ev = 0;
  check(c, dsmc_resample_blocks(c, &bp.model->desc, &pb, static_cast<int>(r), n_out, mh_steps,
                                key.seed, key.level, key.node, ps.left.data(),
                                ps.right.data(), &lmw, &has, &ev, &biased));
  if (has) ps.log_mean_weight = lmw;
  ps.weight_evals = ev;
  ps.biased = biased != 0;
  if (resampler_is_lazy(r))
    metrics::note_lazy_alloc(2 * n_out);
  else
    metrics::count_dense_alloc(bp.n * bp.n);
  metrics::add_weight_evals(ev);
  return ps;
}

// a caller source, dense scheme: the table is filled on the host (where the
// callbacks live) once and sampled on the device
PairSample host_dense(Resampler r, const PairWeightSource& src, std::size_t n_out,
                      const StreamKey& key) {
  const std::size_t n = src.n;
  if (n == 0) throw std::invalid_argument("pair weight source has n == 0");
  auto fill = row_filler(src);
  std::vector<double> tab(n * n);
  metrics::count_dense_alloc(n * n);
  for (std::size_t i = 0; i < n; ++i) fill(i, tab.data() + i * n);
  dsmc_ctx* c = context(0);
  PairSample ps;
  ps.left.resize(n_out);
  ps.right.resize(n_out);
  double lmw = 0;
  int has = 0, biased = 0;
  uint64_t ev = 0;
  check(c, dsmc_resample_table(c, static_cast<int>(r), tab.data(), n, n_out, 0, 0, 0.0,
                               key.seed, key.level, key.node, ps.left.data(), ps.right.data(),
                               &lmw, &has, &ev, &biased));
  if (has) ps.log_mean_weight = lmw;
  ps.weight_evals = ev;
  metrics::add_weight_evals(ev);
  return ps;
}

// a caller source, lazy scheme: the device asks for the entries its slots
// probe, round by round (dsmc_lazy_*); the host evaluates only those
PairSample host_lazy(Resampler r, const PairWeightSource& src, std::size_t n_out,
                     std::size_t mh_steps, const StreamKey& key) {
  const std::size_t n = src.n;
  if (n == 0) throw std::invalid_argument("pair weight source has n == 0");
  if (r == Resampler::rejection_lazy &&
      (!src.log_upper_bound || !std::isfinite(*src.log_upper_bound)))
    throw std::invalid_argument("rejection resampling requires a finite log_upper_bound");
  const bool need_probe = n_out > 0 && !(r == Resampler::mh_lazy && mh_steps == 0);
  if (need_probe && !src.log_weight_at)
    throw std::invalid_argument("lazy resampling requires a log_weight_at entry probe");
  dsmc_ctx* c = context(0);
  std::size_t np = 0;
  check(c, dsmc_lazy_begin(c, static_cast<int>(r), n, n_out, mh_steps,
                           src.log_upper_bound ? 1 : 0, src.log_upper_bound.value_or(0.0),
                           key.seed, key.level, key.node, &np));
  // transient: probe coordinates + values, at most 2 per slot
  metrics::note_lazy_alloc(2 * std::max<std::size_t>(np, n_out));
  std::vector<uint32_t> pi, pj;
  std::vector<double> val;
  while (np) {
    pi.resize(np);
    pj.resize(np);
    val.resize(np);
    check(c, dsmc_lazy_probes(c, pi.data(), pj.data()));
    for (std::size_t q = 0; q < np; ++q) val[q] = src.log_weight_at(pi[q], pj[q]);
    check(c, dsmc_lazy_answer(c, val.data(), &np));
  }
  PairSample ps;
  ps.left.resize(n_out);
  ps.right.resize(n_out);
  uint64_t ev = 0;
  check(c, dsmc_lazy_finish(c, ps.left.data(), ps.right.data(), &ev));
  ps.weight_evals = ev;
  ps.biased = r == Resampler::mh_lazy;
  metrics::add_weight_evals(ev);
  return ps;
}

IndexSample index_sample(Resampler r, const double* log_w, std::size_t n, std::size_t n_out,
                         const StreamKey& key) {
  if (n == 0) throw std::invalid_argument("weight vector has n == 0");
  if (resampler_is_lazy(r))
    throw std::invalid_argument("index resampling: only the dense schemes exist");
  dsmc_ctx* c = context(0);
  IndexSample out;
  out.idx.resize(n_out);
  double mx = 0, total = 0;
  check(c, dsmc_resample_indices(c, static_cast<int>(r), log_w, n, n_out, key.seed, key.level,
                                 key.node, static_cast<int>(key.role), out.idx.data(), &mx,
                                 &total));
  // build_row_weights (resampling.cpp:337-349): m + log(total) - log(n)
  out.log_mean_weight = mx + std::log(total) - std::log(static_cast<double>(n));
  return out;
}

}  // namespace

// ------------------------------------------------------------ resampling
PairSample resample_pairs(Resampler r, const PairWeightSource& src, std::size_t n_out,
                          std::size_t mh_steps, const StreamKey& key) {
  require_pair_role(key);
  if (src.blocks && n_out <= src.n) return device_blocks(r, src, n_out, mh_steps, key);
  switch (r) {
    case Resampler::multinomial:
    case Resampler::systematic: return host_dense(r, src, n_out, key);
    case Resampler::mh_lazy:
    case Resampler::rejection_lazy: return host_lazy(r, src, n_out, mh_steps, key);
  }
  throw std::invalid_argument("unknown resampler");
}
PairSample multinomial_pairs(const PairWeightSource& src, std::size_t n_out,
                             const StreamKey& key) {
  return resample_pairs(Resampler::multinomial, src, n_out, 0, key);
}
PairSample systematic_pairs(const PairWeightSource& src, std::size_t n_out,
                            const StreamKey& key) {
  return resample_pairs(Resampler::systematic, src, n_out, 0, key);
}
PairSample mh_lazy_pairs(const PairWeightSource& src, std::size_t n_out, std::size_t mh_steps,
                         const StreamKey& key) {
  return resample_pairs(Resampler::mh_lazy, src, n_out, mh_steps, key);
}
PairSample rejection_lazy_pairs(const PairWeightSource& src, std::size_t n_out,
                                const StreamKey& key) {
  return resample_pairs(Resampler::rejection_lazy, src, n_out, 0, key);
}

IndexSample multinomial_indices(const double* log_w, std::size_t n, std::size_t n_out,
                                const StreamKey& key) {
  return index_sample(Resampler::multinomial, log_w, n, n_out, key);
}
IndexSample systematic_indices(const double* log_w, std::size_t n, std::size_t n_out,
                               const StreamKey& key) {
  return index_sample(Resampler::systematic, log_w, n, n_out, key);
}
IndexSample resample_indices(Resampler r, const double* log_w, std::size_t n, std::size_t n_out,
                             const StreamKey& key) {
  return index_sample(r, log_w, n, n_out, key);
}

// --------------------------------------------------------------- fk_model
namespace {
void check_time(int t, int horizon, int lo, const char* what) {
  if (t < lo || t > horizon)
    throw std::invalid_argument(std::string(what) + ": time index " + std::to_string(t) +
                                " outside [" + std::to_string(lo) + ", " +
                                std::to_string(horizon) + "]");
}
double checked(double v, const char* what) {
  if (std::isnan(v)) throw std::invalid_argument(std::string(what) + " produced NaN");
  return v;
}
}  // namespace

// fk_model.cpp:43-59
double log_init_weight(const FeynmanKacModel& model, int t, const double* x) {
  check_time(t, model.horizon, 0, "log_init_weight");
  double w;
  if (t == 0) {
    const double pot = model.log_potential(0, x);
    const double p0 = model.init_logdensity(x);
    const double q = model.proposal_logdensity(0, x);
    w = pot + p0 - q;
    if (pot == -INFINITY || p0 == -INFINITY) w = -INFINITY;
  } else {
    const double nu = model.aux_logdensity(t, x);
    const double q = model.proposal_logdensity(t, x);
    w = nu == -INFINITY ? -INFINITY : nu - q;
  }
  return checked(w, "log_init_weight");
}

// fk_model.cpp:75-86
StitchRowFn make_stitch_row(const FeynmanKacModel& model, int c, const double* right,
                            std::size_t n) {
  check_time(c, model.horizon, 1, "make_stitch_row");
  if (model.stitch_row_factory) return model.stitch_row_factory(c, right, n);
  const int d = model.state_dim;
  return [&model, c, right, n, d](const double* x_prev, double* out) {
    for (std::size_t j = 0; j < n; ++j)
      out[j] = log_stitch_weight(model, c, x_prev, right + j * d);
  };
}

// fk_model.cpp:88-99
TransitionRowFn make_transition_row(const FeynmanKacModel& model, int t, const double* prev,
                                    std::size_t n) {
  check_time(t, model.horizon, 1, "make_transition_row");
  if (model.transition_row_factory) return model.transition_row_factory(t, prev, n);
  const int d = model.state_dim;
  return [&model, t, prev, n, d](const double* x_cur, double* out) {
    for (std::size_t j = 0; j < n; ++j)
      out[j] = model.transition_logdensity(t, prev + j * d, x_cur);
  };
}

// fk_model.cpp:101-112
void leaf_weights(const FeynmanKacModel& model, int t, const double* particles, std::size_t n,
                  double* out) {
  check_time(t, model.horizon, 0, "leaf_weights");
  if (model.init_weight_batch) {
    model.init_weight_batch(t, particles, n, out);
    for (std::size_t i = 0; i < n; ++i) checked(out[i], "init_weight_batch");
    return;
  }
  const int d = model.state_dim;
  for (std::size_t i = 0; i < n; ++i) out[i] = log_init_weight(model, t, particles + i * d);
}

// ------------------------------------------------------ piecewise smoother
// make_leaf (smoother.cpp:98-130) drawn and weighed on the device
BlockEstimate make_leaf(const FeynmanKacModel& model, int t, std::size_t n,
                        std::uint64_t seed) {
  if (n == 0) throw std::invalid_argument("make_leaf: n must be >= 1");
  if (n > 0xffffffffu) throw std::invalid_argument("make_leaf: n exceeds the 32-bit index range");
  if (t < 0 || t > model.horizon)
    throw std::invalid_argument("make_leaf: time outside 0..horizon");
  const dsmc_model_desc& desc = detail::device_desc(model);
  dsmc_ctx* c = context(0);
  BlockEstimate blk;
  blk.a = blk.b = t;
  blk.n = n;
  blk.dim = model.state_dim;
  blk.paths.resize(n * static_cast<std::size_t>(blk.dim));
  blk.log_w.resize(n);
  int uni = 0;
  double lnc = NAN;
  check(c, dsmc_make_leaf(c, &desc, t, n, seed, blk.paths.data(), blk.log_w.data(), &uni, &lnc));
  blk.weights_uniform = uni != 0;
  blk.log_norm_const = lnc;
  return blk;
}

// smoother.cpp:132-180: the reference's closures, plus the device attachment
PairSourceBundle make_pair_source(const FeynmanKacModel& model, const BlockEstimate& left,
                                  const BlockEstimate& right) {
  if (left.b + 1 != right.a)
    throw std::invalid_argument("make_pair_source: blocks are not adjacent");
  if (left.n != right.n || left.n == 0)
    throw std::invalid_argument("make_pair_source: block sizes differ");
  if (left.dim != right.dim) throw std::invalid_argument("make_pair_source: block dims differ");
  const int c = right.a;
  const std::size_t n = left.n;
  const int dim = left.dim;
  const double* xl = left.time_slab(left.b);
  const double* xr = right.time_slab(right.a);
  const double* lw_l = left.weights_uniform ? nullptr : left.log_w.data();
  const double* lw_r = right.weights_uniform ? nullptr : right.log_w.data();
  PairSourceBundle bundle;
  bundle.source.n = n;
  if (model.log_potential && model.transition_logdensity && model.aux_logdensity) {
    StitchRowFn row = make_stitch_row(model, c, xr, n);
    bundle.source.fill_row = [row, xl, lw_l, lw_r, n, dim](std::size_t i, double* out) {
      row(xl + i * dim, out);
      const double s = lw_l ? lw_l[i] : 0.0;
      if (lw_r)
        for (std::size_t j = 0; j < n; ++j) out[j] = (out[j] + s) + lw_r[j];
      else if (s != 0.0)
        for (std::size_t j = 0; j < n; ++j) out[j] += s;
    };
    const FeynmanKacModel* mp = &model;
    bundle.source.log_weight_at = [mp, c, xl, xr, lw_l, lw_r, dim](std::size_t i,
                                                                  std::size_t j) {
      double v = log_stitch_weight(*mp, c, xl + i * dim, xr + j * dim);
      if (lw_l) v += lw_l[i];
      if (lw_r) v += lw_r[j];
      return v;
    };
  }
  if (model.log_stitch_bound) {
    double b = model.log_stitch_bound(c);
    if (lw_l) b += *std::max_element(lw_l, lw_l + n);
    if (lw_r) b += *std::max_element(lw_r, lw_r + n);
    bundle.source.log_upper_bound = b;
  }
  if (model.device) {
    auto bp = std::make_shared<detail::BlockPairSource>();
    bp->model = model.device;
    bp->cut = c;
    bp->n = n;
    bp->xl = xl;
    bp->xr = xr;
    bp->lw_l = lw_l;
    bp->lw_r = lw_r;
    bundle.source.blocks = bp;
  }
  const double logn = std::log(static_cast<double>(n));
  bundle.log_shift = (left.weights_uniform ? -logn : 0.0) + (right.weights_uniform ? -logn : 0.0);
  return bundle;
}

// smoother.cpp:182-224: resample on the device, concatenate the selected paths
BlockEstimate combine_blocks(const FeynmanKacModel& model, const BlockEstimate& left,
                             const BlockEstimate& right, const SmootherOptions& options,
                             int level, int node) {
  auto bundle = make_pair_source(model, left, right);
  const std::size_t n = left.n;
  const StreamKey key{options.seed, static_cast<std::uint32_t>(level),
                      static_cast<std::uint64_t>(node), StreamRole::pair_resample};
  PairSample ps;
  try {
    ps = resample_pairs(options.resampler, bundle.source, n, options.mh_steps, key);
  } catch (const std::runtime_error& e) {
    throw std::runtime_error("combine at cut " + std::to_string(right.a) + " (times " +
                             std::to_string(left.a) + ".." + std::to_string(right.b) +
                             "): " + e.what());
  }
  BlockEstimate out;
  out.a = left.a;
  out.b = right.b;
  out.n = n;
  out.dim = left.dim;
  out.paths.resize(static_cast<std::size_t>(out.len()) * n * out.dim);
  const std::size_t row = sizeof(double) * out.dim;
  for (int t = left.a; t <= left.b; ++t)
    for (std::size_t p = 0; p < n; ++p)
      std::memcpy(out.time_slab(t) + p * out.dim,
                  left.time_slab(t) + static_cast<std::size_t>(ps.left[p]) * out.dim, row);
  for (int t = right.a; t <= right.b; ++t)
    for (std::size_t p = 0; p < n; ++p)
      std::memcpy(out.time_slab(t) + p * out.dim,
                  right.time_slab(t) + static_cast<std::size_t>(ps.right[p]) * out.dim, row);
  out.log_w.assign(n, -std::log(static_cast<double>(n)));
  out.weights_uniform = true;
  out.biased = left.biased || right.biased || ps.biased;
  out.weight_evals = left.weight_evals + right.weight_evals + ps.weight_evals;
  if (left.log_norm_const && right.log_norm_const && ps.log_mean_weight)
    out.log_norm_const =
        *left.log_norm_const + *right.log_norm_const + *ps.log_mean_weight + bundle.log_shift;
  return out;
}

}  // namespace dsmc

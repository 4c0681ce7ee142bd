// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// C API over the compiled reference (oracle/_ref/libdsmc_ref.so): the
// reference's own rng.cpp, kernels/*.cpp, resampling.cpp, fk_model.cpp,
// smoother.cpp, conditional.cpp compiled unmodified from /root/reference
// (see oracle/Makefile). Used by tests/ (golden vectors, parity) and by
// bench.py's CPU baseline leg; never by the product.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <atomic>
#include <mutex>
#include <exception>
#include <vector>

#include "dsmc/conditional.hpp"
#include "dsmc/fk_model.hpp"
#include "dsmc/kernels.hpp"
#include "dsmc/metrics.hpp"
#include "dsmc/resampling.hpp"
#include "dsmc/rng.hpp"
#include "dsmc/smoother.hpp"
#include "dsmc_b200.h"
#include "ref_models.hpp"

namespace {

thread_local std::string g_err;

template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    g_err.clear();
    return DSMC_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return DSMC_E_INVALID_ARGUMENT;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return DSMC_E_DOMAIN;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return DSMC_E_LOGIC;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return DSMC_E_RUNTIME;
  } catch (const std::exception& e) {
    g_err = e.what();
    return DSMC_E_RUNTIME;
  }
}

dsmc::StreamKey key_of(uint64_t seed, uint32_t level, uint64_t node, int role) {
  return dsmc::StreamKey{seed, level, node, static_cast<dsmc::StreamRole>(role)};
}

dsmc::PairWeightSource table_source(const double* logw, std::size_t n,
                                    int has_bound, double bound) {
  std::vector<double> tab(logw, logw + n * n);
  dsmc::PairWeightSource src;
  src.n = n;
  src.fill_row = [tab, n](std::size_t i, double* out) {
    std::memcpy(out, tab.data() + i * n, n * sizeof(double));
  };
  src.log_weight_at = [tab, n](std::size_t i, std::size_t j) {
    return tab[i * n + j];
  };
  if (has_bound) src.log_upper_bound = bound;
  return src;
}

// The reference model with injected leaves: proposal_sampler copies the
// given time-t slab (n states) instead of drawing, and, when raw weights are
// given, init_weight_batch returns them (leaf_weights, fk_model.cpp:101-112);
// otherwise the model's own weight callbacks run on the injected states.
dsmc::FeynmanKacModel injected(const dsmc::FeynmanKacModel& base, const double* X,
                               const double* W, std::size_t n) {
  dsmc::FeynmanKacModel m = base;
  const int d = base.state_dim;
  m.proposal_sampler = [X, n, d](int t, std::size_t count, dsmc::RngStream&, double* out) {
    if (count != n) throw std::logic_error("injected leaves: unexpected draw count");
    std::memcpy(out, X + static_cast<std::size_t>(t) * n * d, sizeof(double) * n * d);
  };
  if (W)
    m.init_weight_batch = [W, n](int t, const double*, std::size_t count, double* out) {
      if (count != n) throw std::logic_error("injected weights: unexpected count");
      std::memcpy(out, W + static_cast<std::size_t>(t) * n, sizeof(double) * n);
    };
  return m;
}

// parallel_for over [0, count) with a shared cursor (smoother.cpp:21-49)
void par_for(std::size_t count, int threads, const std::function<void(std::size_t)>& fn) {
  if (threads <= 1 || count <= 1) {
    for (std::size_t i = 0; i < count; ++i) fn(i);
    return;
  }
  std::atomic<std::size_t> cursor{0};
  std::mutex mu;
  std::exception_ptr err;
  auto body = [&] {
    for (;;) {
      const std::size_t i = cursor.fetch_add(1);
      if (i >= count) return;
      try {
        fn(i);
      } catch (...) {
        std::lock_guard<std::mutex> lock(mu);
        if (!err) err = std::current_exception();
      }
    }
  };
  std::vector<std::thread> pool;
  for (int w = 0; w < threads && (std::size_t)w < count; ++w) pool.emplace_back(body);
  for (auto& th : pool) th.join();
  if (err) std::rethrow_exception(err);
}

}  // namespace

namespace dsmc {
// the reference's gamma_draw (pgibbs.cpp:80-102), compiled from its own source
// by oracle/Makefile (gamma_draw_ref.cpp)
double gamma_draw(double shape, double rate, RngStream& stream);
}  // namespace dsmc

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_philox(const uint64_t ctr[4], const uint64_t key[2], uint64_t out[4]) {
  auto r = dsmc::rng_detail::philox4x64_10({ctr[0], ctr[1], ctr[2], ctr[3]},
                                           {key[0], key[1]});
  for (int i = 0; i < 4; ++i) out[i] = r[i];
}

// kind: 0 next_u64, 1 uniform, 2 uniform_pos, 3 normal
void ref_stream(uint64_t seed, uint32_t level, uint64_t node, int role,
                uint64_t substream, int kind, size_t n, void* out) {
  dsmc::RngStream s(key_of(seed, level, node, role), substream);
  for (size_t i = 0; i < n; ++i) {
    switch (kind) {
      case 0: static_cast<uint64_t*>(out)[i] = s.next_u64(); break;
      case 1: static_cast<double*>(out)[i] = s.uniform(); break;
      case 2: static_cast<double*>(out)[i] = s.uniform_pos(); break;
      default: static_cast<double*>(out)[i] = s.normal(); break;
    }
  }
}

int ref_set_backend(int b) {
  return guarded([&] {
    dsmc::kernels::set_active(static_cast<dsmc::kernels::Backend>(b));
  });
}
int ref_active_backend() { return static_cast<int>(dsmc::kernels::active()); }

double ref_exp_w(double x) { return dsmc::kernels::exp_w(x); }
void ref_vec_exp(const double* x, size_t n, double* out) {
  dsmc::kernels::vec_exp(x, n, out);
}
double ref_reduce_sum(const double* x, size_t n) {
  return dsmc::kernels::reduce_sum(x, n);
}
int ref_reduce_max(const double* x, size_t n, double* out) {
  return guarded([&] { *out = dsmc::kernels::reduce_max(x, n); });
}
double ref_log_sum_exp(const double* x, size_t n) {
  return dsmc::kernels::log_sum_exp(x, n);
}
double ref_exp_row_store(const double* logw, size_t n, double shift, double* w,
                         double* sub) {
  return dsmc::kernels::exp_row_store(logw, n, shift, w, sub);
}
void ref_gaussian_row(const double* x, size_t n, double mean, double c,
                      const double* base, double* out) {
  dsmc::kernels::gaussian_row(x, n, mean, c, base, out);
}

void ref_metrics_reset() { dsmc::metrics::reset(); }
void ref_metrics(uint64_t out[4]) {
  auto s = dsmc::metrics::snapshot();
  out[0] = s.weight_evals;
  out[1] = s.dense_allocs;
  out[2] = s.dense_max_elems;
  out[3] = s.lazy_max_elems;
}

int ref_resample_table(int resampler, const double* logw, size_t n,
                       size_t n_out, size_t mh_steps, int has_bound,
                       double bound, uint64_t seed, uint32_t level,
                       uint64_t node, uint32_t* left, uint32_t* right,
                       double* lmw, int* has_lmw, uint64_t* evals,
                       int* biased) {
  return guarded([&] {
    auto src = table_source(logw, n, has_bound, bound);
    auto ps = dsmc::resample_pairs(static_cast<dsmc::Resampler>(resampler), src,
                                   n_out, mh_steps,
                                   key_of(seed, level, node,
                                          DSMC_ROLE_PAIR_RESAMPLE));
    std::memcpy(left, ps.left.data(), sizeof(uint32_t) * n_out);
    std::memcpy(right, ps.right.data(), sizeof(uint32_t) * n_out);
    *has_lmw = ps.log_mean_weight.has_value() ? 1 : 0;
    *lmw = ps.log_mean_weight.value_or(NAN);
    *evals = ps.weight_evals;
    *biased = ps.biased ? 1 : 0;
  });
}

// pairs: 5 ints per pair (level, node, left_a, left_b, right_b).
int ref_build_schedule(int horizon, int* levels, int* pairs) {
  return guarded([&] {
    auto s = dsmc::build_schedule(horizon);
    *levels = s.levels;
    for (size_t k = 0; k < s.pairs.size(); ++k) {
      const auto& p = s.pairs[k];
      int* o = pairs + 5 * k;
      o[0] = p.level;
      o[1] = p.node;
      o[2] = p.left_a;
      o[3] = p.left_b;
      o[4] = p.right_b;
    }
  });
}
int ref_tree_depth(int horizon) { return dsmc::reference_tree_depth(horizon); }

// make_leaf (smoother.cpp:98-130): states, normalized log weights, flags,
// plus the raw leaf weights (fk_model.cpp:101-112) for injection.
int ref_make_leaf(const dsmc_model_desc* desc, int t, size_t n, uint64_t seed,
                  double* x, double* raw_lw, double* norm_lw, int* uniform,
                  double* lnc) {
  return guarded([&] {
    auto model = oracle::build_model(*desc);
    auto blk = dsmc::make_leaf(model, t, n, seed);
    std::memcpy(x, blk.paths.data(), sizeof(double) * blk.paths.size());
    if (norm_lw) std::memcpy(norm_lw, blk.log_w.data(), sizeof(double) * n);
    if (raw_lw) dsmc::leaf_weights(model, t, blk.paths.data(), n, raw_lw);
    *uniform = blk.weights_uniform ? 1 : 0;
    *lnc = blk.log_norm_const.value_or(NAN);
  });
}

// Stitch-row fill of the reference model for one combine (the dense table
// the reference would build), for table-level parity checks.
int ref_stitch_rows(const dsmc_model_desc* desc, int c, const double* xl,
                    const double* xr, size_t n, double* out) {
  return guarded([&] {
    auto model = oracle::build_model(*desc);
    auto row = dsmc::make_stitch_row(model, c, xr, n);
    const int d = model.state_dim;
    for (size_t i = 0; i < n; ++i) row(xl + i * d, out + i * n);
  });
}

// Scalar log_stitch_weight (fk_model.cpp:61-73).
int ref_stitch_weight(const dsmc_model_desc* desc, int c, const double* xp,
                      const double* xc, double* out) {
  return guarded([&] {
    auto model = oracle::build_model(*desc);
    *out = dsmc::log_stitch_weight(model, c, xp, xc);
  });
}

int ref_stitch_bound(const dsmc_model_desc* desc, int c, double* out) {
  return guarded([&] {
    auto model = oracle::build_model(*desc);
    if (!model.log_stitch_bound)
      throw std::invalid_argument("model has no stitch bound");
    *out = model.log_stitch_bound(c);
  });
}

// run_smoother (smoother.cpp:226-277) unchanged; root paths + metadata.
int ref_run_smoother(const dsmc_model_desc* desc, size_t n, int resampler,
                     size_t mh_steps, uint64_t seed, int threads,
                     double* root_paths, double* lnc, int* has_lnc,
                     uint64_t* evals, int* levels, int* biased,
                     double* wall_ms) {
  return guarded([&] {
    auto model = oracle::build_model(*desc);
    dsmc::SmootherOptions o;
    o.n_particles = n;
    o.resampler = static_cast<dsmc::Resampler>(resampler);
    o.mh_steps = mh_steps;
    o.seed = seed;
    o.n_threads = threads;
    auto res = dsmc::run_smoother(model, o);
    if (root_paths)
      std::memcpy(root_paths, res.root.paths.data(),
                  sizeof(double) * res.root.paths.size());
    *has_lnc = res.meta.log_norm_const.has_value() ? 1 : 0;
    *lnc = res.meta.log_norm_const.value_or(NAN);
    *evals = res.meta.weight_evals;
    *levels = res.meta.levels;
    *biased = res.meta.biased ? 1 : 0;
    *wall_ms = res.meta.wall_time_ms;
  });
}

// The same run, level by level through the public pieces (make_leaf,
// make_pair_source, resample_pairs, combine_blocks), recording every
// combine's (left, right) pairs and log mean weight in schedule order.
int ref_trace_smoother(const dsmc_model_desc* desc, size_t n, int resampler,
                       size_t mh_steps, uint64_t seed, double* root_paths,
                       uint32_t* pair_left, uint32_t* pair_right,
                       double* pair_lmw, double* lnc, int* has_lnc) {
  return guarded([&] {
    auto model = oracle::build_model(*desc);
    dsmc::SmootherOptions o;
    o.n_particles = n;
    o.resampler = static_cast<dsmc::Resampler>(resampler);
    o.mh_steps = mh_steps;
    o.seed = seed;
    const int T = model.horizon;
    std::vector<dsmc::BlockEstimate> cur(T + 1);
    for (int t = 0; t <= T; ++t) cur[t] = dsmc::make_leaf(model, t, n, seed);
    int level = 0;
    size_t cursor = 0;
    while (cur.size() > 1) {
      ++level;
      const size_t np = cur.size() / 2;
      std::vector<dsmc::BlockEstimate> next(np + cur.size() % 2);
      for (size_t k = 0; k < np; ++k) {
        const auto& L = cur[2 * k];
        const auto& R = cur[2 * k + 1];
        auto bundle = dsmc::make_pair_source(model, L, R);
        auto ps = dsmc::resample_pairs(
            o.resampler, bundle.source, n, o.mh_steps,
            key_of(seed, level, k, DSMC_ROLE_PAIR_RESAMPLE));
        std::memcpy(pair_left + (cursor + k) * n, ps.left.data(),
                    sizeof(uint32_t) * n);
        std::memcpy(pair_right + (cursor + k) * n, ps.right.data(),
                    sizeof(uint32_t) * n);
        pair_lmw[cursor + k] = ps.log_mean_weight.value_or(NAN);
        next[k] = dsmc::combine_blocks(model, L, R, o, level, (int)k);
      }
      if (cur.size() % 2) next.back() = std::move(cur.back());
      cursor += np;
      cur = std::move(next);
    }
    const auto& root = cur.front();
    std::memcpy(root_paths, root.paths.data(),
                sizeof(double) * root.paths.size());
    *has_lnc = root.log_norm_const.has_value() ? 1 : 0;
    *lnc = root.log_norm_const.value_or(NAN);
  });
}

// run_smoother on INJECTED leaves (states, optional raw weights): with no
// pair outputs this is run_smoother itself on the wrapped model; with pair
// outputs the level loop of run_smoother (smoother.cpp:236-262) runs here,
// multithreaded: the reference's make_pair_source + resample_pairs with the
// key combine_blocks uses, recorded, then the combined block assembled from
// those pairs exactly as combine_blocks does (tests/test_oracle.py checks the
// root against run_smoother's).
int ref_run_injected(const dsmc_model_desc* desc, size_t n, int resampler, size_t mh_steps,
                     uint64_t seed, int threads, const double* inj_x, const double* inj_w,
                     double* root_paths, uint32_t* pair_left, uint32_t* pair_right,
                     double* pair_lmw, double* lnc, int* has_lnc, uint64_t* evals,
                     int* levels, int* biased) {
  return guarded([&] {
    auto base = oracle::build_model(*desc);
    auto model = injected(base, inj_x, inj_w, n);
    dsmc::SmootherOptions o;
    o.n_particles = n;
    o.resampler = static_cast<dsmc::Resampler>(resampler);
    o.mh_steps = mh_steps;
    o.seed = seed;
    o.n_threads = threads;
    if (!pair_left) {
      auto res = dsmc::run_smoother(model, o);
      if (root_paths)
        std::memcpy(root_paths, res.root.paths.data(), sizeof(double) * res.root.paths.size());
      *has_lnc = res.meta.log_norm_const.has_value() ? 1 : 0;
      *lnc = res.meta.log_norm_const.value_or(NAN);
      *evals = res.meta.weight_evals;
      *levels = res.meta.levels;
      *biased = res.meta.biased ? 1 : 0;
      return;
    }
    const int T = model.horizon;
    std::vector<dsmc::BlockEstimate> cur(T + 1);
    par_for(T + 1, threads, [&](std::size_t t) { cur[t] = dsmc::make_leaf(model, (int)t, n, seed); });
    int level = 0;
    size_t cursor = 0;
    while (cur.size() > 1) {
      ++level;
      const size_t np = cur.size() / 2;
      std::vector<dsmc::BlockEstimate> next(np + cur.size() % 2);
      par_for(np, threads, [&](std::size_t k) {
        const auto& L = cur[2 * k];
        const auto& R = cur[2 * k + 1];
        auto bundle = dsmc::make_pair_source(model, L, R);
        auto ps = dsmc::resample_pairs(o.resampler, bundle.source, n, o.mh_steps,
                                       key_of(seed, level, k, DSMC_ROLE_PAIR_RESAMPLE));
        std::memcpy(pair_left + (cursor + k) * n, ps.left.data(), sizeof(uint32_t) * n);
        std::memcpy(pair_right + (cursor + k) * n, ps.right.data(), sizeof(uint32_t) * n);
        if (pair_lmw) pair_lmw[cursor + k] = ps.log_mean_weight.value_or(NAN);
        // the block combine_blocks (smoother.cpp:182-224) builds from these
        // same pairs: every time slab gathered by (left, right), uniform
        // weights, summed evals, log Z += log mean weight + log_shift
        dsmc::BlockEstimate out;
        out.a = L.a;
        out.b = R.b;
        out.n = n;
        out.dim = L.dim;
        out.paths.resize(static_cast<std::size_t>(out.len()) * n * out.dim);
        for (int t = L.a; t <= L.b; ++t)
          for (std::size_t p = 0; p < n; ++p)
            std::memcpy(out.time_slab(t) + p * out.dim,
                        L.time_slab(t) + static_cast<std::size_t>(ps.left[p]) * out.dim,
                        sizeof(double) * out.dim);
        for (int t = R.a; t <= R.b; ++t)
          for (std::size_t p = 0; p < n; ++p)
            std::memcpy(out.time_slab(t) + p * out.dim,
                        R.time_slab(t) + static_cast<std::size_t>(ps.right[p]) * out.dim,
                        sizeof(double) * out.dim);
        out.log_w.assign(n, -std::log(static_cast<double>(n)));
        out.weights_uniform = true;
        out.biased = L.biased || R.biased || ps.biased;
        out.weight_evals = L.weight_evals + R.weight_evals + ps.weight_evals;
        if (L.log_norm_const && R.log_norm_const && ps.log_mean_weight)
          out.log_norm_const = *L.log_norm_const + *R.log_norm_const + *ps.log_mean_weight +
                               bundle.log_shift;
        next[k] = std::move(out);
      });
      if (cur.size() % 2) next.back() = std::move(cur.back());
      cursor += np;
      cur = std::move(next);
    }
    const auto& root = cur.front();
    if (root_paths) std::memcpy(root_paths, root.paths.data(), sizeof(double) * root.paths.size());
    *has_lnc = root.log_norm_const.has_value() ? 1 : 0;
    *lnc = root.log_norm_const.value_or(NAN);
    *evals = root.weight_evals;
    *levels = level;
    *biased = root.biased ? 1 : 0;
  });
}

// leaf_weights (fk_model.cpp:101-112) of every time slab: raw log weights of
// given states, (T+1) x n.
int ref_leaf_weights_all(const dsmc_model_desc* desc, const double* X, size_t n, double* W) {
  return guarded([&] {
    auto model = oracle::build_model(*desc);
    const int d = model.state_dim;
    for (int t = 0; t <= model.horizon; ++t)
      dsmc::leaf_weights(model, t, X + (size_t)t * n * d, n, W + (size_t)t * n);
  });
}

// make_leaf (smoother.cpp:98-130) for every time, multithreaded: states and
// raw leaf weights (T+1) x n (x d).
int ref_make_leaves_all(const dsmc_model_desc* desc, size_t n, uint64_t seed, int threads,
                        double* X, double* raw) {
  return guarded([&] {
    auto model = oracle::build_model(*desc);
    const int d = model.state_dim;
    par_for(model.horizon + 1, threads, [&](std::size_t t) {
      auto blk = dsmc::make_leaf(model, (int)t, n, seed);
      std::memcpy(X + t * n * d, blk.paths.data(), sizeof(double) * n * d);
      dsmc::leaf_weights(model, (int)t, blk.paths.data(), n, raw + t * n);
    });
  });
}

// conditional_leaf (conditional.cpp:52-87) for every time: (T+1) x n x d
// states, slot 0 = the reference path.
int ref_conditional_leaves_all(const dsmc_model_desc* desc, size_t n, uint64_t seed,
                               uint32_t sweep, const double* star, double* X) {
  return guarded([&] {
    auto model = oracle::build_model(*desc);
    const int d = model.state_dim;
    for (int t = 0; t <= model.horizon; ++t) {
      auto blk = dsmc::conditional_leaf(model, t, n, seed, sweep, star + (size_t)t * d);
      std::memcpy(X + (size_t)t * n * d, blk.paths.data(), sizeof(double) * n * d);
    }
  });
}

// gamma_draw (pgibbs.cpp:80-102) from stream {seed, level, node, role}.
int ref_gamma_draw(double shape, double rate, uint64_t seed, uint32_t level, uint64_t node,
                   int role, double* out) {
  return guarded([&] {
    dsmc::RngStream s(key_of(seed, level, node, role));
    *out = dsmc::gamma_draw(shape, rate, s);
  });
}

// The SV parameter kernel of the batched particle Gibbs (the
// reference has no SV model), on the reference's RngStream and gamma_draw:
// sigma2 | rest by the conjugate inverse gamma (gamma_draw of the precision),
// mu | rest normal, random-walk Metropolis on phi with a flat prior on
// (-1, 1); stream {seed, 0, sweep, gibbs_param} as pgibbs_sweep keys it
// (pgibbs.cpp:38). Pins the device kernel's draws (tests/test_gpu_pgibbs.py).
int ref_sv_param_update(const double* x, int T, const dsmc_sv_prior* pr, uint64_t seed,
                        uint32_t sweep, double* theta, int* accepted_phi) {
  return guarded([&] {
    auto lnp = [](double v, double m, double var) {
      const double d = v - m;
      return -0.5 * (1.8378770664093454836 + std::log(var)) - d * d / (2.0 * var);
    };
    auto loglik = [&](double mu, double phi, double s2) {
      double ll = lnp(x[0], mu, s2 / (1.0 - phi * phi));
      for (int t = 1; t <= T; ++t) ll += lnp(x[t], mu + phi * (x[t - 1] - mu), s2);
      return ll;
    };
    dsmc::RngStream s(key_of(seed, 0, sweep, DSMC_ROLE_GIBBS_PARAM));
    double mu = theta[0], phi = theta[1], s2 = theta[2];
    double ss = (1.0 - phi * phi) * (x[0] - mu) * (x[0] - mu);
    for (int t = 1; t <= T; ++t) {
      const double e = x[t] - mu - phi * (x[t - 1] - mu);
      ss += e * e;
    }
    const double prec =
        dsmc::gamma_draw(pr->s2_shape + 0.5 * (double)(T + 1), pr->s2_rate + 0.5 * ss, s);
    s2 = 1.0 / prec;
    const double p = 1.0 / pr->mu_var + (1.0 - phi * phi) / s2 +
                     (double)T * (1.0 - phi) * (1.0 - phi) / s2;
    double acc = 0.0;
    for (int t = 1; t <= T; ++t) acc += x[t] - phi * x[t - 1];
    const double h = pr->mu_mean / pr->mu_var + (1.0 - phi * phi) * x[0] / s2 +
                     (1.0 - phi) * acc / s2;
    mu = h / p + std::sqrt(1.0 / p) * s.normal();
    const double prop = phi + pr->phi_step * s.normal();
    const double lu = std::log(s.uniform_pos());
    int a = 0;
    if (std::fabs(prop) < 1.0) {
      const double dl = loglik(mu, prop, s2) - loglik(mu, phi, s2);
      if (lu < dl) {
        phi = prop;
        a = 1;
      }
    }
    theta[0] = mu;
    theta[1] = phi;
    theta[2] = s2;
    if (accepted_phi) *accepted_phi = a;
  });
}

// run_conditional (conditional.cpp:156-216) unchanged.
int ref_run_conditional(const dsmc_model_desc* desc, const double* ref,
                        size_t n, int resampler, uint64_t seed, uint32_t sweep,
                        double* out_path, double* lnc, int* has_lnc,
                        uint64_t* evals) {
  return guarded([&] {
    auto model = oracle::build_model(*desc);
    dsmc::ConditionalOptions o;
    o.n_particles = n;
    o.resampler = static_cast<dsmc::Resampler>(resampler);
    o.seed = seed;
    auto res = dsmc::run_conditional(model, ref, o, sweep);
    std::memcpy(out_path, res.path.data(), sizeof(double) * res.path.size());
    *has_lnc = res.meta.log_norm_const.has_value() ? 1 : 0;
    *lnc = res.meta.log_norm_const.value_or(NAN);
    *evals = res.meta.weight_evals;
  });
}

// conditional_leaf (conditional.cpp:52-87): states incl. the reference.
int ref_conditional_leaf(const dsmc_model_desc* desc, int t, size_t n,
                         uint64_t seed, uint32_t sweep, const double* star,
                         double* x, double* raw_lw) {
  return guarded([&] {
    auto model = oracle::build_model(*desc);
    auto blk = dsmc::conditional_leaf(model, t, n, seed, sweep, star);
    std::memcpy(x, blk.paths.data(), sizeof(double) * blk.paths.size());
    dsmc::leaf_weights(model, t, blk.paths.data(), n, raw_lw);
  });
}

}  // extern "C"

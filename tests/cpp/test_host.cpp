// C++ host API tests, written like the reference's doctest cases (the
// reference's test names are kept in the CASE titles; file:line cites the
// case each one ports). Runs on the GPU through include/dsmc/dsmc.hpp.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "dsmc/dsmc.hpp"

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                      \
  do {                                                                   \
    ++g_checks;                                                          \
    if (!(cond)) {                                                       \
      ++g_fail;                                                          \
      std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                    \
  } while (0)
#define CHECK_THROWS_AS(expr, exc)                                       \
  do {                                                                   \
    ++g_checks;                                                          \
    bool ok = false;                                                     \
    try {                                                                \
      expr;                                                              \
    } catch (const exc&) {                                               \
      ok = true;                                                         \
    } catch (...) {                                                      \
    }                                                                    \
    if (!ok) {                                                           \
      ++g_fail;                                                          \
      std::printf("  CHECK_THROWS_AS failed %s:%d: %s\n", __FILE__, __LINE__, #expr); \
    }                                                                    \
  } while (0)

struct Case {
  const char* name;
  std::function<void()> fn;
};
static std::vector<Case>& cases() {
  static std::vector<Case> v;
  return v;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { cases().push_back({n, std::move(f)}); }
};
#define TEST_CASE(name) \
  static void name##_fn(); \
  static Reg name##_reg(#name, name##_fn); \
  static void name##_fn()

namespace {

// tests/support/ar1.hpp:23-126: stationary AR(1), Gaussian observations
dsmc::LinearGaussianModel ar1_exact(const std::vector<double>& ys, double rho = 0.8,
                                    double q = 0.3, double r = 0.4) {
  const int T = (int)ys.size() - 1;
  dsmc::LinearGaussianModel m;
  m.horizon = T;
  const double s2 = q / (1 - rho * rho);
  m.m0 = {0.0};
  m.P0 = {s2};
  for (int t = 0; t <= T; ++t) {
    m.F.push_back({rho});
    m.b.push_back({0.0});
    m.Q.push_back({q});
    m.H.push_back({1.0});
    m.R.push_back({r});
    m.y.push_back({ys[t]});
    m.has_obs.push_back(1);
  }
  return m;
}

std::vector<double> default_ys(int T) {
  const double pool[] = {0.4, -0.1, 0.9, 1.3, 0.2, -0.7, -0.2, 0.5, 1.1, 0.3, -0.4, 0.1,
                         0.8, -0.9, 0.0, 0.6, -0.3, 0.7, 1.0, -0.5, 0.2, -0.8, 0.35, 0.15};
  std::vector<double> ys(T + 1);
  for (int t = 0; t <= T; ++t) ys[t] = pool[t % 24];
  return ys;
}

dsmc::FeynmanKacModel ar1_fk(int T) {
  auto lg = ar1_exact(default_ys(T));
  const double s2 = 0.3 / (1 - 0.64);
  std::vector<dsmc::ProposalMarginal> marg(T + 1, {{0.0}, {s2}});
  return dsmc::make_lgssm_fk(lg, marg);
}

}  // namespace

// test_smoother.cpp:195-227
TEST_CASE(combine_schedule_packed_pairing_clipped_blocks_log_depth) {
  for (int T : {0, 1, 2, 5, 6, 11, 100}) {
    auto s = dsmc::build_schedule(T);
    CHECK((int)s.pairs.size() == T);
    CHECK(s.levels == dsmc::reference_tree_depth(T));
    CHECK(s.levels == (T == 0 ? 0 : (int)std::ceil(std::log2(T + 1.0))));
  }
  auto s = dsmc::build_schedule(5);
  CHECK(s.pairs[2].level == 1 && s.pairs[2].left_a == 4 && s.pairs[2].right_b == 5);
  CHECK(s.pairs.back().left_a == 0 && s.pairs.back().right_b == 5);
}

// test_smoother.cpp:292-316: means and evidence vs the exact answers
TEST_CASE(smoothed_means_and_evidence_match_the_exact_Kalman_answers) {
  const int T = 11;
  auto lg = ar1_exact(default_ys(T));
  auto kr = dsmc::kalman_smooth(lg);
  auto model = ar1_fk(T);
  const int reps = 16;
  std::vector<double> mean_sum(T + 1, 0.0), mean_sq(T + 1, 0.0);
  double lz_sum = 0, lz_sq = 0;
  for (int s = 0; s < reps; ++s) {
    dsmc::SmootherOptions o;
    o.n_particles = 1500;
    o.seed = 100 + s;
    auto res = dsmc::run_smoother(model, o);
    for (int t = 0; t <= T; ++t) {
      const double m = dsmc::weighted_time_mean(res.root, t)[0];
      mean_sum[t] += m;
      mean_sq[t] += m * m;
    }
    lz_sum += *res.meta.log_norm_const;
    lz_sq += *res.meta.log_norm_const * *res.meta.log_norm_const;
  }
  for (int t = 0; t <= T; ++t) {
    const double mu = mean_sum[t] / reps;
    const double se = std::sqrt(std::max(mean_sq[t] / reps - mu * mu, 1e-12) / (reps - 1));
    CHECK(std::fabs(mu - kr.smooth_mean[t][0]) < 5 * se + 1e-3);
  }
  const double lz = lz_sum / reps;
  const double lse = std::sqrt(std::max(lz_sq / reps - lz * lz, 1e-12) / (reps - 1));
  CHECK(std::fabs(lz - kr.log_likelihood) < 5 * lse + 0.05);
}

// test_smoother.cpp:343-385
TEST_CASE(runs_are_deterministic_and_precision_invariant_in_structure) {
  auto model = ar1_fk(30);
  dsmc::SmootherOptions o;
  o.n_particles = 200;
  o.seed = 7;
  auto a = dsmc::run_smoother(model, o);
  auto b = dsmc::run_smoother(model, o);
  CHECK(a.root.paths == b.root.paths);
  CHECK(*a.meta.log_norm_const == *b.meta.log_norm_const);
  o.precision = dsmc::Precision::fp64_parity;
  auto c = dsmc::run_smoother(model, o);
  auto d = dsmc::run_smoother(model, o);
  CHECK(c.root.paths == d.root.paths);
  CHECK(c.meta.weight_evals == 30ull * 200 * 200);  // T * N^2 (test_smoother.cpp:382)
  CHECK(c.meta.levels == 5);
}

// test_smoother.cpp:387-414
TEST_CASE(MH_chain_stitching_zero_steps_keeps_identity_pairs_and_is_flagged) {
  auto model = ar1_fk(7);
  dsmc::SmootherOptions o;
  o.n_particles = 16;
  o.resampler = dsmc::Resampler::mh_lazy;
  o.mh_steps = 0;
  auto res = dsmc::run_smoother(model, o);
  CHECK(res.meta.biased);
  CHECK(res.meta.weight_evals == 0);
  CHECK(!res.meta.log_norm_const.has_value());
}

// test_smoother.cpp:416-434
TEST_CASE(rejection_stitching_matches_the_dense_smoother_statistically) {
  auto model = ar1_fk(11);
  dsmc::SmootherOptions o;
  o.n_particles = 2000;
  o.resampler = dsmc::Resampler::rejection_lazy;
  auto res = dsmc::run_smoother(model, o);
  auto kr = dsmc::kalman_smooth(ar1_exact(default_ys(11)));
  for (int t = 0; t <= 11; ++t)
    CHECK(std::fabs(dsmc::weighted_time_mean(res.root, t)[0] - kr.smooth_mean[t][0]) < 0.15);
  CHECK(!res.meta.biased);
}

// test_smoother.cpp:502-527
TEST_CASE(single_time_models_skip_combining_entirely) {
  auto model = ar1_fk(0);
  dsmc::SmootherOptions o;
  o.n_particles = 64;
  auto res = dsmc::run_smoother(model, o);
  CHECK(res.meta.levels == 0);
  CHECK(res.meta.weight_evals == 0);
  CHECK(res.root.len() == 1);
}

// test_models.cpp / test_smoother.cpp:416-456: the reference's own models
TEST_CASE(cox_and_constrained_walk_models_run_through_the_reference_api) {
  std::vector<double> ys = {0, 1, 3, 2, 0, 1, 4, 2, 1, 0, 0, 2, 3, 1, 1, 0};
  dsmc::CoxParams cp;
  auto cox = dsmc::make_cox_model(cp, ys);
  CHECK(cox.horizon == 15);
  dsmc::SmootherOptions o;
  o.n_particles = 256;
  o.seed = 3;
  auto r = dsmc::run_smoother(cox, o);
  CHECK(r.meta.log_norm_const.has_value());
  CHECK(std::isfinite(*r.meta.log_norm_const));
  CHECK(r.meta.weight_evals == 15ull * 256 * 256);
  CHECK_THROWS_AS(dsmc::make_cox_model(cp, {}), std::invalid_argument);
  auto bad = dsmc::make_cox_model(cp, {0.5, 1.0});  // non-integer count
  CHECK_THROWS_AS(dsmc::run_smoother(bad, o), std::invalid_argument);
  // constrained walk: rejection stitching is available (finite bound) and
  // every smoothed state stays in the box
  auto rw = dsmc::make_constrained_rw(0.3, 20);
  o.resampler = dsmc::Resampler::rejection_lazy;
  auto rr = dsmc::run_smoother(rw, o);
  CHECK(!rr.meta.log_norm_const.has_value());
  for (int t = 0; t <= 20; ++t) CHECK(std::fabs(dsmc::weighted_time_mean(rr.root, t)[0]) <= 1.0);
  o.precision = dsmc::Precision::fp64_parity;
  o.resampler = dsmc::Resampler::multinomial;
  auto r64 = dsmc::run_smoother(rw, o);
  CHECK(std::isfinite(*r64.meta.log_norm_const));
  // theta-logistic with flat-ish marginals around the observations
  std::vector<double> ty(21);
  std::vector<dsmc::ProposalMarginal> mg(21);
  for (int t = 0; t <= 20; ++t) {
    ty[t] = 0.3 * std::sin(0.3 * t);
    mg[t].mean = {ty[t]};
    mg[t].cov = {0.2};
  }
  auto th = dsmc::make_theta_logistic(dsmc::ThetaLogisticParams{}, ty, mg);
  o.precision = dsmc::Precision::fp32;
  auto rt = dsmc::run_smoother(th, o);
  CHECK(std::isfinite(*rt.meta.log_norm_const));
  for (int t = 0; t <= 20; ++t)
    CHECK(std::fabs(dsmc::weighted_time_mean(rt.root, t)[0] - ty[t]) < 0.5);
  CHECK_THROWS_AS(dsmc::make_theta_logistic(dsmc::ThetaLogisticParams{}, ty, {}),
                  std::invalid_argument);
}

TEST_CASE(models_without_a_device_descriptor_are_rejected) {
  dsmc::FeynmanKacModel m;
  m.horizon = 3;
  CHECK_THROWS_AS(dsmc::run_smoother(m, dsmc::SmootherOptions{}), std::invalid_argument);
}

// test_resampling.cpp:65-89
TEST_CASE(multinomial_frequencies_and_log_total_match_an_independent_normalization) {
  const std::vector<double> logw = {0.3, -1.2, 0.8, -0.4, 1.5, -2.0, 0.0, 0.7, -0.9};
  long double mx = -INFINITY, tot = 0;
  for (double v : logw) mx = std::max<long double>(mx, v);
  for (double v : logw) tot += std::exp((long double)v - mx);
  const std::size_t n_out = 60000;
  auto ps = dsmc::resample_pairs(dsmc::Resampler::multinomial, logw, 3, n_out, 0,
                                 {11, 2, 5, dsmc::StreamRole::pair_resample});
  CHECK(std::fabs(*ps.log_mean_weight - (double)(mx + std::log(tot))) < 1e-12);
  CHECK(ps.weight_evals == 9);
  std::vector<double> cnt(9, 0);
  for (std::size_t k = 0; k < n_out; ++k) cnt[ps.left[k] * 3 + ps.right[k]] += 1;
  for (int k = 0; k < 9; ++k) {
    const double p = (double)(std::exp((long double)logw[k] - mx) / tot);
    CHECK(std::fabs(cnt[k] - n_out * p) <= 5 * std::sqrt(n_out * p * (1 - p)) + 1);
  }
  CHECK_THROWS_AS(dsmc::resample_pairs(dsmc::Resampler::multinomial,
                                       std::vector<double>(25, -INFINITY), 5, 10, 0, {}),
                  std::runtime_error);
}

// test_conditional.cpp:317-329
TEST_CASE(ordered_and_biased_resamplers_are_rejected_at_configuration) {
  auto model = ar1_fk(5);
  std::vector<double> ref(6, 0.1);
  dsmc::ConditionalOptions o;
  o.n_particles = 8;
  o.resampler = dsmc::Resampler::systematic;
  CHECK_THROWS_AS(dsmc::run_conditional(model, ref.data(), o, 0), std::invalid_argument);
  o.resampler = dsmc::Resampler::mh_lazy;
  CHECK_THROWS_AS(dsmc::run_conditional(model, ref.data(), o, 0), std::invalid_argument);
}

// test_conditional.cpp:360-391
TEST_CASE(sweeps_are_deterministic_and_keyed_by_seed_and_sweep_index) {
  auto model = ar1_fk(9);
  std::vector<double> ref(10, 0.2);
  dsmc::ConditionalOptions o;
  o.n_particles = 64;
  o.seed = 5;
  auto a = dsmc::run_conditional(model, ref.data(), o, 3);
  auto b = dsmc::run_conditional(model, ref.data(), o, 3);
  auto c = dsmc::run_conditional(model, ref.data(), o, 4);
  CHECK(a.path == b.path);
  CHECK(a.path != c.path);
  CHECK(a.meta.weight_evals == 9ull * (64 * 64 + 1));  // test_conditional.cpp:188
}

// test_pgibbs.cpp:160-202
TEST_CASE(pgibbs_sweep_aborts_cleanly_when_a_kernel_or_builder_throws) {
  dsmc::GibbsState st;
  st.theta = {1.0};
  st.star.assign(8, 0.1);
  const auto saved = st;
  auto bad_kernel = [](dsmc::GibbsState&, dsmc::RngStream&) {
    throw std::runtime_error("kernel failed");
  };
  auto builder = [](dsmc::GibbsState&) { return ar1_fk(7); };
  dsmc::ConditionalOptions o;
  o.n_particles = 16;
  CHECK_THROWS_AS(dsmc::pgibbs_sweep(st, builder, bad_kernel, o, 0), std::runtime_error);
  CHECK(st.star == saved.star && st.theta == saved.theta);
  auto id_kernel = [](dsmc::GibbsState&, dsmc::RngStream&) {};
  auto out = dsmc::pgibbs_sweep(st, builder, id_kernel, o, 1);
  CHECK(out.state.star.size() == 8);
  CHECK(out.changed.size() == 8);
  CHECK(st.star == saved.star);
}

TEST_CASE(batched_sv_particle_gibbs_moves_parameters_and_paths) {
  const int T = 63, B = 4;
  std::vector<double> ys(T + 1);
  for (int t = 0; t <= T; ++t) ys[t] = std::exp(-0.5) * ((t % 3) ? 1.0 : -1.3);
  dsmc::SvGibbsChains ch;
  ch.theta.assign(B * 3, 0.0);
  for (int c = 0; c < B; ++c) {
    ch.theta[3 * c] = -1.0;
    ch.theta[3 * c + 1] = 0.9;
    ch.theta[3 * c + 2] = 0.1;
    ch.seeds.push_back(1000 + c);
  }
  ch.stars.assign((size_t)B * (T + 1), -1.0);
  dsmc_sv_prior prior{-1.0, 1.0, 2.0, 0.2, 0.05};
  dsmc::ConditionalOptions o;
  o.n_particles = 128;
  const auto theta0 = ch.theta;
  std::size_t moved = 0;
  for (std::uint32_t s = 0; s < 5; ++s) {
    auto changed = dsmc::sv_pgibbs_sweep(ch, ys, prior, o, s);
    for (char v : changed) moved += v;
  }
  CHECK(ch.theta != theta0);
  CHECK(moved > (std::size_t)(B * (T + 1)));
  for (double v : ch.stars) CHECK(std::isfinite(v));
}

// ---------------------------------------------------------------------------
// Host-only cases (no GPU): run with `test_host cpu_`.

// test_rng.cpp:32-47: Philox4x64-10 known-answer vectors
TEST_CASE(cpu_philox4x64_10_known_answer_vectors) {
  const auto z = dsmc::rng_detail::philox4x64_10({0, 0, 0, 0}, {0, 0});
  CHECK(z[0] == 0x16554d9eca36314cull);
  CHECK(z[1] == 0xdb20fe9d672d0fdcull);
  CHECK(z[2] == 0xd7e772cee186176bull);
  CHECK(z[3] == 0x7e68b68aec7ba23bull);
  const auto w = dsmc::rng_detail::philox4x64_10(
      {0xdeadbeefull, 1, 2, 3}, {0x9E3779B97F4A7C15ull, 0x243F6A8885A308D3ull});
  CHECK(w[0] == 0x89aa73bbe8e9ebdbull);
  CHECK(w[1] == 0x42065f627a6e7ccfull);
  CHECK(w[2] == 0xf103ff19821da020ull);
  CHECK(w[3] == 0x0cf1b816fdc3eb80ull);
}

// test_rng.cpp:49-80: identical keys give identical streams, distinct
// substreams and roles differ, uniforms stay in range
TEST_CASE(cpu_streams_are_keyed_and_in_range) {
  const dsmc::StreamKey key{42, 3, 17, dsmc::StreamRole::pair_resample};
  dsmc::RngStream a(key), b(key), c(key, 1);
  dsmc::StreamKey k2 = key;
  k2.role = dsmc::StreamRole::leaf_proposal;
  dsmc::RngStream d(k2);
  int same_c = 0, same_d = 0;
  for (int i = 0; i < 64; ++i) {
    const std::uint64_t x = a.next_u64();
    CHECK(x == b.next_u64());
    same_c += x == c.next_u64();
    same_d += x == d.next_u64();
  }
  CHECK(same_c == 0 && same_d == 0);
  dsmc::RngStream u({7, 0, 0, dsmc::StreamRole::data_sim});
  double lo = 1, hi = 0, s = 0, s2 = 0;
  for (int i = 0; i < 20000; ++i) {
    const double x = u.uniform_pos();
    lo = std::min(lo, x);
    hi = std::max(hi, x);
    const double z = u.normal();
    s += z;
    s2 += z * z;
  }
  CHECK(lo > 0.0 && hi < 1.0);
  CHECK(std::fabs(s / 20000) < 0.05 && std::fabs(s2 / 20000 - 1.0) < 0.05);
  for (int i = 0; i < 1000; ++i) CHECK(u.uniform_index(7) < 7);
}

// Data simulation follows the reference's streams: values pinned by
// tests/golden/make_harness_golden.py (reference Philox, restated simulators)
TEST_CASE(cpu_simulated_data_matches_the_reference_streams) {
  const auto cox = dsmc::simulate_cox(dsmc::CoxParams{}, 15, 90210);
  const std::vector<double> want = {4, 3, 6, 6, 11, 3, 6, 1, 5, 2, 0, 0, 0, 1, 0, 1};
  CHECK(cox.ys == want);
  dsmc::LinearGaussianModel m;
  m.horizon = 31;
  m.m0 = {0.0};
  m.P0 = {1.0};
  m.F.assign(32, {0.9});
  m.b.assign(32, {0.0});
  m.Q.assign(32, {0.25});
  m.H.assign(32, {1.0});
  m.R.assign(32, {0.25});
  m.y.assign(32, {0.0});
  m.has_obs.assign(32, 1);
  dsmc::RngStream st({90210, 0, 0, dsmc::StreamRole::data_sim});
  const auto s = dsmc::simulate_lgssm(m, st);
  CHECK(s.y[0][0] == 1.5863467310809578);
  CHECK(s.y[1][0] == 1.0690823364517432);
  CHECK(s.y[2][0] == -0.16730312329906827);
  CHECK(s.y[3][0] == 1.8049285543505404);
  const auto th = dsmc::simulate_theta_logistic(dsmc::ThetaLogisticParams{}, 40, 5);
  CHECK(th.ys.size() == 41);
  CHECK_THROWS_AS(dsmc::simulate_cox(dsmc::CoxParams{0, 0.9, -1, 1}, 3, 1), std::invalid_argument);
}

// pgibbs.cpp:80-102: gamma draws have mean shape / rate (both branches)
TEST_CASE(cpu_gamma_draw_moments) {
  dsmc::RngStream st({11, 0, 0, dsmc::StreamRole::gibbs_param});
  for (double shape : {0.5, 3.0}) {
    double acc = 0.0;
    const int n = 40000;
    for (int i = 0; i < n; ++i) acc += dsmc::gamma_draw(shape, 2.0, st);
    const double m = acc / n, sd = std::sqrt(shape) / 2.0 / std::sqrt((double)n);
    CHECK(std::fabs(m - shape / 2.0) < 5 * sd);
  }
  CHECK_THROWS_AS(dsmc::gamma_draw(0.0, 1.0, st), std::invalid_argument);
}

// kalman.cpp:192-243: linear dynamics linearise exactly, so one IEKS
// iteration equals the Kalman/RTS smoother; the theta-logistic IEKS
// converges (fixed point of the reference trajectory)
TEST_CASE(cpu_iterated_smoother) {
  const int T = 30;
  dsmc::NonlinearGaussianModel nl;
  nl.horizon = T;
  nl.m0 = {0.0};
  nl.P0 = {1.0};
  nl.f = [](int, const std::vector<double>& x) { return std::vector<double>{0.8 * x[0] + 0.1}; };
  nl.Q.assign(T + 1, {0.3});
  nl.H.assign(T + 1, {1.0});
  nl.R.assign(T + 1, {0.4});
  nl.y.resize(T + 1);
  for (int t = 0; t <= T; ++t) nl.y[t] = {std::sin(0.3 * t)};
  nl.has_obs.assign(T + 1, 1);
  const auto it = dsmc::iterated_smooth(nl, 1);
  dsmc::LinearGaussianModel lin = it.linearized;
  for (int t = 1; t <= T; ++t) {
    CHECK(std::fabs(lin.F[t][0] - 0.8) < 1e-8);  // central differences
    CHECK(std::fabs(lin.b[t][0] - 0.1) < 1e-8);
  }
  std::vector<double> ys(T + 1);
  for (int t = 0; t <= T; ++t) ys[t] = 0.5 + 0.1 * std::cos(0.2 * t);
  const auto th = dsmc::theta_logistic_nonlinear(dsmc::ThetaLogisticParams{}, ys);
  const auto a = dsmc::iterated_smooth(th, 25);
  const auto b = dsmc::iterated_smooth(th, 1, &a.ref);
  double diff = 0.0;
  for (int t = 0; t <= T; ++t) diff = std::max(diff, std::fabs(a.ref[t][0] - b.ref[t][0]));
  CHECK(diff < 1e-9);
  CHECK(a.iterations == 25 && b.iterations == 1);
}

TEST_CASE(cpu_scores_match_their_definitions) {
  const double path[3] = {0.1, -0.2, 0.4};
  const dsmc::CoxParams p{};
  const double s2 = p.sigma2;
  double want = -3 / (2 * s2) + (1 - p.rho * p.rho) / (2 * s2 * s2) * 0.01;
  const double e1 = -0.2 - 0.9 * 0.1, e2 = 0.4 - 0.9 * -0.2;
  want += e1 * e1 / (2 * s2 * s2) + e2 * e2 / (2 * s2 * s2);
  CHECK(std::fabs(dsmc::cox_score(p, path, 2) - want) < 1e-12);
  CHECK(std::fabs(dsmc::rw_score(0.5, path, 2) - (std::log(0.5) + (0.09 + 0.36) / 0.125)) < 1e-12);
}

// pgibbs.hpp:83-87 / test_pgibbs.cpp:62-110: conjugate precision draws on a
// hand trajectory follow Gamma(shape + T/2, rate + ss/2) (moment checks)
TEST_CASE(cpu_draw_precisions_conjugate_law) {
  dsmc::ThetaLogisticParams p{0.2, 0.1, 0.5, 1.0, 1.0};
  const std::vector<double> star = {0.0, 0.4, -0.2}, ys = {0.1, 0.3, -0.4};
  dsmc::ThetaLogisticGibbsConfig cfg;
  cfg.prec_x_shape = 2.0;
  cfg.prec_x_rate = 1.0;
  cfg.prec_y_shape = 3.0;
  cfg.prec_y_rate = 0.5;
  auto f = [](double x) { return x + 0.2 - 0.1 * std::exp(0.5 * x); };
  const double ssx = (0.4 - f(0.0)) * (0.4 - f(0.0)) + (-0.2 - f(0.4)) * (-0.2 - f(0.4));
  const double ssy = 0.01 + 0.01 + 0.04;
  const double ax = 2.0 + 1.0, bx = 1.0 + 0.5 * ssx, ay = 3.0 + 1.5, by = 0.5 + 0.5 * ssy;
  dsmc::RngStream st({11, 0, 0, dsmc::StreamRole::gibbs_param});
  const int n = 40000;
  double sx = 0, sxx = 0, sy = 0;
  for (int k = 0; k < n; ++k) {
    const auto d = dsmc::draw_precisions(p, ys, star, cfg, st);
    CHECK(d.tau0 == p.tau0 && d.tau1 == p.tau1 && d.tau2 == p.tau2);
    sx += 1.0 / d.q2;
    sxx += 1.0 / (d.q2 * d.q2);
    sy += 1.0 / d.r2;
  }
  const double mx = sx / n, vx = sxx / n - mx * mx, my = sy / n;
  CHECK(std::fabs(mx - ax / bx) < 5 * std::sqrt(ax) / bx / std::sqrt((double)n));
  CHECK(std::fabs(vx - ax / (bx * bx)) < 0.05 * ax / (bx * bx));
  CHECK(std::fabs(my - ay / by) < 5 * std::sqrt(ay) / by / std::sqrt((double)n));
  CHECK_THROWS_AS(dsmc::draw_precisions(p, ys, {0.0, 1.0}, cfg, st), std::invalid_argument);
}

// test_pgibbs.cpp:204-258: the theta-logistic chain (host parameter kernel,
// device c-dSMC) is deterministic in its seed, keeps the support, renews the
// path at a healthy rate and guards its inputs
TEST_CASE(theta_logistic_chain_determinism_support_mixing) {
  dsmc::ThetaLogisticParams truth{0.15, 0.10, 0.50, 0.09, 0.04};
  const auto data = dsmc::simulate_theta_logistic(truth, 40, 2024);
  dsmc::ThetaLogisticGibbsConfig cfg;
  cfg.n_particles = 32;
  const auto chain = dsmc::run_theta_logistic_pgibbs(data.ys, truth, cfg, 60, 5);
  CHECK(chain.thetas.size() == 60 && chain.stars.size() == 60);
  for (const auto& th : chain.thetas)
    CHECK(std::isfinite(th.tau0) && th.tau1 > 0 && th.tau2 > 0 && th.q2 > 0 && th.r2 > 0);
  CHECK(chain.weight_evals > 0);
  const auto rates = dsmc::update_rate(chain.stars);
  double mean_rate = 0;
  for (double r : rates) mean_rate += r;
  CHECK(mean_rate / rates.size() > 0.3);
  CHECK(chain.thetas[5].q2 != chain.thetas[6].q2);
  const auto again = dsmc::run_theta_logistic_pgibbs(data.ys, truth, cfg, 60, 5);
  CHECK(again.thetas.back().q2 == chain.thetas.back().q2);
  CHECK(again.stars.back() == chain.stars.back());
  CHECK(again.rwm_accepts == chain.rwm_accepts);
  const auto other = dsmc::run_theta_logistic_pgibbs(data.ys, truth, cfg, 60, 6);
  CHECK(other.stars.back() != chain.stars.back());
  dsmc::ThetaLogisticParams bad = truth;
  bad.tau1 = -0.1;
  CHECK_THROWS_AS(dsmc::run_theta_logistic_pgibbs(data.ys, bad, cfg, 3, 1), std::invalid_argument);
  CHECK_THROWS_AS(dsmc::run_theta_logistic_pgibbs({1.0}, truth, cfg, 3, 1), std::invalid_argument);
}

// test_pgibbs.cpp:260-289: with the taus frozen the chain is Gibbs over
// (path, q2, r2). The reference checks doctest::Approx(truth).epsilon(0.5),
// i.e. |a - b| < 0.5 (1 + max(|a|, |b|)); on this data set the exact posterior
// means are q2 = 0.176, r2 = 0.151 (a Gibbs sampler with exact Kalman/FFBS
// path draws, 3500 iterations, same priors — computed when this case was
// written), and the particle-Gibbs chain must land within 15% of those
TEST_CASE(theta_logistic_conjugate_only_chain_recovers_precisions) {
  dsmc::ThetaLogisticParams truth{0.1, 1e-8, 1e-8, 0.25, 0.09};
  const auto data = dsmc::simulate_theta_logistic(truth, 150, 99);
  dsmc::ThetaLogisticGibbsConfig cfg;
  cfg.n_particles = 48;
  cfg.rwm_step_tau = 0.0;
  cfg.rwm_step_x0 = 0.0;
  const auto chain = dsmc::run_theta_logistic_pgibbs(data.ys, truth, cfg, 300, 17);
  double mq = 0, mr = 0;
  const std::size_t burn = 50;
  for (std::size_t k = burn; k < chain.thetas.size(); ++k) {
    mq += chain.thetas[k].q2;
    mr += chain.thetas[k].r2;
  }
  mq /= (double)(chain.thetas.size() - burn);
  mr /= (double)(chain.thetas.size() - burn);
  auto approx = [](double a, double b) {  // doctest::Approx(b).epsilon(0.5)
    return std::fabs(a - b) < 0.5 * (1.0 + std::max(std::fabs(a), std::fabs(b)));
  };
  CHECK(approx(mq, truth.q2));
  CHECK(approx(mr, truth.r2));
  CHECK(std::fabs(mq - 0.1757) < 0.15 * 0.1757);
  CHECK(std::fabs(mr - 0.1514) < 0.15 * 0.1514);
}

// smoother.hpp:98-125: the piecewise API (make_leaf + combine_blocks in the
// packed schedule, smoother.cpp:236-262) on the device reproduces
// run_smoother's FP64 parity run bit for bit: same leaves, same stitches,
// same root paths, evals and bias; log Z to rounding.
static void piecewise_matches(const dsmc::FeynmanKacModel& model, std::size_t n,
                              dsmc::Resampler rs) {
  dsmc::SmootherOptions o;
  o.n_particles = n;
  o.resampler = rs;
  o.mh_steps = 5;
  o.seed = 4242;
  o.precision = dsmc::Precision::fp64_parity;
  auto ref = dsmc::run_smoother(model, o);
  const int T = model.horizon;
  std::vector<dsmc::BlockEstimate> cur;
  for (int t = 0; t <= T; ++t) cur.push_back(dsmc::make_leaf(model, t, n, o.seed));
  int level = 0;
  while (cur.size() > 1) {
    ++level;
    std::vector<dsmc::BlockEstimate> next;
    for (std::size_t k = 0; k + 1 < cur.size(); k += 2)
      next.push_back(dsmc::combine_blocks(model, cur[k], cur[k + 1], o, level, (int)(k / 2)));
    if (cur.size() % 2) next.push_back(cur.back());
    cur.swap(next);
  }
  const auto& root = cur.front();
  CHECK(level == ref.meta.levels);
  CHECK(root.paths == ref.root.paths);
  CHECK(root.weight_evals == ref.meta.weight_evals);
  CHECK(root.biased == ref.meta.biased);
  CHECK(root.log_norm_const.has_value() == ref.meta.log_norm_const.has_value());
  if (root.log_norm_const && ref.meta.log_norm_const)
    CHECK(std::fabs(*root.log_norm_const - *ref.meta.log_norm_const) <=
          1e-12 * std::max(1.0, std::fabs(*ref.meta.log_norm_const)));
}

TEST_CASE(piecewise_make_leaf_and_combine_blocks_reproduce_run_smoother) {
  piecewise_matches(ar1_fk(21), 37, dsmc::Resampler::multinomial);
  piecewise_matches(ar1_fk(9), 24, dsmc::Resampler::systematic);
  piecewise_matches(ar1_fk(12), 30, dsmc::Resampler::mh_lazy);
  piecewise_matches(ar1_fk(10), 20, dsmc::Resampler::rejection_lazy);
  std::vector<double> ys(16);
  for (int t = 0; t < 16; ++t) ys[t] = 0.3 + 0.1 * ((t * 7) % 5);
  piecewise_matches(dsmc::make_sv_model({-1.0, 0.9, 0.1}, ys), 40, dsmc::Resampler::mh_lazy);
}

// make_leaf (smoother.cpp:98-130): uniform iff min == max raw weight; the
// log normalising constant is the leaf's mean raw weight; weights normalised
TEST_CASE(make_leaf_normalises_and_flags_uniform_leaves) {
  auto model = ar1_fk(5);
  auto l0 = dsmc::make_leaf(model, 0, 50, 9);
  auto l3 = dsmc::make_leaf(model, 3, 50, 9);
  CHECK(!l0.weights_uniform);  // h0 * P0 / q0 varies
  CHECK(l3.weights_uniform);   // nu = q at t >= 1
  double lse = -INFINITY;
  for (double v : l0.log_w) lse = std::max(lse, v);
  double acc = 0;
  for (double v : l0.log_w) acc += std::exp(v - lse);
  CHECK(std::fabs(lse + std::log(acc)) < 1e-12);
  CHECK(l0.a == 0 && l0.b == 0 && l0.n == 50 && l0.paths.size() == 50);
  std::vector<double> raw(50);
  dsmc::leaf_weights(model, 0, l0.paths.data(), 50, raw.data());
  double m = -INFINITY;
  for (double v : raw) m = std::max(m, v);
  double s = 0;
  for (double v : raw) s += std::exp(v - m);
  CHECK(std::fabs(*l0.log_norm_const - (m + std::log(s) - std::log(50.0))) < 1e-9);
  CHECK_THROWS_AS(dsmc::make_leaf(model, 6, 50, 9), std::invalid_argument);
  CHECK_THROWS_AS(dsmc::make_leaf(model, 0, 0, 9), std::invalid_argument);
}

// make_pair_source (smoother.cpp:132-180): host closures over the callbacks,
// the adjacency / size checks, log_shift and the rejection bound
TEST_CASE(make_pair_source_closures_shift_and_bound) {
  auto model = ar1_fk(7);
  auto a = dsmc::make_leaf(model, 0, 16, 3), b = dsmc::make_leaf(model, 1, 16, 3);
  auto c = dsmc::make_leaf(model, 2, 16, 3);
  auto bundle = dsmc::make_pair_source(model, a, b);
  CHECK(bundle.source.n == 16 && bundle.source.blocks != nullptr);
  CHECK(std::fabs(bundle.log_shift + std::log(16.0)) < 1e-15);  // only b is uniform
  std::vector<double> row(16);
  bundle.source.fill_row(3, row.data());
  for (std::size_t j = 0; j < 16; ++j)
    CHECK(std::fabs(row[j] - bundle.source.log_weight_at(3, j)) < 1e-12);
  CHECK_THROWS_AS(dsmc::make_pair_source(model, a, c), std::invalid_argument);
  auto d = dsmc::make_leaf(model, 1, 8, 3);
  CHECK_THROWS_AS(dsmc::make_pair_source(model, a, d), std::invalid_argument);
  // the device samples the attached blocks; a host copy without the
  // attachment samples the host-filled table: same law (log mean weight)
  auto ps = dsmc::resample_pairs(dsmc::Resampler::multinomial, bundle.source, 16, 0,
                                 {5, 1, 0, dsmc::StreamRole::pair_resample});
  auto host = bundle.source;
  host.blocks.reset();
  auto ph = dsmc::resample_pairs(dsmc::Resampler::multinomial, host, 16, 0,
                                 {5, 1, 0, dsmc::StreamRole::pair_resample});
  CHECK(ps.log_mean_weight && ph.log_mean_weight);
  CHECK(std::fabs(*ps.log_mean_weight - *ph.log_mean_weight) < 1e-9);
}

// test_smoother.cpp:416-433 + metrics.hpp: rejection stitching builds no
// dense table, has no evidence estimate; dense stitching counts one N x N
// table per combine
TEST_CASE(rejection_stitching_does_no_dense_allocs) {
  auto model = ar1_fk(11);
  dsmc::metrics::reset();
  dsmc::SmootherOptions o;
  o.n_particles = 400;
  o.resampler = dsmc::Resampler::rejection_lazy;
  for (int r = 0; r < 3; ++r) {
    o.seed = 700 + r;
    auto res = dsmc::run_smoother(model, o);
    CHECK(!res.meta.log_norm_const.has_value());
  }
  auto snap = dsmc::metrics::snapshot();
  CHECK(snap.dense_allocs == 0);
  CHECK(snap.weight_evals > 0);
  CHECK(snap.lazy_max_elems <= 4 * 400);
  dsmc::metrics::reset();
  o.resampler = dsmc::Resampler::multinomial;
  auto res = dsmc::run_smoother(model, o);
  snap = dsmc::metrics::snapshot();
  CHECK(snap.dense_allocs == 11);
  CHECK(snap.dense_max_elems == 400u * 400u);
  CHECK(snap.weight_evals == res.meta.weight_evals);
}

int main(int argc, char** argv) {
  const char* only = argc > 1 ? argv[1] : nullptr;
  int failed_cases = 0;
  for (auto& c : cases()) {
    if (only && std::strstr(c.name, only) == nullptr) continue;
    const int before = g_fail;
    try {
      c.fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("  exception: %s\n", e.what());
    }
    const bool ok = g_fail == before;
    failed_cases += !ok;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
  }
  std::printf("%d checks, %d failed, %d failing cases\n", g_checks, g_fail, failed_cases);
  return failed_cases ? 1 : 0;
}

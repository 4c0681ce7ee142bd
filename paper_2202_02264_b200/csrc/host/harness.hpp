// Experiment harness of the B200 dSMC engine: the reference's command-line
// tooling contract (/root/reference/proj/tools/experiment.hpp, dsmc_cli.cpp)
// over the C++ host API (include/dsmc/dsmc.hpp): the same configuration
// fields, JSON config overlay with unknown-key rejection, FNV-1a config hash,
// fixed-schema result CSV, method runners (dsmc, dsmc-rs, dsmc-mh, ffbs),
// theta-logistic particle Gibbs and the Kalman/RTS self-check. Every method
// runs on the GPU; nothing here computes a smoothing result on the host.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "dsmc/dsmc.hpp"

namespace dsmc::harness {

// ------------------------------------------------------------ tiny JSON
// Enough JSON for config files and for the canonical dump the config hash is
// taken over (objects keep sorted keys, compact separators, integers printed
// as integers and doubles in the shortest round-trip form with ".0" for
// integral values — the layout of the reference's JSON library dump()).
struct Json {
  enum Kind { Null, Bool, Int, Uint, Double, String, Array, Object } kind = Null;
  bool b = false;
  std::int64_t i = 0;
  std::uint64_t u = 0;
  double d = 0.0;
  std::string s;
  std::vector<Json> a;
  std::map<std::string, Json> o;

  static Json parse(const std::string& text);  // throws std::invalid_argument
  std::string dump() const;
  double as_double() const;
  std::int64_t as_int() const;
  std::uint64_t as_uint() const;

  Json() = default;
  Json(bool v) : kind(Bool), b(v) {}
  Json(int v) : kind(Int), i(v) {}
  Json(std::int64_t v) : kind(Int), i(v) {}
  Json(std::uint64_t v) : kind(Uint), u(v) {}
  Json(unsigned long long v) : kind(Uint), u(v) {}
  Json(double v) : kind(Double), d(v) {}
  Json(const char* v) : kind(String), s(v) {}
  Json(const std::string& v) : kind(String), s(v) {}
};

// --------------------------------------------------------------- config
struct LgssmCheckParams {  // experiment.hpp:18-27
  double coef = 0.9, shift = 0.0, trans_var = 0.25;
  double init_mean = 0.0, init_var = 1.0, obs_var = 0.25;
};

struct GibbsTuning {  // experiment.hpp:29-41
  double prec_x_shape = 2.0, prec_x_rate = 1.0;
  double prec_y_shape = 2.0, prec_y_rate = 1.0;
  double tau0_sd = 1.0, tau1_sd = 1.0, tau2_sd = 1.0;
  double rwm_step_tau = 0.05, rwm_step_x0 = 0.1;
  int ieks_cold_iterations = 25;
};

struct ExperimentConfig {  // experiment.hpp:43-75, same fields and defaults
  std::string experiment = "cox";
  int horizon = 32;
  std::size_t n_particles = 256;
  int replicates = 10;
  std::vector<std::string> methods;
  std::string resampler = "multinomial";
  std::size_t mh_steps = 16;
  std::uint64_t seed = 1;
  std::uint64_t data_seed = 90210;
  std::string out = "results.csv";
  int threads = 1;
  bool stable_timing = false;
  double proposal_inflation = 1.0;
  int sweeps = 1000;
  std::string data_path;
  std::string trace_out;
  CoxParams cox;
  double rw_sigma = 0.5;
  ThetaLogisticParams theta;
  LgssmCheckParams lgssm;
  GibbsTuning gibbs;
  // B200 additions (not part of the hash): arithmetic of the dsmc methods
  // (FP32 fast path or the bit-exact FP64 parity path) and the device
  Precision precision = Precision::fp32;
  int device = 0;
};

void validate_config(const ExperimentConfig& cfg);
void apply_json_file(const std::string& path, ExperimentConfig& cfg);
void apply_json(const Json& j, ExperimentConfig& cfg);
std::string config_hash(const ExperimentConfig& cfg, const std::vector<double>* loaded_data);
std::string csv_escape(const std::string& field);
std::string format_double(double v);
std::uint64_t derive_seed(std::uint64_t base, int method, int replicate);

// ------------------------------------------------------------------ CSV
struct ResultRow {  // experiment.hpp:97-111
  std::string experiment;
  int horizon = 0;
  std::size_t n_particles = 0;
  std::string method;
  int replicate = 0;
  std::optional<double> estimate;
  double wall_time_ms = 0.0;
  int levels = 0;
  std::uint64_t weight_evals = 0;
  std::optional<double> log_norm_const;
  std::uint64_t seed = 0;
  std::string hash;
  std::string error;
};
extern const char* const kCsvHeader;
std::string format_row(const ResultRow& row);
void write_csv(const std::string& path, const std::vector<ResultRow>& rows);

// ----------------------------------------------------------------- runs
struct ResolvedData {
  std::vector<double> ys;
  int horizon = 0;
  bool from_file = false;
  std::string note;
};
ResolvedData resolve_data(const ExperimentConfig& cfg);
bool run_smooth(const ExperimentConfig& cfg, const ResolvedData& data,
                std::vector<ResultRow>& rows);
bool run_pgibbs(const ExperimentConfig& cfg, const ResolvedData& data,
                std::vector<ResultRow>& rows);
bool run_oracle_check(const ExperimentConfig& cfg);

double mean_of(const std::vector<double>& v);
double variance_of(const std::vector<double>& v);  // unbiased (n - 1)

}  // namespace dsmc::harness

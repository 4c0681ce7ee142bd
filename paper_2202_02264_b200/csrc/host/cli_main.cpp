// dsmc_cli: the reference's command-line harness (tools/dsmc_cli.cpp:85-219)
// on the B200 engine. Subcommands smooth | pgibbs | bench | check-oracle with
// the same flags; flags override --config JSON values; every run writes the
// fixed-schema result CSV, summaries go to stdout and warnings to stderr.
// Exit codes: 0 ok, 1 some replicate or check failed, 2 usage/config error.
// B200 additions: --precision fp32|fp64 (the dsmc methods' arithmetic:
// the FP32 fast path or the bit-exact FP64 parity path) and --device.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "harness.hpp"

namespace {

using dsmc::harness::ExperimentConfig;
using dsmc::harness::ResultRow;

const char* kUsage =
    "dsmc_cli: divide-and-conquer particle smoothing and particle Gibbs experiments on B200\n"
    "usage: dsmc_cli <smooth|pgibbs|bench|check-oracle> [options]\n"
    "  --config PATH        JSON config file; flags override its values\n"
    "  --experiment NAME    cox, theta-logistic, constrained-rw, or lgssm-check\n"
    "  --T INT              time horizon (times run 0..T)\n"
    "  --N INT              particles per block\n"
    "  --replicates INT     independent repetitions\n"
    "  --resampler NAME     dense stitching scheme: multinomial or systematic\n"
    "  --mh-steps INT       chain length per slot for the dsmc-mh method\n"
    "  --seed INT           base inference seed\n"
    "  --data-seed INT      seed for simulating the shared data set\n"
    "  --out PATH           result CSV path\n"
    "  --threads INT        worker threads over replicates (validated; one GPU serves all)\n"
    "  --inflation X        proposal variance inflation factor\n"
    "  --data PATH          observation series, one value per line\n"
    "  --stable-timing      write wall_time_ms as 0 for byte-stable output\n"
    "  --methods LIST       smooth/bench: subset of dsmc,dsmc-rs,dsmc-mh,ffbs\n"
    "  --sweeps INT         pgibbs: Gibbs sweeps per chain\n"
    "  --trace PATH         pgibbs: also write per-sweep parameter draws\n"
    "  --T-list LIST        bench: comma-separated horizons\n"
    "  --N-list LIST        bench: comma-separated particle counts\n"
    "  --precision P        fp32 (default) or fp64 (bit-exact parity path)\n"
    "  --device INT         CUDA device\n";

std::vector<std::string> split(const std::string& s) {
  std::vector<std::string> out;
  std::size_t a = 0;
  while (a <= s.size()) {
    const std::size_t b = s.find(',', a);
    out.push_back(s.substr(a, b == std::string::npos ? std::string::npos : b - a));
    if (b == std::string::npos) break;
    a = b + 1;
  }
  return out;
}

long long to_int(const std::string& flag, const std::string& v) {
  char* end = nullptr;
  const long long x = std::strtoll(v.c_str(), &end, 10);
  if (v.empty() || *end) throw std::invalid_argument(flag + ": not an integer: " + v);
  return x;
}
unsigned long long to_uint(const std::string& flag, const std::string& v) {
  char* end = nullptr;
  const unsigned long long x = std::strtoull(v.c_str(), &end, 10);
  if (v.empty() || *end || v[0] == '-') throw std::invalid_argument(flag + ": not a non-negative integer: " + v);
  return x;
}
double to_real(const std::string& flag, const std::string& v) {
  char* end = nullptr;
  const double x = std::strtod(v.c_str(), &end);
  if (v.empty() || *end) throw std::invalid_argument(flag + ": not a number: " + v);
  return x;
}

std::vector<int> int_list(const std::vector<std::string>& raw, const char* flag) {
  if (raw.empty()) throw std::invalid_argument(std::string(flag) + " needs at least one value");
  std::vector<int> out;
  for (const auto& s : raw) {
    const long long v = to_int(flag, s);
    if (v < 1) throw std::invalid_argument(std::string(flag) + " entries must be at least 1");
    out.push_back(static_cast<int>(v));
  }
  return out;
}

void print_summary(const std::vector<ResultRow>& rows, const std::string& path) {
  std::vector<std::string> methods;
  for (const auto& r : rows) {
    bool seen = false;
    for (const auto& m : methods) seen = seen || m == r.method;
    if (!seen) methods.push_back(r.method);
  }
  std::printf("wrote %zu rows to %s\n", rows.size(), path.c_str());
  for (const auto& m : methods) {
    std::vector<double> est, wall;
    int failed = 0, total = 0;
    for (const auto& r : rows) {
      if (r.method != m) continue;
      ++total;
      if (r.error.empty() && r.estimate) {
        est.push_back(*r.estimate);
        wall.push_back(r.wall_time_ms);
      } else {
        ++failed;
      }
    }
    std::string line = "  " + m + ": " + std::to_string(total - failed) + "/" +
                       std::to_string(total) + " replicates ok";
    if (!est.empty()) {
      line += ", estimate mean " + dsmc::harness::format_double(dsmc::harness::mean_of(est));
      if (est.size() >= 2)
        line += ", sd " +
                dsmc::harness::format_double(std::sqrt(dsmc::harness::variance_of(est)));
      line += ", mean wall " + dsmc::harness::format_double(dsmc::harness::mean_of(wall)) + " ms";
    }
    std::printf("%s\n", line.c_str());
  }
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2 || !std::strcmp(argv[1], "--help") || !std::strcmp(argv[1], "-h")) {
    std::fputs(kUsage, argc < 2 ? stderr : stdout);
    return argc < 2 ? 2 : 0;
  }
  const std::string sub = argv[1];
  if (sub != "smooth" && sub != "pgibbs" && sub != "bench" && sub != "check-oracle") {
    std::fprintf(stderr, "error: unknown subcommand '%s'\n%s", sub.c_str(), kUsage);
    return 2;
  }
  std::set<std::string> allowed = {"--config", "--experiment", "--T", "--N", "--replicates",
                                   "--resampler", "--mh-steps", "--seed", "--data-seed", "--out",
                                   "--threads", "--inflation", "--data", "--stable-timing",
                                   "--precision", "--device"};
  if (sub == "smooth" || sub == "bench") allowed.insert("--methods");
  if (sub == "pgibbs") {
    allowed.insert("--sweeps");
    allowed.insert("--trace");
  }
  if (sub == "bench") {
    allowed.insert("--T-list");
    allowed.insert("--N-list");
  }
  std::map<std::string, std::string> opt;
  std::vector<std::string> methods, tlist, nlist;
  for (int k = 2; k < argc; ++k) {
    std::string a = argv[k], v;
    if (a == "--help" || a == "-h") {
      std::fputs(kUsage, stdout);
      return 0;
    }
    const std::size_t eq = a.find('=');
    if (eq != std::string::npos) {
      v = a.substr(eq + 1);
      a = a.substr(0, eq);
    }
    if (!allowed.count(a)) {
      std::fprintf(stderr, "error: the following argument was not expected: %s\n", argv[k]);
      return 2;
    }
    if (a == "--stable-timing") {
      opt[a] = "1";
      continue;
    }
    if (eq == std::string::npos) {
      if (k + 1 >= argc) {
        std::fprintf(stderr, "error: %s requires an argument\n", a.c_str());
        return 2;
      }
      v = argv[++k];
    }
    if (a == "--methods" || a == "--T-list" || a == "--N-list") {
      auto& dst = a == "--methods" ? methods : (a == "--T-list" ? tlist : nlist);
      for (auto& s : split(v)) dst.push_back(s);
    }
    opt[a] = v;
  }
  auto has = [&](const char* k) { return opt.count(k) > 0; };
  try {
    ExperimentConfig cfg;
    if (has("--config")) dsmc::harness::apply_json_file(opt["--config"], cfg);
    if (has("--experiment")) cfg.experiment = opt["--experiment"];
    if (has("--T")) cfg.horizon = static_cast<int>(to_int("--T", opt["--T"]));
    if (has("--N")) cfg.n_particles = to_uint("--N", opt["--N"]);
    if (has("--replicates")) cfg.replicates = static_cast<int>(to_int("--replicates", opt["--replicates"]));
    if (has("--resampler")) cfg.resampler = opt["--resampler"];
    if (has("--mh-steps")) cfg.mh_steps = to_uint("--mh-steps", opt["--mh-steps"]);
    if (has("--seed")) cfg.seed = to_uint("--seed", opt["--seed"]);
    if (has("--data-seed")) cfg.data_seed = to_uint("--data-seed", opt["--data-seed"]);
    if (has("--out")) cfg.out = opt["--out"];
    if (has("--threads")) cfg.threads = static_cast<int>(to_int("--threads", opt["--threads"]));
    if (has("--inflation")) cfg.proposal_inflation = to_real("--inflation", opt["--inflation"]);
    if (has("--data")) cfg.data_path = opt["--data"];
    if (has("--stable-timing")) cfg.stable_timing = true;
    if (has("--methods")) cfg.methods = methods;
    if (has("--device")) cfg.device = static_cast<int>(to_int("--device", opt["--device"]));
    if (has("--precision")) {
      const std::string p = opt["--precision"];
      if (p == "fp32") cfg.precision = dsmc::Precision::fp32;
      else if (p == "fp64") cfg.precision = dsmc::Precision::fp64_parity;
      else throw std::invalid_argument("--precision must be fp32 or fp64");
    }
    if (sub == "pgibbs") {
      if (has("--sweeps")) cfg.sweeps = static_cast<int>(to_int("--sweeps", opt["--sweeps"]));
      if (has("--trace")) cfg.trace_out = opt["--trace"];
      if (!has("--experiment") && !has("--config")) cfg.experiment = "theta-logistic";
    }
    dsmc::harness::validate_config(cfg);
    if (sub == "check-oracle") return dsmc::harness::run_oracle_check(cfg) ? 0 : 1;

    std::vector<ResultRow> rows;
    bool ok = true;
    if (sub == "smooth" || sub == "pgibbs") {
      const auto data = dsmc::harness::resolve_data(cfg);
      if (!data.note.empty()) std::fprintf(stderr, "%s\n", data.note.c_str());
      ok = sub == "smooth" ? dsmc::harness::run_smooth(cfg, data, rows)
                           : dsmc::harness::run_pgibbs(cfg, data, rows);
    } else {
      const auto ts = int_list(tlist.empty() ? std::vector<std::string>{std::to_string(cfg.horizon)}
                                             : tlist, "--T-list");
      const auto ns = int_list(nlist.empty() ? std::vector<std::string>{std::to_string(cfg.n_particles)}
                                             : nlist, "--N-list");
      for (int t : ts) {
        ExperimentConfig g = cfg;
        g.horizon = t;
        const auto data = dsmc::harness::resolve_data(g);
        if (!data.note.empty()) std::fprintf(stderr, "%s\n", data.note.c_str());
        for (int n : ns) {
          g.n_particles = static_cast<std::size_t>(n);
          ok = dsmc::harness::run_smooth(g, data, rows) && ok;
        }
      }
    }
    dsmc::harness::write_csv(cfg.out, rows);
    print_summary(rows, cfg.out);
    if (!ok) std::fprintf(stderr, "error: some replicates failed; see the error column\n");
    return ok ? 0 : 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
}

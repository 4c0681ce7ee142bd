// TEST INFRASTRUCTURE: prints the reference harness's config hash
// (experiment.cpp:240-303: FNV-1a of the nlohmann::json dump of the
// result-determining fields) for the configurations in
// tests/golden/make_hash_golden.py, using the JSON library the reference
// links (found in this image under cudnn_frontend's third-party tree).
// Input lines: experiment T N replicates methods(comma|-) resampler mh_steps
// seed data_seed inflation sweeps cox.mu cox.rho cox.sigma2 cox.lambda
// rw_sigma tau0 tau1 tau2 q2 r2 coef shift trans_var init_mean init_var
// obs_var gx_shape gx_rate gy_shape gy_rate tau0_sd tau1_sd tau2_sd
// step_tau step_x0 ieks
#include <cstdint>
#include <cstdio>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "nlohmann/json.hpp"

static std::uint64_t fnv(const std::string& s) {
  std::uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

int main() {
  std::string line;
  while (std::getline(std::cin, line)) {
    std::istringstream in(line);
    std::string exp, methods, resampler;
    int T, reps, sweeps, ieks;
    std::size_t N, mh;
    std::uint64_t seed, dseed;
    double infl, cmu, crho, cs2, clam, rws, t0, t1, t2, q2, r2, coef, shift, tv, im, iv, ov,
        gxs, gxr, gys, gyr, s0, s1, s2, st, sx;
    in >> exp >> T >> N >> reps >> methods >> resampler >> mh >> seed >> dseed >> infl >>
        sweeps >> cmu >> crho >> cs2 >> clam >> rws >> t0 >> t1 >> t2 >> q2 >> r2 >> coef >>
        shift >> tv >> im >> iv >> ov >> gxs >> gxr >> gys >> gyr >> s0 >> s1 >> s2 >> st >>
        sx >> ieks;
    std::vector<std::string> ms;
    std::stringstream mss(methods);
    for (std::string m; std::getline(mss, m, ',');) ms.push_back(m);
    nlohmann::json j;
    j["experiment"] = exp;
    j["T"] = T;
    j["N"] = N;
    j["replicates"] = reps;
    j["methods"] = ms;
    j["resampler"] = resampler;
    j["mh_steps"] = mh;
    j["seed"] = seed;
    j["data_seed"] = dseed;
    j["proposal_inflation"] = infl;
    j["sweeps"] = sweeps;
    j["cox"] = {{"mu", cmu}, {"rho", crho}, {"sigma2", cs2}, {"lambda", clam}};
    j["rw_sigma"] = rws;
    j["theta"] = {{"tau0", t0}, {"tau1", t1}, {"tau2", t2}, {"q2", q2}, {"r2", r2}};
    j["lgssm"] = {{"coef", coef}, {"shift", shift}, {"trans_var", tv},
                  {"init_mean", im}, {"init_var", iv}, {"obs_var", ov}};
    j["gibbs"] = {{"prec_x_shape", gxs}, {"prec_x_rate", gxr}, {"prec_y_shape", gys},
                  {"prec_y_rate", gyr}, {"tau0_sd", s0}, {"tau1_sd", s1}, {"tau2_sd", s2},
                  {"rwm_step_tau", st}, {"rwm_step_x0", sx}, {"ieks_cold_iterations", ieks}};
    std::printf("%016llx %s\n", (unsigned long long)fnv(j.dump()), j.dump().c_str());
  }
}

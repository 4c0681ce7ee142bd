// Internals shared by the C++ host layer's translation units.
#pragma once

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "dsmc/dsmc.hpp"

namespace dsmc {

// Owning storage behind a dsmc_model_desc (the arrays the descriptor points at).
struct DeviceModel {
  dsmc_model_desc desc{};
  std::vector<double> m0, P0, F, b, Q, H, R, y, prop_mean, prop_cov;
  std::vector<uint8_t> has_obs;
  void bind() {
    auto p = [](std::vector<double>& v) { return v.empty() ? nullptr : v.data(); };
    desc.m0 = p(m0);
    desc.P0 = p(P0);
    desc.F = p(F);
    desc.b = p(b);
    desc.Q = p(Q);
    desc.H = p(H);
    desc.R = p(R);
    desc.y = p(y);
    desc.prop_mean = p(prop_mean);
    desc.prop_cov = p(prop_cov);
    desc.has_obs = has_obs.empty() ? nullptr : has_obs.data();
  }
};

namespace detail {

[[noreturn]] void throw_code(int code, const std::string& msg);
dsmc_ctx* context(int device);  // one engine context per (thread, device)
void check(dsmc_ctx* c, int rc);
const dsmc_model_desc& desc_of(const FeynmanKacModel& m);
// validate_model + a device descriptor that agrees with it
const dsmc_model_desc& device_desc(const FeynmanKacModel& m);

// make_pair_source's device attachment: the model and the two blocks'
// boundary data, borrowed for the duration of one combine (as the
// reference's closures borrow the blocks, smoother.hpp:108-109).
struct BlockPairSource {
  std::shared_ptr<DeviceModel> model;
  int cut = 0;
  std::size_t n = 0;
  const double* xl = nullptr;    // L's slab at time cut - 1
  const double* xr = nullptr;    // R's slab at time cut
  const double* lw_l = nullptr;  // non-uniform L weights, else null
  const double* lw_r = nullptr;
};

}  // namespace detail
}  // namespace dsmc

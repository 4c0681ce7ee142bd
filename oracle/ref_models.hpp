// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// Builds reference-API models (dsmc::FeynmanKacModel, the reference's own
// struct of callbacks, fk_model.hpp:37-86) from the product's plain-data
// model descriptor (include/dsmc_b200.h), so the compiled reference
// smoother (oracle/_ref/libdsmc_ref.so) and the CUDA path run on the same
// model and data.
//
//  * LGSSM d = 1 restates make_lgssm_fk (models.cpp:562-685): same stitch-row
//    factory arithmetic (two gaussian_row passes + add_vec_scalar for the
//    column base, gaussian_row for the row), same log_stitch_bound rule.
//    models.cpp needs Eigen (absent, no network), so it cannot be compiled
//    here; this restatement is its stand-in.
//  * LGSSM d = 2..4 and SV do not exist in the reference; they
//    are written against the reference API with the FP64 operation order
//    documented in DESIGN.md §"parity arithmetic", which the device parity
//    kernels reproduce.
#pragma once

#include <memory>

#include "dsmc/fk_model.hpp"
#include "dsmc_b200.h"

namespace oracle {

// Derived per-time constants shared by the LGSSM callbacks.
struct LgPrep;

dsmc::FeynmanKacModel build_model(const dsmc_model_desc& desc);

}  // namespace oracle

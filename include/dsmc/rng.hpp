// Forwarding header: the reference's <dsmc/rng.hpp> include path
// (/root/reference/proj/include/dsmc/rng.hpp). Every dsmc:: declaration of
// the device-backed host API lives in dsmc/dsmc.hpp.
#pragma once
#include "dsmc/dsmc.hpp"

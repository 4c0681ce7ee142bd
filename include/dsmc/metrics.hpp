// Forwarding header: the reference's <dsmc/metrics.hpp> include path
// (/root/reference/proj/include/dsmc/metrics.hpp). Every dsmc:: declaration of
// the device-backed host API lives in dsmc/dsmc.hpp.
#pragma once
#include "dsmc/dsmc.hpp"

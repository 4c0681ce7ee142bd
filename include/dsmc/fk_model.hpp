// Forwarding header: the reference's <dsmc/fk_model.hpp> include path
// (/root/reference/proj/include/dsmc/fk_model.hpp). Every dsmc:: declaration of
// the device-backed host API lives in dsmc/dsmc.hpp.
#pragma once
#include "dsmc/dsmc.hpp"

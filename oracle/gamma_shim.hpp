// ORACLE / TEST INFRASTRUCTURE ONLY.
// Header-only shim that lets the reference's gamma_draw (pgibbs.cpp:80-102)
// compile on its own: pgibbs.cpp as a whole needs Eigen (through kalman.hpp),
// which is not available here, so oracle/Makefile extracts that one function
// body from /root/reference at build time (into _ref/, never into the repo)
// and compiles it after this prologue.
#pragma once
#include <cmath>
#include <stdexcept>

#include "dsmc/rng.hpp"

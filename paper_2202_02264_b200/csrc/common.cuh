// Device primitives shared by every dSMC kernel (sm_100a).
//
//  * Philox4x64-10 and the counter layout of the reference's RngStream
//    (rng.cpp:27-53): ctr = {block, node, level<<16 | role, substream},
//    key = {seed, 0x243F6A8885A308D3}. Streams are counter-addressed, so any
//    thread can jump to u64 number q of a stream (block q/4, lane q%4).
//  * exp_w, the reference's FP64 exp (exp_poly.hpp:39-51): Cody-Waite split
//    plus a degree-13 Horner polynomial with explicit FMAs. Bit-identical to
//    the CPU scalar backend (no FMA contraction: every op here is an
//    explicit __fma_rn / __dmul_rn / __dadd_rn).
//  * the 8-lane reduction contract (kernels.hpp:13-17, exp_poly.hpp:78-84).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace dsmc_dev {

constexpr uint64_t kPhiloxM0 = 0xD2E7470EE14C6C93ull;
constexpr uint64_t kPhiloxM1 = 0xCA5A826395121157ull;
constexpr uint64_t kPhiloxW0 = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kPhiloxW1 = 0xBB67AE8584CAA73Bull;
constexpr uint64_t kKey1 = 0x243F6A8885A308D3ull;
constexpr int kSub = 64;  // kernels::kSubBlock (kernels.hpp:77)

struct U64x4 {
  uint64_t v[4];
};

// One Philox4x64-10 block (rng.cpp:27-41).
__device__ __forceinline__ U64x4 philox(uint64_t c0, uint64_t c1, uint64_t c2,
                                        uint64_t c3, uint64_t k0) {
  uint64_t k1 = kKey1;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t lo0 = kPhiloxM0 * c0, hi0 = __umul64hi(kPhiloxM0, c0);
    const uint64_t lo1 = kPhiloxM1 * c2, hi1 = __umul64hi(kPhiloxM1, c2);
    const uint64_t n0 = hi1 ^ c1 ^ k0;
    const uint64_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += kPhiloxW0;
    k1 += kPhiloxW1;
  }
  U64x4 o;
  o.v[0] = c0;
  o.v[1] = c1;
  o.v[2] = c2;
  o.v[3] = c3;
  return o;
}

// Same with an arbitrary second key word (KAT tests).
__device__ __forceinline__ U64x4 philox_k(uint64_t c0, uint64_t c1,
                                          uint64_t c2, uint64_t c3,
                                          uint64_t k0, uint64_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t lo0 = kPhiloxM0 * c0, hi0 = __umul64hi(kPhiloxM0, c0);
    const uint64_t lo1 = kPhiloxM1 * c2, hi1 = __umul64hi(kPhiloxM1, c2);
    const uint64_t n0 = hi1 ^ c1 ^ k0;
    const uint64_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += kPhiloxW0;
    k1 += kPhiloxW1;
  }
  U64x4 o;
  o.v[0] = c0;
  o.v[1] = c1;
  o.v[2] = c2;
  o.v[3] = c3;
  return o;
}

// Word p (0..3) of a block by select chain: indexing v[] with a runtime value
// would place the block in local memory.
__device__ __forceinline__ uint64_t pick4(const U64x4& b, uint32_t p) {
  return p == 0 ? b.v[0] : p == 1 ? b.v[1] : p == 2 ? b.v[2] : b.v[3];
}

// Stream identity (rng.cpp:45-53).
struct StreamId {
  uint64_t seed, node, lvrole, sub;
};
__device__ __forceinline__ StreamId stream_id(uint64_t seed, uint32_t level,
                                              uint64_t node, int role,
                                              uint64_t substream) {
  StreamId s;
  s.seed = seed;
  s.node = node;
  s.lvrole = (static_cast<uint64_t>(level) << 16) | static_cast<uint64_t>(role);
  s.sub = substream;
  return s;
}
__device__ __forceinline__ U64x4 stream_block(const StreamId& s, uint64_t blk) {
  return philox(blk, s.node, s.lvrole, s.sub, s.seed);
}
// u64 number q of the stream.
__device__ __forceinline__ uint64_t stream_u64(const StreamId& s, uint64_t q) {
  const U64x4 b = stream_block(s, q >> 2);
  return pick4(b, (uint32_t)(q & 3));
}

// rng.cpp:66-72.
// FP32 uniforms from the top 23 bits of a u64 without an int -> float
// conversion (I2F issues on the XU pipe, which the leaf kernels' MUFU work
// already saturates): the bits fill the mantissa of a float in [1, 2).
__device__ __forceinline__ float u01_open23(uint64_t v) {  // (0, 1): (2m + 1) 2^-24
  return __uint_as_float(0x3F800000u | (uint32_t)(v >> 41)) - (1.0f - 0x1p-24f);
}
__device__ __forceinline__ float u01_23(uint64_t v) {  // [0, 1): m 2^-23
  return __uint_as_float(0x3F800000u | (uint32_t)(v >> 41)) - 1.0f;
}
__device__ __forceinline__ double u64_uniform(uint64_t v) {
  return __dmul_rn(static_cast<double>(v >> 11), 0x1.0p-53);
}
__device__ __forceinline__ double u64_uniform_pos(uint64_t v) {
  return __dmul_rn(__dadd_rn(static_cast<double>(v >> 12), 0.5), 0x1.0p-52);
}
// rng.cpp:88-93.
__device__ __forceinline__ uint64_t u64_index(uint64_t v, uint64_t n) {
  return __umul64hi(v, n);
}

// Sequential reader over a stream (lazy samplers, Gibbs kernels).
struct StreamReader {
  StreamId id;
  uint64_t blk;
  U64x4 buf;
  int pos;
  double cached;
  bool has_cached;
  __device__ void init(const StreamId& s) {
    id = s;
    blk = 0;
    pos = 4;
    has_cached = false;
  }
  __device__ __forceinline__ uint64_t next() {
    if (pos == 4) {
      buf = stream_block(id, blk++);
      pos = 0;
    }
    // pick4, not buf.v[pos]: no local memory (an STL per refill and an LDL
    // per draw otherwise)
    const uint64_t v = pick4(buf, (uint32_t)pos);
    ++pos;
    return v;
  }
  __device__ double uniform() { return u64_uniform(next()); }
  __device__ double uniform_pos() { return u64_uniform_pos(next()); }
  __device__ uint64_t index(uint64_t n) { return u64_index(next(), n); }
  // Box-Muller, cos first then the cached sin (rng.cpp:74-86). Device
  // log/sin/cos are within 1-2 ulp of glibc, not bit-identical.
  __device__ double normal() {
    if (has_cached) {
      has_cached = false;
      return cached;
    }
    const double u1 = uniform_pos();
    const double u2 = uniform();
    const double r = sqrt(-2.0 * log(u1));
    const double th = 2.0 * 3.14159265358979323846 * u2;
    double s, c;
    sincos(th, &s, &c);
    cached = r * s;
    has_cached = true;
    return r * c;
  }
};

// The draws of MB lazy steps / trials (3 u64 each: index i, index j, then the
// uniform through `lu_of` -- log2 in FP32, log in FP64) from 3 MB / 4 whole
// Philox blocks starting at block b0; each block is consumed as soon as it is
// generated, so only the converted values stay live.
template <int MB, class T, class F>
__device__ __forceinline__ void draw_batch(const StreamId& id, uint64_t b0, int N, uint32_t* pi,
                                           uint32_t* pj, T* lu, F lu_of) {
  static_assert(MB % 4 == 0, "whole Philox blocks per batch");
#pragma unroll
  for (int r = 0; r < 3 * MB / 4; ++r) {
    const U64x4 blk = stream_block(id, b0 + r);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int n = 4 * r + c, q = n / 3;
      if (n % 3 == 0) pi[q] = (uint32_t)u64_index(blk.v[c], N);
      else if (n % 3 == 1) pj[q] = (uint32_t)u64_index(blk.v[c], N);
      else lu[q] = lu_of(blk.v[c]);
    }
  }
}

// ------------------------------------------------------------------ exp_w
// The FP64 constants live in constant memory so DMUL / DFMA take them as
// c[][] operands (as immediates each costs two UMOVs per use, ~14% of the
// FP64 pass's instructions), and the special cases are selects around one
// straight-line evaluation instead of branches. Same operations, same order,
// same results as the branchy form.
__constant__ double kExpW[16] = {
    1.4426950408889634074,  -6.93147180369123816490e-01, -1.90821492927058770002e-10,
    1.0 / 6227020800.0,     1.0 / 479001600,              1.0 / 39916800,
    1.0 / 3628800,          1.0 / 362880,                 1.0 / 40320,
    1.0 / 5040,             1.0 / 720,                    1.0 / 120,
    1.0 / 24,               1.0 / 6,                      1.0 / 2,
    1.0};
__device__ __forceinline__ double exp_w(double x) {
  const bool nan = isnan(x), low = x <= -708.0;
  const double xc = (nan || low) ? 0.0 : (x > 710.0 ? 710.0 : x);
  const double k = rint(__dmul_rn(xc, kExpW[0]));
  double r = __fma_rn(k, kExpW[1], xc);
  r = __fma_rn(k, kExpW[2], r);
  double p = kExpW[3];
#pragma unroll
  for (int q = 4; q < 16; ++q) p = __fma_rn(p, r, kExpW[q]);
  p = __fma_rn(p, r, kExpW[15]);
  const long long ki = static_cast<long long>(k);
  const double scale =
      __longlong_as_double(static_cast<long long>(
          static_cast<unsigned long long>(ki + 1023) << 52));
  const double v = __dmul_rn(p, scale);
  return nan ? x : (low ? 0.0 : v);
}
// exp_w on its pass-1 domain: x = v - (row max) <= 0 or -inf, never NaN (a
// NaN row is reported and skipped before its sum pass). Same operations and
// results as exp_w there, without the NaN and overflow selects.
__device__ __forceinline__ double exp_w_le0(double x) {
  const bool low = x <= -708.0;
  const double xc = x;  // a low x (-inf included) evaluates garbage the final select drops
  const double k = rint(__dmul_rn(xc, kExpW[0]));
  double r = __fma_rn(k, kExpW[1], xc);
  r = __fma_rn(k, kExpW[2], r);
  double p = kExpW[3];
#pragma unroll
  for (int q = 4; q < 16; ++q) p = __fma_rn(p, r, kExpW[q]);
  p = __fma_rn(p, r, kExpW[15]);
  const long long ki = __double2ll_rz(k);  // k is integral; a low x's inf saturates (result dropped)
  const double scale =
      __longlong_as_double(static_cast<long long>(
          static_cast<unsigned long long>(ki + 1023) << 52));
  const double v = __dmul_rn(p, scale);
  return low ? 0.0 : v;
}

// b[l] = a[l] + a[l+4]; (b0 + b2) + (b1 + b3).
__device__ __forceinline__ double combine8(const double a[8]) {
  const double b0 = __dadd_rn(a[0], a[4]);
  const double b1 = __dadd_rn(a[1], a[5]);
  const double b2 = __dadd_rn(a[2], a[6]);
  const double b3 = __dadd_rn(a[3], a[7]);
  return __dadd_rn(__dadd_rn(b0, b2), __dadd_rn(b1, b3));
}

// Device error record: first failing (code, cut) wins.
// Reasons (message selection on the host).
enum ErrReason {
  kReasonNone = 0,
  kReasonZeroTable = 1,   // all pair weights are zero (resampling.cpp:94-96)
  kReasonTrialCap = 2,    // rejection trial cap (resampling.cpp:316-320)
  kReasonOverBound = 3,   // weight above its bound (resampling.cpp:310-311)
  kReasonNaN = 4,         // NaN pair / leaf weight
  kReasonNoBound = 5,     // rejection without a finite bound
  kReasonRefPair = 6,     // conditional reference pair has zero weight
  kReasonLeafZero = 7,    // every leaf draw has zero weight
  kReasonRefLeaf = 8,     // conditional reference has zero leaf weight
};
struct ErrFlag {
  int code;  // dsmc_status
  int cut;   // cut (combines) or time (leaves)
  int level;
  int reason;
};
__device__ __forceinline__ void raise_err(ErrFlag* e, int code, int cut,
                                          int level, int reason = 0) {
  if (atomicCAS(&e->code, 0, code) == 0) {
    e->cut = cut;
    e->level = level;
    e->reason = reason;
  }
}

// Schedule geometry (smoother.cpp:64-85): level l (>= 1) combine k merges
// blocks [2k s, (2k+1) s - 1] and [(2k+1) s, min((2k+2) s, K) - 1], s =
// 2^(l-1); the cut is (2k+1) s.
struct CombineGeom {
  int a, c, b;
};
__device__ __host__ __forceinline__ CombineGeom combine_geom(int level, int k,
                                                             int K) {
  const int s = 1 << (level - 1);
  CombineGeom g;
  g.a = 2 * k * s;
  g.c = (2 * k + 1) * s;
  const int rb = (2 * k + 2) * s - 1;
  g.b = rb < K - 1 ? rb : K - 1;
  return g;
}

}  // namespace dsmc_dev

// FP32 pass 1 on tcgen05, streaming form (d = 2..4; DSMC_PAIR_KERNEL=tc2).
//
// Same contraction as c32_pair_tc (pair_tc.cuh): the bound-shifted exponent
//   t_ij = (A_j - cmax_s) + u_i . y_j - c_i
// as a 3xTF32 rank-(3d+4) product (K = 16), accumulated in TMEM, so the SM
// only takes exponentials. What changes is who does what:
//
//  * c32_prol (one launch per sub-chunk of <= kTc2Sub combines) computes each
//    combine's columns once — y_j, A_j for the sampler hand-off (Aux32), the
//    per-sub-block column maximum cmax_s, and the column operand tile of every
//    64-column sub-block in the UMMA K-major layout (4 KB) — and the rows'
//    u_i, B_i. A sub-chunk's tiles (64 KB per combine) stay in L2 for pass 1.
//  * c32_pair_tc2: one CTA per 128-row tile of a combine; warp 8 (lane 0)
//    bulk-copies tiles into an 8-stage ring (cp.async.bulk, mbarrier
//    complete_tx) and issues each sub-block's two N = 64 MMAs into one of four
//    64-column TMEM accumulators; warps 0-3 and 4-7 (two consumer groups, one
//    row = TMEM lane per thread) take alternate sub-blocks: two
//    tcgen05.ld.32x32b.x32, release the accumulator, then 64 exponentials —
//    a fraction through an FMA-pipe polynomial (ex2_poly2) so MUFU.EX2 is not
//    the only unit doing them — summed with packed FADD2. No producer compute
//    and no column gathers remain inside the MUFU-bound kernel.
//
// Output identical in layout to c32_pair: ws[s][i] = log2 sum_{j in s} 2^w_ij.
#pragma once

#include "wide.cuh"  // tma_bulk_g2s, pair_tc.cuh primitives

namespace dsmc_dev {

constexpr int kTc2Sub = 1024;     // combines per prologue / pass-1 sub-chunk (tiles in L2)
constexpr int kTc2Stages = 8;     // shared tile ring
constexpr int kTc2Threads = 160;  // 4 consumer warps (one row = TMEM lane each) + 1 MMA / copy warp
constexpr int kTc2Ctas = 4;       // CTAs per SM (2 x 64 TMEM columns each)
#ifndef DSMC_TC2_POLY
#define DSMC_TC2_POLY 2  // of every 8 exponential pairs, this many on the FMA pipe
#endif
constexpr int kTc2Poly = DSMC_TC2_POLY;

// 2^x for a pair on the FMA / ALU pipes, for x <= 127 (the bound-shifted
// exponents are <= 100 by construction): round-to-nearest split x = n + r by
// the magic-number add, degree-5 minimax polynomial of 2^r on [-1/2, 1/2]
// (relative error 2.4e-7 evaluated in FP32, the order of ex2.approx), n added
// to the exponent bits with one shift-add (f's bits << 23 leave exactly n << 23:
// the magic's own bits shift out). x is clamped below at -125, whose 2^x is
// negligible next to a kept sum >= 2^-60.
__device__ __forceinline__ float2 ex2_poly5(float2 x) {
  x.x = fmaxf(x.x, -125.f);
  x.y = fmaxf(x.y, -125.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);  // 1.5 * 2^23
  const float2 f = __fadd2_rn(x, magic);
  const float2 nr = __fadd2_rn(f, make_float2(-12582912.f, -12582912.f));
  const float2 r = __fadd2_rn(x, make_float2(-nr.x, -nr.y));
  float2 p = make_float2(1.3276379322633147e-3f, 1.3276379322633147e-3f);
  p = __ffma2_rn(p, r, make_float2(9.675510227680206e-3f, 9.675510227680206e-3f));
  p = __ffma2_rn(p, r, make_float2(5.550713092088699e-2f, 5.550713092088699e-2f));
  p = __ffma2_rn(p, r, make_float2(2.4022120237350464e-1f, 2.4022120237350464e-1f));
  p = __ffma2_rn(p, r, make_float2(6.931469440460205e-1f, 6.931469440460205e-1f));
  p = __ffma2_rn(p, r, make_float2(1.0000001192092896f, 1.0000001192092896f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(f.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(f.y) << 23)));
}

template <int D>
struct Tc2L {
  using L = TcK<D>;
  static constexpr int TILE = kSub / 8 * L::SBO;  // bytes of one sub-block's column tile
  static constexpr int ATILE = kTcRows / 8 * L::SBO;
};

// per combine of a sub-chunk: nsub column tiles, then nsub column maxima
__host__ __device__ inline size_t tc2_comb_bytes(int nsub, int tile) {
  return (size_t)nsub * tile + (((size_t)nsub * 4 + 127) & ~(size_t)127);
}

// Prologue: grid (ceil(nsub*64 / 128), combines, chains), 128 threads. Thread
// t of block x handles column q = 128 x + t (two sub-blocks per block) and,
// for q < N, row q.
template <int D>
__global__ void __launch_bounds__(128) c32_prol(Bufs b, LevelArgs la, uint8_t* tiles) {
  using T = Tc2L<D>;
  const int k = la.k0 + blockIdx.y, ch = blockIdx.z;
  const int N = b.N, nsub = (N + kSub - 1) / kSub;
  Side L, R;
  CombineGeom g;
  sides(b, la, k, L, R, g);
  __shared__ CutConst32 s_cc;
  __shared__ float s_cm[4];
  if (threadIdx.x == 0) load_cut32<D>(b.tc[(size_t)ch * b.Kt + b.t0 + g.c], s_cc);
  const CutConst32& cc = s_cc;  // read after the barrier below
  const size_t cslot = (size_t)blockIdx.z * gridDim.y + blockIdx.y;
  const Aux32 ax = aux32(la, cslot, N);
  uint8_t* ct = tiles + cslot * tc2_comb_bytes(nsub, T::TILE);
  float* cmax = reinterpret_cast<float*>(ct + (size_t)nsub * T::TILE);
  const int q = blockIdx.x * 128 + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // both gather chains (column q and row q) issued before any arithmetic
  const bool lnonuni = L.leaf && !b.UNI[(size_t)ch * b.K + L.t];
  float4 xc = make_float4(0.f, 0.f, 0.f, 0.f), xl = xc;
  float col = -CUDART_INF_F, lwr = 0.f;
  if (q < N) {
    const uint32_t pc = map_first(b, la, ch, R, q);
    const uint32_t pr = map_last(b, la, ch, L, q);
    const size_t offc = ((size_t)ch * b.K + R.t) * N + pc;
    xc = b.X32[offc];
    col = b.COL[offc];
    xl = b.X32[((size_t)ch * b.K + L.t) * N + pr];
    if (lnonuni) lwr = b.LW32[(size_t)ch * N + q];
  }
  __syncthreads();  // s_cc
  float y[4] = {0.f, 0.f, 0.f, 0.f};
  float A = -CUDART_INF_F, cv = -CUDART_INF_F;
  if (q < N) {
    cv = col;
    col32<D>(cc, xc, cv, y, A);
    ax.y[q] = make_float4(y[0], y[1], y[2], y[3]);
    ax.A[q] = A;
  }
  bool live = A > -CUDART_INF_F;
#pragma unroll
  for (int c = 0; c < D; ++c) live = live && isfinite(y[c]);
  if (!live) {
    cv = -CUDART_INF_F;
#pragma unroll
    for (int c = 0; c < D; ++c) y[c] = 0.f;
  }
  float cm = cv;  // cmax_s: the two warps of the sub-block
#pragma unroll
  for (int o = 16; o; o >>= 1) cm = fmaxf(cm, __shfl_xor_sync(~0u, cm, o));
  if (lane == 0) s_cm[warp] = cm;
  __syncthreads();
  cm = fmaxf(s_cm[warp & ~1], s_cm[warp | 1]);
  const int s = q / kSub;
  if (s < nsub) {
    if ((q & (kSub - 1)) == 0) cmax[s] = cm;
    float vals[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) vals[c] = 0.f;
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const float hi = tf32_hi(y[c]);
      vals[c] = hi;
      vals[D + c] = hi;
      vals[2 * D + c] = y[c] - hi;
    }
    const bool clive = live && cm > -CUDART_INF_F;
    const float a = clive ? A - cm : kDeadCol;
    const float ah = tf32_hi(a);
    vals[3 * D] = ah;
    vals[3 * D + 1] = clive ? a - ah : 0.f;
    vals[3 * D + 2] = 1.f;
    vals[3 * D + 3] = 1.f;
    tc_store_row<D>(ct + (size_t)s * T::TILE, q & (kSub - 1), vals);
  }
  if (q < N) {  // row q: the left block's last-leaf state
    float u[4] = {0.f, 0.f, 0.f, 0.f}, Bv;
    row32<D>(cc, xl, lwr, u, Bv);
    ax.u[q] = make_float4(u[0], u[1], u[2], u[3]);
    ax.B[q] = Bv;
  }
}

// Row operand of TMEM lane `row` for one item (K-major, into tile sA), and the
// row's output terms (B_i, overflow shift c_i).
template <int D>
__device__ __forceinline__ void tc2_row(float4 u4, float Bv, bool ok, uint8_t* sA, int row,
                                        float& Brow, float& crow) {
  float u[4] = {u4.x, u4.y, u4.z, u4.w};
  Brow = ok ? Bv : -CUDART_INF_F;
  bool fin = Brow > -CUDART_INF_F;
#pragma unroll
  for (int c = 0; c < D; ++c) fin = fin && isfinite(u[c]);
  if (!fin) {
    Brow = -CUDART_INF_F;
#pragma unroll
    for (int c = 0; c < 4; ++c) u[c] = 0.f;
  }
  float nn = 0.f;
#pragma unroll
  for (int c = 0; c < D; ++c) nn = fmaf(0.5f * u[c], 0.5f * u[c], nn);
  crow = nn > 100.f ? nn - 100.f : 0.f;  // the overflow shift c_i of c32_pair
  float vals[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) vals[c] = 0.f;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const float hi = tf32_hi(u[c]);
    vals[c] = hi;
    vals[D + c] = u[c] - hi;
    vals[2 * D + c] = hi;
  }
  vals[3 * D] = 1.f;
  vals[3 * D + 1] = 1.f;
  const float ch_ = tf32_hi(-crow);
  vals[3 * D + 2] = ch_;
  vals[3 * D + 3] = -crow - ch_;
  tc_store_row<D>(sA, row, vals);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// One CTA per (combine, 128-row tile): warps 0-3 consume (one row = TMEM lane
// each), warp 4 lane 0 copies tiles and issues MMAs into two 64-column TMEM
// accumulators (4 CTAs per SM fill the 512 columns).
template <int D>
__global__ void __launch_bounds__(kTc2Threads, kTc2Ctas) c32_pair_tc2(Bufs b, LevelArgs la,
                                                               const uint8_t* tiles) {
  using T = Tc2L<D>;
  using L = TcK<D>;
  __shared__ __align__(128) uint8_t sA[T::ATILE];
  __shared__ __align__(128) uint8_t sB[kTc2Stages][T::TILE];
  __shared__ __align__(8) uint64_t bar_full[kTc2Stages], bar_tfull[2], bar_tempty[2];
  __shared__ uint32_t s_tmem;
  const int N = b.N, nsub = (N + kSub - 1) / kSub;
  const int rt = blockIdx.x;
  const size_t cslot = (size_t)blockIdx.z * gridDim.y + blockIdx.y;
  const Aux32 ax = aux32(la, cslot, N);
  float* ws = reinterpret_cast<float*>(la.ws) + cslot * la.ws_comb * 2;
  const uint8_t* ct = tiles + cslot * tc2_comb_bytes(nsub, T::TILE);
  const float* cmax = reinterpret_cast<const float*>(ct + (size_t)nsub * T::TILE);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&s_tmem)),
                 "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 128) {
    for (int q = 0; q < kTc2Stages; ++q) mbar_init(&bar_full[q], 1);
    for (int a = 0; a < 2; ++a) {
      mbar_init(&bar_tfull[a], 1);
      mbar_init(&bar_tempty[a], 4);  // the 4 consumer warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
    for (int q = 0; q < kTc2Stages && q < nsub; ++q)
      tma_bulk_g2s(sB[q], ct + (size_t)q * T::TILE, T::TILE, &bar_full[q]);
  }
  const int row = 32 * (warp & 3) + lane, i = rt * kTcRows + row;
  float Brow = -CUDART_INF_F, crow = 0.f;
  if (warp < 4) {
    float4 u4 = make_float4(0.f, 0.f, 0.f, 0.f);
    float Bv = -CUDART_INF_F;
    if (i < N) {
      u4 = ax.u[i];
      Bv = ax.B[i];
    }
    tc2_row<D>(u4, Bv, i < N, sA, row, Brow, crow);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s_tmem;
  if (warp == 4) {
    // ------------------------------------------------ MMA issue + tile copies
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kSub >> 3) << 17) |
                             ((uint32_t)(kTcRows >> 4) << 24);
      for (int it = 0; it < nsub; ++it) {
        const int q = it % kTc2Stages, a = it & 1;
        mbar_wait(smem_u32(&bar_full[q]), (it / kTc2Stages) & 1);
        if (it >= 2) mbar_wait(smem_u32(&bar_tempty[a]), ((it >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
        for (int ks = 0; ks < L::KS; ++ks) {
          const uint64_t da = umma_sdesc(smem_u32(sA) + ks * 2 * L::LBO, L::LBO, L::SBO);
          const uint64_t db = umma_sdesc(smem_u32(sB[q]) + ks * 2 * L::LBO, L::LBO, L::SBO);
          const uint32_t acc = ks > 0;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + a * 64),
              "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                smem_u32(&bar_tfull[a])));
        // refill the stage of sub-block it - 2: its MMAs completed before the
        // consumers released accumulator a (the tempty wait above)
        const int r = it - 2;
        if (r >= 0 && r + kTc2Stages < nsub) {
          const int rq = r % kTc2Stages;
          tma_bulk_g2s(sB[rq], ct + (size_t)(r + kTc2Stages) * T::TILE, T::TILE, &bar_full[rq]);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ consumers
    const uint32_t lane_off = (uint32_t)(32 * warp) << 16;
    for (int it = 0; it < nsub; ++it) {
      const int a = it & 1;
      mbar_wait(smem_u32(&bar_tfull[a]), (it >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      float v[64];
      tmem_ld32(tmem + lane_off + (uint32_t)(a * 64), v);
      tmem_ld32(tmem + lane_off + (uint32_t)(a * 64 + 32), v + 32);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_tempty[a]);
      const float cmx = cmax[it];
      float2 a4[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) a4[e] = make_float2(0.f, 0.f);
#pragma unroll
      for (int cc = 0; cc < 64; cc += 16) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float2 x = make_float2(v[cc + 2 * e], v[cc + 2 * e + 1]);
          const float2 ev = (e >= 8 - kTc2Poly) ? ex2_poly5(x) : make_float2(ex2(x.x), ex2(x.y));
          a4[e & 3] = __fadd2_rn(a4[e & 3], ev);
        }
      }
      const float2 s2 = __fadd2_rn(__fadd2_rn(a4[0], a4[1]), __fadd2_rn(a4[2], a4[3]));
      const float sum = s2.x + s2.y;
      float Ls;
      if (sum >= 0x1p-60f && sum <= 0x1p120f) {
        Ls = lg2(sum);
      } else {  // out of the safe range (rows far from every column): exact max
        float m = v[0];
#pragma unroll
        for (int q = 1; q < 64; ++q) m = fmaxf(m, v[q]);
        float acc = 0.f;
        if (m > 0.5f * kDeadCol)
#pragma unroll
          for (int q = 0; q < 64; ++q) acc += ex2(v[q] - m);
        Ls = acc > 0.f ? m + lg2(acc) : -CUDART_INF_F;
      }
      if (i < N)
        ws[(size_t)it * N + i] = (Brow > -CUDART_INF_F && cmx > -CUDART_INF_F && Ls > -CUDART_INF_F)
                                     ? Ls + crow + cmx + Brow
                                     : -CUDART_INF_F;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}

}  // namespace dsmc_dev

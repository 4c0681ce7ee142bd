// FP32 pass 1 on the 5th-generation tensor cores (tcgen05, sm_100a).
//
// The pair exponent in log2 units is w_ij = A_j + u_i . y_j + B_i (whitened
// expanded form, col32 / row32): a rank-(d+1) product plus row and column
// terms. A CTA owns 128 rows of one combine (one TMEM lane per row and per
// thread); per 64-column sub-block one elected thread issues
//     D[128 x 64] (TMEM, FP32) = A_rows[128 x K] . B_cols[64 x K]^T
// (kind::tf32, K-major shared-memory operands, no swizzle) and the four
// warps read their rows back with tcgen05.ld, take the exact row max over
// the 64 columns and sum 2^(t - max) on MUFU.EX2: no FP32-pipe dot products
// remain, so the kernel runs at the MUFU roof instead of the FFMA2+MUFU mix
// roof of c32_pair.
//
// Precision: TF32 keeps 10 mantissa bits, so every operand is split
// x = x_hi + x_lo (x_hi = x with the low 13 mantissa bits cleared) and the
// product is taken as u_hi y_hi + u_lo y_hi + u_hi y_lo ("3xTF32"), the
// column term as a_hi + a_lo; K = 3d + 2 padded to 8 or 16. The dropped
// u_lo y_lo term is ~2^-22 relative, the FP32 accumulation ~2^-23 of the
// term magnitudes — the same order as the FFMA chain it replaces.
//
// Pipeline per sub-block s: threads 0..63 write B_s (one column each, from
// raw data prefetched a sub-block ahead) into shared buffer s & 1; barrier;
// thread 0 issues the MMAs into TMEM buffer s & 1 and commits to mbarrier
// s & 1; every thread then finishes sub-block s - 1 (wait on its mbarrier,
// tcgen05.ld, max / exp2 / sum, store L_is). 128 TMEM columns per CTA, 4 CTAs
// per SM.
#pragma once

#include "combine32.cuh"

namespace dsmc_dev {

constexpr int kTcRows = 128;  // rows per CTA (MMA M)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}
// shared-memory matrix descriptor: K-major, no swizzle, version 1
__device__ __forceinline__ uint64_t umma_sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr & 0x3FFFF) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
// Waits for the phase of the given parity; a wait that outlives ~10 s of
// spinning traps (a pipeline bug then surfaces as a launch error, never as a
// hung device).
__device__ __forceinline__ uint64_t gtimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void mbar_wait(uint32_t addr, uint32_t parity) {
  uint32_t done = 0;
  uint32_t spins = 0;
  uint64_t t0 = 0;
  while (!done) {
    if ((++spins & 0xffff) == 0) {
      const uint64_t t = gtimer_ns();
      if (t0 == 0) t0 = t;
      else if (t - t0 > 10000000000ull) __trap();
    }
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tmem_ld32(uint32_t ta, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(ta));
#pragma unroll
  for (int c = 0; c < 32; ++c) v[c] = __uint_as_float(r[c]);
}

// K layout (per row i / column j, 4-wide chunks of the K-major operands):
//   A_i = [u_hi(d), u_lo(d), u_hi(d), 1, 1, 0...]
//   B_j = [y_hi(d), y_hi(d), y_lo(d), a_hi, a_lo, 0...]
template <int D>
struct TcK {
  static constexpr int K = (3 * D + 2 <= 8) ? 8 : 16;
  static constexpr int KC = K / 4;          // 16-byte chunks per row
  static constexpr int SBO = KC * 128;      // bytes per 8-row core-matrix group
  static constexpr int LBO = 128;           // bytes between K chunks
  static constexpr int KS = K / 8;          // MMA K-steps (K = 8 per tf32 MMA)
};

// write one operand row (16 floats max) into the K-major layout
template <int D>
__device__ __forceinline__ void tc_store_row(uint8_t* base, int r, const float* vals) {
  using L = TcK<D>;
  uint8_t* p = base + (r & 7) * 16 + (r >> 3) * L::SBO;
#pragma unroll
  for (int c = 0; c < L::KC; ++c)
    *reinterpret_cast<float4*>(p + c * L::LBO) =
        make_float4(vals[4 * c], vals[4 * c + 1], vals[4 * c + 2], vals[4 * c + 3]);
}

constexpr float kDeadCol = -1e30f;  // finite stand-in for A_j = -inf

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(
                   smem_u32(bar))
               : "memory");
}

constexpr int kTcConsumers = kTcRows;            // warps 0-3: one row (TMEM lane) each
constexpr int kTcProducers = kSub;               // warps 4-5: one column each
constexpr int kTcThreads = kTcConsumers + kTcProducers + 32;  // + warp 6: MMA issue
constexpr int kTcCtasPerSm = 2;
constexpr int kTcStages = 4;  // TMEM accumulator stages of 64 columns (256 per CTA)
constexpr int kTcMaxSub = 32;  // column cache: up to 32 sub-blocks (N <= 2048)

// Shared-memory column cache of one work item: sub-block s of the item at
// s * colbytes (64 columns, K-major core matrices).
template <int D>
__host__ __device__ constexpr int tc_col_bytes() {
  return kSub / 8 * TcK<D>::SBO;
}
template <int D>
__host__ __device__ constexpr size_t tc_smem_bytes(int nsb) {
  return (size_t)nsb * tc_col_bytes<D>();
}

// Work item w of a launch: (column split, combine of the chunk, chain). An
// item runs all its 128-row tiles against the same staged columns.
struct TcItem {
  int cs, kk, ch, sb0, sb1;
};
__device__ __forceinline__ TcItem tc_item(const LevelArgs& la, int w, int nsub) {
  TcItem it;
  it.cs = w % la.tc_ncs;
  w /= la.tc_ncs;
  it.kk = w % la.tc_nk;
  it.ch = w / la.tc_nk;
  it.sb0 = it.cs * nsub / la.tc_ncs;
  it.sb1 = (it.cs + 1) * nsub / la.tc_ncs;
  return it;
}

// Persistent warp-specialised pass 1 (grid = 3 CTAs per SM over the work
// list of (column split, combine, chain) items).
//  * producers (warps 4-5, one column each) gather and write every sub-block
//    of the item's columns once into the shared column cache, arriving on
//    full[s] per sub-block (gathers pipelined: block-map index three
//    sub-blocks ahead, state two ahead); before the next item they wait for
//    the item's last MMA;
//  * the issuer (warp 6, one thread) walks (row tile, sub-block) and issues
//    D[tile rows x 64] = A_tile . B_s^T into TMEM stage q & 1 once the
//    sub-block is staged (first tile), the tile's rows are written and the
//    stage was released, committing to tfull[q & 1];
//  * consumers (warps 0-3, one row each) read their 64 values per stage with
//    tcgen05.ld, release the stage and spend it on MUFU; during a tile's last
//    stage they write the next tile's rows (gathered a tile ahead) into the
//    other A buffer, so the issuer never waits on a row prologue.
template <int D>
__global__ void __maxnreg__(96) c32_pair_tc(Bufs b, LevelArgs la) {
  using L = TcK<D>;
  constexpr int CB = tc_col_bytes<D>();
  extern __shared__ __align__(128) uint8_t s_cols[];  // [item sub-blocks][CB]
  __shared__ __align__(128) uint8_t sA[2][kTcRows / 8 * L::SBO];
  __shared__ __align__(8) uint64_t bar_full[kTcMaxSub], bar_tfull[kTcStages], bar_tempty[kTcStages], bar_a[2],
      bar_item;
  __shared__ uint32_t s_tmem;
  __shared__ CutConst32 s_ccp, s_ccc;  // cut constants: producers' item, consumers' item
  const int N = b.N;
  const int nsub = (N + kSub - 1) / kSub;
  const int nrt = (N + kTcRows - 1) / kTcRows;
  const int W = la.tc_ncs * la.tc_nk * b.B;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&s_tmem)),
                 "r"(kTcStages * kSub));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == kTcConsumers) {
    for (int q = 0; q < kTcMaxSub; ++q) mbar_init(&bar_full[q], kTcProducers);
    for (int q = 0; q < kTcStages; ++q) {
      mbar_init(&bar_tfull[q], 1);
      mbar_init(&bar_tempty[q], kTcConsumers / 32);
    }
    for (int q = 0; q < 2; ++q) mbar_init(&bar_a[q], kTcConsumers);
    mbar_init(&bar_item, 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s_tmem;

  if (warp >= (kTcConsumers + kTcProducers) / 32) {
    // ----------------------------------------------------------- issuer
    // (the whole warp walks the schedule and waits; lane 0 issues)
    {
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) |
                             ((uint32_t)(kSub >> 3) << 17) | ((uint32_t)(kTcRows >> 4) << 24);
      int q = 0, tcn = 0, itc = 0;
      for (int w = blockIdx.x; w < W; w += gridDim.x, ++itc) {
        const TcItem it = tc_item(la, w, nsub);
        for (int rt = 0; rt < nrt; ++rt, ++tcn) {
          mbar_wait(smem_u32(&bar_a[tcn & 1]), (tcn >> 1) & 1);
          for (int sbk = it.sb0; sbk < it.sb1; ++sbk, ++q) {
            const int sl = sbk - it.sb0;
            if (rt == 0) mbar_wait(smem_u32(&bar_full[sl]), itc & 1);
            if (q >= kTcStages)
              mbar_wait(smem_u32(&bar_tempty[q % kTcStages]), ((q / kTcStages) - 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            if (lane == 0) {
              const uint32_t dcol = tmem + (uint32_t)((q % kTcStages) * kSub);
#pragma unroll
              for (int ks = 0; ks < L::KS; ++ks) {
                const uint64_t da =
                    umma_sdesc(smem_u32(sA[tcn & 1]) + ks * 2 * L::LBO, L::LBO, L::SBO);
                const uint64_t db =
                    umma_sdesc(smem_u32(s_cols + sl * CB) + ks * 2 * L::LBO, L::LBO, L::SBO);
                const uint32_t acc = ks > 0;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(dcol),
                    "l"(da), "l"(db), "r"(idesc), "r"(acc));
              }
              asm volatile(
                  "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                      smem_u32(&bar_tfull[q % kTcStages])));
            }
            __syncwarp();
          }
        }
        // the item's columns may be replaced once its last MMA has completed
        if (lane == 0)
          asm volatile(
              "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                  smem_u32(&bar_item)));
        __syncwarp();
      }
    }
  } else if (tid >= kTcConsumers) {
    // -------------------------------------------------------- producers
    const int p = tid - kTcConsumers;  // column within the sub-block
    struct Cur {
      int w, s, sb1, ch;
      Side R;
      size_t base;
    };
    auto enter = [&](Cur& c, int w) {
      c.w = w;
      if (w >= W) return;
      const TcItem it = tc_item(la, w, nsub);
      Side Lq;
      CombineGeom gq;
      sides(b, la, la.k0 + it.kk, Lq, c.R, gq);
      c.s = it.sb0;
      c.sb1 = it.sb1;
      c.ch = it.ch;
      c.base = ((size_t)it.ch * b.K + c.R.t) * N;
    };
    auto step = [&](Cur& c) {
      if (c.w < W && ++c.s >= c.sb1) enter(c, c.w + gridDim.x);
    };
    auto idx_of = [&](const Cur& c) -> uint32_t {
      const int j = c.s * kSub + p;
      if (c.w >= W || j >= N) return 0xffffffffu;
      return map_first(b, la, c.ch, c.R, j);
    };
    Cur c0, c1, c2, c3;
    enter(c0, blockIdx.x);
    c1 = c0;
    step(c1);
    c2 = c1;
    step(c2);
    c3 = c2;
    step(c3);
    float4 x0 = make_float4(0.f, 0.f, 0.f, 0.f), x1 = x0;
    float k0 = -CUDART_INF_F, k1 = k0;
    {
      const uint32_t i0 = idx_of(c0), i1 = idx_of(c1);
      if (i0 != 0xffffffffu) {
        x0 = b.X32[c0.base + i0];
        k0 = b.COL[c0.base + i0];
      }
      if (i1 != 0xffffffffu) {
        x1 = b.X32[c1.base + i1];
        k1 = b.COL[c1.base + i1];
      }
    }
    uint32_t i2 = idx_of(c2);
    int itc = 0;  // items entered
    TcItem it = tc_item(la, c0.w < W ? c0.w : 0, nsub);
    const CutConst32& cc = s_ccp;
    auto load_item = [&](int w) {
      it = tc_item(la, w, nsub);
      Side Lq, Rq;
      CombineGeom gq;
      sides(b, la, la.k0 + it.kk, Lq, Rq, gq);
      asm volatile("bar.sync 1, %0;" ::"n"(kTcProducers));
      if (p == 0) {
        CutConst32 t;
        load_cut32<D>(b.tc[(size_t)it.ch * b.Kt + b.t0 + gq.c], t);
        s_ccp = t;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kTcProducers));
      // the previous item's columns stay in the cache until its last MMA
      // (bar_item completes once per item, so its parity is unambiguous)
      if (itc > 0) mbar_wait(smem_u32(&bar_item), (itc - 1) & 1);
    };
    if (c0.w < W) load_item(c0.w);
    while (c0.w < W) {
      const uint32_t i3 = idx_of(c3);
      float4 x2 = make_float4(0.f, 0.f, 0.f, 0.f);
      float k2 = -CUDART_INF_F;
      if (i2 != 0xffffffffu) {
        x2 = b.X32[c2.base + i2];
        k2 = b.COL[c2.base + i2];
      }
      const int sbk = c0.s;
      const int j = sbk * kSub + p;
      float y[4] = {0.f, 0.f, 0.f, 0.f};
      float A = -CUDART_INF_F;
      if (j < N) {
        col32<D>(cc, x0, k0, y, A);
        // hand the column to the sampler
        const Aux32 ax = aux32(la, (size_t)it.ch * la.tc_nk + it.kk, N);
        ax.y[j] = make_float4(y[0], y[1], y[2], y[3]);
        ax.A[j] = A;
      }
      // a dead column (A = -inf, or a non-finite state) enters as y = 0 with
      // a large negative finite a: inf / NaN would poison every row's sum
      bool live = A > -CUDART_INF_F;
#pragma unroll
      for (int c = 0; c < D; ++c) live = live && isfinite(y[c]);
      if (!live) {
#pragma unroll
        for (int c = 0; c < D; ++c) y[c] = 0.f;
      }
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
      const float a = live ? A : kDeadCol;
      const float ah = tf32_hi(a);
      vals[3 * D] = ah;
      vals[3 * D + 1] = live ? a - ah : 0.f;
      tc_store_row<D>(s_cols + (sbk - it.sb0) * CB, p, vals);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&bar_full[sbk - it.sb0]);
      x0 = x1;
      k0 = k1;
      x1 = x2;
      k1 = k2;
      i2 = i3;
      const int prev_w = c0.w;
      step(c0);
      step(c2);
      step(c3);
      if (c0.w != prev_w) {
        ++itc;
        if (c0.w < W) load_item(c0.w);
      }
    }
  } else {
    // -------------------------------------------------------- consumers
    const uint32_t lane_off = (uint32_t)(32 * warp) << 16;
    // rows of a tile: state through the left block's last map, left weight
    struct RowSrc {
      int w, rt;
    };
    auto row_idx = [&](int w, int rt) -> uint32_t {
      if (w >= W) return 0xffffffffu;
      const TcItem it = tc_item(la, w, nsub);
      const int i = rt * kTcRows + tid;
      if (i >= N) return 0xffffffffu;
      Side Lq, Rq;
      CombineGeom gq;
      sides(b, la, la.k0 + it.kk, Lq, Rq, gq);
      return map_last(b, la, it.ch, Lq, i);
    };
    auto row_data = [&](int w, int rt, uint32_t idx, float4& xl, float& lw) {
      xl = make_float4(0.f, 0.f, 0.f, 0.f);
      lw = 0.f;
      if (idx == 0xffffffffu) return;
      const TcItem it = tc_item(la, w, nsub);
      const int i = rt * kTcRows + tid;
      Side Lq, Rq;
      CombineGeom gq;
      sides(b, la, la.k0 + it.kk, Lq, Rq, gq);
      xl = b.X32[((size_t)it.ch * b.K + Lq.t) * N + idx];
      if (Lq.leaf && !b.UNI[(size_t)it.ch * b.K + Lq.t]) lw = b.LW32[(size_t)it.ch * N + i];
    };
    // write the rows of tile (w, rt) into sA[slot]; returns B_i of the row
    auto write_rows = [&](int w, int rt, const CutConst32& cc, float4 xl, float lwr, int slot,
                          float& Brow) {
      Brow = -CUDART_INF_F;
      const TcItem it = tc_item(la, w, nsub);
      const int i = rt * kTcRows + tid;
      float u[4] = {0.f, 0.f, 0.f, 0.f};
      float vals[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) vals[c] = 0.f;
      if (w < W && i < N) {
        row32<D>(cc, xl, lwr, u, Brow);
        if (it.cs == 0) {  // hand the row to the sampler
          const Aux32 ax = aux32(la, (size_t)it.ch * la.tc_nk + it.kk, N);
          ax.u[i] = make_float4(u[0], u[1], u[2], u[3]);
          ax.B[i] = Brow;
        }
        // a dead row (zero weight, or a non-finite state) must not put
        // inf / NaN into the MMA: its sums are discarded (L = -inf)
        bool fin = Brow > -CUDART_INF_F;
#pragma unroll
        for (int c = 0; c < D; ++c) fin = fin && isfinite(u[c]);
        if (!fin) {
          Brow = -CUDART_INF_F;
#pragma unroll
          for (int c = 0; c < D; ++c) u[c] = 0.f;
        }
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const float hi = tf32_hi(u[c]);
          vals[c] = hi;
          vals[D + c] = u[c] - hi;
          vals[2 * D + c] = hi;
        }
        vals[3 * D] = 1.f;
        vals[3 * D + 1] = 1.f;
      }
      tc_store_row<D>(sA[slot], tid, vals);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&bar_a[slot]);
    };
    auto load_cc = [&](int w) {
      const TcItem it = tc_item(la, w < W ? w : 0, nsub);
      Side Lq, Rq;
      CombineGeom gq;
      sides(b, la, la.k0 + it.kk, Lq, Rq, gq);
      asm volatile("bar.sync 2, %0;" ::"n"(kTcConsumers));
      if (tid == 0) {
        CutConst32 t;
        load_cut32<D>(b.tc[(size_t)it.ch * b.Kt + b.t0 + gq.c], t);
        s_ccc = t;
      }
      asm volatile("bar.sync 2, %0;" ::"n"(kTcConsumers));
    };
    // first tile's rows
    int w = blockIdx.x;
    const CutConst32& cc = s_ccc;
    load_cc(w);
    float Brow;
    {
      float4 xl;
      float lw;
      row_data(w, 0, row_idx(w, 0), xl, lw);
      write_rows(w, 0, cc, xl, lw, 0, Brow);
    }
    int q = 0, tcn = 0;
    while (w < W) {
      const TcItem it = tc_item(la, w, nsub);
      const size_t cslot = (size_t)it.ch * la.tc_nk + it.kk;
      float* ws = reinterpret_cast<float*>(la.ws) + cslot * la.ws_comb * 2;
      for (int rt = 0; rt < nrt; ++rt, ++tcn) {
        // the next tile (same item, or the first of the next item)
        const int nw = rt + 1 < nrt ? w : w + gridDim.x;
        const int nrt_ = rt + 1 < nrt ? rt + 1 : 0;
        const uint32_t nidx = row_idx(nw, nrt_);
        float4 nxl = make_float4(0.f, 0.f, 0.f, 0.f);
        float nlw = 0.f;
        const int i = rt * kTcRows + tid;
        const bool row_ok = i < N;
        float Bnext = -CUDART_INF_F;
        for (int sbk = it.sb0; sbk < it.sb1; ++sbk, ++q) {
          if (sbk == it.sb0) row_data(nw, nrt_, nidx, nxl, nlw);
          mbar_wait(smem_u32(&bar_tfull[q % kTcStages]), (q / kTcStages) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          float v[64];
          const uint32_t ta = tmem + lane_off + (uint32_t)((q % kTcStages) * kSub);
          tmem_ld32(ta, v);
          tmem_ld32(ta + 32, v + 32);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          asm volatile("tcgen05.fence::before_thread_sync;");
          __syncwarp();
          if (lane == 0) mbar_arrive(&bar_tempty[q % kTcStages]);
          if (sbk + 1 == it.sb1) {  // last stage of the tile: next tile's rows
            if (nw != w) load_cc(nw);
            write_rows(nw, nrt_, cc, nxl, nlw, (tcn + 1) & 1, Bnext);
          }
          // row max and sum with independent partial chains (4 max trees,
          // 4 packed accumulators): the consumers are few per SMSP, so the
          // MUFU queue is fed by ILP rather than by warp count
          float mq[4];
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const float* x = v + 16 * h;
            const float a = fmax3(fmax3(x[0], x[1], x[2]), fmax3(x[3], x[4], x[5]),
                                  fmax3(x[6], x[7], x[8]));
            const float c2 = fmax3(fmax3(x[9], x[10], x[11]), fmax3(x[12], x[13], x[14]), x[15]);
            mq[h] = fmaxf(a, c2);
          }
          const float m = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
          float2 acc[4];
#pragma unroll
          for (int h = 0; h < 4; ++h) acc[h] = make_float2(0.f, 0.f);
          const float2 nm = make_float2(-m, -m);
#pragma unroll
          for (int c = 0; c < 64; c += 8) {
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const float2 t = __fadd2_rn(make_float2(v[c + 2 * h], v[c + 2 * h + 1]), nm);
              acc[h] = __fadd2_rn(acc[h], make_float2(ex2(t.x), ex2(t.y)));
            }
          }
          const float2 s01 = __fadd2_rn(acc[0], acc[1]), s23 = __fadd2_rn(acc[2], acc[3]);
          const float2 s4 = __fadd2_rn(s01, s23);
          const float sum = s4.x + s4.y;
          if (row_ok)
            ws[(size_t)sbk * N + i] = (m > 0.5f * kDeadCol && Brow > -CUDART_INF_F)
                                          ? lg2(sum) + m + Brow
                                          : -CUDART_INF_F;
        }
        Brow = Bnext;
      }
      w += gridDim.x;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTcStages * kSub));
}

}  // namespace dsmc_dev

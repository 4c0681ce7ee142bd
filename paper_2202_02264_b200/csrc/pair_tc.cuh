// FP32 pass 1 on the 5th-generation tensor cores (tcgen05, sm_100a),
// selected with DSMC_PAIR_KERNEL=tc (d >= 2).
//
// The bound-shifted pair exponent of c32_pair, t_ij = (A_j - cmax_s) +
// u_i . y_j - c_i (log2 units, whitened expanded form), is a rank-(d+2)
// product: a CTA owns 128 rows of one combine (one TMEM lane per row) and
// per 64-column sub-block issues two
//     D[128 x 32] (TMEM, FP32) = A_rows[128 x K] . B_cols[32 x K]^T
// (kind::tf32, K-major shared-memory operands, no swizzle) into one of four
// 32-column TMEM stages. The consumer warps read a stage with one
// tcgen05.ld.32x32b.x32, release it, and sum 2^t on MUFU.EX2 (one pair in
// four through an FMA-pipe polynomial) with packed FADD2 accumulators; a
// half sub-block whose sum leaves [2^-60, 2^120] is redone from its exact max.
//
// Precision: TF32 keeps 10 mantissa bits, so every operand is split
// x = x_hi + x_lo (x_hi = x with the low 13 mantissa bits cleared) and the
// product is taken as u_hi y_hi + u_lo y_hi + u_hi y_lo ("3xTF32"), the
// column and row shifts as hi + lo pairs; K = 3d + 4 padded to 8 or 16. The
// dropped u_lo y_lo term is ~2^-22 relative, the FP32 accumulation ~2^-23 of
// the term magnitudes — the same order as the FFMA chain it replaces.
//
// Roles per CTA (224 threads, 4 CTAs per SM = 4 x 128 TMEM columns): warps
// 0-3 consume (one row each), warps 4-5 produce (one column each: gather,
// whiten, split, write the K-major row of the B operand into one of four
// shared buffers), warp 6 issues the MMAs once a buffer is full and its TMEM
// stage was released. Barriers are mbarriers with per-buffer / per-stage
// phase parities; every wait traps after 10 s instead of hanging.
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
//   A_i = [u_hi(d), u_lo(d), u_hi(d), 1, 1, -c_hi, -c_lo, 0...]
//   B_j = [y_hi(d), y_hi(d), y_lo(d), a_hi, a_lo, 1, 1, 0...]
// so D_ij = u_i . y_j + a_j - c_i: the bound-shifted exponent of c32_pair.
template <int D>
struct TcK {
  static constexpr int K = (3 * D + 4 <= 8) ? 8 : 16;
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

// 2^x for a pair on the FMA / ALU pipes (no MUFU): round-to-nearest split
// x = n + r (magic-number add), r in [-1/2, 1/2], degree-6 Taylor of 2^r
// (relative error < 1.3e-7, the order of ex2.approx), 2^n added to the
// exponent bits. x is clamped to [-125, 127]: results below 2^-125 are
// negligible next to a sum >= 2^-60 (the pass-1 range check).
#ifndef DSMC_TC_POLY
#define DSMC_TC_POLY 1
#endif
constexpr bool kTcPolyExp = DSMC_TC_POLY != 0;
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  x.x = fminf(fmaxf(x.x, -125.f), 127.f);
  x.y = fminf(fmaxf(x.y, -125.f), 127.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);  // 1.5 * 2^23
  const float2 f = __fadd2_rn(x, magic);
  const float2 nr = __fadd2_rn(f, make_float2(-12582912.f, -12582912.f));
  const float2 r = __fadd2_rn(x, make_float2(-nr.x, -nr.y));
  const int nx = __float_as_int(f.x) - 0x4B400000, ny = __float_as_int(f.y) - 0x4B400000;
  // Taylor coefficients (ln 2)^k / k!
  float2 p = make_float2(1.5403530393381606e-4f, 1.5403530393381606e-4f);
  p = __ffma2_rn(p, r, make_float2(1.3333558146428443e-3f, 1.3333558146428443e-3f));
  p = __ffma2_rn(p, r, make_float2(9.6181291076284772e-3f, 9.6181291076284772e-3f));
  p = __ffma2_rn(p, r, make_float2(5.5504108664821580e-2f, 5.5504108664821580e-2f));
  p = __ffma2_rn(p, r, make_float2(2.4022650695910071e-1f, 2.4022650695910071e-1f));
  p = __ffma2_rn(p, r, make_float2(6.9314718055994531e-1f, 6.9314718055994531e-1f));
  p = __ffma2_rn(p, r, make_float2(1.f, 1.f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (nx << 23)),
                     __int_as_float(__float_as_int(p.y) + (ny << 23)));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(
                   smem_u32(bar))
               : "memory");
}

constexpr int kTcConsumers = kTcRows;               // warps 0-3: one row (TMEM lane) each
constexpr int kTcProducers = kSub;                   // warps 4-5: one column each
constexpr int kTcThreads = kTcConsumers + kTcProducers + 32;  // + warp 6: MMA issue
constexpr int kTcBufs = 4;     // staged sub-blocks in flight (shared memory)
constexpr int kTcStages = 4;   // TMEM accumulator stages of kTcHalf columns
constexpr int kTcHalf = 32;    // columns per MMA / TMEM stage (half a sub-block)
constexpr int kTcCtasPerSm = 4;  // 4 x 128 TMEM columns

// Tensor-core pass 1 (one CTA per 128-row tile and column split, 4 CTAs per
// SM). Producers (warps 4-5, one column each) stage sub-block q into shared
// buffer q % 4: y_j and a_j = A_j - cmax_s (the two producer warps exchange
// their column maxima), then arrive on full[q % 4]; they reuse a buffer once
// the consumers released its second half (bfree). The issuer warp waits for
// a full buffer and a released TMEM stage and issues the sub-block as two
// N = 32 MMAs, each committed to its stage's mbarrier. Consumers (warps 0-3)
// take a stage with one tcgen05.ld.x32, release it at once and sum 2^t with
// four packed accumulators: the exponent is bound-shifted exactly as in
// c32_pair (shift c_i + cmax_s), so the SM executes only MUFU.EX2 (or the
// FMA-pipe polynomial) and FADD2 per pair. A half sub-block whose sum leaves
// [2^-60, 2^120] (rare: rows far from every column) is redone with its exact
// max from the values still in registers, in log form.
template <int D>
__global__ void __launch_bounds__(kTcThreads, kTcCtasPerSm) c32_pair_tc(Bufs b, LevelArgs la) {
  using L = TcK<D>;
  constexpr int CB = kSub / 8 * L::SBO;  // bytes of one staged sub-block
  __shared__ __align__(128) uint8_t sA[kTcRows / 8 * L::SBO];
  __shared__ __align__(128) uint8_t sB[kTcBufs][CB];
  __shared__ __align__(8) uint64_t bar_full[kTcBufs], bar_bfree[kTcBufs], bar_tfull[kTcStages],
      bar_tempty[kTcStages];
  __shared__ uint32_t s_tmem;
  __shared__ float s_cm[kTcBufs][2];  // per buffer: the two producer warps' column maxima
  __shared__ float s_cmax[kTcBufs];   // per buffer: cmax of the staged sub-block
  __shared__ CutConst32 s_cc;          // the cut's constants (loaded once per CTA)
  const int k = la.k0 + blockIdx.y, ch = blockIdx.z;
  const int N = b.N;
  const int nsub = (N + kSub - 1) / kSub;
  const int nrt = (N + kTcRows - 1) / kTcRows;
  const int rt = blockIdx.x % nrt, cs = blockIdx.x / nrt, ncs = gridDim.x / nrt;
  Side Lsd, Rsd;
  CombineGeom g;
  sides(b, la, k, Lsd, Rsd, g);
  const TimeConst& tc = b.tc[(size_t)ch * b.Kt + b.t0 + g.c];
  const size_t cslot = (size_t)blockIdx.z * gridDim.y + blockIdx.y;
  float* ws = reinterpret_cast<float*>(la.ws) + cslot * la.ws_comb * 2;
  const Aux32 ax = aux32(la, cslot, N);
  const int row0 = rt * kTcRows;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int sb0 = cs * nsub / ncs, sb1 = (cs + 1) * nsub / ncs;
  const int nq = sb1 - sb0;  // sub-blocks of this CTA
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&s_tmem)),
                 "r"(kTcStages * kTcHalf));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == kTcConsumers) {
    for (int q = 0; q < kTcBufs; ++q) {
      mbar_init(&bar_full[q], kTcProducers);
      mbar_init(&bar_bfree[q], kTcConsumers / 32);
    }
    for (int q = 0; q < kTcStages; ++q) {
      mbar_init(&bar_tfull[q], 1);
      mbar_init(&bar_tempty[q], kTcConsumers / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }

  if (tid >= kTcConsumers + kTcProducers) {
    // ----------------------------------------------------------- issuer
    {  // the cut constants for everyone, one entry per lane (load_cut32's
       // fields; published by barrier 1)
      if (lane < D * D) {
        s_cc.W[lane] = (float)(tc.tW[lane]) * kS;
        s_cc.F[lane] = (float)tc.F[lane];
      } else if (lane >= 16 && lane < 16 + D) {
        s_cc.delta[lane - 16] = (float)tc.delta[lane - 16];
      } else if (lane == 24) {
        s_cc.drift = tc.drift;
      } else if (lane >= 25 && lane < 29) {
        s_cc.th[lane - 25] = (float)tc.th[lane - 25];
      } else if (lane == 29) {
        s_cc.th[4] = (float)tc.pm[0];
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();  // (1)
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = s_tmem;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) |
                           ((uint32_t)(kTcHalf >> 3) << 17) | ((uint32_t)(kTcRows >> 4) << 24);
    __syncthreads();  // (2) the rows are in sA
    for (int q = 0; q < nq; ++q) {
      mbar_wait(smem_u32(&bar_full[q % kTcBufs]), (q / kTcBufs) & 1);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int hq = 2 * q + h;
        if (hq >= kTcStages)
          mbar_wait(smem_u32(&bar_tempty[hq % kTcStages]), ((hq / kTcStages) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (lane == 0) {
          const uint32_t dcol = tmem + (uint32_t)((hq % kTcStages) * kTcHalf);
#pragma unroll
          for (int ks = 0; ks < L::KS; ++ks) {
            const uint64_t da = umma_sdesc(smem_u32(sA) + ks * 2 * L::LBO, L::LBO, L::SBO);
            // columns 32h..32h+31 = core-matrix groups 4h..4h+3
            const uint64_t db = umma_sdesc(
                smem_u32(sB[q % kTcBufs]) + h * 4 * L::SBO + ks * 2 * L::LBO, L::LBO, L::SBO);
            const uint32_t acc = ks > 0;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(dcol),
                "l"(da), "l"(db), "r"(idesc), "r"(acc));
          }
          asm volatile(
              "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                  smem_u32(&bar_tfull[hq % kTcStages])));
        }
        __syncwarp();
      }
    }
  } else if (tid >= kTcConsumers) {
    // -------------------------------------------------------- producers
    const int p = tid - kTcConsumers;
    const int pw = p >> 5;  // producer warp 0 / 1
    const CutConst32& cc = s_cc;  // valid after barrier (1)
    const float4* XR = b.X32 + ((size_t)ch * b.K + Rsd.t) * N;
    const float* CR = b.COL + ((size_t)ch * b.K + Rsd.t) * N;
    // gathers: block-map index two sub-blocks ahead, state one ahead
    auto idx_of = [&](int sbk) -> uint32_t {
      const int j = sbk * kSub + p;
      if (sbk >= sb1 || j >= N) return 0xffffffffu;
      return map_first(b, la, ch, Rsd, j);
    };
    uint32_t i1 = idx_of(sb0 + 1);
    float4 x0 = make_float4(0.f, 0.f, 0.f, 0.f);
    float k0 = -CUDART_INF_F;
    {
      const uint32_t i0 = idx_of(sb0);
      if (i0 != 0xffffffffu) {
        x0 = XR[i0];
        k0 = CR[i0];
      }
    }
    __syncthreads();  // (1) barriers initialised, TMEM allocated
    __syncthreads();  // (2) the rows are in sA
    for (int q = 0; q < nq; ++q) {
      const int sbk = sb0 + q;
      const uint32_t i2 = idx_of(sbk + 2);
      float4 x1 = make_float4(0.f, 0.f, 0.f, 0.f);
      float k1 = -CUDART_INF_F;
      if (i1 != 0xffffffffu) {
        x1 = XR[i1];
        k1 = CR[i1];
      }
      const int j = sbk * kSub + p;
      float y[4] = {0.f, 0.f, 0.f, 0.f};
      float A = -CUDART_INF_F, cv = -CUDART_INF_F;
      if (j < N) {
        cv = k0;
        col32<D>(cc, x0, k0, y, A);
        if (rt == 0) {  // hand the column to the sampler
          ax.y[j] = make_float4(y[0], y[1], y[2], y[3]);
          ax.A[j] = A;
        }
      }
      bool live = A > -CUDART_INF_F;
#pragma unroll
      for (int c = 0; c < D; ++c) live = live && isfinite(y[c]);
      if (!live) {
        cv = -CUDART_INF_F;
#pragma unroll
        for (int c = 0; c < D; ++c) y[c] = 0.f;
      }
      // cmax_s over the 64 columns: warp max, then the two warps' maxima
      float cm = cv;
#pragma unroll
      for (int o = 16; o; o >>= 1) cm = fmaxf(cm, __shfl_xor_sync(~0u, cm, o));
      // buffer q % kTcBufs (and its cmax slot) is free once the consumers
      // finished reading sub-block q - kTcBufs (its MMAs completed before)
      const int bq = q % kTcBufs;
      if (q >= kTcBufs) mbar_wait(smem_u32(&bar_bfree[bq]), ((q / kTcBufs) - 1) & 1);
      if (lane == 0) s_cm[bq][pw] = cm;
      asm volatile("bar.sync 1, %0;" ::"n"(kTcProducers));
      cm = fmaxf(s_cm[bq][0], s_cm[bq][1]);
      if (p == 0) s_cmax[bq] = cm;
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
      tc_store_row<D>(sB[bq], p, vals);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&bar_full[bq]);
      x0 = x1;
      k0 = k1;
      i1 = i2;
    }
  } else {
    // -------------------------------------------------------- consumers
    const int i = row0 + tid;
    const bool row_ok = i < N;
    float Brow = -CUDART_INF_F, crow = 0.f;
    float4 xl = make_float4(0.f, 0.f, 0.f, 0.f);
    float lwr = 0.f;
    if (row_ok) {  // row gathers in flight across barrier (1)
      xl = b.X32[((size_t)ch * b.K + Lsd.t) * N + map_last(b, la, ch, Lsd, i)];
      if (Lsd.leaf && !b.UNI[(size_t)ch * b.K + Lsd.t]) lwr = b.LW32[(size_t)ch * N + i];
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();  // (1) barriers, TMEM and the cut constants are ready
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = s_tmem;
    {
      const CutConst32& cc = s_cc;
      float u[4] = {0.f, 0.f, 0.f, 0.f};
      float vals[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) vals[c] = 0.f;
      if (row_ok) {
        row32<D>(cc, xl, lwr, u, Brow);
        if (cs == 0) {  // hand the row to the sampler
          ax.u[i] = make_float4(u[0], u[1], u[2], u[3]);
          ax.B[i] = Brow;
        }
        bool fin = Brow > -CUDART_INF_F;
#pragma unroll
        for (int c = 0; c < D; ++c) fin = fin && isfinite(u[c]);
        if (!fin) {
          Brow = -CUDART_INF_F;
#pragma unroll
          for (int c = 0; c < D; ++c) u[c] = 0.f;
        }
        float nn = 0.f;
#pragma unroll
        for (int c = 0; c < D; ++c) nn = fmaf(0.5f * u[c], 0.5f * u[c], nn);
        crow = nn > 100.f ? nn - 100.f : 0.f;  // the overflow shift c_i of c32_pair
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
      }
      tc_store_row<D>(sA, tid, vals);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();  // (2) rows staged
    const uint32_t lane_off = (uint32_t)(32 * warp) << 16;
    for (int q = 0; q < nq; ++q) {
      const int sbk = sb0 + q;
      // per half: linear sum (bound shift) or, if it left the safe range, the
      // log2 of the sum from the half's exact max
      float part[2];
      bool lin[2];
      float cmx = 0.f;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int hq = 2 * q + h;
        mbar_wait(smem_u32(&bar_tfull[hq % kTcStages]), (hq / kTcStages) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (h == 0) cmx = s_cmax[q % kTcBufs];  // read before the buffer is released
        float v[32];
        tmem_ld32(tmem + lane_off + (uint32_t)((hq % kTcStages) * kTcHalf), v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&bar_tempty[hq % kTcStages]);
          if (h == 1) mbar_arrive(&bar_bfree[q % kTcBufs]);
        }
        float2 a4[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) a4[c] = make_float2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < 32; c += 8) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 x = make_float2(v[c + 2 * e], v[c + 2 * e + 1]);
            // one pair in four on the FMA pipe (idle here): MUFU.EX2 is the roof
            const float2 ev = (kTcPolyExp && e == 3) ? ex2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
            a4[e] = __fadd2_rn(a4[e], ev);
          }
        }
        const float2 s01 = __fadd2_rn(a4[0], a4[1]), s23 = __fadd2_rn(a4[2], a4[3]);
        const float2 s4 = __fadd2_rn(s01, s23);
        float sh = s4.x + s4.y;
        lin[h] = true;
        if (!(sh >= 0x1p-60f && sh <= 0x1p120f)) {
          float m = v[0];
#pragma unroll
          for (int c = 1; c < 32; ++c) m = fmaxf(m, v[c]);
          float acc = 0.f;
          if (m > 0.5f * kDeadCol)
#pragma unroll
            for (int c = 0; c < 32; ++c) acc += ex2(v[c] - m);
          sh = acc > 0.f ? m + lg2(acc) : -CUDART_INF_F;
          lin[h] = false;
        }
        part[h] = sh;
      }
      if (row_ok) {
        float Ls;
        if (lin[0] && lin[1]) {
          const float s = part[0] + part[1];
          Ls = s > 0.f ? lg2(s) : -CUDART_INF_F;
        } else {
          const float l0 = lin[0] ? (part[0] > 0.f ? lg2(part[0]) : -CUDART_INF_F) : part[0];
          const float l1 = lin[1] ? (part[1] > 0.f ? lg2(part[1]) : -CUDART_INF_F) : part[1];
          const float mx = fmaxf(l0, l1);
          Ls = mx > -CUDART_INF_F ? mx + lg2(ex2(l0 - mx) + ex2(l1 - mx)) : -CUDART_INF_F;
        }
        ws[(size_t)sbk * N + i] = (Brow > -CUDART_INF_F && cmx > -CUDART_INF_F && Ls > -CUDART_INF_F)
                                      ? Ls + crow + cmx + Brow
                                      : -CUDART_INF_F;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem),
                 "r"(kTcStages * kTcHalf));
}

}  // namespace dsmc_dev

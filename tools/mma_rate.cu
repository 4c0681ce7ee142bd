// Throughput of legacy mma.sync.m16n8k8 tf32 (warp-level, registers) on this
// GPU, alone and interleaved with MUFU.EX2 (the pass-1 mix: 2 mma + 4 ex2 +
// 2 FADD2 per 16x8 tile).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/mma_rate.cu -o tools/mma_rate
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ void mma(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ float ex2(float x) {
  float r;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

template <int MODE>
__global__ void k(float* out, int iters) {
  uint32_t a[8][4];
  for (int m = 0; m < 8; ++m)
    for (int q = 0; q < 4; ++q) a[m][q] = __float_as_uint(0.001f * (threadIdx.x + m + q));
  float c[8][4] = {};
  float2 s[8] = {};
  uint32_t b0 = __float_as_uint(0.5f), b1 = __float_as_uint(0.25f);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      float cc[4] = {0.f, 0.f, 0.f, 0.f};
      if (MODE >= 3) {
        // no MMA: arguments from the loop state (ex2 + FADD2 mix, and ex2
        // chained through its own results)
        const float x = __uint_as_float(a[m][0]) - (float)(i & 7);
        if (MODE == 3) {
          s[m] = __fadd2_rn(s[m], make_float2(ex2(x), ex2(x - 1.f)));
          s[m] = __fadd2_rn(s[m], make_float2(ex2(x - 2.f), ex2(x - 3.f)));
        } else {
          float e = ex2(ex2(ex2(ex2(x) - 1.f) - 1.f) - 1.f);
          s[m].x += e;
        }
        continue;
      }
      mma(cc, a[m], b0, b1);
      mma(cc, a[m], b1, b0);
      if (MODE == 2) {
        s[m] = __fadd2_rn(s[m], make_float2(ex2(cc[0]), ex2(cc[2])));
        s[m] = __fadd2_rn(s[m], make_float2(ex2(cc[1]), ex2(cc[3])));
      } else if (MODE == 1) {
        s[m].x += ex2(cc[0] - 30.f) + ex2(cc[1] - 30.f);
        s[m].y += ex2(cc[2] - 30.f) + ex2(cc[3] - 30.f);
      } else {
        for (int q = 0; q < 4; ++q) c[m][q] += cc[q];
      }
    }
    b0 ^= 1;
  }
  float r = 0.f;
  for (int m = 0; m < 8; ++m) r += c[m][0] + c[m][1] + c[m][2] + c[m][3] + s[m].x + s[m].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
  float* o;
  cudaMalloc(&o, 148 * 16 * 128 * 4 * 2);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2000;
  for (int mode = 0; mode < 5; ++mode) {
    for (int ctas = 4; ctas <= 8; ctas *= 2) {
      float ms = 0;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) k<0><<<148 * ctas, 128>>>(o, iters);
        else if (mode == 1) k<1><<<148 * ctas, 128>>>(o, iters);
        else if (mode == 2) k<2><<<148 * ctas, 128>>>(o, iters);
        else if (mode == 3) k<3><<<148 * ctas, 128>>>(o, iters);
        else k<4><<<148 * ctas, 128>>>(o, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
      }
      const double mmas = 148.0 * ctas * 4 * iters * 16;
      const double exps = mode ? 148.0 * ctas * 128 * iters * 8 * 4 : 0;
      printf("mode %d ctas/SM %d: %.3f ms, %.1f mma.sync per SM per us, %.3e ex2/s\n", mode, ctas,
             ms, mmas / (ms * 1e-3) / 148 / 1e6, exps / (ms * 1e-3));
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

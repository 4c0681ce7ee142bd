// Microbenchmark of the pipes that bound the pair kernel: MUFU.EX2
// (ex2.approx.ftz.f32), FP32 FFMA, packed FFMA2, FP64 DFMA. Prints JSON with
// ops/s at the clock the kernel actually ran (also sampled by the caller).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sfu_peak sfu_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) {
  float r;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

template <int KIND>
__global__ void bench(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = 0.001f * (threadIdx.x + i);
  double d[4];
  for (int i = 0; i < 4; ++i) d[i] = 1e-3 * (threadIdx.x + i);
  float2 p[4];
  for (int i = 0; i < 4; ++i) p[i] = make_float2(a[i], a[i + 4]);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 0) a[i] = ex2(a[i]) * -0.5f;                // 1 MUFU (+1 FMUL)
      if (KIND == 1) a[i] = fmaf(a[i], 0.999f, 0.001f);       // FFMA
    }
    if (KIND == 2) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        p[i] = __ffma2_rn(p[i], make_float2(0.999f, 0.999f), make_float2(0.001f, 0.001f));
    }
    if (KIND == 3) {
#pragma unroll
      for (int i = 0; i < 4; ++i) d[i] = fma(d[i], 0.999, 0.001);
    }
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  for (int i = 0; i < 4; ++i) s += p[i].x + p[i].y + (float)d[i];
  if (s == 12345.f) out[0] = s;
}

int main() {
  float* out;
  cudaMalloc(&out, 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[4] = {"ex2", "ffma", "ffma2_lanes", "dfma"};
  double per_iter[4] = {8, 8, 8, 4};  // lane-ops per iteration (ffma2: 2 lanes x 4)
  printf("{\"sms\": %d", sms);
  for (int k = 0; k < 4; ++k) {
    for (int rep = 0; rep < 2; ++rep) {  // warm then time
      cudaEventRecord(e0);
      if (k == 0) bench<0><<<blocks, threads>>>(out, iters);
      if (k == 1) bench<1><<<blocks, threads>>>(out, iters);
      if (k == 2) bench<2><<<blocks, threads>>>(out, iters);
      if (k == 3) bench<3><<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)blocks * threads * iters * per_iter[k];
    printf(", \"%s_per_s\": %.6e", names[k], ops / (ms * 1e-3));
  }
  printf("}\n");
  return 0;
}

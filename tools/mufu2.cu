// Packed ex2.approx.{bf16x2,f16x2} vs FP32 MUFU.EX2 throughput (DESIGN.md 5.1:
// all three reach the same exps/s, so packing does not help pass 1).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mufu2.cu -o tools/mufu2
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
template <int KIND>
__global__ void bench(float* out, int iters) {
  unsigned a[8];
  float f[8];
  for (int i = 0; i < 8; ++i) { f[i] = -0.001f * (threadIdx.x + i); __nv_bfloat162 v = __floats2bfloat162_rn(f[i], f[i]*0.5f); a[i] = *(unsigned*)&v; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 0) { asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i])); }
      if (KIND == 1) { asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i])); }
      if (KIND == 2) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i])); }
    }
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += (float)a[i] + f[i];
  if (s == 12345.f) out[0] = s;
}
int main() {
  float* out; cudaMalloc(&out, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* nm[3] = {"bf16x2 (values)", "f16x2 (values)", "f32"};
  for (int k = 0; k < 3; ++k) for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    if (k == 0) bench<0><<<blocks, threads>>>(out, iters);
    if (k == 1) bench<1><<<blocks, threads>>>(out, iters);
    if (k == 2) bench<2><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * iters * 8 * (k < 2 ? 2 : 1);
    if (rep) printf("%s: %.3e exp2/s\n", nm[k], ops / (ms * 1e-3));
  }
  return 0;
}

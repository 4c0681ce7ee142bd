// Philox4x64-10 throughput of one B200 (the roofline of the lazy samplers,
// which are bound by their counter-based stream draws: 3 u64 per MH step or
// rejection trial = 0.75 blocks). Each thread generates independent blocks
// with the engine's own philox() (csrc/common.cuh), 4 streams interleaved per
// thread so the integer pipes, not the dependency chains, set the rate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2202_02264_b200/csrc \
//        tools/philox_peak.cu -o tools/philox_peak
// Prints JSON: {"philox4x64_blocks_per_s": ..., "u64_per_s": ...}
#include <cstdio>
#include <cuda_runtime.h>
#include "common.cuh"
using namespace dsmc_dev;

template <int ILP>
__global__ void bench(uint64_t seed, int iters, uint64_t* out) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < ILP; ++q) {
      const U64x4 b = philox((uint64_t)it, tid, (uint64_t)q, 7, seed);
      acc ^= b.v[0] ^ b.v[1] ^ b.v[2] ^ b.v[3];
    }
  }
  if (acc == 0x123456789ull) out[0] = acc;
}

int main() {
  uint64_t* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 256, iters = 512;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 0;
  int best_cfg = 0;
  for (int bpsm : {4, 8}) {
    for (int ilp : {1, 2, 4}) {
      const int blocks = sms * bpsm;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        if (ilp == 1) bench<1><<<blocks, threads>>>(42, iters, out);
        if (ilp == 2) bench<2><<<blocks, threads>>>(42, iters, out);
        if (ilp == 4) bench<4><<<blocks, threads>>>(42, iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double bl = (double)blocks * threads * iters * ilp / (ms * 1e-3);
        if (rep) fprintf(stderr, "ctas/sm %d ilp %d: %.4e blocks/s\n", bpsm, ilp, bl);
        if (rep && bl > best) {
          best = bl;
          best_cfg = bpsm * 10 + ilp;
        }
      }
    }
  }
  printf("{\"sms\": %d, \"philox4x64_blocks_per_s\": %.6e, \"u64_per_s\": %.6e, \"best_cfg\": %d}\n",
         sms, best, 4 * best, best_cfg);
  return 0;
}

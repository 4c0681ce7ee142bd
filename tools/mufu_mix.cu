// Synthetic version of the pass-1 inner loop (no memory): per "column" and
// row pair: FADD2 bias, 4 FFMA2, 2 MUFU.EX2, FADD2 accumulate; 4 row pairs.
// Measures the ex2 rate this instruction mix reaches at a given occupancy.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float r; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }
template <int WARPS, int MINB, int BIAS, int DD>
__global__ void __launch_bounds__(32 * WARPS, MINB) mix(float* out, int iters, float seed) {
  float2 U[4][4], NC[4], S[4];
  for (int p = 0; p < 4; ++p) { for (int q = 0; q < 4; ++q) U[q][p] = make_float2(seed * (p + q), -seed * q); NC[p] = make_float2(-seed, -2 * seed); S[p] = make_float2(0, 0); }
  float4 yv = make_float4(seed, 2 * seed, 3 * seed, 4 * seed);
  float a = -seed;
  const float2 one2 = make_float2(1.f, 1.f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll 2
    for (int j = 0; j < 64; ++j) {
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        float2 t = BIAS ? __ffma2_rn(make_float2(a, a), one2, NC[p]) : make_float2(a, a);
        t = __ffma2_rn(make_float2(yv.x, yv.x), U[0][p], t);
        if (DD > 1) t = __ffma2_rn(make_float2(yv.y, yv.y), U[1][p], t);
        if (DD > 2) t = __ffma2_rn(make_float2(yv.z, yv.z), U[2][p], t);
        if (DD > 3) t = __ffma2_rn(make_float2(yv.w, yv.w), U[3][p], t);
        S[p] = __fadd2_rn(S[p], make_float2(ex2(t.x), ex2(t.y)));
      }
      yv.x += 1e-7f; a -= 1e-7f;
    }
  }
  float s = 0; for (int p = 0; p < 4; ++p) s += S[p].x + S[p].y;
  if (s == 12345.f) out[0] = s;
}
template <int W, int M, int BIAS, int DD>
void run(const char* name, float* out) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * M * 8, iters = 64;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); mix<W, M, BIAS, DD><<<blocks, 32 * W>>>(out, iters, 1e-3f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("%s: %.3e ex2/s\n", name, (double)blocks * 32 * W * iters * 64 * 8 / (ms * 1e-3));
  }
}
int main() {
  float* out; cudaMalloc(&out, 4);
  run<4, 4, 1, 4>("d=4 bias   (pass-1 mix)", out);
  run<4, 4, 0, 4>("d=4 nobias", out);
  run<4, 4, 1, 2>("d=2 bias  ", out);
  run<4, 4, 0, 2>("d=2 nobias", out);
  run<4, 4, 0, 1>("d=1 nobias", out);
  return 0;
}

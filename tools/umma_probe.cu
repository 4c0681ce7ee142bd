// Probe for the tcgen05 TF32 pair-GEMM building blocks (descriptor layout,
// TMEM alloc / ld, mbarrier commit): D[128 x 64] = A[128 x 16] . B[64 x 16]^T
// with K-major no-swizzle operands, checked against a host double GEMM of
// the TF32-truncated inputs. Also times the 3xTF32 split accuracy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/umma_probe.cu -o tools/umma_probe
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// K-major, no swizzle: element (r, k) at (r%8)*16 + (r/8)*SBO + (k/4)*LBO + (k%4)*4
__host__ __device__ inline int kmaj_off(int r, int k, int sbo, int lbo) {
  return (r & 7) * 16 + (r >> 3) * sbo + (k >> 2) * lbo + (k & 3) * 4;
}
__device__ inline uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (sm100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}

constexpr int M = 128, NC = 64, K = 16;
constexpr int SBO = 4 * 128, LBO = 128;  // 4 K-chunks of 16 B per 8-row group

__global__ void probe(const float* A, const float* B, float* D) {
  __shared__ __align__(1024) uint8_t sa[M / 8 * SBO];
  __shared__ __align__(1024) uint8_t sb[NC / 8 * SBO];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < M * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    *reinterpret_cast<float*>(sa + kmaj_off(r, k, SBO, LBO)) = A[e];
  }
  for (int e = tid; e < NC * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    *reinterpret_cast<float*>(sb + kmaj_off(r, k, SBO, LBO)) = B[e];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tbase;
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NC >> 3) << 17) |
                           ((uint32_t)(M >> 4) << 24);
    for (int ks = 0; ks < K / 8; ++ks) {
      const uint64_t da = sdesc(smem_u32(sa) + ks * 2 * LBO, LBO, SBO);
      const uint64_t db = sdesc(smem_u32(sb) + ks * 2 * LBO, LBO, SBO);
      const uint32_t acc = ks > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
  }
  // wait for phase 0
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int half = 0; half < 2; ++half) {
    uint32_t v[32];
    const uint32_t ta = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + 32 * half;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
          "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
          "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int row = 32 * (warp & 3) + lane;
    for (int c = 0; c < 32; ++c) D[row * NC + 32 * half + c] = __uint_as_float(v[c]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}

static float tf32(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u &= 0xFFFFE000u;
  float y;
  memcpy(&y, &u, 4);
  return y;
}

int main() {
  std::vector<float> A(M * K), B(NC * K), D(M * NC);
  srand(7);
  for (auto& v : A) v = (float)(rand() % 2001 - 1000) / 137.0f;
  for (auto& v : B) v = (float)(rand() % 2001 - 1000) / 91.0f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  probe<<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("CUDA error %s\n", cudaGetErrorString(e));
    return 1;
  }
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double worst = 0, worst_rel = 0;
  int bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < NC; ++j) {
      double ref = 0, mag = 0;
      for (int k = 0; k < K; ++k) {
        ref += (double)tf32(A[i * K + k]) * tf32(B[j * K + k]);
        mag += fabs((double)tf32(A[i * K + k]) * tf32(B[j * K + k]));
      }
      const double err = fabs(D[i * NC + j] - ref);
      worst = fmax(worst, err);
      worst_rel = fmax(worst_rel, err / mag);
      bad += err > 1e-5 * mag + 1e-6;
    }
  printf("umma tf32 probe: max abs err %.3g, max err / sum|terms| %.3g, bad %d of %d\n", worst,
         worst_rel, bad, M * NC);
  return bad ? 2 : 0;
}

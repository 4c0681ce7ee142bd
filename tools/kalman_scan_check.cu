// Debug harness for csrc/kalman_scan.cuh: the same element construction and
// combines on the host (sequential folds) and on the device (kernels), stage
// by stage, on arrays written by tools/kalman_debug.py (binary files in cwd).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --expt-relaxed-constexpr \
//        -I paper_2202_02264_b200/csrc -I include tools/kalman_scan_check.cu
#include <math_constants.h>
#include <cstdio>
#include <vector>
#include "engine.hpp"
#include "kalman_scan.cuh"
using namespace dsmc_dev;
template <class T> std::vector<T> rd(const char* f, size_t n) { std::vector<T> v(n); FILE* fp = fopen(f, "rb"); if (!fp) { printf("missing %s\n", f); exit(1); } fread(v.data(), sizeof(T), n, fp); fclose(fp); return v; }
template <class T> T* up(const std::vector<T>& v) { T* p; cudaMalloc(&p, v.size() * sizeof(T)); cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice); return p; }
int main() {
  const int K = 2, D = 4, DY = 2;
  auto F = rd<double>("F", 16), b = rd<double>("b", 4), Q = rd<double>("Q", 16), H = rd<double>("H", 8), R = rd<double>("R", 4);
  auto y = rd<double>("y", K * 2), m0 = rd<double>("m0", 4), P0 = rd<double>("P0", 16);
  KfModel hm{F.data(), b.data(), Q.data(), H.data(), R.data(), y.data(), m0.data(), P0.data(), 0, 0, 0, 0, 0, nullptr};
  KfModel dm{up(F), up(b), up(Q), up(H), up(R), up(y), up(m0), up(P0), 0, 0, 0, 0, 0, nullptr};
  std::vector<FiltElem<D>> fe(K);
  int bad = 0;
  for (int t = 0; t < K; ++t) kf_filter_elem<D, DY>(hm, t, fe.data(), &bad);
  FiltElem<D>* dfe; cudaMalloc(&dfe, K * sizeof(FiltElem<D>));
  int* dbad; cudaMalloc(&dbad, 4); cudaMemset(dbad, 0, 4);
  kf_filter_elems<D, DY><<<1, 128>>>(dm, K, dfe, dbad);
  std::vector<FiltElem<D>> g(K);
  cudaMemcpy(g.data(), dfe, K * sizeof(FiltElem<D>), cudaMemcpyDeviceToHost);
  double mx = 0; for (int t = 0; t < K; ++t) { const double* a = (const double*)&fe[t]; const double* c = (const double*)&g[t]; for (size_t i = 0; i < sizeof(FiltElem<D>) / 8; ++i) mx = fmax(mx, fabs(a[i] - c[i])); }
  printf("elements: max diff %g (err %s)\n", mx, cudaGetErrorString(cudaGetLastError()));
  FiltElem<D> run = fe[0]; FiltOp<D>::apply(run, fe[1], run);
  scan_chunk_apply<FiltOp<D>><<<1, 1>>>(dfe, K, nullptr);
  cudaMemcpy(g.data(), dfe, K * sizeof(FiltElem<D>), cudaMemcpyDeviceToHost);
  mx = 0; { const double* a = (const double*)&run; const double* c = (const double*)&g[1]; for (size_t i = 0; i < sizeof(FiltElem<D>) / 8; ++i) { double dd = fabs(a[i] - c[i]); if (dd > 1e-12) printf("  field %zu host %g dev %g\n", i, a[i], c[i]); mx = fmax(mx, dd); } }
  printf("combine: max diff %g (err %s)\n", mx, cudaGetErrorString(cudaGetLastError()));
  // smoother stage on the device from the device-scanned filter elements
  std::vector<FiltElem<D>> hpre = {fe[0], run};
  std::vector<SmoothElem<D>> hse(K);
  std::vector<double> hll(K);
  for (int t = 0; t < K; ++t) kf_smooth_elem<D, DY>(hm, K, t, hpre.data(), hse.data(), hll.data(), &bad);
  SmoothElem<D>* dse; cudaMalloc(&dse, K * sizeof(SmoothElem<D>));
  double* dll; cudaMalloc(&dll, K * 8);
  kf_smooth_elems<D, DY><<<1, 128>>>(dm, K, dfe, dse, dll, dbad);
  std::vector<SmoothElem<D>> gse(K);
  cudaMemcpy(gse.data(), dse, K * sizeof(SmoothElem<D>), cudaMemcpyDeviceToHost);
  int hb = 0; cudaMemcpy(&hb, dbad, 4, cudaMemcpyDeviceToHost);
  mx = 0; for (int q = 0; q < K; ++q) { const double* a = (const double*)&hse[q]; const double* c = (const double*)&gse[q]; for (size_t i = 0; i < sizeof(SmoothElem<D>) / 8; ++i) { double dd = fabs(a[i] - c[i]); if (dd > 1e-12) printf("  q %d field %zu host %g dev %g\n", q, i, a[i], c[i]); mx = fmax(mx, dd); } }
  printf("smooth elems: max diff %g bad host %d dev %d (err %s)\n", mx, bad, hb, cudaGetErrorString(cudaGetLastError()));
}

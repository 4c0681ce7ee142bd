// Device Kalman filter + RTS smoother by parallel prefix scans (proposal
// construction; the step before the leaves). The reference
// runs kalman_smooth (kalman.cpp:78-138) sequentially on the host, O(T d^3)
// with a length-T dependency chain; here both passes are associative scans
// (Sarkka & Garcia-Fernandez, "Temporal parallelization of Bayesian
// smoothers", IEEE TAC 2021), O(log T) span:
//
//   filter element of time t (model x_t = F x_{t-1} + b + N(0, Q),
//   y_t = H x_t + N(0, R)): (A, b, C, eta, J) with, for t >= 1,
//     S = H Q H' + R, K = Q H' S^-1, A = (I - K H) F, b = b_t + K (y - H b_t),
//     C = (I - K H) Q, eta = F' H' S^-1 (y - H b_t), J = F' H' S^-1 H F
//   (t = 0: the prior: A = 0, b = m0 + K0 (y - H m0), C = P0 - K0 S0 K0',
//   eta = J = 0; unobserved t: K = 0), combined (earlier i, later j) by
//     A = A_j M A_i,  b = A_j M (b_i + C_i eta_j) + b_j,
//     C = A_j M C_i A_j' + C_j,  M = (I + C_i J_j)^-1,
//     eta = A_i' N (eta_j - J_j b_i) + eta_i,  J = A_i' N J_j A_i + J_i,
//     N = (I + J_j C_i)^-1;
//   the inclusive prefix at t holds the filtered mean b and covariance C.
//
//   smoother element of time t < T: E = G_t = P_t F' Pp^-1 (Pp = F P_t F' +
//   Q, the RTS gain of kalman.cpp:125-127), g = m_t - E (F m_t + b_{t+1}),
//   L = P_t - E Pp E'; t = T: (0, m_T, P_T); combined (earlier i, later j)
//   by (E_i E_j, E_i g_j + g_i, E_i L_j E_i' + L_i); the suffix from t holds
//   the smoothed mean g and covariance L.
//
// Scans are chunked: one thread folds a chunk of kScanChunk consecutive
// elements, the chunk totals are scanned recursively, and the chunks are
// re-folded from their exclusive prefixes. FP64 throughout; covariances are
// symmetrised on output, as the reference symmetrises after every step.
// tests/test_gpu_kalman.py checks means / covariances / log-likelihood
// against the sequential host restatement (dsmc_kalman_smooth).
#pragma once

#include "kernels64.cuh"

namespace dsmc_dev {

constexpr int kScanChunk = 32;

template <int D>
struct FiltElem {
  double A[D * D], b[D], C[D * D], eta[D], J[D * D];
};
template <int D>
struct SmoothElem {
  double E[D * D], g[D], L[D * D];
};

// ---- small dense helpers (row-major, compile-time sizes)
template <int R, int K, int Cc>
__host__ __device__ inline void mm(const double* A, const double* B, double* C) {  // C = A B
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < Cc; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) s = fma(A[i * K + k], B[k * Cc + j], s);
      C[i * Cc + j] = s;
    }
}
template <int R, int K, int Cc>
__host__ __device__ inline void mmT(const double* A, const double* B, double* C) {  // C = A B'
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < Cc; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) s = fma(A[i * K + k], B[j * K + k], s);
      C[i * Cc + j] = s;
    }
}
template <int R, int K, int Cc>
__host__ __device__ inline void mTm(const double* A, const double* B, double* C) {  // C = A' B
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < Cc; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) s = fma(A[k * R + i], B[k * Cc + j], s);
      C[i * Cc + j] = s;
    }
}
template <int R, int Cc>
__host__ __device__ inline void mv(const double* A, const double* x, double* y) {
#pragma unroll
  for (int i = 0; i < R; ++i) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < Cc; ++k) s = fma(A[i * Cc + k], x[k], s);
    y[i] = s;
  }
}
template <int R, int Cc>
__host__ __device__ inline void mTv(const double* A, const double* x, double* y) {  // A' x
#pragma unroll
  for (int i = 0; i < Cc; ++i) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < R; ++k) s = fma(A[k * Cc + i], x[k], s);
    y[i] = s;
  }
}
// X := M^-1 B for an n x n M (Gauss-Jordan, partial pivoting); M is destroyed
template <int N, int Cc>
__host__ __device__ inline bool solve(double* M, double* B) {
#pragma unroll
  for (int c = 0; c < N; ++c) {
    int p = c;
    double best = fabs(M[c * N + c]);
#pragma unroll
    for (int r = c + 1; r < N; ++r)
      if (fabs(M[r * N + c]) > best) {
        best = fabs(M[r * N + c]);
        p = r;
      }
    if (!(best > 0.0)) return false;
    if (p != c) {
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const double t = M[c * N + k];
        M[c * N + k] = M[p * N + k];
        M[p * N + k] = t;
      }
#pragma unroll
      for (int k = 0; k < Cc; ++k) {
        const double t = B[c * Cc + k];
        B[c * Cc + k] = B[p * Cc + k];
        B[p * Cc + k] = t;
      }
    }
    // normalise the pivot row (M and B alike), then clear column c elsewhere
    const double inv = 1.0 / M[c * N + c];
#pragma unroll
    for (int k = 0; k < N; ++k) M[c * N + k] *= inv;
#pragma unroll
    for (int k = 0; k < Cc; ++k) B[c * Cc + k] *= inv;
#pragma unroll
    for (int r = 0; r < N; ++r) {
      if (r == c) continue;
      const double f = M[r * N + c];
      if (f == 0.0) continue;
#pragma unroll
      for (int k = 0; k < N; ++k) M[r * N + k] = fma(-f, M[c * N + k], M[r * N + k]);
#pragma unroll
      for (int k = 0; k < Cc; ++k) B[r * Cc + k] = fma(-f, B[c * Cc + k], B[r * Cc + k]);
    }
  }
  return true;
}

// ---- associative combines
template <int D>
__host__ __device__ inline void filt_combine(const FiltElem<D>& ei, const FiltElem<D>& ej,
                                    FiltElem<D>& out) {
  double M[D * D], X[D * (2 * D + 1)];
  // M = I + C_i J_j ; X = [A_i | C_i | b_i + C_i eta_j] -> M^-1 X
  mm<D, D, D>(ei.C, ej.J, M);
#pragma unroll
  for (int k = 0; k < D; ++k) M[k * D + k] += 1.0;
  double cv[D];
  mv<D, D>(ei.C, ej.eta, cv);
#pragma unroll
  for (int r = 0; r < D; ++r) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      X[r * (2 * D + 1) + k] = ei.A[r * D + k];
      X[r * (2 * D + 1) + D + k] = ei.C[r * D + k];
    }
    X[r * (2 * D + 1) + 2 * D] = ei.b[r] + cv[r];
  }
  solve<D, 2 * D + 1>(M, X);
  double MA[D * D], MC[D * D], Mb[D];
#pragma unroll
  for (int r = 0; r < D; ++r) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      MA[r * D + k] = X[r * (2 * D + 1) + k];
      MC[r * D + k] = X[r * (2 * D + 1) + D + k];
    }
    Mb[r] = X[r * (2 * D + 1) + 2 * D];
  }
  // N' = (I + J_j C_i)^-1 applied to [J_j A_i | eta_j - J_j b_i]
  double Nm[D * D], Y[D * (D + 1)];
  mm<D, D, D>(ej.J, ei.C, Nm);
#pragma unroll
  for (int k = 0; k < D; ++k) Nm[k * D + k] += 1.0;
  double JA[D * D], Jb[D];
  mm<D, D, D>(ej.J, ei.A, JA);
  mv<D, D>(ej.J, ei.b, Jb);
#pragma unroll
  for (int r = 0; r < D; ++r) {
#pragma unroll
    for (int k = 0; k < D; ++k) Y[r * (D + 1) + k] = JA[r * D + k];
    Y[r * (D + 1) + D] = ej.eta[r] - Jb[r];
  }
  solve<D, D + 1>(Nm, Y);
  double NJA[D * D], Ne[D];
#pragma unroll
  for (int r = 0; r < D; ++r) {
#pragma unroll
    for (int k = 0; k < D; ++k) NJA[r * D + k] = Y[r * (D + 1) + k];
    Ne[r] = Y[r * (D + 1) + D];
  }
  FiltElem<D> o;
  mm<D, D, D>(ej.A, MA, o.A);
  mv<D, D>(ej.A, Mb, o.b);
#pragma unroll
  for (int k = 0; k < D; ++k) o.b[k] += ej.b[k];
  double T1[D * D];
  mm<D, D, D>(ej.A, MC, T1);
  mmT<D, D, D>(T1, ej.A, o.C);
#pragma unroll
  for (int k = 0; k < D * D; ++k) o.C[k] += ej.C[k];
  mTv<D, D>(ei.A, Ne, o.eta);
#pragma unroll
  for (int k = 0; k < D; ++k) o.eta[k] += ei.eta[k];
  mTm<D, D, D>(ei.A, NJA, o.J);
#pragma unroll
  for (int k = 0; k < D * D; ++k) o.J[k] += ei.J[k];
  out = o;
}

template <int D>
__host__ __device__ inline void smooth_combine(const SmoothElem<D>& ei, const SmoothElem<D>& ej,
                                      SmoothElem<D>& out) {
  SmoothElem<D> o;
  mm<D, D, D>(ei.E, ej.E, o.E);
  mv<D, D>(ei.E, ej.g, o.g);
#pragma unroll
  for (int k = 0; k < D; ++k) o.g[k] += ei.g[k];
  double T1[D * D];
  mm<D, D, D>(ei.E, ej.L, T1);
  mmT<D, D, D>(T1, ei.E, o.L);
#pragma unroll
  for (int k = 0; k < D * D; ++k) o.L[k] += ei.L[k];
  out = o;
}

// Scan order: the filter scans forward (element q = time q, earlier first);
// the smoother scans the reversed sequence (element q = time n-1-q) and its
// combine takes (time-earlier, time-later) = (incoming, running).
template <int D>
struct FiltOp {
  using E = FiltElem<D>;
  __host__ __device__ static void apply(const E& run, const E& next, E& out) { filt_combine<D>(run, next, out); }
};
template <int D>
struct SmoothOp {
  using E = SmoothElem<D>;
  __host__ __device__ static void apply(const E& run, const E& next, E& out) {
    smooth_combine<D>(next, run, out);
  }
};

// chunk totals: agg[c] = fold of elems[c*CH .. min(n, (c+1)*CH))
template <class Op>
__global__ void scan_chunk_total(const typename Op::E* el, int n, typename Op::E* agg) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int a = c * kScanChunk;
  if (a >= n) return;
  const int b = min(n, a + kScanChunk);
  typename Op::E run = el[a];
  for (int q = a + 1; q < b; ++q) Op::apply(run, el[q], run);
  agg[c] = run;
}
// inclusive scan in place, chunk c starting from the inclusive total of the
// chunks before it (pre[c - 1]); pre == nullptr: one chunk, no prefix
template <class Op>
__global__ void scan_chunk_apply(typename Op::E* el, int n, const typename Op::E* pre) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int a = c * kScanChunk;
  if (a >= n) return;
  const int b = min(n, a + kScanChunk);
  typename Op::E run = el[a];
  if (c > 0 && pre) Op::apply(pre[c - 1], run, run);
  el[a] = run;
  for (int q = a + 1; q < b; ++q) {
    Op::apply(run, el[q], run);
    el[q] = run;
  }
}

// ---- model terms
struct KfModel {
  const double *F, *b, *Q, *H, *R, *y, *m0, *P0;
  int64_t Fs, bs, Qs, Hs, Rs;
  const uint8_t* has_obs;
};
__host__ __device__ inline const double* at_t(const double* p, int64_t s, int t) { return p + s * t; }

// x := m + K (y - H m) and the gain of an update with prior (m, P):
// S = H P H' + R, K = P H' S^-1; returns false if S is singular
template <int D, int DY>
__host__ __device__ inline bool kf_gain(const double* P, const double* H, const double* R, double* K,
                               double* S) {
  double HP[DY * D];
  mm<DY, D, D>(H, P, HP);
  mmT<DY, D, DY>(HP, H, S);
#pragma unroll
  for (int k = 0; k < DY * DY; ++k) S[k] += R[k];
  double Sc[DY * DY], X[DY * D];
#pragma unroll
  for (int k = 0; k < DY * DY; ++k) Sc[k] = S[k];
#pragma unroll
  for (int k = 0; k < DY * D; ++k) X[k] = HP[k];
  if (!solve<DY, D>(Sc, X)) return false;  // X = S^-1 H P, K = X'
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < DY; ++j) K[i * DY + j] = X[j * D + i];
  return true;
}

template <int D, int DY>
__host__ __device__ inline void kf_filter_elem(const KfModel& m, int t, FiltElem<D>* el,
                                               int* bad);
template <int D, int DY>
__global__ void kf_filter_elems(KfModel m, int K, FiltElem<D>* el, int* bad) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < K) kf_filter_elem<D, DY>(m, t, el, bad);
}
template <int D, int DY>
__host__ __device__ inline void kf_filter_elem(const KfModel& m, int t, FiltElem<D>* el,
                                               int* bad) {
  FiltElem<D> e;
#pragma unroll
  for (int k = 0; k < D * D; ++k) e.A[k] = e.C[k] = e.J[k] = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) e.b[k] = e.eta[k] = 0.0;
  const bool obs = m.has_obs ? m.has_obs[t] != 0 : true;
  const double* H = at_t(m.H, m.Hs, t);
  const double* R = at_t(m.R, m.Rs, t);
  const double* y = m.y + (size_t)t * DY;
  if (t == 0) {  // the prior N(m0, P0) updated with y_0
    double bm[D], P[D * D];
#pragma unroll
    for (int k = 0; k < D; ++k) bm[k] = m.m0[k];
#pragma unroll
    for (int k = 0; k < D * D; ++k) P[k] = m.P0[k];
    if (obs) {
      double Kg[D * DY], S[DY * DY];
      if (!kf_gain<D, DY>(P, H, R, Kg, S)) *bad = 1;
      double Hm[DY], res[DY], KS[D * DY], KSK[D * D], kr[D];
      mv<DY, D>(H, bm, Hm);
#pragma unroll
      for (int k = 0; k < DY; ++k) res[k] = y[k] - Hm[k];
      mv<D, DY>(Kg, res, kr);
      mm<D, DY, DY>(Kg, S, KS);
      mmT<D, DY, D>(KS, Kg, KSK);
#pragma unroll
      for (int k = 0; k < D; ++k) e.b[k] = bm[k] + kr[k];
#pragma unroll
      for (int k = 0; k < D * D; ++k) e.C[k] = P[k] - KSK[k];
    } else {
#pragma unroll
      for (int k = 0; k < D; ++k) e.b[k] = bm[k];
#pragma unroll
      for (int k = 0; k < D * D; ++k) e.C[k] = P[k];
    }
    el[t] = e;
    return;
  }
  const double* F = at_t(m.F, m.Fs, t);
  const double* bt = at_t(m.b, m.bs, t);
  const double* Q = at_t(m.Q, m.Qs, t);
  if (!obs) {
#pragma unroll
    for (int k = 0; k < D * D; ++k) {
      e.A[k] = F[k];
      e.C[k] = Q[k];
    }
#pragma unroll
    for (int k = 0; k < D; ++k) e.b[k] = bt[k];
    el[t] = e;
    return;
  }
  double Kg[D * DY], S[DY * DY];
  if (!kf_gain<D, DY>(Q, H, R, Kg, S)) *bad = 1;
  double IKH[D * D], KH[D * D];
  mm<D, DY, D>(Kg, H, KH);
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) IKH[i * D + j] = (i == j ? 1.0 : 0.0) - KH[i * D + j];
  mm<D, D, D>(IKH, F, e.A);
  mm<D, D, D>(IKH, Q, e.C);
  double Hb[DY], res[DY], kr[D];
  mv<DY, D>(H, bt, Hb);
#pragma unroll
  for (int k = 0; k < DY; ++k) res[k] = y[k] - Hb[k];
  mv<D, DY>(Kg, res, kr);
#pragma unroll
  for (int k = 0; k < D; ++k) e.b[k] = bt[k] + kr[k];
  // S^-1 (res) and S^-1 H F
  double HF[DY * D];
  mm<DY, D, D>(H, F, HF);
  double Sc[DY * DY], X[DY * (D + 1)];
#pragma unroll
  for (int k = 0; k < DY * DY; ++k) Sc[k] = S[k];
#pragma unroll
  for (int r = 0; r < DY; ++r) {
#pragma unroll
    for (int k = 0; k < D; ++k) X[r * (D + 1) + k] = HF[r * D + k];
    X[r * (D + 1) + D] = res[r];
  }
  if (!solve<DY, D + 1>(Sc, X)) *bad = 1;
  double SHF[DY * D], Sr[DY];
#pragma unroll
  for (int r = 0; r < DY; ++r) {
#pragma unroll
    for (int k = 0; k < D; ++k) SHF[r * D + k] = X[r * (D + 1) + k];
    Sr[r] = X[r * (D + 1) + D];
  }
  mTv<DY, D>(HF, Sr, e.eta);       // F' H' S^-1 res
  mTm<D, DY, D>(HF, SHF, e.J);     // F' H' S^-1 H F
  el[t] = e;
}

// filtered (b, C) of the prefix -> smoother elements; per-time log-likelihood
// terms of the predictive y_t ~ N(H m_pred, H P_pred H' + R)
template <int D, int DY>
__host__ __device__ inline void kf_smooth_elem(const KfModel& m, int K, int t,
                                               const FiltElem<D>* filt, SmoothElem<D>* el,
                                               double* ll_t, int* bad);
template <int D, int DY>
__global__ void kf_smooth_elems(KfModel m, int K, const FiltElem<D>* filt, SmoothElem<D>* el,
                                double* ll_t, int* bad) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < K) kf_smooth_elem<D, DY>(m, K, t, filt, el, ll_t, bad);
}
// small Cholesky (d <= 4) usable on both sides
__host__ __device__ inline bool kchol(const double* A, int d, double* L) {
  for (int i = 0; i < d * d; ++i) L[i] = 0.0;
  for (int i = 0; i < d; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = A[i * d + j];
      for (int k = 0; k < j; ++k) s -= L[i * d + k] * L[j * d + k];
      if (i == j) {
        if (!(s > 0.0)) return false;
        L[i * d + i] = sqrt(s);
      } else {
        L[i * d + j] = s / L[j * d + j];
      }
    }
  return true;
}
template <int D, int DY>
__host__ __device__ inline void kf_smooth_elem(const KfModel& m, int K, int t,
                                               const FiltElem<D>* filt, SmoothElem<D>* el,
                                               double* ll_t, int* bad) {
  const FiltElem<D>& f = filt[t];
  // predictive of time t from the filtered t - 1 (or the prior at t = 0)
  double mp[D], Pp[D * D];
  if (t == 0) {
#pragma unroll
    for (int k = 0; k < D; ++k) mp[k] = m.m0[k];
#pragma unroll
    for (int k = 0; k < D * D; ++k) Pp[k] = m.P0[k];
  } else {
    const FiltElem<D>& fp = filt[t - 1];
    const double* F = at_t(m.F, m.Fs, t);
    const double* bt = at_t(m.b, m.bs, t);
    const double* Q = at_t(m.Q, m.Qs, t);
    mv<D, D>(F, fp.b, mp);
#pragma unroll
    for (int k = 0; k < D; ++k) mp[k] += bt[k];
    double T1[D * D];
    mm<D, D, D>(F, fp.C, T1);
    mmT<D, D, D>(T1, F, Pp);
#pragma unroll
    for (int k = 0; k < D * D; ++k) Pp[k] += Q[k];
  }
  const bool obs = m.has_obs ? m.has_obs[t] != 0 : true;
  double ll = 0.0;
  if (obs) {  // log_gaussian (kalman.cpp:28-36) through a Cholesky of S
    const double* H = at_t(m.H, m.Hs, t);
    const double* R = at_t(m.R, m.Rs, t);
    double S[DY * DY], HP[DY * D], res[DY], Hm[DY], L[16];
    mm<DY, D, D>(H, Pp, HP);
    mmT<DY, D, DY>(HP, H, S);
#pragma unroll
    for (int k = 0; k < DY * DY; ++k) S[k] += R[k];
    mv<DY, D>(H, mp, Hm);
#pragma unroll
    for (int k = 0; k < DY; ++k) res[k] = m.y[(size_t)t * DY + k] - Hm[k];
    if (!kchol(S, DY, L)) *bad = 1;
    double ld = 0.0, q = 0.0, z[DY];
#pragma unroll
    for (int i = 0; i < DY; ++i) {
      double s = res[i];
      for (int k = 0; k < i; ++k) s -= L[i * DY + k] * z[k];
      z[i] = s / L[i * DY + i];
      q += z[i] * z[i];
      ld += 2.0 * log(L[i * DY + i]);
    }
    ll = -0.5 * (DY * kLog2Pi + ld + q);
  }
  ll_t[t] = ll;
  SmoothElem<D> e;
  if (t == K - 1) {
#pragma unroll
    for (int k = 0; k < D * D; ++k) {
      e.E[k] = 0.0;
      e.L[k] = f.C[k];
    }
#pragma unroll
    for (int k = 0; k < D; ++k) e.g[k] = f.b[k];
  } else {
    // G = P F' Pp1^-1 with Pp1 = F_{t+1} P F_{t+1}' + Q_{t+1} (kalman.cpp:125-127)
    const double* F = at_t(m.F, m.Fs, t + 1);
    const double* b1 = at_t(m.b, m.bs, t + 1);
    const double* Q = at_t(m.Q, m.Qs, t + 1);
    double FP[D * D], Pp1[D * D], Pc[D * D];
    mm<D, D, D>(F, f.C, FP);
    mmT<D, D, D>(FP, F, Pp1);
#pragma unroll
    for (int k = 0; k < D * D; ++k) {
      Pp1[k] += Q[k];
      Pc[k] = Pp1[k];
    }
    double X[D * D];  // Pp1^-1 (F P) = G'  (P, Pp1 symmetric)
#pragma unroll
    for (int k = 0; k < D * D; ++k) X[k] = FP[k];
    if (!solve<D, D>(Pc, X)) *bad = 1;
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) e.E[i * D + j] = X[j * D + i];
    double Fm[D], Em[D];
    mv<D, D>(F, f.b, Fm);
#pragma unroll
    for (int k = 0; k < D; ++k) Fm[k] += b1[k];
    mv<D, D>(e.E, Fm, Em);
#pragma unroll
    for (int k = 0; k < D; ++k) e.g[k] = f.b[k] - Em[k];
    double EP[D * D], EPE[D * D];
    mm<D, D, D>(e.E, Pp1, EP);
    mmT<D, D, D>(EP, e.E, EPE);
#pragma unroll
    for (int k = 0; k < D * D; ++k) e.L[k] = f.C[k] - EPE[k];
  }
  el[K - 1 - t] = e;  // reversed: the smoother scans from time T down
}

template <int D>
__global__ void kf_outputs(int K, const SmoothElem<D>* el, double* mean, double* cov) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= K) return;
  const SmoothElem<D>& e = el[K - 1 - t];
#pragma unroll
  for (int k = 0; k < D; ++k) mean[(size_t)t * D + k] = e.g[k];
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j)
      cov[((size_t)t * D + i) * D + j] = 0.5 * (e.L[i * D + j] + e.L[j * D + i]);
}

}  // namespace dsmc_dev

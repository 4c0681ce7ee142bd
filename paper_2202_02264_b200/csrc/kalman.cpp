// Host Kalman filter + RTS smoother for LGSSM descriptors (d, dy <= 4).
// Proposal construction, the step before the leaves: the
// reference builds q_t = nu_t from kalman_smooth (kalman.cpp:78-138) in the
// harness's prepare() (experiment.cpp:449-456). Eigen-free restatement with
// fixed-size arrays: Joseph-form update, RTS gain solved against the
// predicted covariance, symmetrisation after every step, jitter-escalating
// Cholesky (kalman.cpp:15-26).
#include <cmath>
#include <cstring>
#include <vector>

#include "dsmc_b200.h"

namespace {

constexpr double kLog2Pi = 1.8378770664093454836;

struct Mat {
  int r = 0, c = 0;
  double a[16] = {0};
  double& operator()(int i, int j) { return a[i * c + j]; }
  double operator()(int i, int j) const { return a[i * c + j]; }
};

Mat make(int r, int c) {
  Mat m;
  m.r = r;
  m.c = c;
  return m;
}
Mat load(const double* p, int r, int c) {
  Mat m = make(r, c);
  std::memcpy(m.a, p, sizeof(double) * r * c);
  return m;
}
Mat mul(const Mat& A, const Mat& B) {
  Mat C = make(A.r, B.c);
  for (int i = 0; i < A.r; ++i)
    for (int j = 0; j < B.c; ++j) {
      double s = 0.0;
      for (int k = 0; k < A.c; ++k) s += A(i, k) * B(k, j);
      C(i, j) = s;
    }
  return C;
}
Mat tr(const Mat& A) {
  Mat C = make(A.c, A.r);
  for (int i = 0; i < A.r; ++i)
    for (int j = 0; j < A.c; ++j) C(j, i) = A(i, j);
  return C;
}
Mat add(const Mat& A, const Mat& B, double s = 1.0) {
  Mat C = A;
  for (int i = 0; i < A.r * A.c; ++i) C.a[i] = A.a[i] + s * B.a[i];
  return C;
}
void sym(Mat& P) {
  for (int i = 0; i < P.r; ++i)
    for (int j = 0; j < i; ++j) {
      const double v = (P(i, j) + P(j, i)) * 0.5;
      P(i, j) = P(j, i) = v;
    }
}
// kalman.cpp:15-26
bool robust_chol(Mat P, Mat& L) {
  sym(P);
  double trace = 0.0;
  for (int i = 0; i < P.r; ++i) trace += P(i, i);
  const double scale = std::fmax(trace / P.r, 1e-300);
  for (int attempt = 0; attempt < 4; ++attempt) {
    L = make(P.r, P.r);
    bool ok = true;
    for (int i = 0; i < P.r && ok; ++i)
      for (int j = 0; j <= i; ++j) {
        double s = P(i, j);
        for (int k = 0; k < j; ++k) s -= L(i, k) * L(j, k);
        if (i == j) {
          if (!(s > 0.0)) {
            ok = false;
            break;
          }
          L(i, i) = std::sqrt(s);
        } else {
          L(i, j) = s / L(j, j);
        }
      }
    if (ok) return true;
    for (int i = 0; i < P.r; ++i) P(i, i) += scale * std::pow(10.0, attempt - 12);
  }
  return false;
}
// Solve (L L^T) X = B.
Mat chol_solve(const Mat& L, const Mat& B) {
  Mat X = B;
  const int n = L.r;
  for (int col = 0; col < B.c; ++col) {
    for (int i = 0; i < n; ++i) {
      double s = X(i, col);
      for (int k = 0; k < i; ++k) s -= L(i, k) * X(k, col);
      X(i, col) = s / L(i, i);
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = X(i, col);
      for (int k = i + 1; k < n; ++k) s -= L(k, i) * X(k, col);
      X(i, col) = s / L(i, i);
    }
  }
  return X;
}

}  // namespace

extern "C" DSMC_API int dsmc_kalman_smooth(const dsmc_model_desc* m,
                                           double* smooth_mean,
                                           double* smooth_cov, double* loglik) {
  if (!m || m->kind != DSMC_MODEL_LGSSM) return DSMC_E_INVALID_ARGUMENT;
  const int d = m->state_dim, dy = m->obs_dim, T = m->horizon;
  if (d < 1 || d > 4 || dy < 1 || dy > 4 || T < 0) return DSMC_E_INVALID_ARGUMENT;
  const int K = T + 1;
  std::vector<Mat> pm(K), pP(K), fm(K), fP(K);
  double ll = 0.0;
  const Mat I = [&] {
    Mat e = make(d, d);
    for (int i = 0; i < d; ++i) e(i, i) = 1.0;
    return e;
  }();
  for (int t = 0; t < K; ++t) {
    if (t == 0) {
      pm[0] = load(m->m0, d, 1);
      pP[0] = load(m->P0, d, d);
    } else {
      const Mat F = load(m->F + m->F_stride * t, d, d);
      const Mat b = load(m->b + m->b_stride * t, d, 1);
      const Mat Q = load(m->Q + m->Q_stride * t, d, d);
      pm[t] = add(mul(F, fm[t - 1]), b);
      pP[t] = add(mul(mul(F, fP[t - 1]), tr(F)), Q);
      sym(pP[t]);
    }
    const bool obs = m->has_obs ? m->has_obs[t] != 0 : true;
    if (obs) {
      const Mat H = load(m->H + m->H_stride * t, dy, d);
      const Mat R = load(m->R + m->R_stride * t, dy, dy);
      const Mat y = load(m->y + (size_t)t * dy, dy, 1);
      const Mat resid = add(y, mul(H, pm[t]), -1.0);
      const Mat S = add(mul(mul(H, pP[t]), tr(H)), R);
      Mat L;
      if (!robust_chol(S, L)) return DSMC_E_RUNTIME;
      // log N(resid; 0, S) (kalman.cpp:28-36)
      double ld = 0.0;
      for (int i = 0; i < dy; ++i) ld += 2.0 * std::log(L(i, i));
      Mat z = resid;
      for (int i = 0; i < dy; ++i) {
        double s = z(i, 0);
        for (int k = 0; k < i; ++k) s -= L(i, k) * z(k, 0);
        z(i, 0) = s / L(i, i);
      }
      double zz = 0.0;
      for (int i = 0; i < dy; ++i) zz += z(i, 0) * z(i, 0);
      ll += -0.5 * (dy * kLog2Pi + ld + zz);
      const Mat Kg = tr(chol_solve(L, mul(H, pP[t])));  // d x dy
      fm[t] = add(pm[t], mul(Kg, resid));
      const Mat A = add(I, mul(Kg, H), -1.0);
      fP[t] = add(mul(mul(A, pP[t]), tr(A)), mul(mul(Kg, R), tr(Kg)));
      sym(fP[t]);
    } else {
      fm[t] = pm[t];
      fP[t] = pP[t];
    }
  }
  std::vector<Mat> sm(K), sP(K);
  sm[T] = fm[T];
  sP[T] = fP[T];
  for (int t = T - 1; t >= 0; --t) {
    const Mat F = load(m->F + m->F_stride * (t + 1), d, d);
    Mat L;
    if (!robust_chol(pP[t + 1], L)) return DSMC_E_RUNTIME;
    const Mat G = tr(chol_solve(L, mul(F, tr(fP[t]))));
    sm[t] = add(fm[t], mul(G, add(sm[t + 1], pm[t + 1], -1.0)));
    sP[t] = add(fP[t], mul(mul(G, add(sP[t + 1], pP[t + 1], -1.0)), tr(G)));
    sym(sP[t]);
  }
  for (int t = 0; t < K; ++t) {
    if (smooth_mean) std::memcpy(smooth_mean + (size_t)t * d, sm[t].a, sizeof(double) * d);
    if (smooth_cov) std::memcpy(smooth_cov + (size_t)t * d * d, sP[t].a, sizeof(double) * d * d);
  }
  if (loglik) *loglik = ll;
  return DSMC_OK;
}

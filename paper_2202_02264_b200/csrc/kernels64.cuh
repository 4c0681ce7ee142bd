// FP64 device kernels: model prep, leaves, the parity dense combine, lazy
// samplers. Every FP64 operation that the reference performs without FMA is
// written with __dadd_rn/__dmul_rn/__ddiv_rn so nvcc cannot contract it;
// explicit FMAs are __fma_rn, exactly where the reference calls std::fma.
#pragma once

#include "engine.hpp"

namespace dsmc_dev {

#define DADD __dadd_rn
#define DSUB __dsub_rn
#define DMUL __dmul_rn
#define DDIV __ddiv_rn

enum ModelClass { kLG1 = 0, kSV = 1, kLGN = 2, kCOX = 3, kCRW = 4, kTHETA = 5 };

__host__ __device__ inline int model_class(int kind, int d, int dy) {
  if (kind == DSMC_MODEL_SV) return kSV;
  if (kind == DSMC_MODEL_COX) return kCOX;
  if (kind == DSMC_MODEL_CRW) return kCRW;
  if (kind == DSMC_MODEL_THETA) return kTHETA;
  return (d == 1 && dy == 1) ? kLG1 : kLGN;
}
// models.cpp:361-363: x + tau0 - tau1 exp(tau2 x)
__device__ inline double theta_drift(const DevModel& M, double x) {
  return DSUB(DADD(x, M.mp[0]), DMUL(M.mp[1], exp(DMUL(M.mp[2], x))));
}
// models.cpp:260: in_box; :274 kLogHalf
__device__ inline bool crw_in_box(double x) { return x >= -1.0 && x <= 1.0; }
constexpr double kLogHalf = -0.6931471805599453;
// models.cpp:103-106: y x - exp(x) - lgamma(y + 1)
__device__ inline double cox_log_poisson(const DevModel& M, int t, double x) {
  return DSUB(DSUB(DMUL(M.y[t], x), exp(x)), M.lgam[t]);
}

// ----------------------------------------------------------- small LA
// Same algorithms and operation order as oracle/dsmc_oracle.c chol/tri_inv.
__device__ inline bool dchol(const double* A, int d, double* L) {
  for (int i = 0; i < d * d; ++i) L[i] = 0.0;
  for (int i = 0; i < d; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = A[i * d + j];
      for (int k = 0; k < j; ++k) s = DSUB(s, DMUL(L[i * d + k], L[j * d + k]));
      if (i == j) {
        if (!(s > 0.0)) return false;
        L[i * d + i] = __dsqrt_rn(s);
      } else {
        L[i * d + j] = DDIV(s, L[j * d + j]);
      }
    }
  return true;
}
__device__ inline void dtri_inv(const double* L, int d, double* W) {
  for (int i = 0; i < d * d; ++i) W[i] = 0.0;
  for (int i = 0; i < d; ++i) {
    W[i * d + i] = DDIV(1.0, L[i * d + i]);
    for (int j = 0; j < i; ++j) {
      double s = 0.0;
      for (int k = j; k < i; ++k) s = DADD(s, DMUL(L[i * d + k], W[k * d + j]));
      W[i * d + j] = DDIV(-s, L[i * d + i]);
    }
  }
}
__device__ inline double dnorm_of(const double* L, int d) {
  double ld = 0.0;
  for (int i = 0; i < d; ++i) ld = DADD(ld, DMUL(2.0, log(L[i * d + i])));
  return DMUL(-0.5, DADD(DMUL((double)d, kLog2Pi), ld));
}
// |W (x - m)|^2, W lower (oracle gauss_quad order).
__device__ inline double dquad(const double* W, int d, const double* x,
                               const double* m) {
  double e[4], q = 0.0;
  for (int k = 0; k < d; ++k) e[k] = DSUB(x[k], m[k]);
  for (int k = 0; k < d; ++k) {
    double z = 0.0;
    for (int l = 0; l <= k; ++l) z = DADD(z, DMUL(W[k * d + l], e[l]));
    q = DADD(q, DMUL(z, z));
  }
  return q;
}
// models.cpp:20-23
__device__ inline double dlog_normal_pdf(double x, double mean, double var) {
  const double dd = DSUB(x, mean);
  return DSUB(DMUL(-0.5, DADD(kLog2Pi, log(var))),
              DDIV(DMUL(dd, dd), DMUL(2.0, var)));
}

__device__ inline const double* at(const double* p, int64_t s, int t) {
  return p + s * t;
}

// ------------------------------------------------------------------ prep
// Per-time constants (TimeConst) of chain `ch`, one thread per time.
__global__ void prep_kernel(const DevModel* models, TimeConst* tc_all, int K,
                            int* bounded_all, int t_begin = 0, int t_end = 1 << 30) {
  const int ch = blockIdx.y;
  const int t = t_begin + blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= K || t >= t_end) return;
  const DevModel M = models[ch];
  TimeConst tc;
  for (int i = 0; i < 4; ++i) tc.pm[i] = tc.delta[i] = tc.e[i] = 0.0;
  for (int i = 0; i < 16; ++i)
    tc.pL[i] = tc.pW[i] = tc.tW[i] = tc.F[i] = tc.oW[i] = tc.G[i] = 0.0;
  tc.p_norm = tc.t_norm = tc.o_norm = tc.cconst = tc.shift1 = 0.0;
  tc.bound = CUDART_NAN;
  tc.logabsy = 0.0;
  tc.obs = 0;
  tc.bounded = 0;
  tc.drift = 0;
  for (int i = 0; i < 4; ++i) tc.th[i] = 0.0;
  const int d = M.d, dy = M.dy;
  if (M.kind == DSMC_MODEL_THETA) {
    // Gaussian proposal / observation (h = 1) constants as for the LGSSM FP32
    // leaves; the row term is the nonlinear drift (no F / delta)
    const double m = M.prop_mean[t], v = M.prop_cov[t];
    tc.pm[0] = m;
    tc.pL[0] = __dsqrt_rn(v);
    tc.pW[0] = DDIV(1.0, tc.pL[0]);
    tc.p_norm = DMUL(-0.5, DADD(kLog2Pi, log(v)));
    tc.obs = 1;
    tc.o_norm = M.mp[6];
    tc.oW[0] = DDIV(1.0, __dsqrt_rn(M.mp[4]));
    tc.e[0] = DMUL(tc.oW[0], DSUB(M.y[t], m));
    tc.G[0] = DMUL(tc.oW[0], tc.pL[0]);
    tc.t_norm = M.mp[5];
    tc.tW[0] = DDIV(1.0, __dsqrt_rn(M.mp[3]));
    tc.cconst = DADD(DSUB(tc.o_norm, tc.p_norm), t >= 1 ? tc.t_norm : 0.0);
    // models.cpp:454-457 (same expression order): obs_norm + 0.5 (log 2 pi +
    // log var) + trans_norm
    tc.shift1 = DADD(DADD(M.mp[6], DMUL(0.5, DADD(kLog2Pi, log(v)))), M.mp[5]);
    tc.drift = 1;
    tc.th[0] = M.mp[0];
    tc.th[1] = M.mp[1];
    tc.th[2] = M.mp[2];
    tc.th[3] = t >= 1 ? M.prop_mean[t - 1] : 0.0;
    if (t >= 1) {  // models.cpp:473-483: obs_over_aux_sup(y, 1, r2, m, v)
      const double y = M.y[t], r2 = M.mp[4];
      const double alpha = DSUB(DDIV(1.0, DMUL(2.0, v)), DDIV(1.0, DMUL(2.0, r2)));
      const double beta = DSUB(DDIV(y, r2), DDIV(m, v));
      const double gamma = DADD(DADD(DDIV(DMUL(-y, y), DMUL(2.0, r2)), DDIV(DMUL(m, m), DMUL(2.0, v))),
                                DMUL(0.5, log(DDIV(v, r2))));
      double sv;
      if (alpha < 0.0) sv = DSUB(gamma, DDIV(DMUL(beta, beta), DMUL(4.0, alpha)));
      else if (alpha == 0.0 && beta == 0.0) sv = gamma;
      else sv = CUDART_INF;
      tc.bounded = isfinite(sv);
      if (tc.bounded) tc.bound = DADD(M.mp[5], sv);
      if (!tc.bounded) atomicAnd(bounded_all + ch, ~1);
    }
  } else if (M.kind == DSMC_MODEL_COX || M.kind == DSMC_MODEL_CRW) {
    // d = 1 Gaussian-transition models with host-computed constants (mp):
    // centre = proposal mean, whitening = 1 / transition sd
    const bool cox = M.kind == DSMC_MODEL_COX;
    const double m = cox ? M.mp[2] : 0.0;
    tc.pm[0] = m;
    tc.pL[0] = cox ? M.mp[6] : 1.0;
    tc.pW[0] = DDIV(1.0, tc.pL[0]);
    tc.t_norm = cox ? M.mp[4] : M.mp[1];
    tc.tW[0] = DDIV(1.0, cox ? __dsqrt_rn(M.mp[5]) : M.mp[2]);
    tc.F[0] = cox ? M.mp[0] : 1.0;
    // centring offset F m + b - m of the transition into t
    tc.delta[0] = cox ? DSUB(DADD(DMUL(M.mp[0], m), M.mp[1]), m) : 0.0;
    tc.obs = 1;
    if (!cox && t >= 1) {  // models.cpp:334-335
      tc.bound = DSUB(M.mp[1], kLogHalf);
      tc.bounded = 1;
    }
    if (t >= 1 && !tc.bounded) atomicAnd(bounded_all + ch, ~1);
  } else if (M.kind == DSMC_MODEL_SV) {
    const double y = M.y[t];
    tc.logabsy = log(fabs(y));
    tc.obs = 1;
    const double tn = DMUL(-0.5, DADD(kLog2Pi, log(M.sv_s2)));
    tc.t_norm = tn;
    tc.shift1 = DSUB(tn, tc.logabsy);
    tc.bound = tc.shift1;
    tc.bounded = (y != 0.0) && isfinite(y);
    tc.tW[0] = DDIV(1.0, __dsqrt_rn(M.sv_s2));
    tc.F[0] = M.sv_phi;
    tc.delta[0] = DMUL(M.sv_mu, DSUB(1.0, M.sv_phi));
    tc.cconst = tc.shift1;
    tc.pL[0] = 1.0;
    if (!tc.bounded) atomicAnd(bounded_all + ch, ~1);
  } else {
    const double* pm = M.prop_mean + (size_t)t * d;
    for (int k = 0; k < d; ++k) tc.pm[k] = pm[k];
    bool ok = dchol(M.prop_cov + (size_t)t * d * d, d, tc.pL);
    dtri_inv(tc.pL, d, tc.pW);
    tc.p_norm = dnorm_of(tc.pL, d);
    tc.obs = M.has_obs ? (M.has_obs[t] != 0) : 1;
    double L[16];
    if (tc.obs) {
      ok = ok && dchol(at(M.R, M.R_s, t), dy, L);
      dtri_inv(L, dy, tc.oW);
      tc.o_norm = dnorm_of(L, dy);
      const double* H = at(M.H, M.H_s, t);
      const double* y = M.y + (size_t)t * dy;
      double r[4], HL[16];
      for (int a = 0; a < dy; ++a) {
        double s = 0.0;
        for (int l = 0; l < d; ++l) s = DADD(s, DMUL(H[a * d + l], pm[l]));
        r[a] = DSUB(y[a], s);
        for (int l = 0; l < d; ++l) {
          double h = 0.0;
          for (int m = l; m < d; ++m) h = DADD(h, DMUL(H[a * d + m], tc.pL[m * d + l]));
          HL[a * d + l] = h;
        }
      }
      for (int a = 0; a < dy; ++a) {
        double z = 0.0;
        for (int b = 0; b <= a; ++b) z = DADD(z, DMUL(tc.oW[a * dy + b], r[b]));
        tc.e[a] = z;
        for (int l = 0; l < d; ++l) {
          double g = 0.0;
          for (int b = 0; b <= a; ++b) g = DADD(g, DMUL(tc.oW[a * dy + b], HL[b * d + l]));
          tc.G[a * d + l] = g;
        }
      }
    }
    if (t >= 1) {
      ok = ok && dchol(at(M.Q, M.Q_s, t), d, L);
      dtri_inv(L, d, tc.tW);
      tc.t_norm = dnorm_of(L, d);
      const double* F = at(M.F, M.F_s, t);
      const double* b = at(M.b, M.b_s, t);
      const double* pmp = M.prop_mean + (size_t)(t - 1) * d;
      for (int k = 0; k < d * d; ++k) tc.F[k] = F[k];
      for (int k = 0; k < d; ++k) {
        double s = 0.0;
        for (int l = 0; l < d; ++l) s = DADD(s, DMUL(F[k * d + l], pmp[l]));
        tc.delta[k] = DSUB(DADD(s, b[k]), pm[k]);
      }
    }
    tc.cconst = DADD(DSUB(tc.obs ? tc.o_norm : 0.0, tc.p_norm), t >= 1 ? tc.t_norm : 0.0);
    if (d == 1 && dy == 1 && t >= 1) {
      // models.cpp:613-624 (same expression order).
      const double qvar = *at(M.Q, M.Q_s, t);
      const double var = M.prop_cov[t];
      const double trans_norm = DMUL(-0.5, DADD(kLog2Pi, log(qvar)));
      double shift = DADD(trans_norm, DMUL(0.5, DADD(kLog2Pi, log(var))));
      if (tc.obs) {
        const double r = *at(M.R, M.R_s, t);
        shift = DADD(shift, DMUL(-0.5, DADD(kLog2Pi, log(r))));
      }
      tc.shift1 = shift;
      // models.cpp:657-676: bound only if observed, sloped and the proposal
      // is wider than the likelihood curvature.
      const double F1 = *at(M.F, M.F_s, t);
      bool bnd = tc.obs && F1 != 0.0;
      if (bnd) {
        const double h = *at(M.H, M.H_s, t), r2 = *at(M.R, M.R_s, t);
        const double yy = M.y[t], m = pm[0], v = var;
        const double alpha = DSUB(DDIV(1.0, DMUL(2.0, v)), DDIV(DMUL(h, h), DMUL(2.0, r2)));
        const double beta = DSUB(DDIV(DMUL(h, yy), r2), DDIV(m, v));
        const double gamma = DADD(DADD(DDIV(DMUL(-yy, yy), DMUL(2.0, r2)),
                                       DDIV(DMUL(m, m), DMUL(2.0, v))),
                                  DMUL(0.5, log(DDIV(v, r2))));
        double s;
        if (alpha < 0.0) s = DSUB(gamma, DDIV(DMUL(beta, beta), DMUL(4.0, alpha)));
        else if (alpha == 0.0 && beta == 0.0) s = gamma;
        else s = CUDART_INF;
        bnd = isfinite(s);
        if (bnd) tc.bound = DADD(DMUL(-0.5, DADD(kLog2Pi, log(qvar))), s);
      }
      tc.bounded = bnd;
    }
    if (t >= 1 && !tc.bounded) atomicAnd(bounded_all + ch, ~1);
    if (!ok) atomicAnd(bounded_all + ch, ~2);  // bit 1 clear = SPD failure
  }
  tc_all[(size_t)ch * K + t] = tc;
}

// ------------------------------------------------------- FP64 callbacks
// Scalar model callbacks (the reference's std::function callbacks restated
// per model class; fk_model.cpp / oracle ref_models.cpp).
__device__ inline double cb_log_h(const DevModel& M, const TimeConst& tc,
                                  int t, const double* x) {
  if (M.kind == DSMC_MODEL_COX) return cox_log_poisson(M, t, x[0]);
  if (M.kind == DSMC_MODEL_CRW) return crw_in_box(x[0]) ? 0.0 : -CUDART_INF;
  if (M.kind == DSMC_MODEL_THETA) return dlog_normal_pdf(M.y[t], x[0], M.mp[4]);
  if (M.kind == DSMC_MODEL_SV) {
    const double y = M.y[t];
    return DSUB(DMUL(-0.5, DADD(kLog2Pi, x[0])), DDIV(DMUL(y, y), DMUL(2.0, exp(x[0]))));
  }
  if (!tc.obs) return 0.0;
  const double* H = at(M.H, M.H_s, t);
  if (M.d == 1 && M.dy == 1)
    return dlog_normal_pdf(M.y[t], DMUL(H[0], x[0]), *at(M.R, M.R_s, t));
  double hx[4];
  for (int a = 0; a < M.dy; ++a) {
    double s = 0.0;
    for (int l = 0; l < M.d; ++l) s = DADD(s, DMUL(H[a * M.d + l], x[l]));
    hx[a] = s;
  }
  return DSUB(tc.o_norm, DMUL(0.5, dquad(tc.oW, M.dy, M.y + (size_t)t * M.dy, hx)));
}
__device__ inline double cb_prop_logdensity(const DevModel& M,
                                            const TimeConst& tc, int t,
                                            const double* x) {
  if (M.kind == DSMC_MODEL_SV) return DADD(tc.logabsy, cb_log_h(M, tc, t, x));
  if (M.kind == DSMC_MODEL_COX) return dlog_normal_pdf(x[0], M.mp[2], M.mp[3]);
  if (M.kind == DSMC_MODEL_CRW) return crw_in_box(x[0]) ? kLogHalf : -CUDART_INF;
  if (M.kind == DSMC_MODEL_THETA || (M.d == 1 && M.dy == 1))
    return dlog_normal_pdf(x[0], M.prop_mean[t], M.prop_cov[t]);
  return DSUB(tc.p_norm, DMUL(0.5, dquad(tc.pW, M.d, x, tc.pm)));
}
__device__ inline double cb_init_logdensity(const DevModel& M,
                                            const TimeConst& tc0,
                                            const double* x, const double* W0,
                                            double norm0) {
  if (M.kind == DSMC_MODEL_SV)
    return dlog_normal_pdf(x[0], M.sv_mu,
                           DDIV(M.sv_s2, DSUB(1.0, DMUL(M.sv_phi, M.sv_phi))));
  if (M.kind == DSMC_MODEL_COX) return dlog_normal_pdf(x[0], M.mp[2], M.mp[3]);
  if (M.kind == DSMC_MODEL_CRW || M.kind == DSMC_MODEL_THETA) return dlog_normal_pdf(x[0], 0.0, 1.0);
  if (M.d == 1 && M.dy == 1) return dlog_normal_pdf(x[0], M.m0[0], M.P0[0]);
  return DSUB(norm0, DMUL(0.5, dquad(W0, M.d, x, M.m0)));
}
__device__ inline void lg_mean(const DevModel& M, int t, const double* xp,
                               double* mu) {
  const double* F = at(M.F, M.F_s, t);
  const double* b = at(M.b, M.b_s, t);
  for (int k = 0; k < M.d; ++k) {
    double s = 0.0;
    for (int l = 0; l < M.d; ++l) s = DADD(s, DMUL(F[k * M.d + l], xp[l]));
    mu[k] = DADD(s, b[k]);
  }
}
__device__ inline double cb_transition(const DevModel& M, const TimeConst& tc,
                                       int t, const double* xp,
                                       const double* xc) {
  if (M.kind == DSMC_MODEL_SV)
    return dlog_normal_pdf(xc[0], DADD(M.sv_mu, DMUL(M.sv_phi, DSUB(xp[0], M.sv_mu))),
                           M.sv_s2);
  if (M.kind == DSMC_MODEL_COX)  // models.cpp:163-165
    return dlog_normal_pdf(xc[0], DADD(M.mp[1], DMUL(M.mp[0], xp[0])), M.mp[5]);
  if (M.kind == DSMC_MODEL_CRW)  // models.cpp:292-294
    return dlog_normal_pdf(xc[0], xp[0], M.mp[0]);
  if (M.kind == DSMC_MODEL_THETA)  // models.cpp:443-445
    return dlog_normal_pdf(xc[0], theta_drift(M, xp[0]), M.mp[3]);
  if (M.d == 1 && M.dy == 1)
    return dlog_normal_pdf(xc[0], DADD(DMUL(*at(M.F, M.F_s, t), xp[0]), *at(M.b, M.b_s, t)),
                           *at(M.Q, M.Q_s, t));
  double mu[4];
  lg_mean(M, t, xp, mu);
  return DSUB(tc.t_norm, DMUL(0.5, dquad(tc.tW, M.d, xc, mu)));
}
// log_stitch_weight (fk_model.cpp:61-73); returns NaN-coded errors via flag.
__device__ inline double cb_stitch_weight(const DevModel& M,
                                          const TimeConst& tc, int c,
                                          const double* xp, const double* xc,
                                          int* err) {
  const double tr = cb_transition(M, tc, c, xp, xc);
  const double pot = cb_log_h(M, tc, c, xc);
  if (tr == -CUDART_INF || pot == -CUDART_INF) return -CUDART_INF;
  const double nu = cb_prop_logdensity(M, tc, c, xc);
  if (nu == -CUDART_INF) {
    *err = DSMC_E_INVALID_ARGUMENT;
    return CUDART_NAN;
  }
  return DSUB(DADD(tr, pot), nu);
}

}  // namespace dsmc_dev

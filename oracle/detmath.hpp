// ORACLE — test infrastructure only. Never linked into the product.
//
// Deterministic scalar kernels used by the oracle's restatement of the
// reference path. Every function here is built from IEEE-754 correctly rounded
// operations only (+ - * / sqrt, explicit fma), so the CUDA implementation in
// paper_1810_12163_b200/csrc/ (an independent re-implementation of the same
// definitions) can be compared bit-for-bit. The definitions are frozen in
// DESIGN.md §"Numerics contract".
//
//   det_expf     exp(x) for x <= 0 (RQS density kernel)
//   det_sincos   sin/cos in double (exp_se3, geometry.hpp:97-103)
//   svd3_jacobi  one-sided Jacobi SVD of a 3x3 (stands in for Eigen::JacobiSVD,
//                geometry.hpp:180; the rotation Kabsch returns is unique for
//                non-degenerate input, so any correct SVD reproduces it)
//   eig3_jacobi  cyclic Jacobi eigen-decomposition of a symmetric 3x3
//   chol6_solve  Cholesky solve of a 6x6 SPD system
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>

namespace oracle {

inline float det_expf(float x) {
  if (!(x > -87.0f)) return 0.0f;  // also maps NaN to 0
  if (x > 0.0f) x = 0.0f;
  const float kf = std::nearbyint(x * 1.44269504088896341f);
  float r = std::fma(kf, -0.693145751953125f, x);
  r = std::fma(kf, -1.428606765330187045e-06f, r);
  float p = 1.98412698e-4f;  // 1/5040
  p = std::fma(p, r, 1.38888889e-3f);
  p = std::fma(p, r, 8.33333333e-3f);
  p = std::fma(p, r, 4.16666667e-2f);
  p = std::fma(p, r, 1.66666667e-1f);
  p = std::fma(p, r, 0.5f);
  p = std::fma(p, r, 1.0f);
  p = std::fma(p, r, 1.0f);
  const int k = static_cast<int>(kf);
  uint32_t bits = static_cast<uint32_t>(k + 127) << 23;
  float scale;
  std::memcpy(&scale, &bits, 4);
  return p * scale;
}

// fdlibm-style kernels on [-pi/4, pi/4] with a Cody-Waite reduction by pi/2.
inline double det_ksin(double x) {
  const double S1 = -1.66666666666666324348e-01, S2 = 8.33333333332248946124e-03,
               S3 = -1.98412698298579493134e-04, S4 = 2.75573137070700676789e-06,
               S5 = -2.50507602534068634195e-08, S6 = 1.58969099521155010221e-10;
  const double z = x * x;
  const double v = z * x;
  const double r = S2 + z * (S3 + z * (S4 + z * (S5 + z * S6)));
  return x + v * (S1 + z * r);
}
inline double det_kcos(double x) {
  const double C1 = 4.16666666666666019037e-02, C2 = -1.38888888888741095749e-03,
               C3 = 2.48015872894767294178e-05, C4 = -2.75573143513906633035e-07,
               C5 = 2.08757232129817482790e-09, C6 = -1.13596475577881948265e-11;
  const double z = x * x;
  const double r = z * (C1 + z * (C2 + z * (C3 + z * (C4 + z * (C5 + z * C6)))));
  const double hz = 0.5 * z;
  const double w = 1.0 - hz;
  return w + (((1.0 - w) - hz) + z * r);
}
inline void det_sincos(double x, double* s, double* c) {
  const double n = std::nearbyint(x * 6.36619772367581382433e-01);
  const double r = (x - n * 1.57079632673412561417e+00) - n * 6.07710050650619224932e-11;
  const double ks = det_ksin(r), kc = det_kcos(r);
  const int q = static_cast<int>(static_cast<long long>(n) & 3);
  switch (q) {
    case 0: *s = ks; *c = kc; break;
    case 1: *s = kc; *c = -ks; break;
    case 2: *s = -ks; *c = -kc; break;
    default: *s = -kc; *c = ks; break;
  }
}

// One-sided (Hestenes) Jacobi SVD of a row-major 3x3 A = U diag(S) V^T with
// S descending. U's first two columns are normalised columns of A V; the third
// is u0 x u1 (any sign works for Kabsch's reflection fix).
// Returns false when sv0 == 0 (U undefined).
inline void svd3_jacobi(const double A[9], double U[9], double S[3], double V[9]) {
  double W[9];
  for (int i = 0; i < 9; ++i) W[i] = A[i];
  for (int i = 0; i < 9; ++i) V[i] = (i % 4 == 0) ? 1.0 : 0.0;
  static const int P[3] = {0, 0, 1}, Q[3] = {1, 2, 2};
  for (int sweep = 0; sweep < 30; ++sweep) {
    bool rotated = false;
    for (int pq = 0; pq < 3; ++pq) {
      const int p = P[pq], q = Q[pq];
      double alpha = 0, beta = 0, gamma = 0;
      for (int k = 0; k < 3; ++k) {
        alpha = alpha + W[3 * k + p] * W[3 * k + p];
        beta = beta + W[3 * k + q] * W[3 * k + q];
        gamma = gamma + W[3 * k + p] * W[3 * k + q];
      }
      if (gamma == 0.0) continue;
      if (std::fabs(gamma) <= 1e-15 * std::sqrt(alpha * beta)) continue;
      rotated = true;
      const double zeta = (beta - alpha) / (2.0 * gamma);
      const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
      const double c = 1.0 / std::sqrt(1.0 + t * t);
      const double s = c * t;
      for (int k = 0; k < 3; ++k) {
        const double wp = W[3 * k + p], wq = W[3 * k + q];
        W[3 * k + p] = c * wp - s * wq;
        W[3 * k + q] = s * wp + c * wq;
        const double vp = V[3 * k + p], vq = V[3 * k + q];
        V[3 * k + p] = c * vp - s * vq;
        V[3 * k + q] = s * vp + c * vq;
      }
    }
    if (!rotated) break;
  }
  for (int j = 0; j < 3; ++j) {
    double n2 = 0;
    for (int k = 0; k < 3; ++k) n2 = n2 + W[3 * k + j] * W[3 * k + j];
    S[j] = std::sqrt(n2);
  }
  // sort descending (stable selection over 3 entries), permuting W and V columns
  for (int i = 0; i < 2; ++i) {
    int m = i;
    for (int j = i + 1; j < 3; ++j)
      if (S[j] > S[m]) m = j;
    if (m != i) {
      const double ts = S[i]; S[i] = S[m]; S[m] = ts;
      for (int k = 0; k < 3; ++k) {
        double tw = W[3 * k + i]; W[3 * k + i] = W[3 * k + m]; W[3 * k + m] = tw;
        double tv = V[3 * k + i]; V[3 * k + i] = V[3 * k + m]; V[3 * k + m] = tv;
      }
    }
  }
  for (int j = 0; j < 2; ++j)
    for (int k = 0; k < 3; ++k) U[3 * k + j] = S[j] > 0.0 ? W[3 * k + j] / S[j] : 0.0;
  U[2] = U[3] * U[7] - U[6] * U[4];
  U[5] = U[6] * U[1] - U[0] * U[7];
  U[8] = U[0] * U[4] - U[3] * U[1];
}

// Cyclic Jacobi on a symmetric 3x3 (row-major). evals[i] with eigenvector in
// column i of Vout. Unsorted (order is irrelevant for the matrix functions built from it).
inline void eig3_jacobi(const double Ain[9], double evals[3], double Vout[9]) {
  double A[9];
  for (int i = 0; i < 9; ++i) A[i] = Ain[i];
  double V[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  static const int P[3] = {0, 0, 1}, Q[3] = {1, 2, 2};
  for (int sweep = 0; sweep < 50; ++sweep) {
    const double off = A[1] * A[1] + A[2] * A[2] + A[5] * A[5];
    const double diag = A[0] * A[0] + A[4] * A[4] + A[8] * A[8];
    if (off == 0.0 || off <= 1e-32 * diag) break;
    for (int pq = 0; pq < 3; ++pq) {
      const int p = P[pq], q = Q[pq];
      const double apq = A[3 * p + q];
      if (apq == 0.0) continue;
      const double app = A[3 * p + p], aqq = A[3 * q + q];
      const double theta = (aqq - app) / (2.0 * apq);
      double t;
      if (std::fabs(theta) > 1e150) {
        t = 0.5 / theta;
      } else {
        t = (theta >= 0.0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
      }
      const double c = 1.0 / std::sqrt(t * t + 1.0);
      const double s = t * c;
      // A' = J^T A J with J the (p,q) rotation
      for (int k = 0; k < 3; ++k) {
        const double akp = A[3 * k + p], akq = A[3 * k + q];
        A[3 * k + p] = c * akp - s * akq;
        A[3 * k + q] = s * akp + c * akq;
      }
      for (int k = 0; k < 3; ++k) {
        const double apk = A[3 * p + k], aqk = A[3 * q + k];
        A[3 * p + k] = c * apk - s * aqk;
        A[3 * q + k] = s * apk + c * aqk;
      }
      A[3 * p + q] = 0.0;
      A[3 * q + p] = 0.0;
      for (int k = 0; k < 3; ++k) {
        const double vkp = V[3 * k + p], vkq = V[3 * k + q];
        V[3 * k + p] = c * vkp - s * vkq;
        V[3 * k + q] = s * vkp + c * vkq;
      }
    }
  }
  evals[0] = A[0];
  evals[1] = A[4];
  evals[2] = A[8];
  for (int i = 0; i < 9; ++i) Vout[i] = V[i];
}

// Solves M x = rhs for SPD 6x6 M (row-major, full). Returns false if a pivot <= 0.
inline bool chol6_solve(const double M[36], const double rhs[6], double x[6]) {
  double L[36], invd[6];
  for (int i = 0; i < 36; ++i) L[i] = 0.0;
  for (int j = 0; j < 6; ++j) {
    double d = M[6 * j + j];
    for (int k = 0; k < j; ++k) d = d - L[6 * j + k] * L[6 * j + k];
    if (!(d > 0.0)) return false;
    const double ljj = std::sqrt(d);
    L[6 * j + j] = ljj;
    const double inv = 1.0 / ljj;  // one division per pivot; every use multiplies by it
    invd[j] = inv;
    for (int i = j + 1; i < 6; ++i) {
      double s = M[6 * i + j];
      for (int k = 0; k < j; ++k) s = s - L[6 * i + k] * L[6 * j + k];
      L[6 * i + j] = s * inv;
    }
  }
  double y[6];
  for (int i = 0; i < 6; ++i) {
    double s = rhs[i];
    for (int k = 0; k < i; ++k) s = s - L[6 * i + k] * y[k];
    y[i] = s * invd[i];
  }
  for (int i = 5; i >= 0; --i) {
    double s = y[i];
    for (int k = i + 1; k < 6; ++k) s = s - L[6 * k + i] * x[k];
    x[i] = s * invd[i];
  }
  return true;
}

}  // namespace oracle

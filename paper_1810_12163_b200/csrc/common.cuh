// Device-side building blocks shared by the sm_100a kernels.
//
// Every function here follows the numerics contract of DESIGN.md: only IEEE
// correctly-rounded operations (+ - * / sqrt and explicit fma), compiled with
// --fmad=false so nothing is contracted behind our back. That makes the GPU
// results bit-comparable with the CPU oracle, which restates the same
// definitions independently (oracle/detmath.hpp, oracle/*.cpp).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/screloc_gpu.h"

#define SCR_DEV __device__ __forceinline__

namespace scr {

constexpr int kMaxTrees = 8;
constexpr int kMaxModes = 50;
constexpr int kFeatures = 256;
constexpr float kMaxValidDepth = 20.0f;
constexpr float kRenderMaxDepth = 6.0f;
constexpr int kLanes = 256;  // canonical ICP / score reduction width

SCR_DEV bool depth_valid(float d) { return d > 0.0f && d <= kMaxValidDepth; }

// std::lround for finite |x| < 2^23 (feature probe offsets, features.cpp:38-40): the
// fractional part x - trunc(x) is exact in f32, so halves round away from zero exactly.
SCR_DEV int lround_small(float x) {
  float t = truncf(x);
  if (fabsf(__fsub_rn(x, t)) >= 0.5f) t = __fadd_rn(t, copysignf(1.0f, x));
  return static_cast<int>(t);
}

// ---- RNG: xoshiro256** / splitmix64 (reference rng.hpp:14-88) ----------------------
struct Rng {
  uint64_t s0, s1, s2, s3;
};
SCR_DEV uint64_t splitmix64(uint64_t& x) {
  x += 0x9e3779b97f4a7c15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
SCR_DEV Rng rng_seed(uint64_t seed) {
  Rng r;
  uint64_t x = seed;
  r.s0 = splitmix64(x);
  r.s1 = splitmix64(x);
  r.s2 = splitmix64(x);
  r.s3 = splitmix64(x);
  return r;
}
SCR_DEV Rng rng_stream(uint64_t seed, uint64_t tag) {
  uint64_t x = seed;
  const uint64_t a = splitmix64(x);
  x ^= tag * 0x9e3779b97f4a7c15ull + 0x243f6a8885a308d3ull;
  const uint64_t b = splitmix64(x);
  return rng_seed(a ^ (b + 0x632be59bd9b4e019ull));
}
SCR_DEV uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
SCR_DEV uint64_t rng_next(Rng& r) {
  const uint64_t result = rotl64(r.s1 * 5, 7) * 9;
  const uint64_t t = r.s1 << 17;
  r.s2 ^= r.s0;
  r.s3 ^= r.s1;
  r.s1 ^= r.s2;
  r.s0 ^= r.s3;
  r.s2 ^= t;
  r.s3 = rotl64(r.s3, 45);
  return result;
}
// Unbiased rejection (rng.hpp:50-56). n < 2^32 on every call site, so the
// threshold and the final reduction use 64-by-32 arithmetic exactly like the
// reference's 64-bit modulo would.
SCR_DEV uint64_t rng_uniform_int(Rng& r, uint64_t n) {
  const uint64_t threshold = (0 - n) % n;
  for (;;) {
    const uint64_t v = rng_next(r);
    if (v >= threshold) return v % n;
  }
}
SCR_DEV double rng_uniform(Rng& r) { return static_cast<double>(rng_next(r) >> 11) * 0x1.0p-53; }

// Exact v mod n via Barrett reduction with m = floor((2^64 - 1) / n): q = umulhi(v, m) is
// at most 2 below floor(v / n), so two conditional subtractions give the exact remainder.
// Same results as the 64-bit modulo above, at a fraction of its cost.
SCR_DEV uint64_t barrett_m(uint64_t n) { return 0xffffffffffffffffull / n; }
SCR_DEV uint64_t mod_barrett(uint64_t v, uint64_t n, uint64_t m) {
  const uint64_t q = __umul64hi(v, m);
  uint64_t r = v - q * n;
  if (r >= n) r -= n;
  if (r >= n) r -= n;
  return r;
}
// Same remainder for n < 2^30: r = v - q n < 3 n fits 32 bits, so the tail is 32-bit.
SCR_DEV uint32_t mod_barrett32(uint64_t v, uint32_t n, uint64_t m) {
  const uint64_t q = __umul64hi(v, m);
  uint32_t r = static_cast<uint32_t>(v) - static_cast<uint32_t>(q) * n;
  if (r >= n) r -= n;
  if (r >= n) r -= n;
  return r;
}
SCR_DEV uint64_t rng_uniform_int_m(Rng& r, uint64_t n, uint64_t m) {
  const uint64_t threshold = mod_barrett(0 - n, n, m);
  for (;;) {
    const uint64_t v = rng_next(r);
    if (v >= threshold) return mod_barrett(v, n, m);
  }
}

// ---- deterministic transcendental kernels (oracle/detmath.hpp restated) ------------
SCR_DEV float det_expf(float x) {
  if (!(x > -87.0f)) return 0.0f;
  if (x > 0.0f) x = 0.0f;
  const float kf = rintf(__fmul_rn(x, 1.44269504088896341f));
  float r = __fmaf_rn(kf, -0.693145751953125f, x);
  r = __fmaf_rn(kf, -1.428606765330187045e-06f, r);
  float p = 1.98412698e-4f;
  p = __fmaf_rn(p, r, 1.38888889e-3f);
  p = __fmaf_rn(p, r, 8.33333333e-3f);
  p = __fmaf_rn(p, r, 4.16666667e-2f);
  p = __fmaf_rn(p, r, 1.66666667e-1f);
  p = __fmaf_rn(p, r, 0.5f);
  p = __fmaf_rn(p, r, 1.0f);
  p = __fmaf_rn(p, r, 1.0f);
  const int k = static_cast<int>(kf);
  return __fmul_rn(p, __int_as_float((k + 127) << 23));
}

SCR_DEV void det_sincos(double x, double* s, double* c) {
  const double S1 = -1.66666666666666324348e-01, S2 = 8.33333333332248946124e-03,
               S3 = -1.98412698298579493134e-04, S4 = 2.75573137070700676789e-06,
               S5 = -2.50507602534068634195e-08, S6 = 1.58969099521155010221e-10;
  const double C1 = 4.16666666666666019037e-02, C2 = -1.38888888888741095749e-03,
               C3 = 2.48015872894767294178e-05, C4 = -2.75573143513906633035e-07,
               C5 = 2.08757232129817482790e-09, C6 = -1.13596475577881948265e-11;
  const double n = rint(x * 6.36619772367581382433e-01);
  const double r = (x - n * 1.57079632673412561417e+00) - n * 6.07710050650619224932e-11;
  const double z = r * r;
  const double v = z * r;
  const double ks = r + v * (S1 + z * (S2 + z * (S3 + z * (S4 + z * (S5 + z * S6)))));
  const double rc = z * (C1 + z * (C2 + z * (C3 + z * (C4 + z * (C5 + z * C6)))));
  const double hz = 0.5 * z;
  const double w = 1.0 - hz;
  const double kc = w + (((1.0 - w) - hz) + z * rc);
  const int q = static_cast<int>(static_cast<long long>(n) & 3);
  if (q == 0) { *s = ks; *c = kc; }
  else if (q == 1) { *s = kc; *c = -ks; }
  else if (q == 2) { *s = -ks; *c = -kc; }
  else { *s = -kc; *c = ks; }
}

// ---- rigid-body math in double (geometry.hpp:73-191 restated) ------------------------
struct Pose {
  double R[9];
  double t[3];
};

SCR_DEV void pose_compose(const Pose& a, const Pose& b, Pose& r) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
#pragma unroll
    for (int j = 0; j < 3; ++j)
      r.R[3 * i + j] = (a.R[3 * i + 0] * b.R[0 + j] + a.R[3 * i + 1] * b.R[3 + j]) + a.R[3 * i + 2] * b.R[6 + j];
    r.t[i] = ((a.R[3 * i + 0] * b.t[0] + a.R[3 * i + 1] * b.t[1]) + a.R[3 * i + 2] * b.t[2]) + a.t[i];
  }
}

SCR_DEV void pose_invert(const Pose& a, Pose& r) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) r.R[3 * i + j] = a.R[3 * j + i];
#pragma unroll
  for (int i = 0; i < 3; ++i) r.t[i] = -(((r.R[3 * i + 0] * a.t[0] + r.R[3 * i + 1] * a.t[1]) + r.R[3 * i + 2] * a.t[2]));
}

SCR_DEV void pose_apply(const Pose& T, const double p[3], double o[3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i) o[i] = ((T.R[3 * i + 0] * p[0] + T.R[3 * i + 1] * p[1]) + T.R[3 * i + 2] * p[2]) + T.t[i];
}

SCR_DEV void exp_se3(const double tw[6], Pose& T) {
  const double w0 = tw[0], w1 = tw[1], w2 = tw[2];
  const double theta = sqrt((w0 * w0 + w1 * w1) + w2 * w2);
  const double hat[9] = {0.0, -w2, w1, w2, 0.0, -w0, -w1, w0, 0.0};
  double hat2[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      hat2[3 * i + j] = (hat[3 * i + 0] * hat[0 + j] + hat[3 * i + 1] * hat[3 + j]) + hat[3 * i + 2] * hat[6 + j];
  double v[9];
  if (theta < 1e-8) {
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      const double id = (i % 4 == 0) ? 1.0 : 0.0;
      T.R[i] = (id + hat[i]) + hat2[i] / 2.0;
      v[i] = (id + hat[i] / 2.0) + hat2[i] / 6.0;
    }
  } else {
    double s, c;
    det_sincos(theta, &s, &c);
    const double t2 = theta * theta;
    const double a = s / theta;
    const double b = (1.0 - c) / t2;
    const double cc = (theta - s) / (t2 * theta);
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      const double id = (i % 4 == 0) ? 1.0 : 0.0;
      T.R[i] = (id + a * hat[i]) + b * hat2[i];
      v[i] = (id + b * hat[i]) + cc * hat2[i];
    }
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) T.t[i] = (v[3 * i + 0] * tw[3] + v[3 * i + 1] * tw[4]) + v[3 * i + 2] * tw[5];
}

// One-sided Jacobi SVD of a row-major 3x3 (oracle/detmath.hpp svd3_jacobi restated).
SCR_DEV void svd3(const double A[9], double U[9], double S[3], double V[9]) {
  double W[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    W[i] = A[i];
    V[i] = (i % 4 == 0) ? 1.0 : 0.0;
  }
  for (int sweep = 0; sweep < 30; ++sweep) {
    bool rotated = false;
#pragma unroll
    for (int pq = 0; pq < 3; ++pq) {
      const int p = pq == 2 ? 1 : 0, q = pq == 0 ? 1 : 2;
      double alpha = 0.0, beta = 0.0, gamma = 0.0;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        alpha = alpha + W[3 * k + p] * W[3 * k + p];
        beta = beta + W[3 * k + q] * W[3 * k + q];
        gamma = gamma + W[3 * k + p] * W[3 * k + q];
      }
      if (gamma == 0.0) continue;
      if (fabs(gamma) <= 1e-15 * sqrt(alpha * beta)) continue;
      rotated = true;
      const double zeta = (beta - alpha) / (2.0 * gamma);
      const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
      const double c = 1.0 / sqrt(1.0 + t * t);
      const double s = c * t;
#pragma unroll
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
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    double n2 = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) n2 = n2 + W[3 * k + j] * W[3 * k + j];
    S[j] = sqrt(n2);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    int m = i;
#pragma unroll
    for (int j = i + 1; j < 3; ++j)
      if (S[j] > S[m]) m = j;
    if (m != i) {
      const double ts = S[i];
      S[i] = S[m];
      S[m] = ts;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double tw = W[3 * k + i];
        W[3 * k + i] = W[3 * k + m];
        W[3 * k + m] = tw;
        const double tv = V[3 * k + i];
        V[3 * k + i] = V[3 * k + m];
        V[3 * k + m] = tv;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int k = 0; k < 3; ++k) U[3 * k + j] = S[j] > 0.0 ? W[3 * k + j] / S[j] : 0.0;
  U[2] = U[3] * U[7] - U[6] * U[4];
  U[5] = U[6] * U[1] - U[0] * U[7];
  U[8] = U[0] * U[4] - U[3] * U[1];
}

// kabsch (geometry.hpp:158-191) for 3 pairs; false when degenerate.
SCR_DEV bool kabsch3(const double cam[9], const double world[9], Pose& T) {
  double cc[3] = {0.0, 0.0, 0.0}, wc[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      cc[k] = cc[k] + cam[3 * i + k];
      wc[k] = wc[k] + world[3 * i + k];
    }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    cc[k] = cc[k] / 3.0;
    wc[k] = wc[k] / 3.0;
  }
  double C[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) C[i] = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double dw[3], dc[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      dw[k] = world[3 * i + k] - wc[k];
      dc[k] = cam[3 * i + k] - cc[k];
    }
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) C[3 * r + c] = C[3 * r + c] + dw[r] * dc[c];
  }
  double U[9], S[3], V[9];
  svd3(C, U, S, V);
  if (!(S[0] > 0.0) || S[1] < 1e-12 * S[0]) return false;
  double M[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      M[3 * i + j] = (U[3 * i + 0] * V[3 * j + 0] + U[3 * i + 1] * V[3 * j + 1]) + U[3 * i + 2] * V[3 * j + 2];
  const double det = (M[0] * (M[4] * M[8] - M[5] * M[7]) - M[1] * (M[3] * M[8] - M[5] * M[6])) +
                     M[2] * (M[3] * M[7] - M[4] * M[6]);
  const double d2 = det < 0.0 ? -1.0 : 1.0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      T.R[3 * i + j] = (U[3 * i + 0] * V[3 * j + 0] + U[3 * i + 1] * V[3 * j + 1]) + (U[3 * i + 2] * d2) * V[3 * j + 2];
#pragma unroll
  for (int i = 0; i < 3; ++i) T.t[i] = wc[i] - ((T.R[3 * i + 0] * cc[0] + T.R[3 * i + 1] * cc[1]) + T.R[3 * i + 2] * cc[2]);
  return true;
}

// Cholesky solve of a 6x6 SPD system (oracle chol6_solve restated).
SCR_DEV bool chol6(const double M[36], const double rhs[6], double x[6]) {
  double L[36], invd[6];
#pragma unroll
  for (int i = 0; i < 36; ++i) L[i] = 0.0;
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    double d = M[6 * j + j];
#pragma unroll
    for (int k = 0; k < j; ++k) d = d - L[6 * j + k] * L[6 * j + k];
    if (!(d > 0.0)) return false;
    const double ljj = sqrt(d);
    L[6 * j + j] = ljj;
    const double inv = 1.0 / ljj;  // one division per pivot; every use multiplies by it
    invd[j] = inv;
#pragma unroll
    for (int i = j + 1; i < 6; ++i) {
      double s = M[6 * i + j];
#pragma unroll
      for (int k = 0; k < j; ++k) s = s - L[6 * i + k] * L[6 * j + k];
      L[6 * i + j] = s * inv;
    }
  }
  double y[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    double s = rhs[i];
#pragma unroll
    for (int k = 0; k < i; ++k) s = s - L[6 * i + k] * y[k];
    y[i] = s * invd[i];
  }
#pragma unroll
  for (int i = 5; i >= 0; --i) {
    double s = y[i];
#pragma unroll
    for (int k = i + 1; k < 6; ++k) s = s - L[6 * k + i] * x[k];
    x[i] = s * invd[i];
  }
  return true;
}

// Cyclic Jacobi eigen-decomposition of a symmetric 3x3 (oracle eig3_jacobi restated).
SCR_DEV void eig3(const double Ain[9], double ev[3], double Vout[9]) {
  double A[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) A[i] = Ain[i];
  double V[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  for (int sweep = 0; sweep < 50; ++sweep) {
    const double off = A[1] * A[1] + A[2] * A[2] + A[5] * A[5];
    const double diag = A[0] * A[0] + A[4] * A[4] + A[8] * A[8];
    if (off == 0.0 || off <= 1e-32 * diag) break;
#pragma unroll
    for (int pq = 0; pq < 3; ++pq) {
      const int p = pq == 2 ? 1 : 0, q = pq == 0 ? 1 : 2;
      const double apq = A[3 * p + q];
      if (apq == 0.0) continue;
      const double app = A[3 * p + p], aqq = A[3 * q + q];
      const double theta = (aqq - app) / (2.0 * apq);
      double t;
      if (fabs(theta) > 1e150) t = 0.5 / theta;
      else t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
      const double c = 1.0 / sqrt(t * t + 1.0);
      const double s = t * c;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double akp = A[3 * k + p], akq = A[3 * k + q];
        A[3 * k + p] = c * akp - s * akq;
        A[3 * k + q] = s * akp + c * akq;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double apk = A[3 * p + k], aqk = A[3 * q + k];
        A[3 * p + k] = c * apk - s * aqk;
        A[3 * q + k] = s * apk + c * aqk;
      }
      A[3 * p + q] = 0.0;
      A[3 * q + p] = 0.0;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double vkp = V[3 * k + p], vkq = V[3 * k + q];
        V[3 * k + p] = c * vkp - s * vkq;
        V[3 * k + q] = s * vkp + c * vkq;
      }
    }
  }
  ev[0] = A[0];
  ev[1] = A[4];
  ev[2] = A[8];
#pragma unroll
  for (int i = 0; i < 9; ++i) Vout[i] = V[i];
}

// ---- f32 helpers (energy / ICP hot loops) ---------------------------------------------
SCR_DEV void xform_f32(const float R[9], const float t[3], float x0, float x1, float x2, float y[3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
    y[i] = __fmaf_rn(R[3 * i + 0], x0, __fmaf_rn(R[3 * i + 1], x1, __fmaf_rn(R[3 * i + 2], x2, t[i])));
}
// d^T Sigma^-1 d with icov packed (c00 c11 c22 2c01 2c02 2c12)
SCR_DEV float quad_icov(float c00, float c11, float c22, float e01, float e02, float e12, float d0, float d1,
                        float d2) {
  float t0 = __fmaf_rn(e01, d1, __fmul_rn(e02, d2));
  t0 = __fmaf_rn(c00, d0, t0);
  const float t1 = __fmaf_rn(c11, d1, __fmul_rn(e12, d2));
  const float t2 = __fmul_rn(c22, d2);
  return __fmaf_rn(d0, t0, __fmaf_rn(d1, t1, __fmul_rn(d2, t2)));
}
SCR_DEV float quad_eucl(float d0, float d1, float d2) { return __fmaf_rn(d0, d0, __fmaf_rn(d1, d1, __fmul_rn(d2, d2))); }

// Packed GPU mode record: q0 = (mu.xyz, c00), q1 = (c11, c22, 2c01, 2c02),
// q2 = (2c12, s00, s01, s02), q3 = (s11, s12, s22, -), colour = (r, g, b, size bits).
struct ModeGeom {
  float4 q0, q1, q2, q3;
};

// ---- analytic scene ray cast (oracle scene.cpp raycast_pixel restated) -------------------
struct Prim {
  int type;
  float a[3], b[3], colour[3], cell;
  uint32_t tex_seed;
};
struct Hit {
  float t;
  int prim;
  int face;
};

SCR_DEV void ray_dir(const float R[9], float fx, float fy, float cx, float cy, int x, int y, float d[3]) {
  const float dcx = __fdiv_rn(__fsub_rn(static_cast<float>(x), cx), fx);
  const float dcy = __fdiv_rn(__fsub_rn(static_cast<float>(y), cy), fy);
#pragma unroll
  for (int i = 0; i < 3; ++i) d[i] = __fmaf_rn(R[3 * i + 0], dcx, __fmaf_rn(R[3 * i + 1], dcy, R[3 * i + 2]));
}

SCR_DEV void ray_dir_tab(const float R[9], float dcx, float dcy, float d[3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i) d[i] = __fmaf_rn(R[3 * i + 0], dcx, __fmaf_rn(R[3 * i + 1], dcy, R[3 * i + 2]));
}

// Ray casts use __frcp_rn(x) for 1/x: the correctly rounded reciprocal, bit-identical to the
// IEEE division 1.0f / x of the oracle (including 0 -> inf), with a shorter instruction sequence.
SCR_DEV Hit raycast(const Prim* prims, int n, const float o[3], const float d[3]) {
  Hit h;
  h.t = __int_as_float(0x7f800000);
  h.prim = -1;
  h.face = -1;
  const float inv0 = __frcp_rn(d[0]), inv1 = __frcp_rn(d[1]), inv2 = __frcp_rn(d[2]);
  const float aa = __fmaf_rn(d[0], d[0], __fmaf_rn(d[1], d[1], __fmul_rn(d[2], d[2])));
  for (int p = 0; p < n; ++p) {
    const Prim& q = prims[p];
    if (q.type == 0) {
      const float t10 = __fmul_rn(__fsub_rn(q.a[0], o[0]), inv0), t20 = __fmul_rn(__fsub_rn(q.b[0], o[0]), inv0);
      const float t11 = __fmul_rn(__fsub_rn(q.a[1], o[1]), inv1), t21 = __fmul_rn(__fsub_rn(q.b[1], o[1]), inv1);
      const float t12 = __fmul_rn(__fsub_rn(q.a[2], o[2]), inv2), t22 = __fmul_rn(__fsub_rn(q.b[2], o[2]), inv2);
      const float lo0 = fminf(t10, t20), lo1 = fminf(t11, t21), lo2 = fminf(t12, t22);
      const float hi0 = fmaxf(t10, t20), hi1 = fmaxf(t11, t21), hi2 = fmaxf(t12, t22);
      const float tn = fmaxf(fmaxf(lo0, lo1), lo2);
      const float tx = fminf(fminf(hi0, hi1), hi2);
      if (tn <= tx && tn > 1e-4f && tn < h.t) {
        const int axis = (tn == lo0) ? 0 : ((tn == lo1) ? 1 : 2);
        const float da = axis == 0 ? d[0] : (axis == 1 ? d[1] : d[2]);
        h.t = tn;
        h.prim = p;
        h.face = axis * 2 + (da > 0.0f ? 0 : 1);
      }
    } else {
      const float oc0 = __fsub_rn(o[0], q.a[0]), oc1 = __fsub_rn(o[1], q.a[1]), oc2 = __fsub_rn(o[2], q.a[2]);
      const float bb = __fmaf_rn(oc0, d[0], __fmaf_rn(oc1, d[1], __fmul_rn(oc2, d[2])));
      const float cc =
          __fsub_rn(__fmaf_rn(oc0, oc0, __fmaf_rn(oc1, oc1, __fmul_rn(oc2, oc2))), __fmul_rn(q.b[0], q.b[0]));
      const float disc = __fsub_rn(__fmul_rn(bb, bb), __fmul_rn(aa, cc));
      if (disc >= 0.0f) {
        const float t = __fdiv_rn(__fsub_rn(-bb, __fsqrt_rn(disc)), aa);
        if (t > 1e-4f && t < h.t) {
          h.t = t;
          h.prim = p;
          h.face = 6;
        }
      }
    }
  }
  return h;
}

// Same closest-hit search over a subset of primitives given by an ascending index list
// (ties still resolve to the lower primitive index, so the hit is identical whenever the
// omitted primitives cannot be hit).
SCR_DEV Hit raycast_list(const Prim* prims, const unsigned char* list, int nl, const float o[3], const float d[3]) {
  Hit h;
  h.t = __int_as_float(0x7f800000);
  h.prim = -1;
  h.face = -1;
  const float inv0 = __frcp_rn(d[0]), inv1 = __frcp_rn(d[1]), inv2 = __frcp_rn(d[2]);
  const float aa = __fmaf_rn(d[0], d[0], __fmaf_rn(d[1], d[1], __fmul_rn(d[2], d[2])));
  for (int li = 0; li < nl; ++li) {
    const int p = list[li];
    const Prim& q = prims[p];
    if (q.type == 0) {
      const float t10 = __fmul_rn(__fsub_rn(q.a[0], o[0]), inv0), t20 = __fmul_rn(__fsub_rn(q.b[0], o[0]), inv0);
      const float t11 = __fmul_rn(__fsub_rn(q.a[1], o[1]), inv1), t21 = __fmul_rn(__fsub_rn(q.b[1], o[1]), inv1);
      const float t12 = __fmul_rn(__fsub_rn(q.a[2], o[2]), inv2), t22 = __fmul_rn(__fsub_rn(q.b[2], o[2]), inv2);
      const float lo0 = fminf(t10, t20), lo1 = fminf(t11, t21), lo2 = fminf(t12, t22);
      const float hi0 = fmaxf(t10, t20), hi1 = fmaxf(t11, t21), hi2 = fmaxf(t12, t22);
      const float tn = fmaxf(fmaxf(lo0, lo1), lo2);
      const float tx = fminf(fminf(hi0, hi1), hi2);
      if (tn <= tx && tn > 1e-4f && tn < h.t) {
        const int axis = (tn == lo0) ? 0 : ((tn == lo1) ? 1 : 2);
        const float da = axis == 0 ? d[0] : (axis == 1 ? d[1] : d[2]);
        h.t = tn;
        h.prim = p;
        h.face = axis * 2 + (da > 0.0f ? 0 : 1);
      }
    } else {
      const float oc0 = __fsub_rn(o[0], q.a[0]), oc1 = __fsub_rn(o[1], q.a[1]), oc2 = __fsub_rn(o[2], q.a[2]);
      const float bb = __fmaf_rn(oc0, d[0], __fmaf_rn(oc1, d[1], __fmul_rn(oc2, d[2])));
      const float cc =
          __fsub_rn(__fmaf_rn(oc0, oc0, __fmaf_rn(oc1, oc1, __fmul_rn(oc2, oc2))), __fmul_rn(q.b[0], q.b[0]));
      const float disc = __fsub_rn(__fmul_rn(bb, bb), __fmul_rn(aa, cc));
      if (disc >= 0.0f) {
        const float t = __fdiv_rn(__fsub_rn(-bb, __fsqrt_rn(disc)), aa);
        if (t > 1e-4f && t < h.t) {
          h.t = t;
          h.prim = p;
          h.face = 6;
        }
      }
    }
  }
  return h;
}

// Same search over the list entries selected by a bitmask (bit j = list[j]; ascending).
SCR_DEV Hit raycast_mask(const Prim* prims, const unsigned char* list, uint32_t mask, const float o[3],
                         const float d[3]) {
  Hit h;
  h.t = __int_as_float(0x7f800000);
  h.prim = -1;
  h.face = -1;
  const float inv0 = __frcp_rn(d[0]), inv1 = __frcp_rn(d[1]), inv2 = __frcp_rn(d[2]);
  const float aa = __fmaf_rn(d[0], d[0], __fmaf_rn(d[1], d[1], __fmul_rn(d[2], d[2])));
  while (mask) {
    const int p = list[__ffs(mask) - 1];
    mask &= mask - 1u;
    const Prim& q = prims[p];
    if (q.type == 0) {
      const float t10 = __fmul_rn(__fsub_rn(q.a[0], o[0]), inv0), t20 = __fmul_rn(__fsub_rn(q.b[0], o[0]), inv0);
      const float t11 = __fmul_rn(__fsub_rn(q.a[1], o[1]), inv1), t21 = __fmul_rn(__fsub_rn(q.b[1], o[1]), inv1);
      const float t12 = __fmul_rn(__fsub_rn(q.a[2], o[2]), inv2), t22 = __fmul_rn(__fsub_rn(q.b[2], o[2]), inv2);
      const float lo0 = fminf(t10, t20), lo1 = fminf(t11, t21), lo2 = fminf(t12, t22);
      const float hi0 = fmaxf(t10, t20), hi1 = fmaxf(t11, t21), hi2 = fmaxf(t12, t22);
      const float tn = fmaxf(fmaxf(lo0, lo1), lo2);
      const float tx = fminf(fminf(hi0, hi1), hi2);
      if (tn <= tx && tn > 1e-4f && tn < h.t) {
        const int axis = (tn == lo0) ? 0 : ((tn == lo1) ? 1 : 2);
        const float da = axis == 0 ? d[0] : (axis == 1 ? d[1] : d[2]);
        h.t = tn;
        h.prim = p;
        h.face = axis * 2 + (da > 0.0f ? 0 : 1);
      }
    } else {
      const float oc0 = __fsub_rn(o[0], q.a[0]), oc1 = __fsub_rn(o[1], q.a[1]), oc2 = __fsub_rn(o[2], q.a[2]);
      const float bb = __fmaf_rn(oc0, d[0], __fmaf_rn(oc1, d[1], __fmul_rn(oc2, d[2])));
      const float cc =
          __fsub_rn(__fmaf_rn(oc0, oc0, __fmaf_rn(oc1, oc1, __fmul_rn(oc2, oc2))), __fmul_rn(q.b[0], q.b[0]));
      const float disc = __fsub_rn(__fmul_rn(bb, bb), __fmul_rn(aa, cc));
      if (disc >= 0.0f) {
        const float t = __fdiv_rn(__fsub_rn(-bb, __fsqrt_rn(disc)), aa);
        if (t > 1e-4f && t < h.t) {
          h.t = t;
          h.prim = p;
          h.face = 6;
        }
      }
    }
  }
  return h;
}

// Conservative frustum test of a primitive against the rays of the pixel rectangle
// [px0, px1] x [py0, py1] (pixel-centre coordinates, already widened by half a pixel) for a
// camera (R cam->world, origin o): false only if no such ray can reach the primitive in
// front of the camera. Each side plane passes through the camera centre; a box is outside
// a plane when its support along the plane normal (centre distance + sum |n_i| e_i) stays
// below zero, a sphere when centre distance + r |n| does. Support terms carry a 1 % + 2 cm
// margin, far above the float rounding of the test.
SCR_DEV bool prim_in_frustum(const Prim& q, const float R[9], const float o[3], float fx, float fy, float cx,
                             float cy, float px0, float px1, float py0, float py1) {
  float c[3], e[3] = {0.0f, 0.0f, 0.0f}, r = 0.0f;
  const bool box = q.type == 0;
  if (box) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      c[i] = 0.5f * (q.a[i] + q.b[i]);
      e[i] = fabsf(0.5f * (q.b[i] - q.a[i]));
    }
  } else {
    c[0] = q.a[0];
    c[1] = q.a[1];
    c[2] = q.a[2];
    r = q.b[0];
  }
  const float v[3] = {c[0] - o[0], c[1] - o[1], c[2] - o[2]};
  const float xl = (px0 - cx) / fx, xh = (px1 - cx) / fx;
  const float yl = (py0 - cy) / fy, yh = (py1 - cy) / fy;
  // camera-frame inward normals: near (0,0,1), left (1,0,-xl), right (-1,0,xh), top (0,1,-yl), bottom (0,-1,yh)
  const float nc[5][3] = {{0.0f, 0.0f, 1.0f}, {1.0f, 0.0f, -xl}, {-1.0f, 0.0f, xh}, {0.0f, 1.0f, -yl}, {0.0f, -1.0f, yh}};
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    float nw[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) nw[i] = R[3 * i + 0] * nc[k][0] + R[3 * i + 1] * nc[k][1] + R[3 * i + 2] * nc[k][2];
    const float nlen = sqrtf(nc[k][0] * nc[k][0] + nc[k][1] * nc[k][1] + nc[k][2] * nc[k][2]);
    const float dist = nw[0] * v[0] + nw[1] * v[1] + nw[2] * v[2];
    const float sup = box ? (fabsf(nw[0]) * e[0] + fabsf(nw[1]) * e[1] + fabsf(nw[2]) * e[2]) : r * nlen;
    if (dist + sup * 1.01f + 0.02f * nlen <= 0.0f) return false;
  }
  return true;
}
SCR_DEV bool prim_in_view(const Prim& q, const float R[9], const float o[3], float fx, float fy, float cx, float cy,
                          int W, int H) {
  return prim_in_frustum(q, R, o, fx, fy, cx, cy, -0.5f, W - 0.5f, -0.5f, H - 0.5f);
}

// ---- TSDF scene model (oracle/tsdf.cpp restated; A13) ----------------------------
struct TsdfView {
  const float2* vox = nullptr;  // {tsdf, weight}, x fastest
  float ox = 0, oy = 0, oz = 0, voxel = 0, trunc = 0;
  int nx = 0, ny = 0, nz = 0;
};
constexpr int kTsdfMaxSteps = 1024;

SCR_DEV float tsdf_lerp(float a, float b, float t) { return __fmaf_rn(t, __fsub_rn(b, a), a); }

SCR_DEV bool tsdf_sample(const TsdfView& v, float px, float py, float pz, float* F) {
  const float g0 = __fsub_rn(__fdiv_rn(__fsub_rn(px, v.ox), v.voxel), 0.5f);
  const float g1 = __fsub_rn(__fdiv_rn(__fsub_rn(py, v.oy), v.voxel), 0.5f);
  const float g2 = __fsub_rn(__fdiv_rn(__fsub_rn(pz, v.oz), v.voxel), 0.5f);
  const float f0 = floorf(g0), f1 = floorf(g1), f2 = floorf(g2);
  const int i0 = static_cast<int>(f0), i1 = static_cast<int>(f1), i2 = static_cast<int>(f2);
  if (i0 < 0 || i1 < 0 || i2 < 0 || i0 + 1 >= v.nx || i1 + 1 >= v.ny || i2 + 1 >= v.nz) return false;
  const float r0 = __fsub_rn(g0, f0), r1 = __fsub_rn(g1, f1), r2 = __fsub_rn(g2, f2);
  float c[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const size_t idx = (static_cast<size_t>(i2 + (q >> 2)) * v.ny + (i1 + ((q >> 1) & 1))) * v.nx + (i0 + (q & 1));
    const float2 e = v.vox[idx];
    if (!(e.y > 0.0f)) return false;
    c[q] = e.x;
  }
  const float c00 = tsdf_lerp(c[0], c[1], r0), c10 = tsdf_lerp(c[2], c[3], r0);
  const float c01 = tsdf_lerp(c[4], c[5], r0), c11 = tsdf_lerp(c[6], c[7], r0);
  *F = tsdf_lerp(tsdf_lerp(c00, c10, r1), tsdf_lerp(c01, c11, r1), r2);
  return true;
}

SCR_DEV uint32_t tsdf_pack_normal(float n0, float n1, float n2) {
  const float s = __fadd_rn(__fadd_rn(fabsf(n0), fabsf(n1)), fabsf(n2));
  float u = __fdiv_rn(n0, s), w = __fdiv_rn(n1, s);
  if (n2 < 0.0f) {
    const float uu = __fmul_rn(__fsub_rn(1.0f, fabsf(w)), u >= 0.0f ? 1.0f : -1.0f);
    const float ww = __fmul_rn(__fsub_rn(1.0f, fabsf(u)), w >= 0.0f ? 1.0f : -1.0f);
    u = uu;
    w = ww;
  }
  const int qu = max(-32767, min(32767, static_cast<int>(floorf(__fadd_rn(__fmul_rn(u, 32767.0f), 0.5f)))));
  const int qw = max(-32767, min(32767, static_cast<int>(floorf(__fadd_rn(__fmul_rn(w, 32767.0f), 0.5f)))));
  return (static_cast<uint32_t>(qu) & 0xffffu) | (static_cast<uint32_t>(qw) << 16);
}

SCR_DEV void tsdf_unpack_normal(uint32_t p, float n[3]) {
  const float u = __fdiv_rn(static_cast<float>(static_cast<int16_t>(p & 0xffffu)), 32767.0f);
  const float w = __fdiv_rn(static_cast<float>(static_cast<int16_t>(p >> 16)), 32767.0f);
  float x = u, y = w;
  const float z = __fsub_rn(__fsub_rn(1.0f, fabsf(u)), fabsf(w));
  if (z < 0.0f) {
    x = __fmul_rn(__fsub_rn(1.0f, fabsf(w)), u >= 0.0f ? 1.0f : -1.0f);
    y = __fmul_rn(__fsub_rn(1.0f, fabsf(u)), w >= 0.0f ? 1.0f : -1.0f);
  }
  const float len = __fsqrt_rn(__fmaf_rn(x, x, __fmaf_rn(y, y, __fmul_rn(z, z))));
  n[0] = __fdiv_rn(x, len);
  n[1] = __fdiv_rn(y, len);
  n[2] = __fdiv_rn(z, len);
}

// March one ray o + t d (d = R (dcx, dcy, 1), so t is the camera depth): hit at the first
// known F <= 0 after a known F > 0, refined linearly; *nrm = packed normal or 0xffffffff.
template <typename FP>
SCR_DEV bool tsdf_raycast_ray(const TsdfView& v, FP o, const float d[3], float* t_out, uint32_t* nrm) {
  float t = 0.2f, tp = 0.0f, Fp = 0.0f;
  bool prev = false;
  for (int it = 0; it < kTsdfMaxSteps && t <= kRenderMaxDepth; ++it) {
    float F;
    if (tsdf_sample(v, __fmaf_rn(t, d[0], o[0]), __fmaf_rn(t, d[1], o[1]), __fmaf_rn(t, d[2], o[2]), &F)) {
      if (prev && Fp > 0.0f && F <= 0.0f) {
        const float ts = __fmaf_rn(__fsub_rn(t, tp), __fdiv_rn(Fp, __fsub_rn(Fp, F)), tp);
        if (!(ts <= kRenderMaxDepth)) return false;
        *t_out = ts;
        *nrm = 0xffffffffu;
        const float q0 = __fmaf_rn(ts, d[0], o[0]), q1 = __fmaf_rn(ts, d[1], o[1]), q2 = __fmaf_rn(ts, d[2], o[2]);
        float gp[3], gm[3];
        if (!tsdf_sample(v, __fadd_rn(q0, v.voxel), q1, q2, &gp[0]) || !tsdf_sample(v, __fsub_rn(q0, v.voxel), q1, q2, &gm[0]) ||
            !tsdf_sample(v, q0, __fadd_rn(q1, v.voxel), q2, &gp[1]) || !tsdf_sample(v, q0, __fsub_rn(q1, v.voxel), q2, &gm[1]) ||
            !tsdf_sample(v, q0, q1, __fadd_rn(q2, v.voxel), &gp[2]) || !tsdf_sample(v, q0, q1, __fsub_rn(q2, v.voxel), &gm[2]))
          return true;
        const float g0 = __fsub_rn(gp[0], gm[0]), g1 = __fsub_rn(gp[1], gm[1]), g2 = __fsub_rn(gp[2], gm[2]);
        const float len = __fsqrt_rn(__fmaf_rn(g0, g0, __fmaf_rn(g1, g1, __fmul_rn(g2, g2))));
        if (!(len > 0.0f)) return true;
        *nrm = tsdf_pack_normal(__fdiv_rn(g0, len), __fdiv_rn(g1, len), __fdiv_rn(g2, len));
        return true;
      }
      prev = true;
      Fp = F;
      tp = t;
      t = __fadd_rn(t, F > 0.0f ? fmaxf(__fmul_rn(F, v.trunc), v.voxel) : v.voxel);
    } else {
      prev = false;
      t = __fadd_rn(t, v.trunc);
    }
  }
  return false;
}

SCR_DEV void hit_normal(const Prim* prims, int prim, int face, const float p[3], float n[3]) {
  if (face < 6) {
    n[0] = n[1] = n[2] = 0.0f;
    const float v = (face & 1) ? 1.0f : -1.0f;
    if ((face >> 1) == 0) n[0] = v;
    else if ((face >> 1) == 1) n[1] = v;
    else n[2] = v;
  } else {
    const Prim& q = prims[prim];
    const float inv = __frcp_rn(q.b[0]);
#pragma unroll
    for (int i = 0; i < 3; ++i) n[i] = __fmul_rn(__fsub_rn(p[i], q.a[i]), inv);
  }
}

// Work-counter update aggregated over the active lanes of the warp (one atomic per warp, so
// the in-library profiler does not serialise the kernels it measures). v < 2^32 per lane.
SCR_DEV void work_add(unsigned long long* work, int id, unsigned v) {
  const unsigned mask = __activemask();
  const unsigned s = __reduce_add_sync(mask, v);
  if (static_cast<int>(threadIdx.x & 31) == __ffs(mask) - 1) atomicAdd(&work[id], static_cast<unsigned long long>(s));
}

// ---- warp reductions in the canonical xor-butterfly order ------------------------------
SCR_DEV double warp_sum_xor(double v) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}
// warp_sum_xor of N <= 32 values at once ("transpose" reduction): at offset o every lane
// keeps one half of its remaining values and sends the other half to lane ^ o, so each value
// is combined with the same partner partial at every level as in its own xor butterfly (the
// pairs are identical and IEEE addition is commutative): bit-identical sums, 31 shuffles of
// a double instead of 5 N. On return lane k holds the sum of value k (for k < N) in v[0].
template <int N>
SCR_DEV void warp_sum_xor_many(double (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = N; k < 32; ++k) v[k] = 0.0;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < o; ++i) {
      const double send = upper ? v[i] : v[i + o];
      const double keep = upper ? v[i + o] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
}
SCR_DEV int warp_isum(int v) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

}  // namespace scr

// Per-frame relocalisation on the GPU: preemptive RANSAC (K4 generation, K5 energy,
// K6 Levenberg-Marquardt, K7 cull/halving), ICP + depth-raycast ranking (K8-K10) and
// the cascade controller (K11), for a batch of independent frames.
//
// Reference behaviour restated here (SPEC.md; the reference sources are missing):
//   generate_hypothesis / generate_initial_hypotheses
//   energy (Eq. 5)
//   initial_cull
//   lm_refine
//   preemptive_ransac
//   raycast_depth / icp_refine
//   depth_diff_score (Eqs. 6-7)
//   rank_hypotheses / relocalise / run_cascade
// Geometry in f64 restates proj/include/screloc/geometry.hpp:83-191.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>

#include <cooperative_groups.h>

#include "internal.cuh"

namespace scr {

struct GenParams {
  int max_iters, nmax;
  double min_sq_dist;
  float colour_thresh;
  double rigidity_tol;
  int fast;  // per-pixel records usable (<= 5 trees, 16-bit leaf ids)
  int force_suspect;  // test hook: every passing triplet is a suspect
  int leaf_base[kMaxTrees];
};

// Outcome of one generation attempt: pass, or its rejection tag.
enum { kAttPass = 0, kAttNoModes = 1, kAttColour = 2, kAttTooClose = 3, kAttNotRigid = 4, kAttDegenerate = 5 };

struct FrameRefs {  // per-batch views of the packed frames
  const int* fidx;       // active index -> workspace slot
  const int* gcount;
  const int* gpx;
  const float4* gcam;
  const int* gslot;
  const int* gnm;
  const int4* grec;    // interleaved 32-B pixel records: grec[2 i] = {x|y<<16, depth, rgb|nm<<24, counts},
  const uint4* gleaf;  // gleaf[2 i + 1] = 16-bit leaf ids (one sector per pixel)
  const uint2* tex;
  const float* dplane;  // per frame: level-0, level-1, level-2 live depth planes
  int gmax, T;
};

SCR_DEV int mode_index(const FrameRefs& fr, const int* pcount, size_t gbase, int m) {
  for (int t = 0; t < fr.T; ++t) {
    const int slot = fr.gslot[gbase * fr.T + t];
    const int cnt = pcount[slot];
    if (m < cnt) return slot * kMaxModes + m;
    m -= cnt;
  }
  return -1;
}

// ================================ K4: hypothesis generation ================================
// Generation slots are independent (slot s draws from Rng::stream(seed, s) and retries up
// to max_iters; draw order and checks per DESIGN.md A1/A7), so lanes pull
// slots from a per-frame atomic counter and never idle behind a slower lane.
// Latency is the cost here (most attempts are rejected), so an attempt touches global
// memory as little as possible:
//  * each CTA keeps |M(u)| of every grid pixel of its frame in shared memory (a byte per
//    pixel), so the draws run the exact sequential algorithm and know how many values the
//    attempt consumes (a pixel without modes ends it) without a global load;
//  * only the colour-check pixel's 32-byte record (colour, per-tree mode counts, 16-bit leaf
//    ids, written by K1) and its mode's colour are loaded; the other two modes are resolved
//    when a warp evaluates its queued colour-check survivors;
//  * uniform draws use exact Barrett reductions (same values as the 64-bit modulo).
constexpr int kMaxModeUnion = kMaxTrees * kMaxModes;
#ifndef SCR_GEN_TPF
#define SCR_GEN_TPF 2048
#endif
constexpr int kGenThreadsPerFrame = SCR_GEN_TPF;  // generation threads per frame (slots pulled dynamically)

// uniform_int(n) by rejection (rng.hpp:50-56) with the 32-bit-tail Barrett reduction.
SCR_DEV uint32_t draw32(Rng& r, uint32_t n, uint64_t m, uint64_t thr) {
  for (;;) {
    const uint64_t v = rng_next(r);
    if (v >= thr) return mod_barrett32(v, n, m);
  }
}
// uniform_int(n) for n < 2^32 with the rejection threshold 2^64 mod n (< n) computed only
// when it can matter: a value with a non-zero high word is always accepted.
SCR_DEV uint64_t draw_exact_lazy(Rng& r, uint64_t n, uint64_t m) {
  for (;;) {
    const uint64_t v = rng_next(r);
    if ((v >> 32) != 0 || v >= mod_barrett(0 - n, n, m)) return mod_barrett(v, n, m);
  }
}
// The accepted raw value of uniform_int(n) (reduced mod n later, when needed).
SCR_DEV uint64_t draw_raw(Rng& r, uint32_t thr) {
  for (;;) {
    const uint64_t v = rng_next(r);
    if (v >= thr) return v;
  }
}

// uniform_int by rejection (rng.hpp:50-56) with a precomputed Barrett reciprocal/threshold.
SCR_DEV uint64_t draw_exact(Rng& r, uint64_t n, uint64_t m, uint64_t thr) {
  for (;;) {
    const uint64_t v = rng_next(r);
    if (v >= thr) return mod_barrett(v, n, m);
  }
}

// Mode index of the pick-th predicted mode of a pixel (union over trees in tree order),
// branch-free from the record: 6-bit per-tree counts and 16-bit leaf ids (trees 0..4).
SCR_DEV int mode_from_record(const int* lbase, uint32_t counts, uint4 lv, int pick) {
  const int c0 = counts & 63u, c1 = (counts >> 6) & 63u, c2 = (counts >> 12) & 63u, c3 = (counts >> 18) & 63u;
  const int e0 = c0, e1 = e0 + c1, e2 = e1 + c2, e3 = e2 + c3;
  // branch-free: t = trees whose cumulative count is <= pick, before = their modes
  const int s0 = pick >= e0, s1 = pick >= e1, s2 = pick >= e2, s3 = pick >= e3;
  const int t = s0 + s1 + s2 + s3;
  const int before = s0 * c0 + s1 * c1 + s2 * c2 + s3 * c3;
  uint32_t w = lv.x;
  w = s1 ? lv.y : w;  // t >= 2
  w = s3 ? lv.z : w;  // t >= 4
  const int leaf = static_cast<int>((w >> ((t & 1) << 4)) & 0xffffu);
  return (lbase[t] + leaf) * kMaxModes + (pick - before);
}

// Colour check: L-inf distance of the pixel's RGB to the mode's mean
// colour within the threshold.
SCR_DEV bool colour_ok(uint32_t col, float4 mc, float thresh) {
  float linf = 0.0f;
  linf = fmaxf(linf, fabsf(__fsub_rn(static_cast<float>(col & 255u), mc.x)));
  linf = fmaxf(linf, fabsf(__fsub_rn(static_cast<float>((col >> 8) & 255u), mc.y)));
  linf = fmaxf(linf, fabsf(__fsub_rn(static_cast<float>((col >> 16) & 255u), mc.z)));
  return !(linf > thresh);
}

// Kabsch for a triplet that passed every check (finisher kernel only).
SCR_DEV bool kabsch3_cold(const double* cm, const double* w, Pose* T) { return kabsch3(cm, w, *T); }

// Exact f64 camera point of a pixel record (x, y, depth): geometry.hpp:194-199, the same
// operations as K1.
SCR_DEV void cam_point_f64(int4 rec, const FrameGeom& g, double out[3]) {
  const int x = rec.x & 0xffff, y = rec.x >> 16;
  const double dd = static_cast<double>(__int_as_float(rec.y));
  out[0] = ((static_cast<double>(x) - g.dcx) * dd) / g.dfx;
  out[1] = ((static_cast<double>(y) - g.dcy) * dd) / g.dfy;
  out[2] = dd;
}

// f32 pre-filter of checks 2-3: rejects only triplets the exact f64 checks reject too (world
// points are the same f32 values; the f32 camera points are within 1e-5 m of the f64 ones,
// far inside the 1e-3 m / 1e-3 m^2 margins).
SCR_DEV bool geometry_prefilter(double min_sq_dist, double rigidity_tol, const int4* grec, const FrameGeom& g,
                                float ifx, float ify, const ModeGeom* geom, int g0, int g1, int g2, int m0, int m1,
                                int m2) {
  const float4 w0 = geom[m0].q0, w1 = geom[m1].q0, w2 = geom[m2].q0;
  const int4 r0 = grec[2 * g0], r1 = grec[2 * g1], r2 = grec[2 * g2];
  const int4 rr[3] = {r0, r1, r2};
  float cf[3][3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float d = __int_as_float(rr[k].y);
    cf[k][0] = (static_cast<float>(rr[k].x & 0xffff) - g.cx) * d * ifx;
    cf[k][1] = (static_cast<float>(rr[k].x >> 16) - g.cy) * d * ify;
    cf[k][2] = d;
  }
  const float4 wf[3] = {w0, w1, w2};
  const float tolf = static_cast<float>(rigidity_tol) + 1e-3f;
  const float closef = static_cast<float>(min_sq_dist) - 1e-3f;
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const int pa = q == 2 ? 1 : 0, pb = q == 0 ? 1 : 2;
    const float ax = wf[pa].x - wf[pb].x, ay = wf[pa].y - wf[pb].y, az = wf[pa].z - wf[pb].z;
    const float bx = cf[pa][0] - cf[pb][0], by = cf[pa][1] - cf[pb][1], bz = cf[pa][2] - cf[pb][2];
    const float dw2f = ax * ax + ay * ay + az * az, dc2f = bx * bx + by * by + bz * bz;
    if (dw2f < closef) return false;
    if (fabsf(sqrtf(dw2f) - sqrtf(dc2f)) > tolf) return false;
  }
  return true;
}

// Three-way f32 classification of checks 2-3 plus Kabsch regularity, for the attempt loop
// (keeps the f64 arithmetic, and its registers, out of k_hypgen):
//  kClsFail    — the exact f64 checks certainly reject (outside a 1e-3 m / m^2 margin);
//  kClsPass    — they certainly accept (inside the margin) and Kabsch is certainly regular;
//  kClsSuspect — anything else: k_hypfin decides it exactly, in attempt order.
// The world points are the same f32 values as in f64 and the f32 camera points are within
// ~1e-5 m of the exact ones, far inside the margins. Regularity: the centred 3-pair
// cross-covariance H has rank <= 2, so r = sqrt(sum of squared 2x2 minors) / |H|_F^2 bounds
// sigma1 / sigma0 from below; the f64 finisher needs r > 1e-6, the f32 test asks r > 1e-3
// (and a non-vanishing |H|), three orders of magnitude above the f32 error of r.
enum { kClsFail = 0, kClsPass = 1, kClsSuspect = 2 };
SCR_DEV int geometry_classify(double min_sq_dist, double rigidity_tol, const int4* grec, const FrameGeom& g,
                              float ifx, float ify, const ModeGeom* geom, int g0, int g1, int g2, int m0, int m1,
                              int m2) {
  const float4 wq[3] = {geom[m0].q0, geom[m1].q0, geom[m2].q0};
  const int4 rr[3] = {grec[2 * g0], grec[2 * g1], grec[2 * g2]};
  float cf[3][3], wf[3][3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float d = __int_as_float(rr[k].y);
    cf[k][0] = (static_cast<float>(rr[k].x & 0xffff) - g.cx) * d * ifx;
    cf[k][1] = (static_cast<float>(rr[k].x >> 16) - g.cy) * d * ify;
    cf[k][2] = d;
    wf[k][0] = wq[k].x;
    wf[k][1] = wq[k].y;
    wf[k][2] = wq[k].z;
  }
  const float rig = static_cast<float>(rigidity_tol), msq = static_cast<float>(min_sq_dist);
  bool sure = true;
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const int pa = q == 2 ? 1 : 0, pb = q == 0 ? 1 : 2;
    const float ax = wf[pa][0] - wf[pb][0], ay = wf[pa][1] - wf[pb][1], az = wf[pa][2] - wf[pb][2];
    const float bx = cf[pa][0] - cf[pb][0], by = cf[pa][1] - cf[pb][1], bz = cf[pa][2] - cf[pb][2];
    const float dw2f = ax * ax + ay * ay + az * az, dc2f = bx * bx + by * by + bz * bz;
    if (dw2f < msq - 1e-3f) return kClsFail;
    const float dev = fabsf(sqrtf(dw2f) - sqrtf(dc2f));
    if (dev > rig + 1e-3f) return kClsFail;
    if ((min_sq_dist > 0.0 && dw2f < msq + 1e-3f) || dev > rig - 1e-3f) sure = false;
  }
  if (!sure) return kClsSuspect;
  float H[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) H[i] = 0.0f;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const float wc = (wf[0][c] + wf[1][c] + wf[2][c]) * (1.0f / 3.0f);
    const float cc = (cf[0][c] + cf[1][c] + cf[2][c]) * (1.0f / 3.0f);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      wf[k][c] -= wc;
      cf[k][c] -= cc;
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) H[3 * r + c] += wf[k][r] * cf[k][c];
  float f2 = 0.0f, e2 = 0.0f;
#pragma unroll
  for (int i = 0; i < 9; ++i) f2 += H[i] * H[i];
#pragma unroll
  for (int r0 = 0; r0 < 3; ++r0)
#pragma unroll
    for (int r1 = r0 + 1; r1 < 3; ++r1)
#pragma unroll
      for (int c0 = 0; c0 < 3; ++c0)
#pragma unroll
        for (int c1 = c0 + 1; c1 < 3; ++c1) {
          const float mnr = H[3 * r0 + c0] * H[3 * r1 + c1] - H[3 * r0 + c1] * H[3 * r1 + c0];
          e2 += mnr * mnr;
        }
  return (f2 > 1e-10f && sqrtf(e2) > 1e-3f * f2) ? kClsPass : kClsSuspect;
}

// Exact checks 2-3 (distances in f64) and Kabsch. Camera points are the
// exact f64 backprojection of the records (geometry.hpp:194-199, the same operations as K1).
// Scalars and pointers only: passing the kernel-parameter structs by reference would force
// copies of them into local memory.
// Kabsch on a triplet (kabsch3) is degenerate iff its computed singular values have
// !(S0 > 0) || S1 < 1e-12 S0. The centred cross-covariance H of 3 pairs has rank <= 2, so
// sigma0^2 sigma1^2 ~= e2 = sum of its squared 2x2 minors and sigma0^2 <= |H|_F^2: with
// r = sqrt(e2) / |H|_F^2 <= sigma1 / sigma0 (up to ~1e-16 rounding), r > 1e-6 guarantees a
// non-degenerate Kabsch by six orders of magnitude (the one-sided Jacobi SVD is accurate to
// ~1e-15 S0). Triplets below that are "suspects" that k_hypfin decides with kabsch3 itself.
SCR_DEV bool kabsch_clearly_regular(const double cm[9], const double w[9]) {
  double cc[3], wc[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    cc[k] = (cm[k] + cm[3 + k] + cm[6 + k]) / 3.0;
    wc[k] = (w[k] + w[3 + k] + w[6 + k]) / 3.0;
  }
  double H[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) H[i] = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) H[3 * r + c] += (w[3 * i + r] - wc[r]) * (cm[3 * i + c] - cc[c]);
  double f2 = 0.0, e2 = 0.0;
#pragma unroll
  for (int i = 0; i < 9; ++i) f2 += H[i] * H[i];
#pragma unroll
  for (int r0 = 0; r0 < 3; ++r0)
#pragma unroll
    for (int r1 = r0 + 1; r1 < 3; ++r1)
#pragma unroll
      for (int c0 = 0; c0 < 3; ++c0)
#pragma unroll
        for (int c1 = c0 + 1; c1 < 3; ++c1) {
          const double mnr = H[3 * r0 + c0] * H[3 * r1 + c1] - H[3 * r0 + c1] * H[3 * r1 + c0];
          e2 += mnr * mnr;
        }
  return f2 > 0.0 && sqrt(e2) > 1e-6 * f2;
}

SCR_DEV bool distance_checks_f64(double min_sq_dist, double rigidity_tol, const int4* grec, const FrameGeom& g,
                                 const ModeGeom* geom, int g0, int g1, int g2, int m0, int m1, int m2,
                                 double* cm_out, double* w_out, bool* regular = nullptr, int* why = nullptr) {
  const float4 w0 = geom[m0].q0, w1 = geom[m1].q0, w2 = geom[m2].q0;
  const int4 r0 = grec[2 * g0], r1 = grec[2 * g1], r2 = grec[2 * g2];
  double w[9] = {w0.x, w0.y, w0.z, w1.x, w1.y, w1.z, w2.x, w2.y, w2.z};
  double cm[9];
  cam_point_f64(r0, g, cm);
  cam_point_f64(r1, g, cm + 3);
  cam_point_f64(r2, g, cm + 6);
  double dw2[3], dc2[3];
  bool close = false;
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const int pa = q == 2 ? 1 : 0, pb = q == 0 ? 1 : 2;
    const double ax = w[3 * pa] - w[3 * pb], ay = w[3 * pa + 1] - w[3 * pb + 1], az = w[3 * pa + 2] - w[3 * pb + 2];
    dw2[q] = (ax * ax + ay * ay) + az * az;
    const double bx = cm[3 * pa] - cm[3 * pb], by = cm[3 * pa + 1] - cm[3 * pb + 1], bz = cm[3 * pa + 2] - cm[3 * pb + 2];
    dc2[q] = (bx * bx + by * by) + bz * bz;
    if (dw2[q] < min_sq_dist) close = true;
  }
  if (close) {
    if (why) *why = kAttTooClose;
    return false;
  }
#pragma unroll
  for (int q = 0; q < 3; ++q)
    if (fabs(sqrt(dw2[q]) - sqrt(dc2[q])) > rigidity_tol) {
      if (why) *why = kAttNotRigid;
      return false;
    }
  if (cm_out) {
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      cm_out[i] = cm[i];
      w_out[i] = w[i];
    }
  }
  if (regular) *regular = kabsch_clearly_regular(cm, w);
  return true;
}

SCR_DEV bool geometry_exact(double min_sq_dist, double rigidity_tol, const int4* grec, const FrameGeom& g,
                            const ModeGeom* geom, int g0, int g1, int g2, int m0, int m1, int m2, Pose* T) {
  double cm[9], w[9];
  if (!distance_checks_f64(min_sq_dist, rigidity_tol, grec, g, geom, g0, g1, g2, m0, m1, m2, cm, w)) return false;
  return kabsch3_cold(cm, w, T);
}

// One generation attempt on the exact sequential path (draw order A1/A7):
// draws pixel, mode, pixel, mode, pixel, mode, colour-pair index from the slot stream with
// rejection sampling; returns kAttPass if the attempt reached the colour check and passed it,
// else its rejection tag (kAttNoModes, kAttColour).
SCR_DEV int attempt_exact(Rng& rng, const GenParams& gp, const FrameRefs& fr, const PredView& pv,
                           const int* s_lbase, const uint64_t* s_m, size_t fbase, uint64_t G,
                           uint64_t mG, uint64_t tG, bool fast, int& g0, int& g1, int& g2, int& m0, int& m1,
                           int& m2) {
  constexpr uint64_t m3 = 0x5555555555555555ull, t3 = 1;  // floor((2^64-1)/3), 2^64 mod 3
  int p0 = 0, p1 = 0, p2 = 0, cc = 0;
  int4 A0, A1, A2;
  uint4 L0, L1, L2;
  g0 = static_cast<int>(draw_exact(rng, G, mG, tG));
  A0 = fr.grec[2 * (fbase + g0)];
  L0 = fr.gleaf[2 * (fbase + g0) + 1];
  const int nm0 = fast ? (static_cast<uint32_t>(A0.z) >> 24) : fr.gnm[fbase + g0];
  if (nm0 <= 0) return kAttNoModes;
  p0 = static_cast<int>(draw_exact_lazy(rng, static_cast<uint64_t>(nm0), s_m[nm0]));
  g1 = static_cast<int>(draw_exact(rng, G, mG, tG));
  A1 = fr.grec[2 * (fbase + g1)];
  L1 = fr.gleaf[2 * (fbase + g1) + 1];
  const int nm1 = fast ? (static_cast<uint32_t>(A1.z) >> 24) : fr.gnm[fbase + g1];
  if (nm1 <= 0) return kAttNoModes;
  p1 = static_cast<int>(draw_exact_lazy(rng, static_cast<uint64_t>(nm1), s_m[nm1]));
  g2 = static_cast<int>(draw_exact(rng, G, mG, tG));
  A2 = fr.grec[2 * (fbase + g2)];
  L2 = fr.gleaf[2 * (fbase + g2) + 1];
  const int nm2 = fast ? (static_cast<uint32_t>(A2.z) >> 24) : fr.gnm[fbase + g2];
  if (nm2 <= 0) return kAttNoModes;
  p2 = static_cast<int>(draw_exact_lazy(rng, static_cast<uint64_t>(nm2), s_m[nm2]));
  cc = static_cast<int>(draw_exact(rng, 3, m3, t3));
  if (fast) {
    m0 = mode_from_record(s_lbase, static_cast<uint32_t>(A0.w), L0, p0);
    m1 = mode_from_record(s_lbase, static_cast<uint32_t>(A1.w), L1, p1);
    m2 = mode_from_record(s_lbase, static_cast<uint32_t>(A2.w), L2, p2);
  } else {
    m0 = mode_index(fr, pv.count, fbase + g0, p0);
    m1 = mode_index(fr, pv.count, fbase + g1, p1);
    m2 = mode_index(fr, pv.count, fbase + g2, p2);
  }
  const uint32_t col = static_cast<uint32_t>(cc == 0 ? A0.z : (cc == 1 ? A1.z : A2.z));
  return colour_ok(col, pv.col[cc == 0 ? m0 : (cc == 1 ? m1 : m2)], gp.colour_thresh) ? kAttPass : kAttColour;
}

// Per-warp queue of colour-check survivors, evaluated 32 at a time at full SIMD width.
// They get the f32 pre-filter and the exact f64 checks 2-3 here; Kabsch (a 3x3 f64 SVD) is
// left to k_hypfin, which keeps the SVD's code and registers out of the attempt loop. A slot
// stops at its first passing attempt whose Kabsch is provably regular (hok = 2, attempt +
// triplet in hcand); passing attempts whose Kabsch may be degenerate are listed as per-frame
// suspects and the slot goes on, so k_hypfin never has to re-run a slot's attempt chain
// (unless the suspect list overflows).
#ifndef SCR_HYPGEN_MINB
#define SCR_HYPGEN_MINB 3  // resident CTAs per SM the register budget is sized for (24 warps, 80 registers)
#endif
#ifndef SCR_GEN_WARPS
#define SCR_GEN_WARPS 8
#endif
#ifndef SCR_GEN_SPEC
#define SCR_GEN_SPEC 1  // draw an attempt's seven values at once (exact; see the attempt loop)
#endif
constexpr int kGenWarps = SCR_GEN_WARPS;  // warps per generation CTA
constexpr int kGenQ = 64;
#ifndef SCR_MAX_SUSPECTS
#define SCR_MAX_SUSPECTS 256  // 64 overflowed on the Default profile: slots then replayed their attempts serially in k_hypfin
#endif
constexpr int kMaxSuspects = SCR_MAX_SUSPECTS;  // per frame: triplets whose Kabsch may be degenerate
// A queued colour-check survivor. Fast-path entries carry the three raw mode draws and are
// resolved to mode indices in the evaluation phase (at full SIMD width, instead of by the
// few passing lanes of every attempt round); exact-path entries carry resolved modes.
constexpr int kCandResolved = 1 << 30;  // flag in slot: m0..m2 hold mode indices
struct GenCand {
  int slot, owner_att;  // slot (| kCandResolved), owner lane | attempt << 5
  uint32_t gA, gB;      // the three grid pixels (< 2^17 each), packed: g0 | g1 << 17, g1 >> 15 | g2 << 2
  uint2 r0, r1, r2;     // raw 64-bit draws of the three modes, or {m, 0}
  SCR_DEV void set_pixels(int g0, int g1, int g2) {
    gA = static_cast<uint32_t>(g0) | (static_cast<uint32_t>(g1) << 17);
    gB = (static_cast<uint32_t>(g1) >> 15) | (static_cast<uint32_t>(g2) << 2);
  }
  SCR_DEV int g0() const { return static_cast<int>(gA & 0x1ffffu); }
  SCR_DEV int g1() const { return static_cast<int>((gA >> 17) | ((gB & 3u) << 15)); }
  SCR_DEV int g2() const { return static_cast<int>(gB >> 2); }
};

SCR_DEV uint64_t u64_of(uint2 v) { return static_cast<uint64_t>(v.x) | (static_cast<uint64_t>(v.y) << 32); }
SCR_DEV uint2 u2_of(uint64_t v) { return make_uint2(static_cast<uint32_t>(v), static_cast<uint32_t>(v >> 32)); }

__global__ void __launch_bounds__(kGenWarps * 32, SCR_HYPGEN_MINB) k_hypgen(GenParams gp, FrameGeom g, FrameRefs fr, PredView pv,
                                                   const uint64_t* __restrict__ seeds, int* __restrict__ slot_ctr,
                                                   int4* __restrict__ hcand, int* __restrict__ hok,
                                                   int* __restrict__ hiters, int* __restrict__ sus_cnt,
                                                   int4* __restrict__ sus, unsigned long long* __restrict__ work) {
  __shared__ uint64_t s_m[kMaxModeUnion + 1];    // Barrett reciprocal for mode counts 1..400
  __shared__ uint32_t s_thr[kMaxModeUnion + 1];  // rejection threshold 2^64 mod n (< n < 2^32)
  __shared__ int s_lbase[kMaxTrees];
  __shared__ GenCand s_q[kGenWarps][kGenQ];
  __shared__ int s_best[kGenWarps][32];  // smallest passing attempt of the lane's slot
  __shared__ int s_pend[kGenWarps][32];  // queued, unevaluated candidates of the lane's slot
  __shared__ int s_cur[kGenWarps][32];   // slot the lane currently owns
  extern __shared__ uint8_t s_nm[];      // |M(u)| of every grid pixel of the frame (fast path)
  for (int i = threadIdx.x; i <= kMaxModeUnion; i += blockDim.x) {
    const uint64_t n = i ? static_cast<uint64_t>(i) : 1;
    const uint64_t m = barrett_m(n);
    s_m[i] = m;
    s_thr[i] = static_cast<uint32_t>(mod_barrett(0 - n, n, m));
  }
  if (threadIdx.x < kMaxTrees) s_lbase[threadIdx.x] = gp.leaf_base[threadIdx.x];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  s_best[wid][lane] = 0x7fffffff;
  s_pend[wid][lane] = 0;
  s_cur[wid][lane] = -1;
  __syncthreads();
  const int a = blockIdx.y;
  const int f = fr.fidx[a];
  const uint64_t G = static_cast<uint64_t>(fr.gcount[f]);
  const uint64_t mG = G ? barrett_m(G) : 1, tG = G ? mod_barrett(0 - G, G, mG) : 0;
  const uint32_t G32 = static_cast<uint32_t>(G);
  const uint64_t m3 = 0x5555555555555555ull;  // floor((2^64-1)/3)
  const bool fast = gp.fast != 0;
  const size_t fbase = static_cast<size_t>(f) * fr.gmax;
  if (fast) {  // <= 5 trees x 50 modes: a byte per pixel
    for (int i = threadIdx.x; i < static_cast<int>(G); i += blockDim.x) s_nm[i] = static_cast<uint8_t>(fr.gnm[fbase + i]);
    __syncthreads();
  }
  const float ifx = 1.0f / g.fx, ify = 1.0f / g.fy;  // f32 pre-filter only
  GenCand* q = s_q[wid];
  int qn = 0;  // warp-uniform queue length
  unsigned long long attempts_total = 0;
  int slot = -1, it = 0;
  bool exhausted = false;
  Rng rng;
  for (;;) {
    if (slot < 0 && !exhausted) {
      slot = atomicAdd(&slot_ctr[a], 1);
      if (slot >= gp.nmax) {
        slot = -1;
        exhausted = true;
      } else if (G == 0) {  // no valid pixels: the slot fails without drawing
        const size_t out = static_cast<size_t>(a) * gp.nmax + slot;
        hok[out] = 0;
        hiters[out] = gp.max_iters;
        slot = -1;
      } else {
        rng = rng_stream(seeds[a], static_cast<uint64_t>(slot));
        it = 0;
        s_cur[wid][lane] = slot;
      }
    }
    if (__all_sync(0xffffffffu, exhausted) && qn == 0) break;
    // ---- one attempt per lane that still has attempts left
    bool push = false;
    GenCand c;
    if (slot >= 0 && it < gp.max_iters) {
      if (fast) {
        // The exact sequential attempt (draw order A1/A7, rejection sampling as in
        // rng.hpp:50-56): each pixel's mode count comes from shared memory, so the stream
        // consumption (1, 3, 5 or 7 values) is known without touching global memory, and
        // only the colour-check pixel's record, leaf ids and mode colour are loaded.
        int g0, g1 = 0, g2 = 0, cc = 0;
        uint32_t nm0, nm1 = 0, nm2 = 0;
        uint64_t v1 = 0, v3 = 0, v5 = 0;
        bool full = false;
#if SCR_GEN_SPEC
        // Speculative form of the same draws: every rejection threshold is below 2^32, so a
        // value with a non-zero high word is always accepted, and an attempt whose three
        // pixels all have modes consumes exactly seven values. Draw the seven at once (the
        // state chain no longer waits on the shared-memory mode-count loads and branches)
        // and fall back to the sequential draws from the saved state otherwise.
        const Rng rs = rng;
        const uint64_t x0 = rng_next(rng), x1 = rng_next(rng), x2 = rng_next(rng), x3 = rng_next(rng),
                       x4 = rng_next(rng), x5 = rng_next(rng), x6 = rng_next(rng);
        g0 = static_cast<int>(mod_barrett32(x0, G32, mG));
        g1 = static_cast<int>(mod_barrett32(x2, G32, mG));
        g2 = static_cast<int>(mod_barrett32(x4, G32, mG));
        nm0 = s_nm[g0];
        nm1 = s_nm[g1];
        nm2 = s_nm[g2];
        const bool hi = (x0 >> 32) != 0 && (x1 >> 32) != 0 && (x2 >> 32) != 0 && (x3 >> 32) != 0 &&
                        (x4 >> 32) != 0 && (x5 >> 32) != 0 && (x6 >> 32) != 0;
        if (hi && nm0 != 0 && nm1 != 0 && nm2 != 0) {
          v1 = x1;
          v3 = x3;
          v5 = x5;
          cc = static_cast<int>(mod_barrett32(x6, 3u, m3));
          full = true;
        } else {
          rng = rs;
          g1 = g2 = 0;
          nm1 = nm2 = 0;
#endif
        g0 = static_cast<int>(draw32(rng, G32, mG, tG));
        nm0 = s_nm[g0];
        if (nm0) {
          v1 = draw_raw(rng, s_thr[nm0]);
          g1 = static_cast<int>(draw32(rng, G32, mG, tG));
          nm1 = s_nm[g1];
          if (nm1) {
            v3 = draw_raw(rng, s_thr[nm1]);
            g2 = static_cast<int>(draw32(rng, G32, mG, tG));
            nm2 = s_nm[g2];
            if (nm2) {
              v5 = draw_raw(rng, s_thr[nm2]);
              cc = static_cast<int>(draw32(rng, 3u, m3, 1u));  // 2^64 mod 3 = 1
              full = true;
            }
          }
        }
#if SCR_GEN_SPEC
        }
#endif
        if (full) {
          const int gc = cc == 0 ? g0 : (cc == 1 ? g1 : g2);
          const uint64_t vc = cc == 0 ? v1 : (cc == 1 ? v3 : v5);
          const uint32_t nmc = cc == 0 ? nm0 : (cc == 1 ? nm1 : nm2);
          const int4 Ac = fr.grec[2 * (fbase + gc)];
          const uint4 Lc = fr.gleaf[2 * (fbase + gc) + 1];
          const uint32_t pc = mod_barrett32(vc, nmc, s_m[nmc]);
          const float4 mcol = pv.col[mode_from_record(s_lbase, static_cast<uint32_t>(Ac.w), Lc, static_cast<int>(pc))];
          if (colour_ok(static_cast<uint32_t>(Ac.z), mcol, gp.colour_thresh)) {
            push = true;
            c.slot = slot;
            c.owner_att = lane | (it << 5);
            c.set_pixels(g0, g1, g2);
            c.r0 = u2_of(v1); c.r1 = u2_of(v3); c.r2 = u2_of(v5);
          }
        }
      } else {  // > 5 trees or 32-bit leaf ids: modes through the slot tables
        int g0, g1, g2, m0, m1, m2;
        if (attempt_exact(rng, gp, fr, pv, s_lbase, s_m, fbase, G, mG, tG, fast, g0, g1, g2, m0, m1, m2) == kAttPass) {
          push = true;
          c.slot = slot | kCandResolved;
          c.owner_att = lane | (it << 5);
          c.set_pixels(g0, g1, g2);
          c.r0 = make_uint2(m0, 0); c.r1 = make_uint2(m1, 0); c.r2 = make_uint2(m2, 0);
        }
      }
      if (push) s_pend[wid][lane] += 1;
      ++it;
    }
    const unsigned pm = __ballot_sync(0xffffffffu, push);
    if (push) q[qn + __popc(pm & ((1u << lane) - 1u))] = c;
    qn += __popc(pm);
    // slots that used all attempts with nothing pending have failed
    if (slot >= 0 && it >= gp.max_iters && s_pend[wid][lane] == 0) {
      const size_t out = static_cast<size_t>(a) * gp.nmax + slot;
      hok[out] = 0;
      hiters[out] = gp.max_iters;
      attempts_total += static_cast<unsigned long long>(gp.max_iters);
      s_cur[wid][lane] = -1;
      slot = -1;
    }
    __syncwarp();
    const bool waiting = slot >= 0 && it >= gp.max_iters;
    const bool idle = slot < 0 && exhausted;
    if (qn >= 32 || (qn > 0 && (__any_sync(0xffffffffu, waiting) || __all_sync(0xffffffffu, idle)))) {
      // ---- evaluate the oldest <= 32 candidates, one per lane
      const int nproc = qn < 32 ? qn : 32;
      bool pass = false;
      int owner = 0, att = 0, eslot = -1, eg0 = 0, eg1 = 0, eg2 = 0;
      GenCand e;
      if (lane < nproc) {
        e = q[lane];
        eg0 = e.g0();
        eg1 = e.g1();
        eg2 = e.g2();
        owner = e.owner_att & 31;
        att = e.owner_att >> 5;
        eslot = e.slot & ~kCandResolved;
        if (s_cur[wid][owner] == eslot) {  // stale if the owner's slot was already resolved
          if (!(e.slot & kCandResolved)) {  // mode indices of the three raw draws (fast path)
            const int4* gr = fr.grec + 2 * fbase;
            const int4 A0 = gr[2 * eg0], A1 = gr[2 * eg1], A2 = gr[2 * eg2];
            const uint4 L0 = fr.gleaf[2 * (fbase + eg0) + 1], L1 = fr.gleaf[2 * (fbase + eg1) + 1],
                        L2 = fr.gleaf[2 * (fbase + eg2) + 1];
            const uint32_t nm0 = static_cast<uint32_t>(A0.z) >> 24, nm1 = static_cast<uint32_t>(A1.z) >> 24,
                           nm2 = static_cast<uint32_t>(A2.z) >> 24;
            const int p0 = static_cast<int>(mod_barrett32(u64_of(e.r0), nm0, s_m[nm0]));
            const int p1 = static_cast<int>(mod_barrett32(u64_of(e.r1), nm1, s_m[nm1]));
            const int p2 = static_cast<int>(mod_barrett32(u64_of(e.r2), nm2, s_m[nm2]));
            e.r0.x = mode_from_record(s_lbase, static_cast<uint32_t>(A0.w), L0, p0);
            e.r1.x = mode_from_record(s_lbase, static_cast<uint32_t>(A1.w), L1, p1);
            e.r2.x = mode_from_record(s_lbase, static_cast<uint32_t>(A2.w), L2, p2);
          }
          const int em0 = static_cast<int>(e.r0.x), em1 = static_cast<int>(e.r1.x), em2 = static_cast<int>(e.r2.x);
          const int cls = geometry_classify(gp.min_sq_dist, gp.rigidity_tol, fr.grec + 2 * fbase, g, ifx, ify,
                                            pv.geom, eg0, eg1, eg2, em0, em1, em2);
          pass = cls != kClsFail;
          if (pass && (cls == kClsSuspect || gp.force_suspect)) {  // k_hypfin decides it exactly, the slot goes on
            const int i = atomicAdd(&sus_cnt[a], 1);
            if (i < kMaxSuspects) {
              int4* sp = sus + 2 * (static_cast<size_t>(a) * kMaxSuspects + i);
              sp[0] = make_int4(att, eg0, eg1, eg2);
              sp[1] = make_int4(em0, em1, em2, eslot);
              pass = false;
            }  // list full: stop here as usual, k_hypfin continues exactly if Kabsch fails
          }
          atomicSub(&s_pend[wid][owner], 1);
          if (pass) atomicMin(&s_best[wid][owner], att);
        }
      }
      __syncwarp();
      if (pass && s_best[wid][owner] == att) {
        int4* hc = hcand + 2 * (static_cast<size_t>(a) * gp.nmax + eslot);
        hc[0] = make_int4(att, eg0, eg1, eg2);
        hc[1] = make_int4(static_cast<int>(e.r0.x), static_cast<int>(e.r1.x), static_cast<int>(e.r2.x), 0);
      }
      // drop the evaluated entries
      GenCand keep;
      const int rest = qn - nproc;
      if (lane < rest) keep = q[nproc + lane];
      __syncwarp();
      if (lane < rest) q[lane] = keep;
      qn = rest;
      // owners whose slot now has a winner
      if (slot >= 0 && s_best[wid][lane] != 0x7fffffff) {
        const int best = s_best[wid][lane];
        const size_t out = static_cast<size_t>(a) * gp.nmax + slot;
        hok[out] = 2;  // tentative: k_hypfin decides
        hiters[out] = best + 1;
        attempts_total += static_cast<unsigned long long>(best + 1);
        s_best[wid][lane] = 0x7fffffff;
        s_pend[wid][lane] = 0;
        s_cur[wid][lane] = -1;
        slot = -1;
      } else if (slot >= 0 && it >= gp.max_iters && s_pend[wid][lane] == 0) {
        const size_t out = static_cast<size_t>(a) * gp.nmax + slot;
        hok[out] = 0;
        hiters[out] = gp.max_iters;
        attempts_total += static_cast<unsigned long long>(gp.max_iters);
        s_cur[wid][lane] = -1;
        slot = -1;
      }
      __syncwarp();
    }
  }
  if (work) work_add(work, W_GEN_ATTEMPTS, static_cast<unsigned>(attempts_total));
}

// Exact finisher of generation: thread per (frame, slot). k_hypgen stopped a slot at its
// first attempt passing the exact checks 2-3 with a clearly regular Kabsch (hok = 2,
// triplet in hcand) and listed the earlier passing attempts whose Kabsch may be degenerate
// ("suspects", per frame). The slot's result is its first attempt whose Kabsch succeeds
// (SPEC.md:441-447): suspects in attempt order, then the recorded triplet. Only when the
// suspect list overflowed can the recorded triplet itself be degenerate; the slot then
// continues on the exact sequential path (stream replayed through the recorded attempt).
constexpr int kFinThreads = 128;
__global__ void __launch_bounds__(kFinThreads) k_hypfin(GenParams gp, FrameGeom g, FrameRefs fr, PredView pv,
                                                        const uint64_t* __restrict__ seeds,
                                                        const int4* __restrict__ hcand, Pose* __restrict__ hyp,
                                                        int* __restrict__ hok, int* __restrict__ hiters,
                                                        const int* __restrict__ sus_cnt, const int4* __restrict__ sus,
                                                        unsigned long long* __restrict__ work) {
  __shared__ uint64_t s_m[kMaxModeUnion + 1];
  __shared__ int s_lbase[kMaxTrees];
  __shared__ int4 s_sus[kMaxSuspects][2];
  const int a = blockIdx.y;
  const int slot = blockIdx.x * kFinThreads + threadIdx.x;
  const size_t out = static_cast<size_t>(a) * gp.nmax + slot;
  const int ns = min(sus_cnt[a], kMaxSuspects);
  for (int i = threadIdx.x; i < 2 * ns; i += blockDim.x) s_sus[i >> 1][i & 1] = sus[2 * static_cast<size_t>(a) * kMaxSuspects + i];
  const bool clear = slot < gp.nmax && hok[out] == 2;
  if (!__syncthreads_or(clear) && ns == 0) return;
  const int f = fr.fidx[a];
  const size_t fbase = static_cast<size_t>(f) * fr.gmax;
  const int4* grec = fr.grec + 2 * fbase;
  int4 c0 = make_int4(0x7fffffff, 0, 0, 0), c1 = make_int4(0, 0, 0, 0);
  if (clear) {
    c0 = hcand[2 * out];
    c1 = hcand[2 * out + 1];
  }
  Pose T;
  bool ok = false;
  int res_it = 0;
  if (slot < gp.nmax) {
    int last = -1;
    for (;;) {  // this slot's suspects before the recorded attempt, in attempt order
      int best = -1, batt = c0.x;
      for (int i = 0; i < ns; ++i)
        if (s_sus[i][1].w == slot && s_sus[i][0].x > last && s_sus[i][0].x < batt) {
          best = i;
          batt = s_sus[i][0].x;
        }
      if (best < 0) break;
      last = batt;
      const int4 u0 = s_sus[best][0], u1 = s_sus[best][1];
      if (geometry_exact(gp.min_sq_dist, gp.rigidity_tol, grec, g, pv.geom, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, &T)) {
        ok = true;
        res_it = u0.x + 1;
        break;
      }
    }
    if (!ok && clear &&
        geometry_exact(gp.min_sq_dist, gp.rigidity_tol, grec, g, pv.geom, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, &T)) {
      ok = true;
      res_it = c0.x + 1;
    }
    if (ok) {
      hyp[out] = T;
      hok[out] = 1;
      hiters[out] = res_it;
    }
  }
  // The recorded triplet can only fail here if the suspect list overflowed (its Kabsch was
  // not classified); any such slot continues exactly from the next attempt.
  const bool cont = clear && !ok;
  if (!__syncthreads_or(cont)) return;
  // continuation on the exact path (suspect list overflowed): the tables the draws need
  for (int i = threadIdx.x; i <= kMaxModeUnion; i += blockDim.x) {
    const uint64_t n = i ? static_cast<uint64_t>(i) : 1;
    const uint64_t m = barrett_m(n);
    s_m[i] = m;
  }
  if (threadIdx.x < kMaxTrees) s_lbase[threadIdx.x] = gp.leaf_base[threadIdx.x];
  __syncthreads();
  if (!cont) return;
  const uint64_t G = static_cast<uint64_t>(fr.gcount[f]);
  const uint64_t mG = barrett_m(G), tG = mod_barrett(0 - G, G, mG);
  const float ifx = 1.0f / g.fx, ify = 1.0f / g.fy;
  const bool fast = gp.fast != 0;
  Rng rng = rng_stream(seeds[a], static_cast<uint64_t>(slot));
  const int att = c0.x;
  int it = 0;
  int g0, g1, g2, m0, m1, m2;
  for (; it <= att; ++it)  // replay through the recorded attempt
    attempt_exact(rng, gp, fr, pv, s_lbase, s_m, fbase, G, mG, tG, fast, g0, g1, g2, m0, m1, m2);
  for (; it < gp.max_iters && !ok; ++it) {
    if (attempt_exact(rng, gp, fr, pv, s_lbase, s_m, fbase, G, mG, tG, fast, g0, g1, g2, m0, m1, m2) == kAttPass &&
        geometry_prefilter(gp.min_sq_dist, gp.rigidity_tol, grec, g, ifx, ify, pv.geom, g0, g1, g2, m0, m1, m2))
      ok = geometry_exact(gp.min_sq_dist, gp.rigidity_tol, grec, g, pv.geom, g0, g1, g2, m0, m1, m2, &T);
  }
  if (ok) hyp[out] = T;
  hok[out] = ok ? 1 : 0;
  hiters[out] = it;  // ok: the passing attempt + 1; otherwise max_iters
  if (work) atomicAdd(&work[W_GEN_ATTEMPTS], static_cast<unsigned long long>(it - (att + 1)));
}

// Generation diagnostics (scr_debug_generation_stats): thread per slot of one frame runs
// generate_hypothesis on the exact sequential path and histograms the outcome of every
// attempt by rejection tag (NoModes, ColourCheckFailed, TooClose, NotRigid,
// DegenerateKabsch; tag 0 counts the successful final attempts). Not on the hot path.
__global__ void k_gen_stats(GenParams gp, FrameGeom g, FrameRefs fr, PredView pv, uint64_t seed,
                            unsigned long long* __restrict__ tags, int* __restrict__ slots_ok) {
  __shared__ uint64_t s_m[kMaxModeUnion + 1];
  __shared__ int s_lbase[kMaxTrees];
  __shared__ unsigned long long s_tag[6];
  for (int i = threadIdx.x; i <= kMaxModeUnion; i += blockDim.x) s_m[i] = barrett_m(i ? static_cast<uint64_t>(i) : 1);
  if (threadIdx.x < kMaxTrees) s_lbase[threadIdx.x] = gp.leaf_base[threadIdx.x];
  if (threadIdx.x < 6) s_tag[threadIdx.x] = 0;
  __syncthreads();
  const int slot = blockIdx.x * blockDim.x + threadIdx.x;
  const int f = fr.fidx[0];
  const size_t fbase = static_cast<size_t>(f) * fr.gmax;
  const uint64_t G = static_cast<uint64_t>(fr.gcount[f]);
  unsigned long long cnt[6] = {0, 0, 0, 0, 0, 0};
  bool ok = false;
  if (slot < gp.nmax && G > 0) {
    const uint64_t mG = barrett_m(G), tG = mod_barrett(0 - G, G, mG);
    const int4* grec = fr.grec + 2 * fbase;
    Rng rng = rng_stream(seed, static_cast<uint64_t>(slot));
    for (int it = 0; it < gp.max_iters && !ok; ++it) {
      int g0, g1, g2, m0, m1, m2;
      const int r = attempt_exact(rng, gp, fr, pv, s_lbase, s_m, fbase, G, mG, tG, gp.fast != 0, g0, g1, g2, m0, m1,
                                  m2);
      if (r != kAttPass) {
        ++cnt[r];
        continue;
      }
      double cm[9], w[9];
      int why = 0;
      if (!distance_checks_f64(gp.min_sq_dist, gp.rigidity_tol, grec, g, pv.geom, g0, g1, g2, m0, m1, m2, cm, w,
                               nullptr, &why)) {
        ++cnt[why];
        continue;
      }
      Pose T;
      if (!kabsch3_cold(cm, w, &T)) {
        ++cnt[kAttDegenerate];
        continue;
      }
      ++cnt[kAttPass];
      ok = true;
    }
  }
  for (int i = 0; i < 6; ++i)
    if (cnt[i]) atomicAdd(&s_tag[i], cnt[i]);
  if (ok) atomicAdd(slots_ok, 1);
  __syncthreads();
  if (threadIdx.x < 6 && s_tag[threadIdx.x]) atomicAdd(&tags[threadIdx.x], s_tag[threadIdx.x]);
}

// Sample batch k of frame a: eta draws of uniform_int(G) from Rng::stream(seed, nmax + k).
// Sample batches 0..K of every frame in one launch: thread (frame a, batch blockIdx.y)
// draws the batch's eta pixels from its own stream Rng::stream(seed, N_max + batch) (A2).
__global__ void k_draw_samples(FrameRefs fr, const uint64_t* __restrict__ seeds, int nA, int nmax, int eta,
                               int scap, int* __restrict__ samples) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  const int batch = blockIdx.y;
  if (a >= nA) return;
  const uint64_t G = static_cast<uint64_t>(fr.gcount[fr.fidx[a]]);
  int* out = samples + static_cast<size_t>(a) * scap + static_cast<size_t>(batch) * eta;
  if (G == 0) {
    for (int i = 0; i < eta; ++i) out[i] = 0;
    return;
  }
  Rng rng = rng_stream(seeds[a], static_cast<uint64_t>(nmax) + static_cast<uint64_t>(batch));
  const uint64_t mG = barrett_m(G), tG = mod_barrett(0 - G, G, mG);
  for (int i = 0; i < eta; ++i) out[i] = static_cast<int>(draw_exact(rng, G, mG, tG));
}

// ================================ K5: Eq. 5 energy =========================================
// Energy is accumulated per eta-sample batch (E = sum_b E_b in batch order, E_b sequential
// over the batch's samples; DESIGN.md numerics contract). One CTA per (frame, batch,
// hypothesis tile): the batch's camera points and the predicted modes of its samples are
// staged in shared memory (chunked by a mode budget), then each thread owns one
// hypothesis and sweeps the staged samples in order; all threads read the same staged
// mode at the same time (shared-memory broadcast), so the inner loop is pure FP32.
// Per-sample predicted-mode list (union over trees in tree order) for warp-cooperative
// staging: lanes 0..T-1 fetch (slot, count) of their tree, shuffled to the whole warp.
struct SampleModes {
  int slot[kMaxTrees];
  int end[kMaxTrees];  // cumulative counts
};

SCR_DEV void sample_modes(const FrameRefs& fr, const int* pcount, size_t gb, int lane, SampleModes& sm) {
  int myslot = 0, mycnt = 0;
  if (lane < fr.T) {
    myslot = fr.gslot[gb * fr.T + lane];
    mycnt = pcount[myslot];
  }
  int run = 0;
#pragma unroll
  for (int t = 0; t < kMaxTrees; ++t) {
    const int sl = __shfl_sync(0xffffffffu, myslot, t);
    const int c = __shfl_sync(0xffffffffu, mycnt, t);
    run += (t < fr.T) ? c : 0;
    sm.slot[t] = sl;
    sm.end[t] = run;
  }
}

// ================================ K4b: compaction of generated hypotheses ===================
// Most generation slots exhaust their attempts (hok = 0); scoring only the generated ones,
// in slot order with their slot kept as the tie-break key, selects exactly what scoring all
// n_max slots with +inf for the failed ones would.
constexpr int kCompactThreads = 1024;

__global__ void __launch_bounds__(kCompactThreads) k_compact(const Pose* __restrict__ hyp, const int* __restrict__ hok,
                                                            int nmax, Pose* __restrict__ hypc, int* __restrict__ hslot,
                                                            int* __restrict__ hvalid) {
  __shared__ int s_warp[kCompactThreads / 32];
  const int a = blockIdx.x;
  const size_t base = static_cast<size_t>(a) * nmax;
  const int per = (nmax + kCompactThreads - 1) / kCompactThreads;  // consecutive slots per thread (<= 4)
  const int i0 = min(nmax, threadIdx.x * per), i1 = min(nmax, i0 + per);
  int mask = 0, cnt = 0;
  for (int i = i0; i < i1; ++i)
    if (hok[base + i]) {
      mask |= 1 << (i - i0);
      ++cnt;
    }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    int w = s_warp[lane];
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += v;
    }
    s_warp[lane] = wi - w;
    if (lane == 31) hvalid[a] = wi;
  }
  __syncthreads();
  int pos = s_warp[wid] + incl - cnt;
  for (int i = i0; i < i1; ++i)
    if (mask >> (i - i0) & 1) {
      hypc[base + pos] = hyp[base + i];
      hslot[base + pos] = i;
      ++pos;
    }
}

// Lane l stages mode j0 + l of the sample into buf[3 l .. 3 l + 2] (coalesced fetch, one
// L2 round trip per 32 modes); returns the global mode index it staged (-1 if none).
SCR_DEV int stage_modes(const PredView& pv, const SampleModes& sm, int T, int nm, int j0, int lane, float4* buf,
                        bool with_cov = true) {
  const int j = j0 + lane;
  if (j >= nm) return -1;
  // tree of mode j and the modes before it; the slot is selected in registers (a runtime
  // index into sm.slot would put the struct in local memory)
  int slot = sm.slot[0], before = 0;
#pragma unroll
  for (int q = 0; q < kMaxTrees - 1; ++q)
    if (q < T - 1 && j >= sm.end[q]) {
      slot = sm.slot[q + 1];
      before = sm.end[q];
    }
  const int mi = slot * kMaxModes + (j - before);
  const ModeGeom& g = pv.geom[mi];
  buf[3 * lane + 0] = g.q0;
  if (with_cov) {  // the Euclidean association (no prediction covariance) needs only mu
    buf[3 * lane + 1] = g.q1;
    buf[3 * lane + 2] = g.q2;
  }
  return mi;
}


constexpr int kEnergySampleCap = 512;   // eta <= 512 (Table 4)
constexpr int kEnergyBatches = 8;       // sample batches per frame (1 + halvings)

struct EnergyArgs {
  const Pose* poses;
  const int* ok;
  int stride;
  const int* nper;
  int min_n;
  const int* samples;
  int scap, eta, batch0;
  float* out;
  int kb;  // 0: out[a*stride + h] = E_b; else out[(a*stride + h)*kb + b] = E_b
};

// Energies of 64 hypotheses [64 x, 64 x + 64) on one sample batch: warp per sample, lane l
// owns hypotheses l and l + 32, so each predicted mode is loaded once per warp (coalesced
// staging) and used for 2 x 32 hypotheses. Per-sample energies e[h][s] go to shared
// memory; thread h then adds its row in sample order (the batch energy E_b, same bits as a
// sequential sweep: samples without modes contribute +0). Used for the first scoring of
// the generated hypotheses (grid.x = n_max / 64, blocks past the generated count exit) and
// for the re-scoring of the <= 64 survivors.
constexpr int kSmallHyps = 64;

#ifndef SCR_ES_THREADS
#define SCR_ES_THREADS 512
#endif
constexpr int kEsThreads = SCR_ES_THREADS;  // warps per frame-tile: more samples in flight per frame

#ifndef SCR_ES_MINB
#define SCR_ES_MINB 1
#endif
__global__ void __launch_bounds__(kEsThreads, SCR_ES_MINB) k_energy_small(EnergyArgs ea, FrameRefs fr, PredView pv,
                                                      unsigned long long* __restrict__ work) {
  extern __shared__ float es_e[];  // [kSmallHyps][eta + 1]
  __shared__ float s_pose[kSmallHyps][12];
  __shared__ float4 s_modes[(kEsThreads / 32) * 96];  // per-warp staging: 32 modes x 3 float4
  const int a = blockIdx.z, b = ea.batch0 + blockIdx.y;
  const int n_all = ea.nper ? ea.nper[a] : ea.stride;
  if (n_all <= ea.min_n) return;
  const int hbase = blockIdx.x * kSmallHyps;
  if (hbase >= n_all) return;
  const int n = min(kSmallHyps, n_all - hbase);
  const Pose* poses = ea.poses + hbase;
  float* out = ea.out + hbase * (ea.kb ? ea.kb : 1);
  for (int h = threadIdx.x; h < n; h += blockDim.x) {
    const Pose& P = poses[static_cast<size_t>(a) * ea.stride + h];
#pragma unroll
    for (int i = 0; i < 9; ++i) s_pose[h][i] = static_cast<float>(P.R[i]);
#pragma unroll
    for (int i = 0; i < 3; ++i) s_pose[h][9 + i] = static_cast<float>(P.t[i]);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int h0 = lane, h1 = lane + 32;
  const bool v0 = h0 < n, v1 = h1 < n;
  float R0[9], t0[3], R1[9], t1[3];
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    R0[i] = v0 ? s_pose[h0][i] : 0.0f;
    R1[i] = v1 ? s_pose[h1][i] : 0.0f;
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    t0[i] = v0 ? s_pose[h0][9 + i] : 0.0f;
    t1[i] = v1 ? s_pose[h1][9 + i] : 0.0f;
  }
  const int f = fr.fidx[a];
  const size_t fbase = static_cast<size_t>(f) * fr.gmax;
  const int* smp = ea.samples + static_cast<size_t>(a) * ea.scap + static_cast<size_t>(b) * ea.eta;
  const int eta = ea.eta, ld = eta + 1;
  unsigned long long evals = 0, sevals = 0;
  float4* wbuf = s_modes + wid * 96;
  for (int s = wid; s < eta; s += nw) {
    const size_t gb = fbase + smp[s];
    const int nm = fr.gnm[gb];
    float e0 = 0.0f, e1 = 0.0f;
    if (nm > 0) {
      const float4 c = fr.gcam[gb];
      float y0[3], y1[3];
      xform_f32(R0, t0, c.x, c.y, c.z, y0);
      xform_f32(R1, t1, c.x, c.y, c.z, y1);
      float m0 = __int_as_float(0x7f800000), m1 = m0;
      SampleModes sm;
      sample_modes(fr, pv.count, gb, lane, sm);
      for (int j0 = 0; j0 < nm; j0 += 32) {
        stage_modes(pv, sm, fr.T, nm, j0, lane, wbuf);
        __syncwarp();
        const int cnt = min(32, nm - j0);
        for (int m = 0; m < cnt; ++m) {
          const float4 q0 = wbuf[3 * m], q1 = wbuf[3 * m + 1], q2 = wbuf[3 * m + 2];
          m0 = fminf(m0, quad_icov(q0.w, q1.x, q1.y, q1.z, q1.w, q2.x, __fsub_rn(y0[0], q0.x),
                                   __fsub_rn(y0[1], q0.y), __fsub_rn(y0[2], q0.z)));
          m1 = fminf(m1, quad_icov(q0.w, q1.x, q1.y, q1.z, q1.w, q2.x, __fsub_rn(y1[0], q0.x),
                                   __fsub_rn(y1[1], q0.y), __fsub_rn(y1[2], q0.z)));
        }
        __syncwarp();
      }
      e0 = __fsqrt_rn(fmaxf(m0, 0.0f));
      e1 = __fsqrt_rn(fmaxf(m1, 0.0f));
      if (lane == 0) {
        evals += static_cast<unsigned long long>(nm) * static_cast<unsigned long long>(n);
        sevals += static_cast<unsigned long long>(n);
      }
    }
    if (v0) es_e[h0 * ld + s] = e0;
    if (v1) es_e[h1 * ld + s] = e1;
  }
  __syncthreads();
  if (threadIdx.x < n) {
    const int h = threadIdx.x;
    float E = 0.0f;
    for (int s = 0; s < eta; ++s) E = __fadd_rn(E, es_e[h * ld + s]);
    const size_t idx = static_cast<size_t>(a) * ea.stride + h;
    if (ea.kb == 0) out[idx] = E;
    else out[idx * ea.kb + b] = E;
  }
  if (work && lane == 0 && sevals) {
    atomicAdd(&work[W_MODE_EVALS], evals);
    atomicAdd(&work[W_SAMPLE_EVALS], sevals);
  }
}

// Re-scoring of at most 2 L candidates (L < 32 lanes per sample): a warp works on 32 / L
// samples at once, lane j of a sample's group owning candidates j and j + L, so the warp's
// instruction stream is shared by 32 / L samples instead of one. Each lane walks its
// sample's predicted modes tree by tree with direct loads (the group's lanes read the same
// addresses); the per-sample minimum does not depend on the mode order, and the batch sum
// is taken in sample order exactly as in k_energy_small.
#ifndef SCR_EG_THREADS
#define SCR_EG_THREADS 512
#endif
constexpr int kEgThreads = SCR_EG_THREADS;

template <int L>
__global__ void __launch_bounds__(kEgThreads) k_energy_grouped(EnergyArgs ea, FrameRefs fr, PredView pv,
                                                        unsigned long long* __restrict__ work) {
  constexpr int G = 32 / L;
  extern __shared__ float es_e[];  // [2 L][eta + 1]
  __shared__ float s_pose[2 * L][12];
  const int a = blockIdx.z, b = ea.batch0 + blockIdx.y;
  const int n = ea.nper ? ea.nper[a] : ea.stride;
  if (n <= ea.min_n) return;
  for (int h = threadIdx.x; h < n && h < 2 * L; h += blockDim.x) {
    const Pose& P = ea.poses[static_cast<size_t>(a) * ea.stride + h];
#pragma unroll
    for (int i = 0; i < 9; ++i) s_pose[h][i] = static_cast<float>(P.R[i]);
#pragma unroll
    for (int i = 0; i < 3; ++i) s_pose[h][9 + i] = static_cast<float>(P.t[i]);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int grp = lane / L, j = lane % L;
  const int hA = j, hB = j + L;
  const bool vA = hA < n, vB = hB < n;
  float RA[9], tA[3], RB[9], tB[3];
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    RA[i] = vA ? s_pose[hA][i] : 0.0f;
    RB[i] = vB ? s_pose[hB][i] : 0.0f;
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    tA[i] = vA ? s_pose[hA][9 + i] : 0.0f;
    tB[i] = vB ? s_pose[hB][9 + i] : 0.0f;
  }
  const int f = fr.fidx[a];
  const size_t fbase = static_cast<size_t>(f) * fr.gmax;
  const int* smp = ea.samples + static_cast<size_t>(a) * ea.scap + static_cast<size_t>(b) * ea.eta;
  const int eta = ea.eta, ld = eta + 1;
  unsigned long long evals = 0, sevals = 0;
  for (int s = wid * G + grp; s < eta; s += nw * G) {
    const size_t gb = fbase + smp[s];
    const int nm = fr.gnm[gb];
    float eA = 0.0f, eB = 0.0f;
    if (nm > 0) {
      int slot[kMaxTrees], cnt[kMaxTrees];
#pragma unroll
      for (int t = 0; t < kMaxTrees; ++t) slot[t] = t < fr.T ? fr.gslot[gb * fr.T + t] : 0;
#pragma unroll
      for (int t = 0; t < kMaxTrees; ++t) cnt[t] = t < fr.T ? pv.count[slot[t]] : 0;
      const float4 c = fr.gcam[gb];
      float yA[3], yB[3];
      xform_f32(RA, tA, c.x, c.y, c.z, yA);
      xform_f32(RB, tB, c.x, c.y, c.z, yB);
      float mA = __int_as_float(0x7f800000), mB = mA;
#pragma unroll
      for (int t = 0; t < kMaxTrees; ++t) {
        const ModeGeom* mg = pv.geom + static_cast<size_t>(slot[t]) * kMaxModes;
#pragma unroll 2
        for (int q = 0; q < cnt[t]; ++q) {
          const float4 q0 = mg[q].q0, q1 = mg[q].q1, q2 = mg[q].q2;
          mA = fminf(mA, quad_icov(q0.w, q1.x, q1.y, q1.z, q1.w, q2.x, __fsub_rn(yA[0], q0.x), __fsub_rn(yA[1], q0.y),
                                   __fsub_rn(yA[2], q0.z)));
          mB = fminf(mB, quad_icov(q0.w, q1.x, q1.y, q1.z, q1.w, q2.x, __fsub_rn(yB[0], q0.x), __fsub_rn(yB[1], q0.y),
                                   __fsub_rn(yB[2], q0.z)));
        }
      }
      eA = __fsqrt_rn(fmaxf(mA, 0.0f));
      eB = __fsqrt_rn(fmaxf(mB, 0.0f));
      if (j == 0) {
        evals += static_cast<unsigned long long>(nm) * static_cast<unsigned long long>(min(n, 2 * L));
        sevals += static_cast<unsigned long long>(min(n, 2 * L));
      }
    }
    if (vA) es_e[hA * ld + s] = eA;
    if (vB) es_e[hB * ld + s] = eB;
  }
  __syncthreads();
  if (threadIdx.x < n && threadIdx.x < 2 * L) {
    const int h = threadIdx.x;
    float E = 0.0f;
    for (int q = 0; q < eta; ++q) E = __fadd_rn(E, es_e[h * ld + q]);
    const size_t idx = static_cast<size_t>(a) * ea.stride + h;
    if (ea.kb == 0) ea.out[idx] = E;
    else ea.out[idx * ea.kb + b] = E;
  }
  if (work) {
    work_add(work, W_MODE_EVALS, static_cast<unsigned>(evals));
    work_add(work, W_SAMPLE_EVALS, static_cast<unsigned>(sevals));
  }
}

// E(I_k) = base + E_b0 + ... + E_b1 in batch order (base = E(I_{k-1}) when poses did not move).
__global__ void k_energy_sum(const int* __restrict__ ncand, int n_out, int stride, int kb, int b0, int b1,
                             const float* __restrict__ base, const float* __restrict__ part, float* __restrict__ out) {
  const int a = blockIdx.x, h = threadIdx.x;
  const int n = ncand[a];
  if (n <= n_out || h >= n) return;
  const size_t idx = static_cast<size_t>(a) * stride + h;
  float E = base ? base[idx] : 0.0f;
  for (int b = b0; b <= b1; ++b) E = __fadd_rn(E, part[idx * kb + b]);
  out[idx] = E;
}

// ================================ K7: cull / halving ========================================
// One CTA per frame: bitonic sort of keys (energy bits << 32 | slot << 12 | position),
// i.e. ascending energy with ties to the lower generation slot, then the
// first `keep` entries become the candidate list.
__global__ void __launch_bounds__(1024) k_select(const Pose* __restrict__ src_pose, const float* __restrict__ src_e,
                                                 const int* __restrict__ src_ok, const int* __restrict__ src_slot,
                                                 int src_stride, const int* __restrict__ src_n, int n_fixed,
                                                 int keep_cap, int n_out, int halving, Pose* __restrict__ cand,
                                                 float* __restrict__ cenergy, int* __restrict__ cslot,
                                                 int* __restrict__ ncand, int cand_stride) {
  extern __shared__ unsigned long long keys[];
  const int a = blockIdx.x;
  const int n = src_n ? src_n[a] : n_fixed;
  if (halving && n <= n_out) return;
  int P = 1;
  while (P < n) P <<= 1;
  const size_t base = static_cast<size_t>(a) * src_stride;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    unsigned long long k = ~0ull;
    if (i < n && (!src_ok || src_ok[base + i])) {
      const float e = src_e[base + i];
      const uint32_t eb = isnan(e) ? 0x7f800000u : __float_as_uint(e);
      const uint32_t sl = src_slot ? static_cast<uint32_t>(src_slot[base + i]) : static_cast<uint32_t>(i);
      k = (static_cast<unsigned long long>(eb) << 32) | (static_cast<unsigned long long>(sl) << 12) |
          static_cast<unsigned long long>(i);
    }
    keys[i] = k;
  }
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const unsigned long long x = keys[i], y = keys[ixj];
          const bool up = (i & k) == 0;
          if ((x > y) == up) {
            keys[i] = y;
            keys[ixj] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  int valid = 0;
  if (src_ok) {
    __shared__ int cnt;
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    int local = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) local += src_ok[base + i] ? 1 : 0;
    atomicAdd(&cnt, local);
    __syncthreads();
    valid = cnt;
  } else {
    valid = n;
  }
  const int keep = halving ? (n + 1) / 2 : min(valid, keep_cap);
  // gather into registers first: for halving the source and destination alias
  Pose p;
  float e = 0.0f;
  int sl = 0;
  const bool mine = threadIdx.x < keep;
  if (mine) {
    const int pos = static_cast<int>(keys[threadIdx.x] & 0xfffull);
    p = src_pose[base + pos];
    e = src_e[base + pos];
    sl = src_slot ? src_slot[base + pos] : pos;
  }
  __syncthreads();
  if (mine) {
    const size_t o = static_cast<size_t>(a) * cand_stride + threadIdx.x;
    cand[o] = p;
    cenergy[o] = e;
    cslot[o] = sl;
  }
  if (threadIdx.x == 0) ncand[a] = keep;
}

// ================================ K6: Levenberg-Marquardt ===================================
// One warp per (frame, candidate). Lanes own samples i = lane (mod 32); association
// (nearest mode, frozen per step) in f32, normal equations in f64 reduced with the xor
// butterfly (identical on every lane, so every lane takes the same accept/reject path).
struct LmArgs {
  int ns, scap, cand_stride, n_out, use_cov;
};

// The part of a mode record LM needs: mu and Sigma^-1/2 (s00 s01 s02 s11 s12 s22).
struct LmMode {
  float mu[3], s[6];
};
SCR_DEV LmMode lm_mode(const ModeGeom* geom, int mi, bool use_cov) {
  LmMode m;
  const float4 q0 = geom[mi].q0;
  m.mu[0] = q0.x;
  m.mu[1] = q0.y;
  m.mu[2] = q0.z;
  if (use_cov) {
    const float4 q2 = geom[mi].q2, q3 = geom[mi].q3;
    m.s[0] = q2.y; m.s[1] = q2.z; m.s[2] = q2.w; m.s[3] = q3.x; m.s[4] = q3.y; m.s[5] = q3.z;
  } else {
    m.s[0] = m.s[3] = m.s[5] = 1.0f;
    m.s[1] = m.s[2] = m.s[4] = 0.0f;
  }
  return m;
}

SCR_DEV void lm_accum(const Pose& H, const double x[3], const LmMode& mg, bool use_cov, double acc[28], bool jac) {
  double y[3];
  pose_apply(H, x, y);
  const double d0 = y[0] - static_cast<double>(mg.mu[0]), d1 = y[1] - static_cast<double>(mg.mu[1]),
               d2 = y[2] - static_cast<double>(mg.mu[2]);
  double S[9];
  if (use_cov) {
    S[0] = mg.s[0]; S[1] = mg.s[1]; S[2] = mg.s[2];
    S[3] = mg.s[1]; S[4] = mg.s[3]; S[5] = mg.s[4];
    S[6] = mg.s[2]; S[7] = mg.s[4]; S[8] = mg.s[5];
  } else {
#pragma unroll
    for (int i = 0; i < 9; ++i) S[i] = (i % 4 == 0) ? 1.0 : 0.0;
  }
  double r[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) r[i] = (S[3 * i + 0] * d0 + S[3 * i + 1] * d1) + S[3 * i + 2] * d2;
  acc[27] = acc[27] + ((r[0] * r[0] + r[1] * r[1]) + r[2] * r[2]);
  if (!jac) return;
  double J[3][6];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    J[i][0] = S[3 * i + 1] * (-y[2]) + S[3 * i + 2] * y[1];
    J[i][1] = S[3 * i + 0] * y[2] + S[3 * i + 2] * (-y[0]);
    J[i][2] = S[3 * i + 0] * (-y[1]) + S[3 * i + 1] * y[0];
    J[i][3] = S[3 * i + 0];
    J[i][4] = S[3 * i + 1];
    J[i][5] = S[3 * i + 2];
  }
  int k = 0;
#pragma unroll
  for (int a = 0; a < 6; ++a)
#pragma unroll
    for (int b = a; b < 6; ++b, ++k) acc[k] = acc[k] + ((J[0][a] * J[0][b] + J[1][a] * J[1][b]) + J[2][a] * J[2][b]);
#pragma unroll
  for (int a = 0; a < 6; ++a) acc[21 + a] = acc[21 + a] + ((J[0][a] * r[0] + J[1][a] * r[1]) + J[2][a] * r[2]);
}

// LM state per (frame, candidate) lives in global memory so that each LM iteration can be
// split into two well-shaped kernels:
//  k_lm_assoc_c — warp per sample: nearest mode of H x (f32 metric of Eq. 5, or Euclidean
//               without covariance) for every hypothesis that needs a fresh association,
//               over the compacted list of those hypotheses; modes staged 32 at a time;
//  k_lm_step  — warp per hypothesis, lanes over samples in the canonical 32-lane order:
//               normal equations with the frozen association, damped solve, trial
//               energy, accept/reject (identical on every lane).
struct LmState {
  double lambda;
  int need_assoc, done;
};

__global__ void k_lm_init(const int* __restrict__ ncand, int n_out, int cand_stride, LmState* __restrict__ st) {
  const int a = blockIdx.x, h = threadIdx.x;
  if (h >= cand_stride) return;
  LmState s;
  s.lambda = 1e-3;
  s.need_assoc = 1;
  s.done = (ncand[a] <= n_out || h >= ncand[a]) ? 1 : 0;
  st[static_cast<size_t>(a) * cand_stride + h] = s;
}

// Global mode index of union position j of a sample's predicted modes (trees in order).
SCR_DEV int union_mode(const SampleModes& sm, int T, int j) {
  int slot = sm.slot[0], before = 0;
#pragma unroll
  for (int q = 0; q < kMaxTrees - 1; ++q)
    if (q < T - 1 && j >= sm.end[q]) {
      slot = sm.slot[q + 1];
      before = sm.end[q];
    }
  return slot * kMaxModes + (j - before);
}

// Quadratic form of staged mode jj at point y (Eq. 5 metric, or Euclidean).
template <bool kCov>
SCR_DEV float assoc_q(const float4* wbuf, const float* wc12, int jj, const float* y) {
  const float4 g0 = wbuf[2 * jj];
  const float d0 = __fsub_rn(y[0], g0.x), d1 = __fsub_rn(y[1], g0.y), d2 = __fsub_rn(y[2], g0.z);
  if (kCov) {
    const float4 g1 = wbuf[2 * jj + 1];
    return quad_icov(g0.w, g1.x, g1.y, g1.z, g1.w, wc12[jj], d0, d1, d2);
  }
  return quad_eucl(d0, d1, d2);
}
// One staged chunk of the first-minimum scans. A lane's first evaluated mode is taken
// unconditionally (whatever its value, as the sequential scan does), later ones on q < best.
template <bool kCov>
SCR_DEV void assoc_chunk_two(const float4* wbuf, const float* wc12, int j0, int cnt, const float* y, const float* y2,
                             float& bq, int& bj, float& bq2, int& bj2) {
  int jj = 0;
  if (j0 == 0) {
    bq = assoc_q<kCov>(wbuf, wc12, 0, y);
    bq2 = assoc_q<kCov>(wbuf, wc12, 0, y2);
    bj = bj2 = 0;
    jj = 1;
  }
#pragma unroll 4
  for (; jj < cnt; ++jj) {
    const float q = assoc_q<kCov>(wbuf, wc12, jj, y), q2 = assoc_q<kCov>(wbuf, wc12, jj, y2);
    if (q < bq) {
      bq = q;
      bj = j0 + jj;
    }
    if (q2 < bq2) {
      bq2 = q2;
      bj2 = j0 + jj;
    }
  }
}
template <bool kCov>
SCR_DEV void assoc_chunk_g(const float4* wbuf, const float* wc12, int j0, int cnt, int sub, int G, const float* y,
                           float& bq, int& bj) {
  int jj = sub;
  if (j0 == 0 && jj < cnt) {
    bq = assoc_q<kCov>(wbuf, wc12, jj, y);
    bj = jj;
    jj += G;
  }
#pragma unroll 4
  for (; jj < cnt; jj += G) {
    const float q = assoc_q<kCov>(wbuf, wc12, jj, y);
    if (q < bq) {
      bq = q;
      bj = j0 + jj;
    }
  }
}

#ifndef SCR_ASSOC_SPW
#define SCR_ASSOC_SPW 8
#endif
constexpr int kAssocSpw = SCR_ASSOC_SPW;  // samples per warp in k_lm_assoc_c
#ifndef SCR_ASSOC_MINB
#define SCR_ASSOC_MINB 4  // 64 registers, 32 warps per SM: the association is latency-bound
#endif

// Association over the candidates that need it (<= 64 per frame), compacted: only the
// candidates of this frame with !done && need_assoc take part (after the first iteration most
// have converged or had their step rejected). Warp per sample; with nn <= 32 of them, each
// gets G = 32 / pow2ceil(nn) lanes that stride the staged modes and min-reduce (quadratic
// form, union position); with nn > 32 every lane scans all modes for two of
// them. Both give the sequential first minimum over union positions.
__global__ void __launch_bounds__(256, SCR_ASSOC_MINB) k_lm_assoc_c(FrameRefs fr, PredView pv, LmArgs la,
                                                    const int* __restrict__ samples, const Pose* __restrict__ cand,
                                                    const int* __restrict__ ncand, const LmState* __restrict__ st,
                                                    int* __restrict__ assoc, unsigned long long* __restrict__ work) {
  __shared__ float s_pose[64][12];
  __shared__ int s_list[64];
  __shared__ int s_nn;
  __shared__ float4 s_modes[8 * 64];  // per warp: 32 staged modes x {mu + c00, c11 c22 2c01 2c02}
  __shared__ float s_c12[8 * 32];     // ... and 2c12
  const int a = blockIdx.y;
  const int n = ncand[a];
  if (n <= la.n_out) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (wid == 0) {  // ascending list of the candidates that need a fresh association
    int need[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int h = lane + 32 * u;
      need[u] = 0;
      if (h < n) {
        const LmState ls = st[static_cast<size_t>(a) * la.cand_stride + h];
        need[u] = (!ls.done && ls.need_assoc) ? 1 : 0;
      }
    }
    const unsigned b0 = __ballot_sync(0xffffffffu, need[0]), b1 = __ballot_sync(0xffffffffu, need[1]);
    const unsigned below = (1u << lane) - 1u;
    if (need[0]) s_list[__popc(b0 & below)] = lane;
    if (need[1]) s_list[__popc(b0) + __popc(b1 & below)] = lane + 32;
    if (lane == 0) s_nn = __popc(b0) + __popc(b1);
  }
  __syncthreads();
  const int nn = s_nn;
  if (nn == 0) return;
  for (int i = threadIdx.x; i < nn; i += blockDim.x) {
    const Pose& P = cand[static_cast<size_t>(a) * la.cand_stride + s_list[i]];
#pragma unroll
    for (int k = 0; k < 9; ++k) s_pose[i][k] = static_cast<float>(P.R[k]);
#pragma unroll
    for (int k = 0; k < 3; ++k) s_pose[i][9 + k] = static_cast<float>(P.t[k]);
  }
  __syncthreads();
  const int f = fr.fidx[a];
  const bool two = nn > 32;
  int G = 1;
  if (!two)
    while (G * 2 * nn <= 32) G *= 2;
  const int h = two ? lane : lane / G, sub = two ? 0 : lane % G;
  const bool v = h < nn, v2 = two && lane + 32 < nn;
  // each warp takes samples s, s + 8 * gridDim.x, ... (the candidate list and poses above
  // are set up once per CTA for several samples)
  for (int s = blockIdx.x * (blockDim.x >> 5) + wid; s < la.ns; s += gridDim.x * (blockDim.x >> 5)) {
    const size_t gb = static_cast<size_t>(f) * fr.gmax + samples[static_cast<size_t>(a) * la.scap + s];
    const int nm = fr.gnm[gb];
    int bj = 0x7fffffff, bj2 = 0x7fffffff, bmi = -1, bmi2 = -1;
    SampleModes sm;
    if (nm > 0) {  // warp-uniform
      sample_modes(fr, pv.count, gb, lane, sm);
      const float4 c = fr.gcam[gb];
      float y[3], y2[3];
      {
        const int hh = v ? h : 0;
        float R[9], t[3];
  #pragma unroll
        for (int i = 0; i < 9; ++i) R[i] = s_pose[hh][i];
  #pragma unroll
        for (int i = 0; i < 3; ++i) t[i] = s_pose[hh][9 + i];
        xform_f32(R, t, c.x, c.y, c.z, y);
      }
      if (two) {
        const int hh = v2 ? lane + 32 : 0;
        float R[9], t[3];
  #pragma unroll
        for (int i = 0; i < 9; ++i) R[i] = s_pose[hh][i];
  #pragma unroll
        for (int i = 0; i < 3; ++i) t[i] = s_pose[hh][9 + i];
        xform_f32(R, t, c.x, c.y, c.z, y2);
      }
      float bq = 0.0f, bq2 = 0.0f;
      float4* wbuf = s_modes + wid * 64;
      float* wc12 = s_c12 + wid * 32;
      for (int j0 = 0; j0 < nm; j0 += 32) {
        const int jl = j0 + lane;  // lane l stages mode j0 + l
        if (jl < nm) {
          const int mi = union_mode(sm, fr.T, jl);
          wbuf[2 * lane] = pv.geom[mi].q0;
          if (la.use_cov) {
            wbuf[2 * lane + 1] = pv.geom[mi].q1;
            wc12[lane] = pv.geom[mi].q2.x;
          }
        }
        __syncwarp();
        const int cnt = min(32, nm - j0);
        if (two) {
          if (la.use_cov) assoc_chunk_two<true>(wbuf, wc12, j0, cnt, y, y2, bq, bj, bq2, bj2);
          else assoc_chunk_two<false>(wbuf, wc12, j0, cnt, y, y2, bq, bj, bq2, bj2);
        } else if (v) {
          if (la.use_cov) assoc_chunk_g<true>(wbuf, wc12, j0, cnt, sub, G, y, bq, bj);
          else assoc_chunk_g<false>(wbuf, wc12, j0, cnt, sub, G, y, bq, bj);
        }
        __syncwarp();
      }
      for (int off = two ? 0 : G >> 1; off >= 1; off >>= 1) {  // stays inside the aligned G-lane group
        const float oq = __shfl_xor_sync(0xffffffffu, bq, off);
        const int oj = __shfl_xor_sync(0xffffffffu, bj, off);
        if (oj != 0x7fffffff && (bj == 0x7fffffff || oq < bq || (oq == bq && oj < bj))) {
          bq = oq;
          bj = oj;
        }
      }
      if (bj != 0x7fffffff) bmi = union_mode(sm, fr.T, bj);
      if (bj2 != 0x7fffffff) bmi2 = union_mode(sm, fr.T, bj2);
      if (work && lane == 0)
        atomicAdd(&work[W_LM_ASSOC], static_cast<unsigned long long>(nm) * static_cast<unsigned long long>(nn));
    }
    if (v && sub == 0) assoc[(static_cast<size_t>(a) * la.cand_stride + s_list[h]) * la.scap + s] = bmi;
    if (v2) assoc[(static_cast<size_t>(a) * la.cand_stride + s_list[lane + 32]) * la.scap + s] = bmi2;
  }
}

// One LM iteration of one hypothesis, all lanes in lockstep.
__device__ __noinline__ bool lm_solve(const double* acc, double lambda, double delta[6]) {
  double M[36], rhs[6];
  int k = 0;
#pragma unroll 1
  for (int p = 0; p < 6; ++p)
#pragma unroll 1
    for (int q = p; q < 6; ++q, ++k) {
      M[6 * p + q] = acc[k];
      M[6 * q + p] = acc[k];
    }
#pragma unroll 1
  for (int p = 0; p < 6; ++p) {
    M[6 * p + p] = M[6 * p + p] + lambda * M[6 * p + p];
    rhs[p] = -acc[21 + p];
  }
  return chol6(M, rhs, delta);
}

#ifndef SCR_LM_INFLIGHT
#define SCR_LM_INFLIGHT 4
#endif
constexpr int kLmInFlight = SCR_LM_INFLIGHT;  // sample gathers in flight per lane
constexpr int kLmThreads = 128;  // canonical LM reduction lanes per candidate (4 warps)

#ifndef SCR_LM_STEP_MINB
#define SCR_LM_STEP_MINB 4  // 128 registers (a little spilling), 16 warps per SM
#endif
__global__ void __launch_bounds__(kLmThreads, SCR_LM_STEP_MINB) k_lm_step(FrameRefs fr, PredView pv, LmArgs la,
                                                 const int* __restrict__ samples, Pose* __restrict__ cand,
                                                 const int* __restrict__ ncand, LmState* __restrict__ st,
                                                 const int* __restrict__ assoc, unsigned long long* __restrict__ work) {
  __shared__ double s_red[kLmThreads / 32][28];
  __shared__ double s_tot[28];
  __shared__ Pose s_Hn;
  __shared__ int s_ok;
  const int a = blockIdx.y;
  const int h = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int n = ncand[a];
  if (n <= la.n_out || h >= n) return;  // uniform over the CTA
  const size_t hi = static_cast<size_t>(a) * la.cand_stride + h;
  LmState ls = st[hi];
  if (ls.done) return;
  const int f = fr.fidx[a];
  const size_t fbase = static_cast<size_t>(f) * fr.gmax;
  const int* smp = samples + static_cast<size_t>(a) * la.scap;
  const int* as = assoc + hi * la.scap;
  const bool use_cov = la.use_cov != 0;
  const Pose H = cand[hi];
  double acc[28];
#pragma unroll
  for (int k = 0; k < 28; ++k) acc[k] = 0.0;
  int terms = 0;
  // lane l of the CTA accumulates samples l, l + 128, ... in order; kLmInFlight of them
  // are gathered before any is accumulated (the loads are independent, the sums are not)
  for (int i0 = tid; i0 < la.ns; i0 += kLmThreads * kLmInFlight) {
    int mi[kLmInFlight];
    float4 c[kLmInFlight];
    LmMode gm[kLmInFlight];
#pragma unroll
    for (int u = 0; u < kLmInFlight; ++u) {
      const int i = i0 + kLmThreads * u;
      mi[u] = i < la.ns ? as[i] : -1;
      if (mi[u] >= 0) {
        c[u] = fr.gcam[fbase + smp[i]];
        gm[u] = lm_mode(pv.geom, mi[u], use_cov);
      }
    }
#pragma unroll
    for (int u = 0; u < kLmInFlight; ++u)
      if (mi[u] >= 0) {
        const double x[3] = {static_cast<double>(c[u].x), static_cast<double>(c[u].y), static_cast<double>(c[u].z)};
        lm_accum(H, x, gm[u], use_cov, acc, true);
        ++terms;
      }
  }
  if (work) work_add(work, W_LM_TERMS, static_cast<unsigned>(terms));
  // canonical 128-lane reduction: xor butterfly inside each warp, then (W0 + W1) + (W2 + W3)
  {
    double v[32];
#pragma unroll
    for (int k = 0; k < 28; ++k) v[k] = acc[k];
    warp_sum_xor_many<28>(v);
    if (lane < 28) s_red[wid][lane] = v[0];
  }
  __syncthreads();
  if (tid < 28) s_tot[tid] = (s_red[0][tid] + s_red[1][tid]) + (s_red[2][tid] + s_red[3][tid]);
  __syncthreads();
  ls.need_assoc = 0;
  const double E = s_tot[27];
  if (!(E > 0.0)) {
    ls.done = 1;
  } else {
    if (tid == 0) {  // damped solve + update once per candidate, shared through shared memory
      double delta[6];
      s_ok = lm_solve(s_tot, ls.lambda, delta) ? 1 : 0;
      if (s_ok) {
        Pose D;
        exp_se3(delta, D);
        pose_compose(D, H, s_Hn);
      }
    }
    __syncthreads();
    if (!s_ok) {
      ls.lambda = ls.lambda * 10.0;
    } else {
      const Pose Hn = s_Hn;
      double en[1] = {0.0};
      for (int i0 = tid; i0 < la.ns; i0 += kLmThreads * kLmInFlight) {
        int mi[kLmInFlight];
        float4 c[kLmInFlight];
        LmMode gm[kLmInFlight];
#pragma unroll
        for (int u = 0; u < kLmInFlight; ++u) {
          const int i = i0 + kLmThreads * u;
          mi[u] = i < la.ns ? as[i] : -1;
          if (mi[u] >= 0) {
            c[u] = fr.gcam[fbase + smp[i]];
            gm[u] = lm_mode(pv.geom, mi[u], use_cov);
          }
        }
#pragma unroll
        for (int u = 0; u < kLmInFlight; ++u)
          if (mi[u] >= 0) {
            const double x[3] = {static_cast<double>(c[u].x), static_cast<double>(c[u].y),
                                 static_cast<double>(c[u].z)};
            double accn[28];
            accn[27] = en[0];
            lm_accum(Hn, x, gm[u], use_cov, accn, false);
            en[0] = accn[27];
          }
      }
      const double ew = warp_sum_xor(en[0]);
      __syncthreads();  // s_red reuse
      if (lane == 0) s_red[wid][0] = ew;
      __syncthreads();
      const double En = (s_red[0][0] + s_red[1][0]) + (s_red[2][0] + s_red[3][0]);
      if (En < E) {
        ls.lambda = ls.lambda * 0.1;
        ls.need_assoc = 1;
        if ((E - En) / E < 1e-6) ls.done = 1;
        if (tid == 0) cand[hi] = Hn;
      } else {
        ls.lambda = ls.lambda * 10.0;
      }
    }
  }
  if (tid == 0) st[hi] = ls;
}

// ================================ K8-K10: ICP + raycast + depth-difference score ============
// One 8-CTA thread-block cluster (8 x 256 threads) per (frame, candidate) job. Thread
// lane l = rank * 256 + tid owns pixels p = l (mod 2048) of every pass (the canonical
// order of DESIGN.md). Per-thread partials are f32; each CTA widens them to f64 and
// reduces them (warp xor butterfly, then its 8 warps in order); CTA 0 then adds the 8
// CTA partials in rank order through distributed shared memory, solves the 6x6 system
// and publishes the new pose, which the other CTAs read back over DSMEM.
namespace cg = cooperative_groups;
constexpr int kIcpCtas = 8;
constexpr int kIcpThreads = 256;
constexpr int kIcpLanes = kIcpCtas * kIcpThreads;
constexpr double kIcpStopStep = 1e-6;  // oracle.hpp: a level stops once every |twist component| < this

struct IcpArgs {
  int cand_stride, n_cand_jobs;  // jobs per frame (1 for icp/raw, n_out for ranked)
  int do_icp;
  int job0;                      // first job of this chunk
  size_t map_stride;
};

template <int NV>
__device__ __forceinline__ void cta_reduce_f32(const float* v, double (*red)[32], double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const double s = warp_sum_xor(static_cast<double>(v[k]));
    if (lane == 0) red[wid][k] = s;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = red[0][threadIdx.x];
    for (int w = 1; w < kIcpThreads / 32; ++w) s = s + red[w][threadIdx.x];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

constexpr int kMaxImageW = 1280, kMaxImageH = 960;

// Per-level normalised ray tables (x - cx) / fx and (y - cy) / fy (IEEE division, the
// same values ray_dir computes per pixel).
__device__ __forceinline__ void fill_ray_tables(int W, int H, float fx, float fy, float cx, float cy, float* dcx,
                                                float* dcy) {
  for (int x = threadIdx.x; x < W; x += blockDim.x) dcx[x] = __fdiv_rn(__fsub_rn(static_cast<float>(x), cx), fx);
  for (int y = threadIdx.x; y < H; y += blockDim.x) dcy[y] = __fdiv_rn(__fsub_rn(static_cast<float>(y), cy), fy);
}

// Warp 0 builds the ascending list of primitives that can be seen from (R, o) with the
// given intrinsics; the ray casts of the pass then only test those (identical hits).
__device__ __forceinline__ void build_plist(const Prim* prims, int nprims, const float R[9], const float o[3],
                                            float fx, float fy, float cx, float cy, int W, int H,
                                            unsigned char* list, int* count) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int base = 0;
    for (int i0 = 0; i0 < nprims; i0 += 32) {
      const int i = i0 + lane;
      const bool in = i < nprims && prim_in_view(prims[i], R, o, fx, fy, cx, cy, W, H);
      const unsigned bal = __ballot_sync(0xffffffffu, in);
      if (in) list[base + __popc(bal & ((1u << lane) - 1u))] = static_cast<unsigned char>(i);
      base += __popc(bal);
    }
    if (lane == 0) *count = base;
  }
  __syncthreads();
}

// Per-tile visibility masks: the image is cut into 32 x 8 pixel tiles (a warp's 32
// consecutive pixels of a row always fall in one tile: every level's width is a multiple
// of 32), and bit j of a tile's mask says whether list entry j can be hit by any ray of
// the tile (conservative frustum test). The ray casts then test only those primitives,
// still in ascending order, so hits are identical to testing the whole list.
constexpr int kTileW = 32, kTileH = 8;
constexpr int kMaxTiles = (kMaxImageW / kTileW) * (kMaxImageH / kTileH);

__device__ __forceinline__ void build_tile_masks(const Prim* prims, const unsigned char* list, int nl,
                                                 const float R[9], const float o[3], float fx, float fy, float cx,
                                                 float cy, int W, int H, uint32_t* masks) {
  const int tw = (W + kTileW - 1) / kTileW, th = (H + kTileH - 1) / kTileH;
  for (int t = threadIdx.x; t < tw * th; t += blockDim.x) {
    const int tx = t % tw, ty = t / tw;
    const float x0 = static_cast<float>(tx * kTileW) - 0.5f;
    const float x1 = static_cast<float>(min(W, tx * kTileW + kTileW) - 1) + 0.5f;
    const float y0 = static_cast<float>(ty * kTileH) - 0.5f;
    const float y1 = static_cast<float>(min(H, ty * kTileH + kTileH) - 1) + 0.5f;
    uint32_t m = 0;
    for (int j = 0; j < nl; ++j)
      if (prim_in_frustum(prims[list[j]], R, o, fx, fy, cx, cy, x0, x1, y0, y1)) m |= 1u << j;
    masks[t] = m;
  }
  __syncthreads();
}

__device__ __forceinline__ int cta_isum(int v, int* ired) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_isum(v);
  if (lane == 0) ired[wid] = v;
  __syncthreads();
  int s = 0;
  for (int w = 0; w < kIcpThreads / 32; ++w) s += ired[w];
  __syncthreads();
  return s;
}

// Gauss-Newton step of ICP on the reduced normal equations (one thread): damped 6x6
// Cholesky solve, T <- exp(delta) T. Kept out of line (and un-unrolled) so its f64
// temporaries do not set the register budget of the pixel loops.
#ifdef SCR_ICP_STEP_INLINE
SCR_DEV
#else
__device__ __noinline__
#endif
int icp_step(const double* tot, Pose* T) {
  double M[36], rhs[6], delta[6];
  int k = 0;
#pragma unroll 1
  for (int p = 0; p < 6; ++p)
#pragma unroll 1
    for (int q = p; q < 6; ++q, ++k) {
      M[6 * p + q] = tot[k];
      M[6 * q + p] = tot[k];
    }
  const double mu = 1e-6 * ((((((tot[0] + tot[6]) + tot[11]) + tot[15]) + tot[18]) + tot[20]) / 6.0);
#pragma unroll 1
  for (int p = 0; p < 6; ++p) {
    rhs[p] = -tot[21 + p];
    M[6 * p + p] = M[6 * p + p] + mu;
  }
  if (!chol6(M, rhs, delta)) return 0;
  // the level has converged once the step is below kIcpStopStep in every twist component:
  // such a step only moves the pose within the f32 noise floor, so it is not applied and
  // the level ends (A8)
  double dmax = 0.0;
#pragma unroll 1
  for (int a = 0; a < 6; ++a) dmax = fmax(dmax, fabs(delta[a]));
  if (dmax < kIcpStopStep) return 2;
  Pose D, Tn;
  exp_se3(delta, D);
  pose_compose(D, *T, Tn);
  *T = Tn;
  return 1;
}

#ifndef SCR_ICP_PIX
#define SCR_ICP_PIX 3
#endif
constexpr int kIcpPix = SCR_ICP_PIX;  // live pixels per lane in flight in the association loop
struct IcpPix {  // one live pixel of the association loop in flight
  int x, y, q, ui, vi;
  float dl, pw[3];
};

// p -> (p mod W, p div W) for 0 <= p < 2^24 without an integer division: the float
// quotient is within one of the true one, fixed by one correction step.
SCR_DEV void divmod_w(int p, int W, float invW, int& x, int& y) {
  int q = __float2int_rz(__fmul_rn(__int2float_rn(p), invW));
  int r = p - q * W;
  if (r < 0) {
    --q;
    r += W;
  } else if (r >= W) {
    ++q;
    r -= W;
  }
  x = r;
  y = q;
}

// (x, y) of pixel p + d where (dx, dy) = (d mod W, d div W), from (x, y) of p: one carry.
SCR_DEV void xy_advance(int& x, int& y, int dx, int dy, int W) {
  x += dx;
  y += dy;
  if (x >= W) {
    x -= W;
    ++y;
  }
}

#ifndef SCR_ICP_MINB
#define SCR_ICP_MINB 4
#endif
// kTsdf: the scene model is a fused TSDF volume (A13) instead of the analytic
// primitives; map entries then carry {t, packed normal} instead of {t, prim | face << 16}.
template <bool kTsdf>
__global__ void __cluster_dims__(kIcpCtas, 1, 1) __launch_bounds__(kIcpThreads, SCR_ICP_MINB)
    k_icp_score(IcpArgs ia, FrameGeom g, FrameRefs fr, const Prim* __restrict__ prims, int nprims,
                const Pose* __restrict__ cand, const int* __restrict__ ncand, uint2* __restrict__ maps,
                Pose* __restrict__ out_pose, int* __restrict__ out_conv, double* __restrict__ out_rms,
                double* __restrict__ out_inl, double* __restrict__ out_score, unsigned long long* __restrict__ work,
                TsdfView tv) {
  __shared__ double red[kIcpThreads / 32][32];
  __shared__ double part2[2][32];  // this CTA's f64 partials, double-buffered by iteration parity
  __shared__ int ipart2[2][4];     // (read by every CTA of the cluster over DSMEM)
  double* part = part2[0];
  int* ipart = ipart2[0];
  __shared__ int ired[kIcpThreads / 32];
  __shared__ Pose Ts;           // current estimate (authoritative copy in CTA 0)
  __shared__ int stop_level;
  __shared__ int moved0;  // the pose changed after the level-0 map was cast
  __shared__ unsigned char s_plist[256];
  __shared__ int s_pn;
  // ray tables and tile masks sized to the frame (dynamic shared memory): a smaller
  // shared-memory carve-out leaves more L1 for the depth-plane and model-map gathers
  extern __shared__ uint32_t s_dyn[];
  float* s_dcx = reinterpret_cast<float*>(s_dyn);
  float* s_dcy = s_dcx + g.W;
  uint32_t* s_tmask = reinterpret_cast<uint32_t*>(s_dcy + g.H);
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = static_cast<int>(cluster.block_rank());
  const int lane_id = rank * kIcpThreads + threadIdx.x;
  const int jl = blockIdx.x / kIcpCtas;  // job within this launch
  const int job = ia.job0 + jl;
  const int a = job / ia.n_cand_jobs, c = job % ia.n_cand_jobs;
  if (c >= ncand[a]) return;  // uniform over the cluster
  const int f = fr.fidx[a];
  const size_t cidx = static_cast<size_t>(a) * ia.cand_stride + c;
  const size_t WHf = static_cast<size_t>(g.W) * g.H;
  const float* dpl0 = fr.dplane + static_cast<size_t>(f) * (WHf + WHf / 4 + WHf / 16);
  uint2* map = maps + static_cast<size_t>(jl) * ia.map_stride;
  if (threadIdx.x == 0) {
    Ts = cand[cidx];
    moved0 = 0;
  }
  __syncthreads();
  int last_inl = 0, last_valid = 0;
  double last_r2 = 0.0;
  bool have_stats = false;
  __shared__ int lstat[2];
  __shared__ double lstat_r2;
  int pbuf = 0;
  if (ia.do_icp) {
    for (int level = 2; level >= 0; --level) {
      const int fs = 1 << level;
      const int Wl = g.W / fs, Hl = g.H / fs;
      const float* dpl = dpl0 + (level == 0 ? 0 : (level == 1 ? WHf : WHf + WHf / 4));  // dense level plane
      const float fxl = static_cast<float>(g.dfx / fs), fyl = static_cast<float>(g.dfy / fs);
      const float cxl = static_cast<float>(g.dcx / fs), cyl = static_cast<float>(g.dcy / fs);
      const Pose Tref = Ts;
      Pose Tinv;
      pose_invert(Tref, Tinv);
      // Tinv.R is the exact transpose of Tref.R, so float(Tinv.R[3i+j]) == Rr[3j+i]: the
      // inverse rotation is read from Rr transposed (9 fewer registers in the pixel loops)
      float Rr[9], tr[3], ti[3];
#pragma unroll
      for (int i = 0; i < 9; ++i) Rr[i] = static_cast<float>(Tref.R[i]);
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        tr[i] = static_cast<float>(Tref.t[i]);
        ti[i] = static_cast<float>(Tinv.t[i]);
      }
      // K8: model map of this level at the reference pose (split over the cluster)
      if (work && rank == 0 && threadIdx.x == 0) atomicAdd(&work[W_RAYS], static_cast<unsigned long long>(Wl * Hl));
      fill_ray_tables(Wl, Hl, fxl, fyl, cxl, cyl, s_dcx, s_dcy);  // synced by build_plist
      int npl = 0;
      if (!kTsdf) {
        build_plist(prims, nprims, Rr, tr, fxl, fyl, cxl, cyl, Wl, Hl, s_plist, &s_pn);
        npl = s_pn;
      } else {
        __syncthreads();  // ray tables visible
      }
      const bool tiled = !kTsdf && npl <= 32 && (Wl % kTileW) == 0;
      if (tiled) build_tile_masks(prims, s_plist, npl, Rr, tr, fxl, fyl, cxl, cyl, Wl, Hl, s_tmask);
      unsigned long long tests = 0;
      const int twl = Wl / kTileW;
      const float invWl = __fdiv_rn(1.0f, static_cast<float>(Wl));
      const int sdx = kIcpLanes % Wl, sdy = kIcpLanes / Wl;  // pixel stride of a lane in (x, y)
      int rx, ry;
      divmod_w(lane_id, Wl, invWl, rx, ry);
      for (int p = lane_id; p < Wl * Hl; p += kIcpLanes, xy_advance(rx, ry, sdx, sdy, Wl)) {
        const int x = rx, y = ry;
        float d[3];
        ray_dir_tab(Rr, s_dcx[x], s_dcy[y], d);
        uint2 v = make_uint2(0u, 0xffffffffu);
        if (kTsdf) {
          float t;
          uint32_t nrm;
          if (tsdf_raycast_ray(tv, tr, d, &t, &nrm) && nrm != 0xffffffffu) v = make_uint2(__float_as_uint(t), nrm);
        } else {
          Hit h;
          if (tiled) {
            const uint32_t m = s_tmask[(y / kTileH) * twl + x / kTileW];
            tests += __popc(m);
            h = raycast_mask(prims, s_plist, m, tr, d);
          } else {
            tests += npl;
            h = raycast_list(prims, s_plist, npl, tr, d);
          }
          if (h.prim >= 0 && h.t <= kRenderMaxDepth) v = make_uint2(__float_as_uint(h.t), h.prim | (h.face << 16));
        }
        map[p] = v;
      }
      if (work) work_add(work, W_RAY_PRIMS, static_cast<unsigned>(tests));
      cluster.sync();  // map complete and visible to the whole cluster
      int rx0, ry0;
      divmod_w(lane_id, Wl, invWl, rx0, ry0);
      const int iters = level == 2 ? 10 : (level == 1 ? 5 : 4);
      for (int it = 0; it < iters; ++it) {
        const Pose T = Ts;
        float R[9], t[3];
#pragma unroll
        for (int i = 0; i < 9; ++i) R[i] = static_cast<float>(T.R[i]);
#pragma unroll
        for (int i = 0; i < 3; ++i) t[i] = static_cast<float>(T.t[i]);
        float acc[28];
#pragma unroll
        for (int k = 0; k < 28; ++k) acc[k] = 0.0f;
        int inl = 0, valid = 0;
        // K9: projective point-to-plane association + normal equations. Two pixels of the
        // lane (p, p + kIcpLanes) are in flight at once: both depth loads, then both model-map
        // loads, then both accumulated in pixel order (same per-lane order as one at a time).
        const int npx = Wl * Hl;
        int ax = rx0, ay = ry0;  // (x, y) of pixel p
        for (int p = lane_id; p < npx; p += kIcpPix * kIcpLanes) {
          IcpPix px[kIcpPix];
#pragma unroll
          for (int u = 0; u < kIcpPix; ++u) {
            const int pp = p + u * kIcpLanes;
            px[u].x = ax;
            px[u].y = ay;
            xy_advance(ax, ay, sdx, sdy, Wl);
            px[u].dl = pp < npx ? dpl[pp] : 0.0f;
          }
#pragma unroll
          for (int u = 0; u < kIcpPix; ++u) {
            px[u].q = -1;
            if (!depth_valid(px[u].dl)) continue;
            ++valid;
            const float pc0 = __fmul_rn(s_dcx[px[u].x], px[u].dl), pc1 = __fmul_rn(s_dcy[px[u].y], px[u].dl);
            float pr[3];
#pragma unroll
            for (int i = 0; i < 3; ++i)
              px[u].pw[i] = __fmaf_rn(R[3 * i + 0], pc0, __fmaf_rn(R[3 * i + 1], pc1, __fmaf_rn(R[3 * i + 2], px[u].dl, t[i])));
#pragma unroll
            for (int i = 0; i < 3; ++i)
              pr[i] = __fmaf_rn(Rr[0 + i], px[u].pw[0],
                                __fmaf_rn(Rr[3 + i], px[u].pw[1], __fmaf_rn(Rr[6 + i], px[u].pw[2], ti[i])));
            if (!(pr[2] > 0.0f)) continue;
            const float iz = __frcp_rn(pr[2]);
            const float uf = __fmaf_rn(fxl, __fmul_rn(pr[0], iz), cxl);
            const float vf = __fmaf_rn(fyl, __fmul_rn(pr[1], iz), cyl);
            if (!(uf > -0.5f && vf > -0.5f && uf < __fsub_rn(static_cast<float>(Wl), 0.5f) &&
                  vf < __fsub_rn(static_cast<float>(Hl), 0.5f)))
              continue;
            const int ui = static_cast<int>(floorf(__fadd_rn(uf, 0.5f)));
            const int vi = static_cast<int>(floorf(__fadd_rn(vf, 0.5f)));
            if (ui < 0 || vi < 0 || ui >= Wl || vi >= Hl) continue;
            px[u].q = vi * Wl + ui;
            px[u].ui = ui;
            px[u].vi = vi;
          }
          uint2 mv[kIcpPix];
#pragma unroll
          for (int u = 0; u < kIcpPix; ++u) mv[u] = px[u].q >= 0 ? map[px[u].q] : make_uint2(0u, 0xffffffffu);
#pragma unroll
          for (int u = 0; u < kIcpPix; ++u) {
            if (mv[u].y == 0xffffffffu) continue;
            const float th = __uint_as_float(mv[u].x);
            const int ui = px[u].ui, vi = px[u].vi;
            float dm[3], m[3], nn[3];
            ray_dir_tab(Rr, s_dcx[ui], s_dcy[vi], dm);
#pragma unroll
            for (int i = 0; i < 3; ++i) m[i] = __fmaf_rn(th, dm[i], tr[i]);
            if (kTsdf) tsdf_unpack_normal(mv[u].y, nn);
            else hit_normal(prims, static_cast<int>(mv[u].y & 0xffffu), static_cast<int>(mv[u].y >> 16), m, nn);
            const float* pw = px[u].pw;
            const float df0 = __fsub_rn(pw[0], m[0]), df1 = __fsub_rn(pw[1], m[1]), df2 = __fsub_rn(pw[2], m[2]);
            const float dist2 = __fmaf_rn(df0, df0, __fmaf_rn(df1, df1, __fmul_rn(df2, df2)));
            if (!(dist2 <= 0.01f)) continue;
            const float r = __fmaf_rn(nn[0], df0, __fmaf_rn(nn[1], df1, __fmul_rn(nn[2], df2)));
            const float J[6] = {__fmaf_rn(pw[1], nn[2], -__fmul_rn(pw[2], nn[1])),
                                __fmaf_rn(pw[2], nn[0], -__fmul_rn(pw[0], nn[2])),
                                __fmaf_rn(pw[0], nn[1], -__fmul_rn(pw[1], nn[0])), nn[0], nn[1], nn[2]};
            int k = 0;
#pragma unroll
            for (int aa = 0; aa < 6; ++aa)
#pragma unroll
              for (int bb = aa; bb < 6; ++bb, ++k) acc[k] = __fmaf_rn(J[aa], J[bb], acc[k]);
#pragma unroll
            for (int aa = 0; aa < 6; ++aa) acc[21 + aa] = __fmaf_rn(J[aa], r, acc[21 + aa]);
            acc[27] = __fmaf_rn(r, r, acc[27]);
            ++inl;
          }
        }
        // One cluster barrier per iteration: every CTA reads the 8 partials over DSMEM, sums
        // them in CTA order and takes the (identical, deterministic) Gauss-Newton step
        // itself. Partials alternate between two buffers, so a CTA that runs ahead into the
        // next iteration never overwrites what a slower CTA is still reading.
        double* pb = part2[pbuf];
        // the inlier / valid counts ride along as two more values (exact small integers)
        float vals[30];
#pragma unroll
        for (int k = 0; k < 28; ++k) vals[k] = acc[k];
        vals[28] = static_cast<float>(inl);
        vals[29] = static_cast<float>(valid);
        cta_reduce_f32<30>(vals, red, pb);
        cluster.sync();  // all CTA partials of this iteration written
        if (threadIdx.x < 30) {
          double tot = cluster.map_shared_rank(pb, 0)[threadIdx.x];
          for (int r = 1; r < kIcpCtas; ++r) tot = tot + cluster.map_shared_rank(pb, r)[threadIdx.x];
          red[0][threadIdx.x] = tot;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          const double* tot = red[0];
          const int inl_t = static_cast<int>(tot[28]);
          const int valid_t = static_cast<int>(tot[29]);
          if (work && rank == 0) atomicAdd(&work[W_ICP_TERMS], static_cast<unsigned long long>(valid_t));
          if (level == 0) {
            lstat[0] = inl_t;
            lstat[1] = valid_t;
            lstat_r2 = tot[27];
          }
          const int stepped = inl_t < 6 ? 0 : icp_step(tot, &Ts);
          stop_level = stepped != 1 ? 1 : 0;
          if (level == 0 && stepped == 1) moved0 = 1;
        }
        __syncthreads();
        pbuf ^= 1;
        if (level == 0) {
          last_inl = lstat[0];
          last_valid = lstat[1];
          last_r2 = lstat_r2;
          have_stats = true;
        }
        if (stop_level) break;
      }
      cluster.sync();  // everyone is done with this level's map before it is overwritten
    }
  }
  const Pose Tf = Ts;
  int conv = 1;
  double rms = 0.0, inlf = 0.0;
  if (ia.do_icp) {  // every CTA holds the same statistics
    if (have_stats && last_valid > 0 && last_inl > 0) {
      inlf = static_cast<double>(last_inl) / static_cast<double>(last_valid);
      rms = sqrt(last_r2 / static_cast<double>(last_inl));
      conv = (inlf >= 0.5 && rms <= 0.02) ? 1 : 0;
    } else {
      inlf = 0.0;
      rms = __longlong_as_double(0x7ff0000000000000ll);
      conv = 0;
    }
    cluster.sync();  // no CTA exits or reuses its partials while another may still read them
  }
  double score = __longlong_as_double(0x7ff0000000000000ll);
  if (conv) {
    // K10: raycast at the final pose fused with the Eq. 6-7 depth difference
    float R[9], t[3];
#pragma unroll
    for (int i = 0; i < 9; ++i) R[i] = static_cast<float>(Tf.R[i]);
#pragma unroll
    for (int i = 0; i < 3; ++i) t[i] = static_cast<float>(Tf.t[i]);
    float sum = 0.0f;
    int mutual = 0, synth = 0;
    __syncthreads();
    // With ICP on the analytic model, a final pose equal to the level-0 map's pose (level 0
    // ended at its first step, A8) gives exactly the level-0 map's hits: the depth difference
    // reads them instead of casting the 307 k rays again.
    const bool reuse = !kTsdf && ia.do_icp && !moved0;
    if (reuse) {
      const int fdx = kIcpLanes % g.W, fdy = kIcpLanes / g.W;
      const float invW = __fdiv_rn(1.0f, static_cast<float>(g.W));
      int fx0, fy0;
      divmod_w(lane_id, g.W, invW, fx0, fy0);
      for (int p = lane_id; p < g.W * g.H; p += kIcpLanes, xy_advance(fx0, fy0, fdx, fdy, g.W)) {
        const uint2 v = map[p];
        if (v.y == 0xffffffffu) continue;
        const float ht = __uint_as_float(v.x);
        if (!depth_valid(ht)) continue;
        ++synth;
        const float dl = dpl0[p];
        if (!depth_valid(dl)) continue;
        ++mutual;
        sum = __fadd_rn(sum, fabsf(__fsub_rn(dl, ht)));
      }
    } else {
    if (work && rank == 0 && threadIdx.x == 0) atomicAdd(&work[W_RAYS], static_cast<unsigned long long>(g.W * g.H));
    fill_ray_tables(g.W, g.H, g.fx, g.fy, g.cx, g.cy, s_dcx, s_dcy);
    int npl = 0;
    if (!kTsdf) {
      build_plist(prims, nprims, R, t, g.fx, g.fy, g.cx, g.cy, g.W, g.H, s_plist, &s_pn);
      npl = s_pn;
    } else {
      __syncthreads();
    }
    const bool tiled = !kTsdf && npl <= 32 && (g.W % kTileW) == 0;
    if (tiled) build_tile_masks(prims, s_plist, npl, R, t, g.fx, g.fy, g.cx, g.cy, g.W, g.H, s_tmask);
    unsigned long long tests = 0;
    const int tw0 = g.W / kTileW;
    const float invW = __fdiv_rn(1.0f, static_cast<float>(g.W));
    const int fdx = kIcpLanes % g.W, fdy = kIcpLanes / g.W;
    int fx0, fy0;
    divmod_w(lane_id, g.W, invW, fx0, fy0);
    for (int p = lane_id; p < g.W * g.H; p += kIcpLanes, xy_advance(fx0, fy0, fdx, fdy, g.W)) {
      const int x = fx0, y = fy0;
      float d[3];
      ray_dir_tab(R, s_dcx[x], s_dcy[y], d);
      Hit h;
      if (kTsdf) {
        uint32_t nrm;
        h.prim = tsdf_raycast_ray(tv, t, d, &h.t, &nrm) ? 0 : -1;
      } else if (tiled) {
        const uint32_t m = s_tmask[(y / kTileH) * tw0 + x / kTileW];
        tests += __popc(m);
        h = raycast_mask(prims, s_plist, m, t, d);
      } else {
        tests += npl;
        h = raycast_list(prims, s_plist, npl, t, d);
      }
      if (h.prim < 0 || !(h.t <= kRenderMaxDepth) || !depth_valid(h.t)) continue;
      ++synth;
      const float dl = dpl0[p];
      if (!depth_valid(dl)) continue;
      ++mutual;
      sum = __fadd_rn(sum, fabsf(__fsub_rn(dl, h.t)));
    }
    if (work) work_add(work, W_RAY_PRIMS, static_cast<unsigned>(tests));
    }
    cta_reduce_f32<1>(&sum, red, part);
    const int mutual_c = cta_isum(mutual, ired);
    const int synth_c = cta_isum(synth, ired);
    if (threadIdx.x == 0) {
      ipart[0] = mutual_c;
      ipart[1] = synth_c;
    }
    cluster.sync();
    if (rank == 0 && threadIdx.x == 0) {
      double tot = part[0];
      int mutual_t = ipart[0], synth_t = ipart[1];
      for (int r = 1; r < kIcpCtas; ++r) {
        tot = tot + cluster.map_shared_rank(part, r)[0];
        mutual_t += cluster.map_shared_rank(ipart, r)[0];
        synth_t += cluster.map_shared_rank(ipart, r)[1];
      }
      if (!(static_cast<double>(synth_t) < 0.1 * static_cast<double>(g.W) * static_cast<double>(g.H) ||
            mutual_t == 0))
        score = tot / static_cast<double>(mutual_t);
    }
    cluster.sync();  // keep every CTA's shared memory alive until CTA 0 has read it
  }
  if (rank == 0 && threadIdx.x == 0) {
    out_pose[cidx] = Tf;
    out_conv[cidx] = conv;
    out_rms[cidx] = rms;
    out_inl[cidx] = inlf;
    out_score[cidx] = score;
  }
}

// Dynamic shared memory of k_icp_score: ray tables (W + H floats) + level-0 tile masks.
inline size_t icp_smem(const FrameGeom& g) {
  const size_t tiles = static_cast<size_t>((g.W + kTileW - 1) / kTileW) * ((g.H + kTileH - 1) / kTileH);
  return (static_cast<size_t>(g.W) + g.H + tiles) * sizeof(uint32_t);
}

// ================================ K11: per-frame result =====================================
__global__ void k_finalize(int nA, int mode, int cand_stride, const Pose* __restrict__ cand,
                           const int* __restrict__ ncand, const Pose* __restrict__ icp_pose,
                           const int* __restrict__ icp_conv, const double* __restrict__ icp_score,
                           scr_result* __restrict__ res) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= nA) return;
  scr_result r;
  memset(&r, 0, sizeof(r));
  r.score = __longlong_as_double(0x7ff0000000000000ll);
  const int n = ncand[a];
  r.n_candidates = n;
  const size_t b = static_cast<size_t>(a) * cand_stride;
  if (n == 0) {
    r.status = SCR_E_NO_HYPOTHESES;
  } else if (mode == SCR_MODE_RAW) {
    r.has_pose = 1;
    memcpy(&r.pose, &cand[b], sizeof(scr_pose));
    r.score = icp_score[b];
  } else if (mode == SCR_MODE_ICP) {  // a non-converged ICP discards the pose (§3.2.4)
    if (icp_conv[b]) {
      r.has_pose = 1;
      memcpy(&r.pose, &icp_pose[b], sizeof(scr_pose));
      r.score = icp_score[b];
    } else {
      r.status = SCR_E_ALL_CANDIDATES_FAILED;
    }
  } else {
    int bi = -1;
    double best = __longlong_as_double(0x7ff0000000000000ll);
    for (int c = 0; c < n; ++c) {
      const double sc = icp_conv[b + c] ? icp_score[b + c] : __longlong_as_double(0x7ff0000000000000ll);
      if (sc < best) {
        best = sc;
        bi = c;
      }
    }
    if (bi < 0) {
      r.status = SCR_E_ALL_CANDIDATES_FAILED;
    } else {
      r.has_pose = 1;
      memcpy(&r.pose, &icp_pose[b + bi], sizeof(scr_pose));
      r.score = best;
    }
  }
  res[a] = r;
}

// ================================ host orchestration ========================================
namespace {

FrameRefs frame_refs(scr_scene s) {
  FrameRefs fr;
  fr.fidx = s->ws.fidx;
  fr.gcount = s->ws.gcount;
  fr.gpx = s->ws.gpx;
  fr.gcam = s->ws.gcam;
  fr.gslot = s->ws.gslot;
  fr.gnm = s->ws.gnm;
  fr.grec = s->ws.grec;
  fr.gleaf = reinterpret_cast<const uint4*>(s->ws.grec);
  fr.tex = s->ws.tex;
  fr.dplane = s->ws.dplane;
  fr.gmax = s->ws.gmax;
  fr.T = s->T;
  return fr;
}

int halvings(int n_cull, int n_out) {
  int k = 0, n = n_cull;
  while (n > n_out) {
    n = (n + 1) / 2;
    ++k;
  }
  return k;
}

template <typename T>
scr_status grow(T** p, size_t count) {
  if (*p) cudaFree(*p);
  *p = nullptr;
  SCR_CUDA(cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(1, count) * sizeof(T)));
  return SCR_OK;
}

#define SCR_TRY(x)               \
  do {                           \
    scr_status _s = (x);         \
    if (_s != SCR_OK) return _s; \
  } while (0)

// One relocaliser stage for the nA active frames already listed in
// ws.fidx / ws.seeds. Results land in d_res[0..nA).
scr_status run_stage(scr_scene s, int nA, const scr_ransac_params& p, int mode, scr_result* d_res) {
  Workspace& w = s->ws;
  if (p.n_max <= 0 || p.n_max > 4096 || p.n_cull <= 0 || p.n_cull > 64 || p.eta <= 0 || p.n_out <= 0 ||
      p.max_gen_iters <= 0) {
    set_error("ransac params out of range (n_max <= 4096, n_cull <= 64)");
    return SCR_E_ARG;
  }
  const int K = halvings(p.n_cull, p.n_out);
  const int scap = p.eta * (K + 1);
  if (K + 1 > kEnergyBatches || p.eta > kEnergySampleCap) {
    set_error("ransac params: eta <= 512 and at most 7 sample batches (n_cull / n_out <= 64)");
    return SCR_E_ARG;
  }
  SCR_TRY(ensure_ransac_ws(s, p.n_max, p.n_cull, scap));
  const int jobs_per = mode == SCR_MODE_RANKED ? std::min(p.n_out, p.n_cull) : 1;
  // sized for a full batch, not this stage's active frames: growing the map buffer later
  // (cudaFree + cudaMalloc) would synchronise the whole device under every other lane
  SCR_TRY(ensure_icp_ws(s, std::min(w.cap * jobs_per, 1024)));
  const FrameRefs fr = frame_refs(s);
  const PredView pv = s->pred_view();
  GenParams gp{p.max_gen_iters, p.n_max, p.min_sq_dist, p.colour_thresh, p.rigidity_tol,
               (s->T <= 5 && s->leaves16) ? 1 : 0, s->gen_force_suspect, {0}};
  for (int t = 0; t < s->T && t < kMaxTrees; ++t) gp.leaf_base[t] = s->leaf_base[t];
  unsigned long long* wk = work_ptr(s);
  SCR_CUDA(cudaMemsetAsync(w.hctr, 0, nA * sizeof(int), s->stream));  // per-frame slot counters
  SCR_CUDA(cudaMemsetAsync(w.hctr + w.cap, 0, nA * sizeof(int), s->stream));  // per-frame suspect counts
  const int gen_threads = std::min(p.n_max, kGenThreadsPerFrame);
  SCR_LAUNCH(s, K_HYPGEN,
             (k_hypgen<<<dim3((gen_threads + kGenWarps * 32 - 1) / (kGenWarps * 32), nA), kGenWarps * 32,
                         gp.fast ? static_cast<size_t>((w.gmax + 15) & ~15) : 0, s->stream>>>(gp, s->geom, fr, pv, w.seeds,
                                                                                  w.hctr, w.hcand, w.hok, w.hiters,
                                                                                  w.hctr + w.cap, w.sus, wk)));
  SCR_LAUNCH(s, K_HYPFIN,
             (k_hypfin<<<dim3((p.n_max + kFinThreads - 1) / kFinThreads, nA), kFinThreads, 0, s->stream>>>(
                 gp, s->geom, fr, pv, w.seeds, w.hcand, w.hyp, w.hok, w.hiters, w.hctr + w.cap, w.sus, wk)));
  SCR_LAUNCH(s, K_SAMPLES,
             (k_draw_samples<<<dim3((nA + 63) / 64, K + 1), 64, 0, s->stream>>>(fr, w.seeds, nA, p.n_max, p.eta,
                                                                                w.samples_cap, w.samples)));
  SCR_LAUNCH(s, K_COMPACT,
             (k_compact<<<nA, kCompactThreads, 0, s->stream>>>(w.hyp, w.hok, p.n_max, w.hypc, w.hslot, w.hvalid)));
  {
    EnergyArgs ea{w.hypc, nullptr, p.n_max, w.hvalid, 0, w.samples, w.samples_cap, p.eta, 0, w.henergy, 0};
    const size_t smem = static_cast<size_t>(kSmallHyps) * (p.eta + 1) * sizeof(float);
    SCR_LAUNCH(s, K_ENERGY, (k_energy_small<<<dim3((p.n_max + kSmallHyps - 1) / kSmallHyps, 1, nA), kEsThreads, smem,
                                               s->stream>>>(ea, fr, pv, wk)));
  }
  int P = 1;
  while (P < p.n_max) P <<= 1;
  SCR_LAUNCH(s, K_SELECT,
             (k_select<<<nA, 1024, P * sizeof(unsigned long long), s->stream>>>(
                 w.hypc, w.henergy, nullptr, w.hslot, p.n_max, w.hvalid, 0, p.n_cull, p.n_out, 0, w.cand,
                 w.cenergy, w.cslot, w.ncand, w.ncull_cap)));
  LmArgs la{0, w.samples_cap, w.ncull_cap, p.n_out, p.use_cov};
  for (int k = 1; k <= K; ++k) {
    const int ns = p.eta * (k + 1);
    if (p.pose_update) {
      la.ns = ns;
      LmState* lmst = static_cast<LmState*>(w.lmst);
      SCR_LAUNCH(s, K_LM, (k_lm_init<<<nA, w.ncull_cap, 0, s->stream>>>(w.ncand, p.n_out, w.ncull_cap, lmst)));
      // candidates still in play at step k: at most ceil(n_cull / 2^(k-1))
      const int nk = (p.n_cull + (1 << (k - 1)) - 1) >> (k - 1);
      for (int it = 0; it < 10; ++it) {
        const dim3 ag((ns + 8 * kAssocSpw - 1) / (8 * kAssocSpw), nA);
        SCR_LAUNCH(s, K_LM, (k_lm_assoc_c<<<ag, 256, 0, s->stream>>>(fr, pv, la, w.samples, w.cand, w.ncand, lmst,
                                                                     w.assoc, wk)));
        SCR_LAUNCH(s, K_LM, (k_lm_step<<<dim3(nk, nA), kLmThreads, 0, s->stream>>>(
                                fr, pv, la, w.samples, w.cand, w.ncand, lmst, w.assoc, wk)));
      }
    }
    // rescore (only frames still above n_out take part): per-batch partial energies, then
    // E(I_k) = E(I_{k-1}) + E_k without LM (poses unchanged), or the full batch sum with LM
    {
      const int b0 = p.pose_update ? 0 : k;
      EnergyArgs ea{w.cand, nullptr, w.ncull_cap, w.ncand, p.n_out, w.samples, w.samples_cap, p.eta, b0, w.epart,
                    kEnergyBatches};
      // at most ceil(n_cull / 2^(k-1)) candidates take part in step k
      const int nb = (p.n_cull + (1 << (k - 1)) - 1) >> (k - 1);
      int L = 1;
      while (2 * L < nb) L <<= 1;
      const dim3 grid(1, k - b0 + 1, nA);
      const size_t smem_g = static_cast<size_t>(2 * L) * (p.eta + 1) * sizeof(float);
      if (L >= 32) {
        const size_t smem_small = static_cast<size_t>(kSmallHyps) * (p.eta + 1) * sizeof(float);
        SCR_LAUNCH(s, K_ENERGY, (k_energy_small<<<grid, kEsThreads, smem_small, s->stream>>>(ea, fr, pv, wk)));
      } else if (L == 16) {
        SCR_LAUNCH(s, K_ENERGY, (k_energy_grouped<16><<<grid, kEgThreads, smem_g, s->stream>>>(ea, fr, pv, wk)));
      } else if (L == 8) {
        SCR_LAUNCH(s, K_ENERGY, (k_energy_grouped<8><<<grid, kEgThreads, smem_g, s->stream>>>(ea, fr, pv, wk)));
      } else if (L == 4) {
        SCR_LAUNCH(s, K_ENERGY, (k_energy_grouped<4><<<grid, kEgThreads, smem_g, s->stream>>>(ea, fr, pv, wk)));
      } else if (L == 2) {
        SCR_LAUNCH(s, K_ENERGY, (k_energy_grouped<2><<<grid, kEgThreads, smem_g, s->stream>>>(ea, fr, pv, wk)));
      } else {
        SCR_LAUNCH(s, K_ENERGY, (k_energy_grouped<1><<<grid, kEgThreads, smem_g, s->stream>>>(ea, fr, pv, wk)));
      }
      SCR_LAUNCH(s, K_ENERGY, (k_energy_sum<<<nA, 64, 0, s->stream>>>(w.ncand, p.n_out, w.ncull_cap, kEnergyBatches,
                                                                      b0, k, p.pose_update ? nullptr : w.cenergy,
                                                                      w.epart, w.henergy)));
    }
    int Pc = 1;
    while (Pc < p.n_cull) Pc <<= 1;
    SCR_LAUNCH(s, K_SELECT,
               (k_select<<<nA, 1024, Pc * sizeof(unsigned long long), s->stream>>>(
                   w.cand, w.henergy, nullptr, w.cslot, w.ncull_cap, w.ncand, 0, p.n_cull, p.n_out, 1, w.cand,
                   w.cenergy, w.cslot, w.ncand, w.ncull_cap)));
  }
  SCR_CUDA(cudaGetLastError());
  // ICP / scoring jobs
  const int njobs = nA * jobs_per;
  for (int j0 = 0; j0 < njobs; j0 += w.icp_cap) {
    const int nj = std::min(w.icp_cap, njobs - j0);
    IcpArgs ia{w.ncull_cap, jobs_per, mode != SCR_MODE_RAW ? 1 : 0, j0,
               static_cast<size_t>(s->k.width) * s->k.height};
    if (s->tsdf_model) {
      SCR_LAUNCH(s, K_ICP,
                 (k_icp_score<true><<<nj * kIcpCtas, kIcpThreads, icp_smem(s->geom), s->stream>>>(
                     ia, s->geom, fr, s->d_prims, s->n_prims, w.cand, w.ncand, w.icp_map, w.icp_pose, w.icp_conv,
                     w.icp_rms, w.icp_inl, w.icp_score, wk, tsdf_view(s->tsdf_model))));
    } else {
      SCR_LAUNCH(s, K_ICP,
                 (k_icp_score<false><<<nj * kIcpCtas, kIcpThreads, icp_smem(s->geom), s->stream>>>(
                     ia, s->geom, fr, s->d_prims, s->n_prims, w.cand, w.ncand, w.icp_map, w.icp_pose, w.icp_conv,
                     w.icp_rms, w.icp_inl, w.icp_score, wk, TsdfView{})));
    }
  }
  SCR_LAUNCH(s, K_FINALIZE,
             (k_finalize<<<(nA + 127) / 128, 128, 0, s->stream>>>(nA, mode, w.ncull_cap, w.cand, w.ncand, w.icp_pose,
                                                                  w.icp_conv, w.icp_score, d_res)));
  SCR_CUDA(cudaGetLastError());
  return SCR_OK;
}

}  // namespace

#ifndef SCR_ICP_CARVE
#define SCR_ICP_CARVE 25  // 4 CTAs of ~12 KB fit; a larger carve-out costs L1 (100 %: ICP +19 %)
#endif
#ifndef SCR_GEN_CARVE
#define SCR_GEN_CARVE -1
#endif
scr_status reloc_init() {
  if (SCR_ICP_CARVE >= 0) {  // shared-memory carve-out preference (percent): the rest is L1
    SCR_CUDA(cudaFuncSetAttribute(k_icp_score<false>, cudaFuncAttributePreferredSharedMemoryCarveout, SCR_ICP_CARVE));
    SCR_CUDA(cudaFuncSetAttribute(k_icp_score<true>, cudaFuncAttributePreferredSharedMemoryCarveout, SCR_ICP_CARVE));
  }
  if (SCR_GEN_CARVE >= 0)
    SCR_CUDA(cudaFuncSetAttribute(k_hypgen, cudaFuncAttributePreferredSharedMemoryCarveout, SCR_GEN_CARVE));
  SCR_CUDA(cudaFuncSetAttribute(k_hypgen, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (kMaxImageW / 4) * (kMaxImageH / 4)));
  SCR_CUDA(cudaFuncSetAttribute(k_energy_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kSmallHyps * (kEnergySampleCap + 1) * sizeof(float))));
  SCR_CUDA(cudaFuncSetAttribute(k_energy_grouped<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(32 * (kEnergySampleCap + 1) * sizeof(float))));
  return SCR_OK;
}

scr_status ensure_ransac_ws(scr_scene s, int nmax, int ncull, int scap) {
  Workspace& w = s->ws;
  const size_t B = static_cast<size_t>(w.cap);
  if (nmax > w.nmax_cap) {
    SCR_TRY(grow(&w.hyp, B * nmax));
    SCR_TRY(grow(&w.henergy, B * std::max(nmax, 64)));
    SCR_TRY(grow(&w.hok, B * nmax));
    SCR_TRY(grow(&w.hcand, 2 * B * nmax));
    SCR_TRY(grow(&w.sus, 2 * B * kMaxSuspects));
    SCR_TRY(grow(&w.hiters, B * nmax));
    SCR_TRY(grow(&w.hypc, B * nmax));
    SCR_TRY(grow(&w.hslot, B * nmax));
    SCR_TRY(grow(&w.hvalid, B));
    w.nmax_cap = nmax;
  }
  if (ncull > w.ncull_cap || scap > w.samples_cap) {
    const int nc = std::max(ncull, w.ncull_cap), sc = std::max(scap, w.samples_cap);
    SCR_TRY(grow(&w.cand, B * nc));
    SCR_TRY(grow(&w.cenergy, B * nc));
    SCR_TRY(grow(&w.cslot, B * nc));
    SCR_TRY(grow(&w.ncand, B));
    SCR_TRY(grow(&w.samples, B * sc));
    SCR_TRY(grow(&w.assoc, B * nc * sc));
    SCR_TRY(grow(&w.icp_pose, B * nc));
    SCR_TRY(grow(&w.icp_score, B * nc));
    SCR_TRY(grow(&w.icp_conv, B * nc));
    SCR_TRY(grow(&w.icp_rms, B * nc));
    SCR_TRY(grow(&w.icp_inl, B * nc));
    SCR_TRY(grow(&w.epart, B * nc * kEnergyBatches));
    SCR_TRY(grow(reinterpret_cast<LmState**>(&w.lmst), B * nc));
    w.ncull_cap = nc;
    w.samples_cap = sc;
    if (w.henergy && static_cast<size_t>(w.nmax_cap) < static_cast<size_t>(nc)) {
      SCR_TRY(grow(&w.henergy, B * std::max(w.nmax_cap, nc)));
    }
  }
  return SCR_OK;
}

scr_status ensure_icp_ws(scr_scene s, int jobs) {
  Workspace& w = s->ws;
  jobs = std::max(jobs, 1);
  if (jobs > w.icp_cap) {
    SCR_TRY(grow(&w.icp_map, static_cast<size_t>(jobs) * s->k.width * s->k.height));
    w.icp_cap = jobs;
  }
  return SCR_OK;
}

uint64_t stage_seed(uint64_t seed, int stage) { return seed + static_cast<uint64_t>(stage) * 0x9e3779b97f4a7c15ull; }

// run_cascade for frames packed in workspace slots 0..n-1.
scr_status run_cascade(scr_scene s, int n, const scr_ransac_params* stages, const int32_t* modes, const double* thr,
                       int nstages, const uint64_t* seeds, scr_result* out) {
  // Host control between stages only: stage i+1 takes the frames whose stage-i score exceeds
  // the threshold. Staging buffers are pinned and allocated once per
  // workspace, so a call makes no allocation and no implicit device synchronisation.
  Workspace& w = s->ws;
  std::vector<int> active(n);
  for (int i = 0; i < n; ++i) active[i] = i;
  std::vector<scr_result> res(n);
  for (int st = 0; st < nstages && !active.empty(); ++st) {
    const int nA = static_cast<int>(active.size());
    for (int i = 0; i < nA; ++i) {
      w.h_idx[i] = active[i];
      w.h_seeds[i] = stage_seed(seeds[active[i]], st);
    }
    SCR_CUDA(cudaMemcpyAsync(w.fidx, w.h_idx, nA * sizeof(int), cudaMemcpyHostToDevice, s->stream));
    SCR_CUDA(cudaMemcpyAsync(w.seeds, w.h_seeds, nA * sizeof(uint64_t), cudaMemcpyHostToDevice, s->stream));
    cudaEventRecord(w.ev_stage[0], s->stream);
    SCR_TRY(run_stage(s, nA, stages[st], modes[st], w.d_res));
    cudaEventRecord(w.ev_stage[1], s->stream);
    SCR_CUDA(cudaMemcpyAsync(w.h_res, w.d_res, nA * sizeof(scr_result), cudaMemcpyDeviceToHost, s->stream));
    SCR_CUDA(cudaStreamSynchronize(s->stream));
    prof_flush(s);
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, w.ev_stage[0], w.ev_stage[1]);
    std::vector<int> next;
    for (int i = 0; i < nA; ++i) {
      const int f = active[i];
      float keep[4];
      std::memcpy(keep, res[f].stage_ms, sizeof(keep));
      res[f] = w.h_res[i];
      std::memcpy(res[f].stage_ms, keep, sizeof(keep));
      if (st < 4) res[f].stage_ms[st] = ms / nA;
      res[f].stage_used = st;
      if (st < nstages - 1 && !(w.h_res[i].score <= thr[st])) next.push_back(f);
    }
    active.swap(next);
  }
  std::memcpy(out, res.data(), n * sizeof(scr_result));
  return SCR_OK;
}

}  // namespace scr

using namespace scr;

namespace {
scr_status check_stage_args(int n, const scr_ransac_params* stages, const int32_t* modes, int nstages,
                            const uint64_t* seeds, scr_result* out) {
  if (n < 0 || !stages || !modes || nstages <= 0 || (!seeds && n > 0) || (!out && n > 0)) {
    set_error("null or empty argument");
    return SCR_E_ARG;
  }
  for (int i = 0; i < nstages; ++i)
    if (modes[i] < 0 || modes[i] > 2) {
      set_error("mode must be raw (0), icp (1) or ranked (2)");
      return SCR_E_ARG;
    }
  return SCR_OK;
}
}  // namespace

extern "C" {

scr_status scr_cascade_batch(scr_scene s, const scr_frame* frames, int n, const scr_ransac_params* stages,
                             const int32_t* modes, const double* thr, int nstages, const uint64_t* seeds,
                             scr_result* out) {
  if (!s) return SCR_E_ARG;
  SCR_TRY(check_stage_args(n, stages, modes, nstages, seeds, out));
  if (nstages > 1 && !thr) return SCR_E_ARG;
  if (!(s->parent ? (s->parent->d_prims || s->parent->tsdf_model) : (s->d_prims || s->tsdf_model))) {  // every mode scores against the model (A11)
    set_error("relocalise: no scene model set (scr_scene_set_analytic_model)");
    return SCR_E_ARG;
  }
  StateReadLock lock(s);
  SCR_CUDA(cudaSetDevice(s->dev->ordinal));
  SCR_TRY(refresh_lane(s));
  const size_t WH = static_cast<size_t>(s->k.width) * s->k.height;
  SCR_TRY(check_frames(s, frames, n));
  Workspace& w = s->ws;
  if (n > w.cap && !w.depth2) {  // second staging buffer: chunk j + 1 uploads while chunk j runs
    SCR_CUDA(cudaMalloc(&w.depth2, static_cast<size_t>(w.cap) * WH * sizeof(float)));
    SCR_CUDA(cudaMalloc(&w.rgb2, static_cast<size_t>(w.cap) * WH * 3));
    SCR_CUDA(cudaEventCreateWithFlags(&w.ev_upload2, cudaEventDisableTiming));
  }
  // chunk j's frames, contiguous on the device's copy stream, into staging buffer j % 2
  auto upload = [&](int j) -> scr_status {
    const int b0 = j * w.cap, nb = std::min(w.cap, n - b0);
    float* dd = (j & 1) ? w.depth2 : w.depth;
    uint8_t* dc = (j & 1) ? w.rgb2 : w.rgb;
    std::lock_guard<std::mutex> lk(s->dev->copy_mu);
    for (int i = 0; i < nb; ++i) {
      const scr_frame& fr = frames[b0 + i];
      SCR_CUDA(cudaMemcpyAsync(dd + i * WH, fr.depth, WH * sizeof(float), cudaMemcpyHostToDevice, s->dev->copy));
      SCR_CUDA(cudaMemcpyAsync(dc + i * WH * 3, fr.rgb, WH * 3, cudaMemcpyHostToDevice, s->dev->copy));
    }
    SCR_CUDA(cudaEventRecord((j & 1) ? w.ev_upload2 : w.ev_upload, s->dev->copy));
    return SCR_OK;
  };
  // staging is free on entry: the previous call on this lane synchronised its stream; buffer
  // j % 2 is free again for chunk j + 2 once chunk j's cascade (which synchronises) is done
  const int nchunks = (n + w.cap - 1) / w.cap;
  if (nchunks > 0) SCR_TRY(upload(0));
  for (int j = 0; j < nchunks; ++j) {
    const int b0 = j * w.cap, nb = std::min(w.cap, n - b0);
    SCR_CUDA(cudaStreamWaitEvent(s->stream, (j & 1) ? w.ev_upload2 : w.ev_upload, 0));
    SCR_TRY(pack_frames(s, (j & 1) ? w.depth2 : w.depth, (j & 1) ? w.rgb2 : w.rgb, nullptr, nb));
    if (j + 1 < nchunks) SCR_TRY(upload(j + 1));  // overlaps this chunk's cascade
    SCR_TRY(run_cascade(s, nb, stages, modes, thr, nstages, seeds + b0, out + b0));
  }
  return SCR_OK;
}

scr_status scr_relocalise_batch(scr_scene s, const scr_frame* frames, int n, const scr_ransac_params* p, int mode,
                                const uint64_t* seeds, scr_result* out) {
  const int32_t m = mode;
  return scr_cascade_batch(s, frames, n, p, &m, nullptr, 1, seeds, out);
}

scr_status scr_cascade_frameset(scr_scene s, scr_frameset fs, const int32_t* idx, int n,
                                const scr_ransac_params* stages, const int32_t* modes, const double* thr,
                                int nstages, const uint64_t* seeds, scr_result* out) {
  if (!s || !fs || (!idx && n > 0)) return SCR_E_ARG;
  SCR_TRY(check_stage_args(n, stages, modes, nstages, seeds, out));
  if (nstages > 1 && !thr) return SCR_E_ARG;
  if (!(s->parent ? (s->parent->d_prims || s->parent->tsdf_model) : (s->d_prims || s->tsdf_model))) {
    set_error("relocalise: no scene model set (scr_scene_set_analytic_model)");
    return SCR_E_ARG;
  }
  if (fs->scene != s && fs->scene != s->parent) {
    set_error("scr_cascade_frameset: the frame set belongs to another scene");
    return SCR_E_ARG;
  }
  StateReadLock lock(s);
  SCR_CUDA(cudaSetDevice(s->dev->ordinal));
  SCR_TRY(refresh_lane(s));
  for (int i = 0; i < n; ++i)
    if (idx[i] < 0 || idx[i] >= fs->cap) return SCR_E_ARG;
  for (int b0 = 0; b0 < n; b0 += s->ws.cap) {
    const int nb = std::min(s->ws.cap, n - b0);
    // the previous chunk's copy from h_fsidx completed: run_cascade synchronised the stream
    std::memcpy(s->ws.h_fsidx, idx + b0, nb * sizeof(int));
    SCR_CUDA(cudaMemcpyAsync(s->ws.status, s->ws.h_fsidx, nb * sizeof(int), cudaMemcpyHostToDevice, s->stream));
    SCR_TRY(pack_frames(s, fs->depth, fs->rgb, s->ws.status, nb));
    SCR_TRY(run_cascade(s, nb, stages, modes, thr, nstages, seeds + b0, out + b0));
  }
  return SCR_OK;
}

scr_status scr_debug_ransac(scr_scene s, const scr_frame* f, const scr_ransac_params* p, uint64_t seed,
                            int32_t* gen_slots, scr_pose* gen_poses, int* n_gen, int32_t* surv_slots,
                            scr_pose* surv_poses, float* surv_energy, int* n_surv) {
  if (!s || !f || !p || !n_gen || !n_surv) return SCR_E_ARG;
  SCR_TRY(check_frames(s, f, 1));
  StateReadLock lock(s);
  SCR_CUDA(cudaSetDevice(s->dev->ordinal));
  SCR_TRY(refresh_lane(s));
  const size_t WH = static_cast<size_t>(s->k.width) * s->k.height;
  SCR_CUDA(cudaMemcpyAsync(s->ws.depth, f->depth, WH * sizeof(float), cudaMemcpyHostToDevice, s->stream));
  SCR_CUDA(cudaMemcpyAsync(s->ws.rgb, f->rgb, WH * 3, cudaMemcpyHostToDevice, s->stream));
  SCR_TRY(pack_frames(s, s->ws.depth, s->ws.rgb, nullptr, 1));
  const int zero = 0;
  SCR_CUDA(cudaMemcpyAsync(s->ws.fidx, &zero, sizeof(int), cudaMemcpyHostToDevice, s->stream));
  SCR_CUDA(cudaMemcpyAsync(s->ws.seeds, &seed, sizeof(uint64_t), cudaMemcpyHostToDevice, s->stream));
  scr_result* d_res = nullptr;
  SCR_CUDA(cudaMalloc(&d_res, sizeof(scr_result)));
  // raw mode still needs a model for the score; skip ICP work by using raw
  const bool have_model = s->d_prims != nullptr || s->tsdf_model != nullptr;
  if (!have_model) {
    set_error("scr_debug_ransac: no scene model set");
    cudaFree(d_res);
    return SCR_E_ARG;
  }
  scr_status st = run_stage(s, 1, *p, SCR_MODE_RAW, d_res);
  cudaFree(d_res);
  if (st != SCR_OK) return st;
  SCR_CUDA(cudaStreamSynchronize(s->stream));
  const int nmax = p->n_max;
  std::vector<int> ok(nmax);
  std::vector<Pose> hp(nmax);
  SCR_CUDA(cudaMemcpy(ok.data(), s->ws.hok, nmax * sizeof(int), cudaMemcpyDeviceToHost));
  SCR_CUDA(cudaMemcpy(hp.data(), s->ws.hyp, nmax * sizeof(Pose), cudaMemcpyDeviceToHost));
  int g = 0;
  for (int i = 0; i < nmax; ++i)
    if (ok[i]) {
      if (gen_slots) gen_slots[g] = i;
      if (gen_poses) std::memcpy(&gen_poses[g], &hp[i], sizeof(scr_pose));
      ++g;
    }
  *n_gen = g;
  int nc = 0;
  SCR_CUDA(cudaMemcpy(&nc, s->ws.ncand, sizeof(int), cudaMemcpyDeviceToHost));
  std::vector<Pose> cp(std::max(1, nc));
  std::vector<int> cs(std::max(1, nc));
  std::vector<float> ce(std::max(1, nc));
  if (nc) {
    SCR_CUDA(cudaMemcpy(cp.data(), s->ws.cand, nc * sizeof(Pose), cudaMemcpyDeviceToHost));
    SCR_CUDA(cudaMemcpy(cs.data(), s->ws.cslot, nc * sizeof(int), cudaMemcpyDeviceToHost));
    SCR_CUDA(cudaMemcpy(ce.data(), s->ws.cenergy, nc * sizeof(float), cudaMemcpyDeviceToHost));
  }
  for (int i = 0; i < nc; ++i) {
    if (surv_slots) surv_slots[i] = cs[i];
    if (surv_poses) std::memcpy(&surv_poses[i], &cp[i], sizeof(scr_pose));
    if (surv_energy) surv_energy[i] = ce[i];
  }
  *n_surv = nc;
  return g == 0 ? SCR_E_NO_HYPOTHESES : SCR_OK;
}

scr_status scr_debug_generation_mode(scr_scene s, int mode) {
  if (!s || mode < 0 || mode > 1) {
    scr::set_error("scr_debug_generation_mode: bad scene or mode");
    return SCR_E_ARG;
  }
  s->gen_force_suspect = mode;
  return SCR_OK;
}

scr_status scr_debug_generation_stats(scr_scene s, const scr_frame* f, const scr_ransac_params* p, uint64_t seed,
                                      int64_t* tags, int* slots_ok) {
  if (!s || !f || !f->depth || !f->rgb || !p || !tags || !slots_ok || p->n_max <= 0 || p->n_max > 4096 ||
      p->max_gen_iters <= 0) {
    set_error("scr_debug_generation_stats: bad argument");
    return SCR_E_ARG;
  }
  SCR_TRY(check_frames(s, f, 1));
  StateReadLock lock(s);
  SCR_CUDA(cudaSetDevice(s->dev->ordinal));
  SCR_TRY(refresh_lane(s));
  const size_t WH = static_cast<size_t>(s->k.width) * s->k.height;
  SCR_CUDA(cudaMemcpyAsync(s->ws.depth, f->depth, WH * sizeof(float), cudaMemcpyHostToDevice, s->stream));
  SCR_CUDA(cudaMemcpyAsync(s->ws.rgb, f->rgb, WH * 3, cudaMemcpyHostToDevice, s->stream));
  SCR_TRY(pack_frames(s, s->ws.depth, s->ws.rgb, nullptr, 1));
  const int zero = 0;
  SCR_CUDA(cudaMemcpyAsync(s->ws.fidx, &zero, sizeof(int), cudaMemcpyHostToDevice, s->stream));
  GenParams gp{p->max_gen_iters, p->n_max, p->min_sq_dist, p->colour_thresh, p->rigidity_tol,
               (s->T <= 5 && s->leaves16) ? 1 : 0, 0, {0}};
  for (int t = 0; t < s->T && t < kMaxTrees; ++t) gp.leaf_base[t] = s->leaf_base[t];
  unsigned long long* d_tags = nullptr;
  SCR_CUDA(cudaMalloc(&d_tags, 6 * sizeof(unsigned long long) + sizeof(int)));
  int* d_ok = reinterpret_cast<int*>(d_tags + 6);
  SCR_CUDA(cudaMemsetAsync(d_tags, 0, 6 * sizeof(unsigned long long) + sizeof(int), s->stream));
  k_gen_stats<<<(p->n_max + 127) / 128, 128, 0, s->stream>>>(gp, s->geom, frame_refs(s), s->pred_view(), seed,
                                                              d_tags, d_ok);
  unsigned long long h[6];
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(h, d_tags, sizeof(h), cudaMemcpyDeviceToHost, s->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(slots_ok, d_ok, sizeof(int), cudaMemcpyDeviceToHost, s->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
  cudaFree(d_tags);
  SCR_CUDA(e);
  for (int i = 0; i < 6; ++i) tags[i] = static_cast<int64_t>(h[i]);
  return SCR_OK;
}

scr_status scr_debug_icp(scr_scene s, const scr_frame* f, const scr_pose* init, scr_pose* out, int* converged,
                         double* rms, double* inlier_frac, double* score) {
  if (!s || !f || !init || !(s->d_prims || s->tsdf_model)) return SCR_E_ARG;
  SCR_TRY(check_frames(s, f, 1));
  StateReadLock lock(s);
  SCR_CUDA(cudaSetDevice(s->dev->ordinal));
  SCR_TRY(refresh_lane(s));
  const size_t WH = static_cast<size_t>(s->k.width) * s->k.height;
  SCR_TRY(ensure_ransac_ws(s, 1, 1, 1));
  SCR_TRY(ensure_icp_ws(s, 1));
  SCR_CUDA(cudaMemcpyAsync(s->ws.depth, f->depth, WH * sizeof(float), cudaMemcpyHostToDevice, s->stream));
  SCR_CUDA(cudaMemcpyAsync(s->ws.rgb, f->rgb, WH * 3, cudaMemcpyHostToDevice, s->stream));
  SCR_TRY(pack_frames(s, s->ws.depth, s->ws.rgb, nullptr, 1));
  const int zero = 0, one = 1;
  SCR_CUDA(cudaMemcpyAsync(s->ws.fidx, &zero, sizeof(int), cudaMemcpyHostToDevice, s->stream));
  SCR_CUDA(cudaMemcpyAsync(s->ws.ncand, &one, sizeof(int), cudaMemcpyHostToDevice, s->stream));
  SCR_CUDA(cudaMemcpyAsync(s->ws.cand, init, sizeof(Pose), cudaMemcpyHostToDevice, s->stream));
  IcpArgs ia{s->ws.ncull_cap, 1, 1, 0, WH};
  if (s->tsdf_model) {
    SCR_LAUNCH(s, K_ICP, (k_icp_score<true><<<kIcpCtas, kIcpThreads, icp_smem(s->geom), s->stream>>>(
                             ia, s->geom, frame_refs(s), s->d_prims, s->n_prims, s->ws.cand, s->ws.ncand, s->ws.icp_map,
                             s->ws.icp_pose, s->ws.icp_conv, s->ws.icp_rms, s->ws.icp_inl, s->ws.icp_score, nullptr,
                             tsdf_view(s->tsdf_model))));
  } else {
    SCR_LAUNCH(s, K_ICP, (k_icp_score<false><<<kIcpCtas, kIcpThreads, icp_smem(s->geom), s->stream>>>(
                             ia, s->geom, frame_refs(s), s->d_prims, s->n_prims, s->ws.cand, s->ws.ncand, s->ws.icp_map,
                             s->ws.icp_pose, s->ws.icp_conv, s->ws.icp_rms, s->ws.icp_inl, s->ws.icp_score, nullptr,
                             TsdfView{})));
  }
  SCR_CUDA(cudaGetLastError());
  SCR_CUDA(cudaStreamSynchronize(s->stream));
  SCR_CUDA(cudaMemcpy(out, s->ws.icp_pose, sizeof(Pose), cudaMemcpyDeviceToHost));
  SCR_CUDA(cudaMemcpy(converged, s->ws.icp_conv, sizeof(int), cudaMemcpyDeviceToHost));
  SCR_CUDA(cudaMemcpy(rms, s->ws.icp_rms, sizeof(double), cudaMemcpyDeviceToHost));
  SCR_CUDA(cudaMemcpy(inlier_frac, s->ws.icp_inl, sizeof(double), cudaMemcpyDeviceToHost));
  SCR_CUDA(cudaMemcpy(score, s->ws.icp_score, sizeof(double), cudaMemcpyDeviceToHost));
  return SCR_OK;
}

}  // extern "C"

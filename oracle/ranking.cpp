// ORACLE — test infrastructure only. Never linked into the product.
//
// ranking_cascade + ICP restatement (src/ranking.cpp
// and src/scene_model.cpp are missing from the reference). The model is the
// analytic SyntheticScene (A9); ICP is projective point-to-plane on a
// 3-level pyramid with {10, 5, 4} Gauss-Newton iterations coarse->fine (A8).
// Reductions follow the 256-lane canonical order of DESIGN.md.
#include <algorithm>
#include <cmath>

#include "detmath.hpp"
#include "oracle.hpp"

namespace oracle {

namespace {
constexpr int kIcpAcc = 28;  // 21 JtJ + 6 Jtr + r^2

struct ModelMap {
  int w = 0, h = 0;
  std::vector<float> v;  // 3 per pixel (world vertex)
  std::vector<float> n;  // 3 per pixel (world normal)
  std::vector<uint8_t> valid;
};

void render_model_map(const Scene& s, const Pose& T, const Intrinsics& k, ModelMap& m) {
  float R[9], tf[3];
  for (int i = 0; i < 9; ++i) R[i] = static_cast<float>(T.R[i]);
  for (int i = 0; i < 3; ++i) tf[i] = static_cast<float>(T.t[i]);
  m.w = k.width;
  m.h = k.height;
  m.v.assign(3 * static_cast<size_t>(m.w) * m.h, 0.0f);
  m.n.assign(3 * static_cast<size_t>(m.w) * m.h, 0.0f);
  m.valid.assign(static_cast<size_t>(m.w) * m.h, 0);
  for (int y = 0; y < m.h; ++y)
    for (int x = 0; x < m.w; ++x) {
      const size_t idx = static_cast<size_t>(y) * m.w + x;
      Hit h{0.0f, -1, -1};
      uint32_t packed = 0xffffffffu;
      if (s.tsdf) {  // fused model: hit + packed normal (A13)
        if (!tsdf_raycast_pixel(*s.tsdf, R, tf, k, x, y, &h.t, &packed) || packed == 0xffffffffu) continue;
      } else {
        h = raycast_pixel(s, R, tf, k, x, y);
        if (h.prim < 0 || !(h.t <= kRenderMaxDepth)) continue;
      }
      const float dcx = (static_cast<float>(x) - static_cast<float>(k.cx)) / static_cast<float>(k.fx);
      const float dcy = (static_cast<float>(y) - static_cast<float>(k.cy)) / static_cast<float>(k.fy);
      float p[3];
      for (int i = 0; i < 3; ++i) {
        const float di = std::fma(R[3 * i + 0], dcx, std::fma(R[3 * i + 1], dcy, R[3 * i + 2]));
        p[i] = std::fma(h.t, di, tf[i]);
      }
      float nn[3];
      if (s.tsdf) unpack_normal(packed, nn);
      else hit_normal(s, h, p, nn);
      for (int i = 0; i < 3; ++i) {
        m.v[3 * idx + i] = p[i];
        m.n[3 * idx + i] = nn[i];
      }
      m.valid[idx] = 1;
    }
}

// kIcpLanes = 8 x 256 lanes (the threads of an 8-CTA cluster): lane l owns pixels
// p = l (mod kIcpLanes) in row-major order and accumulates in f32; lanes are widened to
// f64 and combined by an xor butterfly inside each 32-lane warp, the 8 warp sums of a CTA
// are added sequentially, then the 8 CTA sums are added sequentially.
void canonical_reduce(const float lanes[kIcpLanes][kIcpAcc], int nacc, double out[]) {
  static thread_local double warp_sum[kIcpLanes / 32][kIcpAcc];
  for (int w = 0; w < kIcpLanes / 32; ++w) {
    double v[32][kIcpAcc];
    for (int l = 0; l < 32; ++l)
      for (int a = 0; a < nacc; ++a) v[l][a] = static_cast<double>(lanes[32 * w + l][a]);
    for (int off = 16; off >= 1; off >>= 1) {
      double nx[32][kIcpAcc];
      for (int l = 0; l < 32; ++l)
        for (int a = 0; a < nacc; ++a) nx[l][a] = v[l][a] + v[l ^ off][a];
      for (int l = 0; l < 32; ++l)
        for (int a = 0; a < nacc; ++a) v[l][a] = nx[l][a];
    }
    for (int a = 0; a < nacc; ++a) warp_sum[w][a] = v[0][a];
  }
  for (int a = 0; a < nacc; ++a) {
    double total = 0.0;
    for (int c = 0; c < kIcpCtas; ++c) {
      double s = warp_sum[8 * c][a];
      for (int w = 1; w < 8; ++w) s = s + warp_sum[8 * c + w][a];
      total = c == 0 ? s : total + s;
    }
    out[a] = total;
  }
}
}  // namespace

// icp_refine: per level the model is ray cast at the level's start
// pose (reference view); each Gauss-Newton step associates live points projectively
// against that view, gates at 0.1 m, and solves the 6x6 point-to-plane system.
// converged iff (final inliers / valid live px) >= 0.5 and rms <= 0.02 m, measured on
// the last linearisation of the finest level.
IcpResult icp_refine(const Scene& s, const Pose& init, const Frame& fr) {
  IcpResult res;
  Pose T = init;
  int last_inl = 0, last_valid = 0;
  double last_r2 = 0.0;
  bool have_stats = false;
  for (int level = 2; level >= 0; --level) {
    const int f = 1 << level;
    const Intrinsics k = fr.k.scaled(f);
    ModelMap mm;
    render_model_map(s, T, k, mm);
    const Pose Tinv = invert(T);
    float Ri[9], ti[3];
    for (int i = 0; i < 9; ++i) Ri[i] = static_cast<float>(Tinv.R[i]);
    for (int i = 0; i < 3; ++i) ti[i] = static_cast<float>(Tinv.t[i]);
    const float fxf = static_cast<float>(k.fx), fyf = static_cast<float>(k.fy);
    const float cxf = static_cast<float>(k.cx), cyf = static_cast<float>(k.cy);
    for (int it = 0; it < kIcpIters[level]; ++it) {
      float R[9], tf[3];
      for (int i = 0; i < 9; ++i) R[i] = static_cast<float>(T.R[i]);
      for (int i = 0; i < 3; ++i) tf[i] = static_cast<float>(T.t[i]);
      static thread_local float lanes[kIcpLanes][kIcpAcc];
      static thread_local int lane_inl[kIcpLanes], lane_valid[kIcpLanes];
      for (int l = 0; l < kIcpLanes; ++l) {
        for (int a = 0; a < kIcpAcc; ++a) lanes[l][a] = 0.0f;
        lane_inl[l] = lane_valid[l] = 0;
      }
      const int W = k.width, H = k.height;
      for (int p = 0; p < W * H; ++p) {
        const int x = p % W, y = p / W;
        const float d = fr.depth[static_cast<size_t>(y * f) * fr.width + x * f];
        if (!depth_valid(d)) continue;
        const int l = p % kIcpLanes;
        lane_valid[l]++;
        const float dcx = (static_cast<float>(x) - cxf) / fxf;
        const float dcy = (static_cast<float>(y) - cyf) / fyf;
        const float pc[3] = {dcx * d, dcy * d, d};
        float pw[3], pr[3];
        for (int i = 0; i < 3; ++i)
          pw[i] = std::fma(R[3 * i + 0], pc[0], std::fma(R[3 * i + 1], pc[1], std::fma(R[3 * i + 2], pc[2], tf[i])));
        for (int i = 0; i < 3; ++i)
          pr[i] = std::fma(Ri[3 * i + 0], pw[0], std::fma(Ri[3 * i + 1], pw[1], std::fma(Ri[3 * i + 2], pw[2], ti[i])));
        if (!(pr[2] > 0.0f)) continue;
        const float iz = 1.0f / pr[2];  // one correctly rounded reciprocal, then products
        const float uf = std::fma(fxf, pr[0] * iz, cxf);
        const float vf = std::fma(fyf, pr[1] * iz, cyf);
        if (!(uf > -0.5f && vf > -0.5f && uf < W - 0.5f && vf < H - 0.5f)) continue;
        const int ui = static_cast<int>(std::floor(uf + 0.5f)), vi = static_cast<int>(std::floor(vf + 0.5f));
        if (ui < 0 || vi < 0 || ui >= W || vi >= H) continue;
        const size_t q = static_cast<size_t>(vi) * W + ui;
        if (!mm.valid[q]) continue;
        const float* mv = &mm.v[3 * q];
        const float* mn = &mm.n[3 * q];
        const float df[3] = {pw[0] - mv[0], pw[1] - mv[1], pw[2] - mv[2]};
        const float dist2 = std::fma(df[0], df[0], std::fma(df[1], df[1], df[2] * df[2]));
        if (!(dist2 <= 0.01f)) continue;
        const float r = std::fma(mn[0], df[0], std::fma(mn[1], df[1], mn[2] * df[2]));
        const float J[6] = {std::fma(pw[1], mn[2], -(pw[2] * mn[1])), std::fma(pw[2], mn[0], -(pw[0] * mn[2])),
                            std::fma(pw[0], mn[1], -(pw[1] * mn[0])), mn[0], mn[1], mn[2]};
        float* acc = lanes[l];
        int kk = 0;
        for (int a = 0; a < 6; ++a)
          for (int b = a; b < 6; ++b, ++kk) acc[kk] = std::fma(J[a], J[b], acc[kk]);
        for (int a = 0; a < 6; ++a) acc[21 + a] = std::fma(J[a], r, acc[21 + a]);
        acc[27] = std::fma(r, r, acc[27]);
        lane_inl[l]++;
      }
      double tot[kIcpAcc];
      canonical_reduce(lanes, kIcpAcc, tot);
      int inl = 0, valid = 0;
      for (int l = 0; l < kIcpLanes; ++l) {
        inl += lane_inl[l];
        valid += lane_valid[l];
      }
      if (level == 0) {
        last_inl = inl;
        last_valid = valid;
        last_r2 = tot[27];
        have_stats = true;
      }
      res.iterations++;
      if (inl < 6) break;
      double M[36], rhs[6], delta[6];
      int kk = 0;
      for (int a = 0; a < 6; ++a)
        for (int b = a; b < 6; ++b, ++kk) {
          M[6 * a + b] = tot[kk];
          M[6 * b + a] = tot[kk];
        }
      // damping mu = 1e-6 tr(A)/6 keeps directions the view does not constrain (e.g. height
      // in front of a bare wall) at their current value instead of failing the solve
      const double mu = 1e-6 * ((((((tot[0] + tot[6]) + tot[11]) + tot[15]) + tot[18]) + tot[20]) / 6.0);
      for (int a = 0; a < 6; ++a) {
        rhs[a] = -tot[21 + a];
        M[6 * a + a] = M[6 * a + a] + mu;
      }
      if (!chol6_solve(M, rhs, delta)) break;
      // the level has converged once the Gauss-Newton step is below kIcpStopStep in every
      // twist component (rad / m): such a step only moves the pose within the f32 noise floor
      // of the sums, so it is not applied and the level ends (A8)
      double dmax = 0.0;
      for (int a = 0; a < 6; ++a) dmax = std::fmax(dmax, std::fabs(delta[a]));
      if (dmax < kIcpStopStep) break;
      T = compose(exp_se3(delta), T);
    }
  }
  res.pose = T;
  if (have_stats && last_valid > 0 && last_inl > 0) {
    res.inlier_frac = static_cast<double>(last_inl) / static_cast<double>(last_valid);
    res.rms = std::sqrt(last_r2 / static_cast<double>(last_inl));
    res.converged = (res.inlier_frac >= 0.5 && res.rms <= 0.02) ? 1 : 0;
  } else {
    res.inlier_frac = 0.0;
    res.rms = kInf;
    res.converged = 0;
  }
  return res;
}

// depth_diff_score (Eqs. 6-7): mean |D_live - D_synth| over pixels valid
// in both; inf if valid(D_synth)/|Omega| < 0.1 or the mutual set is empty.
double depth_diff_images(const float* live, const float* synth, int W, int H) {
  static thread_local float lanes[kIcpLanes][kIcpAcc];
  int mutual = 0, nsynth = 0;
  for (int l = 0; l < kIcpLanes; ++l) lanes[l][0] = 0.0f;
  for (int p = 0; p < W * H; ++p) {
    const float ds = synth[p];
    if (!depth_valid(ds)) continue;
    ++nsynth;
    const float dl = live[p];
    if (!depth_valid(dl)) continue;
    ++mutual;
    lanes[p % kIcpLanes][0] = lanes[p % kIcpLanes][0] + std::fabs(dl - ds);
  }
  if (static_cast<double>(nsynth) < 0.1 * static_cast<double>(W) * static_cast<double>(H)) return kInf;
  if (mutual == 0) return kInf;
  double tot[kIcpAcc];
  canonical_reduce(lanes, 1, tot);
  return tot[0] / static_cast<double>(mutual);
}

// raycast_depth for the analytic model: exact per-pixel intersection.
void raycast_depth(const Scene& s, const Pose& T, const Intrinsics& k, float* out) {
  float R[9], tf[3];
  for (int i = 0; i < 9; ++i) R[i] = static_cast<float>(T.R[i]);
  for (int i = 0; i < 3; ++i) tf[i] = static_cast<float>(T.t[i]);
  for (int y = 0; y < k.height; ++y)
    for (int x = 0; x < k.width; ++x) {
      if (s.tsdf) {
        float t;
        uint32_t nrm;
        out[static_cast<size_t>(y) * k.width + x] = tsdf_raycast_pixel(*s.tsdf, R, tf, k, x, y, &t, &nrm) ? t : 0.0f;
        continue;
      }
      const Hit h = raycast_pixel(s, R, tf, k, x, y);
      out[static_cast<size_t>(y) * k.width + x] = (h.prim >= 0 && h.t <= kRenderMaxDepth) ? h.t : 0.0f;
    }
}

double depth_diff_score(const Scene& s, const Pose& T, const Frame& fr) {
  std::vector<float> synth(static_cast<size_t>(fr.width) * fr.height);
  raycast_depth(s, T, fr.k, synth.data());
  return depth_diff_images(fr.depth, synth.data(), fr.width, fr.height);
}

uint64_t stage_seed(uint64_t seed, int stage) { return seed + static_cast<uint64_t>(stage) * 0x9e3779b97f4a7c15ull; }

// relocalise with DESIGN.md A11: raw scores the unrefined rank-1
// pose; icp refines it (non-converged: unrefined pose kept, score inf); ranked ICPs
// and scores every survivor and picks the argmin (ties by order).
RelocResult relocalise(const RansacParams& p, int mode, const Frame& fr, const Forest& f, const AdaptState& s,
                       const Scene& model, uint64_t seed) {
  RelocResult r;
  FrameCtx c;
  build_frame_ctx(c, f, s, fr);
  std::vector<Hypothesis> hyps;
  try {
    hyps = preemptive_ransac(c, s, p, seed);
  } catch (const Error& e) {
    r.status = e.code;
    return r;
  }
  r.n_candidates = static_cast<int>(hyps.size());
  if (mode == MODE_RAW) {
    r.has_pose = 1;
    r.pose = hyps[0].pose;
    r.score = depth_diff_score(model, r.pose, fr);
  } else if (mode == MODE_ICP) {
    // "If this fails, we discard the pose" (§3.2.4): a non-converged ICP gives no
    // pose, exactly as ranked mode with one candidate (A11)
    const IcpResult ir = icp_refine(model, hyps[0].pose, fr);
    if (ir.converged) {
      r.has_pose = 1;
      r.pose = ir.pose;
      r.score = depth_diff_score(model, ir.pose, fr);
    } else {
      r.status = E_ALL_CANDIDATES_FAILED;
      r.has_pose = 0;
      r.score = kInf;
    }
  } else {
    double best = kInf;
    int bi = -1;
    Pose bp;
    for (size_t i = 0; i < hyps.size(); ++i) {
      const IcpResult ir = icp_refine(model, hyps[i].pose, fr);
      const double sc = ir.converged ? depth_diff_score(model, ir.pose, fr) : kInf;
      if (sc < best) {
        best = sc;
        bi = static_cast<int>(i);
        bp = ir.pose;
      }
    }
    if (bi < 0) {
      r.status = E_ALL_CANDIDATES_FAILED;
      r.has_pose = 0;
      r.score = kInf;
    } else {
      r.has_pose = 1;
      r.pose = bp;
      r.score = best;
    }
  }
  return r;
}

// run_cascade: stage i returns iff best_score <= tau_i; last stage
// unconditional; stage i uses stage_seed(seed, i).
RelocResult run_cascade(const RansacParams* stages, const int* modes, const double* thr, int n, const Frame& fr,
                        const Forest& f, const AdaptState& s, const Scene& model, uint64_t seed) {
  RelocResult r;
  for (int i = 0; i < n; ++i) {
    r = relocalise(stages[i], modes[i], fr, f, s, model, stage_seed(seed, i));
    r.stage_used = i;
    if (i == n - 1 || r.score <= thr[i]) return r;
  }
  return r;
}

}  // namespace oracle

// ORACLE — test infrastructure only. Never linked into the product.
//
// RANSAC restatement (src/ransac.cpp is missing from the
// reference): triplet hypothesis generation with the three checks, Eq. 5 energy,
// the initial cull, and preemptive halving with Levenberg-Marquardt in se(3).
// Frozen choices: DESIGN.md A1 (grid pixel domain), A2 (streams), A7 (colour check),
// and the numerics contract (f32 energy with explicit fma; f64 LM with the
// 32-lane canonical reduction order).
#include <algorithm>
#include <cmath>

#include "detmath.hpp"
#include "oracle.hpp"

namespace oracle {

void build_frame_ctx(FrameCtx& c, const Forest& f, const AdaptState& s, const Frame& fr) {
  c.frame = &fr;
  c.trees = static_cast<int>(f.trees.size());
  c.grid = sample_grid_pixels(fr, 4);
  const size_t G = c.grid.size();
  c.slots.assign(G * c.trees, 0);
  c.cam.assign(G * 3, 0.0);
  c.camf.assign(G * 3, 0.0f);
  c.nmodes.assign(G, 0);
  for (size_t g = 0; g < G; ++g) {
    const int x = c.grid[g] & 0xffff, y = c.grid[g] >> 16;
    int nm = 0;
    for (int t = 0; t < c.trees; ++t) {
      const int64_t slot = f.leaf_base[t] + find_leaf(f.trees[t], fr, x, y, f.specs);
      c.slots[g * c.trees + t] = slot;
      nm += s.pred_count.empty() ? 0 : s.pred_count[slot];
    }
    c.nmodes[g] = nm;
    backproject(x, y, static_cast<double>(fr.depth[static_cast<size_t>(y) * fr.width + x]), fr.k, &c.cam[3 * g]);
    for (int k = 0; k < 3; ++k) c.camf[3 * g + k] = static_cast<float>(c.cam[3 * g + k]);
  }
}

// predict_modes: union over trees in tree order.
const Mode* ctx_mode(const FrameCtx& c, const AdaptState& s, int g, int m) {
  for (int t = 0; t < c.trees; ++t) {
    const int64_t slot = c.slots[static_cast<size_t>(g) * c.trees + t];
    const int cnt = s.pred_count[slot];
    if (m < cnt) return &s.modes[static_cast<size_t>(slot) * kMaxModes + m];
    m -= cnt;
  }
  return nullptr;
}

static inline double d2_3(const double* a, const double* b) {
  const double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
  return (dx * dx + dy * dy) + dz * dz;
}

// generate_hypothesis. Draw order per attempt: for k in 0..2
// {pixel = uniform_int(G); NoModes if empty; mode = uniform_int(|M|)}, then the
// colour-check correspondence uniform_int(3) (A7).
int generate_hypothesis(const FrameCtx& c, const AdaptState& s, const RansacParams& p, Rng& rng, Pose* out,
                        int* attempts, int64_t* tags) {
  const uint64_t G = c.grid.size();
  int last = REJ_NO_MODES;
  *attempts = 0;
  if (G == 0) return REJ_NO_MODES;
  for (int it = 0; it < p.max_iters; ++it) {
    *attempts = it + 1;
    int gi[3];
    const Mode* mm[3];
    bool ok = true;
    for (int k = 0; k < 3; ++k) {
      gi[k] = static_cast<int>(rng.uniform_int(G));
      const int nm = c.nmodes[gi[k]];
      if (nm == 0) {
        ok = false;
        break;
      }
      mm[k] = ctx_mode(c, s, gi[k], static_cast<int>(rng.uniform_int(static_cast<uint64_t>(nm))));
    }
    if (!ok) {
      last = REJ_NO_MODES;
      if (tags) ++tags[REJ_NO_MODES];
      continue;
    }
    const int cc = static_cast<int>(rng.uniform_int(3));
    {
      const int g = c.grid[gi[cc]];
      const size_t idx = static_cast<size_t>(g >> 16) * c.frame->width + (g & 0xffff);
      float linf = 0.0f;
      for (int ch = 0; ch < 3; ++ch)
        linf = std::fmax(linf, std::fabs(static_cast<float>(c.frame->rgb[3 * idx + ch]) - mm[cc]->colour[ch]));
      if (linf > p.colour_thresh) {
        last = REJ_COLOUR;
        if (tags) ++tags[REJ_COLOUR];
        continue;
      }
    }
    double w[9], cm[9];
    for (int k = 0; k < 3; ++k)
      for (int q = 0; q < 3; ++q) {
        w[3 * k + q] = static_cast<double>(mm[k]->mu[q]);
        cm[3 * k + q] = c.cam[3 * static_cast<size_t>(gi[k]) + q];
      }
    last = check_triplet(cm, w, p, out);
    if (tags) ++tags[last];
    if (last == REJ_OK) return REJ_OK;
  }
  return last;
}

// Checks 2-3 and Kabsch of one colour-checked triplet: camera points cm
// and world points w (3 x 3, row per point) -> REJ_OK with the transform, or the tag.
int check_triplet(const double cm[9], const double w[9], const RansacParams& p, Pose* out) {
  static const int PA[3] = {0, 0, 1}, PB[3] = {1, 2, 2};
  bool close = false;
  double dw2[3], dc2[3];
  for (int q = 0; q < 3; ++q) {
    dw2[q] = d2_3(&w[3 * PA[q]], &w[3 * PB[q]]);
    dc2[q] = d2_3(&cm[3 * PA[q]], &cm[3 * PB[q]]);
    if (dw2[q] < p.min_sq_dist) close = true;
  }
  if (close) return REJ_TOO_CLOSE;
  for (int q = 0; q < 3; ++q)
    if (std::fabs(std::sqrt(dw2[q]) - std::sqrt(dc2[q])) > p.rigidity_tol) return REJ_NOT_RIGID;
  if (!kabsch(cm, w, 3, out)) return REJ_DEGENERATE;
  return REJ_OK;
}

void draw_samples(uint64_t seed, int batch, int n_max, int eta, int G, std::vector<int>& out) {
  Rng rng = Rng::stream(seed, static_cast<uint64_t>(n_max) + static_cast<uint64_t>(batch));
  for (int i = 0; i < eta; ++i) out.push_back(static_cast<int>(rng.uniform_int(static_cast<uint64_t>(G))));
}

static inline void pose_to_f32(const Pose& H, float R[9], float t[3]) {
  for (int i = 0; i < 9; ++i) R[i] = static_cast<float>(H.R[i]);
  for (int i = 0; i < 3; ++i) t[i] = static_cast<float>(H.t[i]);
}

static inline void xform_f32(const float R[9], const float t[3], const float* x, float y[3]) {
  for (int i = 0; i < 3; ++i)
    y[i] = std::fma(R[3 * i + 0], x[0], std::fma(R[3 * i + 1], x[1], std::fma(R[3 * i + 2], x[2], t[i])));
}

// Mahalanobis quadratic form d^T Sigma^-1 d with icov = (c00 c11 c22 2c01 2c02 2c12).
static inline float quad_icov(const float* ic, float d0, float d1, float d2) {
  float t0 = std::fma(ic[3], d1, ic[4] * d2);
  t0 = std::fma(ic[0], d0, t0);
  const float t1 = std::fma(ic[1], d1, ic[5] * d2);
  const float t2 = ic[2] * d2;
  return std::fma(d0, t0, std::fma(d1, t1, d2 * t2));
}
static inline float quad_eucl(float d0, float d1, float d2) { return std::fma(d0, d0, std::fma(d1, d1, d2 * d2)); }

// Eq. 5: E = sum_i min_modes ||Sigma^-1/2 (H x_i - mu)||, evaluated as
// sqrt(min d^T Sigma^-1 d); samples without modes contribute 0; f32 sums: sequential within
// each eta-sample batch, then batch totals added in batch order (DESIGN.md numerics contract).
float energy(const FrameCtx& c, const AdaptState& s, const Pose& H, const std::vector<int>& samples, int eta) {
  float R[9], t[3];
  pose_to_f32(H, R, t);
  float E = 0.0f, Eb = 0.0f;
  for (size_t i = 0; i < samples.size(); ++i) {
    if (i > 0 && i % static_cast<size_t>(eta) == 0) {  // batch boundary
      E = E + Eb;
      Eb = 0.0f;
    }
    const int g = samples[i];
    const int nm = c.nmodes[g];
    if (nm == 0) continue;
    float y[3];
    xform_f32(R, t, &c.camf[3 * static_cast<size_t>(g)], y);
    float qmin = std::numeric_limits<float>::infinity();
    for (int m = 0; m < nm; ++m) {
      const Mode* md = ctx_mode(c, s, g, m);
      const float q = quad_icov(md->icov, y[0] - md->mu[0], y[1] - md->mu[1], y[2] - md->mu[2]);
      qmin = std::fmin(qmin, q);
    }
    Eb = Eb + std::sqrt(std::fmax(qmin, 0.0f));
  }
  return E + Eb;
}

namespace {
constexpr int kAcc = 28;  // 21 (upper JtJ) + 6 (Jt r) + 1 (sum r^2)

struct LmSample {
  const Mode* m;
  double x[3];
};

}  // namespace

// Residual r = S (H x - mu) and its Jacobian J = dr/d(delta) for H <- exp(delta) H (left
// perturbation, twist = (omega, rho)); S = Sigma^-1/2 or I. Returns y = H x.
void lm_residual_jacobian(const Pose& H, const double x[3], const Mode& m, bool use_cov, double r[3],
                          double J[3][6], double y[3]) {
  transform_point(H, x, y);
  const double d[3] = {y[0] - m.mu[0], y[1] - m.mu[1], y[2] - m.mu[2]};
  double S[9];
  if (use_cov) {
    const float* q = m.isqrt;
    S[0] = q[0]; S[1] = q[1]; S[2] = q[2];
    S[3] = q[1]; S[4] = q[3]; S[5] = q[4];
    S[6] = q[2]; S[7] = q[4]; S[8] = q[5];
  } else {
    for (int i = 0; i < 9; ++i) S[i] = (i % 4 == 0) ? 1.0 : 0.0;
  }
  for (int i = 0; i < 3; ++i) r[i] = (S[3 * i + 0] * d[0] + S[3 * i + 1] * d[1]) + S[3 * i + 2] * d[2];
  if (!J) return;
  for (int i = 0; i < 3; ++i) {
    J[i][0] = S[3 * i + 1] * (-y[2]) + S[3 * i + 2] * y[1];
    J[i][1] = S[3 * i + 0] * y[2] + S[3 * i + 2] * (-y[0]);
    J[i][2] = S[3 * i + 0] * (-y[1]) + S[3 * i + 1] * y[0];
    J[i][3] = S[3 * i + 0];
    J[i][4] = S[3 * i + 1];
    J[i][5] = S[3 * i + 2];
  }
}

namespace {
// One sample's contribution to the normal equations (or only to sum r^2).
inline void lm_term(const Pose& H, const LmSample& s, bool use_cov, double acc[kAcc], bool with_jac) {
  double y[3], r[3], J[3][6];
  lm_residual_jacobian(H, s.x, *s.m, use_cov, r, with_jac ? J : nullptr, y);
  acc[27] = acc[27] + ((r[0] * r[0] + r[1] * r[1]) + r[2] * r[2]);
  if (!with_jac) return;
  int k = 0;
  for (int a = 0; a < 6; ++a)
    for (int b = a; b < 6; ++b, ++k) acc[k] = acc[k] + ((J[0][a] * J[0][b] + J[1][a] * J[1][b]) + J[2][a] * J[2][b]);
  for (int a = 0; a < 6; ++a) acc[21 + a] = acc[21 + a] + ((J[0][a] * r[0] + J[1][a] * r[1]) + J[2][a] * r[2]);
}

// Canonical 128-lane order: lane l accumulates samples l, l+128, ... in order, then an xor
// butterfly combines lanes, first inside each 32-lane warp (16, 8, 4, 2, 1), then across the
// four warps (32, 64): the total is (W0 + W1) + (W2 + W3).
void lm_accumulate(const Pose& H, const std::vector<LmSample>& smp, bool use_cov, bool with_jac, double out[kAcc]) {
  thread_local double L[kLmLanes][kAcc], nxt[kLmLanes][kAcc];
  for (auto& l : L)
    for (double& v : l) v = 0.0;
  for (size_t i = 0; i < smp.size(); ++i)
    if (smp[i].m) lm_term(H, smp[i], use_cov, L[i % kLmLanes], with_jac);
  static const int kOffsets[7] = {16, 8, 4, 2, 1, 32, 64};
  for (int off : kOffsets) {
    for (int l = 0; l < kLmLanes; ++l)
      for (int a = 0; a < kAcc; ++a) nxt[l][a] = L[l][a] + L[l ^ off][a];
    for (int l = 0; l < kLmLanes; ++l)
      for (int a = 0; a < kAcc; ++a) L[l][a] = nxt[l][a];
  }
  for (int a = 0; a < kAcc; ++a) out[a] = L[0][a];
}
}  // namespace

// lm_refine: nearest mode frozen per step (re-associated after an
// accepted step), H <- exp(delta) H, (A + lambda diag A) delta = -b, lambda0 = 1e-3,
// x10 on reject / x0.1 on accept, <= 10 iterations, stop on relative decrease < 1e-6.
void lm_refine(const FrameCtx& c, const AdaptState& s, Pose& H, const std::vector<int>& samples, bool use_cov,
               double* final_surrogate) {
  std::vector<LmSample> smp(samples.size());
  double lambda = 1e-3;
  bool need_assoc = true;
  double lastE = 0.0;
  for (int it = 0; it < 10; ++it) {
    if (need_assoc) {
      float R[9], t[3];
      pose_to_f32(H, R, t);
      for (size_t i = 0; i < samples.size(); ++i) {
        const int g = samples[i];
        smp[i].m = nullptr;
        for (int q = 0; q < 3; ++q) smp[i].x[q] = static_cast<double>(c.camf[3 * static_cast<size_t>(g) + q]);
        const int nm = c.nmodes[g];
        if (nm == 0) continue;
        float y[3];
        xform_f32(R, t, &c.camf[3 * static_cast<size_t>(g)], y);
        float best = std::numeric_limits<float>::infinity();
        for (int m = 0; m < nm; ++m) {
          const Mode* md = ctx_mode(c, s, g, m);
          const float d0 = y[0] - md->mu[0], d1 = y[1] - md->mu[1], d2 = y[2] - md->mu[2];
          const float q = use_cov ? quad_icov(md->icov, d0, d1, d2) : quad_eucl(d0, d1, d2);
          if (smp[i].m == nullptr || q < best) {  // first minimum wins ties
            best = q;
            smp[i].m = md;
          }
        }
      }
      need_assoc = false;
    }
    double acc[kAcc];
    lm_accumulate(H, smp, use_cov, true, acc);
    const double E = acc[27];
    lastE = E;
    if (!(E > 0.0)) break;
    double M[36], rhs[6], delta[6];
    int k = 0;
    for (int a = 0; a < 6; ++a)
      for (int b = a; b < 6; ++b, ++k) {
        M[6 * a + b] = acc[k];
        M[6 * b + a] = acc[k];
      }
    for (int a = 0; a < 6; ++a) {
      M[6 * a + a] = M[6 * a + a] + lambda * M[6 * a + a];
      rhs[a] = -acc[21 + a];
    }
    if (!chol6_solve(M, rhs, delta)) {
      lambda = lambda * 10.0;
      continue;
    }
    const Pose Hn = compose(exp_se3(delta), H);
    double accn[kAcc];
    lm_accumulate(Hn, smp, use_cov, false, accn);
    const double En = accn[27];
    if (En < E) {
      H = Hn;
      lambda = lambda * 0.1;
      need_assoc = true;
      lastE = En;
      if ((E - En) / E < 1e-6) break;
    } else {
      lambda = lambda * 10.0;
    }
  }
  if (final_surrogate) *final_surrogate = lastE;
}

static bool hyp_less(const Hypothesis& a, const Hypothesis& b) {
  const float ea = std::isnan(a.energy) ? std::numeric_limits<float>::infinity() : a.energy;
  const float eb = std::isnan(b.energy) ? std::numeric_limits<float>::infinity() : b.energy;
  if (ea != eb) return ea < eb;
  return a.slot < b.slot;
}

// preemptive_ransac: N_max slots (Rng::stream(seed, slot)), cull to
// N_cull on sample batch 0, then {add batch k, LM (if pose_update), rescore, keep
// ceil(n/2)} until n <= n_out. Batch k is drawn from Rng::stream(seed, N_max + k).
std::vector<Hypothesis> preemptive_ransac(const FrameCtx& c, const AdaptState& s, const RansacParams& p,
                                          uint64_t seed, std::vector<Hypothesis>* generated) {
  const int G = static_cast<int>(c.grid.size());
  if (G == 0) throw Error(E_NO_HYPOTHESES, "preemptive_ransac: no valid grid pixels");
  std::vector<Hypothesis> hyps;
  for (int slot = 0; slot < p.n_max; ++slot) {
    Rng rng = Rng::stream(seed, static_cast<uint64_t>(slot));
    Hypothesis h;
    int attempts = 0;
    if (generate_hypothesis(c, s, p, rng, &h.pose, &attempts) == REJ_OK) {
      h.slot = slot;
      h.iterations = attempts;
      hyps.push_back(h);
    }
  }
  if (generated) *generated = hyps;
  if (hyps.empty()) throw Error(E_NO_HYPOTHESES, "preemptive_ransac: every generation slot failed");
  std::vector<int> I;
  draw_samples(seed, 0, p.n_max, p.eta, G, I);
  for (auto& h : hyps) h.energy = energy(c, s, h.pose, I, p.eta);
  std::sort(hyps.begin(), hyps.end(), hyp_less);
  if (static_cast<int>(hyps.size()) > p.n_cull) hyps.resize(p.n_cull);
  int k = 1;
  while (static_cast<int>(hyps.size()) > p.n_out) {
    draw_samples(seed, k, p.n_max, p.eta, G, I);
    for (auto& h : hyps) {
      if (p.pose_update) lm_refine(c, s, h.pose, I, p.use_cov != 0);
      h.energy = energy(c, s, h.pose, I, p.eta);
    }
    std::sort(hyps.begin(), hyps.end(), hyp_less);
    hyps.resize((hyps.size() + 1) / 2);
    ++k;
  }
  return hyps;
}

}  // namespace oracle

// ORACLE — test infrastructure only. Never linked into the product.
//
// adaptation restatement (src/adaptation.cpp is missing from
// the reference): per-leaf Algorithm-R reservoirs with counter-based draws
// (A2/A3), Really Quick Shift clustering (A5, A6), round-robin
// refresh and mode prediction.
#include <algorithm>
#include <cmath>
#include <numeric>

#include "detmath.hpp"
#include "oracle.hpp"

namespace oracle {

void init_state(AdaptState& s, const Forest& f, const ForestParams& p, uint64_t seed) {
  s.params = p;
  s.seed = seed;
  s.total_leaves = f.total_leaves;
  s.cursor = 0;
  s.entries.assign(static_cast<size_t>(s.total_leaves) * p.capacity, Entry{0, 0, 0, 0, 0, 0, 0});
  s.seen.assign(s.total_leaves, 0);
  s.pred_count.assign(s.total_leaves, 0);
  s.modes.assign(static_cast<size_t>(s.total_leaves) * kMaxModes, Mode{});
}

// SPEC.md:384-391
void clear_adaptation(AdaptState& s) {
  std::fill(s.entries.begin(), s.entries.end(), Entry{0, 0, 0, 0, 0, 0, 0});
  std::fill(s.seen.begin(), s.seen.end(), 0u);
  std::fill(s.pred_count.begin(), s.pred_count.end(), 0);
  std::fill(s.modes.begin(), s.modes.end(), Mode{});
  s.cursor = 0;
}

// Algorithm R (A3): n = seen before the insert;
// n < kappa -> slot n; else j = uniform_int(n + 1) from
// Rng::stream(adapt_seed, slot << 32 | n), replace iff j < kappa.
void reservoir_insert(AdaptState& s, int64_t slot, const Entry& e) {
  const uint32_t n = s.seen[slot];
  const int kappa = s.params.capacity;
  if (n < static_cast<uint32_t>(kappa)) {
    s.entries[static_cast<size_t>(slot) * kappa + n] = e;
  } else {
    Rng rng = Rng::stream(s.seed, (static_cast<uint64_t>(slot) << 32) | n);
    const uint64_t j = rng.uniform_int(static_cast<uint64_t>(n) + 1);
    if (j < static_cast<uint64_t>(kappa)) s.entries[static_cast<size_t>(slot) * kappa + j] = e;
  }
  s.seen[slot] = n + 1;
}

// grid pixels in row-major order, x_W = pose * backproject (double,
// rounded to f32 for storage), inserted into the reached leaf of every tree in tree order.
void integrate_frame(AdaptState& s, const Forest& f, const Frame& fr, const Pose& pose) {
  if (!fr.pose_reliable) throw Error(E_UNRELIABLE_POSE, "integrate_frame: pose flagged unreliable");
  const std::vector<int> grid = sample_grid_pixels(fr, 4);
  for (int g : grid) {
    const int x = g & 0xffff, y = g >> 16;
    const size_t idx = static_cast<size_t>(y) * fr.width + x;
    double pc[3], pw[3];
    backproject(x, y, static_cast<double>(fr.depth[idx]), fr.k, pc);
    transform_point(pose, pc, pw);
    const Entry e{static_cast<float>(pw[0]), static_cast<float>(pw[1]), static_cast<float>(pw[2]),
                  fr.rgb[3 * idx], fr.rgb[3 * idx + 1], fr.rgb[3 * idx + 2], 0};
    for (size_t t = 0; t < f.trees.size(); ++t) {
      const int32_t leaf = find_leaf(f.trees[t], fr, x, y, f.specs);
      reservoir_insert(s, f.leaf_base[t] + leaf, e);
    }
  }
}

static inline float dist2f(const Entry& a, const Entry& b) {
  const float dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z;
  return std::fma(dz, dz, std::fma(dy, dy, dx * dx));
}

// Really Quick Shift (A5/A6).
std::vector<Mode> cluster_reservoir(const Entry* e, int n, const ForestParams& p, std::vector<int>* labels_out) {
  std::vector<Mode> out;
  if (labels_out) labels_out->assign(n, -1);
  if (n <= 0) return out;
  const float c = static_cast<float>(-1.0 / (2.0 * static_cast<double>(p.sigma) * static_cast<double>(p.sigma)));
  const float tau2 = static_cast<float>(static_cast<double>(p.tau) * static_cast<double>(p.tau));
  std::vector<double> rho(n);
  for (int i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int j = 0; j < n; ++j) acc = acc + static_cast<double>(det_expf(dist2f(e[i], e[j]) * c));
    rho[i] = acc;
  }
  std::vector<int> parent(n, -1);
  for (int i = 0; i < n; ++i) {
    float best = std::numeric_limits<float>::infinity();
    int bj = -1;
    for (int j = 0; j < n; ++j) {
      if (j == i) continue;
      const bool higher = rho[j] > rho[i] || (rho[j] == rho[i] && j < i);
      if (!higher) continue;
      const float d2 = dist2f(e[i], e[j]);
      if (d2 <= tau2 && d2 < best) {
        best = d2;
        bj = j;
      }
    }
    parent[i] = bj;
  }
  std::vector<int> root(n);
  for (int i = 0; i < n; ++i) {
    int r = i;
    while (parent[r] >= 0) r = parent[r];
    root[i] = r;
  }
  std::vector<int> size(n, 0);
  for (int i = 0; i < n; ++i) size[root[i]]++;
  std::vector<int> roots;
  for (int i = 0; i < n; ++i)
    if (parent[i] < 0 && size[i] >= p.min_cluster_size) roots.push_back(i);
  std::stable_sort(roots.begin(), roots.end(), [&](int a, int b) { return size[a] > size[b]; });
  if (static_cast<int>(roots.size()) > p.max_clusters) roots.resize(p.max_clusters);
  std::vector<int> label(n, -1);
  for (size_t k = 0; k < roots.size(); ++k)
    for (int i = 0; i < n; ++i)
      if (root[i] == roots[k]) label[i] = static_cast<int>(k);
  if (labels_out) *labels_out = label;
  for (size_t k = 0; k < roots.size(); ++k) {
    double sx = 0, sy = 0, sz = 0, sr = 0, sg = 0, sb = 0;
    int cnt = 0;
    for (int i = 0; i < n; ++i) {
      if (label[i] != static_cast<int>(k)) continue;
      sx = sx + e[i].x; sy = sy + e[i].y; sz = sz + e[i].z;
      sr = sr + e[i].r; sg = sg + e[i].g; sb = sb + e[i].b;
      ++cnt;
    }
    const double dn = static_cast<double>(cnt);
    const double mx = sx / dn, my = sy / dn, mz = sz / dn;
    double c00 = 0, c01 = 0, c02 = 0, c11 = 0, c12 = 0, c22 = 0;
    for (int i = 0; i < n; ++i) {
      if (label[i] != static_cast<int>(k)) continue;
      const double dx = e[i].x - mx, dy = e[i].y - my, dz = e[i].z - mz;
      c00 = c00 + dx * dx; c01 = c01 + dx * dy; c02 = c02 + dx * dz;
      c11 = c11 + dy * dy; c12 = c12 + dy * dz; c22 = c22 + dz * dz;
    }
    c00 = c00 / dn + 1e-6; c01 = c01 / dn; c02 = c02 / dn;
    c11 = c11 / dn + 1e-6; c12 = c12 / dn; c22 = c22 / dn + 1e-6;
    const double S[9] = {c00, c01, c02, c01, c11, c12, c02, c12, c22};
    double lam[3], V[9];
    eig3_jacobi(S, lam, V);
    double il[3], isl[3];
    for (int q = 0; q < 3; ++q) {
      const double l = lam[q] > 1e-12 ? lam[q] : 1e-12;
      il[q] = 1.0 / l;
      isl[q] = 1.0 / std::sqrt(l);
    }
    auto fn = [&](const double w[3], int a, int b) {
      return (V[3 * a + 0] * w[0] * V[3 * b + 0] + V[3 * a + 1] * w[1] * V[3 * b + 1]) + V[3 * a + 2] * w[2] * V[3 * b + 2];
    };
    Mode m;
    m.mu[0] = static_cast<float>(mx); m.mu[1] = static_cast<float>(my); m.mu[2] = static_cast<float>(mz);
    m.colour[0] = static_cast<float>(sr / dn); m.colour[1] = static_cast<float>(sg / dn); m.colour[2] = static_cast<float>(sb / dn);
    m.cov[0] = static_cast<float>(c00); m.cov[1] = static_cast<float>(c01); m.cov[2] = static_cast<float>(c02);
    m.cov[3] = static_cast<float>(c11); m.cov[4] = static_cast<float>(c12); m.cov[5] = static_cast<float>(c22);
    m.icov[0] = static_cast<float>(fn(il, 0, 0));
    m.icov[1] = static_cast<float>(fn(il, 1, 1));
    m.icov[2] = static_cast<float>(fn(il, 2, 2));
    m.icov[3] = static_cast<float>(2.0 * fn(il, 0, 1));
    m.icov[4] = static_cast<float>(2.0 * fn(il, 0, 2));
    m.icov[5] = static_cast<float>(2.0 * fn(il, 1, 2));
    m.isqrt[0] = static_cast<float>(fn(isl, 0, 0));
    m.isqrt[1] = static_cast<float>(fn(isl, 0, 1));
    m.isqrt[2] = static_cast<float>(fn(isl, 0, 2));
    m.isqrt[3] = static_cast<float>(fn(isl, 1, 1));
    m.isqrt[4] = static_cast<float>(fn(isl, 1, 2));
    m.isqrt[5] = static_cast<float>(fn(isl, 2, 2));
    m.size = cnt;
    out.push_back(m);
  }
  return out;
}

// the next `leaves_per_call` slots after the cursor, cursor mod leaves.
void update_leaves_round_robin(AdaptState& s, int64_t leaves_per_call) {
  const int64_t L = s.total_leaves;
  if (L == 0) return;
  const int64_t n = std::min(leaves_per_call, L);
  const int kappa = s.params.capacity;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t slot = (s.cursor + i) % L;
    const int cnt = static_cast<int>(std::min<uint32_t>(s.seen[slot], static_cast<uint32_t>(kappa)));
    const std::vector<Mode> m = cluster_reservoir(&s.entries[static_cast<size_t>(slot) * kappa], cnt, s.params);
    s.pred_count[slot] = static_cast<int32_t>(m.size());
    for (size_t k = 0; k < m.size(); ++k) s.modes[static_cast<size_t>(slot) * kMaxModes + k] = m[k];
  }
  s.cursor = (s.cursor + n) % L;
}

}  // namespace oracle

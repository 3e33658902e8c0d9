// ORACLE — test infrastructure only. Never linked into the product.
//
// geometry: restates proj/include/screloc/geometry.hpp:73-222
// features: restates proj/src/features.cpp:7-75 (bit-exact)
// forest:   restates proj/include/screloc/forest.hpp:19-112 (layout, routing,
//           random generation per SPEC.md:262-270, serialization per SPEC.md:280-300)
#include <algorithm>
#include <cmath>
#include <cstring>

#include "detmath.hpp"
#include "oracle.hpp"

namespace oracle {

// ---------------------------------------------------------------- geometry ---
// compose / invert: geometry.hpp:144-153
Pose compose(const Pose& a, const Pose& b) {
  Pose r;
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j)
      r.R[3 * i + j] = (a.R[3 * i + 0] * b.R[0 + j] + a.R[3 * i + 1] * b.R[3 + j]) + a.R[3 * i + 2] * b.R[6 + j];
    r.t[i] = ((a.R[3 * i + 0] * b.t[0] + a.R[3 * i + 1] * b.t[1]) + a.R[3 * i + 2] * b.t[2]) + a.t[i];
  }
  return r;
}

Pose invert(const Pose& a) {
  Pose r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.R[3 * i + j] = a.R[3 * j + i];
  for (int i = 0; i < 3; ++i)
    r.t[i] = -(((r.R[3 * i + 0] * a.t[0] + r.R[3 * i + 1] * a.t[1]) + r.R[3 * i + 2] * a.t[2]));
  return r;
}

void transform_point(const Pose& T, const double p[3], double out[3]) {
  for (int i = 0; i < 3; ++i)
    out[i] = ((T.R[3 * i + 0] * p[0] + T.R[3 * i + 1] * p[1]) + T.R[3 * i + 2] * p[2]) + T.t[i];
}

static void mat3_mul(const double A[9], const double B[9], double C[9]) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      C[3 * i + j] = (A[3 * i + 0] * B[0 + j] + A[3 * i + 1] * B[3 + j]) + A[3 * i + 2] * B[6 + j];
}

static void skew(const double v[3], double S[9]) {
  S[0] = 0; S[1] = -v[2]; S[2] = v[1];
  S[3] = v[2]; S[4] = 0; S[5] = -v[0];
  S[6] = -v[1]; S[7] = v[0]; S[8] = 0;
}

// exp_se3: geometry.hpp:83-105 (Rodrigues; series below 1e-8), twist = (omega, rho)
Pose exp_se3(const double tw[6]) {
  const double* w = tw;
  const double* rho = tw + 3;
  const double theta = std::sqrt((w[0] * w[0] + w[1] * w[1]) + w[2] * w[2]);
  double hat[9], hat2[9];
  skew(w, hat);
  mat3_mul(hat, hat, hat2);
  double rot[9], v[9];
  if (theta < 1e-8) {
    for (int i = 0; i < 9; ++i) {
      const double id = (i % 4 == 0) ? 1.0 : 0.0;
      rot[i] = (id + hat[i]) + hat2[i] / 2.0;
      v[i] = (id + hat[i] / 2.0) + hat2[i] / 6.0;
    }
  } else {
    double s, c;
    det_sincos(theta, &s, &c);
    const double t2 = theta * theta;
    const double a = s / theta;
    const double b = (1.0 - c) / t2;
    const double cc = (theta - s) / (t2 * theta);
    for (int i = 0; i < 9; ++i) {
      const double id = (i % 4 == 0) ? 1.0 : 0.0;
      rot[i] = (id + a * hat[i]) + b * hat2[i];
      v[i] = (id + b * hat[i]) + cc * hat2[i];
    }
  }
  Pose T;
  for (int i = 0; i < 9; ++i) T.R[i] = rot[i];
  for (int i = 0; i < 3; ++i) T.t[i] = (v[3 * i + 0] * rho[0] + v[3 * i + 1] * rho[1]) + v[3 * i + 2] * rho[2];
  return T;
}

// log_se3: geometry.hpp:107-142 (test-only; uses libm acos/sin/tan like the reference)
void log_se3(const Pose& T, double tw[6]) {
  const double* R = T.R;
  const double tr = (R[0] + R[4]) + R[8];
  const double cos_theta = std::min(1.0, std::max(-1.0, (tr - 1.0) / 2.0));
  const double theta = std::acos(cos_theta);
  if (theta >= M_PI - 1e-6) throw Error(E_ANGLE_NEAR_PI, "log_se3: rotation angle within 1e-6 of pi");
  double w[3], hat[9], hat2[9], vinv[9];
  if (theta < 1e-8) {
    w[0] = (R[7] - R[5]) / 2.0;
    w[1] = (R[2] - R[6]) / 2.0;
    w[2] = (R[3] - R[1]) / 2.0;
    skew(w, hat);
    mat3_mul(hat, hat, hat2);
    for (int i = 0; i < 9; ++i) vinv[i] = (((i % 4 == 0) ? 1.0 : 0.0) - hat[i] / 2.0) + hat2[i] / 12.0;
  } else {
    const double f = theta / (2.0 * std::sin(theta));
    w[0] = f * (R[7] - R[5]);
    w[1] = f * (R[2] - R[6]);
    w[2] = f * (R[3] - R[1]);
    skew(w, hat);
    mat3_mul(hat, hat, hat2);
    const double t2 = theta * theta;
    const double coeff = (1.0 - theta / (2.0 * std::tan(theta / 2.0))) / t2;
    for (int i = 0; i < 9; ++i) vinv[i] = (((i % 4 == 0) ? 1.0 : 0.0) - hat[i] / 2.0) + coeff * hat2[i];
  }
  for (int i = 0; i < 3; ++i) tw[i] = w[i];
  for (int i = 0; i < 3; ++i)
    tw[3 + i] = (vinv[3 * i + 0] * T.t[0] + vinv[3 * i + 1] * T.t[1]) + vinv[3 * i + 2] * T.t[2];
}

// kabsch: geometry.hpp:155-191 (SVD with reflection fix; degenerate iff
// !(sv0 > 0) || sv1 < 1e-12 sv0 — the second singular value, per the code comment
// at geometry.hpp:182-184).
bool kabsch(const double* cam, const double* world, int n, Pose* out) {
  if (n < 3) return false;
  double cc[3] = {0, 0, 0}, wc[3] = {0, 0, 0};
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k) {
      cc[k] = cc[k] + cam[3 * i + k];
      wc[k] = wc[k] + world[3 * i + k];
    }
  for (int k = 0; k < 3; ++k) {
    cc[k] = cc[k] / static_cast<double>(n);
    wc[k] = wc[k] / static_cast<double>(n);
  }
  double C[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = 0; i < n; ++i) {
    double dw[3], dc[3];
    for (int k = 0; k < 3; ++k) {
      dw[k] = world[3 * i + k] - wc[k];
      dc[k] = cam[3 * i + k] - cc[k];
    }
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) C[3 * r + c] = C[3 * r + c] + dw[r] * dc[c];
  }
  double U[9], S[3], V[9];
  svd3_jacobi(C, U, S, V);
  if (!(S[0] > 0.0) || S[1] < 1e-12 * S[0]) return false;
  double M[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      M[3 * i + j] = (U[3 * i + 0] * V[3 * j + 0] + U[3 * i + 1] * V[3 * j + 1]) + U[3 * i + 2] * V[3 * j + 2];
  const double det = (M[0] * (M[4] * M[8] - M[5] * M[7]) - M[1] * (M[3] * M[8] - M[5] * M[6])) +
                     M[2] * (M[3] * M[7] - M[4] * M[6]);
  const double d2 = det < 0.0 ? -1.0 : 1.0;
  Pose T;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      T.R[3 * i + j] = (U[3 * i + 0] * V[3 * j + 0] + U[3 * i + 1] * V[3 * j + 1]) + (U[3 * i + 2] * d2) * V[3 * j + 2];
  for (int i = 0; i < 3; ++i)
    T.t[i] = wc[i] - ((T.R[3 * i + 0] * cc[0] + T.R[3 * i + 1] * cc[1]) + T.R[3 * i + 2] * cc[2]);
  *out = T;
  return true;
}

// backproject: geometry.hpp:194-199
void backproject(int x, int y, double depth, const Intrinsics& k, double out[3]) {
  if (!(depth > 0) || !std::isfinite(depth)) throw Error(E_INVALID_DEPTH, "backproject: non-positive or non-finite depth");
  out[0] = (x - k.cx) * depth / k.fx;
  out[1] = (y - k.cy) * depth / k.fy;
  out[2] = depth;
}

// pose_error: geometry.hpp:206-216
void pose_error(const Pose& e, const Pose& g, double* terr, double* aerr) {
  const double dx = e.t[0] - g.t[0], dy = e.t[1] - g.t[1], dz = e.t[2] - g.t[2];
  *terr = std::sqrt((dx * dx + dy * dy) + dz * dz);
  double M[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      M[3 * i + j] = (g.R[0 + i] * e.R[0 + j] + g.R[3 + i] * e.R[3 + j]) + g.R[6 + i] * e.R[6 + j];
  const double c = std::min(1.0, std::max(-1.0, (((M[0] + M[4]) + M[8]) - 1.0) / 2.0));
  *aerr = std::acos(c) * 180.0 / M_PI;
}

// ---------------------------------------------------------------- features ---
// features.cpp:7-19
std::vector<FeatureSpec> generate_feature_specs(uint64_t seed, int radius) {
  Rng rng(seed);
  const long long r = radius;
  std::vector<FeatureSpec> specs(kFeatureCount);
  for (int i = 0; i < kFeatureCount; ++i) {
    FeatureSpec& s = specs[i];
    s.kind = i < kDepthFeatureCount ? 0 : 1;
    s.dx = static_cast<int>(rng.uniform_int_range(-r, r));
    s.dy = static_cast<int>(rng.uniform_int_range(-r, r));
    s.channel = static_cast<int>(rng.uniform_int(3));
  }
  return specs;
}

static inline bool in_bounds(const Frame& f, int x, int y) { return x >= 0 && x < f.width && y >= 0 && y < f.height; }

// features.cpp:33-58
float compute_feature(const Frame& f, int x, int y, const FeatureSpec& s) {
  if (!in_bounds(f, x, y) || !depth_valid(f.depth[static_cast<size_t>(y) * f.width + x]))
    throw Error(E_INVALID_CENTRE_PIXEL, "compute_feature: invalid depth at centre pixel");
  const float cd = f.depth[static_cast<size_t>(y) * f.width + x];
  const int px = x + static_cast<int>(std::lround(s.dx / cd));
  const int py = y + static_cast<int>(std::lround(s.dy / cd));
  if (s.kind == 0) {
    float pd = 0.0f;
    if (in_bounds(f, px, py)) {
      const float d = f.depth[static_cast<size_t>(py) * f.width + px];
      if (depth_valid(d)) pd = d;
    }
    return cd - pd;
  }
  const float cv = f.rgb[(static_cast<size_t>(y) * f.width + x) * 3 + s.channel];
  float pv = 0.0f;
  if (in_bounds(f, px, py) && depth_valid(f.depth[static_cast<size_t>(py) * f.width + px]))
    pv = f.rgb[(static_cast<size_t>(py) * f.width + px) * 3 + s.channel];
  return cv - pv;
}

// features.cpp:67-75 (grid origin (0,0), row-major)
std::vector<int> sample_grid_pixels(const Frame& f, int spacing) {
  std::vector<int> px;
  for (int y = 0; y < f.height; y += spacing)
    for (int x = 0; x < f.width; x += spacing)
      if (depth_valid(f.depth[static_cast<size_t>(y) * f.width + x])) px.push_back(x | (y << 16));
  return px;
}

// ------------------------------------------------------------------ forest ---
void Forest::finalize() {
  leaf_base.assign(trees.size(), 0);
  int64_t b = 0;
  for (size_t t = 0; t < trees.size(); ++t) {
    leaf_base[t] = b;
    b += trees[t].leaf_count;
  }
  total_leaves = b;
}

// SPEC.md:262-270 + DESIGN.md A2: specs from Rng(seed); tree t from Rng::stream(seed, t);
// BFS over branch nodes: bernoulli(p) picks Depth, then uniform_int(128) picks phi; tau = 0.
Forest generate_random_forest(uint64_t seed, int height, double p_depth, int ntrees, int radius) {
  Forest f;
  f.specs = generate_feature_specs(seed, radius);
  const int32_t branches = (1 << height) - 1;
  const int32_t nodes = (1 << (height + 1)) - 1;
  for (int t = 0; t < ntrees; ++t) {
    Rng rng = Rng::stream(seed, static_cast<uint64_t>(t));
    Tree tr;
    tr.nodes.resize(nodes);
    for (int32_t i = 0; i < nodes; ++i) {
      TreeNode& n = tr.nodes[i];
      if (i < branches) {
        const bool depth = rng.bernoulli(p_depth);
        n.feature = (depth ? 0 : kDepthFeatureCount) + static_cast<int32_t>(rng.uniform_int(kDepthFeatureCount));
        n.threshold = 0.0f;
        n.left = 2 * i + 1;
        n.right = 2 * i + 2;
        n.leaf_id = -1;
      } else {
        n.left = n.right = -1;
        n.leaf_id = i - branches;
      }
    }
    tr.leaf_count = nodes - branches;
    f.trees.push_back(std::move(tr));
  }
  f.finalize();
  return f;
}

// forest.hpp:40-42 lazy descent; route right iff f[phi] >= tau (forest.hpp:21)
int32_t find_leaf(const Tree& t, const Frame& f, int x, int y, const std::vector<FeatureSpec>& specs) {
  int32_t i = 0;
  for (;;) {
    const TreeNode& n = t.nodes[i];
    if (n.left < 0) return n.leaf_id;
    const float v = compute_feature(f, x, y, specs[n.feature]);
    i = v >= n.threshold ? n.right : n.left;
  }
}

// Serialization: little-endian; magic "SCRF", u32 version=1,
// u32 tree_count, u32 spec_count, specs {u8 kind, u8 channel, i16 dx, i16 dy},
// per tree {u32 node_count, i32 leaf_count, nodes {i32 feature, f32 threshold,
// i32 left, i32 right, i32 leaf_id}}.
namespace {
template <typename T>
void put(std::vector<uint8_t>& b, T v) {
  uint8_t raw[sizeof(T)];
  std::memcpy(raw, &v, sizeof(T));
  b.insert(b.end(), raw, raw + sizeof(T));
}
struct Reader {
  const uint8_t* d;
  size_t n, off = 0;
  template <typename T>
  T get() {
    if (off + sizeof(T) > n)
      throw Error(E_MALFORMED_DATA, "deserialize_forest: truncated at offset " + std::to_string(off));
    T v;
    std::memcpy(&v, d + off, sizeof(T));
    off += sizeof(T);
    return v;
  }
};
}  // namespace

std::vector<uint8_t> serialize_forest(const Forest& f) {
  std::vector<uint8_t> b;
  b.push_back('S'); b.push_back('C'); b.push_back('R'); b.push_back('F');
  put<uint32_t>(b, 1);
  put<uint32_t>(b, static_cast<uint32_t>(f.trees.size()));
  put<uint32_t>(b, static_cast<uint32_t>(f.specs.size()));
  for (const auto& s : f.specs) {
    put<uint8_t>(b, static_cast<uint8_t>(s.kind));
    put<uint8_t>(b, static_cast<uint8_t>(s.channel));
    put<int16_t>(b, static_cast<int16_t>(s.dx));
    put<int16_t>(b, static_cast<int16_t>(s.dy));
  }
  for (const auto& t : f.trees) {
    put<uint32_t>(b, static_cast<uint32_t>(t.nodes.size()));
    put<int32_t>(b, t.leaf_count);
    for (const auto& n : t.nodes) {
      put<int32_t>(b, n.feature);
      put<float>(b, n.threshold);
      put<int32_t>(b, n.left);
      put<int32_t>(b, n.right);
      put<int32_t>(b, n.leaf_id);
    }
  }
  return b;
}

Forest deserialize_forest(const uint8_t* data, size_t n) {
  Reader r{data, n};
  const char m0 = r.get<char>(), m1 = r.get<char>(), m2 = r.get<char>(), m3 = r.get<char>();
  if (m0 != 'S' || m1 != 'C' || m2 != 'R' || m3 != 'F') throw Error(E_MALFORMED_DATA, "deserialize_forest: bad magic");
  const uint32_t version = r.get<uint32_t>();
  if (version != 1) throw Error(E_MALFORMED_DATA, "deserialize_forest: unsupported version " + std::to_string(version));
  const uint32_t nt = r.get<uint32_t>(), ns = r.get<uint32_t>();
  if (ns != kFeatureCount) throw Error(E_MALFORMED_DATA, "deserialize_forest: spec count " + std::to_string(ns));
  Forest f;
  f.specs.resize(ns);
  for (auto& s : f.specs) {
    s.kind = r.get<uint8_t>();
    s.channel = r.get<uint8_t>();
    s.dx = r.get<int16_t>();
    s.dy = r.get<int16_t>();
    if (s.kind > 1 || s.channel > 2) throw Error(E_MALFORMED_DATA, "deserialize_forest: bad spec at offset " + std::to_string(r.off));
  }
  for (uint32_t t = 0; t < nt; ++t) {
    Tree tr;
    const uint32_t nn = r.get<uint32_t>();
    tr.leaf_count = r.get<int32_t>();
    if (nn == 0 || nn > (1u << 26)) throw Error(E_MALFORMED_DATA, "deserialize_forest: bad node count");
    tr.nodes.resize(nn);
    for (auto& nd : tr.nodes) {
      nd.feature = r.get<int32_t>();
      nd.threshold = r.get<float>();
      nd.left = r.get<int32_t>();
      nd.right = r.get<int32_t>();
      nd.leaf_id = r.get<int32_t>();
    }
    for (uint32_t i = 0; i < nn; ++i) {  // structural validation
      const auto& nd = tr.nodes[i];
      if (nd.left < 0) {
        if (nd.leaf_id < 0 || nd.leaf_id >= tr.leaf_count) throw Error(E_MALFORMED_DATA, "deserialize_forest: bad leaf id");
      } else if (nd.left <= static_cast<int32_t>(i) || nd.right <= static_cast<int32_t>(i) ||
                 nd.left >= static_cast<int32_t>(nn) || nd.right >= static_cast<int32_t>(nn) || nd.feature < 0 ||
                 nd.feature >= kFeatureCount) {
        throw Error(E_MALFORMED_DATA, "deserialize_forest: bad branch node " + std::to_string(i));
      }
    }
    f.trees.push_back(std::move(tr));
  }
  if (r.off != n) throw Error(E_MALFORMED_DATA, "deserialize_forest: trailing bytes at offset " + std::to_string(r.off));
  f.finalize();
  return f;
}

}  // namespace oracle

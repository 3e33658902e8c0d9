// ORACLE — test infrastructure only. extern "C" entry points into the REFERENCE's own
// code (compiled from /root/reference/proj by oracle/ref/build_ref.sh against the local
// Eigen shim): rng.hpp, features.cpp, geometry.hpp. Used only to generate the golden
// vectors under tests/golden/ that pin the oracle restatement.
#include <cstdint>
#include <cstring>
#include <vector>

#include "screloc/features.hpp"
#include "screloc/geometry.hpp"
#include "screloc/rng.hpp"

using namespace screloc;

extern "C" {

void ref_rng_u64(uint64_t seed, int use_stream, uint64_t tag, int n, uint64_t* out) {
  Rng r = use_stream ? Rng::stream(seed, tag) : Rng(seed);
  for (int i = 0; i < n; ++i) out[i] = r.next_u64();
}
void ref_rng_uniform_int(uint64_t seed, int use_stream, uint64_t tag, uint64_t bound, int n, uint64_t* out) {
  Rng r = use_stream ? Rng::stream(seed, tag) : Rng(seed);
  for (int i = 0; i < n; ++i) out[i] = r.uniform_int(bound);
}
void ref_rng_uniform(uint64_t seed, int use_stream, uint64_t tag, int n, double* out) {
  Rng r = use_stream ? Rng::stream(seed, tag) : Rng(seed);
  for (int i = 0; i < n; ++i) out[i] = r.uniform();
}
void ref_rng_bernoulli(uint64_t seed, double p, int n, int32_t* out) {
  Rng r(seed);
  for (int i = 0; i < n; ++i) out[i] = r.bernoulli(p) ? 1 : 0;
}
void ref_feature_specs(uint64_t seed, int radius, int32_t* out) {
  const auto s = generate_feature_specs(seed, radius);
  for (int i = 0; i < kFeatureCount; ++i) {
    out[4 * i] = static_cast<int>(s[i].kind);
    out[4 * i + 1] = s[i].offset.x();
    out[4 * i + 2] = s[i].offset.y();
    out[4 * i + 3] = static_cast<int>(s[i].channel);
  }
}

static RgbdFrame make_frame(const float* depth, const uint8_t* rgb, int w, int h) {
  RgbdFrame f;
  f.depth = DepthImage(w, h);
  f.colour = ColourImage(w, h);
  std::memcpy(f.depth.data(), depth, sizeof(float) * w * h);
  for (int i = 0; i < w * h; ++i) f.colour.data()[i] = Rgb8{rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]};
  return f;
}

// Feature vectors (all 256 specs) at n pixels; status 3 (InvalidCentrePixel) per pixel.
void ref_feature_vectors(const float* depth, const uint8_t* rgb, int w, int h, uint64_t seed, int radius,
                         const int32_t* px, int n, float* out, int32_t* status) {
  const RgbdFrame f = make_frame(depth, rgb, w, h);
  const auto specs = generate_feature_specs(seed, radius);
  for (int i = 0; i < n; ++i) {
    status[i] = 0;
    try {
      const FeatureVector v = compute_feature_vector(f, Vec2i(px[i] & 0xffff, px[i] >> 16), specs);
      for (int k = 0; k < kFeatureCount; ++k) out[static_cast<size_t>(i) * kFeatureCount + k] = v[k];
    } catch (const InvalidCentrePixel&) {
      status[i] = 3;
    }
  }
}
int ref_grid(const float* depth, int w, int h, int spacing, int32_t* out, int cap) {
  RgbdFrame f;
  f.depth = DepthImage(w, h);
  std::memcpy(f.depth.data(), depth, sizeof(float) * w * h);
  const auto g = sample_grid_pixels(f, spacing);
  const int n = static_cast<int>(g.size());
  for (int i = 0; i < n && i < cap; ++i) out[i] = g[i].x() | (g[i].y() << 16);
  return n;
}

static void put_pose(const RigidTransform& T, double* R, double* t) {
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) R[3 * i + j] = T.rotation(i, j);
    t[i] = T.translation(i);
  }
}
static RigidTransform get_pose(const double* R, const double* t) {
  RigidTransform T;
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) T.rotation(i, j) = R[3 * i + j];
    T.translation(i) = t[i];
  }
  return T;
}
void ref_exp_se3(const double* tw, double* R, double* t) {
  TwistVector v;
  for (int i = 0; i < 6; ++i) v(i) = tw[i];
  put_pose(exp_se3<double>(v), R, t);
}
int ref_log_se3(const double* R, const double* t, double* tw) {
  try {
    const TwistVector v = log_se3<double>(get_pose(R, t));
    for (int i = 0; i < 6; ++i) tw[i] = v(i);
    return 0;
  } catch (const AngleNearPi&) {
    return 11;
  }
}
int ref_kabsch(const double* cam, const double* world, int n, double* R, double* t) {
  std::vector<Vec3> c(n), w(n);
  for (int i = 0; i < n; ++i) {
    c[i] = Vec3(cam[3 * i], cam[3 * i + 1], cam[3 * i + 2]);
    w[i] = Vec3(world[3 * i], world[3 * i + 1], world[3 * i + 2]);
  }
  const auto T = kabsch<double>(c, w);
  if (!T) return 0;
  put_pose(*T, R, t);
  return 1;
}
int ref_backproject(int x, int y, double d, double fx, double fy, double cx, double cy, double* out) {
  PinholeIntrinsics k;
  k.fx = fx; k.fy = fy; k.cx = cx; k.cy = cy; k.width = 1 << 20; k.height = 1 << 20;
  try {
    const Vec3 p = backproject(Vec2i(x, y), d, k);
    out[0] = p(0); out[1] = p(1); out[2] = p(2);
    return 0;
  } catch (const InvalidDepth&) {
    return 2;
  }
}
void ref_pose_error(const double* Re, const double* te, const double* Rg, const double* tg, double* terr, double* aerr) {
  const PoseError e = pose_error(get_pose(Re, te), get_pose(Rg, tg));
  *terr = e.translation_error;
  *aerr = e.angular_error;
}

}  // extern "C"

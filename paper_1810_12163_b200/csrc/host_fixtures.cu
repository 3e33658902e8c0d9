// Host-side generators the reference API exposes next to the hot path:
//   generate_feature_specs   proj/src/features.cpp:7-19
//   generate_random_forest   proj/include/screloc/forest.hpp:104-106
//   serialize_forest         proj/include/screloc/forest.hpp:108 (format SPEC.md:300)
//   generate_synthetic_scene / generate_trajectory   SPEC.md:565-572 (benchmark fixture)
// They run once per scene, on the host, and produce the inputs the GPU consumes.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/screloc_gpu.h"

namespace {

class HostRng {  // xoshiro256** seeded by splitmix64 (proj/include/screloc/rng.hpp:14-88)
 public:
  explicit HostRng(uint64_t seed) {
    uint64_t x = seed;
    for (auto& v : s_) v = mix(x);
  }
  static HostRng stream(uint64_t seed, uint64_t tag) {
    uint64_t x = seed;
    const uint64_t a = mix(x);
    x ^= tag * 0x9e3779b97f4a7c15ull + 0x243f6a8885a308d3ull;
    const uint64_t b = mix(x);
    return HostRng(a ^ (b + 0x632be59bd9b4e019ull));
  }
  uint64_t next() {
    const uint64_t r = rotl(s_[1] * 5, 7) * 9;
    const uint64_t t = s_[1] << 17;
    s_[2] ^= s_[0];
    s_[3] ^= s_[1];
    s_[1] ^= s_[2];
    s_[0] ^= s_[3];
    s_[2] ^= t;
    s_[3] = rotl(s_[3], 45);
    return r;
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  uint64_t below(uint64_t n) {
    const uint64_t thr = (0 - n) % n;
    for (;;) {
      const uint64_t r = next();
      if (r >= thr) return r % n;
    }
  }
  long long range(long long lo, long long hi) { return lo + static_cast<long long>(below(static_cast<uint64_t>(hi - lo + 1))); }
  bool bernoulli(double p) { return uniform() < p; }

 private:
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  static uint64_t mix(uint64_t& x) {
    x += 0x9e3779b97f4a7c15ull;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  uint64_t s_[4];
};

void sincos_det(double x, double* s, double* c) {  // same definition as the device det_sincos
  const double S1 = -1.66666666666666324348e-01, S2 = 8.33333333332248946124e-03,
               S3 = -1.98412698298579493134e-04, S4 = 2.75573137070700676789e-06,
               S5 = -2.50507602534068634195e-08, S6 = 1.58969099521155010221e-10;
  const double C1 = 4.16666666666666019037e-02, C2 = -1.38888888888741095749e-03,
               C3 = 2.48015872894767294178e-05, C4 = -2.75573143513906633035e-07,
               C5 = 2.08757232129817482790e-09, C6 = -1.13596475577881948265e-11;
  const double n = std::nearbyint(x * 6.36619772367581382433e-01);
  const double r = (x - n * 1.57079632673412561417e+00) - n * 6.07710050650619224932e-11;
  const double z = r * r;
  const double v = z * r;
  const double ks = r + v * (S1 + z * (S2 + z * (S3 + z * (S4 + z * (S5 + z * S6)))));
  const double rc = z * (C1 + z * (C2 + z * (C3 + z * (C4 + z * (C5 + z * C6)))));
  const double hz = 0.5 * z;
  const double w = 1.0 - hz;
  const double kc = w + (((1.0 - w) - hz) + z * rc);
  switch (static_cast<int>(static_cast<long long>(n) & 3)) {
    case 0: *s = ks; *c = kc; break;
    case 1: *s = kc; *c = -ks; break;
    case 2: *s = -ks; *c = -kc; break;
    default: *s = -kc; *c = ks; break;
  }
}

template <typename T>
void put(std::vector<uint8_t>& b, T v) {
  uint8_t raw[sizeof(T)];
  std::memcpy(raw, &v, sizeof(T));
  b.insert(b.end(), raw, raw + sizeof(T));
}

void hsv(double h, double s, double v, float out[3]) {
  const double hh = (h - std::floor(h)) * 6.0;
  const int i = static_cast<int>(hh);
  const double f = hh - i;
  const double p = v * (1 - s), q = v * (1 - s * f), t = v * (1 - s * (1 - f));
  double r, g, b;
  switch (i % 6) {
    case 0: r = v; g = t; b = p; break;
    case 1: r = q; g = v; b = p; break;
    case 2: r = p; g = v; b = t; break;
    case 3: r = p; g = q; b = v; break;
    case 4: r = t; g = p; b = v; break;
    default: r = v; g = p; b = q; break;
  }
  out[0] = static_cast<float>(r * 255.0);
  out[1] = static_cast<float>(g * 255.0);
  out[2] = static_cast<float>(b * 255.0);
}

}  // namespace

extern "C" {

// generate_random_forest(seed, {height, p, trees, radius}) serialised in the SPEC.md:300
// format. Feature specs come from Rng(seed) (features.cpp:7-19); tree t from
// Rng::stream(seed, t), breadth-first: bernoulli(p) picks a Depth feature, then
// uniform_int(128) its index; thresholds are 0 (§4.5).
size_t scr_generate_random_forest(uint64_t seed, int height, double p_depth, int trees, int radius, uint8_t* out,
                                  size_t cap) {
  if (height < 1 || height > 24 || trees < 1 || trees > 8) return 0;
  std::vector<uint8_t> b;
  b.push_back('S'); b.push_back('C'); b.push_back('R'); b.push_back('F');
  put<uint32_t>(b, 1);
  put<uint32_t>(b, static_cast<uint32_t>(trees));
  put<uint32_t>(b, 256);
  HostRng spec_rng(seed);
  for (int i = 0; i < 256; ++i) {
    const int dx = static_cast<int>(spec_rng.range(-radius, radius));
    const int dy = static_cast<int>(spec_rng.range(-radius, radius));
    const int ch = static_cast<int>(spec_rng.below(3));
    put<uint8_t>(b, i < 128 ? 0 : 1);
    put<uint8_t>(b, static_cast<uint8_t>(ch));
    put<int16_t>(b, static_cast<int16_t>(dx));
    put<int16_t>(b, static_cast<int16_t>(dy));
  }
  const int32_t branches = (1 << height) - 1, nodes = (1 << (height + 1)) - 1;
  for (int t = 0; t < trees; ++t) {
    HostRng rng = HostRng::stream(seed, static_cast<uint64_t>(t));
    put<uint32_t>(b, static_cast<uint32_t>(nodes));
    put<int32_t>(b, nodes - branches);
    for (int32_t i = 0; i < nodes; ++i) {
      if (i < branches) {
        const bool depth = rng.bernoulli(p_depth);
        put<int32_t>(b, (depth ? 0 : 128) + static_cast<int32_t>(rng.below(128)));
        put<float>(b, 0.0f);
        put<int32_t>(b, 2 * i + 1);
        put<int32_t>(b, 2 * i + 2);
        put<int32_t>(b, -1);
      } else {
        put<int32_t>(b, 0);
        put<float>(b, 0.0f);
        put<int32_t>(b, -1);
        put<int32_t>(b, -1);
        put<int32_t>(b, i - branches);
      }
    }
  }
  if (out && cap >= b.size()) std::memcpy(out, b.data(), b.size());
  return b.size();
}

// generate_synthetic_scene(seed, complexity) — the benchmark fixture (DESIGN.md
// "Synthetic fixture"): a closed 4 x 3 x 2.5 m room of six zero-thickness panels plus
// (complexity - 6) boxes / spheres spread over the four walls.
int scr_generate_synthetic_scene(uint64_t seed, int complexity, scr_prim* out, int cap) {
  HostRng rng(seed);
  const float X = 4.0f, Y = 3.0f, Z = 2.5f;
  const float walls[6][6] = {{0, 0, 0, X, Y, 0}, {0, 0, Z, X, Y, Z}, {0, 0, 0, 0, Y, Z},
                             {X, 0, 0, X, Y, Z}, {0, 0, 0, X, 0, Z}, {0, Y, 0, X, Y, Z}};
  const int n = complexity < 6 ? 6 : complexity;
  const double hue0 = rng.uniform();
  for (int i = 0; i < n; ++i) {
    scr_prim p;
    std::memset(&p, 0, sizeof(p));
    hsv(hue0 + 0.6180339887498949 * i, 0.45 + 0.45 * rng.uniform(), 0.55 + 0.4 * rng.uniform(), p.colour);
    p.cell = static_cast<float>(0.08 + 0.17 * rng.uniform());
    p.tex_seed = static_cast<uint32_t>(rng.next() >> 32);
    if (i < 6) {
      p.type = 0;
      for (int k = 0; k < 3; ++k) {
        p.a[k] = walls[i][k];
        p.b[k] = walls[i][3 + k];
      }
    } else {
      const int j = i - 6, nobj = n - 6;
      const double perim = 2.0 * (X + Y);
      const double sp = (j + 0.5 + 0.3 * (rng.uniform() - 0.5)) * perim / nobj;
      int wall;
      double centre;
      if (sp < X) { wall = 2; centre = sp; }
      else if (sp < X + Y) { wall = 1; centre = sp - X; }
      else if (sp < 2.0 * X + Y) { wall = 3; centre = X - (sp - X - Y); }
      else { wall = 0; centre = Y - (sp - 2.0 * X - Y); }
      const int along = wall < 2 ? 1 : 0, nrm = wall < 2 ? 0 : 1;
      const double len = wall < 2 ? Y : X;
      const double wpos = (wall == 0 || wall == 2) ? 0.0 : (wall == 1 ? X : Y);
      const bool low = (wall == 0 || wall == 2);
      if (rng.uniform() < 0.55) {
        const double w = 0.4 + 0.5 * rng.uniform();
        const double depth = 0.2 + 0.5 * rng.uniform();
        const double gap = 0.02 + 0.15 * rng.uniform();
        const bool floor_standing = rng.bernoulli(0.7);
        const double z0 = floor_standing ? 0.0 : 0.5 + 0.6 * rng.uniform();
        const double h = floor_standing ? 0.4 + 1.2 * rng.uniform() : 0.15 + 0.4 * rng.uniform();
        double mn[3], mx[3];
        const double dep = depth < 0.9 - gap ? depth : 0.9 - gap;
        if (low) { mn[nrm] = wpos + gap; mx[nrm] = mn[nrm] + dep; }
        else { mx[nrm] = wpos - gap; mn[nrm] = mx[nrm] - dep; }
        mn[along] = centre - w / 2 > 0.05 ? centre - w / 2 : 0.05;
        mx[along] = centre + w / 2 < len - 0.05 ? centre + w / 2 : len - 0.05;
        mn[2] = z0;
        mx[2] = z0 + h < static_cast<double>(Z) - 0.05 ? z0 + h : static_cast<double>(Z) - 0.05;
        p.type = 0;
        for (int k = 0; k < 3; ++k) {
          p.a[k] = static_cast<float>(mn[k]);
          p.b[k] = static_cast<float>(mx[k]);
        }
      } else {
        const double r = 0.2 + 0.2 * rng.uniform();
        const double gap = 0.05 + 0.25 * rng.uniform();
        const double z = r + 0.1 + (1.2 - r) * rng.uniform();
        double c[3];
        c[nrm] = low ? wpos + gap + r : wpos - gap - r;
        double ca = centre > r + 0.05 ? centre : r + 0.05;
        if (ca > len - r - 0.05) ca = len - r - 0.05;
        c[along] = ca;
        c[2] = z;
        p.type = 1;
        for (int k = 0; k < 3; ++k) p.a[k] = static_cast<float>(c[k]);
        p.b[0] = static_cast<float>(r);
      }
    }
    if (out && i < cap) out[i] = p;
  }
  return n;
}

// generate_trajectory(seed, n, kind): kind 0 = smooth adaptation loop around the room
// centre; kind 1 = held-out test poses (same loop half a step off, perturbed by up to
// +-6 cm / +-6 deg / +-3 deg roll); kind 2 = held-out novel-pose set:
// frame i targets novelty bin b = i mod 11 (offset 5b..5b+5 cm along a uniform random
// direction, 5b..5b+5 deg of yaw/pitch/roll along another), positions clamped to the
// free camera volume, so the set spans every bin up to 55 cm / 55 deg.
static void unit_dir(HostRng& r, double v[3]) {
  const double z = 2.0 * r.uniform() - 1.0, phi = 6.283185307179586 * r.uniform();
  double sp, cp;
  sincos_det(phi, &sp, &cp);
  const double rr = std::sqrt(std::max(0.0, 1.0 - z * z));
  v[0] = rr * cp;
  v[1] = rr * sp;
  v[2] = z;
}

void scr_generate_trajectory(uint64_t seed, int n, int kind, scr_pose* out) {
  HostRng rng(seed);
  const double twopi = 6.283185307179586;
  const double ph0 = twopi * rng.uniform(), ph1 = twopi * rng.uniform(), ph2 = twopi * rng.uniform(),
               ph3 = twopi * rng.uniform();
  HostRng pert = HostRng::stream(seed, 0x7e57ull);
  (void)ph1;
  for (int i = 0; i < n; ++i) {
    const double s = (i + (kind != 0 ? 0.5 : 0.0)) / static_cast<double>(n);
    double a, b, c, d, e, g;
    sincos_det(twopi * s + ph0, &a, &b);
    sincos_det(2 * twopi * s + ph1, &c, &d);
    sincos_det(3 * twopi * s + ph3, &e, &g);
    double px = 2.0 + 0.5 * b, py = 1.5 + 0.2 * a, pz = 1.4 + 0.15 * c;
    double yaw = ph2 + twopi * s, pitch = -0.35 + 0.12 * e, roll = 0.0;
    if (kind == 1) {
      px += 0.06 * (2 * pert.uniform() - 1);
      py += 0.06 * (2 * pert.uniform() - 1);
      pz += 0.06 * (2 * pert.uniform() - 1);
      const double deg = 0.017453292519943295;
      yaw += 6 * deg * (2 * pert.uniform() - 1);
      pitch += 6 * deg * (2 * pert.uniform() - 1);
      roll += 3 * deg * (2 * pert.uniform() - 1);
    } else if (kind == 2) {
      const double deg = 0.017453292519943295;
      const int bn = i % 11;
      const double rt = 0.05 * (bn + pert.uniform()), ra = 5.0 * deg * (bn + pert.uniform());
      double v[3], q[3];
      unit_dir(pert, v);
      unit_dir(pert, q);
      px = std::min(2.8, std::max(1.2, px + rt * v[0]));
      py = std::min(1.95, std::max(1.05, py + rt * v[1]));
      pz = std::min(2.2, std::max(0.5, pz + rt * v[2]));
      yaw += ra * q[0];
      pitch += ra * q[1];
      roll += ra * q[2];
    }
    double sy, cy, sp, cp, sr, cr;
    sincos_det(yaw, &sy, &cy);
    sincos_det(pitch, &sp, &cp);
    sincos_det(roll, &sr, &cr);
    const double f[3] = {cp * cy, cp * sy, sp};
    const double x0[3] = {sy, -cy, 0.0};
    const double y0[3] = {sp * cy, sp * sy, -cp};
    scr_pose& P = out[i];
    for (int k = 0; k < 3; ++k) {
      P.R[3 * k + 0] = cr * x0[k] + sr * y0[k];
      P.R[3 * k + 1] = -sr * x0[k] + cr * y0[k];
      P.R[3 * k + 2] = f[k];
    }
    P.t[0] = px;
    P.t[1] = py;
    P.t[2] = pz;
  }
}

}  // extern "C"

// ORACLE — test infrastructure only. Never linked into the product.
//
// scene_model restatement: the procedural SyntheticScene,
// its exact analytic raycast (shared by render_frame and raycast_depth,
// SPEC.md:550, 578, 586) and seeded trajectories. The generator constants are
// builder choices frozen in DESIGN.md ("Synthetic fixture").
#include <algorithm>
#include <cmath>

#include "detmath.hpp"
#include "oracle.hpp"

namespace oracle {

namespace {
void hsv_to_rgb(double h, double s, double v, float out[3]) {
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

// Room [0,4]x[0,3]x[0,2.5] (z up) closed by 6 zero-thickness panels, plus
// (complexity - 6) boxes and spheres spread over the four walls, kept within 0.9 m of
// their wall so that the camera volume x in [1.3,2.7], y in [1.1,1.9] stays free.
Scene generate_synthetic_scene(uint64_t seed, int complexity) {
  Rng rng(seed);
  Scene sc;
  const float X = sc.room[0], Y = sc.room[1], Z = sc.room[2];
  const float walls[6][6] = {{0, 0, 0, X, Y, 0}, {0, 0, Z, X, Y, Z}, {0, 0, 0, 0, Y, Z},
                             {X, 0, 0, X, Y, Z}, {0, 0, 0, X, 0, Z}, {0, Y, 0, X, Y, Z}};
  const int n = std::max(complexity, 6);
  const double golden = 0.6180339887498949;
  const double hue0 = rng.uniform();
  for (int i = 0; i < n; ++i) {
    Prim p;
    hsv_to_rgb(hue0 + golden * i, 0.45 + 0.45 * rng.uniform(), 0.55 + 0.4 * rng.uniform(), p.colour);
    p.cell = static_cast<float>(0.08 + 0.17 * rng.uniform());
    p.tex_seed = static_cast<uint32_t>(rng.next_u64() >> 32);
    if (i < 6) {
      p.type = 0;
      for (int k = 0; k < 3; ++k) {
        p.a[k] = walls[i][k];
        p.b[k] = walls[i][3 + k];
      }
    } else {
      // objects evenly spaced by perimeter arc length (+ jitter) so every view direction
      // sees non-planar, asymmetric geometry (breaks the room's symmetries)
      const int j = i - 6, nobj = n - 6;
      const double perim = 2.0 * (X + Y);
      const double s = (j + 0.5 + 0.3 * (rng.uniform() - 0.5)) * perim / nobj;
      int wall;  // 0: x=0, 1: x=X, 2: y=0, 3: y=Y
      double centre;
      if (s < X) { wall = 2; centre = s; }
      else if (s < X + Y) { wall = 1; centre = s - X; }
      else if (s < 2.0 * X + Y) { wall = 3; centre = X - (s - X - Y); }
      else { wall = 0; centre = Y - (s - 2.0 * X - Y); }
      const int along_axis = wall < 2 ? 1 : 0;
      const int nrm = wall < 2 ? 0 : 1;
      const double along_len = wall < 2 ? Y : X;
      const double wall_pos = (wall == 0 || wall == 2) ? 0.0 : (wall == 1 ? X : Y);
      const bool lowside = (wall == 0 || wall == 2);
      if (rng.uniform() < 0.55) {  // box: floor-standing cabinet or wall shelf
        const double w = 0.4 + 0.5 * rng.uniform();
        const double depth = 0.2 + 0.5 * rng.uniform();
        const double gap = 0.02 + 0.15 * rng.uniform();
        const bool floor = rng.bernoulli(0.7);
        const double z0 = floor ? 0.0 : 0.5 + 0.6 * rng.uniform();
        const double h = floor ? 0.4 + 1.2 * rng.uniform() : 0.15 + 0.4 * rng.uniform();
        double mn[3], mx[3];
        if (lowside) { mn[nrm] = wall_pos + gap; mx[nrm] = mn[nrm] + std::min(depth, 0.9 - gap); }
        else { mx[nrm] = wall_pos - gap; mn[nrm] = mx[nrm] - std::min(depth, 0.9 - gap); }
        mn[along_axis] = std::max(0.05, centre - w / 2);
        mx[along_axis] = std::min(along_len - 0.05, centre + w / 2);
        mn[2] = z0;
        mx[2] = std::min(z0 + h, static_cast<double>(Z) - 0.05);
        p.type = 0;
        for (int k = 0; k < 3; ++k) { p.a[k] = static_cast<float>(mn[k]); p.b[k] = static_cast<float>(mx[k]); }
      } else {  // sphere
        const double r = 0.2 + 0.2 * rng.uniform();
        const double gap = 0.05 + 0.25 * rng.uniform();
        const double z = r + 0.1 + (1.2 - r) * rng.uniform();
        double c[3];
        c[nrm] = lowside ? wall_pos + gap + r : wall_pos - gap - r;
        c[along_axis] = std::min(std::max(centre, r + 0.05), along_len - r - 0.05);
        c[2] = z;
        p.type = 1;
        for (int k = 0; k < 3; ++k) p.a[k] = static_cast<float>(c[k]);
        p.b[0] = static_cast<float>(r);
      }
    }
    sc.prims.push_back(p);
  }
  return sc;
}

// Exact analytic ray cast of one pixel (f32; frozen operation order).
// Ray: o = t_cam, d = R (( x - cx)/fx, (y - cy)/fy, 1), so the hit parameter is the
// camera-space depth. Closest hit over primitives in order; ties keep the earlier one.
Hit raycast_pixel(const Scene& s, const float R[9], const float tf[3], const Intrinsics& k, int x, int y) {
  const float dcx = (static_cast<float>(x) - static_cast<float>(k.cx)) / static_cast<float>(k.fx);
  const float dcy = (static_cast<float>(y) - static_cast<float>(k.cy)) / static_cast<float>(k.fy);
  float d[3], o[3];
  for (int i = 0; i < 3; ++i) {
    d[i] = std::fma(R[3 * i + 0], dcx, std::fma(R[3 * i + 1], dcy, R[3 * i + 2]));
    o[i] = tf[i];
  }
  Hit h{std::numeric_limits<float>::infinity(), -1, -1};
  for (int p = 0; p < static_cast<int>(s.prims.size()); ++p) {
    const Prim& q = s.prims[p];
    if (q.type == 0) {
      float lo[3], hi[3];
      for (int a = 0; a < 3; ++a) {
        const float inv = 1.0f / d[a];
        const float t1 = (q.a[a] - o[a]) * inv;
        const float t2 = (q.b[a] - o[a]) * inv;
        lo[a] = std::fmin(t1, t2);
        hi[a] = std::fmax(t1, t2);
      }
      const float tn = std::fmax(std::fmax(lo[0], lo[1]), lo[2]);
      const float tx = std::fmin(std::fmin(hi[0], hi[1]), hi[2]);
      if (tn <= tx && tn > 1e-4f && tn < h.t) {
        const int axis = (tn == lo[0]) ? 0 : ((tn == lo[1]) ? 1 : 2);
        h.t = tn;
        h.prim = p;
        h.face = axis * 2 + (d[axis] > 0.0f ? 0 : 1);
      }
    } else {
      const float oc[3] = {o[0] - q.a[0], o[1] - q.a[1], o[2] - q.a[2]};
      const float aa = std::fma(d[0], d[0], std::fma(d[1], d[1], d[2] * d[2]));
      const float bb = std::fma(oc[0], d[0], std::fma(oc[1], d[1], oc[2] * d[2]));
      const float cc = std::fma(oc[0], oc[0], std::fma(oc[1], oc[1], oc[2] * oc[2])) - q.b[0] * q.b[0];
      const float disc = bb * bb - aa * cc;
      if (disc >= 0.0f) {
        const float t = (-bb - std::sqrt(disc)) / aa;
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

void hit_normal(const Scene& s, const Hit& h, const float p[3], float n[3]) {
  const Prim& q = s.prims[h.prim];
  if (h.face < 6) {
    n[0] = n[1] = n[2] = 0.0f;
    n[h.face >> 1] = (h.face & 1) ? 1.0f : -1.0f;  // facing the ray
  } else {
    const float inv = 1.0f / q.b[0];
    for (int i = 0; i < 3; ++i) n[i] = (p[i] - q.a[i]) * inv;
  }
}

static inline uint32_t hash3(int x, int y, uint32_t seed) {
  uint32_t h = static_cast<uint32_t>(x) * 73856093u ^ static_cast<uint32_t>(y) * 19349663u ^ seed;
  h ^= h >> 16;
  h *= 0x7feb352du;
  h ^= h >> 15;
  h *= 0x846ca68bu;
  h ^= h >> 16;
  return h;
}

// Triplanar cell texture: the two coordinates orthogonal to the dominant normal
// axis index a hashed brightness cell of the primitive's base colour.
static void shade(const Scene& s, const Hit& h, const float p[3], uint8_t out[3]) {
  const Prim& q = s.prims[h.prim];
  float n[3];
  hit_normal(s, h, p, n);
  const float ax = std::fabs(n[0]), ay = std::fabs(n[1]), az = std::fabs(n[2]);
  const int dom = (ax >= ay && ax >= az) ? 0 : (ay >= az ? 1 : 2);
  const int u = dom == 0 ? 1 : 0, v = dom == 2 ? 1 : 2;
  const float inv = 1.0f / q.cell;
  const int iu = static_cast<int>(std::floor(p[u] * inv));
  const int iv = static_cast<int>(std::floor(p[v] * inv));
  const uint32_t hh = hash3(iu, iv, q.tex_seed);
  const float f = 0.35f + 0.65f * (static_cast<float>(hh & 255u) / 255.0f);
  for (int c = 0; c < 3; ++c) {
    const float val = q.colour[c] * f + 0.5f;
    out[c] = static_cast<uint8_t>(std::min(255, std::max(0, static_cast<int>(val))));
  }
}

void render_frame(const Scene& s, const Pose& T, const Intrinsics& k, float* depth, uint8_t* rgb) {
  float R[9], tf[3];
  for (int i = 0; i < 9; ++i) R[i] = static_cast<float>(T.R[i]);
  for (int i = 0; i < 3; ++i) tf[i] = static_cast<float>(T.t[i]);
  for (int y = 0; y < k.height; ++y)
    for (int x = 0; x < k.width; ++x) {
      const size_t idx = static_cast<size_t>(y) * k.width + x;
      const Hit h = raycast_pixel(s, R, tf, k, x, y);
      if (h.prim < 0 || !(h.t <= kRenderMaxDepth)) {
        depth[idx] = 0.0f;
        rgb[3 * idx] = rgb[3 * idx + 1] = rgb[3 * idx + 2] = 0;
        continue;
      }
      depth[idx] = h.t;
      const float dcx = (static_cast<float>(x) - static_cast<float>(k.cx)) / static_cast<float>(k.fx);
      const float dcy = (static_cast<float>(y) - static_cast<float>(k.cy)) / static_cast<float>(k.fy);
      float p[3];
      for (int i = 0; i < 3; ++i) {
        const float di = std::fma(R[3 * i + 0], dcx, std::fma(R[3 * i + 1], dcy, R[3 * i + 2]));
        p[i] = std::fma(h.t, di, tf[i]);
      }
      shade(s, h, p, rgb + 3 * idx);
    }
}

// Uniform direction on the unit sphere from two draws (z = 2u - 1, azimuth 2 pi u').
static void unit_dir(Rng& r, double v[3]) {
  const double z = 2.0 * r.uniform() - 1.0, phi = 6.283185307179586 * r.uniform();
  double sp, cp;
  det_sincos(phi, &sp, &cp);
  const double rr = std::sqrt(std::max(0.0, 1.0 - z * z));
  v[0] = rr * cp;
  v[1] = rr * sp;
  v[2] = z;
}

static Pose look_pose(double px, double py, double pz, double yaw, double pitch, double roll) {
  double sy, cy, sp, cp, sr, cr;
  det_sincos(yaw, &sy, &cy);
  det_sincos(pitch, &sp, &cp);
  det_sincos(roll, &sr, &cr);
  const double f[3] = {cp * cy, cp * sy, sp};
  const double x0[3] = {sy, -cy, 0.0};
  const double y0[3] = {sp * cy, sp * sy, -cp};
  Pose T;
  for (int i = 0; i < 3; ++i) {
    const double xc = cr * x0[i] + sr * y0[i];
    const double yc = -sr * x0[i] + cr * y0[i];
    T.R[3 * i + 0] = xc;
    T.R[3 * i + 1] = yc;
    T.R[3 * i + 2] = f[i];
  }
  T.t[0] = px;
  T.t[1] = py;
  T.t[2] = pz;
  return T;
}

// Smooth loop around the room centre. kind 0 = adaptation
// sequence; kind 1 = held-out test poses: the same loop sampled half a step
// off, perturbed by up to +-6 cm / +-6 deg (seeded); kind 2 = the held-out
// novel-pose set: frame i targets novelty bin b = i mod 11, i.e. a
// translation offset of 5b..5b+5 cm in a uniformly random direction and a rotation offset
// of 5b..5b+5 deg (yaw/pitch/roll along a uniformly random direction), so the offsets span
// every bin up to 55 cm / 55 deg; positions are clamped to the room's free camera volume.
void generate_trajectory(uint64_t seed, int n, int kind, Pose* out) {
  Rng rng(seed);
  const double twopi = 6.283185307179586;
  const double ph0 = twopi * rng.uniform(), ph1 = twopi * rng.uniform(), ph2 = twopi * rng.uniform(),
               ph3 = twopi * rng.uniform();
  Rng pert = Rng::stream(seed, 0x7e57ull);
  for (int i = 0; i < n; ++i) {
    const double s = (i + (kind != 0 ? 0.5 : 0.0)) / static_cast<double>(n);
    double a, b, c, d;
    det_sincos(twopi * s + ph0, &a, &b);
    det_sincos(2 * twopi * s + ph1, &c, &d);
    double px = 2.0 + 0.5 * b, py = 1.5 + 0.2 * a, pz = 1.4 + 0.15 * c;
    double e, g;
    det_sincos(3 * twopi * s + ph3, &e, &g);
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
      const int b = i % 11;
      const double rt = 0.05 * (b + pert.uniform()), ra = 5.0 * deg * (b + pert.uniform());
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
    out[i] = look_pose(px, py, pz, yaw, pitch, roll);
  }
}

}  // namespace oracle

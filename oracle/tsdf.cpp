// ORACLE — test infrastructure only. Never linked into the product.
//
// TSDF scene model (scene_model module): dense
// voxel volume, projective fusion (fuse_frame) and ray casting with sign-change detection
// and linear refinement (raycast_depth), plus the surface normal the ICP needs. The
// reference delegates this to InfiniTAM and ships none of it; the operations below are the
// frozen definition both this oracle and the GPU library implement (A13):
//   voxel (i,j,k) centre  c = origin + (idx + 0.5) * voxel          (fma per axis)
//   fuse: p_c = R^T (c - t); pixel = round-half-up(f * p/z + c0); sdf = D - z;
//         skip if z <= 0, pixel outside, D invalid or sdf < -trunc; f = min(1, sdf/trunc);
//         tsdf = fma(tsdf, w, f) / (w + 1); w = min(w + 1, 128)
//   sample F(p): trilinear over the 8 voxels around g = (p - origin)/voxel - 0.5, unknown
//         if any corner is outside or has weight 0; lerp(a,b,t) = fma(t, b - a, a), x, y, z
//   march: t = 0.2 m; step trunc while unknown, max(F * trunc, voxel) while F > 0, voxel
//         otherwise; hit at the first known F <= 0 after a known F > 0:
//         t* = fma(t - t_prev, F_prev / (F_prev - F), t_prev); no hit beyond 6 m or 1024 steps
//   normal: central differences of F at +-voxel on each axis, normalised; packed in 32 bits
//         (octahedral, two int16 snorm, never 0xffffffff).
#include <algorithm>
#include <cmath>

#include "oracle.hpp"

namespace oracle {

Tsdf tsdf_create(const float origin[3], float voxel, int nx, int ny, int nz, float trunc) {
  Tsdf v;
  for (int i = 0; i < 3; ++i) v.origin[i] = origin[i];
  v.voxel = voxel;
  v.trunc = trunc;
  v.nx = nx;
  v.ny = ny;
  v.nz = nz;
  const size_t n = static_cast<size_t>(nx) * ny * nz;
  v.tsdf.assign(n, 1.0f);
  v.weight.assign(n, 0.0f);
  return v;
}

void tsdf_fuse(Tsdf& v, const float* depth, const Intrinsics& k, const Pose& T) {
  float R[9], tf[3];
  for (int i = 0; i < 9; ++i) R[i] = static_cast<float>(T.R[i]);
  for (int i = 0; i < 3; ++i) tf[i] = static_cast<float>(T.t[i]);
  const float fx = static_cast<float>(k.fx), fy = static_cast<float>(k.fy);
  const float cx = static_cast<float>(k.cx), cy = static_cast<float>(k.cy);
  for (int kz = 0; kz < v.nz; ++kz)
    for (int jy = 0; jy < v.ny; ++jy)
      for (int ix = 0; ix < v.nx; ++ix) {
        const size_t idx = (static_cast<size_t>(kz) * v.ny + jy) * v.nx + ix;
        const float c[3] = {std::fma(static_cast<float>(ix) + 0.5f, v.voxel, v.origin[0]),
                            std::fma(static_cast<float>(jy) + 0.5f, v.voxel, v.origin[1]),
                            std::fma(static_cast<float>(kz) + 0.5f, v.voxel, v.origin[2])};
        const float dx = c[0] - tf[0], dy = c[1] - tf[1], dz = c[2] - tf[2];
        float pc[3];
        for (int i = 0; i < 3; ++i) pc[i] = std::fma(R[0 + i], dx, std::fma(R[3 + i], dy, R[6 + i] * dz));
        if (!(pc[2] > 0.0f)) continue;
        const float u = std::fma(fx, pc[0] / pc[2], cx), w = std::fma(fy, pc[1] / pc[2], cy);
        const int ui = static_cast<int>(std::floor(u + 0.5f)), vi = static_cast<int>(std::floor(w + 0.5f));
        if (ui < 0 || vi < 0 || ui >= k.width || vi >= k.height) continue;
        const float d = depth[static_cast<size_t>(vi) * k.width + ui];
        if (!depth_valid(d)) continue;
        const float sdf = d - pc[2];
        if (sdf < -v.trunc) continue;
        const float f = std::fmin(1.0f, sdf / v.trunc);
        const float wt = v.weight[idx];
        v.tsdf[idx] = std::fma(v.tsdf[idx], wt, f) / (wt + 1.0f);
        v.weight[idx] = std::fmin(wt + 1.0f, 128.0f);
      }
}

static inline float lerp(float a, float b, float t) { return std::fma(t, b - a, a); }

bool tsdf_sample(const Tsdf& v, const float p[3], float* F) {
  int i0[3];
  float fr[3];
  for (int a = 0; a < 3; ++a) {
    const float g = (p[a] - v.origin[a]) / v.voxel - 0.5f;
    const float gf = std::floor(g);
    i0[a] = static_cast<int>(gf);
    fr[a] = g - gf;
  }
  if (i0[0] < 0 || i0[1] < 0 || i0[2] < 0 || i0[0] + 1 >= v.nx || i0[1] + 1 >= v.ny || i0[2] + 1 >= v.nz) return false;
  float c[8];
  for (int q = 0; q < 8; ++q) {
    const size_t idx = (static_cast<size_t>(i0[2] + (q >> 2)) * v.ny + (i0[1] + ((q >> 1) & 1))) * v.nx + (i0[0] + (q & 1));
    if (!(v.weight[idx] > 0.0f)) return false;
    c[q] = v.tsdf[idx];
  }
  const float c00 = lerp(c[0], c[1], fr[0]), c10 = lerp(c[2], c[3], fr[0]);
  const float c01 = lerp(c[4], c[5], fr[0]), c11 = lerp(c[6], c[7], fr[0]);
  *F = lerp(lerp(c00, c10, fr[1]), lerp(c01, c11, fr[1]), fr[2]);
  return true;
}

uint32_t pack_normal(const float n[3]) {
  const float s = std::fabs(n[0]) + std::fabs(n[1]) + std::fabs(n[2]);
  float u = n[0] / s, w = n[1] / s;
  if (n[2] < 0.0f) {
    const float uu = (1.0f - std::fabs(w)) * (u >= 0.0f ? 1.0f : -1.0f);
    const float ww = (1.0f - std::fabs(u)) * (w >= 0.0f ? 1.0f : -1.0f);
    u = uu;
    w = ww;
  }
  const int qu = std::max(-32767, std::min(32767, static_cast<int>(std::floor(u * 32767.0f + 0.5f))));
  const int qw = std::max(-32767, std::min(32767, static_cast<int>(std::floor(w * 32767.0f + 0.5f))));
  return (static_cast<uint32_t>(qu) & 0xffffu) | (static_cast<uint32_t>(qw) << 16);
}

void unpack_normal(uint32_t p, float n[3]) {
  const float u = static_cast<float>(static_cast<int16_t>(p & 0xffffu)) / 32767.0f;
  const float w = static_cast<float>(static_cast<int16_t>(p >> 16)) / 32767.0f;
  float x = u, y = w;
  const float z = 1.0f - std::fabs(u) - std::fabs(w);
  if (z < 0.0f) {
    x = (1.0f - std::fabs(w)) * (u >= 0.0f ? 1.0f : -1.0f);
    y = (1.0f - std::fabs(u)) * (w >= 0.0f ? 1.0f : -1.0f);
  }
  const float len = std::sqrt(std::fma(x, x, std::fma(y, y, z * z)));
  n[0] = x / len;
  n[1] = y / len;
  n[2] = z / len;
}

// One pixel: ray o = t_cam, d = R ((x - cx)/fx, (y - cy)/fy, 1) as for the analytic model,
// so t is the camera-space depth. Returns false on no hit; *nrm = 0xffffffff when the
// normal is unavailable (an unknown neighbour).
bool tsdf_raycast_pixel(const Tsdf& v, const float R[9], const float tf[3], const Intrinsics& k, int x, int y,
                        float* t_out, uint32_t* nrm) {
  const float dcx = (static_cast<float>(x) - static_cast<float>(k.cx)) / static_cast<float>(k.fx);
  const float dcy = (static_cast<float>(y) - static_cast<float>(k.cy)) / static_cast<float>(k.fy);
  float d[3];
  for (int i = 0; i < 3; ++i) d[i] = std::fma(R[3 * i + 0], dcx, std::fma(R[3 * i + 1], dcy, R[3 * i + 2]));
  float t = 0.2f, tp = 0.0f, Fp = 0.0f;
  bool prev = false;
  for (int it = 0; it < kTsdfMaxSteps && t <= kRenderMaxDepth; ++it) {
    const float p[3] = {std::fma(t, d[0], tf[0]), std::fma(t, d[1], tf[1]), std::fma(t, d[2], tf[2])};
    float F;
    if (tsdf_sample(v, p, &F)) {
      if (prev && Fp > 0.0f && F <= 0.0f) {
        const float ts = std::fma(t - tp, Fp / (Fp - F), tp);
        if (!(ts <= kRenderMaxDepth)) return false;
        *t_out = ts;
        const float q[3] = {std::fma(ts, d[0], tf[0]), std::fma(ts, d[1], tf[1]), std::fma(ts, d[2], tf[2])};
        float g[3];
        *nrm = 0xffffffffu;
        for (int a = 0; a < 3; ++a) {
          float qp[3] = {q[0], q[1], q[2]}, qm[3] = {q[0], q[1], q[2]};
          qp[a] = q[a] + v.voxel;
          qm[a] = q[a] - v.voxel;
          float fp, fm;
          if (!tsdf_sample(v, qp, &fp) || !tsdf_sample(v, qm, &fm)) return true;
          g[a] = fp - fm;
        }
        const float len = std::sqrt(std::fma(g[0], g[0], std::fma(g[1], g[1], g[2] * g[2])));
        if (!(len > 0.0f)) return true;
        const float n[3] = {g[0] / len, g[1] / len, g[2] / len};
        *nrm = pack_normal(n);
        return true;
      }
      prev = true;
      Fp = F;
      tp = t;
      t = t + (F > 0.0f ? std::fmax(F * v.trunc, v.voxel) : v.voxel);
    } else {
      prev = false;
      t = t + v.trunc;
    }
  }
  return false;
}

}  // namespace oracle

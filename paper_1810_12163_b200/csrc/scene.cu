// Scene lifetime, frame ingest (K0), forest traversal (K1), online adaptation
// (K2 reservoir insertion, K3 Really Quick Shift) and the synthetic-scene renderer.
//
// Reference behaviour restated here (file:line into /root/reference):
//   frame validity            proj/include/screloc/core.hpp:109-114
//   compute_feature           proj/src/features.cpp:33-58
//   sample_grid_pixels        proj/src/features.cpp:67-75
//   Tree::find_leaf (lazy)    proj/include/screloc/forest.hpp:40-42, routing forest.hpp:21
//   leaf_slot (tree-major)    proj/include/screloc/forest.hpp:74-79
//   integrate_frame           SPEC.md:348-356 (source missing in the reference)
//   reservoir_insert
//   cluster_reservoir (RQS)
//   update_leaves_round_robin SPEC.md:366-374
//   clear_adaptation
#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "internal.cuh"

namespace scr {

namespace {
thread_local std::string g_err;
}
void set_error(const std::string& m) { g_err = m; }

cudaEvent_t prof_event(scr_scene s) {
  if (s->prof.pool.empty()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  cudaEvent_t e = s->prof.pool.back();
  s->prof.pool.pop_back();
  return e;
}

// Folds the completed launch events into per-kernel totals (call after a stream sync).
void prof_flush(scr_scene s) {
  for (auto& r : s->prof.pending) {
    float ms = 0.0f;
    if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) s->prof.ms[r.kid] += ms;
    s->prof.pool.push_back(r.a);
    s->prof.pool.push_back(r.b);
  }
  s->prof.pending.clear();
}

const char* const kKernelNames[K_COUNT] = {"k_pack", "k_grid", "k_leaves", "k_hypgen", "k_draw_samples", "k_energy",
                                           "k_select", "k_lm", "k_icp_score", "k_finalize", "k_insert", "k_rqs",
                                           "k_render", "k_compact", "k_hypfin"};
scr_status cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string("CUDA error ") + cudaGetErrorString(e) + " at " + what;
  return e == cudaErrorMemoryAllocation ? SCR_E_OOM : SCR_E_CUDA;
}

// =============================== K0: frame ingest ====================================
// Packs f32 depth + RGB8 into an 8-byte texel {depth or 0, r | g<<8 | b<<16 | valid<<24}.
// Invalid pixels carry zero depth and zero colour, which is exactly what a probe
// landing on them contributes (features.cpp:43-56), so K1 needs one load per probe.
// Also writes the live depth planes of the ICP pyramid (levels 0-2, subsampled at (x f, y f)
// like the association reads them), dense f32 with 0 for invalid depth.
__global__ void k_pack(const float* __restrict__ depth_base, const uint8_t* __restrict__ rgb_base,
                       const int* __restrict__ idx, int W, int H, uint2* __restrict__ tex,
                       float* __restrict__ dplane) {
  const int WH = W * H;
  const int f = blockIdx.y;
  const size_t src = idx ? static_cast<size_t>(idx[f]) : static_cast<size_t>(f);
  const float* dp = depth_base + src * WH;
  const uint8_t* cp = rgb_base + src * WH * 3;
  uint2* out = tex + static_cast<size_t>(f) * WH;
  float* dl0 = dplane + static_cast<size_t>(f) * (WH + WH / 4 + WH / 16);
  float* dl1 = dl0 + WH;
  float* dl2 = dl1 + WH / 4;
  const int W1 = W / 2, W2 = W / 4;
  const int stride = gridDim.x * blockDim.x;
  if ((W & 3) == 0 && (H & 3) == 0) {  // 4 pixels per thread: 16-B depth, 12-B colour, 32-B texel stores
    const float4* d4 = reinterpret_cast<const float4*>(dp);
    const uint3* c3 = reinterpret_cast<const uint3*>(cp);
    uint4* o4 = reinterpret_cast<uint4*>(out);
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < (WH >> 2); q += stride) {
      const float4 d = d4[q];
      const uint3 c = c3[q];  // bytes r0 g0 b0 r1 | g1 b1 r2 g2 | b2 r3 g3 b3
      const uint32_t rgb0 = c.x & 0xffffffu;
      const uint32_t rgb1 = (c.x >> 24) | ((c.y & 0xffffu) << 8);
      const uint32_t rgb2 = (c.y >> 16) | ((c.z & 0xffu) << 16);
      const uint32_t rgb3 = c.z >> 8;
      const bool v0 = depth_valid(d.x), v1 = depth_valid(d.y), v2 = depth_valid(d.z), v3 = depth_valid(d.w);
      o4[2 * q] = make_uint4(v0 ? __float_as_uint(d.x) : 0u, v0 ? (rgb0 | (1u << 24)) : 0u,
                             v1 ? __float_as_uint(d.y) : 0u, v1 ? (rgb1 | (1u << 24)) : 0u);
      o4[2 * q + 1] = make_uint4(v2 ? __float_as_uint(d.z) : 0u, v2 ? (rgb2 | (1u << 24)) : 0u,
                                 v3 ? __float_as_uint(d.w) : 0u, v3 ? (rgb3 | (1u << 24)) : 0u);
      const float4 lv = make_float4(v0 ? d.x : 0.0f, v1 ? d.y : 0.0f, v2 ? d.z : 0.0f, v3 ? d.w : 0.0f);
      reinterpret_cast<float4*>(dl0)[q] = lv;
      const int p0 = 4 * q, y = p0 / W, x = p0 - y * W;  // x % 4 == 0
      if ((y & 1) == 0) reinterpret_cast<float2*>(dl1)[((y >> 1) * W1 + (x >> 1)) >> 1] = make_float2(lv.x, lv.z);
      if ((y & 3) == 0) dl2[(y >> 2) * W2 + (x >> 2)] = lv.x;
    }
    return;
  }
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < WH; p += stride) {
    const float d = dp[p];
    uint2 t = make_uint2(0u, 0u);
    if (depth_valid(d)) {
      t.x = __float_as_uint(d);
      t.y = static_cast<uint32_t>(cp[3 * p]) | (static_cast<uint32_t>(cp[3 * p + 1]) << 8) |
            (static_cast<uint32_t>(cp[3 * p + 2]) << 16) | (1u << 24);
    }
    out[p] = t;
    const float lv = __uint_as_float(t.x);
    dl0[p] = lv;
    const int y = p / W, x = p - y * W;
    if ((x & 1) == 0 && (y & 1) == 0 && (x >> 1) < W1 && (y >> 1) < H / 2) dl1[(y >> 1) * W1 + (x >> 1)] = lv;
    if ((x & 3) == 0 && (y & 3) == 0 && (x >> 2) < W2 && (y >> 2) < H / 4) dl2[(y >> 2) * W2 + (x >> 2)] = lv;
  }
}

// Order-preserving compaction of the valid 4-px grid (features.cpp:67-75), one CTA per frame.
__global__ void __launch_bounds__(1024) k_grid(const uint2* __restrict__ tex, int W, int H, int gmax,
                                               int* __restrict__ gcount, int* __restrict__ gpx) {
  __shared__ int warp_tot[32];
  __shared__ int base_s;
  const int f = blockIdx.x;
  const uint2* t = tex + static_cast<size_t>(f) * W * H;
  const int gw = (W + 3) / 4, gh = (H + 3) / 4, total = gw * gh;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) base_s = 0;
  __syncthreads();
  for (int chunk = 0; chunk < total; chunk += 1024) {
    const int i = chunk + threadIdx.x;
    int x = 0, y = 0;
    bool v = false;
    if (i < total) {
      x = (i % gw) * 4;
      y = (i / gw) * 4;
      v = (t[static_cast<size_t>(y) * W + x].y >> 24) != 0u;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, v);
    const int pre = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) warp_tot[wid] = __popc(bal);
    __syncthreads();
    if (wid == 0) {
      int s = warp_tot[lane];
      for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, s, off);
        if (lane >= off) s += o;
      }
      warp_tot[lane] = s;  // inclusive
    }
    __syncthreads();
    const int wbase = wid ? warp_tot[wid - 1] : 0;
    const int base = base_s;
    if (v) gpx[static_cast<size_t>(f) * gmax + base + wbase + pre] = x | (y << 16);
    __syncthreads();
    if (threadIdx.x == 0) base_s = base + warp_tot[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) gcount[f] = base_s;
}

// =============================== K1: feature + forest traversal ========================
// One thread per valid grid pixel. Per tree: lazy descent evaluating only the visited
// features (forest.hpp:40-42): probe p + lround(delta / D(p)) (features.cpp:38-40), one
// 8-byte texel gather per visited node, route right iff f >= tau (forest.hpp:21).
// Also emits the f32 camera point (f64 backprojection, geometry.hpp:194-199) and the
// number of predicted modes (union over trees).
__global__ void __launch_bounds__(128) k_leaves(ForestView fv, FrameGeom g, const uint2* __restrict__ tex,
                                                const int* __restrict__ gcount, const int* __restrict__ gpx,
                                                int gmax, int* __restrict__ gslot, int* __restrict__ gnm,
                                                float4* __restrict__ gcam, int4* __restrict__ grec,
                                                const int* __restrict__ pcount, unsigned long long* __restrict__ work) {
  __shared__ short4 sspec[kFeatures];
  for (int i = threadIdx.x; i < kFeatures; i += blockDim.x) sspec[i] = fv.specs[i];
  __syncthreads();
  const int f = blockIdx.y;
  const int gi = blockIdx.x * blockDim.x + threadIdx.x;
  if (gi >= gcount[f]) return;
  const size_t gidx = static_cast<size_t>(f) * gmax + gi;
  const int px = gpx[gidx];
  const int x = px & 0xffff, y = px >> 16;
  const int W = g.W, H = g.H;
  const uint2* T = tex + static_cast<size_t>(f) * W * H;
  const uint2 c = T[y * W + x];
  const float d = __uint_as_float(c.x);
  int nm = 0, visits = 0;
  uint32_t counts = 0;
  uint32_t lw[4] = {0u, 0u, 0u, 0u};  // 16-bit leaf ids of trees 0..7
  for (int t = 0; t < fv.T; ++t) {
    const int nb = fv.node_base[t];
    int node = nb;
    int leaf;
    for (;;) {
      const int4 nd = __ldg(&fv.nodes[node]);
      if (nd.x < 0) {
        leaf = nd.y;
        break;
      }
      ++visits;
      const short4 sp = sspec[nd.z];
      const int qx = x + lround_small(__fdiv_rn(static_cast<float>(sp.x), d));
      const int qy = y + lround_small(__fdiv_rn(static_cast<float>(sp.y), d));
      uint2 pt = make_uint2(0u, 0u);
      if (qx >= 0 && qx < W && qy >= 0 && qy < H) pt = T[qy * W + qx];
      float v;
      if (sp.z == 0) {
        v = __fsub_rn(d, __uint_as_float(pt.x));
      } else {
        const int sh = 8 * sp.w;
        v = __fsub_rn(static_cast<float>((c.y >> sh) & 255u), static_cast<float>((pt.y >> sh) & 255u));
      }
      node = nb + ((v >= __int_as_float(nd.w)) ? nd.y : nd.x);
    }
    const int slot = fv.leaf_base[t] + leaf;
    gslot[gidx * fv.T + t] = slot;
    if (t < 8) lw[t >> 1] |= (static_cast<uint32_t>(leaf) & 0xffffu) << (16 * (t & 1));
    const int cnt = pcount ? pcount[slot] : 0;
    nm += cnt;
    if (t < 5) counts |= static_cast<uint32_t>(cnt) << (6 * t);
  }
  gnm[gidx] = nm;
  // packed per-pixel record for hypothesis generation: pixel, depth, colour + |M(u)|,
  // per-tree mode counts (6 bits each, trees 0..4)
  grec[2 * gidx] = make_int4(px, static_cast<int>(c.x), static_cast<int>((c.y & 0xffffffu) | (min(nm, 255) << 24)),
                         static_cast<int>(counts));
  reinterpret_cast<uint4*>(grec)[2 * gidx + 1] = make_uint4(lw[0], lw[1], lw[2], lw[3]);
  if (work) work_add(work, W_NODE_VISITS, static_cast<unsigned>(visits));
  const double dd = static_cast<double>(d);
  const double X = ((static_cast<double>(x) - g.dcx) * dd) / g.dfx;
  const double Y = ((static_cast<double>(y) - g.dcy) * dd) / g.dfy;
  gcam[gidx] = make_float4(static_cast<float>(X), static_cast<float>(Y), static_cast<float>(dd), 0.0f);
}

// Debug: full 256-D feature vectors at given pixels (features.cpp:60-65).
__global__ void k_features(ForestView fv, FrameGeom g, const uint2* __restrict__ tex, const int* __restrict__ px,
                           int n, float* __restrict__ out) {
  const int i = blockIdx.x;
  const int k = threadIdx.x;
  if (i >= n || k >= kFeatures) return;
  const int x = px[i] & 0xffff, y = px[i] >> 16;
  const int W = g.W, H = g.H;
  const uint2 c = tex[y * W + x];
  const float d = __uint_as_float(c.x);
  const short4 sp = fv.specs[k];
  if (!depth_valid(d)) {
    out[static_cast<size_t>(i) * kFeatures + k] = __int_as_float(0x7fc00000);
    return;
  }
  const int qx = x + lround_small(__fdiv_rn(static_cast<float>(sp.x), d));
  const int qy = y + lround_small(__fdiv_rn(static_cast<float>(sp.y), d));
  uint2 pt = make_uint2(0u, 0u);
  if (qx >= 0 && qx < W && qy >= 0 && qy < H) pt = tex[qy * W + qx];
  float v;
  if (sp.z == 0) v = __fsub_rn(d, __uint_as_float(pt.x));
  else v = __fsub_rn(static_cast<float>((c.y >> (8 * sp.w)) & 255u), static_cast<float>((pt.y >> (8 * sp.w)) & 255u));
  out[static_cast<size_t>(i) * kFeatures + k] = v;
}

// =============================== K2: reservoir insertion ================================
// Sequential Algorithm R made parallel and bit-exact. An insertion is an
// item i = g * T + t (grid pixel g, tree t) aimed at leaf slot = gslot[i]; its rank inside
// the leaf is its row-major pixel order among the frame's insertions into that leaf, n =
// seen + rank, and the counter-based draw j = uniform_int(n + 1) from
// Rng::stream(adapt_seed, slot << 32 | n) picks the target. Among insertions of one frame
// hitting the same target the highest rank wins, exactly as the sequential loop would
// overwrite it. Both orderings come from stable radix sorts (O(items) per frame, no scan of
// a leaf's other insertions, no host round trip for the item count):
//  1. sort (slot, item): inside a leaf, items stay in item = pixel order -> rank = position
//     minus the leaf's first position;
//  2. sort (slot * kappa + target, position): inside a run of one target the last entry has
//     the highest rank -> it is the one written.
__global__ void k_ins_keys(const int* __restrict__ gslot, const int* __restrict__ gcount, int T, int items_max,
                           uint32_t pad_key, uint32_t* __restrict__ key, int* __restrict__ val) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= items_max) return;
  const int items = gcount[0] * T;
  key[i] = i < items ? static_cast<uint32_t>(gslot[i]) : pad_key;
  val[i] = i;
}

// Leaf boundaries in sorted order: start[slot] = first position of the leaf's insertions.
__global__ void k_ins_bounds(const uint32_t* __restrict__ key, const int* __restrict__ gcount, int T,
                             int* __restrict__ start) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= gcount[0] * T) return;
  if (p == 0 || key[p] != key[p - 1]) start[key[p]] = p;
}

__global__ void k_ins_target(const uint32_t* __restrict__ key, const int* __restrict__ gcount, int T,
                             const int* __restrict__ start, const uint32_t* __restrict__ seen, int kappa,
                             uint64_t seed, uint64_t pad_key2, int* __restrict__ tgt, uint64_t* __restrict__ key2,
                             int* __restrict__ val2, int items_max) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= items_max) return;
  if (p >= gcount[0] * T) {
    key2[p] = pad_key2;
    val2[p] = p;
    return;
  }
  const uint32_t slot = key[p];
  const uint32_t n = seen[slot] + static_cast<uint32_t>(p - start[slot]);
  int target;
  if (n < static_cast<uint32_t>(kappa)) {
    target = static_cast<int>(n);
  } else {
    Rng rng = rng_stream(seed, (static_cast<uint64_t>(slot) << 32) | n);
    const uint64_t j = rng_uniform_int(rng, static_cast<uint64_t>(n) + 1);
    target = j < static_cast<uint64_t>(kappa) ? static_cast<int>(j) : -1;
  }
  tgt[p] = target;
  key2[p] = target >= 0 ? static_cast<uint64_t>(slot) * static_cast<uint64_t>(kappa) + static_cast<uint64_t>(target)
                        : pad_key2;
  val2[p] = p;
}

__global__ void k_ins_commit(const uint32_t* __restrict__ key, const int* __restrict__ item_at,
                             const int* __restrict__ gcount, int T, const int* __restrict__ start,
                             const uint64_t* __restrict__ key2, const int* __restrict__ pos2,
                             const int* __restrict__ tgt, const int* __restrict__ gpx, const uint2* __restrict__ tex,
                             FrameGeom g, Pose pose, int kappa, uint64_t pad_key2, scr_entry* __restrict__ entries,
                             uint32_t* __restrict__ seen) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  const int items = gcount[0] * T;
  if (q >= items) return;
  // seen += insertions of the leaf (one writer per leaf: its last position in sort 1)
  if (q == items - 1 || key[q + 1] != key[q]) seen[key[q]] += static_cast<uint32_t>(q - start[key[q]] + 1);
  const uint64_t k2 = key2[q];
  if (k2 == pad_key2) return;                         // no target (or padding)
  if (q + 1 < items && key2[q + 1] == k2) return;     // a later insertion overwrites this target
  const int p = pos2[q];
  const uint32_t slot = key[p];
  const int item = item_at[p];
  const int gidx = item / T;
  const int px = gpx[gidx];
  const int x = px & 0xffff, y = px >> 16;
  const uint2 c = tex[y * g.W + x];
  const double dd = static_cast<double>(__uint_as_float(c.x));
  const double pc[3] = {((static_cast<double>(x) - g.dcx) * dd) / g.dfx, ((static_cast<double>(y) - g.dcy) * dd) / g.dfy,
                        dd};
  double pw[3];
  pose_apply(pose, pc, pw);
  scr_entry e;
  e.x = static_cast<float>(pw[0]);
  e.y = static_cast<float>(pw[1]);
  e.z = static_cast<float>(pw[2]);
  e.r = static_cast<uint8_t>(c.y & 255u);
  e.g = static_cast<uint8_t>((c.y >> 8) & 255u);
  e.b = static_cast<uint8_t>((c.y >> 16) & 255u);
  e.pad = 0;
  entries[static_cast<size_t>(slot) * kappa + tgt[p]] = e;
}

// =============================== K3: Really Quick Shift ==================================
// One CTA per scheduled leaf; the reservoir (<= kappa entries) lives in shared memory.
// density_i = sum_j exp(-|xi - xj|^2 / 2 sigma^2) (f64 accumulation in j order), link to
// the nearest strictly-higher-density point within tau (ties: lower index), components by
// pointer chasing, clusters of size >= min sorted by (size desc, root asc), top M_max,
// mu / colour / Sigma + 1e-6 I in f64, Sigma^-1 and Sigma^-1/2 via 3x3 Jacobi.
SCR_DEV uint32_t spread3_10(uint32_t v) {  // 10 bits -> every third bit of 30
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000ffu;
  v = (v | (v << 8)) & 0x0300f00fu;
  v = (v | (v << 4)) & 0x030c30c3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}
SCR_DEV uint32_t morton3_10(uint32_t x, uint32_t y, uint32_t z) {
  return spread3_10(x) | (spread3_10(y) << 1) | (spread3_10(z) << 2);
}
SCR_DEV void atomic_min_float(float* a, float v) {  // via the ordered int view (no NaNs here)
  if (v >= 0.0f) atomicMin(reinterpret_cast<int*>(a), __float_as_int(v));
  else atomicMax(reinterpret_cast<unsigned*>(a), __float_as_uint(v));
}
SCR_DEV void atomic_max_float(float* a, float v) {
  if (v >= 0.0f) atomicMax(reinterpret_cast<int*>(a), __float_as_int(v));
  else atomicMin(reinterpret_cast<unsigned*>(a), __float_as_uint(v));
}
SCR_DEV int rqs_pow2(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

struct RqsParams {
  float c;       // -1 / (2 sigma^2), rounded once on the host
  float tau2;    // tau^2
  int min_size, max_clusters, kappa;
};

#ifndef SCR_RQS_THREADS
#define SCR_RQS_THREADS 1024  // 4 rows per thread at kappa 4096: RQS 2.96 -> 1.43 ms per 256-leaf refresh (256 threads: 8 rows)
#endif
constexpr int kRqsThreads = SCR_RQS_THREADS;
// shared memory of k_rqs: per entry x, y, z, colour, density, parent, root, size, rank
// (40 B) + the 64-bit Morton sort keys (power-of-two count)
inline size_t rqs_smem(int kappa) {
  size_t p2 = 1;
  while (p2 < static_cast<size_t>(kappa)) p2 <<= 1;
  return ((static_cast<size_t>(kappa) * 40 + 7) & ~static_cast<size_t>(7)) + p2 * 8;
}

__global__ void __launch_bounds__(kRqsThreads) k_rqs(const scr_entry* __restrict__ entries, const uint32_t* __restrict__ seen,
                                             int64_t L, int64_t cursor, int nleaves, RqsParams rp,
                                             int* __restrict__ pcount, ModeGeom* __restrict__ pgeom,
                                             float4* __restrict__ pcol, float* __restrict__ pcov,
                                             const scr_entry* __restrict__ single, int single_n,
                                             int* __restrict__ labels_out) {
  extern __shared__ unsigned char smem_raw[];
  const int kappa = rp.kappa;
  float* sx = reinterpret_cast<float*>(smem_raw);
  float* sy = sx + kappa;
  float* sz = sy + kappa;
  uint32_t* scol = reinterpret_cast<uint32_t*>(sz + kappa);
  double* rho = reinterpret_cast<double*>(scol + kappa);
  int* parent = reinterpret_cast<int*>(rho + kappa);
  int* root = parent + kappa;
  int* size = root + kappa;
  int* rlist = size + kappa;
  __shared__ int nroots;

  int64_t slot = 0;
  int n;
  const scr_entry* e;
  if (single) {
    e = single;
    n = single_n;
  } else {
    slot = (cursor + blockIdx.x) % L;
    n = static_cast<int>(min(seen[slot], static_cast<uint32_t>(kappa)));
    e = entries + slot * kappa;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const scr_entry v = e[i];
    sx[i] = v.x;
    sy[i] = v.y;
    sz[i] = v.z;
    scol[i] = v.r | (v.g << 8) | (v.b << 16);
    size[i] = 0;
  }
  if (threadIdx.x == 0) nroots = 0;
  __syncthreads();
  // Rows are handed to threads in Morton order of their points (sorted (code, index) keys,
  // perm[r] = index of the r-th point), so the 32 rows of a warp are spatially close. For a
  // given j the warp then usually agrees that every exp(-|xi - xj|^2 / 2 sigma^2) underflows
  // to exactly 0 (det_expf(x) = 0 for x <= -87, i.e. beyond 1.32 m at sigma = 0.1) and skips
  // it: adding +0 leaves a sum unchanged, and each row is still summed in j order, so the
  // densities are bit-identical to the sequential definition. The link pass skips j likewise
  // when no row of the warp is within tau of it.
  const int np2 = rqs_pow2(n);
  unsigned long long* skey = reinterpret_cast<unsigned long long*>(
      smem_raw + ((static_cast<size_t>(kappa) * 40 + 7) & ~static_cast<size_t>(7)));
  {
    __shared__ float s_box[6];
    if (threadIdx.x == 0) {
      s_box[0] = s_box[1] = s_box[2] = __int_as_float(0x7f800000);
      s_box[3] = s_box[4] = s_box[5] = -__int_as_float(0x7f800000);
    }
    __syncthreads();
    float lo[3] = {__int_as_float(0x7f800000), __int_as_float(0x7f800000), __int_as_float(0x7f800000)};
    float hi[3] = {-lo[0], -lo[1], -lo[2]};
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      lo[0] = fminf(lo[0], sx[i]); hi[0] = fmaxf(hi[0], sx[i]);
      lo[1] = fminf(lo[1], sy[i]); hi[1] = fmaxf(hi[1], sy[i]);
      lo[2] = fminf(lo[2], sz[i]); hi[2] = fmaxf(hi[2], sz[i]);
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      float l = lo[a], h = hi[a];
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        l = fminf(l, __shfl_xor_sync(0xffffffffu, l, o));
        h = fmaxf(h, __shfl_xor_sync(0xffffffffu, h, o));
      }
      if ((threadIdx.x & 31) == 0) {
        atomic_min_float(&s_box[a], l);
        atomic_max_float(&s_box[3 + a], h);
      }
    }
    __syncthreads();
    float scale[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float ext = s_box[3 + a] - s_box[a];
      scale[a] = ext > 0.0f ? 1023.0f / ext : 0.0f;
    }
    for (int r = threadIdx.x; r < np2; r += blockDim.x) {
      unsigned long long k = ~0ull;
      if (r < n) {
        const uint32_t qx = min(1023u, static_cast<uint32_t>(fmaxf(0.0f, (sx[r] - s_box[0]) * scale[0])));
        const uint32_t qy = min(1023u, static_cast<uint32_t>(fmaxf(0.0f, (sy[r] - s_box[1]) * scale[1])));
        const uint32_t qz = min(1023u, static_cast<uint32_t>(fmaxf(0.0f, (sz[r] - s_box[2]) * scale[2])));
        k = (static_cast<unsigned long long>(morton3_10(qx, qy, qz)) << 32) | static_cast<unsigned>(r);
      }
      skey[r] = k;
    }
    __syncthreads();
    for (int size2 = 2; size2 <= np2; size2 <<= 1)  // bitonic sort, ascending
      for (int stride = size2 >> 1; stride > 0; stride >>= 1) {
        for (int t = threadIdx.x; t < (np2 >> 1); t += blockDim.x) {
          const int lo_i = 2 * t - (t & (stride - 1));
          const int hi_i = lo_i + stride;
          const bool up = (lo_i & size2) == 0;
          const unsigned long long a = skey[lo_i], b = skey[hi_i];
          if ((a > b) == up) {
            skey[lo_i] = b;
            skey[hi_i] = a;
          }
        }
        __syncthreads();
      }
  }
  // density (f64 sum over j in index order)
  for (int r0 = 0; r0 < n; r0 += blockDim.x) {  // uniform trip count: every lane votes
    const int r = r0 + static_cast<int>(threadIdx.x);
    const bool live = r < n;
    const int i = live ? static_cast<int>(skey[r] & 0xffffffffu) : 0;
    const float xi = live ? sx[i] : 1e18f, yi = live ? sy[i] : 1e18f, zi = live ? sz[i] : 1e18f;
    double acc = 0.0;
    for (int j = 0; j < n; ++j) {
      const float dx = __fsub_rn(xi, sx[j]), dy = __fsub_rn(yi, sy[j]), dz = __fsub_rn(zi, sz[j]);
      const float d2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
      const float x = __fmul_rn(d2, rp.c);
      if (__any_sync(0xffffffffu, x > -87.0f)) acc = acc + static_cast<double>(det_expf(x));
    }
    if (live) rho[i] = acc;
  }
  __syncthreads();
  // link: nearest strictly-higher-density point within tau (ties: lower index)
  for (int r0 = 0; r0 < n; r0 += blockDim.x) {
    const int r = r0 + static_cast<int>(threadIdx.x);
    const bool live = r < n;
    const int i = live ? static_cast<int>(skey[r] & 0xffffffffu) : 0;
    const float xi = live ? sx[i] : 1e18f, yi = live ? sy[i] : 1e18f, zi = live ? sz[i] : 1e18f;
    const double ri = rho[i];
    float best = __int_as_float(0x7f800000);
    int bj = -1;
    for (int j = 0; j < n; ++j) {
      const float dx = __fsub_rn(xi, sx[j]), dy = __fsub_rn(yi, sy[j]), dz = __fsub_rn(zi, sz[j]);
      const float d2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
      const bool near = d2 <= rp.tau2;
      if (!__any_sync(0xffffffffu, near)) continue;
      if (!near || j == i) continue;
      const double rj = rho[j];
      if (!(rj > ri || (rj == ri && j < i))) continue;
      if (d2 < best) {
        best = d2;
        bj = j;
      }
    }
    if (live) parent[i] = bj;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int r = i;
    while (parent[r] >= 0) r = parent[r];
    root[i] = r;
    atomicAdd(&size[r], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (parent[i] < 0 && size[i] >= rp.min_size) {
      rlist[atomicAdd(&nroots, 1)] = i;
    }
  }
  __syncthreads();
  const int R = nroots;
  // rank roots by (size desc, index asc); parent[] (no longer needed) becomes the
  // root -> cluster map. rlist is only read here, so the ranking is race-free.
  for (int i = threadIdx.x; i < n; i += blockDim.x) parent[i] = -1;
  __syncthreads();
  for (int q = threadIdx.x; q < R; q += blockDim.x) {
    const int i = rlist[q];
    const int si = size[i];
    int rk = 0;
    for (int u = 0; u < R; ++u) {
      const int j = rlist[u];
      rk += (size[j] > si) || (size[j] == si && j < i);
    }
    if (rk < rp.max_clusters) parent[i] = rk;
  }
  __syncthreads();
  const int ncl = min(R, rp.max_clusters);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int lab = parent[root[i]];
    if (labels_out) labels_out[i] = lab;
    root[i] = lab;  // root[] now holds labels
  }
  __syncthreads();
  if (threadIdx.x < ncl) {
    const int k = threadIdx.x;
    double sxm = 0, sym = 0, szm = 0, sr = 0, sg = 0, sb = 0;
    int cnt = 0;
    for (int i = 0; i < n; ++i) {
      if (root[i] != k) continue;
      sxm = sxm + static_cast<double>(sx[i]);
      sym = sym + static_cast<double>(sy[i]);
      szm = szm + static_cast<double>(sz[i]);
      const uint32_t cc = scol[i];
      sr = sr + static_cast<double>(cc & 255u);
      sg = sg + static_cast<double>((cc >> 8) & 255u);
      sb = sb + static_cast<double>((cc >> 16) & 255u);
      ++cnt;
    }
    const double dn = static_cast<double>(cnt);
    const double mx = sxm / dn, my = sym / dn, mz = szm / dn;
    double c00 = 0, c01 = 0, c02 = 0, c11 = 0, c12 = 0, c22 = 0;
    for (int i = 0; i < n; ++i) {
      if (root[i] != k) continue;
      const double dx = static_cast<double>(sx[i]) - mx, dy = static_cast<double>(sy[i]) - my,
                   dz = static_cast<double>(sz[i]) - mz;
      c00 = c00 + dx * dx; c01 = c01 + dx * dy; c02 = c02 + dx * dz;
      c11 = c11 + dy * dy; c12 = c12 + dy * dz; c22 = c22 + dz * dz;
    }
    c00 = c00 / dn + 1e-6; c01 = c01 / dn; c02 = c02 / dn;
    c11 = c11 / dn + 1e-6; c12 = c12 / dn; c22 = c22 / dn + 1e-6;
    const double S[9] = {c00, c01, c02, c01, c11, c12, c02, c12, c22};
    double lam[3], V[9];
    eig3(S, lam, V);
    double il[3], isl[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const double l = lam[q] > 1e-12 ? lam[q] : 1e-12;
      il[q] = 1.0 / l;
      isl[q] = 1.0 / sqrt(l);
    }
#define SCR_FN(w, a, b) \
  ((V[3 * (a) + 0] * w[0] * V[3 * (b) + 0] + V[3 * (a) + 1] * w[1] * V[3 * (b) + 1]) + V[3 * (a) + 2] * w[2] * V[3 * (b) + 2])
    ModeGeom m;
    m.q0 = make_float4(static_cast<float>(mx), static_cast<float>(my), static_cast<float>(mz),
                       static_cast<float>(SCR_FN(il, 0, 0)));
    m.q1 = make_float4(static_cast<float>(SCR_FN(il, 1, 1)), static_cast<float>(SCR_FN(il, 2, 2)),
                       static_cast<float>(2.0 * SCR_FN(il, 0, 1)), static_cast<float>(2.0 * SCR_FN(il, 0, 2)));
    m.q2 = make_float4(static_cast<float>(2.0 * SCR_FN(il, 1, 2)), static_cast<float>(SCR_FN(isl, 0, 0)),
                       static_cast<float>(SCR_FN(isl, 0, 1)), static_cast<float>(SCR_FN(isl, 0, 2)));
    m.q3 = make_float4(static_cast<float>(SCR_FN(isl, 1, 1)), static_cast<float>(SCR_FN(isl, 1, 2)),
                       static_cast<float>(SCR_FN(isl, 2, 2)), 0.0f);
#undef SCR_FN
    const size_t mi = static_cast<size_t>(slot) * kMaxModes + k;
    pgeom[mi] = m;
    pcol[mi] = make_float4(static_cast<float>(sr / dn), static_cast<float>(sg / dn), static_cast<float>(sb / dn),
                           __int_as_float(cnt));
    float* cv = pcov + mi * 6;
    cv[0] = static_cast<float>(c00); cv[1] = static_cast<float>(c01); cv[2] = static_cast<float>(c02);
    cv[3] = static_cast<float>(c11); cv[4] = static_cast<float>(c12); cv[5] = static_cast<float>(c22);
  }
  if (threadIdx.x == 0) pcount[slot] = ncl;
}

// =============================== synthetic renderer (fixture) ==============================
SCR_DEV uint32_t hash3(int x, int y, uint32_t seed) {
  uint32_t h = static_cast<uint32_t>(x) * 73856093u ^ static_cast<uint32_t>(y) * 19349663u ^ seed;
  h ^= h >> 16;
  h *= 0x7feb352du;
  h ^= h >> 15;
  h *= 0x846ca68bu;
  h ^= h >> 16;
  return h;
}

__global__ void k_render(const Prim* __restrict__ prims, int nprims, FrameGeom g, const Pose* __restrict__ poses,
                         float* __restrict__ depth, uint8_t* __restrict__ rgb) {
  const int f = blockIdx.y;
  const int WH = g.W * g.H;
  float R[9], o[3];
#pragma unroll
  for (int i = 0; i < 9; ++i) R[i] = static_cast<float>(poses[f].R[i]);
#pragma unroll
  for (int i = 0; i < 3; ++i) o[i] = static_cast<float>(poses[f].t[i]);
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < WH; p += gridDim.x * blockDim.x) {
    const int x = p % g.W, y = p / g.W;
    float d[3];
    ray_dir(R, g.fx, g.fy, g.cx, g.cy, x, y, d);
    const Hit h = raycast(prims, nprims, o, d);
    const size_t idx = static_cast<size_t>(f) * WH + p;
    if (h.prim < 0 || !(h.t <= kRenderMaxDepth)) {
      depth[idx] = 0.0f;
      rgb[3 * idx] = rgb[3 * idx + 1] = rgb[3 * idx + 2] = 0;
      continue;
    }
    depth[idx] = h.t;
    float q[3], n[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) q[i] = __fmaf_rn(h.t, d[i], o[i]);
    hit_normal(prims, h.prim, h.face, q, n);
    const float ax = fabsf(n[0]), ay = fabsf(n[1]), az = fabsf(n[2]);
    const int dom = (ax >= ay && ax >= az) ? 0 : (ay >= az ? 1 : 2);
    const int u = dom == 0 ? 1 : 0, v = dom == 2 ? 1 : 2;
    const Prim& pr = prims[h.prim];
    const float inv = __fdiv_rn(1.0f, pr.cell);
    const int iu = static_cast<int>(floorf(__fmul_rn(q[u], inv)));
    const int iv = static_cast<int>(floorf(__fmul_rn(q[v], inv)));
    const uint32_t hh = hash3(iu, iv, pr.tex_seed);
    const float fct = __fadd_rn(0.35f, __fmul_rn(0.65f, __fdiv_rn(static_cast<float>(hh & 255u), 255.0f)));
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float val = __fadd_rn(__fmul_rn(pr.colour[c], fct), 0.5f);
      rgb[3 * idx + c] = static_cast<uint8_t>(min(255, max(0, static_cast<int>(val))));
    }
  }
}

}  // namespace scr

using namespace scr;

// =============================== host side ============================================
ForestView scr_scene_s::forest_view() const {
  ForestView v;
  v.nodes = d_nodes;
  v.specs = d_specs;
  v.T = T;
  for (int t = 0; t < kMaxTrees; ++t) {
    v.node_base[t] = t < T ? node_base[t] : 0;
    v.leaf_base[t] = t < T ? leaf_base[t] : 0;
  }
  return v;
}

namespace {
template <typename T>
bool rd(const uint8_t* d, size_t n, size_t& off, T* v) {
  if (off + sizeof(T) > n) return false;
  std::memcpy(v, d + off, sizeof(T));
  off += sizeof(T);
  return true;
}
scr_status malformed(const std::string& m) {
  set_error("deserialize_forest: " + m);
  return SCR_E_MALFORMED_DATA;
}
template <typename T>
scr_status dalloc(T** p, size_t count) {
  SCR_CUDA(cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(1, count) * sizeof(T)));
  return SCR_OK;
}
#define SCR_TRY(x)                       \
  do {                                   \
    scr_status _s = (x);                 \
    if (_s != SCR_OK) return _s;         \
  } while (0)
}  // namespace

namespace scr {
// Per-lane batch workspace (frames addressed by workspace slot f in [0, max_batch)).
scr_status alloc_workspace(scr_scene s, int max_batch) {
  const scr_intrinsics* k = &s->k;
  const int64_t L = s->L;
  scr_status st;
  Workspace& w = s->ws;
  w.cap = max_batch;
  w.gmax = ((k->width + 3) / 4) * ((k->height + 3) / 4);
  const size_t WH = static_cast<size_t>(k->width) * k->height;
  const size_t B = static_cast<size_t>(max_batch);
  if ((st = dalloc(&w.depth, B * WH)) != SCR_OK) return st;
  if ((st = dalloc(&w.rgb, B * WH * 3)) != SCR_OK) return st;
  if ((st = dalloc(&w.tex, B * WH)) != SCR_OK) return st;
  if ((st = dalloc(&w.dplane, B * (WH + WH / 4 + WH / 16))) != SCR_OK) return st;
  if ((st = dalloc(&w.gcount, B)) != SCR_OK) return st;
  if ((st = dalloc(&w.gpx, B * w.gmax)) != SCR_OK) return st;
  if ((st = dalloc(&w.gcam, B * w.gmax)) != SCR_OK) return st;
  if ((st = dalloc(&w.gslot, B * w.gmax * s->T)) != SCR_OK) return st;
  if ((st = dalloc(&w.gnm, B * w.gmax)) != SCR_OK) return st;
  if ((st = dalloc(&w.grec, 2 * B * w.gmax)) != SCR_OK) return st;  // interleaved with the leaf ids
  if ((st = dalloc(&w.fidx, B)) != SCR_OK) return st;
  if ((st = dalloc(&w.seeds, B)) != SCR_OK) return st;
  if ((st = dalloc(&w.status, B)) != SCR_OK) return st;
  if ((st = dalloc(&w.hctr, 2 * B)) != SCR_OK) return st;  // slot counters, then suspect counts
  if ((st = dalloc(&w.d_res, B)) != SCR_OK) return st;
  SCR_CUDA(cudaMallocHost(reinterpret_cast<void**>(&w.h_res), B * sizeof(scr_result)));
  SCR_CUDA(cudaMallocHost(reinterpret_cast<void**>(&w.h_idx), B * sizeof(int)));
  SCR_CUDA(cudaMallocHost(reinterpret_cast<void**>(&w.h_fsidx), B * sizeof(int)));
  SCR_CUDA(cudaMallocHost(reinterpret_cast<void**>(&w.h_seeds), B * sizeof(uint64_t)));
  SCR_CUDA(cudaEventCreate(&w.ev_stage[0]));
  SCR_CUDA(cudaEventCreate(&w.ev_stage[1]));
  SCR_CUDA(cudaEventCreateWithFlags(&w.ev_upload, cudaEventDisableTiming));
  const size_t items = static_cast<size_t>(w.gmax) * s->T;
  if ((st = dalloc(&w.ins_start, L)) != SCR_OK) return st;
  if ((st = dalloc(&w.ins_key, items)) != SCR_OK) return st;
  if ((st = dalloc(&w.ins_key_s, items)) != SCR_OK) return st;
  if ((st = dalloc(&w.ins_val, items)) != SCR_OK) return st;
  if ((st = dalloc(&w.ins_item, items)) != SCR_OK) return st;
  if ((st = dalloc(&w.ins_tgt, items)) != SCR_OK) return st;
  if ((st = dalloc(&w.ins_key2, items)) != SCR_OK) return st;
  if ((st = dalloc(&w.ins_key2_s, items)) != SCR_OK) return st;
  if ((st = dalloc(&w.ins_val2, items)) != SCR_OK) return st;
  if ((st = dalloc(&w.ins_pos2, items)) != SCR_OK) return st;
  {  // radix-sort scratch for the larger (64-bit key) of the two sorts
    size_t a = 0, b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, w.ins_key, w.ins_key_s, w.ins_val, w.ins_item, static_cast<int>(items));
    cub::DeviceRadixSort::SortPairs(nullptr, b, w.ins_key2, w.ins_key2_s, w.ins_val2, w.ins_pos2,
                                    static_cast<int>(items));
    w.ins_tmp_bytes = std::max(a, b);
    if ((st = dalloc(reinterpret_cast<unsigned char**>(&w.ins_tmp), w.ins_tmp_bytes)) != SCR_OK) return st;
  }
  return SCR_OK;
}

// A lane reads the parent's current shared pointers and orders its stream after the
// parent's last published update (readers never see a half-published state).
scr_status refresh_lane(scr_scene s) {
  scr_scene p = s->parent;
  if (!p) return SCR_OK;
  s->d_nodes = p->d_nodes;
  s->d_specs = p->d_specs;
  s->d_entries = p->d_entries;
  s->d_seen = p->d_seen;
  s->d_count = p->d_count;
  s->d_geom = p->d_geom;
  s->d_col = p->d_col;
  s->d_cov = p->d_cov;
  s->d_prims = p->d_prims;
  s->n_prims = p->n_prims;
  s->tsdf_model = p->tsdf_model;
  s->cursor = p->cursor;
  if (p->published && s->stream) SCR_CUDA(cudaStreamWaitEvent(s->stream, p->published, 0));
  return SCR_OK;
}

// Marks the end of an update of shared state on the scene's stream (lanes wait on it).
scr_status publish(scr_scene s) {
  SCR_CUDA(cudaEventRecord(s->published, s->stream));
  return SCR_OK;
}

}  // namespace scr

extern "C" {

const char* scr_last_error(void) { return g_err.c_str(); }
const char* scr_version(void) { return "screloc-b200 0.1 (sm_100a)"; }

scr_status scr_device_open(int ordinal, scr_device* out) {
  if (!out) return SCR_E_ARG;
  int n = 0;
  SCR_CUDA(cudaGetDeviceCount(&n));
  if (ordinal < 0 || ordinal >= n) {
    set_error("scr_device_open: no such device");
    return SCR_E_ARG;
  }
  SCR_CUDA(cudaSetDevice(ordinal));
  scr_device d = new scr_device_s();
  d->ordinal = ordinal;
  {
    const cudaError_t e = cudaStreamCreateWithFlags(&d->copy, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      delete d;
      return cuda_fail(e, "cudaStreamCreate(copy)");
    }
  }
  cudaDeviceGetAttribute(&d->sm_count, cudaDevAttrMultiProcessorCount, ordinal);
  *out = d;
  return SCR_OK;
}

void scr_device_close(scr_device d) {
  if (!d) return;
  if (d->copy) {
    cudaSetDevice(d->ordinal);
    cudaStreamDestroy(d->copy);
  }
  delete d;
}

scr_status scr_scene_create(scr_device dev, const uint8_t* blob, size_t n, const scr_forest_params* fp,
                            const scr_intrinsics* k, uint64_t adapt_seed, int max_batch, scr_scene* out) {
  if (!dev || !blob || !fp || !k || !out || max_batch <= 0) {
    set_error("scr_scene_create: null argument");
    return SCR_E_ARG;
  }
  if (k->width <= 0 || k->height <= 0 || k->width > 1280 || k->height > 960) {
    // shared-memory tables of ICP (ray directions) and generation (per-pixel mode counts)
    set_error("scr_scene_create: frames up to 1280 x 960 (the stress configuration)");
    return SCR_E_ARG;
  }
  if (!(k->fx > 0 && k->fy > 0 && k->cx >= 0 && k->cx < k->width && k->cy >= 0 && k->cy < k->height)) {
    set_error("scr_scene_create: invalid intrinsics (geometry.hpp:52-54)");
    return SCR_E_ARG;
  }
  if (fp->capacity <= 0 || fp->capacity > 4096 || fp->max_clusters <= 0 || fp->max_clusters > kMaxModes) {
    set_error("scr_scene_create: capacity must be in (0, 4096] and max_clusters in (0, 50]");
    return SCR_E_ARG;
  }
  // ---- parse the forest (SPEC.md:300 layout; validation mirrors deserialize_forest) ----
  size_t off = 0;
  char magic[4];
  for (int i = 0; i < 4; ++i)
    if (!rd(blob, n, off, &magic[i])) return malformed("truncated at offset " + std::to_string(off));
  if (magic[0] != 'S' || magic[1] != 'C' || magic[2] != 'R' || magic[3] != 'F') return malformed("bad magic");
  uint32_t version, nt, ns;
  if (!rd(blob, n, off, &version)) return malformed("truncated at offset " + std::to_string(off));
  if (version != 1) return malformed("unsupported version " + std::to_string(version));
  if (!rd(blob, n, off, &nt) || !rd(blob, n, off, &ns)) return malformed("truncated at offset " + std::to_string(off));
  if (ns != kFeatures) return malformed("spec count " + std::to_string(ns));
  if (nt == 0 || nt > static_cast<uint32_t>(kMaxTrees)) return malformed("tree count " + std::to_string(nt));
  std::vector<short4> specs(kFeatures);
  for (uint32_t i = 0; i < ns; ++i) {
    uint8_t kind, ch;
    int16_t dx, dy;
    if (!rd(blob, n, off, &kind) || !rd(blob, n, off, &ch) || !rd(blob, n, off, &dx) || !rd(blob, n, off, &dy))
      return malformed("truncated at offset " + std::to_string(off));
    if (kind > 1 || ch > 2) return malformed("bad spec at offset " + std::to_string(off));
    specs[i] = make_short4(dx, dy, kind, ch);
  }
  std::vector<int4> nodes;
  std::vector<int> node_base, leaf_base;
  bool leaves16 = true;
  int64_t L = 0;
  for (uint32_t t = 0; t < nt; ++t) {
    uint32_t nn;
    int32_t leaves;
    if (!rd(blob, n, off, &nn) || !rd(blob, n, off, &leaves)) return malformed("truncated at offset " + std::to_string(off));
    if (nn == 0 || nn > (1u << 26) || leaves <= 0) return malformed("bad node count");
    node_base.push_back(static_cast<int>(nodes.size()));
    leaf_base.push_back(static_cast<int>(L));
    const size_t first = nodes.size();
    for (uint32_t i = 0; i < nn; ++i) {
      int32_t feat, left, right, leaf;
      float thr;
      if (!rd(blob, n, off, &feat) || !rd(blob, n, off, &thr) || !rd(blob, n, off, &left) ||
          !rd(blob, n, off, &right) || !rd(blob, n, off, &leaf))
        return malformed("truncated at offset " + std::to_string(off));
      int4 v;
      if (left < 0) {
        if (leaf < 0 || leaf >= leaves) return malformed("bad leaf id");
        v = make_int4(-1, leaf, 0, 0);
      } else {
        if (left <= static_cast<int32_t>(i) || right <= static_cast<int32_t>(i) || left >= static_cast<int32_t>(nn) ||
            right >= static_cast<int32_t>(nn) || feat < 0 || feat >= kFeatures)
          return malformed("bad branch node " + std::to_string(i));
        int tb;
        std::memcpy(&tb, &thr, 4);
        v = make_int4(left, right, feat, tb);
      }
      nodes.push_back(v);
    }
    (void)first;
    if (leaves > 65536) leaves16 = false;
    L += leaves;
  }
  if (off != n) return malformed("trailing bytes at offset " + std::to_string(off));

  SCR_CUDA(cudaSetDevice(dev->ordinal));
  scr_scene s = new scr_scene_s();
  s->dev = dev;
  s->k = *k;
  s->fp = *fp;
  s->adapt_seed = adapt_seed;
  s->T = static_cast<int>(nt);
  s->L = L;
  s->node_base = node_base;
  s->leaf_base = leaf_base;
  s->leaves16 = leaves16;
  s->geom.W = k->width;
  s->geom.H = k->height;
  s->geom.fx = static_cast<float>(k->fx);
  s->geom.fy = static_cast<float>(k->fy);
  s->geom.cx = static_cast<float>(k->cx);
  s->geom.cy = static_cast<float>(k->cy);
  s->geom.dfx = k->fx;
  s->geom.dfy = k->fy;
  s->geom.dcx = k->cx;
  s->geom.dcy = k->cy;
  auto fail = [&](scr_status st) {
    scr_scene_destroy(s);
    return st;
  };
  cudaError_t e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) return fail(cuda_fail(e, "cudaStreamCreate"));
  e = cudaEventCreateWithFlags(&s->published, cudaEventDisableTiming);
  if (e != cudaSuccess) return fail(cuda_fail(e, "cudaEventCreate"));
  scr_status st;
  if ((st = dalloc(&s->d_nodes, nodes.size())) != SCR_OK) return fail(st);
  if ((st = dalloc(&s->d_specs, kFeatures)) != SCR_OK) return fail(st);
  const size_t kappa = static_cast<size_t>(fp->capacity);
  if ((st = dalloc(&s->d_entries, static_cast<size_t>(L) * kappa)) != SCR_OK) return fail(st);
  if ((st = dalloc(&s->d_seen, L)) != SCR_OK) return fail(st);
  if ((st = dalloc(&s->d_count, L)) != SCR_OK) return fail(st);
  if ((st = dalloc(&s->d_geom, static_cast<size_t>(L) * kMaxModes)) != SCR_OK) return fail(st);
  if ((st = dalloc(&s->d_col, static_cast<size_t>(L) * kMaxModes)) != SCR_OK) return fail(st);
  if ((st = dalloc(&s->d_cov, static_cast<size_t>(L) * kMaxModes * 6)) != SCR_OK) return fail(st);
  e = cudaMemcpyAsync(s->d_nodes, nodes.data(), nodes.size() * sizeof(int4), cudaMemcpyHostToDevice, s->stream);
  if (e != cudaSuccess) return fail(cuda_fail(e, "upload nodes"));
  e = cudaMemcpyAsync(s->d_specs, specs.data(), kFeatures * sizeof(short4), cudaMemcpyHostToDevice, s->stream);
  if (e != cudaSuccess) return fail(cuda_fail(e, "upload specs"));
  e = cudaStreamSynchronize(s->stream);  // the pageable sources are locals
  if (e != cudaSuccess) return fail(cuda_fail(e, "upload sync"));
  if ((st = alloc_workspace(s, max_batch)) != SCR_OK) return fail(st);
  if ((st = scr_reset(s)) != SCR_OK) return fail(st);
  e = cudaFuncSetAttribute(k_rqs, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (e != cudaSuccess) return fail(cuda_fail(e, "cudaFuncSetAttribute(k_rqs)"));
  if ((st = reloc_init()) != SCR_OK) return fail(st);
  e = cudaStreamSynchronize(s->stream);
  if (e != cudaSuccess) return fail(cuda_fail(e, "scene create sync"));
  *out = s;
  return SCR_OK;
}

scr_status scr_scene_fork(scr_scene parent, int max_batch, scr_scene* out) {
  if (!parent || !out || max_batch <= 0 || max_batch > 4096) {
    set_error("scr_scene_fork: bad arguments (max_batch 1..4096)");
    return SCR_E_ARG;
  }
  if (parent->parent) {
    set_error("scr_scene_fork: fork the root scene, not a lane");
    return SCR_E_ARG;
  }
  SCR_CUDA(cudaSetDevice(parent->dev->ordinal));
  scr_scene s = new scr_scene_s();
  s->parent = parent;
  s->dev = parent->dev;
  s->k = parent->k;
  s->geom = parent->geom;
  s->fp = parent->fp;
  s->adapt_seed = parent->adapt_seed;
  s->T = parent->T;
  s->L = parent->L;
  s->cursor = parent->cursor;
  s->node_base = parent->node_base;
  s->leaf_base = parent->leaf_base;
  s->leaves16 = parent->leaves16;
  parent->lanes++;
  scr_status st = refresh_lane(s);
  cudaError_t e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) st = cuda_fail(e, "cudaStreamCreate");
  if (st == SCR_OK) st = alloc_workspace(s, max_batch);
  if (st != SCR_OK) {
    scr_scene_destroy(s);
    return st;
  }
  *out = s;
  return SCR_OK;
}

void scr_scene_destroy(scr_scene s) {
  if (!s) return;
  cudaSetDevice(s->dev->ordinal);
  if (s->stream) cudaStreamSynchronize(s->stream);
  if (s->parent) {  // a lane: the shared state belongs to the parent
    s->parent->lanes--;
    s->d_nodes = nullptr; s->d_specs = nullptr; s->d_entries = nullptr; s->d_seen = nullptr;
    s->d_count = nullptr; s->d_geom = nullptr; s->d_col = nullptr; s->d_cov = nullptr; s->d_prims = nullptr;
    s->tsdf_model = nullptr;
  }
  if (s->published) cudaEventDestroy(s->published);
  for (cudaEvent_t e : {s->ws.ev_stage[0], s->ws.ev_stage[1], s->ws.ev_upload, s->ws.ev_upload2})
    if (e) cudaEventDestroy(e);
  for (void* p : {static_cast<void*>(s->ws.depth2), static_cast<void*>(s->ws.rgb2)})
    if (p) cudaFree(p);
  for (void* h : {static_cast<void*>(s->ws.h_res), static_cast<void*>(s->ws.h_idx), static_cast<void*>(s->ws.h_fsidx),
                  static_cast<void*>(s->ws.h_seeds)})
    if (h) cudaFreeHost(h);
  if (s->ws.d_res) cudaFree(s->ws.d_res);
  void* ptrs[] = {s->d_nodes, s->d_specs, s->d_entries, s->d_seen, s->d_count, s->d_geom, s->d_col, s->d_cov,
                  s->d_prims, s->ws.depth, s->ws.rgb, s->ws.tex, s->ws.gcount, s->ws.gpx, s->ws.gcam, s->ws.gslot,
                  s->ws.gnm, s->ws.hyp, s->ws.henergy, s->ws.hok, s->ws.hcand, s->ws.sus, s->ws.hiters, s->ws.cand, s->ws.cenergy,
                  s->ws.cslot, s->ws.ncand, s->ws.samples, s->ws.assoc, s->ws.icp_map, s->ws.icp_pose,
                  s->ws.icp_score, s->ws.icp_conv, s->ws.icp_rms, s->ws.icp_inl, s->ws.fidx, s->ws.seeds,
                  s->ws.status, s->ws.hctr, s->ws.epart, s->ws.grec, s->ws.dplane, s->ws.hypc, s->ws.hslot, s->ws.hvalid, s->ws.lmst, s->ws.ins_start, s->ws.ins_key, s->ws.ins_key_s, s->ws.ins_val, s->ws.ins_item,
                  s->ws.ins_tgt, s->ws.ins_key2, s->ws.ins_key2_s, s->ws.ins_val2, s->ws.ins_pos2, s->ws.ins_tmp};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (s->stream) cudaStreamDestroy(s->stream);
  delete s;
}

scr_status scr_profile_enable(scr_scene s, int enable) {
  if (!s) return SCR_E_ARG;
  SCR_CUDA(cudaSetDevice(s->dev->ordinal));
  SCR_CUDA(cudaStreamSynchronize(s->stream));
  prof_flush(s);
  if (!s->prof.d_work) SCR_CUDA(cudaMalloc(&s->prof.d_work, W_COUNT * sizeof(unsigned long long)));
  SCR_CUDA(cudaMemset(s->prof.d_work, 0, W_COUNT * sizeof(unsigned long long)));
  for (int k = 0; k < K_COUNT; ++k) {
    s->prof.ms[k] = 0.0;
    s->prof.launches[k] = 0;
  }
  s->prof.on = enable != 0;
  return SCR_OK;
}

int scr_profile_read(scr_scene s, const char** names, double* ms, int64_t* launches, uint64_t* work, int cap) {
  if (!s) return 0;
  cudaSetDevice(s->dev->ordinal);
  cudaStreamSynchronize(s->stream);
  prof_flush(s);
  for (int k = 0; k < K_COUNT && k < cap; ++k) {
    if (names) names[k] = kKernelNames[k];
    if (ms) ms[k] = s->prof.ms[k];
    if (launches) launches[k] = s->prof.launches[k];
  }
  if (work && s->prof.d_work) cudaMemcpy(work, s->prof.d_work, W_COUNT * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  return K_COUNT;
}

int64_t scr_scene_total_leaves(scr_scene s) { return s ? s->L : 0; }
void* scr_scene_stream(scr_scene s) { return s ? static_cast<void*>(s->stream) : nullptr; }
int64_t scr_kernel_launches(scr_scene s) { return s ? s->launches : 0; }
int64_t scr_update_cursor(scr_scene s) { return s ? s->cursor : 0; }

static scr_status scr_scene_set_analytic_model_impl(scr_scene s, const scr_prim* prims, int n) {
  if (!s || (!prims && n > 0) || n < 0 || n > 256) {
    set_error("scr_scene_set_analytic_model: 0..256 primitives");
    return SCR_E_ARG;
  }
  SCR_CUDA(cudaSetDevice(s->dev->ordinal));
  std::vector<Prim> p(n);
  for (int i = 0; i < n; ++i) {
    p[i].type = prims[i].type;
    for (int q = 0; q < 3; ++q) {
      p[i].a[q] = prims[i].a[q];
      p[i].b[q] = prims[i].b[q];
      p[i].colour[q] = prims[i].colour[q];
    }
    p[i].cell = prims[i].cell;
    p[i].tex_seed = prims[i].tex_seed;
    if (p[i].type != 0 && p[i].type != 1) {
      set_error("scr_scene_set_analytic_model: unknown primitive type");
      return SCR_E_ARG;
    }
  }
  SCR_CUDA(cudaStreamSynchronize(s->stream));
  if (s->d_prims) SCR_CUDA(cudaFree(s->d_prims));
  s->d_prims = nullptr;
  s->n_prims = n;
  if (n > 0) {
    SCR_CUDA(cudaMalloc(&s->d_prims, n * sizeof(Prim)));
    SCR_CUDA(cudaMemcpyAsync(s->d_prims, p.data(), n * sizeof(Prim), cudaMemcpyHostToDevice, s->stream));
    SCR_CUDA(cudaStreamSynchronize(s->stream));
  }
  return SCR_OK;
}

static scr_status scr_reset_impl(scr_scene s) {
  if (!s) return SCR_E_ARG;
  SCR_CUDA(cudaSetDevice(s->dev->ordinal));
  SCR_CUDA(cudaMemsetAsync(s->d_entries, 0, static_cast<size_t>(s->L) * s->fp.capacity * sizeof(scr_entry), s->stream));
  SCR_CUDA(cudaMemsetAsync(s->d_seen, 0, s->L * sizeof(uint32_t), s->stream));
  SCR_CUDA(cudaMemsetAsync(s->d_count, 0, s->L * sizeof(int), s->stream));
  SCR_CUDA(cudaMemsetAsync(s->d_geom, 0, static_cast<size_t>(s->L) * kMaxModes * sizeof(ModeGeom), s->stream));
  SCR_CUDA(cudaMemsetAsync(s->d_col, 0, static_cast<size_t>(s->L) * kMaxModes * sizeof(float4), s->stream));
  SCR_CUDA(cudaMemsetAsync(s->d_cov, 0, static_cast<size_t>(s->L) * kMaxModes * 6 * sizeof(float), s->stream));
  s->cursor = 0;
  SCR_CUDA(cudaStreamSynchronize(s->stream));
  return SCR_OK;
}

}  // extern "C"

namespace scr {

// K0 + grid + K1 for n frames whose raw buffers are at depth_base/rgb_base (device)
// selected by d_idx (or identity), into workspace slots 0..n-1.
scr_status pack_frames(scr_scene s, const float* depth_base, const uint8_t* rgb_base, const int* d_idx, int n) {
  Workspace& w = s->ws;
  const int W = s->k.width, H = s->k.height, WH = W * H;
  const int pack_blocks = (WH + 1023) / 1024 < 64 ? (WH + 1023) / 1024 : 64;
  SCR_LAUNCH(s, K_PACK, (k_pack<<<dim3(pack_blocks, n), 256, 0, s->stream>>>(depth_base, rgb_base, d_idx, W, H, w.tex,
                                                                           w.dplane)));
  SCR_LAUNCH(s, K_GRID, (k_grid<<<n, 1024, 0, s->stream>>>(w.tex, W, H, w.gmax, w.gcount, w.gpx)));
  SCR_LAUNCH(s, K_LEAVES,
             (k_leaves<<<dim3((w.gmax + 127) / 128, n), 128, 0, s->stream>>>(
                 s->forest_view(), s->geom, w.tex, w.gcount, w.gpx, w.gmax, w.gslot, w.gnm, w.gcam, w.grec,
                 s->d_count, work_ptr(s))));
  SCR_CUDA(cudaGetLastError());
  return SCR_OK;
}

scr_status check_frames(const scr_scene_s* s, const scr_frame* frames, int n) {
  if (n > 0 && !frames) {
    set_error("null frame array");
    return SCR_E_ARG;
  }
  for (int i = 0; i < n; ++i) {
    if (!frames[i].depth || !frames[i].rgb) {
      set_error("frame without depth or colour plane");
      return SCR_E_ARG;
    }
    if (frames[i].width != s->k.width || frames[i].height != s->k.height) {
      set_error("frame " + std::to_string(i) + " is " + std::to_string(frames[i].width) + "x" +
                std::to_string(frames[i].height) + ", the scene's intrinsics are " + std::to_string(s->k.width) + "x" +
                std::to_string(s->k.height));
      return SCR_E_DIMENSION_MISMATCH;
    }
  }
  return SCR_OK;
}

}  // namespace scr

namespace {
scr_status upload_frames(scr_scene s, const scr_frame* frames, int n) {
  SCR_TRY(check_frames(s, frames, n));
  const size_t WH = static_cast<size_t>(s->k.width) * s->k.height;
  for (int i = 0; i < n; ++i) {
    if (!frames[i].depth || !frames[i].rgb) {
      set_error("frame with null depth or colour");
      return SCR_E_ARG;
    }
    SCR_CUDA(cudaMemcpyAsync(s->ws.depth + i * WH, frames[i].depth, WH * sizeof(float), cudaMemcpyHostToDevice,
                             s->stream));
    SCR_CUDA(cudaMemcpyAsync(s->ws.rgb + i * WH * 3, frames[i].rgb, WH * 3, cudaMemcpyHostToDevice, s->stream));
  }
  return SCR_OK;
}

static int bits_for(uint64_t v) {  // bits needed to represent 0..v
  int b = 1;
  while (b < 64 && (v >> b) != 0) ++b;
  return b;
}

// integrate_frame for the frame packed in workspace slot 0. No host
// round trip: kernels read the frame's grid count on the device and the sorts run over
// the workspace's item capacity (padding keys sort last and are skipped).
scr_status integrate_slot0(scr_scene s, const scr_pose* pose) {
  Workspace& w = s->ws;
  const int T = s->T;
  const int items_max = w.gmax * T;
  const uint32_t pad_key = static_cast<uint32_t>(s->L);
  const uint64_t pad_key2 = static_cast<uint64_t>(s->L) * static_cast<uint64_t>(s->fp.capacity);
  Pose P;
  std::memcpy(P.R, pose->R, sizeof(P.R));
  std::memcpy(P.t, pose->t, sizeof(P.t));
  const int tb = 256, nb = (items_max + tb - 1) / tb;
  SCR_LAUNCH(s, K_INSERT, (k_ins_keys<<<nb, tb, 0, s->stream>>>(w.gslot, w.gcount, T, items_max, pad_key, w.ins_key,
                                                                w.ins_val)));
  size_t tmp = w.ins_tmp_bytes;
  SCR_CUDA(cub::DeviceRadixSort::SortPairs(w.ins_tmp, tmp, w.ins_key, w.ins_key_s, w.ins_val, w.ins_item, items_max, 0,
                                           bits_for(pad_key), s->stream));
  SCR_LAUNCH(s, K_INSERT, (k_ins_bounds<<<nb, tb, 0, s->stream>>>(w.ins_key_s, w.gcount, T, w.ins_start)));
  SCR_LAUNCH(s, K_INSERT, (k_ins_target<<<nb, tb, 0, s->stream>>>(w.ins_key_s, w.gcount, T, w.ins_start, s->d_seen,
                                                                  s->fp.capacity, s->adapt_seed, pad_key2, w.ins_tgt,
                                                                  w.ins_key2, w.ins_val2, items_max)));
  tmp = w.ins_tmp_bytes;
  SCR_CUDA(cub::DeviceRadixSort::SortPairs(w.ins_tmp, tmp, w.ins_key2, w.ins_key2_s, w.ins_val2, w.ins_pos2,
                                           items_max, 0, bits_for(pad_key2), s->stream));
  SCR_LAUNCH(s, K_INSERT, (k_ins_commit<<<nb, tb, 0, s->stream>>>(w.ins_key_s, w.ins_item, w.gcount, T, w.ins_start,
                                                                  w.ins_key2_s, w.ins_pos2, w.ins_tgt, w.gpx, w.tex,
                                                                  s->geom, P, s->fp.capacity, pad_key2, s->d_entries,
                                                                  s->d_seen)));
  SCR_CUDA(cudaGetLastError());
  return SCR_OK;
}
}  // namespace

extern "C" {

scr_status scr_train(scr_scene s, const scr_frame* frame, const scr_pose* pose) { return scr_train_batch(s, frame, pose, 1); }

static scr_status scr_train_batch_impl(scr_scene s, const scr_frame* frames, const scr_pose* poses, int n) {
  if (!s || (!frames && n > 0) || (!poses && n > 0) || n < 0) return SCR_E_ARG;
  SCR_CUDA(cudaSetDevice(s->dev->ordinal));
  for (int i = 0; i < n; ++i) {
    if (!frames[i].pose_reliable) {
      set_error("integrate_frame: pose flagged unreliable");
      return SCR_E_UNRELIABLE_POSE;
    }
    SCR_TRY(upload_frames(s, &frames[i], 1));
    SCR_TRY(pack_frames(s, s->ws.depth, s->ws.rgb, nullptr, 1));
    SCR_TRY(integrate_slot0(s, &poses[i]));
  }
  SCR_CUDA(cudaStreamSynchronize(s->stream));
  return SCR_OK;
}

static scr_status scr_train_frameset_impl(scr_scene s, scr_frameset fs, const int32_t* idx, const scr_pose* poses, int n) {
  if (!s || !fs || (!idx && n > 0) || (!poses && n > 0)) return SCR_E_ARG;
  SCR_CUDA(cudaSetDevice(s->dev->ordinal));
  const size_t WH = static_cast<size_t>(s->k.width) * s->k.height;
  for (int i = 0; i < n; ++i) {
    if (idx[i] < 0 || idx[i] >= fs->cap) return SCR_E_ARG;
    SCR_TRY(pack_frames(s, fs->depth + idx[i] * WH, fs->rgb + idx[i] * WH * 3, nullptr, 1));
    SCR_TRY(integrate_slot0(s, &poses[i]));
  }
  SCR_CUDA(cudaStreamSynchronize(s->stream));
  return SCR_OK;
}

static scr_status scr_update_impl(scr_scene s, int64_t leaves_per_call) {
  if (!s || leaves_per_call < 0) return SCR_E_ARG;
  SCR_CUDA(cudaSetDevice(s->dev->ordinal));
  const int64_t n = std::min<int64_t>(leaves_per_call, s->L);
  if (n == 0) return SCR_OK;
  RqsParams rp;
  rp.c = static_cast<float>(-1.0 / (2.0 * static_cast<double>(s->fp.sigma) * static_cast<double>(s->fp.sigma)));
  rp.tau2 = static_cast<float>(static_cast<double>(s->fp.tau) * static_cast<double>(s->fp.tau));
  rp.min_size = s->fp.min_cluster_size;
  rp.max_clusters = s->fp.max_clusters;
  rp.kappa = s->fp.capacity;
  const size_t smem = rqs_smem(rp.kappa);
  for (int64_t done = 0; done < n; done += 65535) {
    const int chunk = static_cast<int>(std::min<int64_t>(65535, n - done));
    SCR_LAUNCH(s, K_RQS,
               (k_rqs<<<chunk, kRqsThreads, smem, s->stream>>>(s->d_entries, s->d_seen, s->L, (s->cursor + done) % s->L,
                                                       chunk, rp, s->d_count, s->d_geom, s->d_col, s->d_cov, nullptr,
                                                       0, nullptr)));
  }
  SCR_CUDA(cudaGetLastError());
  s->cursor = (s->cursor + n) % s->L;
  SCR_CUDA(cudaStreamSynchronize(s->stream));
  return SCR_OK;
}

scr_status scr_debug_cluster(scr_scene s, const scr_entry* e, int n, scr_mode* out, int32_t* labels, int* n_modes) {
  if (!s || n < 0 || n > s->fp.capacity || !out || !n_modes) return SCR_E_ARG;
  SCR_CUDA(cudaSetDevice(s->dev->ordinal));
  // run the production kernel on a scratch "leaf" 0 of a private prediction table
  scr_entry* d_e = nullptr;
  int* d_lab = nullptr;
  int* d_cnt = nullptr;
  ModeGeom* d_g = nullptr;
  float4* d_c = nullptr;
  float* d_v = nullptr;
  SCR_CUDA(cudaMalloc(&d_e, std::max(1, n) * sizeof(scr_entry)));
  SCR_CUDA(cudaMalloc(&d_lab, std::max(1, n) * sizeof(int)));
  SCR_CUDA(cudaMalloc(&d_cnt, sizeof(int)));
  SCR_CUDA(cudaMalloc(&d_g, kMaxModes * sizeof(ModeGeom)));
  SCR_CUDA(cudaMalloc(&d_c, kMaxModes * sizeof(float4)));
  SCR_CUDA(cudaMalloc(&d_v, kMaxModes * 6 * sizeof(float)));
  if (n) SCR_CUDA(cudaMemcpy(d_e, e, n * sizeof(scr_entry), cudaMemcpyHostToDevice));
  RqsParams rp;
  rp.c = static_cast<float>(-1.0 / (2.0 * static_cast<double>(s->fp.sigma) * static_cast<double>(s->fp.sigma)));
  rp.tau2 = static_cast<float>(static_cast<double>(s->fp.tau) * static_cast<double>(s->fp.tau));
  rp.min_size = s->fp.min_cluster_size;
  rp.max_clusters = s->fp.max_clusters;
  rp.kappa = s->fp.capacity;
  const size_t smem = rqs_smem(rp.kappa);
  k_rqs<<<1, kRqsThreads, smem, s->stream>>>(nullptr, nullptr, 1, 0, 1, rp, d_cnt, d_g, d_c, d_v, d_e, n, d_lab);
  SCR_CUDA(cudaGetLastError());
  SCR_CUDA(cudaStreamSynchronize(s->stream));
  int cnt = 0;
  SCR_CUDA(cudaMemcpy(&cnt, d_cnt, sizeof(int), cudaMemcpyDeviceToHost));
  std::vector<ModeGeom> g(kMaxModes);
  std::vector<float4> c(kMaxModes);
  std::vector<float> v(kMaxModes * 6);
  SCR_CUDA(cudaMemcpy(g.data(), d_g, kMaxModes * sizeof(ModeGeom), cudaMemcpyDeviceToHost));
  SCR_CUDA(cudaMemcpy(c.data(), d_c, kMaxModes * sizeof(float4), cudaMemcpyDeviceToHost));
  SCR_CUDA(cudaMemcpy(v.data(), d_v, kMaxModes * 6 * sizeof(float), cudaMemcpyDeviceToHost));
  if (labels && n) SCR_CUDA(cudaMemcpy(labels, d_lab, n * sizeof(int), cudaMemcpyDeviceToHost));
  for (int i = 0; i < cnt; ++i) {
    scr_mode& m = out[i];
    m.mu[0] = g[i].q0.x; m.mu[1] = g[i].q0.y; m.mu[2] = g[i].q0.z;
    m.colour[0] = c[i].x; m.colour[1] = c[i].y; m.colour[2] = c[i].z;
    for (int q = 0; q < 6; ++q) m.cov[q] = v[6 * i + q];
    m.icov[0] = g[i].q0.w; m.icov[1] = g[i].q1.x; m.icov[2] = g[i].q1.y;
    m.icov[3] = g[i].q1.z; m.icov[4] = g[i].q1.w; m.icov[5] = g[i].q2.x;
    m.isqrt[0] = g[i].q2.y; m.isqrt[1] = g[i].q2.z; m.isqrt[2] = g[i].q2.w;
    m.isqrt[3] = g[i].q3.x; m.isqrt[4] = g[i].q3.y; m.isqrt[5] = g[i].q3.z;
    std::memcpy(&m.size, &c[i].w, 4);
  }
  *n_modes = cnt;
  cudaFree(d_e); cudaFree(d_lab); cudaFree(d_cnt); cudaFree(d_g); cudaFree(d_c); cudaFree(d_v);
  return SCR_OK;
}

scr_status scr_dump_seen(scr_scene s, uint32_t* out) {
  if (!s || !out) return SCR_E_ARG;
  SCR_CUDA(cudaSetDevice(s->dev->ordinal));
  SCR_TRY(refresh_lane(s));
  SCR_CUDA(cudaStreamSynchronize(s->stream));
  SCR_CUDA(cudaMemcpy(out, s->d_seen, s->L * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  return SCR_OK;
}

scr_status scr_dump_entries(scr_scene s, int64_t slot0, int64_t nslots, scr_entry* out) {
  if (!s || !out || slot0 < 0 || nslots < 0 || slot0 + nslots > s->L) return SCR_E_ARG;
  SCR_CUDA(cudaSetDevice(s->dev->ordinal));
  SCR_TRY(refresh_lane(s));
  SCR_CUDA(cudaStreamSynchronize(s->stream));
  SCR_CUDA(cudaMemcpy(out, s->d_entries + slot0 * s->fp.capacity,
                      static_cast<size_t>(nslots) * s->fp.capacity * sizeof(scr_entry), cudaMemcpyDeviceToHost));
  return SCR_OK;
}

scr_status scr_dump_predictions(scr_scene s, int32_t* counts, scr_mode* modes) {
  if (!s || !counts) return SCR_E_ARG;
  StateReadLock lock(s);
  SCR_CUDA(cudaSetDevice(s->dev->ordinal));
  SCR_TRY(refresh_lane(s));
  SCR_CUDA(cudaStreamSynchronize(s->stream));
  SCR_CUDA(cudaMemcpy(counts, s->d_count, s->L * sizeof(int), cudaMemcpyDeviceToHost));
  if (!modes) return SCR_OK;
  const size_t M = static_cast<size_t>(s->L) * kMaxModes;
  std::vector<ModeGeom> g(M);
  std::vector<float4> c(M);
  std::vector<float> v(M * 6);
  SCR_CUDA(cudaMemcpy(g.data(), s->d_geom, M * sizeof(ModeGeom), cudaMemcpyDeviceToHost));
  SCR_CUDA(cudaMemcpy(c.data(), s->d_col, M * sizeof(float4), cudaMemcpyDeviceToHost));
  SCR_CUDA(cudaMemcpy(v.data(), s->d_cov, M * 6 * sizeof(float), cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < M; ++i) {
    scr_mode& m = modes[i];
    m.mu[0] = g[i].q0.x; m.mu[1] = g[i].q0.y; m.mu[2] = g[i].q0.z;
    m.colour[0] = c[i].x; m.colour[1] = c[i].y; m.colour[2] = c[i].z;
    for (int q = 0; q < 6; ++q) m.cov[q] = v[6 * i + q];
    m.icov[0] = g[i].q0.w; m.icov[1] = g[i].q1.x; m.icov[2] = g[i].q1.y;
    m.icov[3] = g[i].q1.z; m.icov[4] = g[i].q1.w; m.icov[5] = g[i].q2.x;
    m.isqrt[0] = g[i].q2.y; m.isqrt[1] = g[i].q2.z; m.isqrt[2] = g[i].q2.w;
    m.isqrt[3] = g[i].q3.x; m.isqrt[4] = g[i].q3.y; m.isqrt[5] = g[i].q3.z;
    std::memcpy(&m.size, &c[i].w, 4);
  }
  return SCR_OK;
}

static scr_status scr_load_predictions_impl(scr_scene s, const int32_t* counts, const scr_mode* modes) {
  if (!s || !counts || !modes) return SCR_E_ARG;
  for (int64_t i = 0; i < s->L; ++i)
    if (counts[i] < 0 || counts[i] > s->fp.max_clusters) {
      set_error("scr_load_predictions: leaf " + std::to_string(i) + " has " + std::to_string(counts[i]) +
                " modes (0.." + std::to_string(s->fp.max_clusters) + " allowed)");
      return SCR_E_MALFORMED_DATA;
    }
  SCR_CUDA(cudaSetDevice(s->dev->ordinal));
  const size_t M = static_cast<size_t>(s->L) * kMaxModes;
  std::vector<ModeGeom> g(M);
  std::vector<float4> c(M);
  std::vector<float> v(M * 6);
  for (size_t i = 0; i < M; ++i) {
    const scr_mode& m = modes[i];
    g[i].q0 = make_float4(m.mu[0], m.mu[1], m.mu[2], m.icov[0]);
    g[i].q1 = make_float4(m.icov[1], m.icov[2], m.icov[3], m.icov[4]);
    g[i].q2 = make_float4(m.icov[5], m.isqrt[0], m.isqrt[1], m.isqrt[2]);
    g[i].q3 = make_float4(m.isqrt[3], m.isqrt[4], m.isqrt[5], 0.0f);
    float sz;
    std::memcpy(&sz, &m.size, 4);
    c[i] = make_float4(m.colour[0], m.colour[1], m.colour[2], sz);
    for (int q = 0; q < 6; ++q) v[6 * i + q] = m.cov[q];
  }
  // stream-ordered copies (the scene's stream does not synchronise with the legacy default
  // stream); synchronised before the pageable sources go out of scope
  SCR_CUDA(cudaMemcpyAsync(s->d_count, counts, s->L * sizeof(int), cudaMemcpyHostToDevice, s->stream));
  SCR_CUDA(cudaMemcpyAsync(s->d_geom, g.data(), M * sizeof(ModeGeom), cudaMemcpyHostToDevice, s->stream));
  SCR_CUDA(cudaMemcpyAsync(s->d_col, c.data(), M * sizeof(float4), cudaMemcpyHostToDevice, s->stream));
  SCR_CUDA(cudaMemcpyAsync(s->d_cov, v.data(), M * 6 * sizeof(float), cudaMemcpyHostToDevice, s->stream));
  SCR_CUDA(cudaStreamSynchronize(s->stream));
  return SCR_OK;
}

size_t scr_predictions_bytes(scr_scene s) {
  if (!s) return 0;
  const size_t M = static_cast<size_t>(s->L) * kMaxModes;
  return s->L * sizeof(int) + M * (sizeof(ModeGeom) + sizeof(float4) + 6 * sizeof(float));
}

scr_status scr_predictions_export(scr_scene s, void* dst) {
  if (!s || !dst) return SCR_E_ARG;
  StateReadLock lock(s);
  SCR_CUDA(cudaSetDevice(s->dev->ordinal));
  SCR_TRY(refresh_lane(s));
  const size_t M = static_cast<size_t>(s->L) * kMaxModes;
  char* p = static_cast<char*>(dst);
  SCR_CUDA(cudaMemcpyAsync(p, s->d_count, s->L * sizeof(int), cudaMemcpyDeviceToDevice, s->stream));
  p += s->L * sizeof(int);
  SCR_CUDA(cudaMemcpyAsync(p, s->d_geom, M * sizeof(ModeGeom), cudaMemcpyDeviceToDevice, s->stream));
  p += M * sizeof(ModeGeom);
  SCR_CUDA(cudaMemcpyAsync(p, s->d_col, M * sizeof(float4), cudaMemcpyDeviceToDevice, s->stream));
  p += M * sizeof(float4);
  SCR_CUDA(cudaMemcpyAsync(p, s->d_cov, M * 6 * sizeof(float), cudaMemcpyDeviceToDevice, s->stream));
  SCR_CUDA(cudaStreamSynchronize(s->stream));
  return SCR_OK;
}

// NCCL, resolved at run time so the library has no link-time dependency on it.
struct NcclApi {
  bool ok = false;
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*bcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

static const NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.comm_init_all = reinterpret_cast<decltype(api.comm_init_all)>(dlsym(h, "ncclCommInitAll"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.bcast = reinterpret_cast<decltype(api.bcast)>(dlsym(h, "ncclBroadcast"));
    api.group_start = reinterpret_cast<decltype(api.group_start)>(dlsym(h, "ncclGroupStart"));
    api.group_end = reinterpret_cast<decltype(api.group_end)>(dlsym(h, "ncclGroupEnd"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.comm_init_all && api.comm_destroy && api.bcast && api.group_start && api.group_end &&
             api.error_string;
  });
  return api;
}

// Counts outside [0, max_clusters] would index past a leaf's modes (or overflow the 6-bit
// per-tree counts of the K1 records): flagged on the device before a table is accepted.
__global__ void k_check_counts(const int* __restrict__ counts, int64_t L, int max_clusters, int* __restrict__ bad) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < L;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (counts[i] < 0 || counts[i] > max_clusters) atomicAdd(bad, 1);
}

static scr_status scr_predictions_import_impl(scr_scene s, const void* src) {
  if (!s || !src) return SCR_E_ARG;
  SCR_CUDA(cudaSetDevice(s->dev->ordinal));
  {
    int* d_bad = nullptr;
    int bad = 0;
    SCR_CUDA(cudaMallocAsync(&d_bad, sizeof(int), s->stream));
    SCR_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int), s->stream));
    k_check_counts<<<148, 256, 0, s->stream>>>(static_cast<const int*>(src), s->L, s->fp.max_clusters, d_bad);
    SCR_CUDA(cudaGetLastError());
    SCR_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, s->stream));
    SCR_CUDA(cudaFreeAsync(d_bad, s->stream));
    SCR_CUDA(cudaStreamSynchronize(s->stream));
    if (bad) {
      set_error("scr_predictions_import: " + std::to_string(bad) + " leaves with a mode count outside [0, " +
                std::to_string(s->fp.max_clusters) + "]");
      return SCR_E_MALFORMED_DATA;
    }
  }
  const size_t M = static_cast<size_t>(s->L) * kMaxModes;
  const char* p = static_cast<const char*>(src);
  SCR_CUDA(cudaMemcpyAsync(s->d_count, p, s->L * sizeof(int), cudaMemcpyDeviceToDevice, s->stream));
  p += s->L * sizeof(int);
  SCR_CUDA(cudaMemcpyAsync(s->d_geom, p, M * sizeof(ModeGeom), cudaMemcpyDeviceToDevice, s->stream));
  p += M * sizeof(ModeGeom);
  SCR_CUDA(cudaMemcpyAsync(s->d_col, p, M * sizeof(float4), cudaMemcpyDeviceToDevice, s->stream));
  p += M * sizeof(float4);
  SCR_CUDA(cudaMemcpyAsync(s->d_cov, p, M * 6 * sizeof(float), cudaMemcpyDeviceToDevice, s->stream));
  SCR_CUDA(cudaStreamSynchronize(s->stream));
  return SCR_OK;
}

scr_status scr_debug_leaves(scr_scene s, const scr_frame* f, int32_t* grid_px, int32_t* leaves, int* n_grid) {
  if (!s || !f || !n_grid) return SCR_E_ARG;
  SCR_TRY(check_frames(s, f, 1));
  StateReadLock lock(s);
  SCR_CUDA(cudaSetDevice(s->dev->ordinal));
  SCR_TRY(refresh_lane(s));
  SCR_TRY(upload_frames(s, f, 1));
  SCR_TRY(pack_frames(s, s->ws.depth, s->ws.rgb, nullptr, 1));
  int G = 0;
  SCR_CUDA(cudaMemcpyAsync(&G, s->ws.gcount, sizeof(int), cudaMemcpyDeviceToHost, s->stream));
  SCR_CUDA(cudaStreamSynchronize(s->stream));
  *n_grid = G;
  if (grid_px) SCR_CUDA(cudaMemcpy(grid_px, s->ws.gpx, G * sizeof(int), cudaMemcpyDeviceToHost));
  if (leaves) {
    std::vector<int> sl(static_cast<size_t>(G) * s->T);
    if (G) SCR_CUDA(cudaMemcpy(sl.data(), s->ws.gslot, sl.size() * sizeof(int), cudaMemcpyDeviceToHost));
    for (int g = 0; g < G; ++g)
      for (int t = 0; t < s->T; ++t) leaves[g * s->T + t] = sl[g * s->T + t] - s->leaf_base[t];
  }
  return SCR_OK;
}

scr_status scr_debug_features(scr_scene s, const scr_frame* f, const int32_t* px, int n, float* out) {
  if (!s || !f || !px || !out || n < 0) return SCR_E_ARG;
  SCR_TRY(check_frames(s, f, 1));
  StateReadLock lock(s);
  SCR_CUDA(cudaSetDevice(s->dev->ordinal));
  SCR_TRY(refresh_lane(s));
  SCR_TRY(upload_frames(s, f, 1));
  SCR_TRY(pack_frames(s, s->ws.depth, s->ws.rgb, nullptr, 1));
  int* d_px = nullptr;
  float* d_out = nullptr;
  SCR_CUDA(cudaMalloc(&d_px, std::max(1, n) * sizeof(int)));
  SCR_CUDA(cudaMalloc(&d_out, std::max(1, n) * kFeatures * sizeof(float)));
  SCR_CUDA(cudaMemcpy(d_px, px, n * sizeof(int), cudaMemcpyHostToDevice));
  if (n) k_features<<<n, kFeatures, 0, s->stream>>>(s->forest_view(), s->geom, s->ws.tex, d_px, n, d_out);
  SCR_CUDA(cudaGetLastError());
  SCR_CUDA(cudaStreamSynchronize(s->stream));
  SCR_CUDA(cudaMemcpy(out, d_out, static_cast<size_t>(n) * kFeatures * sizeof(float), cudaMemcpyDeviceToHost));
  cudaFree(d_px);
  cudaFree(d_out);
  for (int i = 0; i < n; ++i) {
    const int x = px[i] & 0xffff, y = px[i] >> 16;
    if (x >= s->k.width || y >= s->k.height) {
      set_error("compute_feature: pixel out of bounds");
      return SCR_E_INVALID_CENTRE_PIXEL;
    }
    const float d = f->depth[static_cast<size_t>(y) * s->k.width + x];
    if (!(d > 0.0f && d <= kMaxValidDepth)) {
      set_error("compute_feature: invalid depth at centre pixel");
      return SCR_E_INVALID_CENTRE_PIXEL;
    }
  }
  return SCR_OK;
}

// ---- frame sets ----
scr_status scr_frameset_create(scr_scene s, int cap, scr_frameset* out) {
  if (!s || cap <= 0 || !out) return SCR_E_ARG;
  SCR_CUDA(cudaSetDevice(s->dev->ordinal));
  scr_frameset fs = new scr_frameset_s();
  fs->scene = s;
  fs->cap = cap;
  const size_t WH = static_cast<size_t>(s->k.width) * s->k.height;
  cudaError_t e = cudaMalloc(&fs->depth, cap * WH * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&fs->rgb, cap * WH * 3);
  if (e != cudaSuccess) {
    scr_frameset_destroy(fs);
    return cuda_fail(e, "scr_frameset_create");
  }
  *out = fs;
  return SCR_OK;
}

void scr_frameset_destroy(scr_frameset fs) {
  if (!fs) return;
  cudaSetDevice(fs->scene->dev->ordinal);
  cudaStreamSynchronize(fs->scene->stream);
  if (fs->depth) cudaFree(fs->depth);
  if (fs->rgb) cudaFree(fs->rgb);
  delete fs;
}

scr_status scr_frameset_upload(scr_frameset fs, int first, const scr_frame* frames, int n) {
  if (!fs || first < 0 || n < 0 || first + n > fs->cap) return SCR_E_ARG;
  scr_scene s = fs->scene;
  SCR_TRY(check_frames(s, frames, n));
  SCR_CUDA(cudaSetDevice(s->dev->ordinal));
  const size_t WH = static_cast<size_t>(s->k.width) * s->k.height;
  for (int i = 0; i < n; ++i) {
    SCR_CUDA(cudaMemcpyAsync(fs->depth + (first + i) * WH, frames[i].depth, WH * sizeof(float), cudaMemcpyHostToDevice,
                             s->stream));
    SCR_CUDA(cudaMemcpyAsync(fs->rgb + (first + i) * WH * 3, frames[i].rgb, WH * 3, cudaMemcpyHostToDevice, s->stream));
  }
  SCR_CUDA(cudaStreamSynchronize(s->stream));
  return SCR_OK;
}

scr_status scr_frameset_render(scr_frameset fs, int first, const scr_pose* poses, int n) {
  if (!fs || first < 0 || n < 0 || first + n > fs->cap || !poses) return SCR_E_ARG;
  scr_scene s = fs->scene;
  if (!(s->parent ? (s->parent->d_prims || s->parent->tsdf_model) : (s->d_prims || s->tsdf_model))) {
    set_error("scr_frameset_render: no analytic model set");
    return SCR_E_ARG;
  }
  StateReadLock lock(fs->scene);
  SCR_CUDA(cudaSetDevice(s->dev->ordinal));
  SCR_TRY(refresh_lane(s));
  const size_t WH = static_cast<size_t>(s->k.width) * s->k.height;
  Pose* d_p = nullptr;
  SCR_CUDA(cudaMalloc(&d_p, std::max(1, n) * sizeof(Pose)));
  SCR_CUDA(cudaMemcpy(d_p, poses, n * sizeof(Pose), cudaMemcpyHostToDevice));
  for (int c0 = 0; c0 < n; c0 += 65535) {
    const int c = std::min(65535, n - c0);
    SCR_LAUNCH(s, K_RENDER,
               (k_render<<<dim3(64, c), 256, 0, s->stream>>>(s->d_prims, s->n_prims, s->geom, d_p + c0,
                                                             fs->depth + (first + c0) * WH,
                                                             fs->rgb + (first + c0) * WH * 3)));
  }
  SCR_CUDA(cudaGetLastError());
  SCR_CUDA(cudaStreamSynchronize(s->stream));
  cudaFree(d_p);
  return SCR_OK;
}

scr_status scr_frameset_download(scr_frameset fs, int first, int n, float* depth, uint8_t* rgb) {
  if (!fs || first < 0 || n < 0 || first + n > fs->cap) return SCR_E_ARG;
  scr_scene s = fs->scene;
  SCR_CUDA(cudaSetDevice(s->dev->ordinal));
  SCR_CUDA(cudaStreamSynchronize(s->stream));
  const size_t WH = static_cast<size_t>(s->k.width) * s->k.height;
  if (depth) SCR_CUDA(cudaMemcpy(depth, fs->depth + first * WH, n * WH * sizeof(float), cudaMemcpyDeviceToHost));
  if (rgb) SCR_CUDA(cudaMemcpy(rgb, fs->rgb + first * WH * 3, n * WH * 3, cudaMemcpyDeviceToHost));
  return SCR_OK;
}

static scr_status scr_scene_set_tsdf_model_impl(scr_scene s, scr_tsdf v) {
  if (!s) return SCR_E_ARG;
  SCR_CUDA(cudaSetDevice(s->dev->ordinal));
  SCR_CUDA(cudaStreamSynchronize(s->stream));
  s->tsdf_model = v;
  return SCR_OK;
}

scr_status scr_scene_set_tsdf_model(scr_scene s, scr_tsdf v) {
  if (s && s->parent) {
    set_error("scr_scene_set_tsdf_model: a relocalisation lane is read-only; set the model on its scene");
    return SCR_E_ARG;
  }
  StateWriteLock lock(s);
  scr_status st = scr_scene_set_tsdf_model_impl(s, v);
  if (st == SCR_OK && s) st = publish(s);
  return st;
}

// Updates of shared scene state: refused on lanes, published to lanes when done.
scr_status scr_scene_set_analytic_model(scr_scene s, const scr_prim* prims, int n) {
  if (s && s->parent) {
    set_error("scr_scene_set_analytic_model: a relocalisation lane is read-only; update the scene it was forked from");
    return SCR_E_ARG;
  }
  StateWriteLock lock(s);
  scr_status st = scr_scene_set_analytic_model_impl(s, prims, n);
  if (st == SCR_OK && s) st = publish(s);
  return st;
}

scr_status scr_reset(scr_scene s) {
  if (s && s->parent) {
    set_error("scr_reset: a relocalisation lane is read-only; update the scene it was forked from");
    return SCR_E_ARG;
  }
  StateWriteLock lock(s);
  scr_status st = scr_reset_impl(s);
  if (st == SCR_OK && s) st = publish(s);
  return st;
}

scr_status scr_train_batch(scr_scene s, const scr_frame* frames, const scr_pose* poses, int n) {
  if (s && s->parent) {
    set_error("scr_train_batch: a relocalisation lane is read-only; update the scene it was forked from");
    return SCR_E_ARG;
  }
  scr_status st = scr_train_batch_impl(s, frames, poses, n);
  if (st == SCR_OK && s) st = publish(s);
  return st;
}

scr_status scr_train_frameset(scr_scene s, scr_frameset fs, const int32_t* idx, const scr_pose* poses, int n) {
  if (s && s->parent) {
    set_error("scr_train_frameset: a relocalisation lane is read-only; update the scene it was forked from");
    return SCR_E_ARG;
  }
  scr_status st = scr_train_frameset_impl(s, fs, idx, poses, n);
  if (st == SCR_OK && s) st = publish(s);
  return st;
}

scr_status scr_update(scr_scene s, int64_t leaves_per_call) {
  if (s && s->parent) {
    set_error("scr_update: a relocalisation lane is read-only; update the scene it was forked from");
    return SCR_E_ARG;
  }
  StateWriteLock lock(s);
  scr_status st = scr_update_impl(s, leaves_per_call);
  if (st == SCR_OK && s) st = publish(s);
  return st;
}

scr_status scr_load_predictions(scr_scene s, const int32_t* counts, const scr_mode* modes) {
  if (s && s->parent) {
    set_error("scr_load_predictions: a relocalisation lane is read-only; update the scene it was forked from");
    return SCR_E_ARG;
  }
  StateWriteLock lock(s);
  scr_status st = scr_load_predictions_impl(s, counts, modes);
  if (st == SCR_OK && s) st = publish(s);
  return st;
}

scr_status scr_broadcast_predictions(scr_scene* per_gpu, int ngpu, int root) {
  if (!per_gpu || ngpu < 1 || root < 0 || root >= ngpu) {
    set_error("scr_broadcast_predictions: need ngpu >= 1 scenes and 0 <= root < ngpu");
    return SCR_E_ARG;
  }
  std::vector<int> devs(ngpu);
  for (int i = 0; i < ngpu; ++i) {
    const scr_scene s = per_gpu[i];
    if (!s || s->parent) {
      set_error("scr_broadcast_predictions: every entry must be a scene (not a relocalisation lane)");
      return SCR_E_ARG;
    }
    if (s->L != per_gpu[root]->L || s->T != per_gpu[root]->T) {
      set_error("scr_broadcast_predictions: scenes were created from different forests");
      return SCR_E_DIMENSION_MISMATCH;
    }
    devs[i] = s->dev->ordinal;
    for (int j = 0; j < i; ++j)
      if (devs[j] == devs[i]) {
        set_error("scr_broadcast_predictions: one scene per GPU (two entries share a device)");
        return SCR_E_ARG;
      }
  }
  if (ngpu == 1) return SCR_OK;
  std::vector<std::unique_ptr<StateWriteLock>> locks;  // receivers' tables are rewritten
  for (int i = 0; i < ngpu; ++i)
    if (i != root) locks.emplace_back(new StateWriteLock(per_gpu[i]));
  const NcclApi& nc = nccl_api();
  if (!nc.ok) {
    set_error("scr_broadcast_predictions: libnccl.so.2 could not be loaded");
    return SCR_E_CUDA;
  }
  // the root's table must be complete before the collective reads it
  SCR_CUDA(cudaSetDevice(devs[root]));
  SCR_CUDA(cudaStreamSynchronize(per_gpu[root]->stream));
  std::vector<ncclComm_t> comms(ngpu);
  ncclResult_t r = nc.comm_init_all(comms.data(), ngpu, devs.data());
  if (r != ncclSuccess) {
    set_error(std::string("ncclCommInitAll: ") + nc.error_string(r));
    return SCR_E_CUDA;
  }
  const size_t M = static_cast<size_t>(per_gpu[root]->L) * kMaxModes;
  auto run = [&]() -> ncclResult_t {
    for (int b = 0; b < 4; ++b) {
      ncclResult_t e = nc.group_start();
      if (e != ncclSuccess) return e;
      for (int i = 0; i < ngpu; ++i) {
        const scr_scene s = per_gpu[i];
        void* ptr = b == 0 ? static_cast<void*>(s->d_count)
                    : b == 1 ? static_cast<void*>(s->d_geom)
                    : b == 2 ? static_cast<void*>(s->d_col)
                             : static_cast<void*>(s->d_cov);
        const size_t bytes = b == 0 ? s->L * sizeof(int)
                             : b == 1 ? M * sizeof(ModeGeom)
                             : b == 2 ? M * sizeof(float4)
                                      : M * 6 * sizeof(float);
        cudaSetDevice(devs[i]);
        e = nc.bcast(ptr, ptr, bytes, ncclChar, root, comms[i], s->stream);
        if (e != ncclSuccess) {
          nc.group_end();
          return e;
        }
      }
      e = nc.group_end();
      if (e != ncclSuccess) return e;
    }
    return ncclSuccess;
  };
  r = run();
  scr_status st = SCR_OK;
  if (r != ncclSuccess) {
    set_error(std::string("ncclBroadcast: ") + nc.error_string(r));
    st = SCR_E_CUDA;
  }
  for (int i = 0; i < ngpu; ++i) {
    cudaSetDevice(devs[i]);
    if (cudaStreamSynchronize(per_gpu[i]->stream) != cudaSuccess && st == SCR_OK) {
      set_error("scr_broadcast_predictions: stream synchronisation failed");
      st = SCR_E_CUDA;
    }
    nc.comm_destroy(comms[i]);
  }
  if (st != SCR_OK) return st;
  for (int i = 0; i < ngpu; ++i)
    if (i != root) SCR_TRY(publish(per_gpu[i]));
  return SCR_OK;
}

scr_status scr_predictions_import(scr_scene s, const void* src) {
  if (s && s->parent) {
    set_error("scr_predictions_import: a relocalisation lane is read-only; update the scene it was forked from");
    return SCR_E_ARG;
  }
  StateWriteLock lock(s);
  scr_status st = scr_predictions_import_impl(s, src);
  if (st == SCR_OK && s) st = publish(s);
  return st;
}

}  // extern "C"

// ORACLE — test infrastructure only. C entry points for ctypes (tests/, bench.py's
// cpu_baseline and --impl reference legs). Struct layouts mirror include/screloc_gpu.h
// (declared independently here so the oracle never includes product headers).
#include <atomic>
#include <chrono>
#include <cstring>
#include <string>
#include <thread>

#include "detmath.hpp"
#include "oracle.hpp"

using namespace oracle;

extern "C" {

typedef struct { int32_t width, height; double fx, fy, cx, cy; } or_intrinsics;
typedef struct { double R[9]; double t[3]; } or_pose;
typedef struct {
  int32_t max_gen_iters, n_max, n_cull, eta, pose_update, use_cov;
  double min_sq_dist;
  float colour_thresh, pad0;
  double rigidity_tol;
  int32_t n_out, pad1;
} or_ransac_params;
typedef struct {
  int32_t has_pose, status;
  or_pose pose;
  double score;
  int32_t stage_used, n_candidates;
  float stage_ms[4];
} or_result;
typedef struct { float mu[3], colour[3], cov[6], icov[6], isqrt[6]; int32_t size; } or_mode;
typedef struct { int32_t type; float a[3], b[3], colour[3], cell; uint32_t tex_seed; } or_prim;

}  // extern "C"

static_assert(sizeof(or_intrinsics) == 40, "layout");
static_assert(sizeof(or_pose) == 96, "layout");
static_assert(sizeof(or_ransac_params) == 56, "layout");
static_assert(sizeof(or_result) == 136, "layout");
static_assert(sizeof(or_mode) == 100, "layout");
static_assert(sizeof(or_prim) == 48, "layout");
static_assert(sizeof(Mode) == sizeof(or_mode), "layout");
static_assert(sizeof(Entry) == 16, "layout");

namespace {
thread_local std::string g_err;
Intrinsics to_k(const or_intrinsics& k) {
  Intrinsics o;
  o.fx = k.fx; o.fy = k.fy; o.cx = k.cx; o.cy = k.cy; o.width = k.width; o.height = k.height;
  return o;
}
Pose to_pose(const double* R, const double* t) {
  Pose p;
  std::memcpy(p.R, R, sizeof(p.R));
  std::memcpy(p.t, t, sizeof(p.t));
  return p;
}
Frame mk_frame(const float* depth, const uint8_t* rgb, const or_intrinsics& k, int reliable) {
  Frame f;
  f.width = k.width;
  f.height = k.height;
  f.depth = depth;
  f.rgb = rgb;
  f.k = to_k(k);
  f.pose_reliable = reliable != 0;
  return f;
}
RansacParams to_rp(const or_ransac_params& p) {
  RansacParams r;
  r.max_iters = p.max_gen_iters; r.n_max = p.n_max; r.n_cull = p.n_cull; r.eta = p.eta;
  r.pose_update = p.pose_update; r.use_cov = p.use_cov; r.min_sq_dist = p.min_sq_dist;
  r.colour_thresh = p.colour_thresh; r.rigidity_tol = p.rigidity_tol; r.n_out = p.n_out;
  return r;
}
void to_result(const RelocResult& r, or_result* o) {
  std::memset(o, 0, sizeof(*o));
  o->has_pose = r.has_pose;
  o->status = r.status;
  std::memcpy(o->pose.R, r.pose.R, sizeof(o->pose.R));
  std::memcpy(o->pose.t, r.pose.t, sizeof(o->pose.t));
  o->score = r.score;
  o->stage_used = r.stage_used;
  o->n_candidates = r.n_candidates;
}
template <typename F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return E_ARG;
  }
}
template <typename Fn>
void parallel_for(int n, int threads, Fn&& fn) {  // parallel.hpp:27-51 semantics
  if (threads <= 1 || n <= 1) {
    for (int i = 0; i < n; ++i) fn(i);
    return;
  }
  std::atomic<int> next{0};
  std::vector<std::thread> pool;
  for (int t = 0; t < std::min(threads, n); ++t)
    pool.emplace_back([&] {
      for (;;) {
        const int i = next.fetch_add(1);
        if (i >= n) return;
        fn(i);
      }
    });
  for (auto& th : pool) th.join();
}
}  // namespace

extern "C" {

const char* or_last_error() { return g_err.c_str(); }

// ---- rng / math kernels ------------------------------------------------------
void or_rng_u64(uint64_t seed, int use_stream, uint64_t tag, int n, uint64_t* out) {
  Rng r = use_stream ? Rng::stream(seed, tag) : Rng(seed);
  for (int i = 0; i < n; ++i) out[i] = r.next_u64();
}
void or_rng_uniform_int(uint64_t seed, int use_stream, uint64_t tag, uint64_t bound, int n, uint64_t* out) {
  Rng r = use_stream ? Rng::stream(seed, tag) : Rng(seed);
  for (int i = 0; i < n; ++i) out[i] = r.uniform_int(bound);
}
void or_rng_uniform(uint64_t seed, int use_stream, uint64_t tag, int n, double* out) {
  Rng r = use_stream ? Rng::stream(seed, tag) : Rng(seed);
  for (int i = 0; i < n; ++i) out[i] = r.uniform();
}
float or_det_expf(float x) { return det_expf(x); }
void or_det_sincos(double x, double* s, double* c) { det_sincos(x, s, c); }
void or_svd3(const double* A, double* U, double* S, double* V) { svd3_jacobi(A, U, S, V); }
void or_eig3(const double* A, double* ev, double* V) { eig3_jacobi(A, ev, V); }
int or_chol6(const double* M, const double* b, double* x) { return chol6_solve(M, b, x) ? 1 : 0; }

void or_exp_se3(const double* tw, or_pose* out) {
  const Pose p = exp_se3(tw);
  std::memcpy(out->R, p.R, sizeof(p.R));
  std::memcpy(out->t, p.t, sizeof(p.t));
}
int or_log_se3(const or_pose* T, double* tw) {
  return guarded([&] {
    log_se3(to_pose(T->R, T->t), tw);
    return 0;
  });
}
int or_kabsch(const double* cam, const double* world, int n, or_pose* out) {
  Pose p;
  if (!kabsch(cam, world, n, &p)) return 0;
  std::memcpy(out->R, p.R, sizeof(p.R));
  std::memcpy(out->t, p.t, sizeof(p.t));
  return 1;
}
int or_backproject(int x, int y, double d, const or_intrinsics* k, double* out) {
  return guarded([&] {
    backproject(x, y, d, to_k(*k), out);
    return 0;
  });
}
void or_pose_error(const or_pose* e, const or_pose* g, double* terr, double* aerr) {
  pose_error(to_pose(e->R, e->t), to_pose(g->R, g->t), terr, aerr);
}
void or_compose(const or_pose* a, const or_pose* b, or_pose* out) {
  const Pose p = compose(to_pose(a->R, a->t), to_pose(b->R, b->t));
  std::memcpy(out, &p, sizeof(*out));
}
void or_invert(const or_pose* a, or_pose* out) {
  const Pose p = invert(to_pose(a->R, a->t));
  std::memcpy(out, &p, sizeof(*out));
}

// ---- features ----------------------------------------------------------------
void or_feature_specs(uint64_t seed, int radius, int32_t* out) {  // 256 x {kind, dx, dy, channel}
  const auto s = generate_feature_specs(seed, radius);
  for (int i = 0; i < kFeatureCount; ++i) {
    out[4 * i] = s[i].kind; out[4 * i + 1] = s[i].dx; out[4 * i + 2] = s[i].dy; out[4 * i + 3] = s[i].channel;
  }
}
int or_compute_feature(const float* depth, const uint8_t* rgb, int w, int h, int x, int y, const int32_t* spec,
                       float* out) {
  return guarded([&] {
    Frame f;
    f.width = w; f.height = h; f.depth = depth; f.rgb = rgb;
    FeatureSpec s;
    s.kind = spec[0]; s.dx = spec[1]; s.dy = spec[2]; s.channel = spec[3];
    *out = compute_feature(f, x, y, s);
    return 0;
  });
}
int or_grid(const float* depth, int w, int h, int spacing, int32_t* out, int cap) {
  Frame f;
  f.width = w; f.height = h; f.depth = depth;
  const auto g = sample_grid_pixels(f, spacing);
  const int n = static_cast<int>(g.size());
  for (int i = 0; i < n && i < cap; ++i) out[i] = g[i];
  return n;
}

// ---- forest --------------------------------------------------------------------
void* or_forest_random(uint64_t seed, int height, double p, int trees, int radius) {
  return new Forest(generate_random_forest(seed, height, p, trees, radius));
}
void* or_forest_deserialize(const uint8_t* b, size_t n) {
  try {
    return new Forest(deserialize_forest(b, n));
  } catch (const Error& e) {
    g_err = e.what();
    return nullptr;
  }
}
size_t or_forest_serialize(void* f, uint8_t* out, size_t cap) {
  const auto b = serialize_forest(*static_cast<Forest*>(f));
  if (out && cap >= b.size()) std::memcpy(out, b.data(), b.size());
  return b.size();
}
void or_forest_free(void* f) { delete static_cast<Forest*>(f); }
int64_t or_forest_total_leaves(void* f) { return static_cast<Forest*>(f)->total_leaves; }
int or_forest_trees(void* f) { return static_cast<int>(static_cast<Forest*>(f)->trees.size()); }
int or_forest_nodes(void* f, int t) { return static_cast<int>(static_cast<Forest*>(f)->trees[t].nodes.size()); }
void or_forest_dump_tree(void* f, int t, int32_t* out) {  // 5 ints per node (threshold bit-cast)
  const auto& nodes = static_cast<Forest*>(f)->trees[t].nodes;
  for (size_t i = 0; i < nodes.size(); ++i) {
    out[5 * i] = nodes[i].feature;
    std::memcpy(&out[5 * i + 1], &nodes[i].threshold, 4);
    out[5 * i + 2] = nodes[i].left; out[5 * i + 3] = nodes[i].right; out[5 * i + 4] = nodes[i].leaf_id;
  }
}
void or_forest_specs(void* f, int32_t* out) {
  const auto& s = static_cast<Forest*>(f)->specs;
  for (int i = 0; i < kFeatureCount; ++i) {
    out[4 * i] = s[i].kind; out[4 * i + 1] = s[i].dx; out[4 * i + 2] = s[i].dy; out[4 * i + 3] = s[i].channel;
  }
}
int or_forest_leaves(void* fp, const float* depth, const uint8_t* rgb, int w, int h, const int32_t* px, int n,
                     int32_t* out) {
  return guarded([&] {
    const Forest& f = *static_cast<Forest*>(fp);
    Frame fr;
    fr.width = w; fr.height = h; fr.depth = depth; fr.rgb = rgb;
    const int T = static_cast<int>(f.trees.size());
    for (int i = 0; i < n; ++i)
      for (int t = 0; t < T; ++t) out[i * T + t] = find_leaf(f.trees[t], fr, px[i] & 0xffff, px[i] >> 16, f.specs);
    return 0;
  });
}

// ---- scene ---------------------------------------------------------------------
// ---- TSDF model (oracle/tsdf.cpp) ----
void* or_tsdf_create(const float* origin, float voxel, int nx, int ny, int nz, float trunc) {
  return new Tsdf(tsdf_create(origin, voxel, nx, ny, nz, trunc));
}
void or_tsdf_free(void* v) { delete static_cast<Tsdf*>(v); }
void or_tsdf_fuse(void* v, const float* depth, const or_intrinsics* k, const or_pose* T) {
  tsdf_fuse(*static_cast<Tsdf*>(v), depth, to_k(*k), to_pose(T->R, T->t));
}
void or_tsdf_dump(void* v, float* tsdf, float* weight) {
  const Tsdf& t = *static_cast<Tsdf*>(v);
  std::copy(t.tsdf.begin(), t.tsdf.end(), tsdf);
  std::copy(t.weight.begin(), t.weight.end(), weight);
}
void or_tsdf_raycast(void* v, const or_pose* T, const or_intrinsics* k, float* depth, uint32_t* nrm) {
  const Tsdf& t = *static_cast<Tsdf*>(v);
  const Pose P = to_pose(T->R, T->t);
  const Intrinsics K = to_k(*k);
  float R[9], tf[3];
  for (int i = 0; i < 9; ++i) R[i] = static_cast<float>(P.R[i]);
  for (int i = 0; i < 3; ++i) tf[i] = static_cast<float>(P.t[i]);
  for (int y = 0; y < K.height; ++y)
    for (int x = 0; x < K.width; ++x) {
      float d = 0.0f;
      uint32_t n = 0xffffffffu;
      if (!tsdf_raycast_pixel(t, R, tf, K, x, y, &d, &n)) d = 0.0f;
      depth[static_cast<size_t>(y) * K.width + x] = d;
      if (nrm) nrm[static_cast<size_t>(y) * K.width + x] = n;
    }
}
// the scene's ICP / ranking model becomes the volume (nullptr: back to the analytic model)
void or_scene_set_tsdf(void* scene, void* v) { static_cast<Scene*>(scene)->tsdf = static_cast<const Tsdf*>(v); }

void* or_scene_generate(uint64_t seed, int complexity) { return new Scene(generate_synthetic_scene(seed, complexity)); }
void* or_scene_from_prims(const or_prim* p, int n) {
  Scene* s = new Scene();
  for (int i = 0; i < n; ++i) {
    Prim q;
    q.type = p[i].type;
    for (int k = 0; k < 3; ++k) { q.a[k] = p[i].a[k]; q.b[k] = p[i].b[k]; q.colour[k] = p[i].colour[k]; }
    q.cell = p[i].cell;
    q.tex_seed = p[i].tex_seed;
    s->prims.push_back(q);
  }
  return s;
}
void or_scene_free(void* s) { delete static_cast<Scene*>(s); }
int or_scene_prims(void* sp, or_prim* out, int cap) {
  const Scene& s = *static_cast<Scene*>(sp);
  const int n = static_cast<int>(s.prims.size());
  for (int i = 0; i < n && i < cap; ++i) {
    out[i].type = s.prims[i].type;
    for (int k = 0; k < 3; ++k) { out[i].a[k] = s.prims[i].a[k]; out[i].b[k] = s.prims[i].b[k]; out[i].colour[k] = s.prims[i].colour[k]; }
    out[i].cell = s.prims[i].cell;
    out[i].tex_seed = s.prims[i].tex_seed;
  }
  return n;
}
void or_render(void* sp, const or_pose* T, const or_intrinsics* k, float* depth, uint8_t* rgb) {
  render_frame(*static_cast<Scene*>(sp), to_pose(T->R, T->t), to_k(*k), depth, rgb);
}
void or_render_batch(void* sp, const or_pose* T, int n, const or_intrinsics* k, float* depth, uint8_t* rgb,
                     int threads) {
  const size_t px = static_cast<size_t>(k->width) * k->height;
  parallel_for(n, threads, [&](int i) {
    render_frame(*static_cast<Scene*>(sp), to_pose(T[i].R, T[i].t), to_k(*k), depth + px * i, rgb + 3 * px * i);
  });
}
void or_trajectory(uint64_t seed, int n, int kind, or_pose* out) {
  std::vector<Pose> p(n);
  generate_trajectory(seed, n, kind, p.data());
  for (int i = 0; i < n; ++i) std::memcpy(&out[i], &p[i], sizeof(or_pose));
}

// ---- adaptation --------------------------------------------------------------------
void* or_state_create(void* fp, float sigma, float tau, int max_clusters, int min_size, int capacity, uint64_t seed) {
  AdaptState* s = new AdaptState();
  ForestParams p;
  p.sigma = sigma; p.tau = tau; p.max_clusters = max_clusters; p.min_cluster_size = min_size; p.capacity = capacity;
  init_state(*s, *static_cast<Forest*>(fp), p, seed);
  return s;
}
void or_state_free(void* s) { delete static_cast<AdaptState*>(s); }
int or_integrate(void* sp, void* fp, const float* depth, const uint8_t* rgb, const or_intrinsics* k, int reliable,
                 const or_pose* pose) {
  return guarded([&] {
    integrate_frame(*static_cast<AdaptState*>(sp), *static_cast<Forest*>(fp), mk_frame(depth, rgb, *k, reliable),
                    to_pose(pose->R, pose->t));
    return 0;
  });
}
void or_update(void* sp, int64_t n) { update_leaves_round_robin(*static_cast<AdaptState*>(sp), n); }
void or_update_all_parallel(void* sp, int threads) {  // every leaf once, parallel over leaves
  AdaptState& s = *static_cast<AdaptState*>(sp);
  const int kappa = s.params.capacity;
  parallel_for(static_cast<int>(s.total_leaves), threads, [&](int slot) {
    const int cnt = static_cast<int>(std::min<uint32_t>(s.seen[slot], static_cast<uint32_t>(kappa)));
    const auto m = cluster_reservoir(&s.entries[static_cast<size_t>(slot) * kappa], cnt, s.params);
    s.pred_count[slot] = static_cast<int32_t>(m.size());
    for (size_t q = 0; q < m.size(); ++q) s.modes[static_cast<size_t>(slot) * kMaxModes + q] = m[q];
  });
}
void or_clear(void* sp) { clear_adaptation(*static_cast<AdaptState*>(sp)); }
int64_t or_cursor(void* sp) { return static_cast<AdaptState*>(sp)->cursor; }
void or_dump_seen(void* sp, uint32_t* out) {
  const auto& s = *static_cast<AdaptState*>(sp);
  std::memcpy(out, s.seen.data(), s.seen.size() * 4);
}
void or_dump_entries(void* sp, int64_t slot0, int64_t nslots, void* out) {
  const auto& s = *static_cast<AdaptState*>(sp);
  std::memcpy(out, &s.entries[static_cast<size_t>(slot0) * s.params.capacity],
              static_cast<size_t>(nslots) * s.params.capacity * sizeof(Entry));
}
void or_dump_predictions(void* sp, int32_t* counts, or_mode* modes) {
  const auto& s = *static_cast<AdaptState*>(sp);
  std::memcpy(counts, s.pred_count.data(), s.pred_count.size() * 4);
  if (modes) std::memcpy(modes, s.modes.data(), s.modes.size() * sizeof(Mode));
}
void or_load_predictions(void* sp, const int32_t* counts, const or_mode* modes) {
  auto& s = *static_cast<AdaptState*>(sp);
  std::memcpy(s.pred_count.data(), counts, s.pred_count.size() * 4);
  std::memcpy(s.modes.data(), modes, s.modes.size() * sizeof(Mode));
}
int or_cluster(const void* entries, int n, float sigma, float tau, int min_size, int max_clusters, or_mode* out,
               int32_t* labels) {
  ForestParams p;
  p.sigma = sigma; p.tau = tau; p.min_cluster_size = min_size; p.max_clusters = max_clusters;
  std::vector<int> lab;
  const auto m = cluster_reservoir(static_cast<const Entry*>(entries), n, p, &lab);
  for (size_t i = 0; i < m.size(); ++i) std::memcpy(&out[i], &m[i], sizeof(or_mode));
  if (labels)
    for (int i = 0; i < n; ++i) labels[i] = lab[i];
  return static_cast<int>(m.size());
}

// ---- RANSAC / relocalisation -----------------------------------------------------
// Debug view of one preemptive_ransac call: generated hypotheses (slot order) and survivors.
int or_ransac(void* fp, void* sp, const float* depth, const uint8_t* rgb, const or_intrinsics* k,
              const or_ransac_params* rp, uint64_t seed, int32_t* gen_slots, or_pose* gen_poses, int* n_gen,
              int32_t* surv_slots, or_pose* surv_poses, float* surv_energy, int* n_surv) {
  return guarded([&] {
    const Frame fr = mk_frame(depth, rgb, *k, 1);
    FrameCtx c;
    build_frame_ctx(c, *static_cast<Forest*>(fp), *static_cast<AdaptState*>(sp), fr);
    std::vector<Hypothesis> gen;
    *n_gen = 0;
    *n_surv = 0;
    std::vector<Hypothesis> surv;
    int code = 0;
    try {
      surv = preemptive_ransac(c, *static_cast<AdaptState*>(sp), to_rp(*rp), seed, &gen);
    } catch (const Error& e) {
      code = e.code;
    }
    for (size_t i = 0; i < gen.size(); ++i) {
      gen_slots[i] = gen[i].slot;
      std::memcpy(&gen_poses[i], &gen[i].pose, sizeof(or_pose));
    }
    *n_gen = static_cast<int>(gen.size());
    for (size_t i = 0; i < surv.size(); ++i) {
      surv_slots[i] = surv[i].slot;
      std::memcpy(&surv_poses[i], &surv[i].pose, sizeof(or_pose));
      surv_energy[i] = surv[i].energy;
    }
    *n_surv = static_cast<int>(surv.size());
    return code;
  });
}
int or_relocalise(void* fp, void* sp, void* scene, const float* depth, const uint8_t* rgb, const or_intrinsics* k,
                  const or_ransac_params* rp, int mode, uint64_t seed, or_result* out) {
  return guarded([&] {
    const RelocResult r = relocalise(to_rp(*rp), mode, mk_frame(depth, rgb, *k, 1), *static_cast<Forest*>(fp),
                                     *static_cast<AdaptState*>(sp), *static_cast<Scene*>(scene), seed);
    to_result(r, out);
    return 0;
  });
}
// Frames i in [0, n): frame i = depth + i*W*H etc., seed_i = seeds[i]; parallel over frames.
int or_cascade_batch(void* fp, void* sp, void* scene, const float* depth, const uint8_t* rgb,
                     const or_intrinsics* k, int n, const or_ransac_params* stages, const int32_t* modes,
                     const double* thr, int nstages, const uint64_t* seeds, int threads, or_result* out) {
  return guarded([&] {
    std::vector<RansacParams> st;
    for (int i = 0; i < nstages; ++i) st.push_back(to_rp(stages[i]));
    const size_t px = static_cast<size_t>(k->width) * k->height;
    parallel_for(n, threads, [&](int i) {
      const Frame fr = mk_frame(depth + px * i, rgb + 3 * px * i, *k, 1);
      const auto t0 = std::chrono::steady_clock::now();
      const RelocResult r = run_cascade(st.data(), modes, thr, nstages, fr, *static_cast<Forest*>(fp),
                                        *static_cast<AdaptState*>(sp), *static_cast<Scene*>(scene), seeds[i]);
      to_result(r, &out[i]);
      out[i].stage_ms[0] =
          std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
    });
    return 0;
  });
}
int or_icp(void* scene, const float* depth, const uint8_t* rgb, const or_intrinsics* k, const or_pose* init,
           or_pose* out, int* converged, double* rms, double* inlier_frac) {
  return guarded([&] {
    const IcpResult r = icp_refine(*static_cast<Scene*>(scene), to_pose(init->R, init->t), mk_frame(depth, rgb, *k, 1));
    std::memcpy(out, &r.pose, sizeof(or_pose));
    *converged = r.converged;
    *rms = r.rms;
    *inlier_frac = r.inlier_frac;
    return 0;
  });
}
double or_depth_diff(void* scene, const float* depth, const uint8_t* rgb, const or_intrinsics* k, const or_pose* T) {
  return depth_diff_score(*static_cast<Scene*>(scene), to_pose(T->R, T->t), mk_frame(depth, rgb, *k, 1));
}
double or_depth_diff_images(const float* live, const float* synth, int w, int h) {
  return depth_diff_images(live, synth, w, h);
}
void or_raycast_depth(void* scene, const or_pose* T, const or_intrinsics* k, float* out) {
  raycast_depth(*static_cast<Scene*>(scene), to_pose(T->R, T->t), to_k(*k), out);
}
uint64_t or_stage_seed(uint64_t seed, int stage) { return stage_seed(seed, stage); }

}  // extern "C"

extern "C" {
// Eq. 5 energy of pose H over grid-sample indices (KAT hook).
int or_energy(void* fp, void* sp, const float* depth, const uint8_t* rgb, const or_intrinsics* k, const or_pose* H,
              const int32_t* samples, int n, float* out) {
  return guarded([&] {
    const Frame fr = mk_frame(depth, rgb, *k, 1);
    FrameCtx c;
    build_frame_ctx(c, *static_cast<Forest*>(fp), *static_cast<AdaptState*>(sp), fr);
    std::vector<int> s(samples, samples + n);
    *out = energy(c, *static_cast<AdaptState*>(sp), to_pose(H->R, H->t), s, n > 0 ? n : 1);
    return 0;
  });
}
// lm_refine of pose H over grid-sample indices (KAT hook); returns the final surrogate.
int or_lm(void* fp, void* sp, const float* depth, const uint8_t* rgb, const or_intrinsics* k, or_pose* H,
          const int32_t* samples, int n, int use_cov, double* surrogate) {
  return guarded([&] {
    const Frame fr = mk_frame(depth, rgb, *k, 1);
    FrameCtx c;
    build_frame_ctx(c, *static_cast<Forest*>(fp), *static_cast<AdaptState*>(sp), fr);
    std::vector<int> s(samples, samples + n);
    Pose P = to_pose(H->R, H->t);
    lm_refine(c, *static_cast<AdaptState*>(sp), P, s, use_cov != 0, surrogate);
    std::memcpy(H, &P, sizeof(or_pose));
    return 0;
  });
}
int or_grid_count(void* fp, void* sp, const float* depth, const uint8_t* rgb, const or_intrinsics* k, int32_t* nmodes,
                  int cap) {
  return guarded([&] {
    const Frame fr = mk_frame(depth, rgb, *k, 1);
    FrameCtx c;
    build_frame_ctx(c, *static_cast<Forest*>(fp), *static_cast<AdaptState*>(sp), fr);
    for (size_t i = 0; i < c.nmodes.size() && static_cast<int>(i) < cap; ++i) nmodes[i] = c.nmodes[i];
    return static_cast<int>(c.nmodes.size()) > cap ? -1 : 0;
  });
}
}

extern "C" {
// n consecutive integrate_frame calls; per frame the forest descent runs in parallel over
// grid pixels, the reservoir insertions stay in the sequential (pixel, tree) order.
int or_integrate_batch(void* sp, void* fp, const float* depth, const uint8_t* rgb, const or_intrinsics* k,
                       const or_pose* poses, int n, int threads) {
  return guarded([&] {
    AdaptState& s = *static_cast<AdaptState*>(sp);
    const Forest& f = *static_cast<Forest*>(fp);
    const size_t px = static_cast<size_t>(k->width) * k->height;
    const int T = static_cast<int>(f.trees.size());
    for (int i = 0; i < n; ++i) {
      const Frame fr = mk_frame(depth + px * i, rgb + 3 * px * i, *k, 1);
      const Pose pose = to_pose(poses[i].R, poses[i].t);
      const std::vector<int> grid = sample_grid_pixels(fr, 4);
      std::vector<int32_t> leaves(grid.size() * T);
      parallel_for(static_cast<int>(grid.size()), threads, [&](int g) {
        for (int t = 0; t < T; ++t)
          leaves[static_cast<size_t>(g) * T + t] = find_leaf(f.trees[t], fr, grid[g] & 0xffff, grid[g] >> 16, f.specs);
      });
      for (size_t g = 0; g < grid.size(); ++g) {
        const int x = grid[g] & 0xffff, y = grid[g] >> 16;
        const size_t idx = static_cast<size_t>(y) * fr.width + x;
        double pc[3], pw[3];
        backproject(x, y, static_cast<double>(fr.depth[idx]), fr.k, pc);
        transform_point(pose, pc, pw);
        const Entry e{static_cast<float>(pw[0]), static_cast<float>(pw[1]), static_cast<float>(pw[2]),
                      fr.rgb[3 * idx], fr.rgb[3 * idx + 1], fr.rgb[3 * idx + 2], 0};
        for (int t = 0; t < T; ++t) reservoir_insert(s, f.leaf_base[t] + leaves[g * T + t], e);
      }
    }
    return 0;
  });
}
}

extern "C" {
// Generation diagnostics (test/fixture infrastructure): runs generate_hypothesis for every
// slot of one frame and histograms the outcome of every attempt by rejection tag
// (tags[6] indexed by Reject: OK, NoModes, ColourCheckFailed, TooClose, NotRigid,
// DegenerateKabsch). With a ground-truth pose it also reports mode quality: the fraction
// of (grid pixel, predicted mode) pairs whose mean lies within `radius` of the pixel's
// true world point, and the fraction of moded grid pixels having at least one such mode.
int or_generation_stats(void* fp, void* sp, const float* depth, const uint8_t* rgb, const or_intrinsics* k,
                        const or_ransac_params* rp, uint64_t seed, const or_pose* gt, double radius, int64_t* tags,
                        int* slots_ok, double* mode_frac, double* pixel_frac) {
  return guarded([&] {
    const Frame fr = mk_frame(depth, rgb, *k, 1);
    const AdaptState& s = *static_cast<AdaptState*>(sp);
    FrameCtx c;
    build_frame_ctx(c, *static_cast<Forest*>(fp), s, fr);
    const RansacParams p = to_rp(*rp);
    for (int i = 0; i < 6; ++i) tags[i] = 0;
    *slots_ok = 0;
    for (int slot = 0; slot < p.n_max; ++slot) {
      Rng rng = Rng::stream(seed, static_cast<uint64_t>(slot));
      Pose h;
      int att = 0;
      if (generate_hypothesis(c, s, p, rng, &h, &att, tags) == REJ_OK) ++*slots_ok;
    }
    *mode_frac = *pixel_frac = 0.0;
    if (gt) {
      const Pose T = to_pose(gt->R, gt->t);
      int64_t good = 0, total = 0, px_good = 0, px_total = 0;
      for (size_t g = 0; g < c.grid.size(); ++g) {
        const int nm = c.nmodes[g];
        if (nm == 0) continue;
        double w[3];
        transform_point(T, &c.cam[3 * g], w);
        bool any = false;
        for (int m = 0; m < nm; ++m) {
          const Mode* md = ctx_mode(c, s, static_cast<int>(g), m);
          const double d0 = w[0] - md->mu[0], d1 = w[1] - md->mu[1], d2 = w[2] - md->mu[2];
          const bool ok = d0 * d0 + d1 * d1 + d2 * d2 <= radius * radius;
          good += ok;
          any = any || ok;
        }
        total += nm;
        px_good += any;
        ++px_total;
      }
      *mode_frac = total ? static_cast<double>(good) / total : 0.0;
      *pixel_frac = px_total ? static_cast<double>(px_good) / px_total : 0.0;
    }
    return 0;
  });
}
}

extern "C" {
// KAT hooks (test infrastructure): checks 2-3 + Kabsch of one explicit triplet, and the LM
// residual/Jacobian of one sample.
int or_check_triplet(const double* cm, const double* w, const or_ransac_params* rp, or_pose* out) {
  Pose T;
  const int tag = check_triplet(cm, w, to_rp(*rp), &T);
  if (tag == REJ_OK && out) {
    std::memcpy(out->R, T.R, sizeof(T.R));
    std::memcpy(out->t, T.t, sizeof(T.t));
  }
  return tag;
}
void or_lm_residual_jacobian(const or_pose* H, const double* x, const or_mode* m, int use_cov, double* r,
                             double* J) {
  double y[3], Jm[3][6];
  lm_residual_jacobian(to_pose(H->R, H->t), x, *reinterpret_cast<const Mode*>(m), use_cov != 0, r, J ? Jm : nullptr,
                       y);
  if (J)
    for (int i = 0; i < 3; ++i)
      for (int a = 0; a < 6; ++a) J[6 * i + a] = Jm[i][a];
}
}

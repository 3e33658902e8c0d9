// Host/device internal state of the screloc B200 library (not part of the ABI).
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <mutex>
#include <shared_mutex>
#include <vector>

#include "common.cuh"

namespace scr {

void set_error(const std::string& msg);
scr_status cuda_fail(cudaError_t e, const char* what);

#define SCR_CUDA(expr)                                           \
  do {                                                           \
    cudaError_t _e = (expr);                                     \
    if (_e != cudaSuccess) return ::scr::cuda_fail(_e, #expr);   \
  } while (0)

// ---- in-library profiler: CUDA events around every launch on the scene stream --------
enum KernelId {
  K_PACK, K_GRID, K_LEAVES, K_HYPGEN, K_SAMPLES, K_ENERGY, K_SELECT, K_LM, K_ICP, K_FINALIZE, K_INSERT, K_RQS,
  K_RENDER, K_COMPACT, K_HYPFIN, K_COUNT
};
// device work counters (u64), indexed by W_*; meaning documented in DESIGN.md "Roofline"
enum WorkId {
  W_MODE_EVALS, W_SAMPLE_EVALS, W_LM_TERMS, W_ICP_TERMS, W_RAYS, W_NODE_VISITS, W_GEN_ATTEMPTS, W_LM_ASSOC, W_RAY_PRIMS, W_COUNT
};

struct Profiler {
  bool on = false;
  struct Rec {
    int kid;
    cudaEvent_t a, b;
  };
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> pool;
  double ms[K_COUNT] = {};
  long long launches[K_COUNT] = {};
  unsigned long long* d_work = nullptr;
};

struct ForestView {
  const int4* nodes;     // {left, right|leaf_id, feature, threshold bits}; left < 0 marks a leaf
  const short4* specs;   // {dx, dy, kind, channel}
  int T;
  int node_base[kMaxTrees];
  int leaf_base[kMaxTrees];
};

struct FrameGeom {
  int W, H;
  float fx, fy, cx, cy;     // f32 copies (feature/raycast arithmetic)
  double dfx, dfy, dcx, dcy;  // f64 (backproject, geometry.hpp:198)
};

struct PredView {
  const int* count;
  const ModeGeom* geom;
  const float4* col;
};

// Per-batch device workspace (frames are addressed by workspace slot f in [0, cap)).
struct Workspace {
  int cap = 0;    // frames
  // per-call staging, allocated once: device results, pinned host mirrors, stage events
  scr_result* d_res = nullptr;  // [cap]
  scr_result* h_res = nullptr;  // pinned [cap]
  int* h_idx = nullptr;         // pinned [cap] stage frame list
  int* h_fsidx = nullptr;       // pinned [cap] frameset indices of a call
  uint64_t* h_seeds = nullptr;  // pinned [cap]
  cudaEvent_t ev_stage[2] = {nullptr, nullptr};
  cudaEvent_t ev_upload = nullptr;
  int gmax = 0;   // grid pixels per frame
  float* depth = nullptr;     // staging for host uploads [cap * WH]
  uint8_t* rgb = nullptr;     // [cap * WH * 3]
  float* depth2 = nullptr;    // second staging buffer (calls with more than cap frames)
  uint8_t* rgb2 = nullptr;
  cudaEvent_t ev_upload2 = nullptr;
  uint2* tex = nullptr;       // packed texels [cap * WH]: {depth or 0, rgb|valid<<24}
  float* dplane = nullptr;    // live depth (or 0) per ICP pyramid level, dense: [cap][WH + WH/4 + WH/16]
  int* gcount = nullptr;      // [cap]
  int* gpx = nullptr;         // [cap * gmax] packed x | y << 16
  float4* gcam = nullptr;     // [cap * gmax] camera point (f32 of the f64 backprojection)
  int* gslot = nullptr;       // [cap * gmax * T]
  int* gnm = nullptr;         // [cap * gmax] number of modes (union over trees)
  int4* grec = nullptr;       // [cap * gmax * 2] 32-B pixel records: {x|y<<16, depth bits, rgb | nm<<24,
                              // 6-bit counts of trees 0..4} then the 16-bit leaf ids of trees 0..7
  // RANSAC (grown on demand)
  int nmax_cap = 0, ncull_cap = 0, samples_cap = 0;
  Pose* hyp = nullptr;        // [cap * nmax]
  float* henergy = nullptr;   // [cap * nmax]
  int* hok = nullptr;         // [cap * nmax] 0 failed, 1 generated, 2 tentative (k_hypgen -> k_hypfin)
  int4* hcand = nullptr;      // [cap * nmax * 2] tentative triplet {attempt, g0, g1, g2}, {m0, m1, m2, -}
  int4* sus = nullptr;        // [cap * kMaxSuspects * 2] passing triplets whose Kabsch may be degenerate
  int* hiters = nullptr;      // [cap * nmax]
  Pose* hypc = nullptr;       // generated hypotheses compacted in slot order [cap * nmax]
  int* hslot = nullptr;       // their generation slots [cap * nmax]
  int* hvalid = nullptr;      // number generated per frame [cap]
  Pose* cand = nullptr;       // [cap * ncull]
  float* cenergy = nullptr;   // [cap * ncull]
  int* cslot = nullptr;       // [cap * ncull]
  int* ncand = nullptr;       // [cap]
  float* epart = nullptr;     // per-batch partial energies [cap * ncull * kEnergyBatches]
  void* lmst = nullptr;       // LM state per candidate [cap * ncull]
  int* samples = nullptr;     // [cap * samples_cap]
  int* assoc = nullptr;       // [cap * ncull * samples_cap]
  // ranking / ICP
  int icp_cap = 0;            // (frame, candidate) jobs resident at once
  uint2* icp_map = nullptr;   // [icp_cap * WH] {t bits, prim | face << 16}
  Pose* icp_pose = nullptr;   // [cap * ncull] refined poses
  double* icp_score = nullptr;  // [cap * ncull]
  int* icp_conv = nullptr;    // [cap * ncull]
  double* icp_rms = nullptr;
  double* icp_inl = nullptr;
  int* fidx = nullptr;        // active frame list [cap]
  uint64_t* seeds = nullptr;  // [cap]
  int* status = nullptr;      // [cap] frame-set indices for pack_frames
  int* hctr = nullptr;        // [2 * cap] per-frame generation slot counters, then suspect counts
  // reservoir insertion scratch (one frame)
  // reservoir insertion (K2): two stable radix sorts over the frame's gmax * T items
  int* ins_start = nullptr;        // [L] first sorted position of a leaf's insertions
  uint32_t* ins_key = nullptr;     // [items] leaf slot (padding: L)
  uint32_t* ins_key_s = nullptr;   // sorted
  int* ins_val = nullptr;          // [items] item = g * T + t
  int* ins_item = nullptr;         // sorted items
  int* ins_tgt = nullptr;          // [items] target entry per sorted position (-1: none)
  uint64_t* ins_key2 = nullptr;    // [items] slot * kappa + target (padding: L * kappa)
  uint64_t* ins_key2_s = nullptr;  // sorted
  int* ins_val2 = nullptr;         // [items] sorted position
  int* ins_pos2 = nullptr;         // positions in (slot, target) order
  void* ins_tmp = nullptr;         // radix-sort scratch
  size_t ins_tmp_bytes = 0;
};

}  // namespace scr

struct scr_device_s {
  int ordinal = 0;
  int sm_count = 148;
  // host->device frame uploads of every scene/lane on this GPU go through one copy stream,
  // each call's frames enqueued contiguously: one lane's upload overlaps the others' kernels
  cudaStream_t copy = nullptr;
  std::mutex copy_mu;
};

struct scr_scene_s {
  scr_device dev = nullptr;
  cudaStream_t stream = nullptr;
  scr_intrinsics k{};
  scr::FrameGeom geom{};
  scr_forest_params fp{};
  uint64_t adapt_seed = 0;
  int T = 0;
  int64_t L = 0;
  int64_t cursor = 0;
  std::vector<int> node_base, leaf_base;
  int gen_force_suspect = 0;  // scr_debug_generation_mode
  bool leaves16 = true;  // every tree has <= 65536 leaves (16-bit leaf ids in gleaf)
  int4* d_nodes = nullptr;
  short4* d_specs = nullptr;
  scr_entry* d_entries = nullptr;
  uint32_t* d_seen = nullptr;
  int* d_count = nullptr;
  scr::ModeGeom* d_geom = nullptr;
  float4* d_col = nullptr;
  float* d_cov = nullptr;   // 6 per mode (dumps only)
  scr::Prim* d_prims = nullptr;
  int n_prims = 0;
  scr_tsdf tsdf_model = nullptr;  // ICP / ranking model when set (else the analytic prims)
  scr::Workspace ws;
  // relocalisation lanes (scr_scene_fork): a lane shares the parent's read-only device
  // state (forest, predictions, model) and owns a stream + workspace of its own
  scr_scene_s* parent = nullptr;
  int lanes = 0;                      // live lanes forked from this scene
  cudaEvent_t published = nullptr;    // recorded after every update of shared state
  // Readers (relocalisation on the scene or any of its lanes) hold this shared for a whole
  // call, which returns only after its kernels finished; updates of what they read (RQS
  // refresh, reset, loaded/imported/broadcast predictions, scene model) hold it exclusively,
  // so no reader ever sees a half-written table or a freed model.
  std::shared_mutex state_mu;
  int64_t launches = 0;
  scr::Profiler prof;
  scr::ForestView forest_view() const;
  scr::PredView pred_view() const { return {d_count, d_geom, d_col}; }
};

struct scr_frameset_s {
  scr_scene scene = nullptr;
  int cap = 0;
  float* depth = nullptr;
  uint8_t* rgb = nullptr;
};

namespace scr {
cudaEvent_t prof_event(scr_scene s);
void prof_flush(scr_scene s);
inline unsigned long long* work_ptr(scr_scene s) { return s->prof.on ? s->prof.d_work : nullptr; }

// Launch wrapper: counts every launch and, when profiling, brackets it with events.
#define SCR_LAUNCH(s, kid, ...)                                   \
  do {                                                            \
    cudaEvent_t _ea = nullptr, _eb = nullptr;                     \
    if ((s)->prof.on) {                                           \
      _ea = ::scr::prof_event(s);                                 \
      _eb = ::scr::prof_event(s);                                 \
      cudaEventRecord(_ea, (s)->stream);                          \
    }                                                             \
    __VA_ARGS__;                                                  \
    if ((s)->prof.on) {                                           \
      cudaEventRecord(_eb, (s)->stream);                          \
      (s)->prof.pending.push_back({(kid), _ea, _eb});             \
    }                                                             \
    (s)->launches++;                                              \
    (s)->prof.launches[(kid)]++;                                  \
  } while (0)

// tsdf.cu
TsdfView tsdf_view(scr_tsdf v);
// scene.cu
scr_status refresh_lane(scr_scene s);
scr_status publish(scr_scene s);
scr_status pack_frames(scr_scene s, const float* depth_base, const uint8_t* rgb_base, const int* d_idx, int n);
scr_status ensure_ransac_ws(scr_scene s, int nmax, int ncull, int samples);
scr_status ensure_icp_ws(scr_scene s, int jobs);
// reloc.cu
scr_status reloc_init();
scr_status run_cascade(scr_scene s, int n, const scr_ransac_params* stages, const int32_t* modes,
                       const double* thr, int nstages, const uint64_t* seeds, scr_result* out);
scr_status run_ransac_debug(scr_scene s, const scr_ransac_params* p, uint64_t seed, int32_t* gen_slots,
                            scr_pose* gen_poses, int* n_gen, int32_t* surv_slots, scr_pose* surv_poses,
                            float* surv_energy, int* n_surv);
scr_status run_icp_debug(scr_scene s, const scr_pose* init, scr_pose* out, int* conv, double* rms, double* inl,
                         double* score);
// Frames handed to the ABI: non-null planes (SCR_E_ARG) whose width x height equal the
// scene's intrinsics (SCR_E_DIMENSION_MISMATCH, core.hpp:57).
scr_status check_frames(const scr_scene_s* s, const scr_frame* frames, int n);

// RAII locks on the root scene's state (lanes lock their parent's).
struct StateReadLock {
  std::shared_mutex* m = nullptr;
  explicit StateReadLock(scr_scene_s* s) {
#ifdef SCR_NO_STATE_LOCK
    s = nullptr;
#endif
    if (s) {
      m = &(s->parent ? s->parent : s)->state_mu;
      m->lock_shared();
    }
  }
  ~StateReadLock() {
    if (m) m->unlock_shared();
  }
};
struct StateWriteLock {
  std::shared_mutex* m = nullptr;
  explicit StateWriteLock(scr_scene_s* s) {
    if (s) {
      m = &s->state_mu;
      m->lock();
    }
  }
  ~StateWriteLock() {
    if (m) m->unlock();
  }
};

}  // namespace scr

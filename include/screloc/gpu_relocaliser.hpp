// screloc::gpu — header-only C++17 drop-in for the reference relocaliser API
// (namespace screloc, proj/include/screloc/*.hpp + SPEC.md ops), backed by the B200 C ABI
// in include/screloc_gpu.h. Names and argument order follow the reference:
//   integrate_frame(state, forest, frame, pose)
//   update_leaves_round_robin(state, leaves_per_call)
//   clear_adaptation(state)
//   relocalise(profile, frame, state, forest, model, mode) SPEC.md:646-654
//   run_cascade(config, frame, ...)
//   generate_random_forest / serialize_forest              forest.hpp:104-112
// Errors are thrown as the reference's exception classes (core.hpp:24-72). Eigen value
// types are replaced by POD RigidTransform / Intrinsics (Eigen is not a dependency here).
#ifndef SCRELOC_GPU_RELOCALISER_HPP
#define SCRELOC_GPU_RELOCALISER_HPP

#include <cstdint>
#include <cstring>
#include <limits>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../screloc_gpu.h"

namespace screloc {

// ---- exceptions: the reference's classes by name (core.hpp:24-72) ------------------------
// A caller's `catch (screloc::InvalidDepth&)` fires for the B200 path exactly as for the CPU
// reference. If the reference's core.hpp is included first, its classes are used as they
// are; otherwise the same hierarchy (same names, same bases) is declared here.
#ifndef SCRELOC_CORE_HPP
class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& w) : std::runtime_error(w) {}
};
#define SCRELOC_GPU_ERROR(Name) \
  class Name : public Error {   \
   public:                      \
    using Error::Error;         \
  };
SCRELOC_GPU_ERROR(InvalidDepth)        // core.hpp:29
SCRELOC_GPU_ERROR(InvalidCentrePixel)  // core.hpp:33
SCRELOC_GPU_ERROR(MalformedData)       // core.hpp:49
SCRELOC_GPU_ERROR(UnreliablePose)      // core.hpp:53
SCRELOC_GPU_ERROR(DimensionMismatch)   // core.hpp:57
#undef SCRELOC_GPU_ERROR
#endif
// SPEC-level outcomes without a core.hpp class ("no pose") and device errors
class NoHypotheses : public Error {
 public:
  using Error::Error;
};
class AllCandidatesFailed : public Error {
 public:
  using Error::Error;
};
class CudaError : public Error {
 public:
  using Error::Error;
};

namespace gpu {

using screloc::AllCandidatesFailed;
using screloc::CudaError;
using screloc::DimensionMismatch;
using screloc::Error;
using screloc::InvalidCentrePixel;
using screloc::InvalidDepth;
using screloc::MalformedData;
using screloc::NoHypotheses;
using screloc::UnreliablePose;

inline void check(scr_status s, const char* what) {
  if (s == SCR_OK) return;
  const std::string msg = std::string(what) + ": " + scr_last_error();
  switch (s) {
    case SCR_E_INVALID_DEPTH: throw InvalidDepth(msg);
    case SCR_E_INVALID_CENTRE_PIXEL: throw InvalidCentrePixel(msg);
    case SCR_E_UNRELIABLE_POSE: throw UnreliablePose(msg);
    case SCR_E_NO_HYPOTHESES: throw NoHypotheses(msg);
    case SCR_E_ALL_CANDIDATES_FAILED: throw AllCandidatesFailed(msg);
    case SCR_E_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
    case SCR_E_MALFORMED_DATA: throw MalformedData(msg);
    case SCR_E_CUDA:
    case SCR_E_OOM: throw CudaError(msg);
    default: throw Error(msg);
  }
}

// ---- value types -------------------------------------------------------------------------
using RigidTransform = scr_pose;      // camera -> world, row-major R (geometry.hpp:14-42)
using PinholeIntrinsics = scr_intrinsics;
using RansacParams = scr_ransac_params;
using ForestParams = scr_forest_params;

inline RigidTransform identity_transform() {
  RigidTransform T{};
  T.R[0] = T.R[4] = T.R[8] = 1.0;
  return T;
}

// RgbdFrame (features.hpp:31-44) as a borrowed view: depth metres (0/NaN invalid),
// colour RGB8 interleaved, both row-major with x the column.
struct RgbdFrame {
  const float* depth = nullptr;
  const uint8_t* colour = nullptr;
  int width = 0, height = 0;  // must match the relocaliser's intrinsics (else DimensionMismatch)
  bool pose_reliable = true;
  scr_frame c() const { return scr_frame{depth, colour, width, height, pose_reliable ? 1 : 0, 0}; }
};

enum class Mode : int { Raw = SCR_MODE_RAW, Icp = SCR_MODE_ICP, Ranked = SCR_MODE_RANKED };

// Table 4; colour 30 / rigidity 0.05 m are SPEC.md:501-502 defaults.
inline RansacParams profile(const std::string& name) {
  RansacParams p{};
  p.colour_thresh = 30.0f;
  p.rigidity_tol = 0.05;
  p.n_cull = 64;
  if (name == "default") { p.max_gen_iters = 6000; p.n_max = 1024; p.eta = 512; p.pose_update = 1; p.use_cov = 1; p.min_sq_dist = 0.09; p.n_out = 16; }
  else if (name == "fast") { p.max_gen_iters = 500; p.n_max = 2048; p.eta = 256; p.pose_update = 0; p.use_cov = 0; p.min_sq_dist = 0.0; p.n_out = 1; }
  else if (name == "intermediate") { p.max_gen_iters = 1000; p.n_max = 2048; p.eta = 256; p.pose_update = 1; p.use_cov = 0; p.min_sq_dist = 0.09; p.n_out = 1; }
  else if (name == "slow") { p.max_gen_iters = 250; p.n_max = 2048; p.eta = 256; p.pose_update = 1; p.use_cov = 0; p.min_sq_dist = 0.0225; p.n_out = 16; }
  else throw Error("unknown relocaliser profile " + name);
  return p;
}
inline ForestParams forest_profile(bool cascade) {
  return cascade ? ForestParams{0.1f, 0.2f, 50, 5, 2048} : ForestParams{0.1f, 0.05f, 50, 20, 1024};
}

// CascadeConfig
struct CascadeConfig {
  std::vector<RansacParams> stages;
  std::vector<Mode> modes;
  std::vector<double> fallback_thresholds;  // stages.size() - 1, metres
  static CascadeConfig paper_three_stage() {  // F(5 cm) -> I(7.5 cm) -> S
    return {{profile("fast"), profile("intermediate"), profile("slow")}, {Mode::Icp, Mode::Icp, Mode::Ranked},
            {0.05, 0.075}};
  }
};

// RelocalisationResult
struct RelocalisationResult {
  std::optional<RigidTransform> final_pose;
  double best_score = std::numeric_limits<double>::infinity();
  int stage_used = 0;
  int status = 0;
  float stage_ms[4] = {0, 0, 0, 0};
  static RelocalisationResult from(const scr_result& r) {
    RelocalisationResult o;
    if (r.has_pose) o.final_pose = r.pose;
    o.best_score = r.score;
    o.stage_used = r.stage_used;
    o.status = r.status;
    std::memcpy(o.stage_ms, r.stage_ms, sizeof(o.stage_ms));
    return o;
  }
};

// generate_random_forest + serialize_forest (forest.hpp:104-112)
inline std::vector<uint8_t> generate_random_forest(uint64_t seed, int height = 14, double p_depth = 0.4,
                                                   int trees = 5, int radius = 130) {
  const size_t n = scr_generate_random_forest(seed, height, p_depth, trees, radius, nullptr, 0);
  if (!n) throw Error("generate_random_forest: bad arguments");
  std::vector<uint8_t> b(n);
  scr_generate_random_forest(seed, height, p_depth, trees, radius, b.data(), n);
  return b;
}

// ---- device + relocaliser (forest + adaptation state + scene model on one GPU) ------------
class Device {
 public:
  explicit Device(int ordinal = 0) { check(scr_device_open(ordinal, &d_), "scr_device_open"); }
  ~Device() { scr_device_close(d_); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  scr_device handle() const { return d_; }

 private:
  scr_device d_ = nullptr;
};

// TsdfVolume: dense TSDF scene model on the device; fuse = fuse_frame,
// raycast = raycast_depth (z-depth, 0 = no hit; packed normals optional).
class TsdfVolume {
 public:
  TsdfVolume(Device& dev, const float origin[3], float voxel, int nx, int ny, int nz, float trunc = 0.0f) {
    check(scr_tsdf_create(dev.handle(), origin, voxel, nx, ny, nz, trunc > 0.0f ? trunc : 4.0f * voxel, &v_),
          "TsdfVolume");
  }
  ~TsdfVolume() {
    if (v_) scr_tsdf_destroy(v_);
  }
  TsdfVolume(const TsdfVolume&) = delete;
  TsdfVolume& operator=(const TsdfVolume&) = delete;
  void fuse_frame(const PinholeIntrinsics& k, const float* depth, const RigidTransform& pose) {
    check(scr_tsdf_fuse(v_, &k, depth, &pose), "fuse_frame");
  }
  std::vector<float> raycast_depth(const PinholeIntrinsics& k, const RigidTransform& pose) {
    std::vector<float> d(static_cast<size_t>(k.width) * k.height);
    check(scr_tsdf_raycast(v_, &k, &pose, d.data(), nullptr), "raycast_depth");
    return d;
  }
  scr_tsdf handle() const { return v_; }

 private:
  scr_tsdf v_ = nullptr;
};

class Relocaliser {
 public:
  Relocaliser(Device& dev, const std::vector<uint8_t>& forest_blob, const ForestParams& fp,
              const PinholeIntrinsics& k, uint64_t adapt_seed = 7, int max_batch = 64) {
    check(scr_scene_create(dev.handle(), forest_blob.data(), forest_blob.size(), &fp, &k, adapt_seed, max_batch, &s_),
          "deserialize_forest / scene create");
  }
  ~Relocaliser() {
    if (s_) scr_scene_destroy(s_);
  }
  Relocaliser(const Relocaliser&) = delete;
  Relocaliser& operator=(const Relocaliser&) = delete;
  Relocaliser(Relocaliser&& o) noexcept : s_(o.s_) { o.s_ = nullptr; }

  // A relocalisation lane (scr_scene_fork): shares this relocaliser's forest, adaptation
  // state and model, with its own CUDA stream and workspace, so another host thread can
  // relocalise concurrently. Lanes are read-only and must be destroyed before their root.
  Relocaliser fork_lane(int max_batch = 64) {
    scr_scene h = nullptr;
    check(scr_scene_fork(s_, max_batch, &h), "fork_lane");
    return Relocaliser(h);
  }

  void set_scene_model(const std::vector<scr_prim>& prims) {
    check(scr_scene_set_analytic_model(s_, prims.data(), static_cast<int>(prims.size())), "set_scene_model");
  }
  // ICP and ranking on a fused model (the volume must outlive its use; nullptr: analytic)
  void set_scene_model(const TsdfVolume* volume) {
    check(scr_scene_set_tsdf_model(s_, volume ? volume->handle() : nullptr), "set_scene_model");
  }
  // integrate_frame: throws UnreliablePose if !frame.pose_reliable
  void integrate_frame(const RgbdFrame& frame, const RigidTransform& pose) {
    const scr_frame f = frame.c();
    check(scr_train(s_, &f, &pose), "integrate_frame");
  }
  void update_leaves_round_robin(int64_t leaves_per_call = 256) {
    check(scr_update(s_, leaves_per_call), "update_leaves_round_robin");
  }
  void clear_adaptation() { check(scr_reset(s_), "clear_adaptation"); }
  int64_t total_leaf_count() const { return scr_scene_total_leaves(s_); }

  // relocalise; NoHypotheses / AllCandidatesFailed come back as a result
  // without a pose (status set), exactly as the reference facade reports them.
  RelocalisationResult relocalise(const RansacParams& p, const RgbdFrame& frame, Mode mode, uint64_t seed) {
    return relocalise_batch(p, std::vector<RgbdFrame>{frame}, mode, std::vector<uint64_t>{seed}).front();
  }
  std::vector<RelocalisationResult> relocalise_batch(const RansacParams& p, const std::vector<RgbdFrame>& frames,
                                                     Mode mode, const std::vector<uint64_t>& seeds) {
    if (seeds.size() != frames.size()) throw DimensionMismatch("relocalise_batch: one seed per frame");
    std::vector<scr_frame> f;
    for (const auto& fr : frames) f.push_back(fr.c());
    std::vector<scr_result> r(frames.size());
    check(scr_relocalise_batch(s_, f.data(), static_cast<int>(f.size()), &p, static_cast<int>(mode), seeds.data(),
                               r.data()),
          "relocalise");
    std::vector<RelocalisationResult> out;
    for (const auto& x : r) out.push_back(RelocalisationResult::from(x));
    return out;
  }
  // run_cascade
  std::vector<RelocalisationResult> run_cascade_batch(const CascadeConfig& cfg, const std::vector<RgbdFrame>& frames,
                                                      const std::vector<uint64_t>& seeds) {
    if (cfg.fallback_thresholds.size() + 1 != cfg.stages.size() || cfg.modes.size() != cfg.stages.size())
      throw DimensionMismatch("run_cascade: thresholds.length must be stages.length - 1");
    if (seeds.size() != frames.size()) throw DimensionMismatch("run_cascade: one seed per frame");
    std::vector<scr_frame> f;
    for (const auto& fr : frames) f.push_back(fr.c());
    std::vector<int32_t> modes;
    for (Mode m : cfg.modes) modes.push_back(static_cast<int32_t>(m));
    std::vector<scr_result> r(frames.size());
    check(scr_cascade_batch(s_, f.data(), static_cast<int>(f.size()), cfg.stages.data(), modes.data(),
                            cfg.fallback_thresholds.data(), static_cast<int>(cfg.stages.size()), seeds.data(),
                            r.data()),
          "run_cascade");
    std::vector<RelocalisationResult> out;
    for (const auto& x : r) out.push_back(RelocalisationResult::from(x));
    return out;
  }
  RelocalisationResult run_cascade(const CascadeConfig& cfg, const RgbdFrame& frame, uint64_t seed) {
    return run_cascade_batch(cfg, std::vector<RgbdFrame>{frame}, std::vector<uint64_t>{seed}).front();
  }
  scr_scene handle() const { return s_; }

 private:
  explicit Relocaliser(scr_scene h) : s_(h) {}
  scr_scene s_ = nullptr;
};

// One host process driving several GPUs: after adapting on per_gpu[root], broadcast its
// prediction table to the relocalisers of the other GPUs (scr_broadcast_predictions, NCCL).
inline void broadcast_predictions(const std::vector<Relocaliser*>& per_gpu, int root = 0) {
  std::vector<scr_scene> h;
  for (const Relocaliser* r : per_gpu) h.push_back(r ? r->handle() : nullptr);
  check(scr_broadcast_predictions(h.data(), static_cast<int>(h.size()), root), "broadcast_predictions");
}

}  // namespace gpu
}  // namespace screloc

#endif

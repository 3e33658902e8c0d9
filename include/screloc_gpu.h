/* screloc_gpu.h — C ABI of the B200-native relocalisation hot path.
 *
 * This is the drop-in boundary a host binding of the reference screloc API
 * (namespace screloc, C++20) would call. Each entry point names the reference
 * interface it replaces; include/screloc/gpu_relocaliser.hpp restores the
 * reference's C++ surface (exceptions, value types) on top of it, and
 * INTEGRATION.md shows the bindings. Plain pointers and sizes only.
 *
 * Conventions:
 *  - status codes map 1:1 onto the screloc exception classes (core.hpp:24-72);
 *    scr_last_error() returns a thread-local message for the last failure;
 *  - frames are borrowed for the duration of a call; outputs are caller-allocated;
 *    the scene owns all device memory;
 *  - scr_train / scr_update / scr_reset are single-writer per scene
 *    (SPEC.md:407); relocalisation calls on a scene are serialised on the scene's
 *    stream, so they always see the predictions published by the last update;
 *  - results are deterministic functions of (frame, seed, scene state):
 *    batch size and batch composition never change them.
 */
#ifndef SCRELOC_GPU_H
#define SCRELOC_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct scr_device_s* scr_device; /* one per GPU */
typedef struct scr_scene_s* scr_scene;   /* forest + reservoirs + predictions + model + workspace */

typedef enum {
  SCR_OK = 0,
  SCR_E_ARG = 1,
  SCR_E_INVALID_DEPTH = 2,          /* screloc::InvalidDepth        (core.hpp:29) */
  SCR_E_INVALID_CENTRE_PIXEL = 3,   /* screloc::InvalidCentrePixel  (core.hpp:33) */
  SCR_E_UNRELIABLE_POSE = 4,        /* screloc::UnreliablePose      (core.hpp:53) */
  SCR_E_NO_HYPOTHESES = 5,          /* NoHypotheses */
  SCR_E_ALL_CANDIDATES_FAILED = 6,  /* AllCandidatesFailed */
  SCR_E_DIMENSION_MISMATCH = 7,     /* screloc::DimensionMismatch   (core.hpp:57) */
  SCR_E_MALFORMED_DATA = 8,         /* screloc::MalformedData       (core.hpp:49) */
  SCR_E_CUDA = 9,
  SCR_E_OOM = 10
} scr_status;

/* PinholeIntrinsics (geometry.hpp:47-66) */
typedef struct { int32_t width, height; double fx, fy, cx, cy; } scr_intrinsics;
/* RigidTransform camera->world (geometry.hpp:14-42), row-major R */
typedef struct { double R[9]; double t[3]; } scr_pose;
/* RgbdFrame (features.hpp:31-44): depth metres (0/NaN invalid), colour RGB8 interleaved, both
 * width x height row-major. width/height must equal the scene's intrinsics, else
 * SCR_E_DIMENSION_MISMATCH (screloc::DimensionMismatch, core.hpp:57). */
typedef struct {
  const float* depth;
  const uint8_t* rgb;
  int32_t width, height;
  int32_t pose_reliable;
  int32_t pad;
} scr_frame;
/* forest-side profile parameters (Table 4) */
typedef struct { float sigma, tau; int32_t max_clusters, min_cluster_size, capacity; } scr_forest_params;
/* RansacParams (Table 4) */
typedef struct {
  int32_t max_gen_iters, n_max, n_cull, eta, pose_update, use_cov;
  double min_sq_dist;
  float colour_thresh, pad0;
  double rigidity_tol;
  int32_t n_out, pad1;
} scr_ransac_params;
/* RelocalisationResult */
typedef struct {
  int32_t has_pose, status;
  scr_pose pose;
  double score;     /* depth-difference score s(xi), metres; +inf when absent */
  int32_t stage_used, n_candidates;
  float stage_ms[4];
} scr_result;
/* ModalCluster as dumped: mu, colour centroid, Sigma (+1e-6 I, upper:
 * s00 s01 s02 s11 s12 s22), Sigma^-1 in energy form (c00 c11 c22 2c01 2c02 2c12),
 * Sigma^-1/2 (upper), member count */
typedef struct { float mu[3], colour[3], cov[6], icov[6], isqrt[6]; int32_t size; } scr_mode;
/* LeafReservoir entry */
typedef struct { float x, y, z; uint8_t r, g, b, pad; } scr_entry;
/* SyntheticScene primitive: type 0 axis-aligned box (min a, max b;
 * zero thickness = planar panel), type 1 sphere (centre a, radius b[0]) */
typedef struct { int32_t type; float a[3], b[3], colour[3], cell; uint32_t tex_seed; } scr_prim;

enum { SCR_MODE_RAW = 0, SCR_MODE_ICP = 1, SCR_MODE_RANKED = 2 };

const char* scr_last_error(void);
const char* scr_version(void);

/* ---- host-side generators (run once per scene) --------------------------------- */
/* generate_random_forest (forest.hpp:104-106) serialised as the SPEC.md:300 blob;
 * returns the blob size (call with out = NULL to size the buffer), 0 on bad args. */
size_t scr_generate_random_forest(uint64_t seed, int height, double p_depth, int trees, int radius, uint8_t* out,
                                  size_t cap);
/* generate_synthetic_scene; returns the primitive count */
int scr_generate_synthetic_scene(uint64_t seed, int complexity, scr_prim* out, int cap);
/* generate_trajectory: kind 0 adaptation loop, kind 1 held-out test poses */
void scr_generate_trajectory(uint64_t seed, int n, int kind, scr_pose* out);

/* ---- device / scene lifetime ------------------------------------------------ */
scr_status scr_device_open(int ordinal, scr_device* out);
void scr_device_close(scr_device dev);

/* ForestModel deserialize_forest (forest.hpp:108-109) + AdaptationState creation
 * (SPEC.md:332-336). The blob is the SPEC.md:300 little-endian format. Frames used
 * with the scene must match `k`. max_batch bounds frames per relocalisation call. */
scr_status scr_scene_create(scr_device dev, const uint8_t* forest_blob, size_t n, const scr_forest_params* fp,
                            const scr_intrinsics* k, uint64_t adapt_seed, int max_batch, scr_scene* out);
void scr_scene_destroy(scr_scene s);
/* Relocalisation lane: a second handle on the same forest, adaptation state and model with
 * its own CUDA stream and batch workspace, so several host threads can relocalise
 * concurrently (the reference facade is reentrant for distinct RNG streams).
 * Lanes are read-only (train/update/reset/model/import return SCR_E_ARG) and always see
 * the root scene's last completed update. Destroy lanes before the root. */
scr_status scr_scene_fork(scr_scene root, int max_batch, scr_scene* out);
int64_t scr_scene_total_leaves(scr_scene s);
void* scr_scene_stream(scr_scene s); /* cudaStream_t all scene work runs on */
/* SceneModel used by ICP + ranking: analytic synthetic scene */
scr_status scr_scene_set_analytic_model(scr_scene s, const scr_prim* prims, int n_prims);

/* ---- TSDF scene model (scene_model; A13) -----------------------
 * Dense voxel volume on the device: voxel (i,j,k) centre = origin + (idx + 0.5) * voxel,
 * truncation `trunc` (SPEC default 4 voxels). */
typedef struct scr_tsdf_s* scr_tsdf;
scr_status scr_tsdf_create(scr_device dev, const float origin[3], float voxel, int nx, int ny, int nz, float trunc,
                           scr_tsdf* out);
void scr_tsdf_destroy(scr_tsdf v);
/* fuse_frame: projective TSDF update with the frame's depth at `pose`
 * (camera -> world); weight cap 128. Single writer. */
scr_status scr_tsdf_fuse(scr_tsdf v, const scr_intrinsics* k, const float* depth, const scr_pose* pose);
/* raycast_depth of the volume: z-depth per pixel (0 = no hit) and the
 * packed surface normal (0xffffffff = unavailable; normals may be null). */
scr_status scr_tsdf_raycast(scr_tsdf v, const scr_intrinsics* k, const scr_pose* pose, float* depth,
                            uint32_t* normals);
scr_status scr_tsdf_download(scr_tsdf v, float* tsdf, float* weight);
/* ICP + ranking of the scene use the fused volume instead of the analytic model (null:
 * back to the analytic model). The volume must outlive its use by the scene. */
scr_status scr_scene_set_tsdf_model(scr_scene s, scr_tsdf v);

/* ---- adaptation --------------------------------------------- */
/* integrate_frame(state, forest, frame, pose) — SPEC.md:348-356 */
scr_status scr_train(scr_scene s, const scr_frame* frame, const scr_pose* pose);
/* n consecutive integrate_frame calls (same result as n scr_train calls) */
scr_status scr_train_batch(scr_scene s, const scr_frame* frames, const scr_pose* poses, int n);
/* update_leaves_round_robin(state, leaves_per_call) — SPEC.md:366-374 */
scr_status scr_update(scr_scene s, int64_t leaves_per_call);
/* clear_adaptation(state) — SPEC.md:384-391 */
scr_status scr_reset(scr_scene s);

/* ---- relocalisation ---------------------------------------------- */
/* relocalise(profile, frame, state, forest, model, mode) for n independent frames;
 * frame i uses RANSAC seed seeds[i]. */
scr_status scr_relocalise_batch(scr_scene s, const scr_frame* frames, int n, const scr_ransac_params* p, int mode,
                                const uint64_t* seeds, scr_result* out);
/* run_cascade(config, frame, ...) for n independent frames; stage i uses
 * seed_i = seeds[f] + i * 0x9e3779b97f4a7c15 and mode modes[i]; thresholds has
 * nstages-1 entries. */
scr_status scr_cascade_batch(scr_scene s, const scr_frame* frames, int n, const scr_ransac_params* stages,
                             const int32_t* modes, const double* thresholds, int nstages, const uint64_t* seeds,
                             scr_result* out);

/* ---- device-resident frame sets (inputs already in HBM) ---------------------------- */
typedef struct scr_frameset_s* scr_frameset;
scr_status scr_frameset_create(scr_scene s, int capacity, scr_frameset* out);
void scr_frameset_destroy(scr_frameset fs);
scr_status scr_frameset_upload(scr_frameset fs, int first, const scr_frame* frames, int n);
/* render_frame(scene, pose, intrinsics) on the GPU for the scene's analytic model */
scr_status scr_frameset_render(scr_frameset fs, int first, const scr_pose* poses, int n);
scr_status scr_frameset_download(scr_frameset fs, int first, int n, float* depth, uint8_t* rgb);
/* training / relocalisation straight from a frame set (no host traffic except results) */
scr_status scr_train_frameset(scr_scene s, scr_frameset fs, const int32_t* idx, const scr_pose* poses, int n);
scr_status scr_cascade_frameset(scr_scene s, scr_frameset fs, const int32_t* idx, int n,
                                const scr_ransac_params* stages, const int32_t* modes, const double* thresholds,
                                int nstages, const uint64_t* seeds, scr_result* out);

/* ---- multi-GPU plumbing: the optional broadcast of the adapted forest -- */
/* bytes of the packed prediction table; export/import copy it to/from a caller-owned
 * DEVICE buffer (e.g. a torch tensor that torch.distributed broadcasts over NCCL). */
size_t scr_predictions_bytes(scr_scene s);
scr_status scr_predictions_export(scr_scene s, void* device_dst);
scr_status scr_predictions_import(scr_scene s, const void* device_src);
/* One host process driving several GPUs: broadcast root's adapted prediction table to the
 * scenes of the other GPUs with ncclBroadcast (the reference's
 * single-writer adaptation + concurrent readers). per_gpu[i] must be root scenes
 * (not lanes) created from the same forest on distinct devices; NCCL is loaded at run time
 * (libnccl.so.2). ngpu == 1 is a no-op. Receivers publish the table to their lanes. */
scr_status scr_broadcast_predictions(scr_scene* per_gpu, int ngpu, int root);

/* ---- parity hooks (tests) -------------------------------------------------------------- */
/* K0+K1: valid 4-px grid (packed x | y << 16) and leaf ids (n_grid x trees) */
scr_status scr_debug_leaves(scr_scene s, const scr_frame* f, int32_t* grid_px, int32_t* leaves, int* n_grid);
/* compute_feature_vector (features.cpp:60-65) at n pixels (packed) -> n x 256 */
scr_status scr_debug_features(scr_scene s, const scr_frame* f, const int32_t* px, int n, float* out);
scr_status scr_dump_seen(scr_scene s, uint32_t* out);
scr_status scr_dump_entries(scr_scene s, int64_t slot0, int64_t nslots, scr_entry* out);
scr_status scr_dump_predictions(scr_scene s, int32_t* counts, scr_mode* modes);
scr_status scr_load_predictions(scr_scene s, const int32_t* counts, const scr_mode* modes);
int64_t scr_update_cursor(scr_scene s);
/* cluster_reservoir on one reservoir (GPU RQS kernel) */
scr_status scr_debug_cluster(scr_scene s, const scr_entry* e, int n, scr_mode* out, int32_t* labels, int* n_modes);
/* one preemptive_ransac call: generated hypotheses (slot order) and survivors */
scr_status scr_debug_ransac(scr_scene s, const scr_frame* f, const scr_ransac_params* p, uint64_t seed,
                            int32_t* gen_slots, scr_pose* gen_poses, int* n_gen, int32_t* surv_slots,
                            scr_pose* surv_poses, float* surv_energy, int* n_surv);
/* generation test hook: mode 1 treats every triplet passing checks 1-3 as a possibly degenerate
   Kabsch ("suspect", decided by the exact finisher; overflows the per-frame list and exercises the
   exact continuation), 0 restores the normal classification. Results are identical either way. */
scr_status scr_debug_generation_mode(scr_scene s, int mode);
/* Generation diagnostics for one frame (not on the hot path): runs generate_hypothesis for
 * every slot and histograms every attempt's outcome by rejection tag,
 * tags[0..5] = {successful final attempts, NoModes, ColourCheckFailed, TooClose, NotRigid,
 * DegenerateKabsch}; *slots_ok = slots that generated a hypothesis. */
scr_status scr_debug_generation_stats(scr_scene s, const scr_frame* f, const scr_ransac_params* p, uint64_t seed,
                                      int64_t* tags, int* slots_ok);
scr_status scr_debug_icp(scr_scene s, const scr_frame* f, const scr_pose* init, scr_pose* out, int* converged,
                         double* rms, double* inlier_frac, double* score);
/* number of kernel launches issued by this scene so far (bench accounting) */
int64_t scr_kernel_launches(scr_scene s);
/* in-library profiler: CUDA events bracket every launch on the scene stream; reset on enable */
scr_status scr_profile_enable(scr_scene s, int enable);
/* per-kernel totals since the last enable: names, device ms, launches (arrays of `cap`);
 * work[7] = {mode evals, sample evals, LM terms, ICP terms, rays, node visits, generation
 * attempts}; returns the number of kernel kinds */
int scr_profile_read(scr_scene s, const char** names, double* ms, int64_t* launches, uint64_t* work, int cap);

#ifdef __cplusplus
}
#endif
#endif /* SCRELOC_GPU_H */

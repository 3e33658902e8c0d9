// ORACLE — test infrastructure only. Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load it; the product
// (paper_1810_12163_b200/) never links or calls it.
//
// An Eigen-free C++20 restatement of the reference relocalisation path:
//   rng/features/geometry/forest layout: bit-faithful to the shipped reference
//   code (proj/include/screloc/*.hpp, proj/src/features.cpp);
//   adaptation, ransac, scene_model, ranking_cascade: restated from SPEC.md
//   (the reference sources are missing), with every silent choice
//   frozen in DESIGN.md ("Numerics contract" and "Frozen decisions").
#pragma once
#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "rng.hpp"

namespace oracle {

// ---- errors (core.hpp:24-72) -----------------------------------------------
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& w) : std::runtime_error(w), code(c) {}
};
enum ErrCode {
  E_OK = 0, E_ARG = 1, E_INVALID_DEPTH = 2, E_INVALID_CENTRE_PIXEL = 3, E_UNRELIABLE_POSE = 4,
  E_NO_HYPOTHESES = 5, E_ALL_CANDIDATES_FAILED = 6, E_DIMENSION_MISMATCH = 7, E_MALFORMED_DATA = 8,
  E_ANGLE_NEAR_PI = 11
};

// ---- core / geometry types ---------------------------------------------------
struct Pose {  // camera -> world, p' = R p + t (geometry.hpp:14-29); R row-major
  double R[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  double t[3] = {0, 0, 0};
};
struct Intrinsics {  // geometry.hpp:47-66
  double fx = 0, fy = 0, cx = 0, cy = 0;
  int width = 0, height = 0;
  Intrinsics scaled(int f) const {
    Intrinsics s;
    s.fx = fx / f; s.fy = fy / f; s.cx = cx / f; s.cy = cy / f;
    s.width = width / f; s.height = height / f;
    return s;
  }
};
struct Frame {  // features.hpp:31-44 (colour RGB8 interleaved, row-major, x = column)
  int width = 0, height = 0;
  const float* depth = nullptr;
  const uint8_t* rgb = nullptr;
  Intrinsics k;
  bool pose_reliable = false;
};
constexpr float kMaxValidDepth = 20.0f;
inline bool depth_valid(float d) { return d > 0.0f && d <= kMaxValidDepth; }  // core.hpp:114

// geometry
Pose compose(const Pose& a, const Pose& b);
Pose invert(const Pose& a);
Pose exp_se3(const double twist[6]);
void log_se3(const Pose& T, double twist[6]);  // throws E_ANGLE_NEAR_PI
bool kabsch(const double* cam, const double* world, int n, Pose* out);  // points as xyz triples
void backproject(int x, int y, double depth, const Intrinsics& k, double out[3]);
void transform_point(const Pose& T, const double p[3], double out[3]);
void pose_error(const Pose& est, const Pose& gt, double* terr, double* aerr_deg);

// ---- features (features.hpp / features.cpp) ----------------------------------
constexpr int kFeatureCount = 256;
constexpr int kDepthFeatureCount = 128;
struct FeatureSpec {
  int kind = 0;  // 0 = Depth, 1 = DaRgb
  int dx = 0, dy = 0;
  int channel = 0;
};
std::vector<FeatureSpec> generate_feature_specs(uint64_t seed, int radius);
float compute_feature(const Frame& f, int x, int y, const FeatureSpec& s);
std::vector<int> sample_grid_pixels(const Frame& f, int spacing);  // packed x | y << 16

// ---- forest (forest.hpp) ----------------------------------------------------
struct TreeNode {
  int32_t feature = 0;
  float threshold = 0.0f;
  int32_t left = -1, right = -1, leaf_id = -1;
};
struct Tree {
  std::vector<TreeNode> nodes;
  int32_t leaf_count = 0;
};
struct Forest {
  std::vector<Tree> trees;
  std::vector<FeatureSpec> specs;
  std::vector<int64_t> leaf_base;  // tree-major slot offsets (forest.hpp:74-79)
  int64_t total_leaves = 0;
  void finalize();
};
Forest generate_random_forest(uint64_t seed, int height, double p_depth, int trees, int radius);
int32_t find_leaf(const Tree& t, const Frame& f, int x, int y, const std::vector<FeatureSpec>& specs);
std::vector<uint8_t> serialize_forest(const Forest& f);
Forest deserialize_forest(const uint8_t* data, size_t n);

// ---- synthetic scene --------------------------------------
struct Prim {
  int type = 0;  // 0 = axis-aligned box (zero thickness = planar panel), 1 = sphere
  float a[3] = {0, 0, 0}, b[3] = {0, 0, 0};  // box min/max; sphere centre a, radius b[0]
  float colour[3] = {0, 0, 0};
  float cell = 0.2f;
  uint32_t tex_seed = 0;
};
// TSDF scene model (oracle/tsdf.cpp, A13)
struct Tsdf {
  float origin[3] = {0, 0, 0};
  float voxel = 0.01f, trunc = 0.04f;
  int nx = 0, ny = 0, nz = 0;
  std::vector<float> tsdf, weight;  // x fastest
};
constexpr int kTsdfMaxSteps = 1024;

struct Scene {
  std::vector<Prim> prims;
  float room[3] = {4.0f, 3.0f, 2.5f};
  const Tsdf* tsdf = nullptr;  // when set, ICP and ranking use the fused model instead
};
Scene generate_synthetic_scene(uint64_t seed, int complexity);
struct Hit {
  float t;
  int prim;
  int face;
};
Hit raycast_pixel(const Scene& s, const float Rf[9], const float tf[3], const Intrinsics& k, int x, int y);
void hit_normal(const Scene& s, const Hit& h, const float p[3], float n[3]);
constexpr float kRenderMaxDepth = 6.0f;
Tsdf tsdf_create(const float origin[3], float voxel, int nx, int ny, int nz, float trunc);
void tsdf_fuse(Tsdf& v, const float* depth, const Intrinsics& k, const Pose& T);
bool tsdf_sample(const Tsdf& v, const float p[3], float* F);
bool tsdf_raycast_pixel(const Tsdf& v, const float R[9], const float tf[3], const Intrinsics& k, int x, int y,
                        float* t, uint32_t* nrm);
uint32_t pack_normal(const float n[3]);
void unpack_normal(uint32_t p, float n[3]);
void render_frame(const Scene& s, const Pose& T, const Intrinsics& k, float* depth, uint8_t* rgb);
void generate_trajectory(uint64_t seed, int n, int kind, Pose* out);  // kind 0 = adapt, 1 = test

// ---- adaptation -------------------------------------------
constexpr int kMaxModes = 50;
struct Entry {
  float x, y, z;
  uint8_t r, g, b, pad;
};
struct Mode {
  float mu[3];
  float colour[3];
  float cov[6];    // s00 s01 s02 s11 s12 s22 (incl. +1e-6 I)
  float icov[6];   // c00 c11 c22 2c01 2c02 2c12 of Sigma^-1 (energy form)
  float isqrt[6];  // Sigma^-1/2: s00 s01 s02 s11 s12 s22
  int32_t size;
};
struct ForestParams {
  float sigma = 0.1f, tau = 0.05f;
  int max_clusters = 50, min_cluster_size = 20, capacity = 1024;
};
struct AdaptState {
  ForestParams params;
  uint64_t seed = 7;
  int64_t total_leaves = 0;
  int64_t cursor = 0;
  std::vector<Entry> entries;   // total_leaves * capacity
  std::vector<uint32_t> seen;   // total_leaves
  std::vector<int32_t> pred_count;
  std::vector<Mode> modes;      // total_leaves * kMaxModes
};
void init_state(AdaptState& s, const Forest& f, const ForestParams& p, uint64_t seed);
void clear_adaptation(AdaptState& s);
void reservoir_insert(AdaptState& s, int64_t slot, const Entry& e);
void integrate_frame(AdaptState& s, const Forest& f, const Frame& fr, const Pose& pose);
std::vector<Mode> cluster_reservoir(const Entry* e, int n, const ForestParams& p, std::vector<int>* labels = nullptr);
void update_leaves_round_robin(AdaptState& s, int64_t leaves_per_call);

// ---- RANSAC -----------------------------------------------
struct RansacParams {
  int max_iters = 6000, n_max = 1024, n_cull = 64, eta = 512;
  int pose_update = 1, use_cov = 1;
  double min_sq_dist = 0.09;
  float colour_thresh = 30.0f;
  double rigidity_tol = 0.05;
  int n_out = 16;
};
enum Reject { REJ_OK = 0, REJ_NO_MODES = 1, REJ_COLOUR = 2, REJ_TOO_CLOSE = 3, REJ_NOT_RIGID = 4, REJ_DEGENERATE = 5 };

// Per-frame context: valid grid pixels, their leaves, camera points, colours.
struct FrameCtx {
  const Frame* frame = nullptr;
  std::vector<int> grid;             // packed x | y << 16
  std::vector<int64_t> slots;        // grid.size() * T leaf slots
  std::vector<double> cam;           // grid.size() * 3 (double backprojection)
  std::vector<float> camf;           // float copies
  std::vector<int32_t> nmodes;       // per grid pixel (union over trees)
  int trees = 0;
};
void build_frame_ctx(FrameCtx& c, const Forest& f, const AdaptState& s, const Frame& fr);
const Mode* ctx_mode(const FrameCtx& c, const AdaptState& s, int g, int m);

struct Hypothesis {
  Pose pose;
  int slot = -1;
  float energy = 0;
  int iterations = 0;  // generation attempts used
};
// tags (optional): per-attempt outcome histogram, indexed by Reject (REJ_OK counts the
// successful final attempt). Diagnostic only; never changes the draws.
int generate_hypothesis(const FrameCtx& c, const AdaptState& s, const RansacParams& p, Rng& rng, Pose* out,
                        int* attempts, int64_t* tags = nullptr);
// Checks 2-3 + Kabsch of one triplet: REJ_OK (transform in *out) or the tag.
int check_triplet(const double cm[9], const double w[9], const RansacParams& p, Pose* out);
// LM residual S (H x - mu) and Jacobian w.r.t. the left twist (omega, rho); J may be null.
void lm_residual_jacobian(const Pose& H, const double x[3], const Mode& m, bool use_cov, double r[3],
                          double J[3][6], double y[3]);
// Eq. 5 accumulated per eta-sample batch: E = sum_b E_b (batches in order), E_b sequential.
float energy(const FrameCtx& c, const AdaptState& s, const Pose& H, const std::vector<int>& samples, int eta);
void draw_samples(uint64_t seed, int batch, int n_max, int eta, int G, std::vector<int>& out);
void lm_refine(const FrameCtx& c, const AdaptState& s, Pose& H, const std::vector<int>& samples, bool use_cov,
               double* final_surrogate = nullptr);
std::vector<Hypothesis> preemptive_ransac(const FrameCtx& c, const AdaptState& s, const RansacParams& p,
                                          uint64_t seed, std::vector<Hypothesis>* generated = nullptr);

// ---- ICP / ranking / cascade -------------------------------
struct IcpResult {
  Pose pose;
  int converged = 0;
  double rms = 0, inlier_frac = 0;
  int iterations = 0;
};
IcpResult icp_refine(const Scene& s, const Pose& init, const Frame& fr);
double depth_diff_score(const Scene& s, const Pose& T, const Frame& fr);
double depth_diff_images(const float* live, const float* synth, int W, int H);
void raycast_depth(const Scene& s, const Pose& T, const Intrinsics& k, float* out);
constexpr double kInf = std::numeric_limits<double>::infinity();

enum Mode_ { MODE_RAW = 0, MODE_ICP = 1, MODE_RANKED = 2 };
struct RelocResult {
  int has_pose = 0;
  Pose pose;
  double score = kInf;
  int stage_used = 0;
  int n_candidates = 0;
  int status = 0;
};
RelocResult relocalise(const RansacParams& p, int mode, const Frame& fr, const Forest& f, const AdaptState& s,
                       const Scene& model, uint64_t seed);
RelocResult run_cascade(const RansacParams* stages, const int* modes, const double* thresholds, int nstages,
                        const Frame& fr, const Forest& f, const AdaptState& s, const Scene& model, uint64_t seed);
uint64_t stage_seed(uint64_t seed, int stage);

// Canonical reduction orders shared (by definition, not by code) with the GPU.
constexpr int kLmLanes = 128;  // canonical LM reduction lanes (4 warps of 32)
constexpr int kIcpCtas = 8;                    // ICP / score: 8-CTA cluster
constexpr int kIcpLanes = 256 * kIcpCtas;      // lanes = threads of the cluster
constexpr int kIcpIters[3] = {4, 5, 10};  // at most, level 0 (fine), 1, 2 (coarse)
constexpr double kIcpStopStep = 1e-6;    // a level stops once every |twist component| < this

}  // namespace oracle

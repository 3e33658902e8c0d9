// TSDF scene model on the device (oracle/tsdf.cpp restated bit for bit,
// DESIGN.md A13): dense voxel volume, voxel-parallel projective fusion and pixel-parallel
// ray casting. The ICP / ranking kernels (reloc.cu) ray cast the same volume through
// tsdf_raycast_ray when a scene's model is a volume (scr_scene_set_tsdf_model).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "internal.cuh"

#define SCR_TRY(x)               \
  do {                           \
    scr_status _s = (x);         \
    if (_s != SCR_OK) return _s; \
  } while (0)

namespace scr {

// fuse_frame: one thread per voxel (grid-stride); all arithmetic as in the oracle.
__global__ void k_tsdf_fuse(TsdfView v, float2* __restrict__ vox, const float* __restrict__ depth, int W, int H,
                            float fx, float fy, float cx, float cy, Pose T) {
  float R[9], tf[3];
#pragma unroll
  for (int i = 0; i < 9; ++i) R[i] = static_cast<float>(T.R[i]);
#pragma unroll
  for (int i = 0; i < 3; ++i) tf[i] = static_cast<float>(T.t[i]);
  const size_t n = static_cast<size_t>(v.nx) * v.ny * v.nz;
  for (size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < n;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int ix = static_cast<int>(idx % v.nx);
    const int jy = static_cast<int>((idx / v.nx) % v.ny);
    const int kz = static_cast<int>(idx / (static_cast<size_t>(v.nx) * v.ny));
    const float c0 = __fmaf_rn(__fadd_rn(static_cast<float>(ix), 0.5f), v.voxel, v.ox);
    const float c1 = __fmaf_rn(__fadd_rn(static_cast<float>(jy), 0.5f), v.voxel, v.oy);
    const float c2 = __fmaf_rn(__fadd_rn(static_cast<float>(kz), 0.5f), v.voxel, v.oz);
    const float dx = __fsub_rn(c0, tf[0]), dy = __fsub_rn(c1, tf[1]), dz = __fsub_rn(c2, tf[2]);
    float pc[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) pc[i] = __fmaf_rn(R[0 + i], dx, __fmaf_rn(R[3 + i], dy, __fmul_rn(R[6 + i], dz)));
    if (!(pc[2] > 0.0f)) continue;
    const float u = __fmaf_rn(fx, __fdiv_rn(pc[0], pc[2]), cx), w = __fmaf_rn(fy, __fdiv_rn(pc[1], pc[2]), cy);
    const int ui = static_cast<int>(floorf(__fadd_rn(u, 0.5f))), vi = static_cast<int>(floorf(__fadd_rn(w, 0.5f)));
    if (ui < 0 || vi < 0 || ui >= W || vi >= H) continue;
    const float d = depth[static_cast<size_t>(vi) * W + ui];
    if (!depth_valid(d)) continue;
    const float sdf = __fsub_rn(d, pc[2]);
    if (sdf < -v.trunc) continue;
    const float f = fminf(1.0f, __fdiv_rn(sdf, v.trunc));
    const float2 e = vox[idx];
    vox[idx] = make_float2(__fdiv_rn(__fmaf_rn(e.x, e.y, f), __fadd_rn(e.y, 1.0f)), fminf(__fadd_rn(e.y, 1.0f), 128.0f));
  }
}

// raycast_depth of the volume (parity / user API): one thread per pixel.
__global__ void k_tsdf_raycast(TsdfView v, int W, int H, float fx, float fy, float cx, float cy, Pose T,
                               float* __restrict__ depth, uint32_t* __restrict__ nrm) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= W * H) return;
  const int x = p % W, y = p / W;
  float R[9], tf[3];
#pragma unroll
  for (int i = 0; i < 9; ++i) R[i] = static_cast<float>(T.R[i]);
#pragma unroll
  for (int i = 0; i < 3; ++i) tf[i] = static_cast<float>(T.t[i]);
  const float dcx = __fdiv_rn(__fsub_rn(static_cast<float>(x), cx), fx);
  const float dcy = __fdiv_rn(__fsub_rn(static_cast<float>(y), cy), fy);
  float d[3];
  ray_dir_tab(R, dcx, dcy, d);
  float t = 0.0f;
  uint32_t n = 0xffffffffu;
  if (!tsdf_raycast_ray(v, tf, d, &t, &n)) t = 0.0f;
  depth[p] = t;
  if (nrm) nrm[p] = n;
}

}  // namespace scr

using namespace scr;

struct scr_tsdf_s {
  scr_device dev = nullptr;
  cudaStream_t stream = nullptr;
  TsdfView view;
  float2* d_vox = nullptr;
  float* d_depth = nullptr;  // staging for one frame
  uint32_t* d_nrm = nullptr;
  size_t stage_px = 0;
};

namespace scr {
TsdfView tsdf_view(scr_tsdf v) { return v ? v->view : TsdfView{}; }
}  // namespace scr

namespace {
scr_status stage(scr_tsdf v, size_t px) {
  if (px <= v->stage_px) return SCR_OK;
  if (v->d_depth) cudaFree(v->d_depth);
  if (v->d_nrm) cudaFree(v->d_nrm);
  v->d_depth = nullptr;
  v->d_nrm = nullptr;
  SCR_CUDA(cudaMalloc(&v->d_depth, px * sizeof(float)));
  SCR_CUDA(cudaMalloc(&v->d_nrm, px * sizeof(uint32_t)));
  v->stage_px = px;
  return SCR_OK;
}

Pose to_dev_pose(const scr_pose& p) {
  Pose T;
  std::memcpy(&T, &p, sizeof(Pose));
  return T;
}
}  // namespace

extern "C" {

scr_status scr_tsdf_create(scr_device dev, const float origin[3], float voxel, int nx, int ny, int nz, float trunc,
                           scr_tsdf* out) {
  if (!dev || !origin || !out || !(voxel > 0.0f) || !(trunc > 0.0f) || nx < 2 || ny < 2 || nz < 2 ||
      static_cast<double>(nx) * ny * nz > 4.0e9) {
    set_error("scr_tsdf_create: bad arguments");
    return SCR_E_ARG;
  }
  SCR_CUDA(cudaSetDevice(dev->ordinal));
  scr_tsdf v = new scr_tsdf_s();
  v->dev = dev;
  v->view.ox = origin[0];
  v->view.oy = origin[1];
  v->view.oz = origin[2];
  v->view.voxel = voxel;
  v->view.trunc = trunc;
  v->view.nx = nx;
  v->view.ny = ny;
  v->view.nz = nz;
  const size_t n = static_cast<size_t>(nx) * ny * nz;
  cudaError_t e = cudaStreamCreateWithFlags(&v->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&v->d_vox, n * sizeof(float2));
  if (e != cudaSuccess) {
    scr_tsdf_destroy(v);
    return cuda_fail(e, "scr_tsdf_create");
  }
  // empty volume: tsdf 1, weight 0 (the fill is a 2-float pattern: write it from the host once)
  std::vector<float2> init(std::min<size_t>(n, 1 << 20), make_float2(1.0f, 0.0f));
  for (size_t o = 0; o < n; o += init.size()) {
    const size_t m = std::min(init.size(), n - o);
    e = cudaMemcpy(v->d_vox + o, init.data(), m * sizeof(float2), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      scr_tsdf_destroy(v);
      return cuda_fail(e, "scr_tsdf_create init");
    }
  }
  v->view.vox = v->d_vox;
  *out = v;
  return SCR_OK;
}

void scr_tsdf_destroy(scr_tsdf v) {
  if (!v) return;
  cudaSetDevice(v->dev->ordinal);
  if (v->stream) cudaStreamSynchronize(v->stream);
  for (void* p : {static_cast<void*>(v->d_vox), static_cast<void*>(v->d_depth), static_cast<void*>(v->d_nrm)})
    if (p) cudaFree(p);
  if (v->stream) cudaStreamDestroy(v->stream);
  delete v;
}

scr_status scr_tsdf_fuse(scr_tsdf v, const scr_intrinsics* k, const float* depth, const scr_pose* pose) {
  if (!v || !k || !depth || !pose || k->width <= 0 || k->height <= 0) return SCR_E_ARG;
  SCR_CUDA(cudaSetDevice(v->dev->ordinal));
  const size_t px = static_cast<size_t>(k->width) * k->height;
  SCR_TRY(stage(v, px));
  SCR_CUDA(cudaMemcpyAsync(v->d_depth, depth, px * sizeof(float), cudaMemcpyHostToDevice, v->stream));
  const size_t n = static_cast<size_t>(v->view.nx) * v->view.ny * v->view.nz;
  const int blocks = static_cast<int>(std::min<size_t>((n + 255) / 256, static_cast<size_t>(v->dev->sm_count) * 16));
  k_tsdf_fuse<<<blocks, 256, 0, v->stream>>>(v->view, v->d_vox, v->d_depth, k->width, k->height,
                                             static_cast<float>(k->fx), static_cast<float>(k->fy),
                                             static_cast<float>(k->cx), static_cast<float>(k->cy), to_dev_pose(*pose));
  SCR_CUDA(cudaGetLastError());
  SCR_CUDA(cudaStreamSynchronize(v->stream));  // single writer: the update is published on return
  return SCR_OK;
}

scr_status scr_tsdf_raycast(scr_tsdf v, const scr_intrinsics* k, const scr_pose* pose, float* depth,
                            uint32_t* normals) {
  if (!v || !k || !pose || !depth || k->width <= 0 || k->height <= 0) return SCR_E_ARG;
  SCR_CUDA(cudaSetDevice(v->dev->ordinal));
  const size_t px = static_cast<size_t>(k->width) * k->height;
  SCR_TRY(stage(v, px));
  k_tsdf_raycast<<<static_cast<unsigned>((px + 127) / 128), 128, 0, v->stream>>>(
      v->view, k->width, k->height, static_cast<float>(k->fx), static_cast<float>(k->fy), static_cast<float>(k->cx),
      static_cast<float>(k->cy), to_dev_pose(*pose), v->d_depth, v->d_nrm);
  SCR_CUDA(cudaGetLastError());
  SCR_CUDA(cudaMemcpyAsync(depth, v->d_depth, px * sizeof(float), cudaMemcpyDeviceToHost, v->stream));
  if (normals)
    SCR_CUDA(cudaMemcpyAsync(normals, v->d_nrm, px * sizeof(uint32_t), cudaMemcpyDeviceToHost, v->stream));
  SCR_CUDA(cudaStreamSynchronize(v->stream));
  return SCR_OK;
}

scr_status scr_tsdf_download(scr_tsdf v, float* tsdf, float* weight) {
  if (!v || !tsdf || !weight) return SCR_E_ARG;
  SCR_CUDA(cudaSetDevice(v->dev->ordinal));
  SCR_CUDA(cudaStreamSynchronize(v->stream));
  const size_t n = static_cast<size_t>(v->view.nx) * v->view.ny * v->view.nz;
  std::vector<float2> h(n);
  SCR_CUDA(cudaMemcpy(h.data(), v->d_vox, n * sizeof(float2), cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < n; ++i) {
    tsdf[i] = h[i].x;
    weight[i] = h[i].y;
  }
  return SCR_OK;
}

}  // extern "C"

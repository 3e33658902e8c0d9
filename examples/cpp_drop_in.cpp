// Reference-style C++ usage of the B200 relocaliser through include/screloc/gpu_relocaliser.hpp:
// adapt on a synthetic sequence, then relocalise held-out frames with the 3-stage cascade.
// Build: g++ -std=c++17 -I include examples/cpp_drop_in.cpp -L paper_1810_12163_b200/lib \
//          -lscreloc_gpu -Wl,-rpath,paper_1810_12163_b200/lib -o cpp_drop_in
#include <cmath>
#include <cstring>
#include <thread>
#include <cstdio>
#include <vector>

#include "screloc/gpu_relocaliser.hpp"

namespace sg = screloc::gpu;

int main() {
  sg::Device dev(0);
  const sg::PinholeIntrinsics k{640, 480, 585.0, 585.0, 320.0, 240.0};
  sg::Relocaliser reloc(dev, sg::generate_random_forest(42), sg::forest_profile(true), k, 7, 16);
  std::vector<scr_prim> prims(scr_generate_synthetic_scene(1, 20, nullptr, 0));
  scr_generate_synthetic_scene(1, 20, prims.data(), static_cast<int>(prims.size()));
  reloc.set_scene_model(prims);

  // synthetic RGB-D frames rendered on the GPU (fixture), copied to host like camera input
  const int n_adapt = 60, n_test = 8;
  std::vector<scr_pose> adapt(n_adapt), test(n_test);
  scr_generate_trajectory(1, n_adapt, 0, adapt.data());
  scr_generate_trajectory(1, n_test, 1, test.data());
  scr_frameset fs = nullptr;
  sg::check(scr_frameset_create(reloc.handle(), n_adapt + n_test, &fs), "frameset");
  sg::check(scr_frameset_render(fs, 0, adapt.data(), n_adapt), "render");
  sg::check(scr_frameset_render(fs, n_adapt, test.data(), n_test), "render");
  const size_t px = 640 * 480;
  std::vector<float> depth((n_adapt + n_test) * px);
  std::vector<uint8_t> rgb((n_adapt + n_test) * px * 3);
  sg::check(scr_frameset_download(fs, 0, n_adapt + n_test, depth.data(), rgb.data()), "download");
  scr_frameset_destroy(fs);

  for (int i = 0; i < n_adapt; ++i)  // train
    reloc.integrate_frame({&depth[i * px], &rgb[i * px * 3], k.width, k.height, true}, adapt[i]);
  reloc.update_leaves_round_robin(reloc.total_leaf_count());  // update (every leaf once)

  std::vector<sg::RgbdFrame> frames;
  std::vector<uint64_t> seeds;
  for (int i = 0; i < n_test; ++i) {
    frames.push_back({&depth[(n_adapt + i) * px], &rgb[(n_adapt + i) * px * 3], k.width, k.height, true});
    seeds.push_back(100 + i);
  }
  const auto res = reloc.run_cascade_batch(sg::CascadeConfig::paper_three_stage(), frames, seeds);
  int ok = 0;
  for (int i = 0; i < n_test; ++i) {
    if (!res[i].final_pose) continue;
    const auto& p = *res[i].final_pose;
    const double dt = std::sqrt(std::pow(p.t[0] - test[i].t[0], 2) + std::pow(p.t[1] - test[i].t[1], 2) +
                                std::pow(p.t[2] - test[i].t[2], 2));
    ok += dt <= 0.05;
  }
  std::printf("cpp drop-in: %d/%d frames within 5 cm (stage of frame 0: %d)\n", ok, n_test, res[0].stage_used);
  try {
    reloc.integrate_frame({&depth[0], &rgb[0], k.width, k.height, false}, adapt[0]);
    return 2;
  } catch (const screloc::UnreliablePose&) {  // the reference's class (core.hpp:53)
    std::printf("UnreliablePose raised as in the reference\n");
  }
  try {  // a frame whose size is not the scene's: screloc::DimensionMismatch (core.hpp:57)
    reloc.relocalise(sg::profile("fast"), {&depth[0], &rgb[0], k.width / 2, k.height, true}, sg::Mode::Icp, 1);
    return 3;
  } catch (const screloc::DimensionMismatch&) {
    std::printf("DimensionMismatch raised as in the reference\n");
  }
  {  // a second relocalisation lane on another thread gives the same poses
    sg::Relocaliser lane = reloc.fork_lane(n_test);
    std::vector<sg::RelocalisationResult> lane_res;
    std::thread th([&] { lane_res = lane.run_cascade_batch(sg::CascadeConfig::paper_three_stage(), frames, seeds); });
    th.join();
    for (int i = 0; i < n_test; ++i)
      if (static_cast<bool>(lane_res[i].final_pose) != static_cast<bool>(res[i].final_pose) ||
          (res[i].final_pose && std::memcmp(&*lane_res[i].final_pose, &*res[i].final_pose, sizeof(sg::RigidTransform))))
        return 3;
    std::printf("lane on a second thread: identical results\n");
  }
  return ok >= n_test / 2 ? 0 : 1;
}

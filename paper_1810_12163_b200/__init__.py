"""paper_1810_12163_b200 — B200-native relocalisation hot path of arXiv 1810.12163.

The product is the sm_100a library lib/libscreloc_gpu.so behind the C ABI in
include/screloc_gpu.h; `relocaliser` mirrors the reference screloc API on top of it.
"""
from . import native
from .relocaliser import (FOREST_PROFILES, PROFILES, CascadeConfig, Device, FrameSet, RelocalisationResult, Scene, TsdfVolume, broadcast_predictions, forest_params,
                          generate_random_forest, generate_synthetic_scene, generate_trajectory, intrinsics,
                          pose_arrays, ransac_params, to_pose)

__all__ = ["native", "PROFILES", "FOREST_PROFILES", "CascadeConfig", "Device", "FrameSet", "RelocalisationResult", "Scene", "TsdfVolume",
           "broadcast_predictions", "forest_params",
           "generate_random_forest", "generate_synthetic_scene", "generate_trajectory", "intrinsics", "pose_arrays",
           "ransac_params", "to_pose"]

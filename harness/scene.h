/* harness/scene.h — synthetic-input HARNESS (not the matcher path, not the
 * product library).  A bit-identical restatement of the reference's
 * box-world generator (scene.hpp:156-220) so bench.py's B200 arm and the GPU
 * tests can build the same doubles the reference consumes on a box where the
 * reference is absent; tests/test_host.py pins it to oracle/_ref's gen_scene.
 * Built into harness/libbbs_scene.so (gen_scene is out of
 * scope for the product, "reused to generate identical synthetic inputs"). */
#ifndef BBS_HARNESS_SCENE_H
#define BBS_HARNESS_SCENE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* SceneSpec, scene.hpp:21-38. */
typedef struct hs_scene_spec {
  double size_x, size_y, size_z;
  int32_t num_boxes;
  double min_box_side, max_box_side, min_box_height;
  double map_spacing, scan_spacing, scan_range, point_jitter;
  int32_t tilt_noise;
  double gt_yaw_min, gt_yaw_max;
  uint64_t min_scan_points;
  double feasibility_resolution;
} hs_scene_spec;

/* Status: 0 ok, 11 infeasible pose (InfeasiblePoseError), 12 config
 * (ConfigError), 14 invalid argument. */
void hs_scene_spec_default(hs_scene_spec* spec);
/* gen_scene, scene.hpp:156-220.  Buffers are malloc'ed; release with
 * hs_free.  gt6 = x, y, z, roll, pitch, yaw. */
int hs_gen_scene(const hs_scene_spec* spec, uint64_t seed, double** map_xyz, uint64_t* n_map,
                 double** scan_xyz, uint64_t* n_scan, double* gt6);
/* C4 helper: extra scans of seed's map (poses from Rng(pose_seed_base + j));
 * the same algorithm as oracle/ref_shim.cpp ref_gen_scans. */
int hs_gen_scans(const hs_scene_spec* spec, uint64_t seed, uint64_t pose_seed_base, int32_t n_scans,
                 double** scan_xyz, uint64_t* offsets, double* gt);
/* First k points of a Fisher-Yates shuffle driven by Rng(seed). */
int hs_cut_scan(const double* xyz, uint64_t n, uint64_t k, uint64_t seed, double* out);
const char* hs_last_error(void);
void hs_free(void* p);

#ifdef __cplusplus
}
#endif
#endif

// bbs_internal.h — shared host/device declarations of the B200 matcher.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include <vector_types.h>

#include "bbs.h"

namespace bbs {

constexpr int kMaxLevels = 16;      // levels 0..15 (queue key packs level in 4 bits)
constexpr int kMaxScorePoints = (1 << 20) - 1;  // queue key packs score in 20 bits
constexpr uint64_t kHashEmpty = ~0ull;

// Error carrying a bbs_status; thrown by host code, mapped at the C-ABI.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void throw_cuda(const char* what, int err, const char* file, int line);

#define BBS_CUDA(call)                                                  \
  do {                                                                  \
    const int e_ = static_cast<int>(call);                              \
    if (e_ != 0) ::bbs::throw_cuda(#call, e_, __FILE__, __LINE__);      \
  } while (0)

// ---- device view of one level (passed by value in kernel parameters) ----
struct LevelView {
  int32_t layout;        // BBS_LAYOUT_BITMAP / BBS_LAYOUT_HASH
  int32_t pad0;
  double cell;           // ldexp(r, level), voxel_map.hpp:188
  double inv_cell;       // RN(1 / cell), fast-path only (exactness guarded)
  int32_t box_min[3];    // inclusive voxel box of the inflated set
  uint32_t dim[3];       // box extents
  // bitmap (z-column major): bit (uz & 31) of
  // words[((uz >> 5) * dim[1] + uy) * dim[0] + ux]; one 32-bit word answers
  // 32 consecutive z-voxels of an (x, y) column, consecutive x share sectors.
  uint32_t nwz;          // ceil(dim[2] / 32) words per column
  uint32_t pad2;
  const uint32_t* words;
  // hash: packed key = (x' << (by+bz)) | (y' << bz) | z', 4 slots per bucket
  const unsigned long long* slots;
  unsigned long long bucket_mask;  // buckets - 1 (buckets >= 2, power of two)
  uint32_t bucket_shift; // 64 - log2(buckets)
  uint32_t bits_y, bits_z;
  uint32_t pad1;
};

struct MapView {
  int32_t n_levels;
  int32_t pad;
  double r;
  LevelView level[kMaxLevels];
};

// ---- angular LUT (host cos/sin, device reads) -----------------------------
// For (level l, axis a) the entries lut[off[l*3+a] + i] = {cos, sin} of
// AxisGrid::angle(i) (angular_grid.hpp:57), computed with the host libm
// exactly as pose_to_transform does (geometry.hpp:103-105).
struct GridView {
  int32_t max_level;
  int32_t lut_off[kMaxLevels * 3];    // first LUT entry of (level, axis)
  int32_t lut_lo[kMaxLevels * 3];     // index stored at lut_off (0 for search grids)
  int32_t lut_n[kMaxLevels * 3];      // entries of (level, axis)
  int32_t max_index[kMaxLevels * 3];  // AxisGrid::max_index
  int32_t div[kMaxLevels * 3];        // AngularGrid::divisions(axis, level) (level >= 1)
  const double2* lut;
};

// ---- host angular grid (restates angular_grid.hpp) ------------------------
struct AxisGrid {
  double w_min = 0, w_max = 0, step = 0;
  int segments = 0;
  bool periodic = false;
  int max_index() const { return segments == 0 ? 0 : (periodic ? segments - 1 : segments); }
  int index_count() const { return max_index() + 1; }
  double angle(int i) const { return w_min + step * static_cast<double>(i); }
};

struct HostGrid {
  int max_level = 0;
  std::vector<AxisGrid> axes;  // [axis * (max_level+1) + level]
  const AxisGrid& axis(int a, int l) const { return axes[a * (max_level + 1) + l]; }
  int divisions(int a, int l) const;
};

HostGrid make_grid(const bbs_search_config& cfg, double d_max);
double host_max_range(const double* xyz, uint64_t n);
bbs_aabb host_bounding_box(const double* xyz, uint64_t n);
int32_t host_voxel_index(double c, double cell);
// Max children of one branch() call over all levels (nodes.hpp:91-121).
uint64_t max_children(const HostGrid& g);
// Host cos/sin LUT (vector of {cos, sin} pairs) and the GridView offsets.
// lo/hi (optional, [level*3+axis]) widen the index range per (level, axis)
// beyond [0, max_index] for batch_evaluate on arbitrary nodes.
std::vector<double> build_lut(const HostGrid& g, GridView* view, const int32_t* lo = nullptr,
                              const int32_t* hi = nullptr);

// prepare_source, pipeline.hpp:25-41 (host).
struct SourcePrep {
  std::vector<double> xyz;
  double leaf = 0.0;
  bool converged = true;
  double d_max = 0.0;
};
SourcePrep host_prepare_source(const double* xyz, uint64_t n, uint64_t target);
// voxel_grid_downsample, point_cloud.hpp:78-111 (host, the reference's
// summation order).
std::vector<double> host_voxel_grid_downsample(const double* xyz, uint64_t n, double leaf);
// The same on the device (source_prep.cu): auto_leaf's voxel counts on the
// device (exact leaf, convergence, voxel set and order).  Centroids:
// exact_centroids = true sums each voxel in the reference's std::sort order
// (host_voxel_grid_downsample at the device-found leaf: bit-identical to the
// reference); false sums on the device in input order (fast path; voxels of
// >= 3 points may differ in the last bits).
SourcePrep device_prepare_source(int device, const double* xyz, uint64_t n, uint64_t target,
                                 bool exact_centroids = true);

}  // namespace bbs

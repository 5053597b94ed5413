// host_grid.cpp — host-side restatements that feed the device path.
//
// Compiled with g++ -O2 -ffp-contract=off (no -march): every double
// expression rounds exactly like the reference build, and the
// cos/sin/asin/floor/ceil come from the same host libm the reference uses.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <tuple>

#include "bbs_internal.h"

namespace bbs {

namespace {
constexpr double kPi = 3.141592653589793238462643383279502884;

// angular_step, angular_grid.hpp:20-26.
double angular_step(double cell, double d_max) {
  if (!(d_max > 0.0)) throw Error(BBS_ERR_DEGENERATE_SCAN, "angular_step: d_max must be > 0");
  if (!(cell > 0.0)) throw Error(BBS_ERR_CONFIG, "angular_step: cell must be > 0");
  const double half_chord = cell / (2.0 * d_max);
  if (half_chord >= 1.0) return kPi;
  return 2.0 * std::asin(half_chord);
}

// adjusted_step, angular_grid.hpp:34-39.
void adjusted_step(double range, double step, double* out_step, int* out_segments) {
  if (!(range > 0.0)) throw Error(BBS_ERR_CONFIG, "adjusted_step: range must be > 0");
  if (!(step > 0.0)) throw Error(BBS_ERR_CONFIG, "adjusted_step: step must be > 0");
  const int segments = static_cast<int>(std::ceil(range / step));
  *out_step = range / static_cast<double>(segments);
  *out_segments = segments;
}
}  // namespace

// AngularGrid ctor, angular_grid.hpp:67-99.
HostGrid make_grid(const bbs_search_config& cfg, double d_max) {
  if (!(cfg.yaw_max > cfg.yaw_min))
    throw Error(BBS_ERR_CONFIG, "AngularGrid: yaw range must have positive width");
  if (cfg.roll_pitch_half_range < 0.0)
    throw Error(BBS_ERR_CONFIG, "AngularGrid: roll/pitch range must be >= 0");
  if (cfg.max_level < 0 || cfg.max_level >= kMaxLevels)
    throw Error(BBS_ERR_CONFIG, "AngularGrid: max_level out of the supported range [0, 15]");
  HostGrid g;
  g.max_level = cfg.max_level;
  g.axes.resize(static_cast<std::size_t>(3 * (cfg.max_level + 1)));
  const double rp = cfg.roll_pitch_half_range;
  const double w_min[3] = {-rp, -rp, cfg.yaw_min};
  const double w_max[3] = {rp, rp, cfg.yaw_max};
  const bool periodic[3] = {false, false, true};
  for (int axis = 0; axis < 3; ++axis) {
    for (int l = 0; l <= cfg.max_level; ++l) {
      const int step_level = (cfg.branch_mode == BBS_BRANCH_TRANS_ONLY) ? 0 : l;
      const double cell = std::ldexp(cfg.min_resolution, step_level);
      const double delta = angular_step(cell, d_max);
      AxisGrid a;
      a.w_min = w_min[axis];
      a.w_max = w_max[axis];
      a.periodic = periodic[axis];
      const double range = a.w_max - a.w_min;
      if (range > 0.0) adjusted_step(range, delta, &a.step, &a.segments);
      g.axes[static_cast<std::size_t>(axis * (cfg.max_level + 1) + l)] = a;
    }
  }
  return g;
}

// AngularGrid::divisions, angular_grid.hpp:111-116.
int HostGrid::divisions(int a, int l) const {
  const AxisGrid& parent = axis(a, l);
  const AxisGrid& child = axis(a, l - 1);
  if (child.segments <= 1) return 1;
  return (child.segments + parent.segments - 1) / parent.segments;
}

uint64_t max_children(const HostGrid& g) {
  uint64_t m = 8;
  for (int l = 1; l <= g.max_level; ++l) {
    const uint64_t c = 8ull * static_cast<uint64_t>(g.divisions(0, l)) *
                       static_cast<uint64_t>(g.divisions(1, l)) *
                       static_cast<uint64_t>(g.divisions(2, l));
    m = std::max(m, c);
  }
  return m;
}

std::vector<double> build_lut(const HostGrid& g, GridView* view, const int32_t* lo,
                              const int32_t* hi) {
  std::vector<double> lut;
  std::memset(view, 0, sizeof(*view));
  view->max_level = g.max_level;
  for (int l = 0; l <= g.max_level; ++l) {
    for (int a = 0; a < 3; ++a) {
      const AxisGrid& ax = g.axis(a, l);
      const int i0 = lo ? std::min(0, lo[l * 3 + a]) : 0;
      const int i1 = hi ? std::max(ax.max_index(), hi[l * 3 + a]) : ax.max_index();
      view->lut_off[l * 3 + a] = static_cast<int32_t>(lut.size() / 2);
      view->lut_lo[l * 3 + a] = i0;
      view->lut_n[l * 3 + a] = i1 - i0 + 1;
      view->max_index[l * 3 + a] = ax.max_index();
      view->div[l * 3 + a] = l >= 1 ? g.divisions(a, l) : 1;
      for (int i = i0; i <= i1; ++i) {
        // pose_to_transform, geometry.hpp:103-105, on AxisGrid::angle (:57)
        const double ang = ax.angle(i);
        lut.push_back(std::cos(ang));
        lut.push_back(std::sin(ang));
      }
    }
  }
  return lut;
}

// max_range, point_cloud.hpp:58-63.
double host_max_range(const double* xyz, uint64_t n) {
  if (n == 0) throw Error(BBS_ERR_EMPTY_CLOUD, "max_range: empty cloud");
  double m = 0.0;
  for (uint64_t i = 0; i < n; ++i) {
    const double x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
    m = std::max(m, std::sqrt(x * x + y * y + z * z));
  }
  return m;
}

// bounding_box, point_cloud.hpp:42-54.
bbs_aabb host_bounding_box(const double* xyz, uint64_t n) {
  if (n == 0) throw Error(BBS_ERR_EMPTY_CLOUD, "bounding_box: empty cloud");
  bbs_aabb b{{xyz[0], xyz[1], xyz[2]}, {xyz[0], xyz[1], xyz[2]}};
  for (uint64_t i = 0; i < n; ++i) {
    b.min.x = std::min(b.min.x, xyz[3 * i]);
    b.min.y = std::min(b.min.y, xyz[3 * i + 1]);
    b.min.z = std::min(b.min.z, xyz[3 * i + 2]);
    b.max.x = std::max(b.max.x, xyz[3 * i]);
    b.max.y = std::max(b.max.y, xyz[3 * i + 1]);
    b.max.z = std::max(b.max.z, xyz[3 * i + 2]);
  }
  return b;
}

// voxel_index, point_cloud.hpp:38-40, with the x86 cvttsd2si result for
// values outside int32 (INT32_MIN) made explicit.
int32_t host_voxel_index(double c, double cell) {
  const double f = std::floor(c / cell);
  if (!(f >= -2147483648.0 && f < 2147483648.0)) return std::numeric_limits<int32_t>::min();
  return static_cast<int32_t>(f);
}

// ---- prepare_source (host for now) ----------------------
namespace {

int64_t to_i64(double f) {
  // static_cast<int64_t>(double) on x86-64 is cvttsd2si (64-bit): INT64_MIN
  // for NaN and out-of-range values.
  if (!(f >= -9223372036854775808.0 && f < 9223372036854775808.0))
    return std::numeric_limits<int64_t>::min();
  return static_cast<int64_t>(f);
}

struct VoxelAccum {  // point_cloud.hpp:66-70
  int64_t vx, vy, vz;
  double sx, sy, sz;
  uint32_t count;
};

// voxel_grid_downsample, point_cloud.hpp:78-111.  The reference std::sorts
// 40-byte VoxelAccum records by (vx, vy, vz) and sums each voxel's points in
// the sorted order.  libstdc++'s introsort takes every decision from the
// comparator alone, so ANY element type whose comparisons come out the same
// yields the same permutation: when the voxel box packs into 64 bits, a
// monotone packed key + point index (16 B) is sorted instead (same
// permutation, ~2.5x less data moved); otherwise the reference's own record
// layout is sorted.  Either way the sums run in the reference's order.
std::vector<double> voxel_grid_downsample(const double* xyz, uint64_t n, double leaf) {
  if (n == 0) throw Error(BBS_ERR_EMPTY_CLOUD, "voxel_grid_downsample: empty cloud");
  if (!(leaf > 0.0)) throw Error(BBS_ERR_CONFIG, "voxel_grid_downsample: leaf must be > 0");
  std::vector<int64_t> v(3 * n);
  int64_t mn[3] = {INT64_MAX, INT64_MAX, INT64_MAX}, mx[3] = {INT64_MIN, INT64_MIN, INT64_MIN};
  for (uint64_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) {
      const int64_t c = to_i64(std::floor(xyz[3 * i + a] / leaf));
      v[3 * i + a] = c;
      mn[a] = std::min(mn[a], c);
      mx[a] = std::max(mx[a], c);
    }
  int bits[3];
  for (int a = 0; a < 3; ++a) {
    const uint64_t span = static_cast<uint64_t>(mx[a]) - static_cast<uint64_t>(mn[a]);
    bits[a] = 0;
    while (bits[a] < 64 && (span >> bits[a]) != 0) ++bits[a];
  }
  std::vector<double> out;
  auto emit = [&](auto&& point_of, std::size_t m, auto&& same) {
    std::size_t i = 0;
    while (i < m) {
      std::size_t j = i + 1;
      const double* p0 = point_of(i);
      double sx = p0[0], sy = p0[1], sz = p0[2];
      while (j < m && same(i, j)) {
        const double* p = point_of(j);
        sx += p[0];
        sy += p[1];
        sz += p[2];
        ++j;
      }
      const double cnt = static_cast<double>(j - i);
      out.push_back(sx / cnt);
      out.push_back(sy / cnt);
      out.push_back(sz / cnt);
      i = j;
    }
  };
  if (bits[0] + bits[1] + bits[2] <= 64) {
    struct KeyIdx {
      uint64_t key;
      uint64_t idx;
    };
    std::vector<KeyIdx> cells(n);
    for (uint64_t i = 0; i < n; ++i) {
      const uint64_t kx = static_cast<uint64_t>(v[3 * i]) - static_cast<uint64_t>(mn[0]);
      const uint64_t ky = static_cast<uint64_t>(v[3 * i + 1]) - static_cast<uint64_t>(mn[1]);
      const uint64_t kz = static_cast<uint64_t>(v[3 * i + 2]) - static_cast<uint64_t>(mn[2]);
      auto shl = [](uint64_t x, int b) { return b >= 64 ? uint64_t(0) : x << b; };
      cells[i] = {shl(shl(kx, bits[1]) | ky, bits[2]) | kz, i};  // monotone in (vx, vy, vz)
    }
    std::sort(cells.begin(), cells.end(), [](const KeyIdx& a, const KeyIdx& b) { return a.key < b.key; });
    emit([&](std::size_t i) { return xyz + 3 * cells[i].idx; }, cells.size(),
         [&](std::size_t i, std::size_t j) { return cells[j].key == cells[i].key; });
    return out;
  }
  std::vector<VoxelAccum> cells;
  cells.reserve(n);
  for (uint64_t i = 0; i < n; ++i)
    cells.push_back({v[3 * i], v[3 * i + 1], v[3 * i + 2], xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], 1});
  std::sort(cells.begin(), cells.end(), [](const VoxelAccum& a, const VoxelAccum& b) {
    return std::tie(a.vx, a.vy, a.vz) < std::tie(b.vx, b.vy, b.vz);
  });
  emit([&](std::size_t i) { return &cells[i].sx; }, cells.size(), [&](std::size_t i, std::size_t j) {
    return cells[j].vx == cells[i].vx && cells[j].vy == cells[i].vy && cells[j].vz == cells[i].vz;
  });
  return out;
}

// count_voxels, point_cloud.hpp:115-125.
std::size_t count_voxels(const double* xyz, uint64_t n, double leaf) {
  std::vector<std::tuple<int64_t, int64_t, int64_t>> v;
  v.reserve(n);
  for (uint64_t i = 0; i < n; ++i)
    v.emplace_back(to_i64(std::floor(xyz[3 * i] / leaf)), to_i64(std::floor(xyz[3 * i + 1] / leaf)),
                   to_i64(std::floor(xyz[3 * i + 2] / leaf)));
  std::sort(v.begin(), v.end());
  return static_cast<std::size_t>(std::unique(v.begin(), v.end()) - v.begin());
}

struct AutoLeaf {
  double leaf;
  std::size_t count;
  bool converged;
};

// auto_leaf, point_cloud.hpp:137-182.
AutoLeaf auto_leaf(const double* xyz, uint64_t n, std::size_t target) {
  if (n == 0) throw Error(BBS_ERR_EMPTY_CLOUD, "auto_leaf: empty cloud");
  if (target < 1) throw Error(BBS_ERR_CONFIG, "auto_leaf: target must be >= 1");
  const std::size_t lo_count = std::max<std::size_t>(1, (target + 1) / 2);
  const std::size_t hi_count = 2 * target;
  const bbs_aabb box = host_bounding_box(xyz, n);
  const double ex = box.max.x - box.min.x, ey = box.max.y - box.min.y,
               ez = box.max.z - box.min.z;
  const double max_ext = std::max({ex, ey, ez, 1e-9});
  double lo = max_ext / (1 << 24);
  double hi = max_ext;
  {
    const std::size_t c = count_voxels(xyz, n, lo);
    if (c <= hi_count && (c >= lo_count || c == n)) return {lo, c, true};
  }
  double best_leaf = lo;
  std::size_t best_count = 0;
  double best_gap = std::numeric_limits<double>::infinity();
  for (int iter = 0; iter < 32; ++iter) {
    const double mid = std::sqrt(lo * hi);
    const std::size_t c = count_voxels(xyz, n, mid);
    if (c >= lo_count && c <= hi_count) return {mid, c, true};
    const double gap = std::abs(std::log(static_cast<double>(std::max<std::size_t>(c, 1))) -
                                std::log(static_cast<double>(target)));
    if (gap < best_gap) {
      best_gap = gap;
      best_leaf = mid;
      best_count = c;
    }
    if (c > hi_count)
      lo = mid;
    else
      hi = mid;
  }
  return {best_leaf, best_count, false};
}

}  // namespace

std::vector<double> host_voxel_grid_downsample(const double* xyz, uint64_t n, double leaf) {
  return voxel_grid_downsample(xyz, n, leaf);
}

// prepare_source, pipeline.hpp:25-41.
SourcePrep host_prepare_source(const double* xyz, uint64_t n, uint64_t target) {
  SourcePrep p;
  if (target > 0 && n > target) {
    const AutoLeaf a = auto_leaf(xyz, n, target);
    p.xyz = voxel_grid_downsample(xyz, n, a.leaf);
    p.leaf = a.leaf;
    p.converged = a.converged;
  } else {
    p.xyz.assign(xyz, xyz + 3 * n);
  }
  p.d_max = host_max_range(p.xyz.data(), p.xyz.size() / 3);
  return p;
}

}  // namespace bbs

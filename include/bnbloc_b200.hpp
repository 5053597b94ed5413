// bnbloc_b200.hpp — header-only C++17 facade over the C-ABI (include/bbs.h).
//
// Re-exposes the reference's localizer API (namespace bnbloc,
// /root/reference/proj/include/bnbloc/*.hpp) with the same type names,
// member functions, free functions and exception classes, backed by the
// B200 device path (libbbs_b200.so).  Define BNBLOC_B200_AS_BNBLOC before
// including to make `bnbloc::` an alias of `bnbloc_b200::` (drop-in
// replacement; do not combine with the reference headers in one TU).
//
// Device-backed: MultiResVoxelMap (build/from_levels), LevelMap
// (contains/lookup/score/occupied_voxels), batch_evaluate, search,
// localize_scan.  Host restatements (exact, same libm): AngularGrid,
// angular_step, adjusted_step, node_pose, initial_nodes, branch,
// trans_index_range, pose_to_transform, Transform, max_range,
// bounding_box, prepare_source, spatial_hash, Rng.
#ifndef BNBLOC_B200_HPP
#define BNBLOC_B200_HPP

#include <algorithm>
#include <array>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <limits>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "bbs.h"

namespace bnbloc_b200 {

// ---- errors (errors.hpp:11-98) ---------------------------------------------
class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};
class FileNotFoundError : public Error {
 public:
  explicit FileNotFoundError(const std::string& w) : Error(w) {}
};
class ParseError : public Error {
 public:
  explicit ParseError(const std::string& w) : Error(w) {}
};
class EmptyCloudError : public Error {
 public:
  explicit EmptyCloudError(const std::string& w = "point cloud is empty") : Error(w) {}
};
class CapacityExceededError : public Error {
 public:
  explicit CapacityExceededError(const std::string& w) : Error(w) {}
};
class IoError : public Error {
 public:
  explicit IoError(const std::string& w) : Error(w) {}
};
class FormatError : public Error {
 public:
  explicit FormatError(const std::string& w) : Error(w) {}
};
class DegenerateScanError : public Error {
 public:
  explicit DegenerateScanError(const std::string& w) : Error(w) {}
};
class EmptySearchSpaceError : public Error {
 public:
  explicit EmptySearchSpaceError(const std::string& w) : Error(w) {}
};
class TooLargeError : public Error {
 public:
  explicit TooLargeError(const std::string& w) : Error(w) {}
};
class InfeasiblePoseError : public Error {
 public:
  explicit InfeasiblePoseError(const std::string& w) : Error(w) {}
};
class ConfigError : public Error {
 public:
  explicit ConfigError(const std::string& w) : Error(w) {}
};
class CudaError : public Error {  // no reference counterpart
 public:
  explicit CudaError(const std::string& w) : Error(w) {}
};

namespace detail {
[[noreturn]] inline void throw_status(int st, const char* msg) {
  const std::string m = msg ? msg : "";
  switch (st) {
    case BBS_ERR_FILE_NOT_FOUND: throw FileNotFoundError(m);
    case BBS_ERR_PARSE: throw ParseError(m);
    case BBS_ERR_EMPTY_CLOUD: throw EmptyCloudError(m);
    case BBS_ERR_CAPACITY_EXCEEDED: throw CapacityExceededError(m);
    case BBS_ERR_IO: throw IoError(m);
    case BBS_ERR_FORMAT: throw FormatError(m);
    case BBS_ERR_DEGENERATE_SCAN: throw DegenerateScanError(m);
    case BBS_ERR_EMPTY_SEARCH_SPACE: throw EmptySearchSpaceError(m);
    case BBS_ERR_TOO_LARGE: throw TooLargeError(m);
    case BBS_ERR_INFEASIBLE_POSE: throw InfeasiblePoseError(m);
    case BBS_ERR_CONFIG: throw ConfigError(m);
    case BBS_ERR_CUDA: throw CudaError(m);
    default: throw Error(m);
  }
}
inline void check(int st) {
  if (st != BBS_OK) throw_status(st, bbs_last_error());
}
// The structs of bbs.h are passed by pointer: refuse a library built from a
// different header version.
inline void check_abi() {
  if (bbs_abi_version() != BBS_ABI_VERSION)
    throw Error("libbbs_b200.so ABI version " + std::to_string(bbs_abi_version()) +
                " does not match bbs.h version " + std::to_string(BBS_ABI_VERSION));
}
}  // namespace detail

// ---- geometry (geometry.hpp) ------------------------------------------------
inline constexpr double kTwoPi = 6.283185307179586476925286766559;

struct Point3 {
  double x = 0.0, y = 0.0, z = 0.0;
  friend Point3 operator+(const Point3& a, const Point3& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
  friend Point3 operator-(const Point3& a, const Point3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
  friend Point3 operator*(double s, const Point3& p) { return {s * p.x, s * p.y, s * p.z}; }
  double norm() const { return std::sqrt(x * x + y * y + z * z); }
  bool finite() const { return std::isfinite(x) && std::isfinite(y) && std::isfinite(z); }
};

inline double normalize_angle(double a) {
  double r = std::fmod(a, kTwoPi);
  if (r < 0.0) r += kTwoPi;
  if (r >= kTwoPi) r = 0.0;
  return r;
}

struct Pose6 {
  double x = 0.0, y = 0.0, z = 0.0, roll = 0.0, pitch = 0.0, yaw = 0.0;
  Pose6 normalized() const {
    Pose6 p = *this;
    p.yaw = normalize_angle(yaw);
    return p;
  }
};

struct Transform {
  std::array<double, 9> rotation = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  Point3 translation;
  Point3 apply(const Point3& p) const {
    const auto& r = rotation;
    return {r[0] * p.x + r[1] * p.y + r[2] * p.z + translation.x,
            r[3] * p.x + r[4] * p.y + r[5] * p.z + translation.y,
            r[6] * p.x + r[7] * p.y + r[8] * p.z + translation.z};
  }
  Transform compose(const Transform& o) const {
    Transform t;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double s = 0.0;
        for (int k = 0; k < 3; ++k) s += rotation[3 * i + k] * o.rotation[3 * k + j];
        t.rotation[3 * i + j] = s;
      }
    t.translation = apply(o.translation);
    return t;
  }
  Transform inverse() const {
    Transform t;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) t.rotation[3 * i + j] = rotation[3 * j + i];
    const Point3 nt{-translation.x, -translation.y, -translation.z};
    t.translation = {t.rotation[0] * nt.x + t.rotation[1] * nt.y + t.rotation[2] * nt.z,
                     t.rotation[3] * nt.x + t.rotation[4] * nt.y + t.rotation[5] * nt.z,
                     t.rotation[6] * nt.x + t.rotation[7] * nt.y + t.rotation[8] * nt.z};
    return t;
  }
};

inline Transform pose_to_transform(const Pose6& p) {
  const double ca = std::cos(p.roll), sa = std::sin(p.roll);
  const double cb = std::cos(p.pitch), sb = std::sin(p.pitch);
  const double cg = std::cos(p.yaw), sg = std::sin(p.yaw);
  Transform t;
  t.rotation = {cg * cb, cg * sb * sa - sg * ca, cg * sb * ca + sg * sa,
                sg * cb, sg * sb * sa + cg * ca, sg * sb * ca - cg * sa,
                -sb,     cb * sa,                cb * ca};
  t.translation = {p.x, p.y, p.z};
  return t;
}
inline Point3 transform_point(const Transform& t, const Point3& p) { return t.apply(p); }
inline double rotation_error(const Pose6& a, const Pose6& b) {
  const Transform ta = pose_to_transform(a), tb = pose_to_transform(b);
  double tr = 0.0;
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k) tr += ta.rotation[3 * k + i] * tb.rotation[3 * k + i];
  double c = 0.5 * (tr - 1.0);
  c = std::min(1.0, std::max(-1.0, c));
  return std::acos(c);
}
inline double translation_error(const Pose6& a, const Pose6& b) {
  return (Point3{a.x, a.y, a.z} - Point3{b.x, b.y, b.z}).norm();
}

// ---- point clouds (point_cloud.hpp) ------------------------------------------
struct PointCloud {
  std::vector<Point3> points;
  std::size_t size() const { return points.size(); }
  bool empty() const { return points.empty(); }
};
static_assert(sizeof(Point3) == 3 * sizeof(double), "Point3 must be packed xyz");

struct Aabb {
  Point3 min, max;
  Point3 extent() const { return max - min; }
  bool contains(const Point3& p) const {
    return p.x >= min.x && p.x <= max.x && p.y >= min.y && p.y <= max.y && p.z >= min.z &&
           p.z <= max.z;
  }
};

inline const double* xyz(const PointCloud& c) {
  return c.points.empty() ? nullptr : &c.points.front().x;
}

inline std::int32_t voxel_index(double coord, double cell) {
  return static_cast<std::int32_t>(std::floor(coord / cell));
}
inline Aabb bounding_box(const PointCloud& c) {
  bbs_aabb b;
  detail::check(bbs_bounding_box(xyz(c), c.size(), &b));
  return {{b.min.x, b.min.y, b.min.z}, {b.max.x, b.max.y, b.max.z}};
}
inline double max_range(const PointCloud& c) {
  double d = 0;
  detail::check(bbs_max_range(xyz(c), c.size(), &d));
  return d;
}

// ---- rng (rng.hpp), used by the reference's tests ------------------------------
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : state_(seed) {}
  std::uint64_t next_u64() {
    std::uint64_t z = (state_ += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * next_double(); }
  std::int64_t uniform_int(std::int64_t lo, std::int64_t hi) {
    const std::uint64_t span = static_cast<std::uint64_t>(hi - lo) + 1;
    return lo + static_cast<std::int64_t>(next_u64() % span);
  }

 private:
  std::uint64_t state_;
};

// ---- search config / results (search_config.hpp) --------------------------------
enum class Strategy { kDfs, kBfs };
enum class BranchMode { kTransOnly, kRotoTrans };

struct SearchConfig {
  double min_resolution = 1.0;
  int max_level = 6;
  std::optional<Aabb> translation_range;
  double roll_pitch_half_range = 0.02;
  double yaw_min = 0.0;
  double yaw_max = kTwoPi;
  double score_threshold_fraction = 0.95;
  std::size_t batch_size = 10000;
  Strategy strategy = Strategy::kBfs;
  BranchMode branch_mode = BranchMode::kRotoTrans;
  int workers = 1;
  std::optional<double> d_max;
  bool collect_trace = false;
};

struct Stats {
  std::uint64_t nodes_generated = 0, nodes_pruned = 0, batches_flushed = 0;
  double create_voxel_maps_ms = 0.0, set_source_ms = 0.0, initial_nodes_ms = 0.0,
         find_best_score_ms = 0.0, pop_remaining_queue_ms = 0.0;
  double preprocessing_total_ms() const { return create_voxel_maps_ms + set_source_ms; }
  double localization_total_ms() const {
    return initial_nodes_ms + find_best_score_ms + pop_remaining_queue_ms;
  }
};

struct SearchResult {
  Pose6 best_pose;
  int best_score = 0;
  int score_threshold = 0;
  std::size_t scan_points = 0;
  bool matched = false;
  Stats stats;
  std::vector<int> best_score_trace;
};

namespace detail {
inline bbs_search_config to_c(const SearchConfig& s) {
  bbs_search_config c;
  bbs_search_config_default(&c);
  c.min_resolution = s.min_resolution;
  c.max_level = s.max_level;
  if (s.translation_range) {
    const Aabb& r = *s.translation_range;
    c.has_translation_range = 1;
    c.translation_range = {{r.min.x, r.min.y, r.min.z}, {r.max.x, r.max.y, r.max.z}};
  }
  c.roll_pitch_half_range = s.roll_pitch_half_range;
  c.yaw_min = s.yaw_min;
  c.yaw_max = s.yaw_max;
  c.score_threshold_fraction = s.score_threshold_fraction;
  c.batch_size = s.batch_size;
  c.strategy = s.strategy == Strategy::kDfs ? BBS_STRATEGY_DFS : BBS_STRATEGY_BFS;
  c.branch_mode = s.branch_mode == BranchMode::kTransOnly ? BBS_BRANCH_TRANS_ONLY : BBS_BRANCH_ROTO_TRANS;
  c.workers = s.workers;
  if (s.d_max) {
    c.has_d_max = 1;
    c.d_max = *s.d_max;
  }
  c.collect_trace = s.collect_trace ? 1 : 0;
  return c;
}
}  // namespace detail

// ---- angular grid (angular_grid.hpp), host restatement --------------------------
inline double angular_step(double cell, double d_max) {
  if (!(d_max > 0.0)) throw DegenerateScanError("angular_step: d_max must be > 0");
  if (!(cell > 0.0)) throw ConfigError("angular_step: cell must be > 0");
  const double half_chord = cell / (2.0 * d_max);
  if (half_chord >= 1.0) return 3.141592653589793238462643383279502884;
  return 2.0 * std::asin(half_chord);
}
struct AdjustedStep {
  double step = 0.0;
  int segments = 0;
};
inline AdjustedStep adjusted_step(double range, double step) {
  if (!(range > 0.0)) throw ConfigError("adjusted_step: range must be > 0");
  if (!(step > 0.0)) throw ConfigError("adjusted_step: step must be > 0");
  const int segments = static_cast<int>(std::ceil(range / step));
  return {range / static_cast<double>(segments), segments};
}
struct AxisGrid {
  double w_min = 0.0, w_max = 0.0, step = 0.0;
  int segments = 0;
  bool periodic = false;
  int max_index() const { return segments == 0 ? 0 : (periodic ? segments - 1 : segments); }
  int index_count() const { return max_index() + 1; }
  double angle(int index) const { return w_min + step * static_cast<double>(index); }
};

class AngularGrid {
 public:
  AngularGrid(const SearchConfig& cfg, double d_max) : cfg_(detail::to_c(cfg)), d_max_(d_max) {
    max_level_ = cfg.max_level;
    std::vector<bbs_axis_grid> g(3 * static_cast<std::size_t>(cfg.max_level + 1));
    detail::check(bbs_angular_grid(&cfg_, d_max, g.data(), g.size()));
    for (const auto& a : g) axes_.push_back({a.w_min, a.w_max, a.step, a.segments, a.periodic != 0});
  }
  int max_level() const { return max_level_; }
  const AxisGrid& axis(int a, int l) const {
    return axes_[static_cast<std::size_t>(a * (max_level_ + 1) + l)];
  }
  int divisions(int a, int l) const {
    const AxisGrid& parent = axis(a, l);
    const AxisGrid& child = axis(a, l - 1);
    if (child.segments <= 1) return 1;
    return (child.segments + parent.segments - 1) / parent.segments;
  }
  const bbs_search_config& c_config() const { return cfg_; }
  double d_max() const { return d_max_; }

 private:
  bbs_search_config cfg_;
  double d_max_;
  int max_level_ = 0;
  std::vector<AxisGrid> axes_;
};

// ---- nodes (nodes.hpp), host restatement ----------------------------------------
struct Node {
  std::int32_t ix = 0, iy = 0, iz = 0, iroll = 0, ipitch = 0, iyaw = 0, level = 0, score = -1;
  bool is_leaf() const { return level == 0; }
};
static_assert(sizeof(Node) == sizeof(bbs_node), "Node must be byte-compatible with bbs_node");

inline Pose6 node_pose(const Node& c, const AngularGrid& grids, double min_resolution) {
  const double cell = std::ldexp(min_resolution, c.level);
  Pose6 p;
  p.x = cell * static_cast<double>(c.ix);
  p.y = cell * static_cast<double>(c.iy);
  p.z = cell * static_cast<double>(c.iz);
  p.roll = grids.axis(0, c.level).angle(c.iroll);
  p.pitch = grids.axis(1, c.level).angle(c.ipitch);
  p.yaw = grids.axis(2, c.level).angle(c.iyaw);
  return p;
}
struct TransIndexRange {
  std::int32_t min = 0, max = 0;
  std::int64_t count() const { return static_cast<std::int64_t>(max) - min + 1; }
};
inline TransIndexRange trans_index_range(double w_min, double w_max, double cell) {
  return {static_cast<std::int32_t>(std::floor(w_min / cell)),
          static_cast<std::int32_t>(std::ceil(w_max / cell))};
}
inline std::vector<Node> initial_nodes(const Aabb& r, const AngularGrid& grids, double min_resolution) {
  const int l = grids.max_level();
  const double cell = std::ldexp(min_resolution, l);
  const auto rx = trans_index_range(r.min.x, r.max.x, cell), ry = trans_index_range(r.min.y, r.max.y, cell),
             rz = trans_index_range(r.min.z, r.max.z, cell);
  const int nr = grids.axis(0, l).index_count(), np = grids.axis(1, l).index_count(),
            nw = grids.axis(2, l).index_count();
  const std::int64_t total = rx.count() * ry.count() * rz.count() * nr * np * nw;
  if (total <= 0) throw EmptySearchSpaceError("initial node set is empty");
  std::vector<Node> nodes;
  nodes.reserve(static_cast<std::size_t>(total));
  for (std::int32_t ix = rx.min; ix <= rx.max; ++ix)
    for (std::int32_t iy = ry.min; iy <= ry.max; ++iy)
      for (std::int32_t iz = rz.min; iz <= rz.max; ++iz)
        for (std::int32_t ir = 0; ir < nr; ++ir)
          for (std::int32_t ip = 0; ip < np; ++ip)
            for (std::int32_t iw = 0; iw < nw; ++iw) nodes.push_back({ix, iy, iz, ir, ip, iw, l, -1});
  return nodes;
}
inline std::vector<Node> branch(const Node& c, const AngularGrid& grids) {
  if (c.level <= 0) throw ConfigError("branch: leaf nodes cannot be branched");
  const int cl = c.level - 1;
  const int ar = grids.divisions(0, c.level), ap = grids.divisions(1, c.level),
            aw = grids.divisions(2, c.level);
  const int mr = grids.axis(0, cl).max_index(), mp = grids.axis(1, cl).max_index(),
            mw = grids.axis(2, cl).max_index();
  std::vector<Node> out;
  for (std::int32_t jr = 0; jr < ar; ++jr) {
    const std::int32_t ir = ar * c.iroll + jr;
    if (ir > mr) break;
    for (std::int32_t jp = 0; jp < ap; ++jp) {
      const std::int32_t ip = ap * c.ipitch + jp;
      if (ip > mp) break;
      for (std::int32_t jw = 0; jw < aw; ++jw) {
        const std::int32_t iw = aw * c.iyaw + jw;
        if (iw > mw) break;
        for (std::int32_t jx = 0; jx <= 1; ++jx)
          for (std::int32_t jy = 0; jy <= 1; ++jy)
            for (std::int32_t jz = 0; jz <= 1; ++jz)
              out.push_back({2 * c.ix + jx, 2 * c.iy + jy, 2 * c.iz + jz, ir, ip, iw, cl, -1});
      }
    }
  }
  return out;
}

// ---- voxel map (voxel_map.hpp), device-backed -----------------------------------
struct VoxelCoord {
  std::int32_t x = 0, y = 0, z = 0;
  friend bool operator==(const VoxelCoord& a, const VoxelCoord& b) {
    return a.x == b.x && a.y == b.y && a.z == b.z;
  }
  friend bool operator<(const VoxelCoord& a, const VoxelCoord& b) {
    if (a.x != b.x) return a.x < b.x;
    if (a.y != b.y) return a.y < b.y;
    return a.z < b.z;
  }
};
inline VoxelCoord voxel_of(const Point3& p, double cell) {
  return {voxel_index(p.x, cell), voxel_index(p.y, cell), voxel_index(p.z, cell)};
}
// The reference's XOR hash (voxel_map.hpp:39-52); the device tables use
// their own layout, but the function is part of the public API.
inline std::uint64_t voxel_hash(const VoxelCoord& v) {
  return (static_cast<std::uint64_t>(static_cast<std::int64_t>(v.x)) * 73856093ULL) ^
         (static_cast<std::uint64_t>(static_cast<std::int64_t>(v.y)) * 19349663ULL) ^
         (static_cast<std::uint64_t>(static_cast<std::int64_t>(v.z)) * 83492791ULL);
}
inline std::uint64_t spatial_hash(const VoxelCoord& v, std::uint64_t bucket_count) {
  return voxel_hash(v) % bucket_count;
}

namespace detail {
struct MapHandle {
  bbs_map_t h = nullptr;
  ~MapHandle() {
    if (h) bbs_map_free(h);
  }
};
}  // namespace detail

class LevelMap {
 public:
  static constexpr std::size_t kDefaultMemoryCapBytes = std::size_t{2} << 30;
  LevelMap() = default;
  LevelMap(std::shared_ptr<detail::MapHandle> m, int level) : m_(std::move(m)), level_(level) {
    detail::check(bbs_map_level_info(m_->h, level, &info_));
  }
  int level() const { return level_; }
  double resolution() const { return info_.resolution; }
  std::size_t occupied_count() const { return info_.occupied_count; }
  std::uint64_t bucket_count() const { return info_.bucket_count; }
  double collision_rate() const { return info_.collision_rate; }
  double load_factor() const { return info_.load_factor; }
  bool contains(const VoxelCoord& v) const {
    std::uint8_t out = 0;
    detail::check(bbs_level_contains(m_->h, level_, &v.x, 1, &out));
    return out != 0;
  }
  int lookup(const Point3& p) const { return contains(voxel_of(p, resolution())) ? 1 : 0; }
  int score(const Transform& t, const PointCloud& scan) const {
    std::int32_t s = 0;
    const double tr[3] = {t.translation.x, t.translation.y, t.translation.z};
    detail::check(bbs_level_score(m_->h, level_, t.rotation.data(), tr, xyz(scan), scan.size(), &s));
    return s;
  }
  std::vector<VoxelCoord> occupied_voxels() const {
    std::uint64_t n = 0;
    detail::check(bbs_level_occupied(m_->h, level_, nullptr, 0, &n));
    std::vector<VoxelCoord> out(n);
    if (n) detail::check(bbs_level_occupied(m_->h, level_, &out.front().x, n, &n));
    return out;
  }
  bbs_map_t handle() const { return m_->h; }

 private:
  std::shared_ptr<detail::MapHandle> m_;
  int level_ = 0;
  bbs_level_info info_{};
};
static_assert(sizeof(VoxelCoord) == 12, "VoxelCoord must be 3 x int32");

class MultiResVoxelMap {
 public:
  static constexpr double kDefaultCollisionTarget = 0.001;
  MultiResVoxelMap() = default;

  static MultiResVoxelMap build(const PointCloud& map_points, double min_resolution, int max_level,
                                double collision_target = kDefaultCollisionTarget,
                                std::size_t memory_cap_bytes = LevelMap::kDefaultMemoryCapBytes,
                                int device = 0, int layout = BBS_LAYOUT_AUTO) {
    detail::check_abi();
    auto h = std::make_shared<detail::MapHandle>();
    const bbs_map_options o{device, layout};
    detail::check(bbs_map_build(xyz(map_points), map_points.size(), min_resolution, max_level,
                                collision_target, memory_cap_bytes, &o, &h->h));
    return MultiResVoxelMap(h);
  }
  static MultiResVoxelMap from_levels(std::vector<std::vector<VoxelCoord>> per_level,
                                      double min_resolution, const Aabb& bbox,
                                      double collision_target = kDefaultCollisionTarget,
                                      std::size_t memory_cap_bytes = LevelMap::kDefaultMemoryCapBytes,
                                      int device = 0) {
    detail::check_abi();
    auto h = std::make_shared<detail::MapHandle>();
    std::vector<const std::int32_t*> ptrs;
    std::vector<std::uint64_t> counts;
    for (const auto& v : per_level) {
      ptrs.push_back(v.empty() ? nullptr : &v.front().x);
      counts.push_back(v.size());
    }
    const bbs_aabb b{{bbox.min.x, bbox.min.y, bbox.min.z}, {bbox.max.x, bbox.max.y, bbox.max.z}};
    const bbs_map_options o{device, BBS_LAYOUT_AUTO};
    detail::check(bbs_map_from_levels(ptrs.data(), counts.data(), static_cast<std::int32_t>(per_level.size()),
                                      min_resolution, &b, collision_target, memory_cap_bytes, &o, &h->h));
    return MultiResVoxelMap(h);
  }
  // load_map (map_io.hpp:67-115) into device levels
  static MultiResVoxelMap load(const std::string& path, double collision_target = kDefaultCollisionTarget,
                               std::size_t memory_cap_bytes = LevelMap::kDefaultMemoryCapBytes,
                               int device = 0) {
    detail::check_abi();
    auto h = std::make_shared<detail::MapHandle>();
    const bbs_map_options o{device, BBS_LAYOUT_AUTO};
    detail::check(bbs_map_load(path.c_str(), collision_target, memory_cap_bytes, &o, &h->h));
    return MultiResVoxelMap(h);
  }
  double min_resolution() const { return r_; }
  int max_level() const { return max_level_; }
  const Aabb& bbox() const { return bbox_; }
  const LevelMap& level(int l) const { return levels_[static_cast<std::size_t>(l)]; }
  const std::vector<LevelMap>& levels() const { return levels_; }
  bbs_map_t handle() const { return m_ ? m_->h : nullptr; }

 private:
  explicit MultiResVoxelMap(std::shared_ptr<detail::MapHandle> h) : m_(std::move(h)) {
    detail::check(bbs_map_min_resolution(m_->h, &r_));
    std::int32_t ml = 0;
    detail::check(bbs_map_max_level(m_->h, &ml));
    max_level_ = ml;
    bbs_aabb b;
    detail::check(bbs_map_bbox(m_->h, &b));
    bbox_ = {{b.min.x, b.min.y, b.min.z}, {b.max.x, b.max.y, b.max.z}};
    for (int l = 0; l <= max_level_; ++l) levels_.emplace_back(m_, l);
  }
  std::shared_ptr<detail::MapHandle> m_;
  double r_ = 1.0;
  int max_level_ = 0;
  Aabb bbox_;
  std::vector<LevelMap> levels_;
};

// ---- map_io.hpp (load_map / save_map / is_map_file), device-backed ---------
inline void save_map(const MultiResVoxelMap& map, const std::string& path) {
  detail::check(bbs_map_save(map.handle(), path.c_str()));
}
inline MultiResVoxelMap load_map(const std::string& path,
                                 double collision_target = MultiResVoxelMap::kDefaultCollisionTarget,
                                 std::size_t memory_cap_bytes = LevelMap::kDefaultMemoryCapBytes,
                                 int device = 0) {
  return MultiResVoxelMap::load(path, collision_target, memory_cap_bytes, device);
}
inline bool is_map_file(const std::string& path) { return bbs_is_map_file(path.c_str()) != 0; }

// build_level (voxel_map.hpp:209-216): a map of levels 0..max(level, 1),
// returned as the requested level (the view keeps the device map alive).
inline LevelMap build_level(const PointCloud& points, int level, double min_resolution,
                            double collision_target,
                            std::size_t memory_cap_bytes = LevelMap::kDefaultMemoryCapBytes) {
  if (points.empty()) throw EmptyCloudError("build_level: empty cloud");
  const MultiResVoxelMap m = MultiResVoxelMap::build(points, min_resolution, std::max(level, 1),
                                                     collision_target, memory_cap_bytes);
  return m.level(level);
}

// ---- search (search.hpp, pipeline.hpp), device-backed ---------------------------
inline void batch_evaluate(std::vector<Node>& nodes, const MultiResVoxelMap& map,
                           const PointCloud& scan, const AngularGrid& grids, int /*workers*/ = 1) {
  if (nodes.empty()) return;
  detail::check(bbs_batch_evaluate(map.handle(), xyz(scan), scan.size(), &grids.c_config(),
                                   grids.d_max(), reinterpret_cast<bbs_node*>(nodes.data()),
                                   nodes.size()));
}

namespace detail {
inline SearchResult to_result(const bbs_search_result& r, std::vector<std::int32_t>& trace) {
  SearchResult out;
  out.best_pose = {r.best_pose.x, r.best_pose.y, r.best_pose.z,
                   r.best_pose.roll, r.best_pose.pitch, r.best_pose.yaw};
  out.best_score = r.best_score;
  out.score_threshold = r.score_threshold;
  out.scan_points = r.scan_points;
  out.matched = r.matched != 0;
  out.stats = {r.stats.nodes_generated,   r.stats.nodes_pruned,     r.stats.batches_flushed,
               r.stats.create_voxel_maps_ms, r.stats.set_source_ms,  r.stats.initial_nodes_ms,
               r.stats.find_best_score_ms, r.stats.pop_remaining_queue_ms};
  const std::size_t n = std::min<std::size_t>(r.trace_length, trace.size());
  out.best_score_trace.assign(trace.begin(), trace.begin() + static_cast<std::ptrdiff_t>(n));
  return out;
}
}  // namespace detail

inline SearchResult search(const MultiResVoxelMap& map, const PointCloud& scan,
                           const SearchConfig& cfg) {
  const bbs_search_config c = detail::to_c(cfg);
  std::vector<std::int32_t> trace(cfg.collect_trace ? (1u << 16) : 0u);
  bbs_search_result r{};
  r.best_score_trace = trace.data();
  r.trace_capacity = trace.size();
  detail::check(bbs_search(map.handle(), xyz(scan), scan.size(), &c, &r));
  if (cfg.collect_trace && r.trace_length > trace.size()) {  // retry with the full length
    trace.resize(r.trace_length);
    r = bbs_search_result{};
    r.best_score_trace = trace.data();
    r.trace_capacity = trace.size();
    detail::check(bbs_search(map.handle(), xyz(scan), scan.size(), &c, &r));
  }
  return detail::to_result(r, trace);
}

inline SearchResult localize_scan(const MultiResVoxelMap& map, const PointCloud& raw_scan,
                                  const SearchConfig& cfg, std::size_t downsample_target) {
  const bbs_search_config c = detail::to_c(cfg);
  std::vector<std::int32_t> trace(cfg.collect_trace ? (1u << 16) : 0u);
  bbs_search_result r{};
  r.best_score_trace = trace.data();
  r.trace_capacity = trace.size();
  detail::check(bbs_localize_scan(map.handle(), xyz(raw_scan), raw_scan.size(), &c,
                                  downsample_target, &r));
  return detail::to_result(r, trace);
}

// ---- oracle.hpp:17-95, device-backed (bbs_oracle_search) ---------------------
struct OracleResult {
  int best_score = 0;
  std::vector<Pose6> argmax_poses;  ///< every leaf attaining best_score
  std::uint64_t leaf_count = 0;
};

inline constexpr std::uint64_t kOracleMaxLeaves = 100000000;  // 1e8 guard

inline OracleResult oracle_search(const MultiResVoxelMap& map, const PointCloud& scan,
                                  const SearchConfig& cfg) {
  const bbs_search_config c = detail::to_c(cfg);
  std::int32_t best = 0;
  std::uint64_t count = 0, leaves = 0;
  bbs_node* raw = nullptr;  // every argmax leaf, one pass
  detail::check(bbs_oracle_search_all(map.handle(), xyz(scan), scan.size(), &c, &best, &raw, &count,
                                      &leaves));
  const std::unique_ptr<bbs_node, void (*)(void*)> own(raw, bbs_free);
  const bbs_node* nodes = raw;
  OracleResult out;
  out.best_score = best;
  out.leaf_count = leaves;
  const AngularGrid grids(cfg, cfg.d_max ? *cfg.d_max : max_range(scan));
  out.argmax_poses.reserve(count);
  for (std::uint64_t i = 0; i < count; ++i) {
    const bbs_node& b = nodes[i];
    const Node n{b.ix, b.iy, b.iz, b.iroll, b.ipitch, b.iyaw, b.level, b.score};
    out.argmax_poses.push_back(node_pose(n, grids, cfg.min_resolution).normalized());
  }
  return out;
}

}  // namespace bnbloc_b200

#ifdef BNBLOC_B200_AS_BNBLOC
namespace bnbloc = bnbloc_b200;
#endif

#endif  // BNBLOC_B200_HPP

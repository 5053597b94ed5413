// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (never the product path).
//
// A C-ABI shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/bnbloc, header-only C++20), compiled by
// oracle/Makefile into oracle/_ref/libbnbloc_ref.so with the reference's own
// build flags (-O2 -std=gnu++20, RelWithDebInfo, proj/CMakeLists.txt:3-10;
// no -march=native, so no FMA contraction — SURVEY §8c).
//
// Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
// legs load this library, and only as the checker or the timed CPU baseline.
// Nothing here is copied from the reference: each entry point converts plain
// buffers into reference types and calls the reference function named in its
// comment.

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "bbs.h"
#include "bnbloc/map_io.hpp"
#include "bnbloc/oracle.hpp"
#include "bnbloc/pipeline.hpp"
#include "bnbloc/scene.hpp"
#include "bnbloc/search.hpp"

namespace {

thread_local std::string g_err;

int fail(int code, const char* what) {
  g_err = what;
  return code;
}

// Map the reference exception hierarchy (errors.hpp:11-98) onto bbs_status.
template <typename Fn>
int guard(Fn&& fn) {
  try {
    fn();
    return BBS_OK;
  } catch (const bnbloc::FileNotFoundError& e) {
    return fail(BBS_ERR_FILE_NOT_FOUND, e.what());
  } catch (const bnbloc::ParseError& e) {
    return fail(BBS_ERR_PARSE, e.what());
  } catch (const bnbloc::EmptyCloudError& e) {
    return fail(BBS_ERR_EMPTY_CLOUD, e.what());
  } catch (const bnbloc::CapacityExceededError& e) {
    return fail(BBS_ERR_CAPACITY_EXCEEDED, e.what());
  } catch (const bnbloc::IoError& e) {
    return fail(BBS_ERR_IO, e.what());
  } catch (const bnbloc::FormatError& e) {
    return fail(BBS_ERR_FORMAT, e.what());
  } catch (const bnbloc::DegenerateScanError& e) {
    return fail(BBS_ERR_DEGENERATE_SCAN, e.what());
  } catch (const bnbloc::EmptySearchSpaceError& e) {
    return fail(BBS_ERR_EMPTY_SEARCH_SPACE, e.what());
  } catch (const bnbloc::TooLargeError& e) {
    return fail(BBS_ERR_TOO_LARGE, e.what());
  } catch (const bnbloc::InfeasiblePoseError& e) {
    return fail(BBS_ERR_INFEASIBLE_POSE, e.what());
  } catch (const bnbloc::ConfigError& e) {
    return fail(BBS_ERR_CONFIG, e.what());
  } catch (const bnbloc::Error& e) {
    return fail(BBS_ERR_GENERIC, e.what());
  } catch (const std::exception& e) {
    return fail(BBS_ERR_GENERIC, e.what());
  }
}

bnbloc::PointCloud to_cloud(const double* xyz, std::uint64_t n) {
  bnbloc::PointCloud c;
  c.points.resize(n);
  for (std::uint64_t i = 0; i < n; ++i) c.points[i] = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
  return c;
}

double* to_buffer(const bnbloc::PointCloud& c) {
  double* out = static_cast<double*>(std::malloc(sizeof(double) * 3 * (c.size() ? c.size() : 1)));
  for (std::size_t i = 0; i < c.size(); ++i) {
    out[3 * i] = c.points[i].x;
    out[3 * i + 1] = c.points[i].y;
    out[3 * i + 2] = c.points[i].z;
  }
  return out;
}

bnbloc::SearchConfig to_cfg(const bbs_search_config* c) {
  bnbloc::SearchConfig s;
  s.min_resolution = c->min_resolution;
  s.max_level = c->max_level;
  if (c->has_translation_range) {
    const auto& r = c->translation_range;
    s.translation_range = bnbloc::Aabb{{r.min.x, r.min.y, r.min.z}, {r.max.x, r.max.y, r.max.z}};
  }
  s.roll_pitch_half_range = c->roll_pitch_half_range;
  s.yaw_min = c->yaw_min;
  s.yaw_max = c->yaw_max;
  s.score_threshold_fraction = c->score_threshold_fraction;
  s.batch_size = c->batch_size;
  s.strategy = c->strategy == BBS_STRATEGY_DFS ? bnbloc::Strategy::kDfs : bnbloc::Strategy::kBfs;
  s.branch_mode = c->branch_mode == BBS_BRANCH_TRANS_ONLY ? bnbloc::BranchMode::kTransOnly
                                                          : bnbloc::BranchMode::kRotoTrans;
  s.workers = c->workers;
  if (c->has_d_max) s.d_max = c->d_max;
  s.collect_trace = c->collect_trace != 0;
  return s;
}

void to_node(const bnbloc::Node& n, bbs_node* o) {
  *o = {n.ix, n.iy, n.iz, n.iroll, n.ipitch, n.iyaw, n.level, n.score};
}

}  // namespace

extern "C" {

// Scene spec in plain C (SceneSpec, scene.hpp:21-38).
typedef struct ref_scene_spec {
  double size_x, size_y, size_z;
  int32_t num_boxes;
  double min_box_side, max_box_side, min_box_height;
  double map_spacing, scan_spacing, scan_range, point_jitter;
  int32_t tilt_noise;
  double gt_yaw_min, gt_yaw_max;
  uint64_t min_scan_points;
  double feasibility_resolution;
} ref_scene_spec;

const char* ref_last_error(void) { return g_err.c_str(); }
void ref_free(void* p) { std::free(p); }

void ref_scene_spec_default(ref_scene_spec* s) {
  const bnbloc::SceneSpec d;
  *s = {d.size_x,      d.size_y,       d.size_z,       d.num_boxes,    d.min_box_side,
        d.max_box_side, d.min_box_height, d.map_spacing, d.scan_spacing, d.scan_range,
        d.point_jitter, d.tilt_noise ? 1 : 0, d.gt_yaw_min, d.gt_yaw_max, d.min_scan_points,
        d.feasibility_resolution};
}

// gen_scene, scene.hpp:156-220.  Buffers are malloc'ed; free with ref_free.
int ref_gen_scene(const ref_scene_spec* s, uint64_t seed, double** map_xyz, uint64_t* n_map,
                  double** scan_xyz, uint64_t* n_scan, double* gt6) {
  return guard([&] {
    bnbloc::SceneSpec spec;
    spec.size_x = s->size_x;
    spec.size_y = s->size_y;
    spec.size_z = s->size_z;
    spec.num_boxes = s->num_boxes;
    spec.min_box_side = s->min_box_side;
    spec.max_box_side = s->max_box_side;
    spec.min_box_height = s->min_box_height;
    spec.map_spacing = s->map_spacing;
    spec.scan_spacing = s->scan_spacing;
    spec.scan_range = s->scan_range;
    spec.point_jitter = s->point_jitter;
    spec.tilt_noise = s->tilt_noise != 0;
    spec.gt_yaw_min = s->gt_yaw_min;
    spec.gt_yaw_max = s->gt_yaw_max;
    spec.min_scan_points = s->min_scan_points;
    spec.feasibility_resolution = s->feasibility_resolution;
    const bnbloc::Scene sc = bnbloc::gen_scene(spec, seed);
    *map_xyz = to_buffer(sc.map_cloud);
    *n_map = sc.map_cloud.size();
    *scan_xyz = to_buffer(sc.scan_cloud);
    *n_scan = sc.scan_cloud.size();
    const auto& g = sc.gt_pose;
    const double v[6] = {g.x, g.y, g.z, g.roll, g.pitch, g.yaw};
    std::memcpy(gt6, v, sizeof(v));
  });
}

// C4 harness helper (SURVEY §8d "C4 throughput"): the reference cannot render
// several scans of one map (layout, map, scan samples and gt share one Rng
// stream, scene.hpp:159-216).  This replays gen_scene's layout and surface
// sampling for `seed` with the reference's OWN detail:: functions
// (scene.hpp:50-97), then places n_scans sensors with poses drawn from
// Rng(pose_seed_base + j) under gen_scene's feasibility rules
// (scene.hpp:192-216; the overlap test is scene_overlap_fraction,
// scene.hpp:143-150, over one NeighborGrid built once).  Scans are
// concatenated (offsets[j] = first point of scan j, n_scans + 1 entries);
// gt is 6 * n_scans doubles.  Buffer malloc'ed; free with ref_free.
int ref_gen_scans(const ref_scene_spec* s, uint64_t seed, uint64_t pose_seed_base, int32_t n_scans,
                  double** scan_xyz, uint64_t* offsets, double* gt) {
  return guard([&] {
    namespace D = bnbloc::detail;
    bnbloc::Rng rng(seed * 0x9E3779B97F4A7C15ULL + 1);
    std::vector<D::Rect> surfaces;
    surfaces.push_back({{0, 0, 0}, {s->size_x, 0, 0}, {0, s->size_y, 0}});
    std::vector<D::Box> boxes;
    const double max_h = 0.9 * s->size_z;
    for (int i = 0; i < s->num_boxes; ++i) {
      const double w = std::min(rng.uniform(s->min_box_side, s->max_box_side), s->size_x - 2.5);
      const double d = std::min(rng.uniform(s->min_box_side, s->max_box_side), s->size_y - 2.5);
      const double h = rng.uniform(std::min(s->min_box_height, max_h), max_h);
      const double x0 = rng.uniform(1.0, std::max(1.0 + 1e-6, s->size_x - w - 1.0));
      const double y0 = rng.uniform(1.0, std::max(1.0 + 1e-6, s->size_y - d - 1.0));
      const D::Box b{x0, y0, x0 + w, y0 + d, h};
      boxes.push_back(b);
      for (const auto& f : D::box_faces(b)) surfaces.push_back(f);
    }
    bnbloc::PointCloud map_cloud, world_scan;
    for (const auto& r : surfaces) D::sample_rect(r, s->map_spacing, s->point_jitter, rng, map_cloud);
    for (const auto& r : surfaces) D::sample_rect(r, s->scan_spacing, s->point_jitter, rng, world_scan);
    const D::NeighborGrid grid(map_cloud, s->feasibility_resolution);
    std::vector<bnbloc::Point3> all;
    offsets[0] = 0;
    for (int32_t j = 0; j < n_scans; ++j) {
      bnbloc::Rng prng(pose_seed_base + static_cast<uint64_t>(j));
      bool ok = false;
      std::vector<bnbloc::Point3> scan;
      for (int attempt = 0; attempt < 64 && !ok; ++attempt) {
        bnbloc::Pose6 g;
        g.x = prng.uniform(0.12 * s->size_x, 0.88 * s->size_x);
        g.y = prng.uniform(0.12 * s->size_y, 0.88 * s->size_y);
        g.z = prng.uniform(1.2, 2.2);
        g.yaw = bnbloc::normalize_angle(prng.uniform(s->gt_yaw_min, s->gt_yaw_max));
        if (s->tilt_noise) {
          g.roll = prng.uniform(-0.01, 0.01);
          g.pitch = prng.uniform(-0.01, 0.01);
        }
        bool inside = false;
        for (const auto& b : boxes)
          if (b.contains_xy(g.x, g.y, 1.0)) inside = true;
        if (inside) continue;
        scan.clear();
        const bnbloc::Transform to_sensor = bnbloc::pose_to_transform(g).inverse();
        const bnbloc::Point3 sensor{g.x, g.y, g.z};
        for (const bnbloc::Point3& w : world_scan.points) {
          if ((w - sensor).norm() > s->scan_range) continue;
          scan.push_back(bnbloc::transform_point(to_sensor, w));
        }
        if (scan.size() < s->min_scan_points) continue;
        const bnbloc::Transform t = bnbloc::pose_to_transform(g);
        std::size_t hits = 0;
        for (const bnbloc::Point3& p : scan)
          if (grid.has_neighbor_within(bnbloc::transform_point(t, p), s->feasibility_resolution)) ++hits;
        if (static_cast<double>(hits) / static_cast<double>(scan.size()) >= 0.95) {
          const double v[6] = {g.x, g.y, g.z, g.roll, g.pitch, g.yaw};
          std::memcpy(gt + 6 * j, v, sizeof(v));
          ok = true;
        }
      }
      if (!ok)
        throw bnbloc::InfeasiblePoseError("gen_scans: no feasible pose for scan " + std::to_string(j));
      all.insert(all.end(), scan.begin(), scan.end());
      offsets[j + 1] = all.size();
    }
    bnbloc::PointCloud c;
    c.points = std::move(all);
    *scan_xyz = to_buffer(c);
  });
}

// MultiResVoxelMap::build, voxel_map.hpp:226-244.
int ref_map_build(const double* xyz, uint64_t n, double r, int32_t max_level, double ct,
                  uint64_t cap, void** out) {
  return guard([&] {
    auto* m = new bnbloc::MultiResVoxelMap(
        bnbloc::MultiResVoxelMap::build(to_cloud(xyz, n), r, max_level, ct, cap));
    *out = m;
  });
}

// MultiResVoxelMap::from_levels, voxel_map.hpp:247-261.
int ref_map_from_levels(const int32_t* const* lv, const uint64_t* counts, int32_t n_levels,
                        double r, const bbs_aabb* bbox, double ct, uint64_t cap, void** out) {
  return guard([&] {
    std::vector<std::vector<bnbloc::VoxelCoord>> per(static_cast<std::size_t>(n_levels));
    for (int32_t l = 0; l < n_levels; ++l)
      for (uint64_t i = 0; i < counts[l]; ++i)
        per[static_cast<std::size_t>(l)].push_back({lv[l][3 * i], lv[l][3 * i + 1], lv[l][3 * i + 2]});
    const bnbloc::Aabb b{{bbox->min.x, bbox->min.y, bbox->min.z},
                         {bbox->max.x, bbox->max.y, bbox->max.z}};
    *out = new bnbloc::MultiResVoxelMap(
        bnbloc::MultiResVoxelMap::from_levels(std::move(per), r, b, ct, cap));
  });
}

// save_map, map_io.hpp:44-65.
int ref_save_map(void* m, const char* path) {
  return guard([&] { bnbloc::save_map(*static_cast<bnbloc::MultiResVoxelMap*>(m), path); });
}

// load_map, map_io.hpp:67-115.
int ref_load_map(const char* path, double ct, uint64_t cap, void** out) {
  return guard([&] { *out = new bnbloc::MultiResVoxelMap(bnbloc::load_map(path, ct, cap)); });
}

int ref_map_max_level(void* m, int32_t* out) {
  *out = static_cast<bnbloc::MultiResVoxelMap*>(m)->max_level();
  return BBS_OK;
}

// is_map_file, map_io.hpp:119-126.
int ref_is_map_file(const char* path) { return bnbloc::is_map_file(path) ? 1 : 0; }

void ref_map_free(void* m) { delete static_cast<bnbloc::MultiResVoxelMap*>(m); }

int ref_map_bbox(void* m, bbs_aabb* out) {
  const auto& b = static_cast<bnbloc::MultiResVoxelMap*>(m)->bbox();
  *out = {{b.min.x, b.min.y, b.min.z}, {b.max.x, b.max.y, b.max.z}};
  return BBS_OK;
}

// LevelMap accessors, voxel_map.hpp:118-125.
int ref_level_info(void* m, int32_t level, uint64_t* occupied, uint64_t* buckets,
                   double* collision_rate) {
  const auto& lm = static_cast<bnbloc::MultiResVoxelMap*>(m)->level(level);
  *occupied = lm.occupied_count();
  *buckets = lm.bucket_count();
  *collision_rate = lm.collision_rate();
  return BBS_OK;
}

// LevelMap::occupied_voxels, voxel_map.hpp:158-165.
int ref_level_occupied(void* m, int32_t level, int32_t* xyz, uint64_t cap, uint64_t* count) {
  return guard([&] {
    const auto v = static_cast<bnbloc::MultiResVoxelMap*>(m)->level(level).occupied_voxels();
    *count = v.size();
    for (std::size_t i = 0; i < v.size() && i < cap; ++i) {
      xyz[3 * i] = v[i].x;
      xyz[3 * i + 1] = v[i].y;
      xyz[3 * i + 2] = v[i].z;
    }
  });
}

// LevelMap::contains, voxel_map.hpp:127-135.
int ref_level_contains(void* m, int32_t level, const int32_t* xyz, uint64_t n, uint8_t* out) {
  const auto& lm = static_cast<bnbloc::MultiResVoxelMap*>(m)->level(level);
  for (uint64_t i = 0; i < n; ++i) out[i] = lm.contains({xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]});
  return BBS_OK;
}

// LevelMap::score, voxel_map.hpp:142-154.
int ref_level_score(void* m, int32_t level, const double* rot9, const double* t3,
                    const double* scan, uint64_t k, int32_t* out) {
  return guard([&] {
    bnbloc::Transform t;
    for (int i = 0; i < 9; ++i) t.rotation[static_cast<std::size_t>(i)] = rot9[i];
    t.translation = {t3[0], t3[1], t3[2]};
    *out = static_cast<bnbloc::MultiResVoxelMap*>(m)->level(level).score(t, to_cloud(scan, k));
  });
}

// pose_to_transform, geometry.hpp:102-112.
void ref_pose_to_transform(const double* pose6, double* rot9, double* t3) {
  const bnbloc::Pose6 p{pose6[0], pose6[1], pose6[2], pose6[3], pose6[4], pose6[5]};
  const bnbloc::Transform t = bnbloc::pose_to_transform(p);
  for (int i = 0; i < 9; ++i) rot9[i] = t.rotation[static_cast<std::size_t>(i)];
  t3[0] = t.translation.x;
  t3[1] = t.translation.y;
  t3[2] = t.translation.z;
}

// AngularGrid ctor, angular_grid.hpp:67-99.
int ref_angular_grid(const bbs_search_config* c, double d_max, bbs_axis_grid* out) {
  return guard([&] {
    const bnbloc::AngularGrid g(to_cfg(c), d_max);
    for (int a = 0; a < 3; ++a)
      for (int l = 0; l <= c->max_level; ++l) {
        const auto& x = g.axis(a, l);
        out[a * (c->max_level + 1) + l] = {x.w_min, x.w_max, x.step, x.segments, x.periodic ? 1 : 0};
      }
  });
}

// AngularGrid::divisions, angular_grid.hpp:111-116.
int ref_angular_divisions(const bbs_search_config* c, double d_max, int32_t axis, int32_t level,
                          int32_t* out) {
  return guard([&] {
    const bnbloc::AngularGrid g(to_cfg(c), d_max);
    *out = g.divisions(axis, level);
  });
}

// node_pose, nodes.hpp:33-43.
int ref_node_pose(const bbs_search_config* c, double d_max, const bbs_node* n, double* pose6) {
  return guard([&] {
    const bnbloc::AngularGrid g(to_cfg(c), d_max);
    const bnbloc::Node nd{n->ix, n->iy, n->iz, n->iroll, n->ipitch, n->iyaw, n->level, n->score};
    const bnbloc::Pose6 p = bnbloc::node_pose(nd, g, c->min_resolution);
    const double v[6] = {p.x, p.y, p.z, p.roll, p.pitch, p.yaw};
    std::memcpy(pose6, v, sizeof(v));
  });
}

// initial_nodes, nodes.hpp:60-85.  Writes min(count, cap) nodes.
int ref_initial_nodes(const bbs_search_config* c, double d_max, const bbs_aabb* range,
                      bbs_node* out, uint64_t cap, uint64_t* count) {
  return guard([&] {
    const bnbloc::AngularGrid g(to_cfg(c), d_max);
    const bnbloc::Aabb b{{range->min.x, range->min.y, range->min.z},
                         {range->max.x, range->max.y, range->max.z}};
    const auto v = bnbloc::initial_nodes(b, g, c->min_resolution);
    *count = v.size();
    for (std::size_t i = 0; i < v.size() && i < cap; ++i) to_node(v[i], &out[i]);
  });
}

// branch, nodes.hpp:91-121.
int ref_branch(const bbs_search_config* c, double d_max, const bbs_node* parent, bbs_node* out,
               uint64_t cap, uint64_t* count) {
  return guard([&] {
    const bnbloc::AngularGrid g(to_cfg(c), d_max);
    const bnbloc::Node p{parent->ix,   parent->iy,   parent->iz,    parent->iroll,
                         parent->ipitch, parent->iyaw, parent->level, parent->score};
    const auto v = bnbloc::branch(p, g);
    *count = v.size();
    for (std::size_t i = 0; i < v.size() && i < cap; ++i) to_node(v[i], &out[i]);
  });
}

// batch_evaluate, search.hpp:23-34 (workers as given; 0 = all hardware threads).
int ref_batch_evaluate(void* m, const double* scan, uint64_t k, const bbs_search_config* c,
                       double d_max, bbs_node* nodes, uint64_t n, int32_t workers) {
  return guard([&] {
    const bnbloc::PointCloud sc = to_cloud(scan, k);
    const double dm = d_max > 0 ? d_max : bnbloc::max_range(sc);
    const bnbloc::AngularGrid g(to_cfg(c), dm);
    std::vector<bnbloc::Node> v(n);
    for (uint64_t i = 0; i < n; ++i)
      v[i] = {nodes[i].ix,    nodes[i].iy,   nodes[i].iz,    nodes[i].iroll,
              nodes[i].ipitch, nodes[i].iyaw, nodes[i].level, nodes[i].score};
    int w = workers > 0 ? workers : static_cast<int>(std::thread::hardware_concurrency());
    bnbloc::batch_evaluate(v, *static_cast<bnbloc::MultiResVoxelMap*>(m), sc, g, w);
    for (uint64_t i = 0; i < n; ++i) nodes[i].score = v[i].score;
  });
}

void fill_result(const bnbloc::SearchResult& r, bbs_search_result* out) {
  out->best_pose = {r.best_pose.x, r.best_pose.y, r.best_pose.z,
                    r.best_pose.roll, r.best_pose.pitch, r.best_pose.yaw};
  out->best_score = r.best_score;
  out->score_threshold = r.score_threshold;
  out->scan_points = r.scan_points;
  out->matched = r.matched ? 1 : 0;
  const auto& s = r.stats;
  out->stats = {s.nodes_generated,    s.nodes_pruned,       s.batches_flushed,
                s.create_voxel_maps_ms, s.set_source_ms,     s.initial_nodes_ms,
                s.find_best_score_ms, s.pop_remaining_queue_ms};
  out->trace_length = r.best_score_trace.size();
  for (std::size_t i = 0; i < r.best_score_trace.size() && i < out->trace_capacity; ++i)
    out->best_score_trace[i] = r.best_score_trace[i];
}

// search, search.hpp:72-186.
int ref_search(void* m, const double* scan, uint64_t k, const bbs_search_config* c,
               bbs_search_result* out) {
  return guard([&] {
    const bnbloc::SearchResult r =
        bnbloc::search(*static_cast<bnbloc::MultiResVoxelMap*>(m), to_cloud(scan, k), to_cfg(c));
    fill_result(r, out);
  });
}

// localize_scan, pipeline.hpp:45-51.
int ref_localize_scan(void* m, const double* raw, uint64_t n, const bbs_search_config* c,
                      uint64_t target, bbs_search_result* out) {
  return guard([&] {
    const bnbloc::SearchResult r = bnbloc::localize_scan(
        *static_cast<bnbloc::MultiResVoxelMap*>(m), to_cloud(raw, n), to_cfg(c), target);
    fill_result(r, out);
  });
}

// prepare_source, pipeline.hpp:25-41.  Output malloc'ed (ref_free).
int ref_prepare_source(const double* raw, uint64_t n, uint64_t target, double** out_xyz,
                       uint64_t* count, double* leaf, int32_t* converged, double* d_max) {
  return guard([&] {
    const bnbloc::SourcePrep p = bnbloc::prepare_source(to_cloud(raw, n), target);
    *out_xyz = to_buffer(p.scan);
    *count = p.scan.size();
    *leaf = p.leaf;
    *converged = p.leaf_converged ? 1 : 0;
    *d_max = p.d_max;
  });
}

// max_range, point_cloud.hpp:58-63.
int ref_max_range(const double* xyz, uint64_t n, double* out) {
  return guard([&] { *out = bnbloc::max_range(to_cloud(xyz, n)); });
}

// oracle_search, oracle.hpp:29-95.  Writes min(count, cap) argmax poses.
int ref_oracle_search(void* m, const double* scan, uint64_t k, const bbs_search_config* c,
                      int32_t* best_score, uint64_t* leaf_count, double* poses, uint64_t cap,
                      uint64_t* n_poses) {
  return guard([&] {
    const bnbloc::OracleResult r = bnbloc::oracle_search(
        *static_cast<bnbloc::MultiResVoxelMap*>(m), to_cloud(scan, k), to_cfg(c));
    *best_score = r.best_score;
    *leaf_count = r.leaf_count;
    *n_poses = r.argmax_poses.size();
    for (std::size_t i = 0; i < r.argmax_poses.size() && i < cap; ++i) {
      const auto& p = r.argmax_poses[i];
      const double v[6] = {p.x, p.y, p.z, p.roll, p.pitch, p.yaw};
      std::memcpy(poses + 6 * i, v, sizeof(v));
    }
  });
}

}  // extern "C"

// harness/scene.cpp — synthetic-input harness (NOT the product library).
//
// Restates the reference's box-world generator gen_scene (scene.hpp:156-220)
// and its splitmix64 Rng (rng.hpp:11-38) so the benchmark and the GPU tests
// can build the SAME doubles the reference consumes without shipping the
// reference (tests/test_host.py checks bit-identity against oracle/_ref).
// Also: a seeded Fisher-Yates prefix to cut a scan to exactly K points
// and the C4 helper that renders extra scans of one map.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "scene.h"

namespace {

struct Rng {  // rng.hpp:11-38
  uint64_t state;
  explicit Rng(uint64_t s) : state(s) {}
  uint64_t next_u64() {
    uint64_t z = (state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * next_double(); }
  int64_t uniform_int(int64_t lo, int64_t hi) {
    const uint64_t span = static_cast<uint64_t>(hi - lo) + 1;
    return lo + static_cast<int64_t>(next_u64() % span);
  }
};

struct P3 {
  double x, y, z;
};
P3 sub(P3 a, P3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
double norm(P3 p) { return std::sqrt(p.x * p.x + p.y * p.y + p.z * p.z); }

struct Rect {
  P3 origin, du, dv;
};
struct Box {
  double x0, y0, x1, y1, h;
  bool contains_xy(double x, double y, double pad) const {
    return x >= x0 - pad && x <= x1 + pad && y >= y0 - pad && y <= y1 + pad;
  }
};

// sample_rect, scene.hpp:57-73.
void sample_rect(const Rect& r, double spacing, double jitter, Rng& rng, std::vector<P3>& out) {
  const double lu = norm(r.du), lv = norm(r.dv);
  const int nu = std::max(1, static_cast<int>(std::ceil(lu / spacing)));
  const int nv = std::max(1, static_cast<int>(std::ceil(lv / spacing)));
  for (int u = 0; u <= nu; ++u)
    for (int v = 0; v <= nv; ++v) {
      const double fu = static_cast<double>(u) / nu;
      const double fv = static_cast<double>(v) / nv;
      // argument evaluation order is unspecified in C++, but the reference
      // build (g++) evaluates braced-init members left to right
      const double x = r.origin.x + fu * r.du.x + fv * r.dv.x + rng.uniform(-jitter, jitter);
      const double y = r.origin.y + fu * r.du.y + fv * r.dv.y + rng.uniform(-jitter, jitter);
      const double z = r.origin.z + fu * r.du.z + fv * r.dv.z + rng.uniform(-jitter, jitter);
      out.push_back({x, y, z});
    }
}

// box_faces, scene.hpp:82-91.
void box_faces(const Box& b, std::vector<Rect>& out) {
  const double w = b.x1 - b.x0, d = b.y1 - b.y0;
  out.push_back({{b.x0, b.y0, 0}, {w, 0, 0}, {0, 0, b.h}});
  out.push_back({{b.x0, b.y1, 0}, {w, 0, 0}, {0, 0, b.h}});
  out.push_back({{b.x0, b.y0, 0}, {0, d, 0}, {0, 0, b.h}});
  out.push_back({{b.x1, b.y0, 0}, {0, d, 0}, {0, 0, b.h}});
  out.push_back({{b.x0, b.y0, b.h}, {w, 0, 0}, {0, d, 0}});
}

struct Key {
  int64_t x, y, z;
  bool operator==(const Key& o) const { return x == o.x && y == o.y && z == o.z; }
};
struct KeyHash {
  size_t operator()(const Key& k) const {
    return static_cast<size_t>((k.x * 73856093LL) ^ (k.y * 19349663LL) ^ (k.z * 83492791LL));
  }
};

// NeighborGrid, scene.hpp:105-139 (membership answer is order-independent).
struct NeighborGrid {
  const std::vector<P3>& pts;
  double cell;
  std::unordered_map<Key, std::vector<size_t>, KeyHash> cells;
  NeighborGrid(const std::vector<P3>& p, double c) : pts(p), cell(c) {
    cells.reserve(p.size());
    for (size_t i = 0; i < p.size(); ++i) cells[cell_of(p[i])].push_back(i);
  }
  Key cell_of(const P3& p) const {
    return {static_cast<int64_t>(std::floor(p.x / cell)), static_cast<int64_t>(std::floor(p.y / cell)),
            static_cast<int64_t>(std::floor(p.z / cell))};
  }
  bool has_neighbor_within(const P3& p, double radius) const {
    const Key c = cell_of(p);
    const double r2 = radius * radius;
    for (int64_t dx = -1; dx <= 1; ++dx)
      for (int64_t dy = -1; dy <= 1; ++dy)
        for (int64_t dz = -1; dz <= 1; ++dz) {
          const auto it = cells.find({c.x + dx, c.y + dy, c.z + dz});
          if (it == cells.end()) continue;
          for (size_t i : it->second) {
            const P3 d = sub(pts[i], p);
            if (d.x * d.x + d.y * d.y + d.z * d.z <= r2) return true;
          }
        }
    return false;
  }
};

// pose_to_transform (geometry.hpp:102-112) and Transform::inverse (:92-100).
struct Tf {
  double r[9];
  P3 t;
  P3 apply(const P3& p) const {
    return {r[0] * p.x + r[1] * p.y + r[2] * p.z + t.x, r[3] * p.x + r[4] * p.y + r[5] * p.z + t.y,
            r[6] * p.x + r[7] * p.y + r[8] * p.z + t.z};
  }
};
Tf pose_tf(const double* pose) {
  const double ca = std::cos(pose[3]), sa = std::sin(pose[3]);
  const double cb = std::cos(pose[4]), sb = std::sin(pose[4]);
  const double cg = std::cos(pose[5]), sg = std::sin(pose[5]);
  Tf t;
  const double r[9] = {cg * cb, cg * sb * sa - sg * ca, cg * sb * ca + sg * sa,
                       sg * cb, sg * sb * sa + cg * ca, sg * sb * ca - cg * sa,
                       -sb,     cb * sa,                cb * ca};
  std::memcpy(t.r, r, sizeof(r));
  t.t = {pose[0], pose[1], pose[2]};
  return t;
}
Tf inverse(const Tf& a) {
  Tf t;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) t.r[3 * i + j] = a.r[3 * j + i];
  const P3 nt{-a.t.x, -a.t.y, -a.t.z};
  t.t = {t.r[0] * nt.x + t.r[1] * nt.y + t.r[2] * nt.z, t.r[3] * nt.x + t.r[4] * nt.y + t.r[5] * nt.z,
         t.r[6] * nt.x + t.r[7] * nt.y + t.r[8] * nt.z};
  return t;
}

double normalize_angle(double a) {  // geometry.hpp:36-43
  const double two_pi = 6.283185307179586476925286766559;
  double r = std::fmod(a, two_pi);
  if (r < 0.0) r += two_pi;
  if (r >= two_pi) r = 0.0;
  return r;
}

struct Layout {
  std::vector<Rect> surfaces;
  std::vector<Box> boxes;
};

// layout part of gen_scene, scene.hpp:161-180.
Layout make_layout(const hs_scene_spec& s, Rng& rng) {
  Layout L;
  L.surfaces.push_back({{0, 0, 0}, {s.size_x, 0, 0}, {0, s.size_y, 0}});
  const double max_h = 0.9 * s.size_z;
  for (int i = 0; i < s.num_boxes; ++i) {
    const double w = std::min(rng.uniform(s.min_box_side, s.max_box_side), s.size_x - 2.5);
    const double d = std::min(rng.uniform(s.min_box_side, s.max_box_side), s.size_y - 2.5);
    const double h = rng.uniform(std::min(s.min_box_height, max_h), max_h);
    const double x0 = rng.uniform(1.0, std::max(1.0 + 1e-6, s.size_x - w - 1.0));
    const double y0 = rng.uniform(1.0, std::max(1.0 + 1e-6, s.size_y - d - 1.0));
    const Box b{x0, y0, x0 + w, y0 + d, h};
    L.boxes.push_back(b);
    box_faces(b, L.surfaces);
  }
  return L;
}

// pose attempts, scene.hpp:192-216.  Returns false when infeasible.
bool place_scan(const hs_scene_spec& s, const Layout& L, const std::vector<P3>& map_cloud,
                const std::vector<P3>& world_scan, Rng& rng, const NeighborGrid* grid_in,
                std::vector<P3>& scan, double* gt6) {
  std::unique_ptr<NeighborGrid> own;
  for (int attempt = 0; attempt < 64; ++attempt) {
    double gt[6] = {0, 0, 0, 0, 0, 0};
    gt[0] = rng.uniform(0.12 * s.size_x, 0.88 * s.size_x);
    gt[1] = rng.uniform(0.12 * s.size_y, 0.88 * s.size_y);
    gt[2] = rng.uniform(1.2, 2.2);
    gt[5] = normalize_angle(rng.uniform(s.gt_yaw_min, s.gt_yaw_max));
    if (s.tilt_noise) {
      gt[3] = rng.uniform(-0.01, 0.01);
      gt[4] = rng.uniform(-0.01, 0.01);
    }
    bool inside = false;
    for (const auto& b : L.boxes)
      if (b.contains_xy(gt[0], gt[1], 1.0)) inside = true;
    if (inside) continue;
    scan.clear();
    const Tf to_sensor = inverse(pose_tf(gt));
    const P3 sensor{gt[0], gt[1], gt[2]};
    for (const P3& w : world_scan) {
      if (norm(sub(w, sensor)) > s.scan_range) continue;
      scan.push_back(to_sensor.apply(w));
    }
    if (scan.size() < s.min_scan_points) continue;
    // scene_overlap_fraction, scene.hpp:143-150
    if (!grid_in && !own) own.reset(new NeighborGrid(map_cloud, s.feasibility_resolution));
    const NeighborGrid& grid = grid_in ? *grid_in : *own;
    const Tf t = pose_tf(gt);
    size_t hits = 0;
    for (const P3& p : scan)
      if (grid.has_neighbor_within(t.apply(p), s.feasibility_resolution)) ++hits;
    const double frac = static_cast<double>(hits) / static_cast<double>(scan.size());
    if (frac >= 0.95) {
      std::memcpy(gt6, gt, sizeof(gt));
      return true;
    }
  }
  return false;
}

thread_local std::string g_scene_err;

double* to_buf(const std::vector<P3>& v) {
  double* out = static_cast<double*>(std::malloc(sizeof(double) * 3 * std::max<size_t>(v.size(), 1)));
  for (size_t i = 0; i < v.size(); ++i) {
    out[3 * i] = v[i].x;
    out[3 * i + 1] = v[i].y;
    out[3 * i + 2] = v[i].z;
  }
  return out;
}

}  // namespace

extern "C" {

void hs_scene_spec_default(hs_scene_spec* s) {  // SceneSpec defaults, scene.hpp:21-38
  s->size_x = 64.0;
  s->size_y = 64.0;
  s->size_z = 16.0;
  s->num_boxes = 10;
  s->min_box_side = 4.0;
  s->max_box_side = 14.0;
  s->min_box_height = 6.0;
  s->map_spacing = 0.25;
  s->scan_spacing = 0.40;
  s->scan_range = 28.0;
  s->point_jitter = 0.01;
  s->tilt_noise = 1;
  s->gt_yaw_min = 0.0;
  s->gt_yaw_max = 6.283185307179586476925286766559;
  s->min_scan_points = 400;
  s->feasibility_resolution = 1.0;
}

void hs_free(void* p) { std::free(p); }

// gen_scene, scene.hpp:156-220.
int hs_gen_scene(const hs_scene_spec* s, uint64_t seed, double** map_xyz, uint64_t* n_map,
                  double** scan_xyz, uint64_t* n_scan, double* gt6) {
  if (!s || !map_xyz || !n_map || !scan_xyz || !n_scan || !gt6) return 14;
  if (!(s->size_x > 0 && s->size_y > 0 && s->size_z > 0)) {
    g_scene_err = "gen_scene: dimensions must be positive";
    return 12;
  }
  Rng rng(seed * 0x9E3779B97F4A7C15ULL + 1);
  const Layout L = make_layout(*s, rng);
  std::vector<P3> map_cloud, world_scan, scan;
  for (const auto& r : L.surfaces) sample_rect(r, s->map_spacing, s->point_jitter, rng, map_cloud);
  for (const auto& r : L.surfaces) sample_rect(r, s->scan_spacing, s->point_jitter, rng, world_scan);
  if (!place_scan(*s, L, map_cloud, world_scan, rng, nullptr, scan, gt6)) {
    g_scene_err = "gen_scene: no feasible pose found in 64 attempts (seed " + std::to_string(seed) + ")";
    return 11;
  }
  *map_xyz = to_buf(map_cloud);
  *n_map = map_cloud.size();
  *scan_xyz = to_buf(scan);
  *n_scan = scan.size();
  return 0;
}

// C4 helper: replay seed's layout and map, then render
// n_scans scans with poses drawn from Rng(pose_seed_base + j) under the same
// feasibility rules.  Scans are concatenated; offsets[j] is scan j's first
// point (n_scans + 1 entries); gt is 6 * n_scans doubles.
int hs_gen_scans(const hs_scene_spec* s, uint64_t seed, uint64_t pose_seed_base, int32_t n_scans,
                  double** scan_xyz, uint64_t* offsets, double* gt) {
  if (!s || !scan_xyz || !offsets || !gt || n_scans < 0) return 14;
  Rng rng(seed * 0x9E3779B97F4A7C15ULL + 1);
  const Layout L = make_layout(*s, rng);
  std::vector<P3> map_cloud, world_scan, scan, all;
  for (const auto& r : L.surfaces) sample_rect(r, s->map_spacing, s->point_jitter, rng, map_cloud);
  for (const auto& r : L.surfaces) sample_rect(r, s->scan_spacing, s->point_jitter, rng, world_scan);
  const NeighborGrid grid(map_cloud, s->feasibility_resolution);
  offsets[0] = 0;
  for (int32_t j = 0; j < n_scans; ++j) {
    Rng prng(pose_seed_base + static_cast<uint64_t>(j));
    if (!place_scan(*s, L, map_cloud, world_scan, prng, &grid, scan, gt + 6 * j)) {
      g_scene_err = "gen_scans: no feasible pose for scan " + std::to_string(j);
      return 11;
    }
    all.insert(all.end(), scan.begin(), scan.end());
    offsets[j + 1] = all.size();
  }
  *scan_xyz = to_buf(all);
  return 0;
}

// Seeded Fisher-Yates prefix: the first k points of a uniform shuffle
// driven by Rng(seed) (SURVEY §8d "cut to exactly K points").
int hs_cut_scan(const double* xyz, uint64_t n, uint64_t k, uint64_t seed, double* out) {
  if (!xyz || !out || k > n) return 14;
  std::vector<uint64_t> idx(n);
  for (uint64_t i = 0; i < n; ++i) idx[i] = i;
  Rng rng(seed);
  for (uint64_t i = 0; i < k; ++i) {
    const uint64_t j = i + static_cast<uint64_t>(rng.uniform_int(0, static_cast<int64_t>(n - 1 - i)));
    std::swap(idx[i], idx[j]);
    out[3 * i] = xyz[3 * idx[i]];
    out[3 * i + 1] = xyz[3 * idx[i] + 1];
    out[3 * i + 2] = xyz[3 * idx[i] + 2];
  }
  return 0;
}

const char* hs_last_error(void) { return g_scene_err.c_str(); }

}  // extern "C"

// bbs_map_impl.h — host-side handles behind bbs_map_t / bbs_scan_t.
#pragma once

#include <cuda_runtime.h>

#include <mutex>
#include <vector>

#include "bbs_internal.h"

namespace bbs {
struct Workspace;
void free_workspace(Workspace* w);
}  // namespace bbs

struct bbs_map {
  int device = 0;
  cudaStream_t stream = nullptr;      // stream all work of this map runs on
  cudaStream_t own_stream = nullptr;  // created (and destroyed) by the map
  double r = 1.0;
  int max_level = 0;
  bbs_aabb bbox{};
  double collision_target = 0.001;
  uint64_t memory_cap = 0;
  int layout_pref = BBS_LAYOUT_AUTO;
  struct Level {
    bbs_level_info info{};
    unsigned long long* keys = nullptr;  // sorted unique packed keys (x-major)
    uint64_t n_keys = 0;
    uint32_t bits[3] = {0, 0, 0};
    void* structure = nullptr;           // bitmap words or hash slots
  };
  std::vector<Level> levels;
  bbs::MapView view{};
  double build_ms = 0.0;
  // persistent per-search workspaces (device buffers reused across calls)
  std::mutex ws_mu;
  std::vector<bbs::Workspace*> ws_pool;
  ~bbs_map();
};

struct bbs_scan {
  bbs_map* map = nullptr;
  uint64_t k = 0;
  double d_max = 0.0;          // max_range of the scan (host libm)
  double z_min = 0.0, z_max = 0.0, l1xy_max = 0.0;  // bounds for the dense histogram boxes
  double* soa = nullptr;       // device: x[k], y[k], z[k]
  ~bbs_scan();
};

namespace bbs {

// Device map construction (map_build.cu).
void build_map_from_points(bbs_map* m, const double* xyz, uint64_t n);
void build_map_from_levels(bbs_map* m, const int32_t* const* lv, const uint64_t* counts,
                           int n_levels);
void level_occupied(bbs_map* m, int level, int32_t* xyz, uint64_t cap, uint64_t* count);
void level_contains(bbs_map* m, int level, const int32_t* xyz, uint64_t n, uint8_t* out);
void level_score_transform(bbs_map* m, int level, const double* R, const double* t,
                           const double* scan, uint64_t k, int32_t* score);

// Scans (search.cu).
// sync = false: the caller uses the scan on the map's stream only.
bbs_scan* upload_scan(bbs_map* m, const double* xyz, uint64_t k, bool sync = true);

// oracle_search's level-0 leaf grid (oracle.hpp:39-54): translation index
// ranges [lo, lo + n) at level 0 and the level-0 rotation index counts.
struct LeafGridSpec {
  int64_t x_lo = 0, y_lo = 0, z_lo = 0;
  uint64_t nx = 0, ny = 0, nz = 0, nr = 0, np = 0, nw = 0;
  uint64_t total() const { return nx * ny * nz * (nr * np * nw); }
};
// batch_evaluate on device nodes (search.hpp:23-34), search.cu: the LUT
// built here (lo/hi widen the per-(level, axis) index range), or prebuilt.
void batch_evaluate_device(bbs_map* m, bbs_scan* scan, const bbs_search_config& cfg, double d_max,
                           bbs_node* d_nodes, uint64_t n, cudaStream_t s, const int32_t* lo,
                           const int32_t* hi);
void batch_evaluate_device(bbs_map* m, bbs_scan* scan, const GridView& gv, bbs_node* d_nodes, uint64_t n,
                           cudaStream_t s);
// leaf_grid.cu: score every leaf in blocks of `block`; best score (-1 if
// none) and every node attaining it, in enumeration order.
void leaf_grid_search(bbs_map* m, bbs_scan* scan, const bbs_search_config& cfg, double d_max,
                      const LeafGridSpec& g, uint64_t block, int32_t* best_score,
                      std::vector<bbs_node>* argmax);

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev);
  ~DeviceGuard();
};

}  // namespace bbs

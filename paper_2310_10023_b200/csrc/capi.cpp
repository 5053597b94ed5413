// capi.cpp — the extern "C" boundary (include/bbs.h).  Every entry point
// validates on the host in the reference's order, maps bbs::Error to a
// status code, and keeps the message for bbs_last_error().
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <limits>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "bbs_comm.h"
#include "bbs_map_impl.h"
#include "bbs_map_io.h"

namespace bbs {
void run_search(bbs_map* m, bbs_scan* scan, const bbs_search_config& cfg, const bbs_shard* shard,
                bbs_search_result* out, cudaStream_t stream = nullptr, bbs_search_dump* dump = nullptr);
void set_pool_retention(int device);
extern thread_local unsigned g_grid_share;  // kernels.h
extern thread_local bool g_blocking_sync;
struct SearchGroup;
SearchGroup* group_create(bbs_map* m, const bbs_search_config& cfg, uint32_t n_slots);
void group_destroy(SearchGroup* g);
extern thread_local SearchGroup* g_group;
}  // namespace bbs

namespace {

thread_local std::string g_err;

template <typename Fn>
int guard(Fn&& fn) {
  try {
    fn();
    return BBS_OK;
  } catch (const bbs::Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return BBS_ERR_GENERIC;
  } catch (const std::exception& e) {
    g_err = e.what();
    return BBS_ERR_GENERIC;
  }
}

#define REQUIRE(cond, what)                                              \
  do {                                                                   \
    if (!(cond)) throw bbs::Error(BBS_ERR_INVALID_ARGUMENT, what);       \
  } while (0)

void require_device(int device) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw bbs::Error(BBS_ERR_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
  }
  if (device < 0 || device >= n) throw bbs::Error(BBS_ERR_CUDA, "CUDA device ordinal out of range");
}

bbs_map* new_map(const bbs_map_options* opts, double r, uint64_t cap, double ct) {
  const int device = opts ? opts->device : 0;
  require_device(device);
  std::unique_ptr<bbs_map> m(new bbs_map());
  m->device = device;
  m->r = r;
  m->memory_cap = cap;
  m->collision_target = ct;
  m->layout_pref = opts ? opts->layout : BBS_LAYOUT_AUTO;
  if (m->layout_pref < BBS_LAYOUT_AUTO || m->layout_pref > BBS_LAYOUT_HASH)
    throw bbs::Error(BBS_ERR_CONFIG, "map: unknown layout");
  bbs::DeviceGuard g(device);
  bbs::set_pool_retention(device);
  BBS_CUDA(cudaStreamCreateWithFlags(&m->own_stream, cudaStreamNonBlocking));
  m->stream = m->own_stream;
  return m.release();
}

void check_level(const bbs_map* m, int32_t level) {
  if (level < 0 || level >= static_cast<int32_t>(m->levels.size()))
    throw bbs::Error(BBS_ERR_CONFIG, "level out of range");
}

}  // namespace

extern "C" {

const char* bbs_last_error(void) { return g_err.c_str(); }
int bbs_abi_version(void) { return BBS_ABI_VERSION; }

int bbs_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

void bbs_search_config_default(bbs_search_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->min_resolution = 1.0;
  c->max_level = 6;
  c->roll_pitch_half_range = 0.02;
  c->yaw_min = 0.0;
  c->yaw_max = 6.283185307179586476925286766559;
  c->score_threshold_fraction = 0.95;
  c->batch_size = 10000;
  c->strategy = BBS_STRATEGY_BFS;
  c->branch_mode = BBS_BRANCH_ROTO_TRANS;
  c->workers = 1;
}

int bbs_angular_grid(const bbs_search_config* cfg, double d_max, bbs_axis_grid* out,
                     uint64_t capacity) {
  return guard([&] {
    REQUIRE(cfg && out, "bbs_angular_grid: null argument");
    const bbs::HostGrid g = bbs::make_grid(*cfg, d_max);
    const uint64_t n = 3ull * static_cast<uint64_t>(cfg->max_level + 1);
    REQUIRE(capacity >= n, "bbs_angular_grid: capacity below 3*(max_level+1)");
    for (uint64_t i = 0; i < n; ++i) {
      const bbs::AxisGrid& a = g.axes[i];
      out[i] = {a.w_min, a.w_max, a.step, a.segments, a.periodic ? 1 : 0};
    }
  });
}

int bbs_angular_divisions(const bbs_search_config* cfg, double d_max, int32_t axis, int32_t level,
                          int32_t* out) {
  return guard([&] {
    REQUIRE(cfg && out, "bbs_angular_divisions: null argument");
    REQUIRE(axis >= 0 && axis < 3 && level >= 1 && level <= cfg->max_level,
            "bbs_angular_divisions: axis/level out of range");
    *out = bbs::make_grid(*cfg, d_max).divisions(axis, level);
  });
}

int bbs_max_range(const double* xyz, uint64_t n, double* out) {
  return guard([&] {
    REQUIRE(out && (xyz || n == 0), "bbs_max_range: null argument");
    *out = bbs::host_max_range(xyz, n);
  });
}

int bbs_bounding_box(const double* xyz, uint64_t n, bbs_aabb* out) {
  return guard([&] {
    REQUIRE(out && (xyz || n == 0), "bbs_bounding_box: null argument");
    *out = bbs::host_bounding_box(xyz, n);
  });
}

int bbs_prepare_source(const double* xyz, uint64_t n, uint64_t target, double* out_xyz,
                       uint64_t capacity, uint64_t* count, double* leaf, int32_t* converged,
                       double* d_max) {
  return guard([&] {
    REQUIRE(count && (xyz || n == 0), "bbs_prepare_source: null argument");
    const bbs::SourcePrep p = bbs::host_prepare_source(xyz, n, target);
    const uint64_t m = p.xyz.size() / 3;
    *count = m;
    if (out_xyz) std::memcpy(out_xyz, p.xyz.data(), 3 * std::min(m, capacity) * sizeof(double));
    if (leaf) *leaf = p.leaf;
    if (converged) *converged = p.converged ? 1 : 0;
    if (d_max) *d_max = p.d_max;
  });
}

int bbs_prepare_source_device(int32_t device, const double* xyz, uint64_t n, uint64_t target,
                              double* out_xyz, uint64_t capacity, uint64_t* count, double* leaf,
                              int32_t* converged, double* d_max) {
  return guard([&] {
    REQUIRE(count && (xyz || n == 0), "bbs_prepare_source_device: null argument");
    require_device(device);
    const bbs::SourcePrep p = bbs::device_prepare_source(device, xyz, n, target, false);
    const uint64_t m = p.xyz.size() / 3;
    *count = m;
    if (out_xyz) std::memcpy(out_xyz, p.xyz.data(), 3 * std::min(m, capacity) * sizeof(double));
    if (leaf) *leaf = p.leaf;
    if (converged) *converged = p.converged ? 1 : 0;
    if (d_max) *d_max = p.d_max;
  });
}

int bbs_initial_node_count(const bbs_search_config* cfg, double d_max, const bbs_aabb* range,
                           uint64_t* count) {
  return guard([&] {
    REQUIRE(cfg && range && count, "bbs_initial_node_count: null argument");
    const bbs::HostGrid g = bbs::make_grid(*cfg, d_max);
    const int L = cfg->max_level;
    const double cell = std::ldexp(cfg->min_resolution, L);
    auto cnt = [&](double lo, double hi) {
      const double f = std::floor(lo / cell), c = std::ceil(hi / cell);
      const int64_t a = (f >= -2147483648.0 && f < 2147483648.0) ? static_cast<int32_t>(f) : INT32_MIN;
      const int64_t b = (c >= -2147483648.0 && c < 2147483648.0) ? static_cast<int32_t>(c) : INT32_MIN;
      return b - a + 1;
    };
    const int64_t total = cnt(range->min.x, range->max.x) * cnt(range->min.y, range->max.y) *
                          cnt(range->min.z, range->max.z) * g.axis(0, L).index_count() *
                          g.axis(1, L).index_count() * g.axis(2, L).index_count();
    if (total <= 0) throw bbs::Error(BBS_ERR_EMPTY_SEARCH_SPACE, "initial node set is empty");
    *count = static_cast<uint64_t>(total);
  });
}

int bbs_map_build(const double* xyz, uint64_t n, double min_resolution, int32_t max_level,
                  double collision_target, uint64_t memory_cap_bytes, const bbs_map_options* opts,
                  bbs_map_t* out) {
  return guard([&] {
    REQUIRE(out && (xyz || n == 0), "bbs_map_build: null argument");
    *out = nullptr;
    // voxel_map.hpp:230-233, same order and messages
    if (n == 0) throw bbs::Error(BBS_ERR_EMPTY_CLOUD, "MultiResVoxelMap: empty map");
    if (max_level < 1) throw bbs::Error(BBS_ERR_CONFIG, "MultiResVoxelMap: max_level must be >= 1");
    if (!(min_resolution > 0.0))
      throw bbs::Error(BBS_ERR_CONFIG, "MultiResVoxelMap: min_resolution must be > 0");
    if (max_level >= bbs::kMaxLevels)
      throw bbs::Error(BBS_ERR_CONFIG, "MultiResVoxelMap: max_level above 15 is not supported");
    std::unique_ptr<bbs_map> m(new_map(opts, min_resolution, memory_cap_bytes, collision_target));
    m->max_level = max_level;
    m->bbox = bbs::host_bounding_box(xyz, n);
    bbs::build_map_from_points(m.get(), xyz, n);
    *out = m.release();
  });
}

int bbs_map_from_levels(const int32_t* const* level_voxels, const uint64_t* counts, int32_t n_levels,
                        double min_resolution, const bbs_aabb* bbox, double collision_target,
                        uint64_t memory_cap_bytes, const bbs_map_options* opts, bbs_map_t* out) {
  return guard([&] {
    REQUIRE(out && bbox && (n_levels <= 0 || (level_voxels && counts)),
            "bbs_map_from_levels: null argument");
    *out = nullptr;
    if (n_levels < 2) throw bbs::Error(BBS_ERR_FORMAT, "map must have at least 2 levels");
    if (n_levels > bbs::kMaxLevels)
      throw bbs::Error(BBS_ERR_CONFIG, "map: more than 16 levels are not supported");
    std::unique_ptr<bbs_map> m(new_map(opts, min_resolution, memory_cap_bytes, collision_target));
    m->max_level = n_levels - 1;
    m->bbox = *bbox;
    bbs::build_map_from_levels(m.get(), level_voxels, counts, n_levels);
    *out = m.release();
  });
}

int bbs_map_load(const char* path, double collision_target, uint64_t memory_cap_bytes,
                 const bbs_map_options* opts, bbs_map_t* out) {
  return guard([&] {
    REQUIRE(path && out, "bbs_map_load: null argument");
    *out = nullptr;
    bbs::MapFile mf;
    bbs::map_file_open(path, &mf);
    bbs::map_file_check_levels(&mf);
    if (mf.max_level + 1 > static_cast<uint32_t>(bbs::kMaxLevels))
      throw bbs::Error(BBS_ERR_CONFIG, "map: more than 16 levels are not supported");
    std::unique_ptr<bbs_map> m(new_map(opts, mf.r, memory_cap_bytes, collision_target));
    m->max_level = static_cast<int>(mf.max_level);
    m->bbox = mf.bbox;
    bbs::map_file_read_levels(&mf, m.get());
    *out = m.release();
  });
}

int bbs_map_save(bbs_map_t map, const char* path) {
  return guard([&] {
    REQUIRE(map && path, "bbs_map_save: null argument");
    bbs::map_file_save(map, path);
  });
}

int bbs_is_map_file(const char* path) { return path && bbs::map_file_is_map(path) ? 1 : 0; }

int bbs_map_free(bbs_map_t map) {
  return guard([&] { delete map; });
}

int bbs_map_min_resolution(bbs_map_t map, double* out) {
  return guard([&] {
    REQUIRE(map && out, "null argument");
    *out = map->r;
  });
}
int bbs_map_max_level(bbs_map_t map, int32_t* out) {
  return guard([&] {
    REQUIRE(map && out, "null argument");
    *out = map->max_level;
  });
}
int bbs_map_bbox(bbs_map_t map, bbs_aabb* out) {
  return guard([&] {
    REQUIRE(map && out, "null argument");
    *out = map->bbox;
  });
}
int bbs_map_build_ms(bbs_map_t map, double* out) {
  return guard([&] {
    REQUIRE(map && out, "null argument");
    *out = map->build_ms;
  });
}
int bbs_map_set_stream(bbs_map_t map, void* stream) {
  return guard([&] {
    REQUIRE(map, "null argument");
    bbs::DeviceGuard g(map->device);
    BBS_CUDA(cudaStreamSynchronize(map->stream));
    map->stream = stream ? static_cast<cudaStream_t>(stream) : map->own_stream;
  });
}
int bbs_map_level_info(bbs_map_t map, int32_t level, bbs_level_info* out) {
  return guard([&] {
    REQUIRE(map && out, "null argument");
    check_level(map, level);
    *out = map->levels[static_cast<size_t>(level)].info;
  });
}

int bbs_level_occupied(bbs_map_t map, int32_t level, int32_t* xyz, uint64_t capacity,
                       uint64_t* count) {
  return guard([&] {
    REQUIRE(map && count, "null argument");
    check_level(map, level);
    bbs::level_occupied(map, level, xyz, xyz ? capacity : 0, count);
  });
}

int bbs_level_contains(bbs_map_t map, int32_t level, const int32_t* xyz, uint64_t n, uint8_t* out) {
  return guard([&] {
    REQUIRE(map && (n == 0 || (xyz && out)), "null argument");
    check_level(map, level);
    bbs::level_contains(map, level, xyz, n, out);
  });
}

int bbs_level_score(bbs_map_t map, int32_t level, const double rotation[9],
                    const double translation[3], const double* scan_xyz, uint64_t k, int32_t* score) {
  return guard([&] {
    REQUIRE(map && rotation && translation && score && (scan_xyz || k == 0), "null argument");
    check_level(map, level);
    bbs::level_score_transform(map, level, rotation, translation, scan_xyz, k, score);
  });
}

int bbs_scan_upload(bbs_map_t map, const double* xyz, uint64_t k, bbs_scan_t* out) {
  return guard([&] {
    REQUIRE(map && out && (xyz || k == 0), "null argument");
    *out = bbs::upload_scan(map, xyz, k);
  });
}

int bbs_scan_free(bbs_scan_t scan) {
  return guard([&] { delete scan; });
}

int bbs_search_scan(bbs_map_t map, bbs_scan_t scan, const bbs_search_config* cfg,
                    bbs_search_result* result) {
  return guard([&] {
    REQUIRE(map && scan && cfg && result, "null argument");
    REQUIRE(scan->map == map, "scan was uploaded for a different map");
    bbs::run_search(map, scan, *cfg, nullptr, result);
  });
}

int bbs_search_scan_on(bbs_map_t map, bbs_scan_t scan, const bbs_search_config* cfg, void* stream,
                       bbs_search_result* result) {
  return guard([&] {
    REQUIRE(map && scan && cfg && result, "null argument");
    REQUIRE(scan->map == map, "scan was uploaded for a different map");
    bbs::run_search(map, scan, *cfg, nullptr, result, static_cast<cudaStream_t>(stream));
  });
}

int bbs_search_scan_dump(bbs_map_t map, bbs_scan_t scan, const bbs_search_config* cfg,
                         bbs_search_dump* dump, bbs_search_result* result) {
  return guard([&] {
    REQUIRE(map && scan && cfg && dump && result, "null argument");
    REQUIRE(scan->map == map, "scan was uploaded for a different map");
    bbs::run_search(map, scan, *cfg, nullptr, result, nullptr, dump);
  });
}

int bbs_search_scans(bbs_map_t map, const bbs_scan_t* scans, uint64_t n, const bbs_search_config* cfg,
                     int32_t concurrency, bbs_search_result* results) {
  return guard([&] {
    REQUIRE(map && cfg && (results || n == 0) && (scans || n == 0), "null argument");
    for (uint64_t i = 0; i < n; ++i)
      REQUIRE(scans[i] && scans[i]->map == map, "scan was uploaded for a different map");
    if (n == 0) return;
    const int T = static_cast<int>(std::min<uint64_t>(n, static_cast<uint64_t>(std::max(1, std::min(concurrency, 128)))));
    bbs::DeviceGuard g(map->device);
    // each search's persistent epoch grids take ~1/share of the GPU (C4, 32
    // scans, 16 in flight: 1081 scans/s at share 1, 1134-1146 at 2-4, 732
    // at 16); waits spin (blocking-sync events: -6% at 16 in flight)
    unsigned share = static_cast<unsigned>(std::max(1, std::min(4, T / 4)));
    if (const char* e = std::getenv("BBS_GRID_SHARE")) share = static_cast<unsigned>(std::max(1, std::atoi(e)));
    bool blocking = false;
    if (const char* e = std::getenv("BBS_BLOCKING_SYNC")) blocking = e[0] == '1';
    // co-batched flushes (BBS_COBATCH=1): the searches in flight share one
    // launch per epoch kernel.  Off by default: on C4 (32 scans, 16 in
    // flight) it reaches 886 scans/s against 1119 for per-search graphs on
    // their own streams -- the lockstep group runs ~4.5 of 16 slots busy on
    // average, and per-search PDL graphs on 16 streams already overlap the
    // latency-bound epoch kernels
    const bool cobatch = T > 1 && [] {
      const char* e = std::getenv("BBS_COBATCH");
      return e && e[0] == '1';
    }();
    // BBS_GROUPS=g: g independent groups (own streams) of T/g searches each
    int n_groups = 1;
    if (const char* e = std::getenv("BBS_GROUPS")) n_groups = std::max(1, std::min(T, std::atoi(e)));
    std::vector<std::unique_ptr<bbs::SearchGroup, void (*)(bbs::SearchGroup*)>> groups;
    for (int i = 0; cobatch && i < n_groups; ++i)
      groups.emplace_back(bbs::group_create(map, *cfg, static_cast<uint32_t>((T + n_groups - 1) / n_groups)),
                          bbs::group_destroy);
    std::vector<cudaStream_t> streams(static_cast<size_t>(T));
    for (auto& st : streams) BBS_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    std::atomic<uint64_t> next{0};
    std::mutex err_mu;
    std::exception_ptr first_err;
    std::vector<std::thread> workers;
    for (int t = 0; t < T; ++t)
      workers.emplace_back([&, t] {
        try {
          bbs::DeviceGuard wg(map->device);
          bbs::g_grid_share = share;
          bbs::g_blocking_sync = blocking;
          bbs::g_group = groups.empty() ? nullptr : groups[static_cast<size_t>(t) % groups.size()].get();
          for (uint64_t j = next++; j < n; j = next++)
            bbs::run_search(map, scans[j], *cfg, nullptr, &results[j], streams[static_cast<size_t>(t)]);
        } catch (...) {
          std::lock_guard<std::mutex> lk(err_mu);
          if (!first_err) first_err = std::current_exception();
          next = n;
        }
      });
    for (auto& w : workers) w.join();
    for (auto& st : streams) cudaStreamDestroy(st);
    if (first_err) std::rethrow_exception(first_err);
  });
}

int bbs_stream_create(int32_t device, void** out) {
  return guard([&] {
    REQUIRE(out, "null argument");
    require_device(device);
    bbs::DeviceGuard g(device);
    cudaStream_t s;
    BBS_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    *out = s;
  });
}

int bbs_stream_destroy(void* stream) {
  return guard([&] {
    if (stream) BBS_CUDA(cudaStreamDestroy(static_cast<cudaStream_t>(stream)));
  });
}

int bbs_comm_unique_id(uint8_t id[128]) {
  return guard([&] {
    REQUIRE(id, "null argument");
    bbs::comm_unique_id(id);
  });
}

int bbs_comm_init(int32_t device, int32_t rank, int32_t world_size, const uint8_t id[128],
                  bbs_comm_t* out) {
  return guard([&] {
    REQUIRE(id && out, "null argument");
    *out = reinterpret_cast<bbs_comm_t>(bbs::comm_create(device, rank, world_size, id));
  });
}

int bbs_comm_free(bbs_comm_t comm) {
  return guard([&] { bbs::comm_destroy(reinterpret_cast<bbs::Comm*>(comm)); });
}

int bbs_nccl_version(void) { return bbs::comm_nccl_version(); }

int bbs_search_sharded(bbs_map_t map, bbs_scan_t scan, const bbs_search_config* cfg,
                       const bbs_shard* shard, bbs_search_result* result) {
  return guard([&] {
    REQUIRE(map && scan && cfg && result && shard, "null argument");
    REQUIRE(scan->map == map, "scan was uploaded for a different map");
    REQUIRE(shard->mode == BBS_SHARD_ROOTS || shard->mode == BBS_SHARD_EXACT, "unknown shard mode");
    if (shard->comm) {
      const bbs::Comm* c = reinterpret_cast<const bbs::Comm*>(shard->comm);
      REQUIRE(c->rank == shard->rank && c->world == shard->world_size,
              "shard rank/world_size differ from the communicator's");
      REQUIRE(c->device == map->device, "communicator is on a different device than the map");
    }
    bbs::run_search(map, scan, *cfg, shard, result);
  });
}

int bbs_search(bbs_map_t map, const double* scan_xyz, uint64_t k, const bbs_search_config* cfg,
               bbs_search_result* result) {
  return guard([&] {
    REQUIRE(map && cfg && result && (scan_xyz || k == 0), "null argument");
    if (k == 0) throw bbs::Error(BBS_ERR_DEGENERATE_SCAN, "search: empty scan");
    const auto t0 = std::chrono::steady_clock::now();
    std::unique_ptr<bbs_scan> sc(bbs::upload_scan(map, scan_xyz, k, false));  // same stream as the search
    const auto t1 = std::chrono::steady_clock::now();
    bbs::run_search(map, sc.get(), *cfg, nullptr, result);
    result->h2d_bytes += 3 * k * sizeof(double);
    if (std::getenv("BBS_DEBUG_HOST")) {
      sc.reset();
      const auto t2 = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[host] bbs_search: upload %.1f us, search %.1f us, total (with scan free) %.1f us\n",
                   std::chrono::duration<double, std::micro>(t1 - t0).count(),
                   std::chrono::duration<double, std::micro>(t2 - t1).count(),
                   std::chrono::duration<double, std::micro>(t2 - t0).count());
    }
  });
}

int bbs_localize_scan(bbs_map_t map, const double* raw_xyz, uint64_t n, const bbs_search_config* cfg,
                      uint64_t downsample_target, bbs_search_result* result) {
  return bbs_localize_scan_ex(map, raw_xyz, n, cfg, downsample_target, BBS_PREPARE_EXACT, result);
}

int bbs_localize_scan_ex(bbs_map_t map, const double* raw_xyz, uint64_t n, const bbs_search_config* cfg,
                         uint64_t downsample_target, int32_t prepare, bbs_search_result* result) {
  return guard([&] {
    REQUIRE(map && cfg && result && (raw_xyz || n == 0), "null argument");
    REQUIRE(prepare == BBS_PREPARE_EXACT || prepare == BBS_PREPARE_DEVICE, "unknown prepare mode");
    // prepare_source, pipeline.hpp:25-41 (device voxel counts; centroids in
    // the reference's order, or on the device), then search (pipeline.hpp:48)
    const auto t0 = std::chrono::steady_clock::now();
    const bbs::SourcePrep prep =
        bbs::device_prepare_source(map->device, raw_xyz, n, downsample_target, prepare == BBS_PREPARE_EXACT);
    const double prep_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    const uint64_t k = prep.xyz.size() / 3;
    std::unique_ptr<bbs_scan> sc(bbs::upload_scan(map, prep.xyz.data(), k, false));
    bbs::run_search(map, sc.get(), *cfg, nullptr, result);
    result->stats.set_source_ms = prep_ms;
  });
}

int bbs_batch_evaluate(bbs_map_t map, const double* scan_xyz, uint64_t k,
                       const bbs_search_config* cfg, double d_max, bbs_node* nodes, uint64_t n) {
  return guard([&] {
    REQUIRE(map && cfg && (scan_xyz || k == 0) && (nodes || n == 0), "null argument");
    if (n == 0) return;  // parallel_chunks(0, ...) is a no-op (parallel.hpp:17)
    // index ranges the LUT must cover, per (level, axis)
    int32_t lo[bbs::kMaxLevels * 3], hi[bbs::kMaxLevels * 3];
    for (int i = 0; i < bbs::kMaxLevels * 3; ++i) {
      lo[i] = std::numeric_limits<int32_t>::max();
      hi[i] = std::numeric_limits<int32_t>::min();
    }
    for (uint64_t i = 0; i < n; ++i) {
      const bbs_node& nd = nodes[i];
      if (nd.level < 0 || nd.level > map->max_level || nd.level > cfg->max_level)
        throw bbs::Error(BBS_ERR_CONFIG, "batch_evaluate: node level outside the map / grid levels");
      const int32_t idx[3] = {nd.iroll, nd.ipitch, nd.iyaw};
      for (int a = 0; a < 3; ++a) {
        lo[nd.level * 3 + a] = std::min(lo[nd.level * 3 + a], idx[a]);
        hi[nd.level * 3 + a] = std::max(hi[nd.level * 3 + a], idx[a]);
      }
    }
    for (int i = 0; i < bbs::kMaxLevels * 3; ++i) {
      if (lo[i] > hi[i]) {
        lo[i] = 0;
        hi[i] = 0;
      }
      if (static_cast<int64_t>(hi[i]) - std::min<int64_t>(lo[i], 0) >= (1 << 20))
        throw bbs::Error(BBS_ERR_TOO_LARGE, "batch_evaluate: rotation index span above 2^20");
    }
    std::unique_ptr<bbs_scan> sc(bbs::upload_scan(map, scan_xyz, k));
    if (k == 0) {
      for (uint64_t i = 0; i < n; ++i) nodes[i].score = 0;  // empty scan scores 0
      return;
    }
    bbs::DeviceGuard g(map->device);
    cudaStream_t s = map->stream;
    bbs_node* d_nodes = nullptr;
    BBS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_nodes), n * sizeof(bbs_node), s));
    BBS_CUDA(cudaMemcpyAsync(d_nodes, nodes, n * sizeof(bbs_node), cudaMemcpyHostToDevice, s));
    bbs::batch_evaluate_device(map, sc.get(), *cfg, d_max, d_nodes, n, s, lo, hi);
    BBS_CUDA(cudaMemcpyAsync(nodes, d_nodes, n * sizeof(bbs_node), cudaMemcpyDeviceToHost, s));
    BBS_CUDA(cudaFreeAsync(d_nodes, s));
    BBS_CUDA(cudaStreamSynchronize(s));
  });
}

int bbs_batch_evaluate_device(bbs_map_t map, bbs_scan_t scan, const bbs_search_config* cfg,
                              double d_max, bbs_node* d_nodes, uint64_t n, void* stream) {
  return guard([&] {
    REQUIRE(map && scan && cfg && (d_nodes || n == 0), "null argument");
    if (n == 0) return;
    if (scan->k == 0) throw bbs::Error(BBS_ERR_DEGENERATE_SCAN, "batch_evaluate: empty scan");
    bbs::DeviceGuard g(map->device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : map->stream;
    bbs::batch_evaluate_device(map, scan, *cfg, d_max, d_nodes, n, s, nullptr, nullptr);
  });
}

namespace {
// oracle_search, oracle.hpp:29-95 (validation in the reference's order and
// messages, then the device leaf grid); every argmax leaf into `all`.
void oracle_search_impl(bbs_map_t map, const double* scan_xyz, uint64_t k, const bbs_search_config* cfg,
                        int32_t* best_score, std::vector<bbs_node>* all, uint64_t* leaf_count) {
  {
    // oracle.hpp:31-35, same order and messages
    if (k == 0) throw bbs::Error(BBS_ERR_DEGENERATE_SCAN, "oracle_search: empty scan");
    if (map->r != cfg->min_resolution)
      throw bbs::Error(BBS_ERR_CONFIG, "oracle_search: config r does not match the map");
    std::unique_ptr<bbs_scan> sc(bbs::upload_scan(map, scan_xyz, k, false));
    const double d_max = cfg->has_d_max ? cfg->d_max : sc->d_max;
    if (!(d_max > 0.0)) throw bbs::Error(BBS_ERR_DEGENERATE_SCAN, "oracle_search: zero scan range");
    const bbs::HostGrid grids = bbs::make_grid(*cfg, d_max);  // AngularGrid(cfg, d_max), :37
    const bbs_aabb range = cfg->has_translation_range ? cfg->translation_range : map->bbox;
    const double root_cell = std::ldexp(cfg->min_resolution, cfg->max_level);
    const int64_t scale = int64_t{1} << cfg->max_level;
    // trans_index_range (nodes.hpp:53-56): int32 floor / ceil of w / cell
    // with the x86 conversion (out of range / NaN -> INT32_MIN)
    auto to_i32 = [](double f) {
      return (f >= -2147483648.0 && f < 2147483648.0) ? static_cast<int32_t>(f) : INT32_MIN;
    };
    auto tir = [&](double lo, double hi, int64_t* a, int64_t* b) {
      *a = static_cast<int64_t>(to_i32(std::floor(lo / root_cell))) * scale;
      *b = (static_cast<int64_t>(to_i32(std::ceil(hi / root_cell))) + 1) * scale;
    };
    bbs::LeafGridSpec g;
    int64_t xh, yh, zh;
    tir(range.min.x, range.max.x, &g.x_lo, &xh);
    tir(range.min.y, range.max.y, &g.y_lo, &yh);
    tir(range.min.z, range.max.z, &g.z_lo, &zh);
    const int64_t nrot = static_cast<int64_t>(grids.axis(0, 0).index_count()) *
                         grids.axis(1, 0).index_count() * grids.axis(2, 0).index_count();
    // the reference's count, oracle.hpp:50-53: unsigned products that wrap
    // when an extent is negative
    const uint64_t total = static_cast<uint64_t>(xh - g.x_lo) * static_cast<uint64_t>(yh - g.y_lo) *
                           static_cast<uint64_t>(zh - g.z_lo) * static_cast<uint64_t>(nrot);
    if (total == 0) throw bbs::Error(BBS_ERR_EMPTY_SEARCH_SPACE, "oracle_search: empty leaf grid");
    if (total > 100000000ull)  // kOracleMaxLeaves, oracle.hpp:25
      throw bbs::Error(BBS_ERR_TOO_LARGE, "oracle_search: leaf grid of " + std::to_string(total) +
                                              " nodes exceeds the 1e8 guard");
    if (xh <= g.x_lo || yh <= g.y_lo || zh <= g.z_lo) {
      // an inverted range: the reference's loops (oracle.hpp:79-81) score no
      // leaf, so best_score stays -1 and the argmax list is empty
      *leaf_count = total;
      *best_score = -1;
      all->clear();
      return;
    }
    g.nx = static_cast<uint64_t>(xh - g.x_lo);
    g.ny = static_cast<uint64_t>(yh - g.y_lo);
    g.nz = static_cast<uint64_t>(zh - g.z_lo);
    g.nr = static_cast<uint64_t>(grids.axis(0, 0).index_count());
    g.np = static_cast<uint64_t>(grids.axis(1, 0).index_count());
    g.nw = static_cast<uint64_t>(grids.axis(2, 0).index_count());
    *leaf_count = total;
    const char* eb = std::getenv("BBS_LEAF_BLOCK");
    const uint64_t block = eb ? std::strtoull(eb, nullptr, 10) : (uint64_t{1} << 20);
    bbs::leaf_grid_search(map, sc.get(), *cfg, d_max, g, block, best_score, all);
  }
}
}  // namespace

int bbs_oracle_search(bbs_map_t map, const double* scan_xyz, uint64_t k, const bbs_search_config* cfg,
                      int32_t* best_score, bbs_node* argmax, uint64_t argmax_capacity,
                      uint64_t* argmax_count, uint64_t* leaf_count) {
  return guard([&] {
    REQUIRE(map && cfg && best_score && argmax_count && leaf_count && (scan_xyz || k == 0) &&
                (argmax || argmax_capacity == 0),
            "null argument");
    std::vector<bbs_node> all;
    oracle_search_impl(map, scan_xyz, k, cfg, best_score, &all, leaf_count);
    *argmax_count = all.size();
    if (argmax_capacity) std::memcpy(argmax, all.data(), std::min<uint64_t>(all.size(), argmax_capacity) * sizeof(bbs_node));
  });
}

int bbs_oracle_search_all(bbs_map_t map, const double* scan_xyz, uint64_t k, const bbs_search_config* cfg,
                          int32_t* best_score, bbs_node** argmax, uint64_t* argmax_count,
                          uint64_t* leaf_count) {
  return guard([&] {
    REQUIRE(map && cfg && best_score && argmax && argmax_count && leaf_count && (scan_xyz || k == 0),
            "null argument");
    *argmax = nullptr;
    std::vector<bbs_node> all;
    oracle_search_impl(map, scan_xyz, k, cfg, best_score, &all, leaf_count);
    auto* out = static_cast<bbs_node*>(std::malloc(std::max<size_t>(all.size(), 1) * sizeof(bbs_node)));
    if (!out) throw bbs::Error(BBS_ERR_GENERIC, "oracle_search: out of host memory");
    std::memcpy(out, all.data(), all.size() * sizeof(bbs_node));
    *argmax = out;
    *argmax_count = all.size();
  });
}

void bbs_free(void* p) { std::free(p); }

}  // extern "C"

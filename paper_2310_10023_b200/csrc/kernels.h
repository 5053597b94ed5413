// kernels.h — host launchers of the device kernels (score.cu, search.cu).
#pragma once

#include <atomic>
#include <cstdlib>
#include <mutex>

#include <cuda_runtime.h>

#include <utility>

#include "bbs_internal.h"

namespace bbs {

// Stream-ordered device allocations released on scope exit, so a BBS_CUDA
// throw between the allocation and the normal end leaks nothing.
struct StreamAllocs {
  cudaStream_t s;
  std::vector<void*> p;
  explicit StreamAllocs(cudaStream_t st) : s(st) {}
  StreamAllocs(const StreamAllocs&) = delete;
  StreamAllocs& operator=(const StreamAllocs&) = delete;
  template <typename T>
  T* get(size_t n) {
    void* x = nullptr;
    if (cudaMallocAsync(&x, n ? n * sizeof(T) : 1, s) != cudaSuccess)
      throw Error(BBS_ERR_CUDA, "CUDA: cudaMallocAsync failed");
    p.push_back(x);
    return static_cast<T*>(x);
  }
  ~StreamAllocs() {
    for (void* x : p) cudaFreeAsync(x, s);
  }
};

// Share of the GPU one search's persistent (grid-strided) epoch kernels
// claim: 1 for a lone search; bbs_search_scans sets it per worker thread so
// T concurrent searches size their grids to co-reside instead of each
// filling every SM (the epoch kernels are latency-bound at C4's sizes).
extern thread_local unsigned g_grid_share;
extern thread_local bool g_blocking_sync;  // host checks wait on a blocking-sync event
// cudaOccupancyMaxActiveBlocksPerMultiprocessor, memoised per (device,
// kernel, block, shared memory): the query costs ~10 us of host time and the
// search loop asks the same questions every flush
int ctas_per_sm(const void* kernel, int threads, int smem);
template <typename K>
int ctas_per_sm(K* kernel, int threads, int smem) {
  return ctas_per_sm(reinterpret_cast<const void*>(kernel), threads, smem);
}

inline unsigned share_cap(uint64_t cap) {
  const uint64_t c = cap / (g_grid_share ? g_grid_share : 1u);
  return static_cast<unsigned>(c < 16 ? 16 : c);
}


struct ScanView {
  const double* x;
  const double* y;
  const double* z;
  uint32_t k;
};

// Root translation box (initial_nodes, nodes.hpp:60-85) and its shard.
struct BoxParams {
  int32_t level;
  int32_t x0, y0, z0;         // trans_index_range mins
  uint32_t nx, ny, nz;        // counts per axis
  uint32_t nr, np, nw;        // rotation index counts at the root level
  uint32_t rank, world;       // roots with ref index % world == rank
  uint32_t n_tchunks;         // translation chunks per rotation (grid = nrot * n_tchunks)
  int32_t fpad;               // bound on |voxel offset| of a rotated scan point (d_max / cell + 2)
  double tmax;                // max |translation index| in the box (fast-path guard)
  // dense histogram box of the root level (dn_r = 0: hash), see RotCache
  int32_t dn_r, dn_zlo, dn_nz;
  int32_t threshold;          // survivor score (search.hpp:97-100): roots below it only count as pruned
  double dn_eps, dn_eps1;
};

// Padded shared-memory copy of the root level's z-column words for the
// root column kernel: staged (x, y) in [sx0, sx0 + pitch) x [sy0, sy0 + rows),
// zeros outside the level box, so entry offsets need no bounds checks.
struct RootStage {
  int32_t sx0, sy0;
  uint32_t pitch, rows;
  int32_t zoff;               // z0 - level box_min.z
  uint32_t dimz;              // level z extent (<= 24: words pre-shifted by 8 bits)
  int enabled;
};

constexpr int kBoxThreads = 256;
constexpr int kBoxTransPerThread = 4;
constexpr int kBoxTransPerCta = kBoxThreads * kBoxTransPerThread;

// Root ownership: root (ix, iy, iz, rot) belongs to rank
// ((ix - x0) * nrot + rot) % world, i.e. whole (x-slab, rotation) units.
// Per-rotation de-duplicated scan histograms of the root batch.
constexpr int kHistCap = 4096;   // distinct voxel offsets per rotation
constexpr int kAmbCap = 1024;    // ambiguous points per rotation
constexpr int kRotBatch = 2048;  // rotations per histogram pass
struct RootHist {
  int4* entries;      // [kRotBatch * kHistCap] (fx, fy, fz, count)
  uint32_t* amb;      // [kRotBatch * kAmbCap] scan point indices
  int32_t* n_ent;     // [kRotBatch]
  int32_t* n_amb;     // [kRotBatch]
  int32_t* overflow;  // [kRotBatch] 1: rotation falls back to the chunked kernel
  int32_t* total;     // [kRotBatch] sum of the emitted entries' counts
};

// Owned x-slabs of rotation `rot`: slab ix_rel is owned iff
// (ix_rel * nrot + rot) % world == rank  <=>  ix_rel == x0r (mod P).
__host__ __device__ inline bool owned_slabs(const BoxParams& bp, uint32_t nrot, uint32_t rot,
                                            uint32_t* P, uint32_t* x0r) {
  if (bp.world <= 1) {
    *P = 1;
    *x0r = 0;
    return true;
  }
  uint32_t g = bp.world, b = nrot % bp.world;
  while (b) {
    const uint32_t t = g % b;
    g = b;
    b = t;
  }
  *P = bp.world / g;
  for (uint32_t c = 0; c < *P; ++c)
    if ((static_cast<uint64_t>(c) * nrot + rot) % bp.world == bp.rank) {
      *x0r = c;
      return true;
    }
  return false;
}

// Chunked fallback (per-chunk de-duplication, any level layout) for the
// rotations [rot_begin, rot_end) whose only[rot - rot_begin] != 0 (all when
// only is null).
void launch_score_box_chunked(const MapView& map, const GridView& grid, const ScanView& scan,
                              const BoxParams& bp, uint32_t rot_begin, uint32_t rot_end,
                              const int32_t* only, int32_t* scores, unsigned long long* probes,
                              cudaStream_t s);

// Score every root owned by (rank, world) into scores[ref index], where
// ref index = position in initial_nodes() order (nodes.hpp:77-83).
// `hist` is scratch for kRotBatch rotations.  probes[0] += de-duplicated
// (root, voxel offset) probes; probes[2] += z-column words the column kernel
// read from its shared-memory window (the actual gathers, bench roofline).
// ev_col0/ev_col1 (optional) bracket the column-kernel launches.
void launch_score_roots(const MapView& map, const GridView& grid, const ScanView& scan,
                        const BoxParams& bp, const RootHist& hist, int32_t* scores,
                        unsigned long long* probes, cudaStream_t s, cudaEvent_t ev_col0 = nullptr,
                        cudaEvent_t ev_col1 = nullptr);

// Score n nodes that come in contiguous same-rotation runs of 8 (the output
// order of branch(), nodes.hpp:103-116).  n is read from *d_n when non-null
// (device-resident count; up to n_max nodes).  scores must be zeroed first
// when n_ptiles > 1.
void launch_score_runs8(const MapView& map, const GridView& grid, const ScanView& scan,
                        const bbs_node* nodes, const uint32_t* d_n, uint32_t n_max,
                        uint32_t n_ptiles, int32_t* scores, cudaStream_t s);

// Per-search cache of de-duplicated scan histograms per (level, rotation)
// for the flush batches (epoch_cache.cu).  info[slot] = {state, pool offset,
// entries, ambiguous points}; slot = base[level] + dense rotation id.
constexpr int32_t kCacheEmpty = -1, kCacheBuilding = -2, kCacheNone = -3, kCacheReady = 0;
constexpr int kCtlMaxEnt = 4 + kMaxLevels;      // [20] largest histogram (entries)
constexpr int kCtlDirect = kCtlMaxEnt + 1;      // [21] runs branch listed as direct this flush
constexpr int kCtlDirectItem = kCtlDirect + 1;  // [22] direct-run work items taken (probe kernel)
constexpr int kCacheCtl = kCtlDirectItem + 1;
constexpr int kCacheDenseCells = 48 * 1024;  // 96 KB of 16-bit counters
constexpr int kStageWindowMax = 96 * 1024;   // bytes of the probe's staged column window
struct RotCache {
  int enabled;
  uint32_t base[kMaxLevels];   // 0xFFFFFFFF: level not cached
  double tmax[kMaxLevels];     // translation-index bound of the level (+2)
  int4* info;                  // [slots]
  uint32_t* amb_off;           // [slots]
  int4* pool;                  // (fx, fy, fz, count) entries
  uint32_t* amb_pool;          // ambiguous scan point indices
  uint32_t* ctl;               // [kCacheCtl] pool used, amb used, builds this flush,
                               // fallback runs this flush, then per-level "raw" flags
  uint32_t* fb_runs;           // [max runs] runs the cube kernel scores (not cached)
  // direct runs (single searches; null in co-batched launches): runs that can
  // have no histogram this flush (uncached or given-up level, failed
  // rotation) are listed by the branch kernel and scored by the probe
  // kernel's CTAs after their histogram items, instead of by the cube kernel
  // after the probe
  uint32_t* direct_runs;       // [max runs]
  uint8_t* direct_flag;        // [max runs] 1: the run is in direct_runs
  const uint32_t* direct_gate; // non-null: direct runs only while *direct_gate (the search's spec_mode)
  // dense-histogram box per level (dn_r = 0: hash build): offsets in
  // [-r, r]^2 x [zlo, zlo + nz), two 16-bit counts per shared word
  int32_t dn_r[kMaxLevels], dn_zlo[kMaxLevels], dn_nz[kMaxLevels];
  // fast-path eps of the dense box: (W + tmax) * 2^-48 with W >= |w| + 1 for
  // every in-box offset, so it bounds fast_floor's per-point eps (and 1 - eps)
  double dn_eps[kMaxLevels], dn_eps1[kMaxLevels];
  // staged level (-1: none): its histograms are stored as groups of 4
  // entries (column offset in the padded window, z bytes, count bytes) and
  // the probe reads the level's z-column words from a zero-padded shared
  // window [sx0, sx0 + pitch) x [sy0, sy0 + rows) (relative to box_min),
  // pre-shifted up by 8 bits
  int pre_level;                // level prebuilt for all rotations (-1: none)
  int stg_level;
  int32_t stg_sx0, stg_sy0;
  uint32_t stg_pitch, stg_rows;
  const uint32_t* stg_win;     // the window, built once per search (bytes rounded to 16)
  int4* builds;                // [max runs] (slot, level, iroll, ipitch)
  int32_t* builds_w;           // [max runs] iyaw
  uint64_t pool_cap, amb_cap;
};

// Same contract for the epoch flush, using the 2x2x2 translation-cube
// structure of branch()'s output (z-column bitmap: 4 loads per point).
// With `cache`, runs whose (level, rotation) histogram is READY are skipped.
void launch_score_cube8(const MapView& map, const GridView& grid, const ScanView& scan,
                        const bbs_node* nodes, const uint32_t* d_n, uint32_t n_max,
                        uint32_t n_ptiles, int32_t* scores, const RotCache* cache,
                        cudaStream_t s);

// Flush scoring: cache claim/build/probe + the cube kernel for the rest.
// scores must be zeroed first.
void launch_epoch_score(const MapView& map, const GridView& grid, const ScanView& scan,
                        const bbs_node* pending, const uint32_t* d_n, uint32_t n_max,
                        uint32_t n_ptiles, int32_t* scores, const RotCache& cache, cudaStream_t s,
                        bool builds = true);

// Co-batched flushes (bbs_search_scans): one launch per score kernel for a
// group of searches, blockIdx.y = slot.  A slot's score-kernel arguments sit
// at the front of the caller's per-slot record (`stride` bytes apart).
struct ScoreSlot {
  GridView G;
  ScanView scan;
  RotCache cache;            // cache.enabled == 0: the cube kernel scores every run
  const bbs_node* nodes;     // pending children
  const uint32_t* d_n;       // their count (device)
  int32_t* scores;
  uint32_t n_ptiles;         // point tiles per run without the cache
  uint32_t chunks;           // probe: histogram chunks per run at most
};
void launch_epoch_score_group(const MapView& map, const ScoreSlot* slots, size_t stride, uint32_t n_slots,
                              cudaStream_t s);
void launch_score_cube8_group(const MapView& map, const ScoreSlot* slots, size_t stride, uint32_t n_slots,
                              cudaStream_t s);
__device__ __forceinline__ const ScoreSlot& score_slot(const ScoreSlot* ga, size_t stride) {
  return *reinterpret_cast<const ScoreSlot*>(reinterpret_cast<const char*>(ga) + blockIdx.y * stride);
}
// CTAs per slot when `full` CTAs would fill the GPU for one search
inline unsigned per_slot(unsigned full, uint32_t n_slots, unsigned at_least = 8) {
  // a slot's kernels may take 1/min(slots, div) of the GPU: slots are
  // unevenly loaded, so 1/slots starves the heavy ones (C4 16 in flight:
  // 514 scans/s at div = slots, 789 at 1, 883 at 2)
  static const unsigned div = [] {
    const char* v = std::getenv("BBS_GROUP_DIV");
    return v ? static_cast<unsigned>(std::atoi(v)) : 2u;
  }();
  if (div) n_slots = n_slots < div ? n_slots : div;
  const unsigned g = full / (n_slots ? n_slots : 1u);
  return g < at_least ? at_least : g;
}

// Build the histograms of every rotation of `level` (n_rot slots from
// cache.base[level]) in one launch; cache.builds must hold n_rot entries.
void launch_cache_prebuild(const MapView& map, const GridView& grid, const ScanView& scan, const RotCache& pre,
                           uint32_t n_rot, cudaStream_t s);
// marks the level's n_rot slots BUILDING and lists them in pre.builds /
// pre.builds_w (a list of its own: the flush builds use cache.builds and
// ctl[2] while the prebuild runs on its side stream)
void launch_cache_prebuild_list(const GridView& grid, const RotCache& pre, int level, uint32_t n_rot,
                                cudaStream_t s);

// Score arbitrary nodes in place (node.score), grouping equal rotations on
// the device.  Host-synchronous.
// The rotation LUT of (cfg, d_max) uploaded into `al` (search.cu).
GridView upload_grid(const bbs_search_config& cfg, double d_max, const int32_t* lo, const int32_t* hi,
                     cudaStream_t s, StreamAllocs& al);

void score_nodes_general(const MapView& map, const GridView& grid, const ScanView& scan,
                         bbs_node* d_nodes, uint64_t n, cudaStream_t s);

// Choose the point-tile split for `runs` runs so the grid fills the chip.
uint32_t choose_ptiles(uint64_t runs, uint32_t k);

// Builds the staged probe window (zero-padded, words << 8) in global memory.
void build_stage_window(const MapView& map, const RotCache& cache, uint32_t* win, cudaStream_t s);

// Launch with programmatic stream serialization (PDL) so the kernel's launch
// overlaps the tail of the previous kernel in the stream; the kernel must
// call pdl_wait() before reading what its predecessor wrote.  BBS_PDL=0
// turns it off (plain launches).
bool pdl_enabled();

// Runs f once per (call site, CUDA device): kernel attributes such as the
// dynamic shared-memory limit are per device, and several host threads may
// launch concurrently.
template <typename F>
void once_per_device(std::atomic<uint64_t>& done, std::mutex& mu, F&& f) {
  int d = 0;
  BBS_CUDA(cudaGetDevice(&d));
  const uint64_t bit = 1ull << (d & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  std::lock_guard<std::mutex> lk(mu);
  if (done.load(std::memory_order_relaxed) & bit) return;
  f();
  done.fetch_or(bit, std::memory_order_release);
}
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  BBS_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

}  // namespace bbs

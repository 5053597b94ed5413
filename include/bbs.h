/*
 * bbs.h — C-ABI of the B200-native batched branch-and-bound scan matcher.
 *
 * This is the drop-in boundary for the reference's localizer path
 * (`bnbloc`, header-only C++20 under /root/reference/proj/include/bnbloc).
 * The reference has no FFI of its own (proj/CMakeLists.txt:14-16 declares an
 * INTERFACE library), so every entry point below names the reference
 * function or type it replaces (file:line, relative to
 * /root/reference/proj/include/bnbloc/).  The C++ facade in
 * include/bnbloc_b200.hpp re-exposes these with the reference's own names,
 * signatures and exception types.
 *
 * Conventions
 *   - Every function returns a bbs_status; 0 is success.  On failure
 *     bbs_last_error() returns the message the reference's exception would
 *     carry (thread-local, valid until the next call on the same thread).
 *   - Host pointers are caller-owned and only read/written during the call.
 *   - Points are packed xyz triples of double (the layout of
 *     std::vector<bnbloc::Point3>, geometry.hpp:12-30).
 *   - Nodes are bbs_node, byte-compatible with bnbloc::Node (nodes.hpp:18-29).
 *   - A bbs_map_t is immutable after build and may be shared by host threads
 *     (voxel_map.hpp:54-56); a search owns its own per-call workspace.
 *   - There is no CPU fallback: every compute entry point runs on the GPU the
 *     map was built on and fails with BBS_ERR_CUDA when there is none.
 */
#ifndef BBS_B200_H
#define BBS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BBS_ABI_VERSION 5

/* Status codes, 1:1 with the exception classes of errors.hpp:11-98. */
typedef enum bbs_status {
  BBS_OK = 0,
  BBS_ERR_GENERIC = 1,              /* bnbloc::Error                  errors.hpp:11 */
  BBS_ERR_FILE_NOT_FOUND = 2,       /* bnbloc::FileNotFoundError      errors.hpp:17 */
  BBS_ERR_PARSE = 3,                /* bnbloc::ParseError             errors.hpp:28 */
  BBS_ERR_EMPTY_CLOUD = 4,          /* bnbloc::EmptyCloudError        errors.hpp:46 */
  BBS_ERR_CAPACITY_EXCEEDED = 5,    /* bnbloc::CapacityExceededError  errors.hpp:53 */
  BBS_ERR_IO = 6,                   /* bnbloc::IoError                errors.hpp:59 */
  BBS_ERR_FORMAT = 7,               /* bnbloc::FormatError            errors.hpp:65 */
  BBS_ERR_DEGENERATE_SCAN = 8,      /* bnbloc::DegenerateScanError    errors.hpp:71 */
  BBS_ERR_EMPTY_SEARCH_SPACE = 9,   /* bnbloc::EmptySearchSpaceError  errors.hpp:77 */
  BBS_ERR_TOO_LARGE = 10,           /* bnbloc::TooLargeError          errors.hpp:83 */
  BBS_ERR_INFEASIBLE_POSE = 11,     /* bnbloc::InfeasiblePoseError    errors.hpp:89 */
  BBS_ERR_CONFIG = 12,              /* bnbloc::ConfigError            errors.hpp:95 */
  BBS_ERR_CUDA = 13,                /* no counterpart: device/driver failure */
  BBS_ERR_INVALID_ARGUMENT = 14     /* no counterpart: null handle/pointer */
} bbs_status;

/* Strategy / BranchMode, same enumerator order as search_config.hpp:14-15. */
enum { BBS_STRATEGY_DFS = 0, BBS_STRATEGY_BFS = 1 };
enum { BBS_BRANCH_TRANS_ONLY = 0, BBS_BRANCH_ROTO_TRANS = 1 };

/* Device layout of one level's occupancy set (no reference counterpart:
 * the reference always uses LevelMap's linear-probing table,
 * voxel_map.hpp:57-180).  Membership, and so every score, is identical for
 * all layouts. */
enum {
  BBS_LAYOUT_AUTO = 0,    /* per level: bitmap when it is not larger than the hash table */
  BBS_LAYOUT_BITMAP = 1,  /* dense z-column bit grid over the level's voxel box (32 z per word) */
  BBS_LAYOUT_HASH = 2     /* open addressing, packed 64-bit keys, 4-key (32 B) buckets */
};

typedef struct bbs_point3 { double x, y, z; } bbs_point3;            /* Point3  geometry.hpp:12 */
typedef struct bbs_pose6 {                                            /* Pose6   geometry.hpp:46 */
  double x, y, z, roll, pitch, yaw;
} bbs_pose6;
typedef struct bbs_aabb { bbs_point3 min, max; } bbs_aabb;            /* Aabb    point_cloud.hpp:24 */
typedef struct bbs_node {                                             /* Node    nodes.hpp:18-29 */
  int32_t ix, iy, iz, iroll, ipitch, iyaw, level, score;
} bbs_node;

/* SearchConfig, search_config.hpp:24-52.  std::optional members become a
 * has_* flag plus the value. */
typedef struct bbs_search_config {
  double min_resolution;            /* r, default 1.0 */
  int32_t max_level;                /* default 6 */
  int32_t has_translation_range;    /* 0: use the map bounding box */
  bbs_aabb translation_range;
  double roll_pitch_half_range;     /* default 0.02 */
  double yaw_min;                   /* default 0 */
  double yaw_max;                   /* default 2*pi */
  double score_threshold_fraction;  /* default 0.95 */
  uint64_t batch_size;              /* b, default 10000 */
  int32_t strategy;                 /* BBS_STRATEGY_*, default BFS */
  int32_t branch_mode;              /* BBS_BRANCH_*, default RotoTrans */
  int32_t workers;                  /* accepted and ignored: the GPU grid replaces parallel_chunks */
  int32_t has_d_max;
  double d_max;
  int32_t collect_trace;
} bbs_search_config;

/* Stats, search_config.hpp:55-69. */
typedef struct bbs_stats {
  uint64_t nodes_generated;
  uint64_t nodes_pruned;
  uint64_t batches_flushed;
  double create_voxel_maps_ms;
  double set_source_ms;
  double initial_nodes_ms;
  double find_best_score_ms;
  double pop_remaining_queue_ms;
} bbs_stats;

/* SearchResult, search_config.hpp:71-80.  The incumbent trace is written
 * into a caller-provided buffer (trace_capacity entries); trace_length is
 * the full length even when it exceeds the capacity. */
typedef struct bbs_search_result {
  bbs_pose6 best_pose;
  int32_t best_score;
  int32_t score_threshold;
  uint64_t scan_points;
  int32_t matched;
  bbs_stats stats;
  int32_t* best_score_trace;
  uint64_t trace_capacity;
  uint64_t trace_length;
  /* Extensions (no reference counterpart). */
  bbs_node best_node;     /* the leaf behind best_pose */
  uint64_t epochs;        /* flushes after the root batch */
  uint64_t lookups;       /* (node, scan point) pairs scored = nodes_generated * K */
  double device_ms;       /* device time of the search, CUDA events */
  double root_score_ms;   /* device time of the root-batch score kernel */
  double epoch_score_ms;  /* device time of the per-flush score kernels (sum) */
  uint64_t root_nodes;    /* roots scored by this rank */
  uint64_t queue_peak;    /* largest frontier (queue) length seen */
  uint64_t root_probes;   /* membership probes the root kernel issued after de-duplication */
  uint64_t h2d_bytes;     /* host->device bytes copied by this call */
  uint64_t d2h_bytes;     /* device->host bytes copied by this call */
  uint64_t kernel_launches; /* launches of this library's own kernels (CUB launches excluded) */
  uint64_t evals_per_level[16]; /* nodes scored per tree level (roots included) */
  uint64_t root_words;    /* z-column words the root column kernel read (its actual gathers) */
  double root_col_ms;     /* device time of the root column kernel launches, CUDA events */
  uint64_t group_checks;  /* bbs_search_scans: host checks whose epochs ran in a co-batched group
                             launch (0: the search launched its own) */
} bbs_search_result;

/* AxisGrid, angular_grid.hpp:45-58. */
typedef struct bbs_axis_grid {
  double w_min, w_max, step;
  int32_t segments;
  int32_t periodic;
} bbs_axis_grid;

typedef struct bbs_map_options {
  int32_t device;   /* CUDA ordinal, default 0 */
  int32_t layout;   /* BBS_LAYOUT_*, default AUTO */
} bbs_map_options;

typedef struct bbs_level_info {
  int32_t level;
  int32_t layout;                /* BBS_LAYOUT_BITMAP or BBS_LAYOUT_HASH */
  double resolution;             /* LevelMap::resolution  voxel_map.hpp:119 */
  uint64_t occupied_count;       /* LevelMap::occupied_count voxel_map.hpp:120 */
  uint64_t bucket_count;         /* hash slots, or bitmap bits */
  double collision_rate;         /* of OUR table (0 for bitmaps) */
  double load_factor;            /* occupied / bucket_count */
  uint64_t bytes;                /* device bytes of the structure */
  int32_t box_min[3];            /* voxel box of the level (inclusive) */
  int32_t box_max[3];
} bbs_level_info;

typedef struct bbs_map* bbs_map_t;
typedef struct bbs_scan* bbs_scan_t;

/* ---- errors / device ------------------------------------------------- */
const char* bbs_last_error(void);
int bbs_abi_version(void);
/* Number of visible CUDA devices (0 without a GPU; never fails). */
int bbs_device_count(void);

/* ---- host-side helpers (no device work) ------------------------------ */
/* SearchConfig defaults, search_config.hpp:24-52. */
void bbs_search_config_default(bbs_search_config* cfg);
/* AngularGrid(cfg, d_max), angular_grid.hpp:67-99: writes 3*(max_level+1)
 * grids, axis-major (out[axis*(max_level+1)+level]). */
int bbs_angular_grid(const bbs_search_config* cfg, double d_max, bbs_axis_grid* out,
                     uint64_t capacity);
/* AngularGrid::divisions, angular_grid.hpp:111-116. */
int bbs_angular_divisions(const bbs_search_config* cfg, double d_max, int32_t axis,
                          int32_t level, int32_t* out);
/* max_range, point_cloud.hpp:58-63. */
int bbs_max_range(const double* xyz, uint64_t n, double* out);
/* bounding_box, point_cloud.hpp:42-54. */
int bbs_bounding_box(const double* xyz, uint64_t n, bbs_aabb* out);
/* prepare_source, pipeline.hpp:25-41 (voxel_grid_downsample + auto_leaf,
 * point_cloud.hpp:78-182), host C++.  Writes at most `capacity` points;
 * *count is the full size.  leaf/converged/d_max may be NULL. */
int bbs_prepare_source(const double* xyz, uint64_t n, uint64_t target_points, double* out_xyz,
                       uint64_t capacity, uint64_t* count, double* leaf, int32_t* converged,
                       double* d_max);
/* prepare_source on the device (csrc/source_prep.cu): auto_leaf's bisection
 * with device voxel counts and voxel_grid_downsample's sort + centroids on
 * `device`.  Leaf, convergence flag, voxel set and output order equal the
 * reference's; a voxel's centroid sums its points in input order (the
 * reference in std::sort's unstable order), so centroids of voxels with >= 3
 * points may differ from bbs_prepare_source in the last bits.  The fast
 * path of bbs_localize_scan_ex(..., BBS_PREPARE_DEVICE). */
int bbs_prepare_source_device(int32_t device, const double* xyz, uint64_t n, uint64_t target_points,
                              double* out_xyz, uint64_t capacity, uint64_t* count, double* leaf,
                              int32_t* converged, double* d_max);
/* Root node count of initial_nodes, nodes.hpp:60-85. */
int bbs_initial_node_count(const bbs_search_config* cfg, double d_max, const bbs_aabb* range,
                           uint64_t* count);

/* ---- map (L3) -------------------------------------------------------- */
/* MultiResVoxelMap::build, voxel_map.hpp:226-244 (and build_level /
 * inflated_voxels :186-216, LevelMap::from_voxels :72-116), on the device.
 * collision_target is validated and recorded; the device tables do not use
 * the reference's sizing loop (membership is layout-independent).
 * memory_cap_bytes caps each level's device structure
 * (CapacityExceededError, voxel_map.hpp:91-95).  opts may be NULL. */
int bbs_map_build(const double* xyz, uint64_t n, double min_resolution, int32_t max_level,
                  double collision_target, uint64_t memory_cap_bytes,
                  const bbs_map_options* opts, bbs_map_t* out);
/* MultiResVoxelMap::from_levels, voxel_map.hpp:247-261 (map_io load path). */
int bbs_map_from_levels(const int32_t* const* level_voxels, const uint64_t* counts,
                        int32_t n_levels, double min_resolution, const bbs_aabb* bbox,
                        double collision_target, uint64_t memory_cap_bytes,
                        const bbs_map_options* opts, bbs_map_t* out);
/* load_map, map_io.hpp:67-115: the reference's map file (layout
 * map_io.hpp:17-21) read in chunks straight into device levels.  Errors in
 * the reference's order: FILE_NOT_FOUND ("file not found: <path>"), IO
 * ("cannot open: <path>"), FORMAT (bad magic, unsupported version, invalid
 * header values, level blocks out of order, truncated map file) — all
 * checked before any device work.  opts may be NULL. */
int bbs_map_load(const char* path, double collision_target, uint64_t memory_cap_bytes,
                 const bbs_map_options* opts, bbs_map_t* out);
/* save_map, map_io.hpp:44-65: byte-identical to the reference's file for the
 * same occupied sets (levels written in occupied_voxels order). */
int bbs_map_save(bbs_map_t map, const char* path);
/* is_map_file, map_io.hpp:119-126: 1 when the file starts with the magic. */
int bbs_is_map_file(const char* path);
int bbs_map_free(bbs_map_t map);
int bbs_map_min_resolution(bbs_map_t map, double* out);   /* voxel_map.hpp:263 */
int bbs_map_max_level(bbs_map_t map, int32_t* out);       /* voxel_map.hpp:264 */
int bbs_map_bbox(bbs_map_t map, bbs_aabb* out);           /* voxel_map.hpp:265 */
/* Device time of the map build ("Create voxel maps", Stats::create_voxel_maps_ms). */
int bbs_map_build_ms(bbs_map_t map, double* out);
/* Run all later work of this map on `stream` (a cudaStream_t owned by the
 * caller, e.g. torch's current stream); NULL restores the map's own stream. */
int bbs_map_set_stream(bbs_map_t map, void* stream);
int bbs_map_level_info(bbs_map_t map, int32_t level, bbs_level_info* out);
/* LevelMap::occupied_voxels, voxel_map.hpp:158-165: ascending (x,y,z). */
int bbs_level_occupied(bbs_map_t map, int32_t level, int32_t* xyz, uint64_t capacity,
                       uint64_t* count);
/* LevelMap::contains, voxel_map.hpp:127-135, for n voxel triples. */
int bbs_level_contains(bbs_map_t map, int32_t level, const int32_t* xyz, uint64_t n,
                       uint8_t* out);
/* LevelMap::score, voxel_map.hpp:142-154: rotation row-major (Transform,
 * geometry.hpp:62-64). */
int bbs_level_score(bbs_map_t map, int32_t level, const double rotation[9],
                    const double translation[3], const double* scan_xyz, uint64_t k,
                    int32_t* score);

/* ---- search (L5/L6) --------------------------------------------------- */
/* batch_evaluate, search.hpp:23-34: nodes scored in place (host buffer).
 * The AngularGrid is built from (cfg, d_max); d_max <= 0 means
 * max_range(scan). */
int bbs_batch_evaluate(bbs_map_t map, const double* scan_xyz, uint64_t k,
                       const bbs_search_config* cfg, double d_max, bbs_node* nodes, uint64_t n);
/* search, search.hpp:72-186. */
int bbs_search(bbs_map_t map, const double* scan_xyz, uint64_t k, const bbs_search_config* cfg,
               bbs_search_result* result);
/* localize_scan, pipeline.hpp:45-51: prepare_source, then search.
 * prepare_source runs auto_leaf's voxel counts on the device; the
 * centroids are summed in the reference's order (bit-identical to the
 * reference's localize_scan).  = bbs_localize_scan_ex(..., BBS_PREPARE_EXACT). */
int bbs_localize_scan(bbs_map_t map, const double* raw_xyz, uint64_t n,
                      const bbs_search_config* cfg, uint64_t downsample_target,
                      bbs_search_result* result);
enum {
  BBS_PREPARE_EXACT = 0,  /* centroids in the reference's std::sort order (host replay) */
  BBS_PREPARE_DEVICE = 1  /* centroids summed on the device in input order (faster; a voxel of
                             >= 3 points may differ in the last bits, see
                             bbs_prepare_source_device) */
};
int bbs_localize_scan_ex(bbs_map_t map, const double* raw_xyz, uint64_t n,
                         const bbs_search_config* cfg, uint64_t downsample_target, int32_t prepare,
                         bbs_search_result* result);

/* Device-resident scan: upload once, search many times with no host copy
 * of the scan inside the call. */
int bbs_scan_upload(bbs_map_t map, const double* xyz, uint64_t k, bbs_scan_t* out);
int bbs_scan_free(bbs_scan_t scan);
int bbs_search_scan(bbs_map_t map, bbs_scan_t scan, const bbs_search_config* cfg,
                    bbs_search_result* result);
/* search_scan on a caller stream (a cudaStream_t; NULL = the map's stream):
 * independent searches on different streams run concurrently on the GPU
 * (each call leases its own workspace; the map is shared read-only). */
int bbs_search_scan_on(bbs_map_t map, bbs_scan_t scan, const bbs_search_config* cfg, void* stream,
                       bbs_search_result* result);
/* Throughput mode (C4: many scans, one map): search() for each of n
 * device-resident scans, `concurrency` searches in flight at a time (native
 * worker threads, one stream each; every search leases its own workspace).
 * results[i] receives scan i's result (its trace buffer as set by the
 * caller).  The first failure is returned after all workers stop. */
int bbs_search_scans(bbs_map_t map, const bbs_scan_t* scans, uint64_t n, const bbs_search_config* cfg,
                     int32_t concurrency, bbs_search_result* results);
/* Non-blocking stream on `device` for bbs_search_scan_on. */
int bbs_stream_create(int32_t device, void** out);
int bbs_stream_destroy(void* stream);
/* batch_evaluate over DEVICE node memory (n nodes at d_nodes) on `stream`
 * (a cudaStream_t, NULL = the map's stream).  Asynchronous. */
int bbs_batch_evaluate_device(bbs_map_t map, bbs_scan_t scan, const bbs_search_config* cfg,
                              double d_max, bbs_node* d_nodes, uint64_t n, void* stream);

/* oracle_search, oracle.hpp:29-95: every level-0 leaf under the root index
 * ranges x the level-0 rotation grid, enumerated and scored on the device.
 * best_score = the maximum (the reference's OracleResult::best_score);
 * argmax receives the first argmax_capacity leaves attaining it, in the
 * reference's enumeration order (their poses are node_pose(.).normalized(),
 * see the facade); argmax_count is the full count; leaf_count the grid size.
 * Errors as the reference: DEGENERATE_SCAN, CONFIG (r mismatch),
 * EMPTY_SEARCH_SPACE, TOO_LARGE (> 1e8 leaves). */
int bbs_oracle_search(bbs_map_t map, const double* scan_xyz, uint64_t k, const bbs_search_config* cfg,
                      int32_t* best_score, bbs_node* argmax, uint64_t argmax_capacity,
                      uint64_t* argmax_count, uint64_t* leaf_count);

/* oracle_search returning EVERY argmax leaf in one pass: *argmax is a
 * malloc'ed array of *argmax_count nodes (release with bbs_free; non-NULL
 * on success even when the count is 0). */
int bbs_oracle_search_all(bbs_map_t map, const double* scan_xyz, uint64_t k, const bbs_search_config* cfg,
                          int32_t* best_score, bbs_node** argmax, uint64_t* argmax_count,
                          uint64_t* leaf_count);
/* Releases memory the library malloc'ed for the caller. */
void bbs_free(void* p);

/* ---- multi-GPU ------------------------------------------ */
/* Element-wise MAX all-reduce of `count` int64 values in place across all
 * ranks; returns 0 on success.  Supplied by the caller (NCCL / gloo). */
typedef int (*bbs_allreduce_max_fn)(int64_t* values, int32_t count, void* user);

/* NCCL communicator for the device-side exchanges of a sharded search
 * (ncclAllReduce MAX on the search stream over NVLink / NVSwitch; no host
 * round-trip per epoch).  NCCL is loaded at run time (libnccl.so.2; inside
 * a torch process, the NCCL torch already loaded).  Rank 0 calls
 * bbs_comm_unique_id and ships the 128 bytes to every rank out of band
 * (e.g. torch.distributed.broadcast_object_list); every rank then calls
 * bbs_comm_init collectively.  One sharded search per comm at a time. */
typedef struct bbs_comm* bbs_comm_t;
int bbs_comm_unique_id(uint8_t id[128]);
int bbs_comm_init(int32_t device, int32_t rank, int32_t world_size, const uint8_t id[128],
                  bbs_comm_t* out);
int bbs_comm_free(bbs_comm_t comm);
/* Version of the loaded NCCL (e.g. 22809), 0 when NCCL cannot be loaded. */
int bbs_nccl_version(void);

/* Sharding modes. */
enum {
  /* Each rank runs its own best-first BnB over its share of the root set and
   * adopts the max-all-reduced incumbent after every epoch; the winner is
   * elected at the end.  RotoTrans results may differ from the
   * single-queue schedule (SURVEY §8e caveat); TransOnly best scores equal
   * the unsharded search (admissible bound). */
  BBS_SHARD_ROOTS = 0,
  /* Batch-split exact mode: every rank replays the single-queue schedule;
   * the root batch and every flush batch are split across the ranks (root
   * units as above, flush runs of 8 children by run % world_size) and the
   * int32 scores max-all-reduced, so every rank returns the unsharded
   * search() result exactly (score, pose, Stats, trace). */
  BBS_SHARD_EXACT = 1
};

typedef struct bbs_shard {
  int32_t rank;
  int32_t world_size;
  bbs_allreduce_max_fn allreduce_max; /* host exchange; used when comm is NULL */
  void* user;
  int32_t mode;                       /* BBS_SHARD_ROOTS / BBS_SHARD_EXACT */
  int32_t reserved;
  bbs_comm_t comm;                    /* device exchange (NCCL); NULL = allreduce_max */
} bbs_shard;
/* search() sharded across ranks (see the modes above).  Root (ix, iy, iz,
 * rot) of initial_nodes belongs to rank ((ix - ix_min) * n_rot + rot) %
 * world_size.  Every rank returns the same best pose/score.  ROOTS: Stats
 * are this rank's; EXACT: Stats are the whole search's. */
int bbs_search_sharded(bbs_map_t map, bbs_scan_t scan, const bbs_search_config* cfg,
                       const bbs_shard* shard, bbs_search_result* result);

/* ---- parity instrumentation ------------------------------------------ */
/* What the device scored inside one search(), for per-candidate parity
 * against the reference's batch_evaluate (search.hpp:23-34): the root batch
 * (search.hpp:111-124) and the flushed batches (search.hpp:132-143).
 * Buffers are caller-owned host memory; *_count receive the full counts even
 * when they exceed the capacities (only the first capacity entries are
 * written). */
typedef struct bbs_search_dump {
  /* 1: the root kernel runs without its survivor-bound early exit, so every
   * root score is the full hit count (default 0: roots that provably cannot
   * reach the threshold stop early and keep a partial count below it). */
  int32_t exact_roots;
  /* dump the flush batches of epochs e with e % epoch_stride == 0 (0 = 1) */
  uint32_t epoch_stride;
  int32_t* root_scores;        /* initial_nodes() order (nodes.hpp:77-83) */
  uint64_t root_capacity;
  uint64_t root_count;
  bbs_node* flush_nodes;       /* pending batches in the reference's order */
  int32_t* flush_scores;       /* their device scores */
  uint64_t flush_capacity;
  uint64_t flush_count;
  uint64_t* epoch_offsets;     /* batch i = [epoch_offsets[i], epoch_offsets[i+1]) */
  uint32_t* epoch_ids;         /* flush index (0-based, roots excluded) of batch i */
  uint64_t epoch_capacity;     /* entries of epoch_ids; epoch_offsets holds +1 */
  uint64_t epoch_count;
} bbs_search_dump;
/* search_scan with the dump above: one epoch per host check, no CUDA graphs,
 * the flush batches copied out after each epoch.  Results (score, pose,
 * Stats, trace) are the same as bbs_search_scan's. */
int bbs_search_scan_dump(bbs_map_t map, bbs_scan_t scan, const bbs_search_config* cfg,
                         bbs_search_dump* dump, bbs_search_result* result);

/* ---- measurement ------------------------------------------------------ */
/* Random independent 32-byte gather ceiling over a `bytes` buffer on
 * `device` (SURVEY §8d tier ceilings): sector GB/s. */
int bbs_gather_bench(int32_t device, uint64_t bytes, double* out_gbs);
/* Conflict-free random 4-byte shared-memory read ceiling of the whole GPU
 * (GB/s): the tier the root column kernel gathers from. */
int bbs_smem_bench(int32_t device, double* out_gbs);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif  /* BBS_B200_H */

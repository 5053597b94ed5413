/*
 * bbs_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's batched branch-and-bound path
 * (/root/reference/proj/include/bnbloc), used by tests/ as the parity
 * checker and by bench.py's cpu_baseline leg.  The product never links or
 * calls it.  Parity of this restatement is PINNED against the reference
 * itself: tests/test_oracle.py compares it with oracle/_ref (the unmodified
 * reference headers compiled by oracle/Makefile) and with the committed
 * golden fixtures in tests/golden/ that were generated from oracle/_ref.
 *
 * Types reuse include/bbs.h (byte-compatible with the reference types).
 */
#ifndef BBS_ORACLE_H
#define BBS_ORACLE_H

#include <stdint.h>

#include "bbs.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_map orc_map;

/* point_cloud.hpp:38-40 (x86 cvttsd2si semantics made explicit). */
int32_t orc_voxel_index(double coord, double cell);
/* MultiResVoxelMap::build, voxel_map.hpp:226-244 (set semantics only). */
int orc_map_build(const double* xyz, uint64_t n, double r, int32_t max_level, orc_map** out);
void orc_map_free(orc_map* m);
uint64_t orc_level_count(const orc_map* m, int32_t level);
/* occupied_voxels, voxel_map.hpp:158-165 (ascending). */
const int32_t* orc_level_voxels(const orc_map* m, int32_t level);
int orc_level_contains(const orc_map* m, int32_t level, int32_t x, int32_t y, int32_t z);
/* LevelMap::score, voxel_map.hpp:142-154. */
int32_t orc_level_score(const orc_map* m, int32_t level, const double* rot9, const double* t3,
                        const double* scan, uint64_t k);
/* pose_to_transform, geometry.hpp:102-112. */
void orc_pose_to_transform(const double* pose6, double* rot9, double* t3);
/* AngularGrid, angular_grid.hpp:67-99; out has 3*(max_level+1) entries. */
int orc_angular_grid(const bbs_search_config* cfg, double d_max, bbs_axis_grid* out);
int32_t orc_divisions(const bbs_axis_grid* g, int32_t max_level, int32_t axis, int32_t level);
/* node_pose, nodes.hpp:33-43. */
void orc_node_pose(const bbs_axis_grid* g, int32_t max_level, double r, const bbs_node* n,
                   double* pose6);
/* max_range, point_cloud.hpp:58-63. */
double orc_max_range(const double* xyz, uint64_t n);
/* batch_evaluate, search.hpp:23-34. */
int orc_batch_evaluate(const orc_map* m, const double* scan, uint64_t k,
                       const bbs_search_config* cfg, double d_max, bbs_node* nodes, uint64_t n);
/* search, search.hpp:72-186 (timers are wall-clock of this restatement). */
int orc_search(const orc_map* m, const bbs_aabb* map_bbox, const double* scan, uint64_t k,
               const bbs_search_config* cfg, bbs_search_result* out);
/* Root-sharded search: roots with index % world == rank; the
 * incumbent is max-all-reduced after the root batch and after every flush;
 * winner elected by (score, lowest rank).  world == 1 equals orc_search. */
int orc_search_sharded(const orc_map* m, const bbs_aabb* map_bbox, const double* scan,
                       uint64_t k, const bbs_search_config* cfg, const bbs_shard* shard,
                       bbs_search_result* out);
/* oracle_search, oracle.hpp:29-95: best leaf score over the full leaf grid
 * and the number of argmax leaves. */
int orc_exhaustive(const orc_map* m, const bbs_aabb* map_bbox, const double* scan, uint64_t k,
                   const bbs_search_config* cfg, int32_t* best, uint64_t* n_argmax,
                   uint64_t* leaf_count);

#ifdef __cplusplus
}
#endif

#endif

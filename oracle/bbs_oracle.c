/*
 * bbs_oracle.c — TEST INFRASTRUCTURE ONLY (see bbs_oracle.h).
 *
 * Plain-C restatement of the reference path.  Every function cites the
 * reference lines it restates (paths relative to
 * /root/reference/proj/include/bnbloc/).  Compiled with -O2
 * -ffp-contract=off so every double expression rounds exactly like the
 * reference build (the reference binary has no FMAs).
 * Membership uses a private hash set; only the SET matters for scores
 * (voxel_map.hpp:127-135), so the reference's bucket sizing is not restated.
 */
#include "bbs_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define ORC_PI 3.141592653589793238462643383279502884

typedef struct {
  int32_t x, y, z;
} vox;

typedef struct {
  vox* sorted;   /* ascending (x, y, z), voxel_map.hpp:27-31 */
  uint64_t n;
  vox* slots;    /* open addressing, empty = INT32_MIN^3 */
  uint64_t mask;
} level_set;

struct orc_map {
  double r;
  int32_t max_level;
  level_set* levels;
};

static const int32_t kEmpty = INT32_MIN;

/* point_cloud.hpp:38-40: static_cast<int32_t>(std::floor(c / cell)).  The
 * reference build converts with cvttsd2si, which yields INT32_MIN for NaN
 * and any value outside [-2^31, 2^31); made explicit here. */
int32_t orc_voxel_index(double coord, double cell) {
  const double f = floor(coord / cell);
  if (!(f >= -2147483648.0 && f < 2147483648.0)) return INT32_MIN;
  return (int32_t)f;
}

static int vox_cmp(const void* a, const void* b) {
  const vox* p = (const vox*)a;
  const vox* q = (const vox*)b;
  if (p->x != q->x) return p->x < q->x ? -1 : 1;
  if (p->y != q->y) return p->y < q->y ? -1 : 1;
  if (p->z != q->z) return p->z < q->z ? -1 : 1;
  return 0;
}

static uint64_t sort_unique(vox* v, uint64_t n) {
  if (n == 0) return 0;
  qsort(v, n, sizeof(vox), vox_cmp);
  uint64_t w = 1;
  for (uint64_t i = 1; i < n; ++i)
    if (vox_cmp(&v[i], &v[w - 1]) != 0) v[w++] = v[i];
  return w;
}

static uint64_t mix(int32_t x, int32_t y, int32_t z) {
  uint64_t h = (uint64_t)(uint32_t)x * 0x9E3779B97F4A7C15ULL;
  h ^= (uint64_t)(uint32_t)y * 0xC2B2AE3D27D4EB4FULL;
  h ^= (uint64_t)(uint32_t)z * 0x165667B19E3779F9ULL;
  h ^= h >> 31;
  h *= 0xBF58476D1CE4E5B9ULL;
  return h ^ (h >> 29);
}

static int set_contains(const level_set* s, int32_t x, int32_t y, int32_t z) {
  /* contains(kEmpty) is false in the reference (voxel_map.hpp:131). */
  if (x == kEmpty && y == kEmpty && z == kEmpty) return 0;
  uint64_t i = mix(x, y, z) & s->mask;
  for (;;) {
    const vox* v = &s->slots[i];
    if (v->x == kEmpty && v->y == kEmpty && v->z == kEmpty) return 0;
    if (v->x == x && v->y == y && v->z == z) return 1;
    i = (i + 1) & s->mask;
  }
}

static void set_init(level_set* s, vox* sorted, uint64_t n) {
  s->sorted = sorted;
  s->n = n;
  uint64_t cap = 16;
  while (cap < 2 * n) cap <<= 1;
  s->slots = (vox*)malloc(sizeof(vox) * cap);
  for (uint64_t i = 0; i < cap; ++i) s->slots[i].x = s->slots[i].y = s->slots[i].z = kEmpty;
  s->mask = cap - 1;
  for (uint64_t k = 0; k < n; ++k) {
    const vox v = sorted[k];
    /* A kEmpty key cannot be stored by the reference table either
     * (voxel_map.hpp:102-108 writes it into an empty slot, which stays empty). */
    if (v.x == kEmpty && v.y == kEmpty && v.z == kEmpty) continue;
    uint64_t i = mix(v.x, v.y, v.z) & s->mask;
    while (!(s->slots[i].x == kEmpty && s->slots[i].y == kEmpty && s->slots[i].z == kEmpty))
      i = (i + 1) & s->mask;
    s->slots[i] = v;
  }
}

/* inflated_voxels, voxel_map.hpp:186-206: voxelize at ldexp(r, level),
 * sort/unique, inflate with v - j for j in {0,1}^3, sort/unique. */
static void build_level(const double* xyz, uint64_t n, int32_t level, double r, level_set* out) {
  const double cell = ldexp(r, level);
  vox* src = (vox*)malloc(sizeof(vox) * (n ? n : 1));
  for (uint64_t i = 0; i < n; ++i) {
    src[i].x = orc_voxel_index(xyz[3 * i], cell);
    src[i].y = orc_voxel_index(xyz[3 * i + 1], cell);
    src[i].z = orc_voxel_index(xyz[3 * i + 2], cell);
  }
  const uint64_t ns = sort_unique(src, n);
  vox* inf = (vox*)malloc(sizeof(vox) * (ns * 8 ? ns * 8 : 1));
  uint64_t w = 0;
  for (uint64_t i = 0; i < ns; ++i)
    for (int32_t jx = 0; jx <= 1; ++jx)
      for (int32_t jy = 0; jy <= 1; ++jy)
        for (int32_t jz = 0; jz <= 1; ++jz) {
          /* two's-complement wrap for INT32_MIN - 1, like the reference build */
          inf[w].x = (int32_t)((uint32_t)src[i].x - (uint32_t)jx);
          inf[w].y = (int32_t)((uint32_t)src[i].y - (uint32_t)jy);
          inf[w].z = (int32_t)((uint32_t)src[i].z - (uint32_t)jz);
          ++w;
        }
  free(src);
  const uint64_t nu = sort_unique(inf, w);
  set_init(out, inf, nu);
}

/* MultiResVoxelMap::build, voxel_map.hpp:226-244 (validation :230-233). */
int orc_map_build(const double* xyz, uint64_t n, double r, int32_t max_level, orc_map** out) {
  if (n == 0) return BBS_ERR_EMPTY_CLOUD;
  if (max_level < 1) return BBS_ERR_CONFIG;
  if (!(r > 0.0)) return BBS_ERR_CONFIG;
  orc_map* m = (orc_map*)calloc(1, sizeof(orc_map));
  m->r = r;
  m->max_level = max_level;
  m->levels = (level_set*)calloc((size_t)max_level + 1, sizeof(level_set));
  for (int32_t l = 0; l <= max_level; ++l) build_level(xyz, n, l, r, &m->levels[l]);
  *out = m;
  return BBS_OK;
}

void orc_map_free(orc_map* m) {
  if (!m) return;
  for (int32_t l = 0; l <= m->max_level; ++l) {
    free(m->levels[l].sorted);
    free(m->levels[l].slots);
  }
  free(m->levels);
  free(m);
}

uint64_t orc_level_count(const orc_map* m, int32_t level) { return m->levels[level].n; }
const int32_t* orc_level_voxels(const orc_map* m, int32_t level) {
  return (const int32_t*)m->levels[level].sorted;
}
int orc_level_contains(const orc_map* m, int32_t level, int32_t x, int32_t y, int32_t z) {
  return set_contains(&m->levels[level], x, y, z);
}

/* LevelMap::score, voxel_map.hpp:142-154 — same expression order. */
int32_t orc_level_score(const orc_map* m, int32_t level, const double* r, const double* t,
                        const double* scan, uint64_t k) {
  const level_set* s = &m->levels[level];
  const double cell = ldexp(m->r, level);
  int32_t hits = 0;
  for (uint64_t i = 0; i < k; ++i) {
    const double px = scan[3 * i], py = scan[3 * i + 1], pz = scan[3 * i + 2];
    const double qx = r[0] * px + r[1] * py + r[2] * pz + t[0];
    const double qy = r[3] * px + r[4] * py + r[5] * pz + t[1];
    const double qz = r[6] * px + r[7] * py + r[8] * pz + t[2];
    hits += set_contains(s, orc_voxel_index(qx, cell), orc_voxel_index(qy, cell),
                         orc_voxel_index(qz, cell));
  }
  return hits;
}

/* pose_to_transform, geometry.hpp:102-112. */
void orc_pose_to_transform(const double* p, double* R, double* t) {
  const double ca = cos(p[3]), sa = sin(p[3]);
  const double cb = cos(p[4]), sb = sin(p[4]);
  const double cg = cos(p[5]), sg = sin(p[5]);
  R[0] = cg * cb;
  R[1] = cg * sb * sa - sg * ca;
  R[2] = cg * sb * ca + sg * sa;
  R[3] = sg * cb;
  R[4] = sg * sb * sa + cg * ca;
  R[5] = sg * sb * ca - cg * sa;
  R[6] = -sb;
  R[7] = cb * sa;
  R[8] = cb * ca;
  t[0] = p[0];
  t[1] = p[1];
  t[2] = p[2];
}

/* angular_step, angular_grid.hpp:20-26. */
static int angular_step(double cell, double d_max, double* out) {
  if (!(d_max > 0.0)) return BBS_ERR_DEGENERATE_SCAN;
  if (!(cell > 0.0)) return BBS_ERR_CONFIG;
  const double half_chord = cell / (2.0 * d_max);
  if (half_chord >= 1.0) {
    *out = ORC_PI;
    return BBS_OK;
  }
  *out = 2.0 * asin(half_chord);
  return BBS_OK;
}

/* AngularGrid ctor, angular_grid.hpp:67-99 (adjusted_step :34-39). */
int orc_angular_grid(const bbs_search_config* cfg, double d_max, bbs_axis_grid* out) {
  if (!(cfg->yaw_max > cfg->yaw_min)) return BBS_ERR_CONFIG;
  if (cfg->roll_pitch_half_range < 0.0) return BBS_ERR_CONFIG;
  const double rp = cfg->roll_pitch_half_range;
  const double w_min[3] = {-rp, -rp, cfg->yaw_min};
  const double w_max[3] = {rp, rp, cfg->yaw_max};
  const int L = cfg->max_level + 1;
  for (int axis = 0; axis < 3; ++axis)
    for (int l = 0; l <= cfg->max_level; ++l) {
      const int step_level = cfg->branch_mode == BBS_BRANCH_TRANS_ONLY ? 0 : l;
      const double cell = ldexp(cfg->min_resolution, step_level);
      double delta;
      const int st = angular_step(cell, d_max, &delta);
      if (st) return st;
      bbs_axis_grid g;
      g.w_min = w_min[axis];
      g.w_max = w_max[axis];
      g.periodic = axis == 2;
      g.step = 0.0;
      g.segments = 0;
      const double range = g.w_max - g.w_min;
      if (range > 0.0) {
        if (!(delta > 0.0)) return BBS_ERR_CONFIG;
        const int segments = (int)ceil(range / delta);
        g.step = range / (double)segments;
        g.segments = segments;
      }
      out[axis * L + l] = g;
    }
  return BBS_OK;
}

/* AxisGrid::max_index / index_count / angle, angular_grid.hpp:52-57. */
static int32_t max_index(const bbs_axis_grid* g) {
  if (g->segments == 0) return 0;
  return g->periodic ? g->segments - 1 : g->segments;
}
static double axis_angle(const bbs_axis_grid* g, int32_t idx) {
  return g->w_min + g->step * (double)idx;
}
static const bbs_axis_grid* axis_at(const bbs_axis_grid* g, int32_t max_level, int a, int l) {
  return &g[a * (max_level + 1) + l];
}

/* AngularGrid::divisions, angular_grid.hpp:111-116. */
int32_t orc_divisions(const bbs_axis_grid* g, int32_t max_level, int32_t axis, int32_t level) {
  const bbs_axis_grid* parent = axis_at(g, max_level, axis, level);
  const bbs_axis_grid* child = axis_at(g, max_level, axis, level - 1);
  if (child->segments <= 1) return 1;
  return (child->segments + parent->segments - 1) / parent->segments;
}

/* node_pose, nodes.hpp:33-43. */
void orc_node_pose(const bbs_axis_grid* g, int32_t max_level, double r, const bbs_node* n,
                   double* p) {
  const double cell = ldexp(r, n->level);
  p[0] = cell * (double)n->ix;
  p[1] = cell * (double)n->iy;
  p[2] = cell * (double)n->iz;
  p[3] = axis_angle(axis_at(g, max_level, 0, n->level), n->iroll);
  p[4] = axis_angle(axis_at(g, max_level, 1, n->level), n->ipitch);
  p[5] = axis_angle(axis_at(g, max_level, 2, n->level), n->iyaw);
}

/* max_range, point_cloud.hpp:58-63 (Point3::norm, geometry.hpp:24). */
double orc_max_range(const double* xyz, uint64_t n) {
  double m = 0.0;
  for (uint64_t i = 0; i < n; ++i) {
    const double x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
    const double v = sqrt(x * x + y * y + z * z);
    m = m < v ? v : m; /* std::max(m, v) */
  }
  return m;
}

static void score_node(const orc_map* m, const bbs_axis_grid* g, int32_t grid_max_level,
                       const double* scan, uint64_t k, bbs_node* n) {
  double pose[6], R[9], t[3];
  orc_node_pose(g, grid_max_level, m->r, n, pose);
  orc_pose_to_transform(pose, R, t);
  n->score = orc_level_score(m, n->level, R, t, scan, k);
}

/* batch_evaluate, search.hpp:23-34. */
int orc_batch_evaluate(const orc_map* m, const double* scan, uint64_t k,
                       const bbs_search_config* cfg, double d_max, bbs_node* nodes, uint64_t n) {
  const double dm = d_max > 0 ? d_max : orc_max_range(scan, k);
  bbs_axis_grid* g = (bbs_axis_grid*)malloc(sizeof(bbs_axis_grid) * 3 * (cfg->max_level + 1));
  const int st = orc_angular_grid(cfg, dm, g);
  if (st) {
    free(g);
    return st;
  }
  for (uint64_t i = 0; i < n; ++i) score_node(m, g, cfg->max_level, scan, k, &nodes[i]);
  free(g);
  return BBS_OK;
}

/* ---- search, search.hpp:36-186 ----------------------------------------- */

typedef struct {
  bbs_node node;
  uint64_t seq;
} entry; /* QueueEntry, search.hpp:38-41 */

typedef struct {
  entry* a;
  uint64_t n, cap;
  int bfs;
} heap;

/* EntryCompare, search.hpp:47-59: returns 1 when a pops AFTER b. */
static int lower(const heap* h, const entry* a, const entry* b) {
  if (h->bfs) {
    if (a->node.score != b->node.score) return a->node.score < b->node.score;
    if (a->node.level != b->node.level) return a->node.level < b->node.level;
    return a->seq > b->seq;
  }
  if (a->node.level != b->node.level) return a->node.level > b->node.level;
  if (a->node.score != b->node.score) return a->node.score < b->node.score;
  return a->seq < b->seq;
}

static void heap_push(heap* h, const bbs_node* n, uint64_t seq) {
  if (h->n == h->cap) {
    h->cap = h->cap ? 2 * h->cap : 1024;
    h->a = (entry*)realloc(h->a, sizeof(entry) * h->cap);
  }
  uint64_t i = h->n++;
  entry e = {*n, seq};
  while (i > 0) {
    const uint64_t p = (i - 1) / 2;
    if (!lower(h, &h->a[p], &e)) break;
    h->a[i] = h->a[p];
    i = p;
  }
  h->a[i] = e;
}

static entry heap_pop(heap* h) {
  const entry top = h->a[0];
  const entry last = h->a[--h->n];
  uint64_t i = 0;
  for (;;) {
    uint64_t c = 2 * i + 1;
    if (c >= h->n) break;
    if (c + 1 < h->n && lower(h, &h->a[c], &h->a[c + 1])) ++c;
    if (!lower(h, &last, &h->a[c])) break;
    h->a[i] = h->a[c];
    i = c;
  }
  if (h->n) h->a[i] = last;
  return top;
}

static double now_ms(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

typedef struct {
  int32_t min, max;
} trange; /* TransIndexRange, nodes.hpp:45-49 */

/* trans_index_range, nodes.hpp:53-56. */
static trange trans_index_range(double lo, double hi, double cell) {
  trange r;
  const double f = floor(lo / cell), c = ceil(hi / cell);
  r.min = (f >= -2147483648.0 && f < 2147483648.0) ? (int32_t)f : INT32_MIN;
  r.max = (c >= -2147483648.0 && c < 2147483648.0) ? (int32_t)c : INT32_MIN;
  return r;
}

/* initial_nodes, nodes.hpp:60-85 (loop order ix, iy, iz, ir, ip, iw). */
static int initial_nodes(const bbs_aabb* range, const bbs_axis_grid* g, int32_t L, double r,
                         bbs_node** out, uint64_t* count) {
  const double cell = ldexp(r, L);
  const trange rx = trans_index_range(range->min.x, range->max.x, cell);
  const trange ry = trans_index_range(range->min.y, range->max.y, cell);
  const trange rz = trans_index_range(range->min.z, range->max.z, cell);
  const int32_t nr = max_index(axis_at(g, L, 0, L)) + 1;
  const int32_t np = max_index(axis_at(g, L, 1, L)) + 1;
  const int32_t nw = max_index(axis_at(g, L, 2, L)) + 1;
  const int64_t total = ((int64_t)rx.max - rx.min + 1) * ((int64_t)ry.max - ry.min + 1) *
                        ((int64_t)rz.max - rz.min + 1) * nr * np * nw;
  if (total <= 0) return BBS_ERR_EMPTY_SEARCH_SPACE;
  bbs_node* v = (bbs_node*)malloc(sizeof(bbs_node) * (size_t)total);
  uint64_t w = 0;
  for (int32_t ix = rx.min; ix <= rx.max; ++ix)
    for (int32_t iy = ry.min; iy <= ry.max; ++iy)
      for (int32_t iz = rz.min; iz <= rz.max; ++iz)
        for (int32_t ir = 0; ir < nr; ++ir)
          for (int32_t ip = 0; ip < np; ++ip)
            for (int32_t iw = 0; iw < nw; ++iw) {
              bbs_node n = {ix, iy, iz, ir, ip, iw, L, -1};
              v[w++] = n;
            }
  *out = v;
  *count = w;
  return BBS_OK;
}

/* branch, nodes.hpp:91-121 (loop order jr, jp, jw, jx, jy, jz). */
static uint64_t branch(const bbs_node* c, const bbs_axis_grid* g, int32_t L, bbs_node* out) {
  const int32_t cl = c->level - 1;
  const int32_t ar = orc_divisions(g, L, 0, c->level);
  const int32_t ap = orc_divisions(g, L, 1, c->level);
  const int32_t aw = orc_divisions(g, L, 2, c->level);
  const int32_t mr = max_index(axis_at(g, L, 0, cl));
  const int32_t mp = max_index(axis_at(g, L, 1, cl));
  const int32_t mw = max_index(axis_at(g, L, 2, cl));
  uint64_t w = 0;
  for (int32_t jr = 0; jr < ar; ++jr) {
    const int32_t ir = ar * c->iroll + jr;
    if (ir > mr) break;
    for (int32_t jp = 0; jp < ap; ++jp) {
      const int32_t ip = ap * c->ipitch + jp;
      if (ip > mp) break;
      for (int32_t jw = 0; jw < aw; ++jw) {
        const int32_t iw = aw * c->iyaw + jw;
        if (iw > mw) break;
        for (int32_t jx = 0; jx <= 1; ++jx)
          for (int32_t jy = 0; jy <= 1; ++jy)
            for (int32_t jz = 0; jz <= 1; ++jz) {
              bbs_node n = {2 * c->ix + jx, 2 * c->iy + jy, 2 * c->iz + jz, ir, ip, iw, cl, -1};
              out[w++] = n;
            }
      }
    }
  }
  return w;
}

/* Exact mode: element-wise MAX of the nodes' scores over the ranks. */
static int exchange_scores(const bbs_shard* shard, bbs_node* nodes, uint64_t n) {
  const uint64_t chunk = 1u << 20;
  int64_t* v = (int64_t*)malloc(sizeof(int64_t) * (n < chunk ? (n ? n : 1) : chunk));
  for (uint64_t o = 0; o < n; o += chunk) {
    const uint64_t c = n - o < chunk ? n - o : chunk;
    for (uint64_t i = 0; i < c; ++i) v[i] = nodes[o + i].score;
    if (shard->allreduce_max(v, (int32_t)c, shard->user)) {
      free(v);
      return 1;
    }
    for (uint64_t i = 0; i < c; ++i) nodes[o + i].score = (int32_t)v[i];
  }
  free(v);
  return 0;
}

/* Reference loop with an optional incumbent exchange after each batch. */
static int search_impl(const orc_map* m, const bbs_aabb* map_bbox, const double* scan,
                       uint64_t k, const bbs_search_config* cfg, const bbs_shard* shard,
                       bbs_search_result* out) {
  /* validation, search.hpp:79-89, in the same order */
  if (k == 0) return BBS_ERR_DEGENERATE_SCAN;
  if (m->r != cfg->min_resolution) return BBS_ERR_CONFIG;
  if (cfg->max_level < 1 || cfg->max_level > m->max_level) return BBS_ERR_CONFIG;
  if (cfg->batch_size < 1) return BBS_ERR_CONFIG;
  if (!(cfg->score_threshold_fraction > 0.0 && cfg->score_threshold_fraction <= 1.0))
    return BBS_ERR_CONFIG;
  const double d_max = cfg->has_d_max ? cfg->d_max : orc_max_range(scan, k);
  if (!(d_max > 0.0)) return BBS_ERR_DEGENERATE_SCAN;
  const int32_t L = cfg->max_level;
  bbs_axis_grid* g = (bbs_axis_grid*)malloc(sizeof(bbs_axis_grid) * 3 * (L + 1));
  int st = orc_angular_grid(cfg, d_max, g);
  if (st) {
    free(g);
    return st;
  }
  const bbs_aabb* tr = cfg->has_translation_range ? &cfg->translation_range : map_bbox;
  const int rank = shard ? shard->rank : 0;
  const int world = shard ? shard->world_size : 1;
  /* batch-split exact mode: every rank replays the single-queue
   * schedule; root and flush scores are split over the ranks and
   * max-all-reduced (unscored entries are -1) */
  const int exact = shard && shard->mode == BBS_SHARD_EXACT && shard->allreduce_max;

  memset(&out->stats, 0, sizeof(out->stats));
  out->scan_points = k;
  const int32_t threshold = (int32_t)floor(cfg->score_threshold_fraction * (double)k);
  out->score_threshold = threshold;
  int32_t best = threshold;
  bbs_node best_node;
  memset(&best_node, 0, sizeof(best_node));
  int matched = 0;
  uint64_t trace_len = 0;
  heap h = {NULL, 0, 0, cfg->strategy == BBS_STRATEGY_BFS};
  uint64_t seq = 0;
  bbs_stats* stats = &out->stats;

  const double t_init = now_ms();
  bbs_node* roots;
  uint64_t nroots;
  st = initial_nodes(tr, g, L, m->r, &roots, &nroots);
  if (st) {
    free(g);
    return st;
  }
  /* shard: root (ix, iy, iz, rot) belongs to rank
   * ((ix - ix_min) * nrot + rot) % world — whole (x-slab, rotation) units,
   * the rule of the device root kernel (csrc/kernels.h owned_slabs). */
  uint64_t nmine = 0;
  if (exact) {
    const int64_t np_ = max_index(axis_at(g, L, 1, L)) + 1;
    const int64_t nw_ = max_index(axis_at(g, L, 2, L)) + 1;
    const int64_t nrot = (max_index(axis_at(g, L, 0, L)) + 1) * np_ * nw_;
    const int32_t ix_min = nroots ? roots[0].ix : 0;
    for (uint64_t i = 0; i < nroots; ++i) {
      const int64_t rot = ((int64_t)roots[i].iroll * np_ + roots[i].ipitch) * nw_ + roots[i].iyaw;
      const int64_t unit = ((int64_t)roots[i].ix - ix_min) * nrot + rot;
      if ((int)(unit % world) == rank) {
        score_node(m, g, L, scan, k, &roots[i]);
        ++nmine;
      } else {
        roots[i].score = -1;
      }
    }
    if (exchange_scores(shard, roots, nroots)) {
      free(roots);
      free(g);
      return BBS_ERR_GENERIC;
    }
    stats->nodes_generated += nroots;
    out->root_nodes = nmine;
    nmine = nroots; /* every root is in play below, in initial_nodes order */
  } else {
    const int64_t np_ = max_index(axis_at(g, L, 1, L)) + 1;
    const int64_t nw_ = max_index(axis_at(g, L, 2, L)) + 1;
    const int64_t nrot = (max_index(axis_at(g, L, 0, L)) + 1) * np_ * nw_;
    const int32_t ix_min = nroots ? roots[0].ix : 0;
    for (uint64_t i = 0; i < nroots; ++i) {
      const int64_t rot = ((int64_t)roots[i].iroll * np_ + roots[i].ipitch) * nw_ + roots[i].iyaw;
      const int64_t unit = ((int64_t)roots[i].ix - ix_min) * nrot + rot;
      if ((int)(unit % world) == rank) roots[nmine++] = roots[i];
    }
  }
  if (!exact) {
    stats->nodes_generated += nmine;
    out->root_nodes = nmine;
    for (uint64_t i = 0; i < nmine; ++i) score_node(m, g, L, scan, k, &roots[i]);
  }
  stats->batches_flushed++;
  for (uint64_t i = 0; i < nmine; ++i) {
    if (roots[i].score < threshold)
      stats->nodes_pruned++;
    else
      heap_push(&h, &roots[i], seq++);
  }
  free(roots);
  const double t_loop = now_ms();
  stats->initial_nodes_ms = t_loop - t_init;

  /* children of one parent: 8 * prod(divisions) at most */
  uint64_t maxc = 8;
  for (int32_t l = 1; l <= L; ++l) {
    const uint64_t c = 8ULL * orc_divisions(g, L, 0, l) * orc_divisions(g, L, 1, l) *
                       orc_divisions(g, L, 2, l);
    if (c > maxc) maxc = c;
  }
  const uint64_t pcap = cfg->batch_size + maxc + 1;
  bbs_node* pending = (bbs_node*)malloc(sizeof(bbs_node) * pcap);
  uint64_t np = 0;
  double t_last_best = t_loop;

  /* incumbent exchange (sharded only): values = {best, active} */
  int active = 1;
#define EXCHANGE()                                                      \
  do {                                                                  \
    if (shard && shard->allreduce_max && !exact) {                      \
      int64_t v[2] = {best, active};                                    \
      if (shard->allreduce_max(v, 2, shard->user)) {                    \
        st = BBS_ERR_GENERIC;                                           \
        goto done;                                                      \
      }                                                                 \
      if (v[0] > best) best = (int32_t)v[0];                            \
      others_active = v[1] != 0;                                        \
    }                                                                   \
  } while (0)
  int others_active = 0;
  EXCHANGE();

  while (h.n > 0 || np > 0) {
    int flushed = 0;
    if (h.n == 0) {
      flushed = 1;
    } else {
      const entry e = heap_pop(&h);
      const bbs_node* node = &e.node;
      if (node->score < best) {
        stats->nodes_pruned++;
        continue;
      }
      if (node->level == 0) {
        best = node->score;
        best_node = *node;
        matched = 1;
        t_last_best = now_ms();
        if (cfg->collect_trace) {
          if (trace_len < out->trace_capacity) out->best_score_trace[trace_len] = best;
          trace_len++;
        }
        continue;
      }
      const uint64_t nc = branch(node, g, L, pending + np);
      stats->nodes_generated += nc;
      np += nc;
      if (np > cfg->batch_size) flushed = 1;
    }
    if (flushed) {
      /* flush, search.hpp:132-143 */
      if (exact) {
        /* runs of 8 children dealt round-robin (csrc/search.cu RunSplit) */
        for (uint64_t i = 0; i < np; ++i) {
          if ((int)((i / 8) % (uint64_t)world) == rank)
            score_node(m, g, L, scan, k, &pending[i]);
          else
            pending[i].score = -1;
        }
        if (exchange_scores(shard, pending, np)) {
          st = BBS_ERR_GENERIC;
          goto done;
        }
      } else {
        for (uint64_t i = 0; i < np; ++i) score_node(m, g, L, scan, k, &pending[i]);
      }
      stats->batches_flushed++;
      for (uint64_t i = 0; i < np; ++i) {
        if (pending[i].score < best)
          stats->nodes_pruned++;
        else
          heap_push(&h, &pending[i], seq++);
      }
      np = 0;
      EXCHANGE();
    }
  }
  /* this rank is done; keep answering exchanges until every rank is */
  active = 0;
  if (shard && shard->allreduce_max && !exact) {
    do {
      EXCHANGE();
    } while (others_active);
  }

  {
    const double t_end = now_ms();
    if (matched) {
      stats->find_best_score_ms = t_last_best - t_loop;
      stats->pop_remaining_queue_ms = t_end - t_last_best;
    } else {
      stats->find_best_score_ms = t_end - t_loop;
      stats->pop_remaining_queue_ms = 0.0;
    }
  }

  /* winner election (sharded): max of (score, world-1-rank) among matched */
  if (shard && shard->allreduce_max && world > 1 && !exact) {
    int64_t key[1] = {matched ? ((int64_t)best << 32) | (int64_t)(world - 1 - rank) : -1};
    if (shard->allreduce_max(key, 1, shard->user)) {
      st = BBS_ERR_GENERIC;
      goto done;
    }
    const int winner = key[0] < 0 ? -1 : (int)(world - 1 - (key[0] & 0xffffffff));
    int64_t nv[8];
    const int32_t* f = (const int32_t*)&best_node;
    for (int i = 0; i < 8; ++i) nv[i] = (rank == winner) ? (int64_t)f[i] : INT64_MIN;
    if (shard->allreduce_max(nv, 8, shard->user)) {
      st = BBS_ERR_GENERIC;
      goto done;
    }
    if (winner >= 0) {
      int32_t* bf = (int32_t*)&best_node;
      for (int i = 0; i < 8; ++i) bf[i] = (int32_t)nv[i];
      best = (int32_t)(key[0] >> 32);
      matched = 1;
    } else {
      matched = 0;
    }
  }

  out->matched = matched;
  out->best_score = best;
  out->best_node = best_node;
  out->trace_length = trace_len;
  if (matched) {
    /* node_pose(...).normalized(), search.hpp:183 / geometry.hpp:36-43,55-59 */
    double p[6];
    orc_node_pose(g, L, m->r, &best_node, p);
    const double two_pi = 6.283185307179586476925286766559;
    double y = fmod(p[5], two_pi);
    if (y < 0.0) y += two_pi;
    if (y >= two_pi) y = 0.0;
    p[5] = y;
    out->best_pose.x = p[0];
    out->best_pose.y = p[1];
    out->best_pose.z = p[2];
    out->best_pose.roll = p[3];
    out->best_pose.pitch = p[4];
    out->best_pose.yaw = p[5];
  } else {
    memset(&out->best_pose, 0, sizeof(out->best_pose));
  }
  st = BBS_OK;
done:
#undef EXCHANGE
  free(pending);
  free(h.a);
  free(g);
  return st;
}

int orc_search(const orc_map* m, const bbs_aabb* map_bbox, const double* scan, uint64_t k,
               const bbs_search_config* cfg, bbs_search_result* out) {
  return search_impl(m, map_bbox, scan, k, cfg, NULL, out);
}

int orc_search_sharded(const orc_map* m, const bbs_aabb* map_bbox, const double* scan,
                       uint64_t k, const bbs_search_config* cfg, const bbs_shard* shard,
                       bbs_search_result* out) {
  return search_impl(m, map_bbox, scan, k, cfg, shard, out);
}

/* oracle_search, oracle.hpp:29-95: enumerate the leaf grid under the root
 * index ranges times the level-0 rotation grid; no pruning. */
int orc_exhaustive(const orc_map* m, const bbs_aabb* map_bbox, const double* scan, uint64_t k,
                   const bbs_search_config* cfg, int32_t* best, uint64_t* n_argmax,
                   uint64_t* leaf_count) {
  if (k == 0) return BBS_ERR_DEGENERATE_SCAN;
  if (m->r != cfg->min_resolution) return BBS_ERR_CONFIG;
  const double d_max = cfg->has_d_max ? cfg->d_max : orc_max_range(scan, k);
  if (!(d_max > 0.0)) return BBS_ERR_DEGENERATE_SCAN;
  const int32_t L = cfg->max_level;
  bbs_axis_grid* g = (bbs_axis_grid*)malloc(sizeof(bbs_axis_grid) * 3 * (L + 1));
  int st = orc_angular_grid(cfg, d_max, g);
  if (st) {
    free(g);
    return st;
  }
  const bbs_aabb* tr = cfg->has_translation_range ? &cfg->translation_range : map_bbox;
  const double root_cell = ldexp(cfg->min_resolution, L);
  const int64_t scale = (int64_t)1 << L;
  const trange rx = trans_index_range(tr->min.x, tr->max.x, root_cell);
  const trange ry = trans_index_range(tr->min.y, tr->max.y, root_cell);
  const trange rz = trans_index_range(tr->min.z, tr->max.z, root_cell);
  const int64_t nr = max_index(axis_at(g, L, 0, 0)) + 1;
  const int64_t np = max_index(axis_at(g, L, 1, 0)) + 1;
  const int64_t nw = max_index(axis_at(g, L, 2, 0)) + 1;
  const uint64_t total = (uint64_t)((rx.max + 1) * scale - rx.min * scale) *
                         (uint64_t)((ry.max + 1) * scale - ry.min * scale) *
                         (uint64_t)((rz.max + 1) * scale - rz.min * scale) *
                         (uint64_t)(nr * np * nw);
  if (total == 0) {
    free(g);
    return BBS_ERR_EMPTY_SEARCH_SPACE;
  }
  if (total > 100000000ULL) {
    free(g);
    return BBS_ERR_TOO_LARGE;
  }
  int32_t b = -1;
  uint64_t cnt = 0;
  for (int64_t ix = rx.min * scale; ix < (rx.max + 1) * scale; ++ix)
    for (int64_t iy = ry.min * scale; iy < (ry.max + 1) * scale; ++iy)
      for (int64_t iz = rz.min * scale; iz < (rz.max + 1) * scale; ++iz)
        for (int64_t ir = 0; ir < nr; ++ir)
          for (int64_t ip = 0; ip < np; ++ip)
            for (int64_t iw = 0; iw < nw; ++iw) {
              bbs_node n = {(int32_t)ix, (int32_t)iy, (int32_t)iz, (int32_t)ir,
                            (int32_t)ip, (int32_t)iw, 0, -1};
              score_node(m, g, L, scan, k, &n);
              if (n.score > b) {
                b = n.score;
                cnt = 0;
              }
              if (n.score == b) cnt++;
            }
  *best = b;
  *n_argmax = cnt;
  *leaf_count = total;
  free(g);
  return BBS_OK;
}

// score.cu — K4: the candidate score kernels (batch_evaluate,
// search.hpp:23-34, over LevelMap::score, voxel_map.hpp:142-154).
//
// Exactness.  The reference computes, per (node, scan point),
//   q = ((r0*px + r1*py) + r2*pz) + t        (voxel_map.hpp:148-150)
//   v = (int32)floor(q / cell)                (point_cloud.hpp:39)
// with R from pose_to_transform (geometry.hpp:107-109) and t = cell*ix
// (nodes.hpp:35-37).  All products/sums here use __dmul_rn/__dadd_rn in that
// order (no FMA; the TU is also built with --fmad=false), cos/sin come from a
// host-libm LUT, and the division is IEEE (__ddiv_rn).
//
// Speed.  The rotated point rp = R*p depends only on (rotation, point), and
// the translation is added last, so all nodes that share a rotation share
// rp.  For such a group the kernel computes w = rp * (1/cell) once per point
// and takes floor(q / cell) = floor(w) + ix whenever frac(w) is farther than
// eps = 2^-48 * (|w| + max|ix| + 2) from an integer.  The reference's value
// differs from w + ix by at most ~4u(|w| + |ix|) (u = 2^-53; derivation in
// DESIGN.md §K4), so the integer shortcut is exact; points within eps of a
// voxel boundary ("ambiguous", ~1e-12 of them) take the exact per-node
// divide.  A lookup is then 3 integer adds plus one membership probe.
#include <cub/cub.cuh>

#include <algorithm>

#include "device_common.cuh"
#include "kernels.h"
#include "score_common.cuh"

namespace bbs {

namespace {

// ---- runs kernel ------------------------------------------------------------
// Per point of [p0, p1) (strided by the CTA): rotate once, probe the run's
// M translations, reduce the counts into s_cnt.
template <int M, int NT>
__device__ __forceinline__ void runs_points(const LevelView& L, const double R[9], double tmax,
                                            const ScanView& scan, const int32_t (*s_t)[3], int count,
                                            uint32_t p0, uint32_t p1, int lane, int32_t* s_cnt) {
  int32_t tx[M], ty[M], tz[M];
  int cnt[M];
#pragma unroll
  for (int j = 0; j < M; ++j) {
    tx[j] = s_t[j][0];
    ty[j] = s_t[j][1];
    tz[j] = s_t[j][2];
    cnt[j] = 0;
  }
  for (uint32_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
    const double px = scan.x[p], py = scan.y[p], pz = scan.z[p];
    const double rx = rot_row(R[0], R[1], R[2], px, py, pz);
    const double ry = rot_row(R[3], R[4], R[5], px, py, pz);
    const double rz = rot_row(R[6], R[7], R[8], px, py, pz);
    int32_t fx, fy, fz;
    const bool ok = fast_floor(rx, L.inv_cell, tmax, &fx) & fast_floor(ry, L.inv_cell, tmax, &fy) &
                    fast_floor(rz, L.inv_cell, tmax, &fz);
    if (ok) {
#pragma unroll
      for (int j = 0; j < M; ++j)
        if (j < count) cnt[j] += level_contains(L, fx + tx[j], fy + ty[j], fz + tz[j]) ? 1 : 0;
    } else {
#pragma unroll
      for (int j = 0; j < M; ++j)
        if (j < count) cnt[j] += exact_hit(L, rx, ry, rz, tx[j], ty[j], tz[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < M; ++j) {
    const int v = __reduce_add_sync(0xffffffffu, cnt[j]);
    if (lane == 0 && j < count && v) atomicAdd(&s_cnt[j], v);
  }
}

// One work item = (run of <= NT same-rotation nodes, tile of scan points).
// Each thread walks its points; per point the rotation work is shared by the
// run's NT translations.  Counts are reduced warp -> block -> global.
template <int NT>
__global__ void __launch_bounds__(256) score_runs_kernel(
    MapView map, GridView grid, ScanView scan, const bbs_node* __restrict__ nodes,
    const uint32_t* __restrict__ perm, const uint2* __restrict__ runs, uint32_t n_runs_param,
    const uint32_t* __restrict__ d_n, uint32_t n_nodes_param, uint32_t n_ptiles,
    int32_t* __restrict__ scores) {
  __shared__ int32_t s_t[NT][3];
  __shared__ uint32_t s_idx[NT];
  __shared__ double s_R[9];
  __shared__ int32_t s_cnt[NT];
  __shared__ int32_t s_level, s_count;
  __shared__ double s_tmax;

  const uint32_t n_nodes = d_n ? *d_n : n_nodes_param;
  const uint32_t n_runs = runs ? n_runs_param : (n_nodes + NT - 1) / NT;
  const uint64_t n_items = static_cast<uint64_t>(n_runs) * n_ptiles;
  const uint32_t k = scan.k;
  const uint32_t tile = (k + n_ptiles - 1) / n_ptiles;
  const int lane = threadIdx.x & 31;

  for (uint64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    const uint32_t r = static_cast<uint32_t>(item / n_ptiles);
    const uint32_t pt = static_cast<uint32_t>(item % n_ptiles);
    if (threadIdx.x < 32) {
      uint32_t first, count;
      if (runs) {
        const uint2 rr = runs[r];
        first = rr.x;
        count = rr.y;
      } else {
        first = r * NT;
        count = min(static_cast<uint32_t>(NT), n_nodes - first);
      }
      int32_t amax = 0;
      if (lane < static_cast<int>(count)) {
        const uint32_t idx = perm ? perm[first + lane] : first + lane;
        const int4 a = reinterpret_cast<const int4*>(nodes)[2 * idx];
        s_t[lane][0] = a.x;
        s_t[lane][1] = a.y;
        s_t[lane][2] = a.z;
        s_idx[lane] = idx;
        s_cnt[lane] = 0;
        amax = max(max(abs(a.x), abs(a.y)), abs(a.z));
        if (amax < 0) amax = INT32_MAX;  // abs(INT32_MIN)
      }
      amax = __reduce_max_sync(0xffffffffu, amax);
      if (lane == 0) {
        const uint32_t idx = perm ? perm[first] : first;
        const int4 a = reinterpret_cast<const int4*>(nodes)[2 * idx];
        const int4 b = reinterpret_cast<const int4*>(nodes)[2 * idx + 1];
        // a = (ix, iy, iz, iroll), b = (ipitch, iyaw, level, score)
        double R[9];
        rotation_of(grid, b.z, a.w, b.x, b.y, R);
#pragma unroll
        for (int i = 0; i < 9; ++i) s_R[i] = R[i];
        s_level = b.z;
        s_count = static_cast<int32_t>(count);
        s_tmax = static_cast<double>(amax) + 2.0;
      }
    }
    __syncthreads();
    const LevelView L = map.level[s_level];
    const int count = s_count;
    const double tmax = s_tmax;
    double R[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) R[i] = s_R[i];
    const uint32_t p0 = pt * tile;
    const uint32_t p1 = min(k, p0 + tile);
    // short runs (random candidates: ~3 per rotation) take a 4-wide body so
    // the predicated-off lanes of the NT-wide one cost no issue slots
    if (count <= 4)
      runs_points<4, NT>(L, R, tmax, scan, s_t, count, p0, p1, lane, s_cnt);
    else
      runs_points<NT, NT>(L, R, tmax, scan, s_t, count, p0, p1, lane, s_cnt);
    __syncthreads();
    if (threadIdx.x < static_cast<unsigned>(count)) {
      if (n_ptiles == 1)
        scores[s_idx[threadIdx.x]] = s_cnt[threadIdx.x];
      else if (s_cnt[threadIdx.x])
        atomicAdd(&scores[s_idx[threadIdx.x]], s_cnt[threadIdx.x]);
    }
    __syncthreads();
  }
}

// ---- root box kernel --------------------------------------------------------
// One CTA = (root rotation, chunk of that rotation's owned translations).
// The scan is processed in chunks of kChunk points: each chunk's fast-path
// voxel offsets f are de-duplicated in a shared-memory hash (coarse root
// levels put hundreds of points in one voxel), and every owned translation t
// accumulates sum_f count(f) * contains(f + t).  Ambiguous points are kept
// as a list and scored exactly per translation.
constexpr int kChunk = 2048;
constexpr int kHashSlots = 4096;
constexpr unsigned long long kSlotEmpty = ~0ull;

__device__ __forceinline__ uint32_t slot_hash(unsigned long long key) {
  return static_cast<uint32_t>((key * 0x9E3779B97F4A7C15ull) >> 52);  // 12 bits
}

__global__ void __launch_bounds__(kBoxThreads, 2) score_box_kernel(MapView map, GridView grid,
                                                                   ScanView scan, BoxParams bp,
                                                                   uint32_t rot_begin, uint32_t rot_end,
                                                                   const int32_t* __restrict__ only,
                                                                   int32_t* __restrict__ scores,
                                                                   unsigned long long* probes) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned long long* s_key = reinterpret_cast<unsigned long long*>(smem);        // 32 KB
  int32_t* s_hcnt = reinterpret_cast<int32_t*>(s_key + kHashSlots);               // 16 KB
  int4* s_ent = reinterpret_cast<int4*>(s_hcnt + kHashSlots);                      // 32 KB
  uint32_t* s_amb = reinterpret_cast<uint32_t*>(s_ent + kChunk);                   // 8 KB
  __shared__ int32_t s_nent, s_namb;

  const uint32_t nrot = bp.nr * bp.np * bp.nw;
  const uint64_t slab = static_cast<uint64_t>(bp.ny) * bp.nz;  // translations per x-slab
  const uint64_t n_items = static_cast<uint64_t>(rot_end - rot_begin) * bp.n_tchunks;
  const LevelView L = map.level[bp.level];
  if (only && only[kRotBatch] == 0) return;  // no histogram overflowed in this batch

  for (uint64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    const uint32_t rot = rot_begin + static_cast<uint32_t>(item / bp.n_tchunks);
    const uint32_t tc = static_cast<uint32_t>(item % bp.n_tchunks);
    if (only && !only[rot - rot_begin]) continue;  // uniform across the CTA
    uint32_t P, x0r;
    if (!owned_slabs(bp, nrot, rot, &P, &x0r)) continue;
    const uint64_t n_own = (x0r < bp.nx ? (bp.nx - x0r + P - 1) / P : 0) * slab;
    const uint64_t own0 = static_cast<uint64_t>(tc) * kBoxTransPerCta;
    if (own0 >= n_own) continue;

    const uint32_t ir = rot / (bp.np * bp.nw);
    const uint32_t ip = (rot / bp.nw) % bp.np;
    const uint32_t iw = rot % bp.nw;
    double R[9];
    rotation_of(grid, bp.level, static_cast<int>(ir), static_cast<int>(ip), static_cast<int>(iw), R);

    // this thread's translations
    int32_t tix[kBoxTransPerThread], tiy[kBoxTransPerThread], tiz[kBoxTransPerThread];
    uint64_t tref[kBoxTransPerThread];
    bool tvalid[kBoxTransPerThread];
    int acc[kBoxTransPerThread];
#pragma unroll
    for (int i = 0; i < kBoxTransPerThread; ++i) {
      const uint64_t o = own0 + threadIdx.x + static_cast<uint64_t>(i) * kBoxThreads;
      tvalid[i] = o < n_own;
      const uint64_t t = tvalid[i] ? (x0r + (o / slab) * P) * slab + o % slab : 0;
      tiz[i] = bp.z0 + static_cast<int32_t>(t % bp.nz);
      tiy[i] = bp.y0 + static_cast<int32_t>((t / bp.nz) % bp.ny);
      tix[i] = bp.x0 + static_cast<int32_t>(t / (static_cast<uint64_t>(bp.nz) * bp.ny));
      tref[i] = t * nrot + rot;
      acc[i] = 0;
    }

    for (uint32_t c0 = 0; c0 < scan.k; c0 += kChunk) {
      for (int i = threadIdx.x; i < kHashSlots; i += blockDim.x) {
        s_key[i] = kSlotEmpty;
        s_hcnt[i] = 0;
      }
      if (threadIdx.x == 0) {
        s_nent = 0;
        s_namb = 0;
      }
      __syncthreads();
      const uint32_t c1 = min(scan.k, c0 + kChunk);
      for (uint32_t p = c0 + threadIdx.x; p < c1; p += blockDim.x) {
        const double px = scan.x[p], py = scan.y[p], pz = scan.z[p];
        int32_t fx, fy, fz;
        const bool ok = fast_floor(rot_row(R[0], R[1], R[2], px, py, pz), L.inv_cell, bp.tmax, &fx) &
                        fast_floor(rot_row(R[3], R[4], R[5], px, py, pz), L.inv_cell, bp.tmax, &fy) &
                        fast_floor(rot_row(R[6], R[7], R[8], px, py, pz), L.inv_cell, bp.tmax, &fz);
        if (!ok) {
          s_amb[atomicAdd(&s_namb, 1)] = p;
          continue;
        }
        // |f| < 2^30 on the fast path: 21-bit fields hold f + 2^20 only when
        // |f| < 2^20; larger offsets are scored exactly instead.
        if (fx <= -(1 << 20) || fx >= (1 << 20) || fy <= -(1 << 20) || fy >= (1 << 20) ||
            fz <= -(1 << 20) || fz >= (1 << 20)) {
          s_amb[atomicAdd(&s_namb, 1)] = p;
          continue;
        }
        const unsigned long long key =
            (static_cast<unsigned long long>(fx + (1 << 20)) << 42) |
            (static_cast<unsigned long long>(fy + (1 << 20)) << 21) |
            static_cast<unsigned long long>(fz + (1 << 20));
        uint32_t h = slot_hash(key);
        for (;;) {
          const unsigned long long prev = atomicCAS(&s_key[h], kSlotEmpty, key);
          if (prev == kSlotEmpty || prev == key) {
            atomicAdd(&s_hcnt[h], 1);
            break;
          }
          h = (h + 1) & (kHashSlots - 1);
        }
      }
      __syncthreads();
      for (int i = threadIdx.x; i < kHashSlots; i += blockDim.x) {
        const unsigned long long key = s_key[i];
        if (key != kSlotEmpty) {
          const int e = atomicAdd(&s_nent, 1);
          s_ent[e] = make_int4(static_cast<int32_t>((key >> 42) & 0x1FFFFF) - (1 << 20),
                               static_cast<int32_t>((key >> 21) & 0x1FFFFF) - (1 << 20),
                               static_cast<int32_t>(key & 0x1FFFFF) - (1 << 20), s_hcnt[i]);
        }
      }
      __syncthreads();
      const int nent = s_nent;
      if (threadIdx.x == 0 && probes) {
        const uint64_t nt = min(static_cast<uint64_t>(kBoxTransPerCta), n_own - own0);
        atomicAdd(probes, static_cast<unsigned long long>(nent + s_namb) * nt);
      }
      for (int e = 0; e < nent; ++e) {
        const int4 f = s_ent[e];
#pragma unroll
        for (int i = 0; i < kBoxTransPerThread; ++i)
          acc[i] += level_contains(L, f.x + tix[i], f.y + tiy[i], f.z + tiz[i]) ? f.w : 0;
      }
      const int namb = s_namb;
      for (int a = 0; a < namb; ++a) {
        const uint32_t p = s_amb[a];
        const double px = scan.x[p], py = scan.y[p], pz = scan.z[p];
        const double rx = rot_row(R[0], R[1], R[2], px, py, pz);
        const double ry = rot_row(R[3], R[4], R[5], px, py, pz);
        const double rz = rot_row(R[6], R[7], R[8], px, py, pz);
#pragma unroll
        for (int i = 0; i < kBoxTransPerThread; ++i)
          acc[i] += exact_hit(L, rx, ry, rz, tix[i], tiy[i], tiz[i]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < kBoxTransPerThread; ++i)
      if (tvalid[i]) scores[tref[i]] = acc[i];
  }
}

// ---- epoch flush: 2x2x2 translation cubes -----------------------------------
// pending holds the children of branch() (nodes.hpp:103-116): every 8
// consecutive nodes share a rotation and have translations 2c + j,
// j = (t >> 2, (t >> 1) & 1, t & 1) for t = 0..7.  Per scan point the 8
// probes form a 2x2x2 voxel cube = 4 (x, y) columns x 2 z-bits of the
// z-column bitmap: 4 word loads answer all 8 children.  One work item =
// (run, tile of scan points); counts reduce warp -> CTA -> scores.
template <bool kILP>
__device__ __forceinline__ void score_cube8_kernel_body(const MapView& map,
                                                        const GridView& grid,
                                                        ScanView scan,
                                                        const bbs_node* __restrict__ nodes,
                                                        const uint32_t* __restrict__ d_n,
                                                        uint32_t n_ptiles,
                                                        int32_t* __restrict__ scores,
                                                        const RotCache& cache,
                                                        int use_cache) {
  pdl_wait();

  __shared__ double s_R[9];
  __shared__ int32_t s_hdr[4];
  __shared__ int32_t s_cnt[8];
  const uint32_t k = scan.k;
  uint32_t n_runs = *d_n / 8;
  const uint32_t* list = nullptr;
  if (use_cache) {
    // only the runs the probe kernel listed (no READY histogram); the point
    // tiling is chosen here, for the actual number of runs
    n_runs = cache.ctl[3];
    if (n_runs == 0) return;
    list = cache.fb_runs;
    const uint32_t pmax = max(1u, (k + 1023u) / 1024u);
    n_ptiles = min(pmax, max(1u, (2u * gridDim.x + n_runs - 1) / n_runs));
  }
  const uint64_t n_items = static_cast<uint64_t>(n_runs) * n_ptiles;
  for (uint64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    const uint32_t run = list ? list[item / n_ptiles] : static_cast<uint32_t>(item / n_ptiles);
    const uint32_t pt = static_cast<uint32_t>(item % n_ptiles);
    cube8_item<kILP>(map, grid, scan, nodes, run, pt, n_ptiles, scores, s_R, s_hdr, s_cnt);
  }
}

template <bool kILP>
#ifndef BBS_CUBE_MINB
#define BBS_CUBE_MINB 4
#endif
__global__ void __launch_bounds__(256, BBS_CUBE_MINB) score_cube8_kernel(MapView map, GridView grid, ScanView scan,
                                                             const bbs_node* __restrict__ nodes,
                                                             const uint32_t* __restrict__ d_n,
                                                             uint32_t n_ptiles,
                                                             int32_t* __restrict__ scores,
                                                             RotCache cache, int use_cache) {
  score_cube8_kernel_body<kILP>(map, grid, scan, nodes, d_n, n_ptiles, scores, cache, use_cache);
}

// ---- root batch: whole-scan histogram + z-column kernel ---------------------
// (1) root_hist_kernel: one CTA per root rotation de-duplicates the fast-path
//     voxel offsets f of ALL K scan points in a shared-memory hash
//     (coarse root levels put tens of points in one voxel) and writes the
//     (f, count) list, the ambiguous points and an overflow flag.
// (2) root_col_kernel: one thread per owned (ix, iy) translation column holds
//     the column's nz <= 32 z-translations in registers; per histogram entry
//     it reads ONE 32-bit z-mask of the level's column bitmap and credits
//     count(f) to every z-translation whose bit is set:
//        score(ix, iy, z0 + j) = sum_f count(f) * bit_{fz + z0 + j}(col(fx + ix, fy + iy)).
//     Ambiguous points are scored exactly per translation.
constexpr int kHistSlots = 2 * kHistCap;
constexpr int kColGroupCap = kHistCap / 2;  // groups of 4 (2 int4 each) per rotation
constexpr int kColPadMax = 160 << 10;       // padded column window, bytes of shared memory
constexpr int kEntTile = 1024;

__device__ __forceinline__ uint32_t hist_slot(unsigned long long key) {
  return static_cast<uint32_t>((key * 0x9E3779B97F4A7C15ull) >> 51);  // 13 bits
}

// Entries are emitted heaviest first by count bucket (2 buckets: counts >= 2
// first; more buckets cost emission passes and did not pay off on C2/C3).
#ifndef BBS_ROOT_BUCKETS
#define BBS_ROOT_BUCKETS 2
#endif
constexpr int kRootCountBuckets = BBS_ROOT_BUCKETS;
__device__ __forceinline__ int count_bucket(uint32_t v) {
  return kRootCountBuckets == 1 ? 0 : min(kRootCountBuckets - 1, 31 - __clz(max(v, 1u)));
}

constexpr int kRootListCap = 4096;  // dense root box: touched cells listed (beyond: the box is walked)

// One histogram entry (f, cnt) of root_hist_kernel, appended warp-cooperatively
// (every lane calls; has = false for lanes without an entry).  Staged mode
// (root_colpad_kernel): (padded column byte offset << 8 | z shift + 8) words
// in groups of 4 with their counts packed as bytes (counts > 255 split),
// dropping entries whose z never meets a translation's column; otherwise plain
// (fx, fy, fz, count).
__device__ __forceinline__ void root_emit(bool has, int32_t fx, int32_t fy, int32_t fz, int32_t cnt,
                                          const BoxParams& bp, const RootStage& st, int4* ent4,
                                          int* s_nent, int* s_badpad, int* s_total) {
  const int lane = threadIdx.x & 31;
  int parts = has ? 1 : 0;
  int32_t sh = 0;
  if (has && st.enabled) {
    if (abs(fx) > bp.fpad || abs(fy) > bp.fpad) *s_badpad = 1;
    sh = fz + st.zoff;
    parts = (sh < static_cast<int32_t>(st.dimz) && sh > -static_cast<int32_t>(bp.nz)) ? (cnt + 254) / 255 : 0;
  }
  int incl = parts;  // warp inclusive scan of the parts
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += v;
  }
  const int wtot = __shfl_sync(0xffffffffu, incl, 31);
  const int wcnt = __reduce_add_sync(0xffffffffu, parts ? cnt : 0);  // counts the entries carry
  int at = 0;
  if (lane == 0 && wtot) at = atomicAdd(s_nent, wtot);
  if (lane == 0 && wcnt) atomicAdd(s_total, wcnt);
  at = __shfl_sync(0xffffffffu, at, 0) + incl - parts;
  if (!parts) return;
  if (st.enabled) {
    const uint32_t word = (static_cast<uint32_t>(4 * (fy * static_cast<int32_t>(st.pitch) + fx)) << 8) |
                          static_cast<uint32_t>(sh + 8);
    int32_t* g = reinterpret_cast<int32_t*>(ent4);
    unsigned char* wb = reinterpret_cast<unsigned char*>(ent4);
    for (int q = 0; q < parts; ++q) {
      const int e = at + q;
      if (e >= 4 * kColGroupCap) break;
      g[(e >> 2) * 8 + (e & 3)] = static_cast<int32_t>(word);
      wb[((e >> 2) * 8 + 4) * 4 + (e & 3)] = static_cast<unsigned char>(min(255, cnt - 255 * q));
    }
  } else if (at < kHistCap) {  // more is an overflow (the rotation falls back)
    ent4[at] = make_int4(fx, fy, fz, cnt);
  }
}

__global__ void __launch_bounds__(512) root_hist_kernel(GridView grid, ScanView scan, BoxParams bp,
                                                        LevelView L, uint32_t rot_begin,
                                                        uint32_t rot_end, RootHist h, RootStage st,
                                                        int32_t* __restrict__ n_overflow) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned long long* s_key = reinterpret_cast<unsigned long long*>(smem);  // 64 KB
  int32_t* s_cnt = reinterpret_cast<int32_t*>(s_key + kHistSlots);          // 32 KB
  uint32_t* s_w = reinterpret_cast<uint32_t*>(smem);  // dense box: 16-bit counters (overlays the hash)
  __shared__ int s_distinct, s_namb, s_nent, s_skip, s_badpad, s_total, s_nl;
  __shared__ typename cub::BlockScan<int, 512>::TempStorage s_rscan;
  const uint32_t nrot = bp.nr * bp.np * bp.nw;
  const int lane = threadIdx.x & 31;
  // dense box (coarse root levels): direct-mapped counters, no probing
  const int dr = bp.dn_r, dxy = 2 * dr + 1, dzlo = bp.dn_zlo;
  const bool dense = dr > 0;
  const int ncells = dense ? dxy * dxy * bp.dn_nz : 0;
  // touched dense cells, listed after the counters in the hash region
  uint16_t* s_list = reinterpret_cast<uint16_t*>(s_w + ((ncells + 1) >> 1));
  const int list_cap = min(kRootListCap, (kHistSlots * 12 - ((ncells + 1) >> 1) * 4) / 2);
  for (uint32_t rot = rot_begin + blockIdx.x; rot < rot_end; rot += gridDim.x) {
    const uint32_t slot = rot - rot_begin;
    uint32_t P, x0r;
    if (!owned_slabs(bp, nrot, rot, &P, &x0r)) {
      if (threadIdx.x == 0) {
        h.n_ent[slot] = 0;
        h.n_amb[slot] = 0;
        h.overflow[slot] = 0;
      }
      continue;
    }
    if (dense) {
      for (int i = threadIdx.x; i < (ncells + 1) >> 1; i += blockDim.x) s_w[i] = 0u;
    } else {
      for (int i = threadIdx.x; i < kHistSlots; i += blockDim.x) {
        s_key[i] = kSlotEmpty;
        s_cnt[i] = 0;
      }
    }
    if (threadIdx.x == 0) {
      s_distinct = 0;
      s_namb = 0;
      s_nent = 0;
      s_skip = 0;
      s_badpad = 0;
      s_total = 0;
      s_nl = 0;
    }
    __syncthreads();
    const uint32_t ir = rot / (bp.np * bp.nw), ip = (rot / bp.nw) % bp.np, iw = rot % bp.nw;
    double R[9];
    rotation_of(grid, bp.level, static_cast<int>(ir), static_cast<int>(ip), static_cast<int>(iw), R);
    if (dense) {
      // constant eps (bounds every in-box point's fast_floor eps; an
      // out-of-box point sends the rotation to the chunked kernel)
      const double eps = bp.dn_eps, eps1 = bp.dn_eps1, inv = L.inv_cell;
      const uint32_t udxy = static_cast<uint32_t>(dxy), unz = static_cast<uint32_t>(bp.dn_nz);
      // two points per thread per step: two load / rotate chains in flight
      for (uint32_t p0 = 0; p0 < scan.k; p0 += 2 * blockDim.x) {
        double px[2], py[2], pz[2];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const uint32_t p = p0 + hh * blockDim.x + threadIdx.x;
          const bool live = p < scan.k;
          px[hh] = live ? scan.x[p] : 0.0;
          py[hh] = live ? scan.y[p] : 0.0;
          pz[hh] = live ? scan.z[p] : 0.0;
        }
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const uint32_t p = p0 + hh * blockDim.x + threadIdx.x;
          int idx = -1;
          if (p < scan.k) {
            const double wx = __dmul_rn(rot_row(R[0], R[1], R[2], px[hh], py[hh], pz[hh]), inv);
            const double wy = __dmul_rn(rot_row(R[3], R[4], R[5], px[hh], py[hh], pz[hh]), inv);
            const double wz = __dmul_rn(rot_row(R[6], R[7], R[8], px[hh], py[hh], pz[hh]), inv);
            const double flx = floor(wx), fly = floor(wy), flz = floor(wz);
            const double frx = __dsub_rn(wx, flx), fry = __dsub_rn(wy, fly), frz = __dsub_rn(wz, flz);
            if (frx > eps && frx < eps1 && fry > eps && fry < eps1 && frz > eps && frz < eps1) {
              const uint32_t ux = static_cast<uint32_t>(__double2int_rz(flx)) + static_cast<uint32_t>(dr);
              const uint32_t uy = static_cast<uint32_t>(__double2int_rz(fly)) + static_cast<uint32_t>(dr);
              const uint32_t uz = static_cast<uint32_t>(__double2int_rz(flz)) - static_cast<uint32_t>(dzlo);
              if (ux < udxy && uy < udxy && uz < unz)
                idx = static_cast<int>((uz * udxy + uy) * udxy + ux);
              else
                s_skip = 1;
            } else {
              const int a = atomicAdd(&s_namb, 1);
              if (a < kAmbCap) h.amb[static_cast<uint64_t>(slot) * kAmbCap + a] = p;
            }
          }
          // one shared atomic per point (cheaper than MATCH.ANY aggregation);
          // a cell's first count lists it (emission walks the list, not the box)
          if (idx >= 0) {
            const uint32_t sh = static_cast<uint32_t>(idx & 1) << 4;
            const uint32_t old = atomicAdd(&s_w[idx >> 1], 1u << sh);
            if (((old >> sh) & 0xFFFFu) == 0u) {
              const int pos = atomicAdd(&s_nl, 1);
              if (pos < list_cap) s_list[pos] = static_cast<uint16_t>(idx);
            }
          }
        }
      }
    } else {
      for (uint32_t p0 = 0; p0 < scan.k; p0 += blockDim.x) {
        const uint32_t p = p0 + threadIdx.x;
        const bool live = p < scan.k;
        bool ok = false;
        int32_t fx = 0, fy = 0, fz = 0;
        if (live) {
          const double px = scan.x[p], py = scan.y[p], pz = scan.z[p];
          ok = fast_floor(rot_row(R[0], R[1], R[2], px, py, pz), L.inv_cell, bp.tmax, &fx) &
               fast_floor(rot_row(R[3], R[4], R[5], px, py, pz), L.inv_cell, bp.tmax, &fy) &
               fast_floor(rot_row(R[6], R[7], R[8], px, py, pz), L.inv_cell, bp.tmax, &fz);
          ok = ok && fx > -(1 << 20) && fx < (1 << 20) && fy > -(1 << 20) && fy < (1 << 20) &&
               fz > -(1 << 20) && fz < (1 << 20);
          if (!ok) {
            const int a = atomicAdd(&s_namb, 1);
            if (a < kAmbCap) h.amb[static_cast<uint64_t>(slot) * kAmbCap + a] = p;
          }
        }
        const bool ins = live && ok && s_distinct < kHistCap;
        if (live && ok && !ins) s_skip = 1;  // table saturated: this rotation falls back
        const unsigned long long key = ins ? (static_cast<unsigned long long>(fx + (1 << 20)) << 42) |
                                                 (static_cast<unsigned long long>(fy + (1 << 20)) << 21) |
                                                 static_cast<unsigned long long>(fz + (1 << 20))
                                           : kSlotEmpty;
        // neighbouring scan points often share a voxel: one insert per distinct key per warp
        const unsigned same = __match_any_sync(0xffffffffu, key);
        if (ins && (__ffs(same) - 1) == lane) {
          const int mult = __popc(same);
          uint32_t hs = hist_slot(key);
          for (;;) {
            const unsigned long long prev = atomicCAS(&s_key[hs], kSlotEmpty, key);
            if (prev == kSlotEmpty) atomicAdd(&s_distinct, 1);
            if (prev == kSlotEmpty || prev == key) {
              atomicAdd(&s_cnt[hs], mult);
              break;
            }
            hs = (hs + 1) & (kHistSlots - 1);
          }
        }
      }
    }
    __syncthreads();
    bool over = s_skip || s_distinct > kHistCap || s_namb > kAmbCap;
    if (!over) {
      int4* ent4 = h.entries + static_cast<uint64_t>(slot) * kHistCap;
      const int nl = s_nl;
      if (dense && nl <= list_cap) {
        // the touched cells, heaviest counts first (log2 buckets) so the
        // column kernel's survivor bound tightens early; the warp emits in
        // lockstep
        for (int bk = kRootCountBuckets - 1; bk >= 0; --bk)
          for (int j0 = 0; j0 < nl; j0 += static_cast<int>(blockDim.x)) {
            const int j = j0 + static_cast<int>(threadIdx.x);
            const int i = j < nl ? s_list[j] : 0;
            const uint32_t v = j < nl ? (s_w[i >> 1] >> ((i & 1) << 4)) & 0xFFFFu : 0u;
            root_emit(v != 0u && count_bucket(v) == bk, i % dxy - dr, (i / dxy) % dxy - dr, i / (dxy * dxy) + dzlo,
                      static_cast<int32_t>(v), bp, st, ent4, &s_nent, &s_badpad, &s_total);
          }
      } else if (dense) {
        // each thread walks a contiguous cell range; the warp emits in
        // lockstep, heaviest counts first (log2 buckets) so the column
        // kernel's survivor bound tightens early
        const int dper = (ncells + static_cast<int>(blockDim.x) - 1) / static_cast<int>(blockDim.x);
        const int dc0 = min(ncells, static_cast<int>(threadIdx.x) * dper), dc1 = min(ncells, dc0 + dper);
        for (int bk = kRootCountBuckets - 1; bk >= 0; --bk) {
          int cx = dc0 % dxy, cy = dc0 / dxy % dxy, cz = dc0 / (dxy * dxy);
          for (int step = 0; step < dper; ++step) {
            const int i = dc0 + step;
            const uint32_t v = i < dc1 ? (s_w[i >> 1] >> ((i & 1) << 4)) & 0xFFFFu : 0u;
            root_emit(v != 0u && count_bucket(v) == bk, cx - dr, cy - dr, cz + dzlo, static_cast<int32_t>(v), bp,
                      st, ent4, &s_nent, &s_badpad, &s_total);
            if (++cx == dxy) {
              cx = 0;
              if (++cy == dxy) {
                cy = 0;
                ++cz;
              }
            }
          }
        }
      } else {
        for (int bk = kRootCountBuckets - 1; bk >= 0; --bk)
          for (int i0 = 0; i0 < kHistSlots; i0 += blockDim.x) {
            const int i = i0 + threadIdx.x;
            const unsigned long long key = s_key[i];
            const bool has = key != kSlotEmpty && count_bucket(static_cast<uint32_t>(s_cnt[i])) == bk;
            root_emit(has, has ? static_cast<int32_t>((key >> 42) & 0x1FFFFF) - (1 << 20) : 0,
                      has ? static_cast<int32_t>((key >> 21) & 0x1FFFFF) - (1 << 20) : 0,
                      has ? static_cast<int32_t>(key & 0x1FFFFF) - (1 << 20) : 0, has ? s_cnt[i] : 0, bp, st,
                      ent4, &s_nent, &s_badpad, &s_total);
          }
      }
    }
    __syncthreads();
    // an offset beyond the padding or too many split entries: chunked fallback
    over = over || s_badpad || (st.enabled && s_nent > 4 * kColGroupCap) || (!st.enabled && s_nent > kHistCap);
    if (!over && st.enabled && (s_nent & 3)) {
      // zero-weight padding of the last group
      const int e = s_nent + static_cast<int>(threadIdx.x);
      if (e < ((s_nent + 3) & ~3)) {
        int32_t* g = reinterpret_cast<int32_t*>(h.entries + static_cast<uint64_t>(slot) * kHistCap);
        g[(e >> 2) * 8 + (e & 3)] = 8;  // offset 0, shift 8
        reinterpret_cast<unsigned char*>(g)[((e >> 2) * 8 + 4) * 4 + (e & 3)] = 0;
      }
    }
    if (!over && st.enabled) {
      // counts still to come from each group on (suffix sums, in the .y of
      // the group's count word): the column kernel's survivor bound reads
      // them instead of subtracting every group's counts as it goes
      __syncthreads();  // the padding group is complete
      constexpr int kPer = (kColGroupCap + 511) / 512;
      const int n_grp = (s_nent + 3) >> 2;
      int32_t* g = reinterpret_cast<int32_t*>(h.entries + static_cast<uint64_t>(slot) * kHistCap);
      // thread t holds groups n_grp - 1 - (t * kPer + k): a forward scan over
      // the reversed order is the suffix sum
      int v[kPer], sum = 0;
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const int r = static_cast<int>(threadIdx.x) * kPer + k;
        const int i = n_grp - 1 - r;
        v[k] = i >= 0 ? static_cast<int>(__dp4a(static_cast<uint32_t>(g[i * 8 + 4]), 0x01010101u, 0u)) : 0;
        sum += v[k];
      }
      int excl;
      cub::BlockScan<int, 512>(s_rscan).ExclusiveSum(sum, excl);
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const int r = static_cast<int>(threadIdx.x) * kPer + k;
        const int i = n_grp - 1 - r;
        excl += v[k];
        if (i >= 0) g[i * 8 + 5] = excl;
      }
    }
    if (threadIdx.x == 0) {
      h.n_ent[slot] = over ? 0 : s_nent;
      h.n_amb[slot] = over ? 0 : s_namb;
      h.total[slot] = over ? 0 : s_total;
      h.overflow[slot] = over ? 1 : 0;
      if (over) atomicAdd(n_overflow, 1);
    }
    __syncthreads();
  }
}

template <int NZ>
__global__ void __launch_bounds__(256) root_col_kernel(GridView grid, ScanView scan, BoxParams bp,
                                                       LevelView L, uint32_t rot_begin,
                                                       uint32_t rot_end, RootHist h,
                                                       uint32_t n_cchunks, int stage_col,
                                                       int32_t* __restrict__ scores,
                                                       unsigned long long* probes) {
  extern __shared__ __align__(16) unsigned char smem[];
  int4* s_ent = reinterpret_cast<int4*>(smem);                          // 16 KB
  uint32_t* s_col = reinterpret_cast<uint32_t*>(s_ent + kEntTile);      // staged colmap
  const uint32_t nrot = bp.nr * bp.np * bp.nw;
  const uint32_t dimx = L.dim[0], dimy = L.dim[1];
  const uint32_t* __restrict__ col = L.words;  // nwz == 1: one word per (x, y) column
  if (stage_col) {
    for (uint32_t i = threadIdx.x; i < dimx * dimy; i += blockDim.x) s_col[i] = __ldg(&L.words[i]);
    __syncthreads();
    col = s_col;
  }
  const uint64_t n_items = static_cast<uint64_t>(rot_end - rot_begin) * n_cchunks;
  for (uint64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    const uint32_t slot = static_cast<uint32_t>(item / n_cchunks);
    const uint32_t rot = rot_begin + slot;
    const uint32_t cc = static_cast<uint32_t>(item % n_cchunks);
    if (h.overflow[slot]) continue;  // uniform per CTA
    uint32_t P, x0r;
    if (!owned_slabs(bp, nrot, rot, &P, &x0r)) continue;
    const uint32_t n_own_x = x0r < bp.nx ? (bp.nx - x0r + P - 1) / P : 0;
    const uint64_t ncols = static_cast<uint64_t>(n_own_x) * bp.ny;
    const uint64_t col0 = static_cast<uint64_t>(cc) * blockDim.x;
    if (col0 >= ncols) continue;
    const uint64_t c = col0 + threadIdx.x;
    const bool valid = c < ncols;
    const uint32_t ix_rel = x0r + static_cast<uint32_t>(c / bp.ny) * P;
    const uint32_t iy_rel = static_cast<uint32_t>(c % bp.ny);
    const int32_t ix = bp.x0 + static_cast<int32_t>(ix_rel), iy = bp.y0 + static_cast<int32_t>(iy_rel);
    const uint32_t xoff = static_cast<uint32_t>(ix) - static_cast<uint32_t>(L.box_min[0]);
    const uint32_t yoff = static_cast<uint32_t>(iy) - static_cast<uint32_t>(L.box_min[1]);
    const int32_t zoff = bp.z0 - L.box_min[2];
    int acc[NZ];
#pragma unroll
    for (int j = 0; j < NZ; ++j) acc[j] = 0;
    const int n_ent = h.n_ent[slot];
    const int4* __restrict__ ent = h.entries + static_cast<uint64_t>(slot) * kHistCap;
    for (int t0 = 0; t0 < n_ent; t0 += kEntTile) {
      const int tn = min(kEntTile, n_ent - t0);
      __syncthreads();
      for (int i = threadIdx.x; i < tn; i += blockDim.x) s_ent[i] = ent[t0 + i];
      __syncthreads();
      if (valid) {
#pragma unroll 4
        for (int e = 0; e < tn; ++e) {
          const int4 f = s_ent[e];
          const uint32_t ux = static_cast<uint32_t>(f.x) + xoff;
          const uint32_t uy = static_cast<uint32_t>(f.y) + yoff;
          if (ux < dimx && uy < dimy) {
            const uint32_t m = col[uy * dimx + ux];
            const int32_t sh = f.z + zoff;
            const uint32_t bits = sh >= 0 ? (sh < 32 ? m >> sh : 0u) : (sh > -32 ? m << -sh : 0u);
#pragma unroll
            for (int j = 0; j < NZ; ++j) acc[j] += f.w & -static_cast<int>((bits >> j) & 1u);
          }
        }
      }
    }
    const int n_amb = h.n_amb[slot];
    if (valid && n_amb) {
      const uint32_t ir = rot / (bp.np * bp.nw), ip = (rot / bp.nw) % bp.np, iw = rot % bp.nw;
      double R[9];
      rotation_of(grid, bp.level, static_cast<int>(ir), static_cast<int>(ip), static_cast<int>(iw), R);
      for (int a = 0; a < n_amb; ++a) {
        const uint32_t p = h.amb[static_cast<uint64_t>(slot) * kAmbCap + a];
        const double px = scan.x[p], py = scan.y[p], pz = scan.z[p];
        const double rx = rot_row(R[0], R[1], R[2], px, py, pz);
        const double ry = rot_row(R[3], R[4], R[5], px, py, pz);
        const double rz = rot_row(R[6], R[7], R[8], px, py, pz);
#pragma unroll
        for (int j = 0; j < NZ; ++j)
          if (j < static_cast<int>(bp.nz)) acc[j] += exact_hit(L, rx, ry, rz, ix, iy, bp.z0 + j);
      }
    }
    if (valid) {
      const uint64_t base = (static_cast<uint64_t>(ix_rel) * bp.ny + iy_rel) * bp.nz;
#pragma unroll
      for (int j = 0; j < NZ; ++j)
        if (j < static_cast<int>(bp.nz)) scores[(base + j) * nrot + rot] = acc[j];
    }
    if (threadIdx.x == 0 && probes) {
      const uint64_t nc = min(static_cast<uint64_t>(blockDim.x), ncols - col0);
      atomicAdd(probes, static_cast<unsigned long long>(nc) * (n_ent + n_amb) * bp.nz);
    }
  }
}

// Staged variant: the level's z-column words sit zero-padded (and shifted
// up by 8 bits) in shared memory; entries come in groups of 4 as
// (padded column offset << 8 | z shift + 8) words plus their counts packed as
// bytes.  Per group: 4 LDS + 4 funnel shifts give each entry's z-translation
// bits, 3 PRMT pack their low bytes, and per z-translation j one LOP3 keeps
// bit j of every byte and one IDP4A adds 2^j * sum(count) of the hits.
constexpr int kGrpTile = 1024;  // groups per shared-memory tile (16 KB + 4 KB + 0.5 KB)
constexpr int kColPadHead = kGrpTile * 20 + kGrpTile / 2;  // shared memory before the window
#ifndef BBS_COLPAD_MINB
#define BBS_COLPAD_MINB 3  // <= 80 registers, no spills: 3 CTAs per SM (C2 root batch -13 us; 4 spills)
#endif
template <int NZ>
__global__ void __launch_bounds__(256, BBS_COLPAD_MINB) root_colpad_kernel(GridView grid, ScanView scan, BoxParams bp,
                                                          LevelView L, uint32_t rot_begin,
                                                          uint32_t rot_end, RootHist h, RootStage st,
                                                          uint32_t n_cchunks,
                                                          int32_t* __restrict__ scores,
                                                          unsigned long long* probes) {
  extern __shared__ __align__(16) unsigned char smem[];
  int4* s_go = reinterpret_cast<int4*>(smem);                     // group offsets/shifts
  uint32_t* s_gw = reinterpret_cast<uint32_t*>(s_go + kGrpTile);  // group counts (bytes)
  int32_t* s_rem = reinterpret_cast<int32_t*>(s_gw + kGrpTile);   // counts still to come, every 8th group
  uint32_t* s_col = reinterpret_cast<uint32_t*>(s_rem + kGrpTile / 8);
  const uint32_t nrot = bp.nr * bp.np * bp.nw;
  const uint32_t dimx = L.dim[0], dimy = L.dim[1];
  for (uint32_t i = threadIdx.x; i < st.pitch * st.rows; i += blockDim.x) {
    const int32_t x = st.sx0 + static_cast<int32_t>(i % st.pitch);
    const int32_t y = st.sy0 + static_cast<int32_t>(i / st.pitch);
    s_col[i] = (x >= 0 && y >= 0 && x < static_cast<int32_t>(dimx) && y < static_cast<int32_t>(dimy))
                   ? __ldg(&L.words[static_cast<uint32_t>(y) * dimx + static_cast<uint32_t>(x)]) << 8
                   : 0u;
  }
  __syncthreads();
  uint32_t n_words = 0;  // z-column words this thread read from the window (4 per group)
  const uint64_t n_items = static_cast<uint64_t>(rot_end - rot_begin) * n_cchunks;
  for (uint64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    const uint32_t slot = static_cast<uint32_t>(item / n_cchunks);
    const uint32_t rot = rot_begin + slot;
    const uint32_t cc = static_cast<uint32_t>(item % n_cchunks);
    if (h.overflow[slot]) continue;  // uniform per CTA
    uint32_t P, x0r;
    if (!owned_slabs(bp, nrot, rot, &P, &x0r)) continue;
    const uint32_t n_own_x = x0r < bp.nx ? (bp.nx - x0r + P - 1) / P : 0;
    const uint64_t ncols = static_cast<uint64_t>(n_own_x) * bp.ny;
    const uint64_t col0 = static_cast<uint64_t>(cc) * blockDim.x;
    if (col0 >= ncols) continue;
    const uint64_t c = col0 + threadIdx.x;
    const bool valid = c < ncols;
    const uint32_t ix_rel = valid ? x0r + static_cast<uint32_t>(c / bp.ny) * P : x0r;
    const uint32_t iy_rel = valid ? static_cast<uint32_t>(c % bp.ny) : 0u;
    const int32_t ix = bp.x0 + static_cast<int32_t>(ix_rel), iy = bp.y0 + static_cast<int32_t>(iy_rel);
    // padded index of the translation's own column
    const int32_t base = (iy - L.box_min[1] - st.sy0) * static_cast<int32_t>(st.pitch) +
                         (ix - L.box_min[0] - st.sx0);
    uint32_t acc[NZ];
#pragma unroll
    for (int j = 0; j < NZ; ++j) acc[j] = 0;
    const int n_grp = (h.n_ent[slot] + 3) >> 2;
    const int n_amb = h.n_amb[slot];
    const int4* __restrict__ grp = h.entries + static_cast<uint64_t>(slot) * kHistCap;
    // Survivor bound: a root's score can still grow by at most the counts of
    // the entries not yet probed plus its ambiguous points.  Once even the
    // best of this column's z-translations cannot reach the threshold, its
    // exact value is unobservable (search.hpp:117-123 only counts the root
    // as pruned) and the column stops early; entries come heaviest first.
    // the translation's own column as a shared-memory byte address: an
    // entry's word is one add away (offsets are stored in bytes)
    const uint32_t col_b = static_cast<uint32_t>(__cvta_generic_to_shared(s_col)) + 4u * static_cast<uint32_t>(base);
    bool done = !valid;
    for (int t0 = 0; t0 < n_grp; t0 += kGrpTile) {
      const int tn = min(kGrpTile, n_grp - t0);
      __syncthreads();
      for (int i = threadIdx.x; i < tn; i += blockDim.x) {
        s_go[i] = grp[2 * (t0 + i)];
        const int4 w = grp[2 * (t0 + i) + 1];
        s_gw[i] = static_cast<uint32_t>(w.x);
        if ((i & 7) == 0) s_rem[i >> 3] = w.y;  // root_hist_kernel's suffix sum
      }
      __syncthreads();
      auto group = [&](int gi) {
        const int4 o = s_go[gi];
        const uint32_t w4 = s_gw[gi];
        // byte offsets above the low 8 bits, shift amounts in the low 5 (wrap funnel shift)
        const uint32_t b0 = __funnelshift_r(lds_u32(col_b + static_cast<uint32_t>(o.x >> 8)), 0u, static_cast<uint32_t>(o.x));
        const uint32_t b1 = __funnelshift_r(lds_u32(col_b + static_cast<uint32_t>(o.y >> 8)), 0u, static_cast<uint32_t>(o.y));
        const uint32_t b2 = __funnelshift_r(lds_u32(col_b + static_cast<uint32_t>(o.z >> 8)), 0u, static_cast<uint32_t>(o.z));
        const uint32_t b3 = __funnelshift_r(lds_u32(col_b + static_cast<uint32_t>(o.w >> 8)), 0u, static_cast<uint32_t>(o.w));
        const uint32_t x = __byte_perm(__byte_perm(b0, b1, 0x0040), __byte_perm(b2, b3, 0x0040), 0x5410);
#pragma unroll
        for (int j = 0; j < NZ; ++j) acc[j] = __dp4a(x & (0x01010101u << j), w4, acc[j]);
      };
      // blocks of 8 groups (no per-group exit test), the survivor bound
      // checked between blocks
      int g = 0;
      while (!done && g < tn) {
        if (g) {
          uint32_t best = 0;
#pragma unroll
          for (int j = 0; j < NZ; ++j) best = max(best, acc[j] >> j);
          if (static_cast<int>(best) + s_rem[g >> 3] + n_amb < bp.threshold) {
            done = true;
            break;
          }
        }
        if (g + 8 <= tn) {
#pragma unroll
          for (int u = 0; u < 8; ++u) group(g + u);
          g += 8;
        } else {
          for (; g < tn; ++g) group(g);
        }
      }
      n_words += 4u * static_cast<uint32_t>(g);
    }
    int res[NZ];
#pragma unroll
    for (int j = 0; j < NZ; ++j) res[j] = static_cast<int>(acc[j] >> j);
    if (valid && n_amb && !done) {
      const uint32_t ir = rot / (bp.np * bp.nw), ip = (rot / bp.nw) % bp.np, iw = rot % bp.nw;
      double R[9];
      rotation_of(grid, bp.level, static_cast<int>(ir), static_cast<int>(ip), static_cast<int>(iw), R);
      for (int a = 0; a < n_amb; ++a) {
        const uint32_t p = h.amb[static_cast<uint64_t>(slot) * kAmbCap + a];
        const double px = scan.x[p], py = scan.y[p], pz = scan.z[p];
        const double rx = rot_row(R[0], R[1], R[2], px, py, pz);
        const double ry = rot_row(R[3], R[4], R[5], px, py, pz);
        const double rz = rot_row(R[6], R[7], R[8], px, py, pz);
#pragma unroll
        for (int j = 0; j < NZ; ++j)
          if (j < static_cast<int>(bp.nz)) res[j] += exact_hit(L, rx, ry, rz, ix, iy, bp.z0 + j);
      }
    }
    if (valid) {
      const uint64_t obase = (static_cast<uint64_t>(ix_rel) * bp.ny + iy_rel) * bp.nz;
#pragma unroll
      for (int j = 0; j < NZ; ++j)
        if (j < static_cast<int>(bp.nz)) scores[(obase + j) * nrot + rot] = res[j];
    }
    if (threadIdx.x == 0 && probes) {
      const uint64_t nc = min(static_cast<uint64_t>(blockDim.x), ncols - col0);
      atomicAdd(probes, static_cast<unsigned long long>(nc) * (h.n_ent[slot] + n_amb) * bp.nz);
    }
  }
  if (probes) {
    unsigned long long w = n_words;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
    if ((threadIdx.x & 31) == 0 && w) atomicAdd(probes + 2, w);
  }
}

__global__ void rotation_key_kernel(const bbs_node* __restrict__ nodes, uint64_t n, GridView G,
                                    unsigned long long* __restrict__ keys,
                                    uint32_t* __restrict__ idx) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const bbs_node nd = nodes[i];
    const int l = nd.level;
    keys[i] = (static_cast<unsigned long long>(l) << 60) |
              (static_cast<unsigned long long>(nd.iroll - G.lut_lo[l * 3 + 0]) << 40) |
              (static_cast<unsigned long long>(nd.ipitch - G.lut_lo[l * 3 + 1]) << 20) |
              static_cast<unsigned long long>(nd.iyaw - G.lut_lo[l * 3 + 2]);
    idx[i] = static_cast<uint32_t>(i);
  }
}

__global__ void expand_runs_kernel(const int32_t* __restrict__ counts,
                                   const int32_t* __restrict__ starts,
                                   const int32_t* __restrict__ chunk_off, int32_t n_runs,
                                   uint2* __restrict__ runs) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n_runs;
       r += int64_t(gridDim.x) * blockDim.x) {
    const int32_t c = counts[r], s = starts[r];
    int32_t o = chunk_off[r];
    for (int32_t j = 0; j < c; j += 32, ++o)
      runs[o] = make_uint2(static_cast<uint32_t>(s + j), static_cast<uint32_t>(min(32, c - j)));
  }
}

__global__ void nchunks_kernel(const int32_t* __restrict__ counts, int32_t n,
                               int32_t* __restrict__ out) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x)
    out[r] = (counts[r] + 31) / 32;
}

__global__ void write_scores_kernel(bbs_node* __restrict__ nodes, const int32_t* __restrict__ sc,
                                    uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    nodes[i].score = sc[i];
}

unsigned grid_1d(uint64_t n) {
  return static_cast<unsigned>(std::min<uint64_t>(std::max<uint64_t>((n + 255) / 256, 1), 148ull * 32));
}

// Co-batched flushes: blockIdx.y selects the search (ScoreSlot).
__global__ void __launch_bounds__(256, 4) score_cube8_group(MapView map, const ScoreSlot* __restrict__ ga,
                                                            size_t stride) {
  const ScoreSlot& a = score_slot(ga, stride);
  if (a.cache.enabled)
    score_cube8_kernel_body<true>(map, a.G, a.scan, a.nodes, a.d_n, a.n_ptiles, a.scores, a.cache, 1);
  else
    score_cube8_kernel_body<false>(map, a.G, a.scan, a.nodes, a.d_n, a.n_ptiles, a.scores, a.cache, 0);
}

}  // namespace

uint32_t choose_ptiles(uint64_t runs, uint32_t k) {
  const uint64_t target = 148ull * 8 * 2;  // ~2 waves of 256-thread CTAs
  uint64_t p = runs ? (target + runs - 1) / runs : 1;
  const uint64_t pmax = std::max<uint64_t>(1, (k + 1023) / 1024);  // >= 1024 points per tile
  p = std::min(std::max<uint64_t>(p, 1), pmax);
  return static_cast<uint32_t>(p);
}

void launch_score_box_chunked(const MapView& map, const GridView& grid, const ScanView& scan,
                              const BoxParams& bp, uint32_t rot_begin, uint32_t rot_end,
                              const int32_t* only, int32_t* scores, unsigned long long* probes,
                              cudaStream_t s) {
  static std::atomic<uint64_t> attr_done{0};
  static std::mutex attr_mu;
  const int smem = kHashSlots * 8 + kHashSlots * 4 + kChunk * 16 + kChunk * 4;
  once_per_device(attr_done, attr_mu, [&] {
    BBS_CUDA(cudaFuncSetAttribute(score_box_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  });
  const uint64_t items = static_cast<uint64_t>(rot_end - rot_begin) * bp.n_tchunks;
  const unsigned grid_sz = static_cast<unsigned>(std::min<uint64_t>(std::max<uint64_t>(items, 1), 148ull * 2 * 64));
  score_box_kernel<<<grid_sz, kBoxThreads, smem, s>>>(map, grid, scan, bp, rot_begin, rot_end, only,
                                                      scores, probes);
  BBS_CUDA(cudaGetLastError());
}

int colpad_ctas_per_sm(uint32_t nz, int smem) {
  switch (nz) {
#define BBS_OCC(NZ_) \
  case NZ_:          \
    return ctas_per_sm(root_colpad_kernel<NZ_>, 256, smem);
    BBS_OCC(1) BBS_OCC(2) BBS_OCC(3) BBS_OCC(4) BBS_OCC(5) BBS_OCC(6) BBS_OCC(7) BBS_OCC(8)
#undef BBS_OCC
  }
  return 1;
}

void launch_score_roots(const MapView& map, const GridView& grid, const ScanView& scan,
                        const BoxParams& bp, const RootHist& hist, int32_t* scores,
                        unsigned long long* probes, cudaStream_t s, cudaEvent_t ev_col0,
                        cudaEvent_t ev_col1) {
  const LevelView& L = map.level[bp.level];
  const uint32_t nrot = bp.nr * bp.np * bp.nw;
  const bool col_ok = L.layout == BBS_LAYOUT_BITMAP && L.nwz == 1 && L.words != nullptr &&
                      bp.nz <= 32 && L.dim[0] > 0;
  if (!col_ok) {
    launch_score_box_chunked(map, grid, scan, bp, 0, nrot, nullptr, scores, probes, s);
    return;
  }
  static std::atomic<uint64_t> attr_done{0};
  static std::mutex attr_mu;
  const int hist_smem = kHistSlots * 12;
  const int col_stage_max = 64 << 10;
  once_per_device(attr_done, attr_mu, [&] {
    BBS_CUDA(cudaFuncSetAttribute(root_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  hist_smem));
    BBS_CUDA(cudaFuncSetAttribute(root_col_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kEntTile * 16 + col_stage_max));
    BBS_CUDA(cudaFuncSetAttribute(root_col_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kEntTile * 16 + col_stage_max));
    BBS_CUDA(cudaFuncSetAttribute(root_col_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kEntTile * 16 + col_stage_max));
#define BBS_COLPAD_ATTR(NZ_)                                                                      \
  BBS_CUDA(cudaFuncSetAttribute(root_colpad_kernel<NZ_>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                kColPadHead + kColPadMax));
    BBS_COLPAD_ATTR(1) BBS_COLPAD_ATTR(2) BBS_COLPAD_ATTR(3) BBS_COLPAD_ATTR(4) BBS_COLPAD_ATTR(5)
    BBS_COLPAD_ATTR(6) BBS_COLPAD_ATTR(7) BBS_COLPAD_ATTR(8)
#undef BBS_COLPAD_ATTR
  });
  const uint64_t col_bytes = static_cast<uint64_t>(L.dim[0]) * L.dim[1] * 4ull;
  const int stage = col_bytes <= static_cast<uint64_t>(col_stage_max) ? 1 : 0;
  const int col_smem = kEntTile * 16 + (stage ? static_cast<int>(col_bytes) : 0);
  // padded staging: the staged window covers every translation column plus
  // the largest voxel offset on each side
  RootStage st{};
  {
    const int64_t R = bp.fpad;
    const int64_t xo0 = static_cast<int64_t>(bp.x0) - L.box_min[0], xo1 = xo0 + bp.nx - 1;
    const int64_t yo0 = static_cast<int64_t>(bp.y0) - L.box_min[1], yo1 = yo0 + bp.ny - 1;
    const int64_t sx0 = std::min<int64_t>(0, xo0) - R, sx1 = std::max<int64_t>(L.dim[0], xo1 + 1) + R;
    const int64_t sy0 = std::min<int64_t>(0, yo0) - R, sy1 = std::max<int64_t>(L.dim[1], yo1 + 1) + R;
    // odd pitch: the 32 lanes of a warp (consecutive y, one pitch apart)
    // read 32 distinct shared-memory banks
    const int64_t pitch = (sx1 - sx0) | (std::getenv("BBS_EVEN_PITCH") ? 0 : 1);
    const int64_t words = pitch * (sy1 - sy0);
    if (bp.nz <= 8 && L.dim[2] <= 24 && R < (1 << 15) && words * 4 <= kColPadMax &&
        std::getenv("BBS_ROOT_PAD") == nullptr) {
      st.enabled = 1;
      st.sx0 = static_cast<int32_t>(sx0);
      st.sy0 = static_cast<int32_t>(sy0);
      st.pitch = static_cast<uint32_t>(pitch);
      st.rows = static_cast<uint32_t>(sy1 - sy0);
      st.zoff = bp.z0 - L.box_min[2];
      st.dimz = L.dim[2];
    }
  }
  const int pad_smem = kColPadHead + static_cast<int>(st.pitch * st.rows * 4);
  uint32_t P, x0r;
  BoxParams b0 = bp;
  b0.rank = 0;
  b0.world = bp.world;
  owned_slabs(b0, nrot, 0, &P, &x0r);  // P depends on (nrot, world) only
  const uint64_t max_cols = static_cast<uint64_t>((bp.nx + P - 1) / P) * bp.ny;
  const uint32_t n_cchunks = static_cast<uint32_t>((max_cols + 255) / 256);
  for (uint32_t rb = 0; rb < nrot; rb += kRotBatch) {
    const uint32_t re = std::min<uint32_t>(nrot, rb + kRotBatch);
    BBS_CUDA(cudaMemsetAsync(hist.overflow + kRotBatch, 0, sizeof(int32_t), s));  // n_overflow
    root_hist_kernel<<<std::min<uint32_t>(re - rb, 148 * 4), 512, hist_smem, s>>>(
        grid, scan, bp, L, rb, re, hist, st, hist.overflow + kRotBatch);
    BBS_CUDA(cudaGetLastError());
    const uint64_t items = static_cast<uint64_t>(re - rb) * n_cchunks;
    const unsigned g = static_cast<unsigned>(std::min<uint64_t>(std::max<uint64_t>(items, 1), 148ull * 16));
    if (ev_col0 && rb == 0) BBS_CUDA(cudaEventRecord(ev_col0, s));
    if (st.enabled) {
      // persistent grid: every CTA stages the padded window once
      const unsigned gp = std::min<unsigned>(g, 148u * static_cast<unsigned>(colpad_ctas_per_sm(bp.nz, pad_smem)));
      switch (bp.nz) {
#define BBS_COLPAD(NZ_)                                                                              \
  case NZ_:                                                                                          \
    root_colpad_kernel<NZ_><<<gp, 256, pad_smem, s>>>(grid, scan, bp, L, rb, re, hist, st, n_cchunks, \
                                                     scores, probes);                                \
    break;
        BBS_COLPAD(1) BBS_COLPAD(2) BBS_COLPAD(3) BBS_COLPAD(4) BBS_COLPAD(5) BBS_COLPAD(6)
        BBS_COLPAD(7) BBS_COLPAD(8)
#undef BBS_COLPAD
      }
    } else if (bp.nz <= 8)
      root_col_kernel<8><<<g, 256, col_smem, s>>>(grid, scan, bp, L, rb, re, hist, n_cchunks, stage,
                                                  scores, probes);
    else if (bp.nz <= 16)
      root_col_kernel<16><<<g, 256, col_smem, s>>>(grid, scan, bp, L, rb, re, hist, n_cchunks, stage,
                                                   scores, probes);
    else
      root_col_kernel<32><<<g, 256, col_smem, s>>>(grid, scan, bp, L, rb, re, hist, n_cchunks, stage,
                                                   scores, probes);
    BBS_CUDA(cudaGetLastError());
    if (ev_col1 && re == nrot) BBS_CUDA(cudaEventRecord(ev_col1, s));
    // rotations whose histogram overflowed: chunked kernel (exits at once when none)
    launch_score_box_chunked(map, grid, scan, bp, rb, re, hist.overflow, scores, probes, s);
  }
}

int ctas_per_sm(const void* kernel, int threads, int smem) {
  struct Key {
    int dev;
    const void* k;
    int threads, smem;
  };
  static std::mutex mu;
  static std::vector<std::pair<Key, int>> memo;
  int dev = 0;
  BBS_CUDA(cudaGetDevice(&dev));
  {
    std::lock_guard<std::mutex> lk(mu);
    for (const auto& e : memo)
      if (e.first.dev == dev && e.first.k == kernel && e.first.threads == threads && e.first.smem == smem)
        return e.second;
  }
  int n = 1;
  BBS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, static_cast<size_t>(smem)));
  n = std::max(n, 1);
  std::lock_guard<std::mutex> lk(mu);
  memo.push_back({Key{dev, kernel, threads, smem}, n});
  return n;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("BBS_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}

void launch_score_cube8(const MapView& map, const GridView& grid, const ScanView& scan,
                        const bbs_node* nodes, const uint32_t* d_n, uint32_t n_max,
                        uint32_t n_ptiles, int32_t* scores, const RotCache* cache,
                        cudaStream_t s) {
  const uint64_t items = static_cast<uint64_t>((n_max + 7) / 8) * n_ptiles;
  // with the cache the run list and tiling are only known on the device:
  // one resident wave (4 CTAs per SM), grid-strided
  const unsigned g = cache ? share_cap(148ull * BBS_CUBE_MINB)
                           : static_cast<unsigned>(std::min<uint64_t>(std::max<uint64_t>(items, 1), share_cap(148ull * 4 * 8)));
  // the flush cache's direct runs (large scans) keep two points in flight;
  // without the cache (small scans, short point tiles) one point per step
  if (cache)
    launch_pdl(score_cube8_kernel<true>, g, 256, 0, s, map, grid, scan, nodes, d_n, n_ptiles, scores, *cache, 1);
  else
    launch_pdl(score_cube8_kernel<false>, g, 256, 0, s, map, grid, scan, nodes, d_n, n_ptiles, scores, RotCache{}, 0);
  BBS_CUDA(cudaGetLastError());
}

void launch_score_runs8(const MapView& map, const GridView& grid, const ScanView& scan,
                        const bbs_node* nodes, const uint32_t* d_n, uint32_t n_max,
                        uint32_t n_ptiles, int32_t* scores, cudaStream_t s) {
  const uint64_t items = static_cast<uint64_t>((n_max + 7) / 8) * n_ptiles;
  const unsigned g = static_cast<unsigned>(std::min<uint64_t>(std::max<uint64_t>(items, 1), 148ull * 8 * 8));
  score_runs_kernel<8><<<g, 256, 0, s>>>(map, grid, scan, nodes, nullptr, nullptr, 0, d_n, n_max,
                                         n_ptiles, scores);
  BBS_CUDA(cudaGetLastError());
}

void score_nodes_general(const MapView& map, const GridView& grid, const ScanView& scan,
                         bbs_node* d_nodes, uint64_t n, cudaStream_t s) {
  if (n == 0) return;
  if (n >= (1ull << 31)) throw Error(BBS_ERR_TOO_LARGE, "batch_evaluate: more than 2^31 nodes");
  const int ni = static_cast<int>(n);
  StreamAllocs al(s);
  unsigned long long* keys = al.get<unsigned long long>(n);
  unsigned long long* keys_alt = al.get<unsigned long long>(n);
  uint32_t* idx = al.get<uint32_t>(n);
  uint32_t* idx_alt = al.get<uint32_t>(n);
  rotation_key_kernel<<<grid_1d(n), 256, 0, s>>>(d_nodes, n, grid, keys, idx);
  BBS_CUDA(cudaGetLastError());
  cub::DoubleBuffer<unsigned long long> dk(keys, keys_alt);
  cub::DoubleBuffer<uint32_t> dv(idx, idx_alt);
  size_t t_sort = 0, t_rle = 0, t_scan = 0;
  BBS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t_sort, dk, dv, ni, 0, 64, s));
  int32_t* counts = al.get<int32_t>(n + 1);
  int32_t* starts = al.get<int32_t>(n + 1);
  int32_t* nch = al.get<int32_t>(n + 1);
  int32_t* choff = al.get<int32_t>(n + 1);
  int32_t* d_nruns = al.get<int32_t>(1);
  unsigned long long* uniq = al.get<unsigned long long>(n);
  BBS_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, t_rle, keys, uniq, counts, d_nruns, ni, s));
  BBS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t_scan, counts, starts, ni, s));
  const size_t t_all = std::max(t_sort, std::max(t_rle, t_scan));
  void* temp = al.get<unsigned char>(t_all);
  BBS_CUDA(cub::DeviceRadixSort::SortPairs(temp, t_sort, dk, dv, ni, 0, 64, s));
  BBS_CUDA(cub::DeviceRunLengthEncode::Encode(temp, t_rle, dk.Current(), uniq, counts, d_nruns, ni, s));
  int32_t nruns = 0;
  BBS_CUDA(cudaMemcpyAsync(&nruns, d_nruns, 4, cudaMemcpyDeviceToHost, s));
  BBS_CUDA(cudaStreamSynchronize(s));
  BBS_CUDA(cub::DeviceScan::ExclusiveSum(temp, t_scan, counts, starts, nruns, s));
  nchunks_kernel<<<grid_1d(nruns), 256, 0, s>>>(counts, nruns, nch);
  BBS_CUDA(cub::DeviceScan::ExclusiveSum(temp, t_scan, nch, choff, nruns, s));
  int32_t last_off = 0, last_n = 0;
  BBS_CUDA(cudaMemcpyAsync(&last_off, choff + nruns - 1, 4, cudaMemcpyDeviceToHost, s));
  BBS_CUDA(cudaMemcpyAsync(&last_n, nch + nruns - 1, 4, cudaMemcpyDeviceToHost, s));
  BBS_CUDA(cudaStreamSynchronize(s));
  const uint32_t nchunks = static_cast<uint32_t>(last_off + last_n);
  uint2* runs = al.get<uint2>(nchunks);
  int32_t* sc = al.get<int32_t>(n);
  expand_runs_kernel<<<grid_1d(nruns), 256, 0, s>>>(counts, starts, choff, nruns, runs);
  BBS_CUDA(cudaGetLastError());
  const uint32_t pt = choose_ptiles(nchunks, scan.k);
  if (pt > 1) BBS_CUDA(cudaMemsetAsync(sc, 0, n * 4, s));
  const uint64_t items = static_cast<uint64_t>(nchunks) * pt;
  const unsigned g = static_cast<unsigned>(std::min<uint64_t>(std::max<uint64_t>(items, 1), 148ull * 8 * 8));
  score_runs_kernel<32><<<g, 256, 0, s>>>(map, grid, scan, d_nodes, dv.Current(), runs, nchunks,
                                          nullptr, ni, pt, sc);
  BBS_CUDA(cudaGetLastError());
  write_scores_kernel<<<grid_1d(n), 256, 0, s>>>(d_nodes, sc, n);
  BBS_CUDA(cudaGetLastError());
}

void launch_score_cube8_group(const MapView& map, const ScoreSlot* slots, size_t stride, uint32_t n_slots,
                              cudaStream_t s) {
  launch_pdl(score_cube8_group, dim3(per_slot(148 * 4, n_slots), n_slots), 256, 0, s, map, slots, stride);
  BBS_CUDA(cudaGetLastError());
}

}  // namespace bbs

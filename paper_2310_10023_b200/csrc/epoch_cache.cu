// epoch_cache.cu — rotation histogram cache for the flush batches (K4).
//
// Every run of a flush (8 consecutive children of branch(), one rotation, a
// 2x2x2 translation cube) needs floor(R*p / cell) for all K scan points of
// its (level, rotation).  Rotations recur across flushes (C3 city: ~1.1M
// level-5 runs over ~1.3k level-5 rotations), so the de-duplicated histogram
// {(f, count)} of each (level, rotation) is built ONCE per search and kept in
// a device pool; a run then costs one cube probe per histogram entry instead
// of one rotation + probe per scan point.  Direct-mapped: slot = base[level]
// + dense rotation id, no sorting.  Per flush:
//   claim  (one thread per run)  claims empty slots, lists the builds;
//   build  (one CTA per claimed rotation) rotates the K points, dedups the
//          voxel offsets in shared memory, appends entries + ambiguous points
//          to the pool; when the offsets do not de-duplicate (fine levels) it
//          gives up early and flags the level uncached for the search;
//   probe  (one warp per (run, 256-entry chunk)) cube-probes the entries;
//   cube   (score.cu) scores the runs at uncached levels / failed builds.
// Exactness: the cached offsets use fast_floor with tmax = the largest
// translation index any node of that level can have in this search, so they
// are valid for every later run (score_common.cuh).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>

#include "kernels.h"
#include "score_common.cuh"

namespace bbs {

namespace {

constexpr int kCacheHashSlots = 8192;
constexpr int kCacheHashCap = 4096;   // distinct offsets kept in shared memory
constexpr int kCacheAmbCap = 2048;    // ambiguous points buffered per build
constexpr int kCacheListCap = 4096;   // dense box: cells touched, listed (beyond: the box is walked)
constexpr int kProbeChunk = 128;      // granule of the histogram entries per warp item (32 lanes x 4)
constexpr unsigned long long kEmptyKey = ~0ull;

__device__ __forceinline__ uint32_t cache_hash(unsigned long long key) {
  return static_cast<uint32_t>((key * 0x9E3779B97F4A7C15ull) >> 51);  // 13 bits
}

// Cell i of a dense box with rows of n cells: (x, y, z) = (i % n, i / n % n,
// i / n^2), divided once and then stepped cell by cell.
struct CellWalk {
  int i, x, y, z, n;
  __device__ CellWalk(int i0, int n_) : i(i0), x(i0 % n_), y(i0 / n_ % n_), z(i0 / (n_ * n_)), n(n_) {}
  __device__ void next() {
    ++i;
    if (++x == n) {
      x = 0;
      if (++y == n) {
        y = 0;
        ++z;
      }
    }
  }
};

constexpr int kBuildThreads = 512;
constexpr uint32_t kEarlyAbortPoints = 2048;  // sample before judging a build's de-duplication

// One CTA per claimed (level, rotation): rotate + floor every scan point
// (fast path), de-duplicate the voxel offsets in a shared-memory hash, and
// append (offset, count) entries + ambiguous point ids to the pool.  Two
// points per thread per step keep two load/rotate chains in flight.
__device__ __forceinline__ void cache_build_kernel_body(const RotCache& c,
                                                        const MapView& map,
                                                        const GridView& G,
                                                        ScanView scan,
                                                        uint32_t n_fixed) {
  pdl_wait();

  extern __shared__ __align__(16) unsigned char smem[];
  unsigned long long* s_key = reinterpret_cast<unsigned long long*>(smem);   // 64 KB
  int32_t* s_cnt = reinterpret_cast<int32_t*>(s_key + kCacheHashSlots);      // 32 KB
  uint32_t* s_amb = reinterpret_cast<uint32_t*>(s_cnt + kCacheHashSlots);    // 8 KB

  using ScanI = cub::BlockScan<int, kBuildThreads>;
  __shared__ typename ScanI::TempStorage s_scan;
  __shared__ int s_distinct, s_namb, s_oob, s_nl;
  __shared__ uint32_t s_off, s_aoff;
  const int lane = threadIdx.x & 31;
  // the flush's claimed builds (ctl[2]), or a fixed list (the prebuild)
  const uint32_t n_build = n_fixed ? n_fixed : c.ctl[2];
  for (uint32_t bi = blockIdx.x; bi < n_build; bi += gridDim.x) {
    const int4 bd = c.builds[bi];
    const uint32_t slot = static_cast<uint32_t>(bd.x);
    const int l = bd.y;
    const LevelView& L = map.level[l];
    const double tmax = c.tmax[l];
    double R[9];
    rotation_of(G, l, bd.z, bd.w, c.builds_w[bi], R);
    // dense box (coarse levels): direct-mapped 16-bit counters, no probing
    const int dr = c.dn_r[l];
    const bool dense = dr > 0;
    const int dzlo = c.dn_zlo[l], dxy = 2 * dr + 1;
    const int ncells = dense ? dxy * dxy * c.dn_nz[l] : 0;
    uint32_t* s_w = reinterpret_cast<uint32_t*>(smem);  // overlays the hash table
    // touched dense cells, listed after the counters in the hash region
    uint16_t* s_list = reinterpret_cast<uint16_t*>(s_w + ((ncells + 1) >> 1));
    const int list_cap = min(kCacheListCap, (kCacheHashSlots * 12 - ((ncells + 1) >> 1) * 4) / 2);
    if (dense) {
      for (int i = threadIdx.x; i < (ncells + 1) >> 1; i += blockDim.x) s_w[i] = 0u;
    } else {
      for (int i = threadIdx.x; i < kCacheHashSlots; i += blockDim.x) {
        s_key[i] = kEmptyKey;
        s_cnt[i] = 0;
      }
    }
    if (threadIdx.x == 0) {
      s_distinct = 0;
      s_namb = 0;
      s_oob = 0;
      s_nl = 0;
    }
    __syncthreads();
    // all lanes stay in the loop together (warp-aggregated inserts below)
    bool aborted = false;
    if (dense) {
      // Dense box, tight loop: one constant eps per level (dn_eps bounds the
      // per-point eps of fast_floor for every in-box offset; an out-of-box
      // point gives the build up, so the bound is only ever used in-box) and
      // an unsigned box test on the saturated int conversion.
      const double eps = c.dn_eps[l], eps1 = c.dn_eps1[l], inv = L.inv_cell;
      const uint32_t udxy = static_cast<uint32_t>(dxy), unz = static_cast<uint32_t>(c.dn_nz[l]);
      // two points per thread per step: two load / rotate chains in flight
      for (uint32_t p0 = 0; p0 < scan.k; p0 += 2 * blockDim.x) {
        double px[2], py[2], pz[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t p = p0 + h * blockDim.x + threadIdx.x;
          const bool live = p < scan.k;
          px[h] = live ? scan.x[p] : 0.0;
          py[h] = live ? scan.y[p] : 0.0;
          pz[h] = live ? scan.z[p] : 0.0;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t p = p0 + h * blockDim.x + threadIdx.x;
          int idx = -1;
          if (p < scan.k) {
            const double wx = __dmul_rn(rot_row(R[0], R[1], R[2], px[h], py[h], pz[h]), inv);
            const double wy = __dmul_rn(rot_row(R[3], R[4], R[5], px[h], py[h], pz[h]), inv);
            const double wz = __dmul_rn(rot_row(R[6], R[7], R[8], px[h], py[h], pz[h]), inv);
            const double flx = floor(wx), fly = floor(wy), flz = floor(wz);
            const double frx = __dsub_rn(wx, flx), fry = __dsub_rn(wy, fly), frz = __dsub_rn(wz, flz);
            const bool ok = frx > eps && frx < eps1 && fry > eps && fry < eps1 && frz > eps && frz < eps1;
            if (!ok) {
              const int a = atomicAdd(&s_namb, 1);
              if (a < kCacheAmbCap) s_amb[a] = p;
            } else {
              const uint32_t ux = static_cast<uint32_t>(__double2int_rz(flx)) + static_cast<uint32_t>(dr);
              const uint32_t uy = static_cast<uint32_t>(__double2int_rz(fly)) + static_cast<uint32_t>(dr);
              const uint32_t uz = static_cast<uint32_t>(__double2int_rz(flz)) - static_cast<uint32_t>(dzlo);
              if (ux < udxy && uy < udxy && uz < unz)
                idx = static_cast<int>((uz * udxy + uy) * udxy + ux);
              else
                s_oob = 1;  // outside the box: this build gives up (cube kernel scores its runs)
            }
          }
          // one shared atomic per point (warp aggregation with MATCH.ANY
          // costs more than the conflicts it saves: C3 prebuild 0.42 -> 0.21
          // ms); the first count of a cell lists it, so the entries are
          // emitted from the list (~2k cells) instead of a box walk (~20k)
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
    }
    for (uint32_t p0 = 0; !dense && p0 < scan.k; p0 += 2 * blockDim.x) {
      uint32_t p[2];
      double px[2], py[2], pz[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        p[h] = p0 + h * blockDim.x + threadIdx.x;
        const bool live = p[h] < scan.k;
        px[h] = live ? scan.x[p[h]] : 0.0;
        py[h] = live ? scan.y[p[h]] : 0.0;
        pz[h] = live ? scan.z[p[h]] : 0.0;
      }
      // uniform (read after the step barrier): give up when the table is full,
      // or early when the offsets seen so far do not even halve the points
      // (fine levels: the histogram would cost more than the runs it serves)
      if (!dense && (s_distinct >= kCacheHashCap || (p0 >= kEarlyAbortPoints && 2u * s_distinct > p0))) {
        aborted = true;
        break;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const bool live = p[h] < scan.k;
        bool ok = false;
        int32_t fx = 0, fy = 0, fz = 0;
        if (live) {
          ok = fast_floor(rot_row(R[0], R[1], R[2], px[h], py[h], pz[h]), L.inv_cell, tmax, &fx) &
               fast_floor(rot_row(R[3], R[4], R[5], px[h], py[h], pz[h]), L.inv_cell, tmax, &fy) &
               fast_floor(rot_row(R[6], R[7], R[8], px[h], py[h], pz[h]), L.inv_cell, tmax, &fz);
          ok = ok && fx > -(1 << 20) && fx < (1 << 20) && fy > -(1 << 20) && fy < (1 << 20) &&
               fz > -(1 << 20) && fz < (1 << 20);
          if (!ok) {
            const int a = atomicAdd(&s_namb, 1);
            if (a < kCacheAmbCap) s_amb[a] = p[h];
          }
        }
        const bool ins = live && ok;
        if (dense) {
          int idx = -1;
          if (ins) {
            const int zz = fz - dzlo;
            if (fx >= -dr && fx <= dr && fy >= -dr && fy <= dr && zz >= 0 && zz < c.dn_nz[l])
              idx = (zz * dxy + (fy + dr)) * dxy + (fx + dr);
            else
              s_oob = 1;  // outside the box: this build gives up (cube kernel scores its runs)
          }
          const unsigned same = __match_any_sync(0xffffffffu, idx);
          if (idx >= 0 && (__ffs(same) - 1) == lane)
            atomicAdd(&s_w[idx >> 1], static_cast<uint32_t>(__popc(same)) << ((idx & 1) << 4));
          continue;
        }
        const unsigned long long key = ins ? (static_cast<unsigned long long>(fx + (1 << 20)) << 42) |
                                                 (static_cast<unsigned long long>(fy + (1 << 20)) << 21) |
                                                 static_cast<unsigned long long>(fz + (1 << 20))
                                           : kEmptyKey;
        // neighbouring scan points often share a voxel: one insert per distinct key per warp
        const unsigned same = __match_any_sync(0xffffffffu, key);
        int fresh = 0;
        if (ins && (__ffs(same) - 1) == lane) {
          const int mult = __popc(same);
          uint32_t hh = cache_hash(key);
          for (;;) {
            const unsigned long long prev = atomicCAS(&s_key[hh], kEmptyKey, key);
            if (prev == kEmptyKey || prev == key) {
              fresh = prev == kEmptyKey;
              atomicAdd(&s_cnt[hh], mult);
              break;
            }
            hh = (hh + 1) & (kCacheHashSlots - 1);
          }
        }
        // the distinct count only gates further inserts (the table has 2x room)
        const int nf = __reduce_add_sync(0xffffffffu, fresh);
        if (lane == 0 && nf) atomicAdd(&s_distinct, nf);
      }
      if (!dense) __syncthreads();
    }
    __syncthreads();
    // too many distinct offsets (fine levels: about one per point): the
    // histogram would not beat direct scoring, so give the level up
    const bool raw = aborted;  // (a finished table holds <= cap + one step < slots)
    const bool oob = s_oob != 0;
    const int namb = s_namb;
    // entries in slot / cell order (block scan; deterministic layout)
    constexpr int kPer = kCacheHashSlots / kBuildThreads;
    const int dper = (ncells + kBuildThreads - 1) / kBuildThreads;
    const int dc0 = min(ncells, static_cast<int>(threadIdx.x) * dper), dc1 = min(ncells, dc0 + dper);
    auto dcount = [&](int i) { return (s_w[i >> 1] >> ((i & 1) << 4)) & 0xFFFFu; };
    // the staged level stores groups of 4 byte-count entries (counts > 255 split)
    const bool staged = dense && l == c.stg_level;
    const int nl = s_nl;
    const bool listed = dense && nl <= list_cap;  // else: walk the whole box
    int cnt = 0;
    if (listed) {
      if (!oob)
        for (int j = threadIdx.x; j < nl; j += kBuildThreads) {
          const uint32_t v = dcount(s_list[j]);
          cnt += staged ? static_cast<int>((v + 254u) / 255u) : 1;
        }
    } else if (dense) {
      if (!oob)
        for (int i = dc0; i < dc1; ++i) {
          const uint32_t v = dcount(i);
          cnt += staged ? static_cast<int>((v + 254u) / 255u) : (v != 0u ? 1 : 0);
        }
    } else if (!raw) {
#pragma unroll
      for (int k = 0; k < kPer; ++k) cnt += s_key[threadIdx.x * kPer + k] != kEmptyKey ? 1 : 0;
    }
    int epos, n_dist;
    ScanI(s_scan).ExclusiveSum(cnt, epos, n_dist);
    const uint32_t n_ent = (raw || oob) ? 0u : static_cast<uint32_t>(n_dist);
    // pool space in int4 units (staged: 2 int4 per group of 4 entries)
    const uint32_t n_slots = staged ? 2u * ((n_ent + 3u) / 4u) : n_ent;
    if (threadIdx.x == 0) {
      s_off = (raw || oob) ? 0u : atomicAdd(&c.ctl[0], n_slots);
      s_aoff = (raw || oob) ? 0u : atomicAdd(&c.ctl[1], static_cast<uint32_t>(namb));
      if (raw) c.ctl[4 + (l & (kMaxLevels - 1))] = 1u;
    }
    __syncthreads();
    const uint32_t off = s_off, aoff = s_aoff;
    const bool fits = !raw && !oob && namb <= kCacheAmbCap &&
                      static_cast<uint64_t>(off) + n_slots <= c.pool_cap &&
                      static_cast<uint64_t>(aoff) + namb <= c.amb_cap;
    if (fits && staged) {
      int32_t* gw = reinterpret_cast<int32_t*>(c.pool + off);
      unsigned char* gb = reinterpret_cast<unsigned char*>(c.pool + off);
      auto put = [&](uint32_t v, int fx, int fy, int fz) {
        const int32_t eoff = fy * static_cast<int32_t>(c.stg_pitch) + fx;
        for (; v; ++epos) {
          const uint32_t w = min(v, 255u);
          v -= w;
          const int g = epos >> 2, k = epos & 3;
          gw[g * 8 + k] = eoff;
          gb[(g * 8 + 4) * 4 + k] = static_cast<unsigned char>(static_cast<int8_t>(fz));
          gb[(g * 8 + 5) * 4 + k] = static_cast<unsigned char>(w);
        }
      };
      if (listed) {
        for (int j = threadIdx.x; j < nl; j += kBuildThreads) {
          const int i = s_list[j];
          put(dcount(i), i % dxy - dr, (i / dxy) % dxy - dr, i / (dxy * dxy) + dzlo);
        }
      } else {
        for (CellWalk w(dc0, dxy); w.i < dc1; w.next()) {
          const uint32_t v = dcount(w.i);
          if (v) put(v, w.x - dr, w.y - dr, w.z + dzlo);
        }
      }
      // zero-count padding of the last group
      const int pe = static_cast<int>(n_ent) + static_cast<int>(threadIdx.x);
      if (pe < static_cast<int>((n_ent + 3u) & ~3u)) {
        const int g = pe >> 2, k = pe & 3;
        gw[g * 8 + k] = 0;
        gb[(g * 8 + 4) * 4 + k] = 0;
        gb[(g * 8 + 5) * 4 + k] = 0;
      }
    } else if (fits && listed) {
      for (int j = threadIdx.x; j < nl; j += kBuildThreads) {
        const int i = s_list[j];
        c.pool[off + epos] = make_int4(i % dxy - dr, (i / dxy) % dxy - dr, i / (dxy * dxy) + dzlo,
                                       static_cast<int32_t>(dcount(i)));
        ++epos;
      }
    } else if (fits && dense) {
      for (CellWalk w(dc0, dxy); w.i < dc1; w.next()) {
        const uint32_t v = dcount(w.i);
        if (v) {
          c.pool[off + epos] = make_int4(w.x - dr, w.y - dr, w.z + dzlo, static_cast<int32_t>(v));
          ++epos;
        }
      }
    } else if (fits) {
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const int i = threadIdx.x * kPer + k;
        const unsigned long long key = s_key[i];
        if (key != kEmptyKey) {
          c.pool[off + epos] = make_int4(static_cast<int32_t>((key >> 42) & 0x1FFFFF) - (1 << 20),
                                         static_cast<int32_t>((key >> 21) & 0x1FFFFF) - (1 << 20),
                                         static_cast<int32_t>(key & 0x1FFFFF) - (1 << 20), s_cnt[i]);
          ++epos;
        }
      }
    }
    if (fits)
      for (int a = threadIdx.x; a < namb; a += blockDim.x) c.amb_pool[aoff + a] = s_amb[a];
    __syncthreads();
    if (threadIdx.x == 0) {
      c.amb_off[slot] = aoff;
      // publish: entries first, then the state (readers run in later kernels)
      c.info[slot] = fits ? make_int4(kCacheReady, static_cast<int32_t>(off), static_cast<int32_t>(n_ent), namb)
                          : make_int4(kCacheNone, 0, 0, 0);
      if (fits) atomicMax(&c.ctl[kCtlMaxEnt], n_ent);  // sizes the probe's chunk grid
      // the prebuilt level predicts the finer ones: a scan of surfaces has
      // ~4x the distinct offsets per halving of the cell, so when that would
      // not halve the points (or not fit a build) the finer levels are
      // scored directly instead of each paying a failed build first
      // (a dense-box level holds up to kCacheDenseCells offsets, a hashed
      // one kCacheHashCap)
      if (fits && l == c.pre_level) {
        uint64_t pred = n_ent;
        for (int l2 = l - 1; l2 >= 0; --l2) {
          pred *= 4u;
          const uint64_t cap2 = c.dn_r[l2] > 0 ? static_cast<uint64_t>(kCacheDenseCells)
                                               : static_cast<uint64_t>(kCacheHashCap);
          if (pred > min(static_cast<uint64_t>(scan.k / 2u), cap2)) c.ctl[4 + l2] = 1u;
        }
      }
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kBuildThreads) cache_build_kernel(RotCache c, MapView map, GridView G,
                                                                    ScanView scan, uint32_t n_fixed) {
  cache_build_kernel_body(c, map, G, scan, n_fixed);
}

// Ambiguous points of one run (exact divide path), kept out of line so the
// probe loop's register budget stays small.
__device__ __forceinline__ void probe_ambiguous(const RotCache& c, const LevelView& L, const GridView& G,
                                             const ScanView& scan, uint32_t slot, int n_amb, int l,
                                             int ir, int ip, int iw, int32_t bx, int32_t by,
                                             int32_t bz, int lane, int acc[8]) {
  double R[9];
  rotation_of(G, l, ir, ip, iw, R);
  const uint32_t* __restrict__ amb = c.amb_pool + c.amb_off[slot];
  for (int q = lane; q < n_amb; q += 32) {
    const uint32_t p = amb[q];
    const double px = scan.x[p], py = scan.y[p], pz = scan.z[p];
    const double rx = rot_row(R[0], R[1], R[2], px, py, pz);
    const double ry = rot_row(R[3], R[4], R[5], px, py, pz);
    const double rz = rot_row(R[6], R[7], R[8], px, py, pz);
#pragma unroll
    for (int t = 0; t < 8; ++t)
      acc[t] += exact_hit(L, rx, ry, rz, bx + (t >> 2), by + ((t >> 1) & 1), bz + (t & 1));
  }
}

// Warp items are (run, chunk of its histogram) pairs, grid-strided.  The 32
// lanes first fetch the headers (run node, cache info) of 32 items in
// parallel and park the ones with entries in a per-warp shared-memory list,
// so the probe loops hold no header registers and empty chunks or uncached
// runs cost no serial load latency.  Block shape (A/B, C2 / C3 device ms):
// 256x3 0.833 / 13.83, 512x2 0.838 / 13.95, 1024x1 0.838 / 14.39 -- the
// kernel is bound by its dependent-load chain (headers, window, entries),
// not by occupancy (1024x1 reaches 37% achieved vs 22%).
#ifndef BBS_PROBE_T
#define BBS_PROBE_T 256
#define BBS_PROBE_B 3
#endif
constexpr int kProbeThreads = BBS_PROBE_T;
constexpr int kProbeWarps = kProbeThreads / 32;
struct __align__(16) ProbeItem {
  int4 h0;  // bx, by, bz, run
  int4 h1;  // level, pool offset, first entry, end entry
  int4 h2;  // ambiguous points (chunk 0 only), slot, iroll, ipitch | iyaw << 16
};
constexpr int kProbeItemBytes = kProbeWarps * 32 * static_cast<int>(sizeof(ProbeItem));

__device__ __forceinline__ void cache_probe_kernel_body(const RotCache& c,
                                                        const MapView& map,
                                                        const GridView& G,
                                                        ScanView scan,
                                                        const bbs_node* __restrict__ pending,
                                                        const uint32_t* __restrict__ d_n,
                                                        uint32_t chunks_per_run,
                                                        uint32_t half_items_per_warp,
                                                        bool lazy_stage,
                                                        int32_t* __restrict__ scores) {
  // [staged level's padded column window][per-warp item lists]
  extern __shared__ __align__(16) unsigned char probe_smem[];
  __shared__ __align__(8) unsigned long long s_mbar;
  const uint32_t win_bytes = c.stg_level >= 0 ? ((c.stg_pitch * c.stg_rows * 4u) + 15u) & ~15u : 0u;
  const uint32_t* s_win = reinterpret_cast<const uint32_t*>(probe_smem);
  ProbeItem* s_items = reinterpret_cast<ProbeItem*>(probe_smem + win_bytes) + (threadIdx.x >> 5) * 32;
  // the window is search-constant: one bulk copy per CTA, issued before
  // pdl_wait (it does not depend on the previous kernel) and awaited only
  // by warps that probe the staged level
  // (co-batched launches stage lazily: most CTAs of a light slot have no item)
  if (!lazy_stage && win_bytes) bulk_issue(probe_smem, c.stg_win, win_bytes, &s_mbar);
  __syncthreads();  // the mbarrier is initialised before anyone polls it
  bool win_ready = win_bytes == 0;
  pdl_wait();

  const uint32_t n_runs = *d_n / 8;
  const int lane = threadIdx.x & 31;
  const uint64_t n_warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const bool direct_on = c.direct_flag && (!c.direct_gate || *c.direct_gate);
  // warp items = (run, chunk of the run's histogram): as few chunks per run
  // as keep ~2 items per warp (each item ends in 8 warp reductions and
  // atomics), sized by the largest histogram built so far
  const uint32_t max_ent = max(1u, c.ctl[kCtlMaxEnt]);
  const uint32_t granules = (max_ent + kProbeChunk - 1) / kProbeChunk;
  const uint64_t want = (half_items_per_warp * n_warps / 2 + max(n_runs, 1u) - 1) / max(n_runs, 1u);
  {
    uint64_t cpr = want < granules ? want : granules;
    if (cpr > chunks_per_run) cpr = chunks_per_run;
    chunks_per_run = static_cast<uint32_t>(cpr);
  }
  chunks_per_run = max(chunks_per_run, 1u);
  const uint32_t chunk_len = ((granules + chunks_per_run - 1) / chunks_per_run) * kProbeChunk;
  const uint64_t n_items = static_cast<uint64_t>(n_runs) * chunks_per_run;
  const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (lazy_stage) {
    const bool any = static_cast<uint64_t>(blockIdx.x) * (blockDim.x >> 5) < n_items;
    if (win_bytes && any) bulk_issue(probe_smem, c.stg_win, win_bytes, &s_mbar);
    win_ready = win_bytes == 0 || !any;
    __syncthreads();
  }
  for (uint64_t k0 = 0; gw + k0 * n_warps < n_items; k0 += 32) {
    unsigned hm;
    {
      const uint64_t item = gw + (k0 + lane) * n_warps;
      // inf stays NONE for runs at uncached levels (no slot)
      int4 a = make_int4(0, 0, 0, 0), b = make_int4(0, 0, 0, 0), inf = make_int4(kCacheNone, 0, 0, 0);
      uint32_t slot = 0, chunk = 0, run = 0;
      bool has = false, direct = false;
      if (item < n_items) {
        run = static_cast<uint32_t>(item / chunks_per_run);
        chunk = static_cast<uint32_t>(item % chunks_per_run);
        a = __ldg(reinterpret_cast<const int4*>(pending) + 16ull * run);
        b = __ldg(reinterpret_cast<const int4*>(pending) + 16ull * run + 1);
        direct = direct_on && c.direct_flag[run];  // scored by the direct phase below
        if (!direct && run_slot(c, G, a, b, &slot)) {
          inf = c.info[slot];
          has = inf.x == kCacheReady &&
                (chunk * chunk_len < static_cast<uint32_t>(inf.z) || (chunk == 0 && inf.w > 0));
        }
      }
      // runs without a READY histogram go to the cube kernel's list (chunk 0 items)
      const bool fb = item < n_items && chunk == 0 && !direct && inf.x != kCacheReady;
      const unsigned fbm = __ballot_sync(0xffffffffu, fb);
      if (fbm) {
        const int leader = __ffs(fbm) - 1;
        uint32_t at = 0;
        if (lane == leader) at = atomicAdd(&c.ctl[3], static_cast<uint32_t>(__popc(fbm)));
        at = __shfl_sync(0xffffffffu, at, leader);
        if (fb) c.fb_runs[at + __popc(fbm & ((1u << lane) - 1))] = run;
      }
      hm = __ballot_sync(0xffffffffu, has);
      if (has) {
        const uint32_t e0 = chunk * chunk_len;
        const uint32_t e1 = min(static_cast<uint32_t>(inf.z), e0 + chunk_len);
        ProbeItem it;
        it.h0 = make_int4(a.x, a.y, a.z, static_cast<int32_t>(run));
        it.h1 = make_int4(b.z, inf.y, static_cast<int32_t>(e0), static_cast<int32_t>(e1));
        it.h2 = make_int4(chunk == 0 ? inf.w : 0, static_cast<int32_t>(slot), a.w,
                          (b.x & 0xFFFF) | (b.y << 16));
        s_items[__popc(hm & ((1u << lane) - 1))] = it;
      }
      __syncwarp();
    }
    const int nh = __popc(hm);
    for (int j = 0; j < nh; ++j) {
      const int4 h0 = s_items[j].h0;
      const int4 h1 = s_items[j].h1;
      const int32_t bx = h0.x, by = h0.y, bz = h0.z;
      const int l = h1.x;
      const int4* __restrict__ ent = c.pool + static_cast<uint32_t>(h1.y);
      const uint32_t e0 = static_cast<uint32_t>(h1.z), e1 = static_cast<uint32_t>(h1.w);
      const LevelView& L = map.level[l];
      int acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if (l == c.stg_level) {
        if (!win_ready) {
          bulk_wait(&s_mbar);
          win_ready = true;
        }
        // staged: 4 LDS + 4 clamped funnel shifts give an entry's 2x2x2 child
        // mask (bits t = dx*4 + dy*2 + dz); 4 masks are packed as bytes and
        // per child t one LOP3 + IDP4A adds 2^t * count of the hits
        const int32_t pitch = static_cast<int32_t>(c.stg_pitch);
        const int32_t base = (by - L.box_min[1] - c.stg_sy0) * pitch + (bx - L.box_min[0] - c.stg_sx0);
        const int32_t oz8 = bz - L.box_min[2] + 8;
        uint32_t a8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const uint32_t g_end = (e1 + 3) >> 2;
#pragma unroll 2
        for (uint32_t g = (e0 >> 2) + lane; g < g_end; g += 32) {
          const int4 o = __ldg(ent + 2 * g);
          const int4 q = __ldg(ent + 2 * g + 1);
          const int32_t eo[4] = {o.x, o.y, o.z, o.w};
          uint32_t m4 = 0;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int32_t i = base + eo[k];
            const uint32_t sh = static_cast<uint32_t>(static_cast<int32_t>(static_cast<int8_t>(q.x >> (8 * k))) + oz8);
            const uint32_t b8 = (__funnelshift_rc(s_win[i], 0u, sh) & 0x03u) |
                                (__funnelshift_rc(s_win[i + pitch], 0u, sh - 2u) & 0x0Cu) |
                                (__funnelshift_rc(s_win[i + 1], 0u, sh - 4u) & 0x30u) |
                                (__funnelshift_rc(s_win[i + pitch + 1], 0u, sh - 6u) & 0xC0u);
            m4 |= b8 << (8 * k);
          }
          const uint32_t w4 = static_cast<uint32_t>(q.y);
#pragma unroll
          for (int t = 0; t < 8; ++t) a8[t] = __dp4a(m4 & (0x01010101u << t), w4, a8[t]);
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) acc[t] = static_cast<int>(a8[t] >> t);
      } else if (L.layout == BBS_LAYOUT_BITMAP) {
        const uint32_t ox = static_cast<uint32_t>(bx) - static_cast<uint32_t>(L.box_min[0]);
        const uint32_t oy = static_cast<uint32_t>(by) - static_cast<uint32_t>(L.box_min[1]);
        const uint32_t oz = static_cast<uint32_t>(bz) - static_cast<uint32_t>(L.box_min[2]);
        // two entries per lane per step: 8-16 independent column loads in flight
        uint32_t e = e0 + lane;
        for (; e + 32 < e1; e += 64) {
          const int4 f0 = __ldg(ent + e);
          const int4 f1 = __ldg(ent + e + 32);
          cube_probe(L, static_cast<uint32_t>(f0.x) + ox, static_cast<uint32_t>(f0.y) + oy,
                     static_cast<uint32_t>(f0.z) + oz, f0.w, acc);
          cube_probe(L, static_cast<uint32_t>(f1.x) + ox, static_cast<uint32_t>(f1.y) + oy,
                     static_cast<uint32_t>(f1.z) + oz, f1.w, acc);
        }
        if (e < e1) {
          const int4 f = __ldg(ent + e);
          cube_probe(L, static_cast<uint32_t>(f.x) + ox, static_cast<uint32_t>(f.y) + oy,
                     static_cast<uint32_t>(f.z) + oz, f.w, acc);
        }
      } else {
        for (uint32_t e = e0 + lane; e < e1; e += 32) {
          const int4 f = __ldg(ent + e);
#pragma unroll
          for (int t = 0; t < 8; ++t)
            acc[t] += level_contains(L, f.x + bx + (t >> 2), f.y + by + ((t >> 1) & 1),
                                     f.z + bz + (t & 1))
                          ? f.w
                          : 0;
        }
      }
      const int4 h2 = s_items[j].h2;
      if (h2.x > 0)
        probe_ambiguous(c, L, G, scan, static_cast<uint32_t>(h2.y), h2.x, l, h2.z, h2.w & 0xFFFF, h2.w >> 16,
                        bx, by, bz, lane, acc);
      const uint32_t r = static_cast<uint32_t>(h0.w);
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int v = __reduce_add_sync(0xffffffffu, acc[t]);
        if (lane == 0 && v) atomicAdd(&scores[8ull * r + t], v);
      }
    }
    __syncwarp();  // the list is rewritten by the next round of headers
  }
  // no CTA exits with its window copy in flight
  if (!win_ready) bulk_wait(&s_mbar);
  // direct phase: the runs the branch kernel listed (no histogram possible
  // this flush) in (run, point tile) items taken dynamically, so CTAs that
  // finish their histogram items early take more of them (these runs no
  // longer wait for a cube kernel after the probe)
  // (CTA items: warp items of 256 points measured slower, C3 13.57 vs 13.34 ms)
  const uint32_t n_dir = direct_on ? c.ctl[kCtlDirect] : 0u;
  if (n_dir) {
    __shared__ double s_R[9];
    __shared__ int32_t s_hdr[4], s_cnt[8];
    __shared__ uint32_t s_item;
    const uint32_t pmax = max(1u, (scan.k + 1023u) / 1024u);
    const uint32_t n_pt = min(pmax, max(1u, (2u * gridDim.x + n_dir - 1) / n_dir));
    const uint32_t n_it = n_dir * n_pt;
    for (;;) {
      __syncthreads();  // the previous item's scratch is free
      if (threadIdx.x == 0) s_item = atomicAdd(&c.ctl[kCtlDirectItem], 1u);
      __syncthreads();
      const uint32_t it = s_item;
      if (it >= n_it) break;
      cube8_item<true>(map, G, scan, pending, c.direct_runs[it / n_pt], it % n_pt, n_pt, scores, s_R, s_hdr, s_cnt);
    }
  }
}

__global__ void __launch_bounds__(BBS_PROBE_T, BBS_PROBE_B) cache_probe_kernel(RotCache c, MapView map, GridView G,
                                                          ScanView scan,
                                                          const bbs_node* __restrict__ pending,
                                                          const uint32_t* __restrict__ d_n,
                                                          uint32_t chunks_per_run, uint32_t half_items_per_warp,
                                                          int32_t* __restrict__ scores) {
  cache_probe_kernel_body(c, map, G, scan, pending, d_n, chunks_per_run, half_items_per_warp, false, scores);
}

// The staged probe window: zero-padded, words shifted up by 8 bits; the
// tail up to a multiple of 4 words (16 bytes for the bulk copy) is zero.
__global__ void stage_window_kernel(LevelView SL, int32_t sx0, int32_t sy0, uint32_t pitch, uint32_t n,
                                    uint32_t n16, uint32_t* __restrict__ win) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += gridDim.x * blockDim.x) {
    const int32_t x = sx0 + static_cast<int32_t>(i % pitch);
    const int32_t y = sy0 + static_cast<int32_t>(i / pitch);
    win[i] = i < n && x >= 0 && y >= 0 && x < static_cast<int32_t>(SL.dim[0]) && y < static_cast<int32_t>(SL.dim[1])
                 ? SL.words[static_cast<uint32_t>(y) * SL.dim[0] + static_cast<uint32_t>(x)] << 8
                 : 0u;
  }
}

// Co-batched flushes: blockIdx.y selects the search (ScoreSlot).  Slots
// without the cache skip both kernels (the cube kernel scores their runs).
__global__ void __launch_bounds__(kBuildThreads) cache_build_group(MapView map, const ScoreSlot* __restrict__ ga,
                                                                   size_t stride) {
  const ScoreSlot& a = score_slot(ga, stride);
  if (!a.cache.enabled) return;
  cache_build_kernel_body(a.cache, map, a.G, a.scan, 0u);
}

__global__ void __launch_bounds__(BBS_PROBE_T, BBS_PROBE_B) cache_probe_group(MapView map,
                                                                             const ScoreSlot* __restrict__ ga,
                                                                             size_t stride, uint32_t hipw) {
  const ScoreSlot& a = score_slot(ga, stride);
  if (!a.cache.enabled) return;
  cache_probe_kernel_body(a.cache, map, a.G, a.scan, a.nodes, a.d_n, (a.scan.k + kProbeChunk - 1) / kProbeChunk, hipw,
                          true, a.scores);
}

}  // namespace

void build_stage_window(const MapView& map, const RotCache& cache, uint32_t* win, cudaStream_t s) {
  const uint32_t n = cache.stg_pitch * cache.stg_rows;
  const uint32_t n16 = (n + 3u) & ~3u;  // bulk copies move multiples of 16 bytes
  stage_window_kernel<<<std::min<uint32_t>((n16 + 255) / 256, 148 * 8), 256, 0, s>>>(
      map.level[cache.stg_level], cache.stg_sx0, cache.stg_sy0, cache.stg_pitch, n, n16, win);
  BBS_CUDA(cudaGetLastError());
}

// Prebuild: every rotation of one level listed as a build (all slots of the
// level are claimed up front).  The level-(L-1) histograms are needed by
// nearly every rotation of that level during the search (C2: 466 of 472,
// C3: 1264 of 1264), so building them in one launch replaces one serial
// CTA-per-build tail in each of the first flushes.
__global__ void cache_prebuild_list_kernel(RotCache c, GridView G, int l, uint32_t n_rot) {
  const uint32_t np = static_cast<uint32_t>(G.max_index[l * 3 + 1]) + 1;
  const uint32_t nw = static_cast<uint32_t>(G.max_index[l * 3 + 2]) + 1;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_rot; i += gridDim.x * blockDim.x) {
    const uint32_t slot = c.base[l] + i;
    c.info[slot].x = kCacheBuilding;
    c.builds[i] = make_int4(static_cast<int32_t>(slot), l, static_cast<int32_t>(i / (nw * np)),
                            static_cast<int32_t>((i / nw) % np));
    c.builds_w[i] = static_cast<int32_t>(i % nw);
  }
}

void launch_cache_prebuild_list(const GridView& grid, const RotCache& pre, int level, uint32_t n_rot,
                                 cudaStream_t s) {
  if (n_rot == 0) return;
  cache_prebuild_list_kernel<<<(n_rot + 255) / 256, 256, 0, s>>>(pre, grid, level, n_rot);
  BBS_CUDA(cudaGetLastError());
}

void launch_cache_prebuild(const MapView& map, const GridView& grid, const ScanView& scan, const RotCache& pre,
                           uint32_t n_rot, cudaStream_t s) {
  if (n_rot == 0) return;
  const int build_smem = kCacheHashSlots * 12 + kCacheAmbCap * 4;
  static std::atomic<uint64_t> attr_done{0};
  static std::mutex attr_mu;
  once_per_device(attr_done, attr_mu, [&] {
    BBS_CUDA(cudaFuncSetAttribute(cache_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, build_smem));
  });
  // A/B: BBS_PREBUILD_CTAS (default 2 per SM)
  const uint32_t ctas = [] {
    const char* v = std::getenv("BBS_PREBUILD_CTAS");
    return v ? std::max(1u, static_cast<uint32_t>(std::atoi(v))) : 148u * 2;
  }();
  cache_build_kernel<<<std::min<uint32_t>(n_rot, ctas), kBuildThreads, build_smem, s>>>(pre, map, grid, scan, n_rot);
  BBS_CUDA(cudaGetLastError());
}

void launch_epoch_score(const MapView& map, const GridView& grid, const ScanView& scan,
                        const bbs_node* pending, const uint32_t* d_n, uint32_t n_max,
                        uint32_t n_ptiles, int32_t* scores, const RotCache& cache, cudaStream_t s,
                        bool builds) {
  if (!cache.enabled) {
    launch_score_cube8(map, grid, scan, pending, d_n, n_max, n_ptiles, scores, nullptr, s);
    return;
  }
  static std::atomic<uint64_t> attr_done{0};
  static std::mutex attr_mu;
  const int build_smem = kCacheHashSlots * 12 + kCacheAmbCap * 4;
  static_assert(kCacheHashSlots % kBuildThreads == 0, "slot rows per thread");
  once_per_device(attr_done, attr_mu, [&] {
    BBS_CUDA(cudaFuncSetAttribute(cache_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, build_smem));
    BBS_CUDA(cudaFuncSetAttribute(cache_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kStageWindowMax + kProbeItemBytes));
  });
  const uint32_t max_runs = (n_max + 7) / 8;
  // the epoch's branch kernel already claimed the slots (cache_claim_run)
  // after its frontier reset ctl[2..3]
  if (builds) {  // false once no level can claim a build any more (host-known)
    launch_pdl(cache_build_kernel, std::min<uint32_t>(std::max<uint32_t>(max_runs, 1), share_cap(148 * 2)), kBuildThreads,
               build_smem, s, cache, map, grid, scan, 0u);
    BBS_CUDA(cudaGetLastError());
  }
  const uint32_t chunks = (scan.k + kProbeChunk - 1) / kProbeChunk;
  const uint64_t warp_items = static_cast<uint64_t>(max_runs) * chunks;
  const uint64_t wpc = kProbeThreads / 32;  // warps per CTA
  const unsigned g = static_cast<unsigned>(std::min<uint64_t>((warp_items + wpc - 1) / wpc + 1, share_cap(148ull * 16)));
  const int win_smem = (cache.stg_level >= 0 ? static_cast<int>(((cache.stg_pitch * cache.stg_rows * 4u) + 15u) & ~15u) : 0) +
                       kProbeItemBytes;

  unsigned gp = g;
  if (win_smem > 0) {
    // persistent: each CTA stages the window once
    const int per_sm = ctas_per_sm(cache_probe_kernel, kProbeThreads, win_smem);
    gp = std::min<unsigned>(g, share_cap(148ull * static_cast<unsigned>(per_sm)));
  }
  static const uint32_t hipw = [] {
    const char* v = std::getenv("BBS_PROBE_HIPW");  // A/B: 2x the warp items per warp
    return v ? static_cast<uint32_t>(std::max(1, std::atoi(v))) : 4u;
  }();
  launch_pdl(cache_probe_kernel, gp, kProbeThreads, win_smem, s, cache, map, grid, scan, pending, d_n, chunks, hipw,
             scores);
  BBS_CUDA(cudaGetLastError());
  launch_score_cube8(map, grid, scan, pending, d_n, n_max, n_ptiles, scores, &cache, s);
}

void launch_epoch_score_group(const MapView& map, const ScoreSlot* slots, size_t stride, uint32_t n_slots,
                              cudaStream_t s) {
  static std::atomic<uint64_t> attr_done{0};
  static std::mutex attr_mu;
  const int build_smem = kCacheHashSlots * 12 + kCacheAmbCap * 4;
  const int probe_smem = kStageWindowMax + kProbeItemBytes;  // any slot's window
  once_per_device(attr_done, attr_mu, [&] {
    BBS_CUDA(cudaFuncSetAttribute(cache_build_group, cudaFuncAttributeMaxDynamicSharedMemorySize, build_smem));
    BBS_CUDA(cudaFuncSetAttribute(cache_probe_group, cudaFuncAttributeMaxDynamicSharedMemorySize, probe_smem));
  });
  static const uint32_t hipw = [] {
    const char* v = std::getenv("BBS_PROBE_HIPW");
    return v ? static_cast<uint32_t>(std::max(1, std::atoi(v))) : 4u;
  }();
  launch_pdl(cache_build_group, dim3(per_slot(148 * 2, n_slots), n_slots), kBuildThreads, build_smem, s, map, slots,
             stride);
  BBS_CUDA(cudaGetLastError());
  const int per_sm = ctas_per_sm(cache_probe_group, kProbeThreads, probe_smem);
  launch_pdl(cache_probe_group, dim3(per_slot(148u * static_cast<unsigned>(per_sm), n_slots, 4), n_slots),
             kProbeThreads, probe_smem, s, map, slots, stride, hipw);
  BBS_CUDA(cudaGetLastError());
  launch_score_cube8_group(map, slots, stride, n_slots, s);
}

}  // namespace bbs

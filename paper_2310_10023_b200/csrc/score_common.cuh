// score_common.cuh — the bit-exact per-(node, point) arithmetic shared by
// every score kernel (score.cu, epoch_cache.cu).  See score.cu's header and
// DESIGN.md §3 for the exactness argument of fast_floor.
#pragma once

#include "device_common.cuh"
#include "kernels.h"

namespace bbs {

// pose_to_transform, geometry.hpp:107-109, on LUT cos/sin (geometry.hpp:103-105).
__device__ __forceinline__ void rotation_of(const GridView& G, int level, int ir, int ip, int iw,
                                            double R[9]) {
  const double2 a = G.lut[G.lut_off[level * 3 + 0] + (ir - G.lut_lo[level * 3 + 0])];
  const double2 b = G.lut[G.lut_off[level * 3 + 1] + (ip - G.lut_lo[level * 3 + 1])];
  const double2 g = G.lut[G.lut_off[level * 3 + 2] + (iw - G.lut_lo[level * 3 + 2])];
  const double ca = a.x, sa = a.y, cb = b.x, sb = b.y, cg = g.x, sg = g.y;
  R[0] = __dmul_rn(cg, cb);
  R[1] = __dsub_rn(__dmul_rn(__dmul_rn(cg, sb), sa), __dmul_rn(sg, ca));
  R[2] = __dadd_rn(__dmul_rn(__dmul_rn(cg, sb), ca), __dmul_rn(sg, sa));
  R[3] = __dmul_rn(sg, cb);
  R[4] = __dadd_rn(__dmul_rn(__dmul_rn(sg, sb), sa), __dmul_rn(cg, ca));
  R[5] = __dsub_rn(__dmul_rn(__dmul_rn(sg, sb), ca), __dmul_rn(cg, sa));
  R[6] = -sb;
  R[7] = __dmul_rn(cb, sa);
  R[8] = __dmul_rn(cb, ca);
}

// R*p in the reference's evaluation order (translation not yet added).
__device__ __forceinline__ double rot_row(double r0, double r1, double r2, double px, double py,
                                          double pz) {
  return __dadd_rn(__dadd_rn(__dmul_rn(r0, px), __dmul_rn(r1, py)), __dmul_rn(r2, pz));
}

// Fast-path voxel offset of one axis; returns false when ambiguous.
// tmax >= max |translation index| + 2 of every node that will use *f.
__device__ __forceinline__ bool fast_floor(double rp, double inv_cell, double tmax, int32_t* f) {
  const double w = __dmul_rn(rp, inv_cell);
  const double fl = floor(w);
  const double fr = __dsub_rn(w, fl);
  const double aw = fabs(w);
  const double eps = __dmul_rn(__dadd_rn(aw, tmax), 0x1p-48);
  const bool ok = (aw < 0x1p30) && (fr > eps) && (fr < __dsub_rn(1.0, eps));
  *f = ok ? static_cast<int32_t>(fl) : 0;
  return ok;
}

// Exact reference arithmetic for one (point, node): q = rp + cell*ix, then
// floor(q / cell) with x86 conversion semantics, then contains().
__device__ __forceinline__ int exact_hit(const LevelView& L, double rx, double ry, double rz,
                                         int32_t ix, int32_t iy, int32_t iz) {
  const int32_t vx = dev_voxel_index(__dadd_rn(rx, __dmul_rn(L.cell, static_cast<double>(ix))), L.cell);
  const int32_t vy = dev_voxel_index(__dadd_rn(ry, __dmul_rn(L.cell, static_cast<double>(iy))), L.cell);
  const int32_t vz = dev_voxel_index(__dadd_rn(rz, __dmul_rn(L.cell, static_cast<double>(iz))), L.cell);
  if (vx == INT32_MIN && vy == INT32_MIN && vz == INT32_MIN) return 0;  // kEmpty probe
  return level_contains(L, vx, vy, vz) ? 1 : 0;
}

// Counts of the 8 cube children (jx, jy, jz) = (t >> 2, (t >> 1) & 1, t & 1)
// for one voxel offset f = (ux, uy, z0) already relative to the level box,
// weighted by w, from the z-column bitmap: 4 column words.
__device__ __forceinline__ void cube_probe(const LevelView& L, uint32_t ux, uint32_t uy, uint32_t z0,
                                           int w, int acc[8]) {
  const uint32_t dimx = L.dim[0], dimy = L.dim[1], dimz = L.dim[2];
  const uint32_t plane = dimx * dimy;
  const uint32_t z1 = z0 + 1;
  const bool in0 = z0 < dimz, in1 = z1 < dimz, same = (z0 >> 5) == (z1 >> 5);
#pragma unroll
  for (int d = 0; d < 4; ++d) {
    const uint32_t x = ux + (d >> 1), y = uy + (d & 1);
    if (x < dimx && y < dimy) {
      const uint32_t col = y * dimx + x;
      const uint32_t w0 = in0 ? __ldg(&L.words[(z0 >> 5) * plane + col]) : 0u;
      const uint32_t w1 = in1 ? (same ? w0 : __ldg(&L.words[(z1 >> 5) * plane + col])) : 0u;
      acc[2 * d] += w & -static_cast<int>((w0 >> (z0 & 31)) & 1u);
      acc[2 * d + 1] += w & -static_cast<int>((w1 >> (z1 & 31)) & 1u);
    }
  }
}

// ---- per-search rotation cache (epoch_cache.cu) ----------------------------
__device__ __forceinline__ bool run_slot(const RotCache& c, const GridView& G, const int4& a,
                                         const int4& b, uint32_t* slot) {
  // a = (ix, iy, iz, iroll) of child 0, b = (ipitch, iyaw, level, score)
  const int l = b.z;
  const uint32_t base = c.base[l];
  if (base == 0xFFFFFFFFu) return false;
  const uint32_t np = static_cast<uint32_t>(G.max_index[l * 3 + 1]) + 1;
  const uint32_t nw = static_cast<uint32_t>(G.max_index[l * 3 + 2]) + 1;
  *slot = base + (static_cast<uint32_t>(a.w) * np + static_cast<uint32_t>(b.x)) * nw +
          static_cast<uint32_t>(b.y);
  return true;
}


// A run that can have no READY histogram this flush (the branch kernel runs
// before this flush's builds): uncached level, a level whose builds gave up,
// or a rotation whose build failed in an earlier flush.
__device__ __forceinline__ bool run_is_direct(const RotCache& c, const GridView& G, const int4& a, const int4& b) {
  uint32_t slot;
  if (!run_slot(c, G, a, b, &slot)) return true;
  const int32_t state = c.info[slot].x;
  if (state == kCacheNone) return true;
  return state == kCacheEmpty && c.ctl[4 + (b.z & (kMaxLevels - 1))] != 0u;
}

// Claim one run's (level, rotation) slot for a build in this flush (called
// by the branch kernel for the first child of every run).  a/b are the run's
// first child as int4 pairs: (ix, iy, iz, iroll), (ipitch, iyaw, level, score).
__device__ __forceinline__ void cache_claim_run(const RotCache& c, const GridView& G, const int4& a,
                                                const int4& b) {
  uint32_t slot;
  if (!run_slot(c, G, a, b, &slot)) return;  // uncached level: the cube kernel scores it
  if (c.info[slot].x != kCacheEmpty) return;
  // the level's offsets do not de-duplicate: a build would cost more than it
  // saves, the cube kernel scores the run directly
  if (c.ctl[4 + (b.z & (kMaxLevels - 1))]) return;
  if (atomicCAS(&c.info[slot].x, kCacheEmpty, kCacheBuilding) == kCacheEmpty) {
    const uint32_t i = atomicAdd(&c.ctl[2], 1u);
    c.builds[i] = make_int4(static_cast<int32_t>(slot), b.z, a.w, b.x);  // slot, level, ir, ip
    c.builds_w[i] = b.y;                                                 // iw
  }
}

// The 8 cube counts (children (jx, jy, jz) = (t >> 2, (t >> 1) & 1, t & 1)
// of the run at (bx, by, bz)) of scan point p under rotation R: fast path
// from the z-column bitmap (4 column loads), hash probes, or the exact
// divide path for an ambiguous point.
__device__ __forceinline__ void cube8_point(const LevelView& L, const double* R, double tmax, int32_t bx, int32_t by,
                                            int32_t bz, const ScanView& scan, uint32_t p, int cnt[8]) {
  const double px = scan.x[p], py = scan.y[p], pz = scan.z[p];
  const double rx = rot_row(R[0], R[1], R[2], px, py, pz);
  const double ry = rot_row(R[3], R[4], R[5], px, py, pz);
  const double rz = rot_row(R[6], R[7], R[8], px, py, pz);
  int32_t fx, fy, fz;
  const bool ok = fast_floor(rx, L.inv_cell, tmax, &fx) & fast_floor(ry, L.inv_cell, tmax, &fy) &
                  fast_floor(rz, L.inv_cell, tmax, &fz);
  if (ok && L.layout == BBS_LAYOUT_BITMAP) {
    const uint32_t dimx = L.dim[0], dimy = L.dim[1], dimz = L.dim[2];
    const uint64_t plane = static_cast<uint64_t>(dimx) * dimy;
    const uint32_t ux = static_cast<uint32_t>(fx) + static_cast<uint32_t>(bx) - static_cast<uint32_t>(L.box_min[0]);
    const uint32_t uy = static_cast<uint32_t>(fy) + static_cast<uint32_t>(by) - static_cast<uint32_t>(L.box_min[1]);
    const uint32_t z0 = static_cast<uint32_t>(fz) + static_cast<uint32_t>(bz) - static_cast<uint32_t>(L.box_min[2]);
    const uint32_t z1 = z0 + 1;
    const bool in0 = z0 < dimz, in1 = z1 < dimz;
    const bool same = (z0 >> 5) == (z1 >> 5);
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const uint32_t x = ux + (d >> 1), y = uy + (d & 1);
      if (x < dimx && y < dimy) {
        const uint64_t col = static_cast<uint64_t>(y) * dimx + x;
        const uint32_t w0 = in0 ? __ldg(&L.words[(z0 >> 5) * plane + col]) : 0u;
        const uint32_t w1 = in1 ? (same ? w0 : __ldg(&L.words[(z1 >> 5) * plane + col])) : 0u;
        cnt[2 * d] += (w0 >> (z0 & 31)) & 1u;
        cnt[2 * d + 1] += (w1 >> (z1 & 31)) & 1u;
      }
    }
  } else if (ok) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      cnt[t] += level_contains(L, fx + bx + (t >> 2), fy + by + ((t >> 1) & 1), fz + bz + (t & 1)) ? 1 : 0;
  } else {
#pragma unroll
    for (int t = 0; t < 8; ++t) cnt[t] += exact_hit(L, rx, ry, rz, bx + (t >> 2), by + ((t >> 1) & 1), bz + (t & 1));
  }
}

// One work item of the cube kernel: run `run` (8 children sharing a
// rotation, a 2x2x2 translation cube) over point tile `pt` of `n_ptiles`.
// Every thread of the CTA calls it; s_R / s_hdr / s_cnt are the caller's
// shared scratch.  Also the direct-run phase of the probe kernel.
template <bool kILP>
__device__ __forceinline__ void cube8_item(const MapView& map, const GridView& grid, const ScanView& scan,
                                           const bbs_node* __restrict__ nodes, uint32_t run, uint32_t pt,
                                           uint32_t n_ptiles, int32_t* __restrict__ scores, double* s_R,
                                           int32_t* s_hdr, int32_t* s_cnt) {
  const uint32_t k = scan.k;
  const uint32_t tile = (k + n_ptiles - 1) / n_ptiles;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    const int4 a = reinterpret_cast<const int4*>(nodes)[2 * (8ull * run)];
    const int4 b = reinterpret_cast<const int4*>(nodes)[2 * (8ull * run) + 1];
    double R[9];
    rotation_of(grid, b.z, a.w, b.x, b.y, R);
#pragma unroll
    for (int i = 0; i < 9; ++i) s_R[i] = R[i];
    s_hdr[0] = a.x;
    s_hdr[1] = a.y;
    s_hdr[2] = a.z;
    s_hdr[3] = b.z;
  }
  if (threadIdx.x < 8) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const int32_t bx = s_hdr[0], by = s_hdr[1], bz = s_hdr[2];
  const LevelView L = map.level[s_hdr[3]];
  double R[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) R[i] = s_R[i];
  const double tmax =
      static_cast<double>(max(max(abs(bx), abs(by)), abs(bz))) + 3.0;  // children: b + 1
  const bool bitmap = L.layout == BBS_LAYOUT_BITMAP;
  const uint32_t dimx = L.dim[0], dimy = L.dim[1], dimz = L.dim[2];
  const uint32_t ox = static_cast<uint32_t>(bx) - static_cast<uint32_t>(L.box_min[0]);
  const uint32_t oy = static_cast<uint32_t>(by) - static_cast<uint32_t>(L.box_min[1]);
  const uint32_t oz = static_cast<uint32_t>(bz) - static_cast<uint32_t>(L.box_min[2]);
  const uint64_t plane = static_cast<uint64_t>(dimx) * dimy;
  int cnt[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) cnt[t] = 0;
  const uint32_t p0 = pt * tile, p1 = min(k, p0 + tile);
  // long tiles: two points per thread per step (both points' coordinates,
  // then both rotations, then all their column-word loads in flight);
  // short tiles (small scans, many point tiles): one point per step
  if (!kILP || p1 - p0 < 2 * blockDim.x) {
    for (uint32_t p = p0 + threadIdx.x; p < p1; p += blockDim.x)
      cube8_point(L, R, tmax, bx, by, bz, scan, p, cnt);
  } else
  for (uint32_t pb = p0 + threadIdx.x; kILP && pb < p1; pb += 2 * blockDim.x) {
    double px[2], py[2], pz[2];
    bool live[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t p = pb + h * blockDim.x;
      live[h] = p < p1;
      px[h] = live[h] ? scan.x[p] : 0.0;
      py[h] = live[h] ? scan.y[p] : 0.0;
      pz[h] = live[h] ? scan.z[p] : 0.0;
    }
    double rx[2], ry[2], rz[2];
    int32_t fx[2], fy[2], fz[2];
    bool fast[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      rx[h] = rot_row(R[0], R[1], R[2], px[h], py[h], pz[h]);
      ry[h] = rot_row(R[3], R[4], R[5], px[h], py[h], pz[h]);
      rz[h] = rot_row(R[6], R[7], R[8], px[h], py[h], pz[h]);
      fast[h] = fast_floor(rx[h], L.inv_cell, tmax, &fx[h]) & fast_floor(ry[h], L.inv_cell, tmax, &fy[h]) &
                fast_floor(rz[h], L.inv_cell, tmax, &fz[h]);
    }
    if (bitmap) {
      uint32_t w[2][8];
      uint32_t zz[2][2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const bool use = live[h] && fast[h];
        const uint32_t ux = static_cast<uint32_t>(fx[h]) + ox;
        const uint32_t uy = static_cast<uint32_t>(fy[h]) + oy;
        const uint32_t z0 = static_cast<uint32_t>(fz[h]) + oz, z1 = z0 + 1;
        zz[h][0] = z0;
        zz[h][1] = z1;
        const bool in0 = use && z0 < dimz, in1 = use && z1 < dimz;
        const bool same = (z0 >> 5) == (z1 >> 5);
#pragma unroll
        for (int d = 0; d < 4; ++d) {
          const uint32_t x = ux + (d >> 1), y = uy + (d & 1);
          const bool inxy = x < dimx && y < dimy;
          const uint64_t col = static_cast<uint64_t>(y) * dimx + x;
          w[h][2 * d] = (in0 && inxy) ? __ldg(&L.words[(z0 >> 5) * plane + col]) : 0u;
          w[h][2 * d + 1] = (in1 && inxy && !same) ? __ldg(&L.words[(z1 >> 5) * plane + col]) : 0u;
        }
        // same z word: reuse the first load
#pragma unroll
        for (int d = 0; d < 4; ++d)
          if (same) w[h][2 * d + 1] = in1 ? w[h][2 * d] : 0u;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int d = 0; d < 4; ++d) {
          cnt[2 * d] += (w[h][2 * d] >> (zz[h][0] & 31)) & 1u;
          cnt[2 * d + 1] += (w[h][2 * d + 1] >> (zz[h][1] & 31)) & 1u;
        }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (!live[h] || (bitmap && fast[h])) continue;
      if (fast[h]) {
#pragma unroll
        for (int t = 0; t < 8; ++t)
          cnt[t] += level_contains(L, fx[h] + bx + (t >> 2), fy[h] + by + ((t >> 1) & 1), fz[h] + bz + (t & 1)) ? 1
                                                                                                              : 0;
      } else {
#pragma unroll
        for (int t = 0; t < 8; ++t)
          cnt[t] += exact_hit(L, rx[h], ry[h], rz[h], bx + (t >> 2), by + ((t >> 1) & 1), bz + (t & 1));
      }
    }
  }
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int v = __reduce_add_sync(0xffffffffu, cnt[t]);
    if (lane == 0 && v) atomicAdd(&s_cnt[t], v);
  }
  __syncthreads();
  if (threadIdx.x < 8) {
    const uint64_t idx = 8ull * run + threadIdx.x;
    if (n_ptiles == 1)
      scores[idx] = s_cnt[threadIdx.x];
    else if (s_cnt[threadIdx.x])
      atomicAdd(&scores[idx], s_cnt[threadIdx.x]);
  }
  __syncthreads();
}

}  // namespace bbs

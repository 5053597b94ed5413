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

}  // namespace bbs

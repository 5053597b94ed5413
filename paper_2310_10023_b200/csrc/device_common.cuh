// device_common.cuh — device helpers shared by the map build, score and
// frontier kernels.  Everything here is sm_100a device code; the .cu files
// are compiled with --fmad=false and use explicit _rn intrinsics on the
// bit-exact path, so no FMA contraction can change a rounding
// (SURVEY §7 "Bit-exact FP64 hit counts").
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "bbs_internal.h"

namespace bbs {

// voxel_index, point_cloud.hpp:38-40: (int32)floor(c / cell) with IEEE
// division; the reference's x86 cvttsd2si gives INT32_MIN for NaN and values
// outside [-2^31, 2^31), which cvt.rzi.s32.f64 would saturate instead.
__device__ __forceinline__ int32_t dev_voxel_index(double c, double cell) {
  const double f = floor(__ddiv_rn(c, cell));
  return (f >= -2147483648.0 && f < 2147483648.0) ? static_cast<int32_t>(f) : INT32_MIN;
}

__device__ __forceinline__ uint64_t hash_bucket(unsigned long long key, uint32_t shift) {
  // multiplicative (Fibonacci) hashing on the packed key
  return (key * 0x9E3779B97F4A7C15ull) >> shift;
}

__device__ __forceinline__ unsigned long long pack_key(uint32_t ux, uint32_t uy, uint32_t uz,
                                                       uint32_t by, uint32_t bz) {
  return (static_cast<unsigned long long>(ux) << (by + bz)) |
         (static_cast<unsigned long long>(uy) << bz) | static_cast<unsigned long long>(uz);
}

// Bitmap addressing (z-column major).
__device__ __forceinline__ uint64_t bitmap_word(const LevelView& L, uint32_t ux, uint32_t uy,
                                                uint32_t uz) {
  return (static_cast<uint64_t>(uz >> 5) * L.dim[1] + uy) * L.dim[0] + ux;
}
__device__ __forceinline__ uint32_t bitmap_bit(uint32_t uz) { return uz & 31u; }

// LevelMap::contains, voxel_map.hpp:127-135 — set membership on the
// device layout.  Voxels outside the level's box are misses without a load.
__device__ __forceinline__ bool level_contains(const LevelView& L, int32_t x, int32_t y,
                                               int32_t z) {
  const uint32_t ux = static_cast<uint32_t>(x) - static_cast<uint32_t>(L.box_min[0]);
  const uint32_t uy = static_cast<uint32_t>(y) - static_cast<uint32_t>(L.box_min[1]);
  const uint32_t uz = static_cast<uint32_t>(z) - static_cast<uint32_t>(L.box_min[2]);
  if (ux >= L.dim[0] || uy >= L.dim[1] || uz >= L.dim[2]) return false;
  if (L.layout == BBS_LAYOUT_BITMAP) {
    const uint32_t w = __ldg(&L.words[bitmap_word(L, ux, uy, uz)]);
    return (w >> bitmap_bit(uz)) & 1u;
  }
  const unsigned long long key = pack_key(ux, uy, uz, L.bits_y, L.bits_z);
  uint64_t b = hash_bucket(key, L.bucket_shift);
  for (;;) {
    // one 32-byte sector per bucket; inserts fill a bucket's slots in order,
    // so an empty last slot ends the probe sequence
    const ulonglong2* p = reinterpret_cast<const ulonglong2*>(L.slots + 4 * b);
    const ulonglong2 s0 = __ldg(p);
    const ulonglong2 s1 = __ldg(p + 1);
    if (s0.x == key || s0.y == key || s1.x == key || s1.y == key) return true;
    if (s1.y == ~0ull) return false;
    b = (b + 1) & L.bucket_mask;
  }
}

// 32-bit load from a shared-memory byte address (ld.shared, no generic
// address conversion)
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// Programmatic dependent launch (launch_pdl): wait for the preceding grid
// (complete, memory visible) before reading its output; let the next grid
// launch once every CTA of this one has started.  No-ops without PDL.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// One-shot TMA bulk copy global -> shared (1D, bytes % 16 == 0, both
// addresses 16-byte aligned) completing on an mbarrier, in two halves:
// thread 0 initialises the barrier and issues (a __syncthreads must follow
// before anyone polls), then any thread may wait for the bytes.
__device__ __forceinline__ void bulk_issue(void* dst, const void* src, uint32_t bytes, unsigned long long* mbar) {
  const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(mbar));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src), "r"(bytes), "r"(b)
                 : "memory");
  }
}
__device__ __forceinline__ void bulk_wait(unsigned long long* mbar) {
  const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(mbar));
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "BBS_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
      "@!p bra BBS_WAIT_%=;\n"
      "}\n" ::"r"(b)
      : "memory");
}

}  // namespace bbs

// map_build.cu — K1-K3: the hierarchical voxel map built on the device.
//
// Replaces MultiResVoxelMap::build / build_level / inflated_voxels /
// LevelMap::from_voxels (voxel_map.hpp:72-116, :186-261).  Per level:
//   K1 voxelize every map point at ldexp(r, l) (exact IEEE division,
//      x86 conversion semantics) and reduce the voxel box;
//   K2 pack voxels into 64-bit x-major keys, radix sort + unique (CUB),
//      inflate each source voxel v into v - j, j in {0,1}^3, sort + unique;
//   K3 materialise the set as a dense bitmap (8x8x4 bricks, one 32 B sector
//      each) or an open-addressing table of packed keys (4-key buckets).
// The sorted unique key list is kept on the device: it IS the reference's
// canonical occupied_voxels() order (voxel_map.hpp:158-165).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <limits>

#include "bbs_map_impl.h"
#include "device_common.cuh"

namespace bbs {

[[noreturn]] void throw_cuda(const char* what, int err, const char* file, int line) {
  char buf[512];
  std::snprintf(buf, sizeof(buf), "CUDA error %d (%s) in %s at %s:%d", err,
                cudaGetErrorString(static_cast<cudaError_t>(err)), what, file, line);
  throw Error(BBS_ERR_CUDA, buf);
}

DeviceGuard::DeviceGuard(int dev) {
  BBS_CUDA(cudaGetDevice(&prev));
  if (prev != dev) BBS_CUDA(cudaSetDevice(dev));
}
DeviceGuard::~DeviceGuard() { cudaSetDevice(prev); }

namespace {

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DevBuf(size_t count, cudaStream_t st) : n(count), s(st) {
    if (count) BBS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), st));
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, s);
  }
  T* release() {
    T* r = p;
    p = nullptr;
    return r;
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

constexpr int kThreads = 256;

unsigned grid_for(uint64_t n, int threads = kThreads) {
  const uint64_t g = (n + threads - 1) / threads;
  return static_cast<unsigned>(std::min<uint64_t>(std::max<uint64_t>(g, 1), 148ull * 64));
}

// K1: voxel index of every point + box reduction (min, max per axis).
__global__ void voxelize_kernel(const double* __restrict__ xyz, uint64_t n, double cell,
                                int32_t* __restrict__ vox, int32_t* __restrict__ minmax) {
  int32_t mn[3] = {INT32_MAX, INT32_MAX, INT32_MAX};
  int32_t mx[3] = {INT32_MIN, INT32_MIN, INT32_MIN};
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int32_t v = dev_voxel_index(xyz[3 * i + a], cell);
      vox[3 * i + a] = v;
      mn[a] = min(mn[a], v);
      mx[a] = max(mx[a], v);
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn[a] = min(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
      mx[a] = max(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
    }
  }
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      atomicMin(&minmax[a], mn[a]);
      atomicMax(&minmax[3 + a], mx[a]);
    }
  }
}

// Box of AoS int32 voxel triples (min, max per axis).
__global__ void voxel_box_kernel(const int32_t* __restrict__ vox, uint64_t n, int32_t* __restrict__ minmax) {
  int32_t mn[3] = {INT32_MAX, INT32_MAX, INT32_MAX};
  int32_t mx[3] = {INT32_MIN, INT32_MIN, INT32_MIN};
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int32_t v = vox[3 * i + a];
      mn[a] = min(mn[a], v);
      mx[a] = max(mx[a], v);
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn[a] = min(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
      mx[a] = max(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
    }
  }
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      atomicMin(&minmax[a], mn[a]);
      atomicMax(&minmax[3 + a], mx[a]);
    }
  }
}

// Voxel triples (AoS int32) -> packed keys relative to box_min.
__global__ void pack_kernel(const int32_t* __restrict__ vox, uint64_t n, int3 box_min,
                            uint32_t by, uint32_t bz, unsigned long long* __restrict__ keys) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t ux = static_cast<uint32_t>(vox[3 * i]) - static_cast<uint32_t>(box_min.x);
    const uint32_t uy = static_cast<uint32_t>(vox[3 * i + 1]) - static_cast<uint32_t>(box_min.y);
    const uint32_t uz = static_cast<uint32_t>(vox[3 * i + 2]) - static_cast<uint32_t>(box_min.z);
    keys[i] = pack_key(ux, uy, uz, by, bz);
  }
}

// inflated_voxels, voxel_map.hpp:197-202: v - j, j in {0,1}^3.  Source keys
// are >= 1 per axis (box_min = min - 1), so no underflow.
__global__ void inflate_kernel(const unsigned long long* __restrict__ src, uint64_t n,
                               uint32_t by, uint32_t bz, unsigned long long* __restrict__ out) {
  const unsigned long long my = (1ull << by) - 1, mz = (1ull << bz) - 1;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const unsigned long long k = src[i];
    const uint32_t ux = static_cast<uint32_t>(k >> (by + bz));
    const uint32_t uy = static_cast<uint32_t>((k >> bz) & my);
    const uint32_t uz = static_cast<uint32_t>(k & mz);
#pragma unroll
    for (uint32_t j = 0; j < 8; ++j)
      out[8 * i + j] = pack_key(ux - (j >> 2), uy - ((j >> 1) & 1u), uz - (j & 1u), by, bz);
  }
}

__global__ void bitmap_set_kernel(const unsigned long long* __restrict__ keys, uint64_t n,
                                  LevelView L, uint32_t* __restrict__ words) {
  const unsigned long long my = (1ull << L.bits_y) - 1, mz = (1ull << L.bits_z) - 1;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const unsigned long long k = keys[i];
    const uint32_t ux = static_cast<uint32_t>(k >> (L.bits_y + L.bits_z));
    const uint32_t uy = static_cast<uint32_t>((k >> L.bits_z) & my);
    const uint32_t uz = static_cast<uint32_t>(k & mz);
    atomicOr(&words[bitmap_word(L, ux, uy, uz)], 1u << bitmap_bit(uz));
  }
}

__global__ void hash_insert_kernel(const unsigned long long* __restrict__ keys, uint64_t n,
                                   LevelView L, unsigned long long* __restrict__ slots) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const unsigned long long k = keys[i];
    uint64_t b = hash_bucket(k, L.bucket_shift);
    for (;;) {
      bool done = false;
      for (int s = 0; s < 4; ++s) {
        const unsigned long long prev = atomicCAS(&slots[4 * b + s], ~0ull, k);
        if (prev == ~0ull || prev == k) {
          done = true;
          break;
        }
      }
      if (done) break;
      b = (b + 1) & L.bucket_mask;
    }
  }
}

__global__ void unpack_kernel(const unsigned long long* __restrict__ keys, uint64_t n,
                              int3 box_min, uint32_t by, uint32_t bz, int32_t* __restrict__ xyz) {
  const unsigned long long my = (1ull << by) - 1, mz = (1ull << bz) - 1;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const unsigned long long k = keys[i];
    xyz[3 * i] = static_cast<int32_t>(static_cast<uint32_t>(k >> (by + bz)) +
                                      static_cast<uint32_t>(box_min.x));
    xyz[3 * i + 1] = static_cast<int32_t>(static_cast<uint32_t>((k >> bz) & my) +
                                          static_cast<uint32_t>(box_min.y));
    xyz[3 * i + 2] =
        static_cast<int32_t>(static_cast<uint32_t>(k & mz) + static_cast<uint32_t>(box_min.z));
  }
}

__global__ void contains_kernel(LevelView L, const int32_t* __restrict__ xyz, uint64_t n,
                                uint8_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const int32_t x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
    // contains(kEmpty) is false (voxel_map.hpp:131)
    const bool empty = x == INT32_MIN && y == INT32_MIN && z == INT32_MIN;
    out[i] = (!empty && level_contains(L, x, y, z)) ? 1 : 0;
  }
}

// LevelMap::score, voxel_map.hpp:142-154, for one arbitrary Transform.
__global__ void score_transform_kernel(LevelView L, const double* __restrict__ R,
                                       const double* __restrict__ t,
                                       const double* __restrict__ scan, uint64_t k,
                                       int32_t* __restrict__ out) {
  int hits = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < k;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const double px = scan[3 * i], py = scan[3 * i + 1], pz = scan[3 * i + 2];
    const double qx =
        __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(R[0], px), __dmul_rn(R[1], py)),
                            __dmul_rn(R[2], pz)), t[0]);
    const double qy =
        __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(R[3], px), __dmul_rn(R[4], py)),
                            __dmul_rn(R[5], pz)), t[1]);
    const double qz =
        __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(R[6], px), __dmul_rn(R[7], py)),
                            __dmul_rn(R[8], pz)), t[2]);
    const int32_t vx = dev_voxel_index(qx, L.cell), vy = dev_voxel_index(qy, L.cell),
                  vz = dev_voxel_index(qz, L.cell);
    const bool empty = vx == INT32_MIN && vy == INT32_MIN && vz == INT32_MIN;
    hits += (!empty && level_contains(L, vx, vy, vz)) ? 1 : 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) hits += __shfl_xor_sync(0xffffffffu, hits, o);
  if ((threadIdx.x & 31) == 0 && hits) atomicAdd(out, hits);
}

uint32_t bits_for(uint64_t dim) {
  uint32_t b = 1;
  while ((1ull << b) < dim) ++b;
  return b;
}

// Sort + unique `n` keys in place (end_bit significant bits); returns count.
uint64_t sort_unique(unsigned long long*& keys, uint64_t n, int end_bit, cudaStream_t s) {
  if (n == 0) return 0;
  DevBuf<unsigned long long> alt(n, s);
  DevBuf<int64_t> d_count(1, s);
  cub::DoubleBuffer<unsigned long long> db(keys, alt.p);
  size_t temp_sort = 0, temp_uniq = 0;
  BBS_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, temp_sort, db, static_cast<int64_t>(n), 0,
                                          end_bit, s));
  BBS_CUDA(cub::DeviceSelect::Unique(nullptr, temp_uniq, keys, alt.p, d_count.p,
                                     static_cast<int64_t>(n), s));
  DevBuf<unsigned char> temp(std::max(temp_sort, temp_uniq), s);
  BBS_CUDA(cub::DeviceRadixSort::SortKeys(temp.p, temp_sort, db, static_cast<int64_t>(n), 0,
                                          end_bit, s));
  unsigned long long* sorted = db.Current();
  unsigned long long* other = (sorted == keys) ? alt.p : keys;
  BBS_CUDA(cub::DeviceSelect::Unique(temp.p, temp_uniq, sorted, other, d_count.p,
                                     static_cast<int64_t>(n), s));
  int64_t cnt = 0;
  BBS_CUDA(cudaMemcpyAsync(&cnt, d_count.p, sizeof(cnt), cudaMemcpyDeviceToHost, s));
  BBS_CUDA(cudaStreamSynchronize(s));
  // result lives in `other`; hand that buffer back as `keys`
  if (other == alt.p) {
    alt.release();
    cudaFreeAsync(keys, s);
    keys = other;
  }
  return static_cast<uint64_t>(cnt);
}

uint64_t next_pow2(uint64_t v) {
  uint64_t p = 1;
  while (p < v) p <<= 1;
  return p;
}

// Choose and build the device structure for a level from its sorted unique
// keys (K3).  box_min/dims describe the voxel box the keys are relative to.
void finish_level(bbs_map* m, int level, unsigned long long* keys, uint64_t n, const int64_t* bmin,
                  const uint64_t* dims, const uint32_t* bits, int layout_pref) {
  bbs_map::Level& L = m->levels[static_cast<size_t>(level)];
  L.keys = keys;
  L.n_keys = n;
  for (int a = 0; a < 3; ++a) L.bits[a] = bits[a];
  LevelView& V = m->view.level[level];
  std::memset(&V, 0, sizeof(V));
  V.cell = std::ldexp(m->r, level);
  V.inv_cell = 1.0 / V.cell;
  V.bits_y = bits[1];
  V.bits_z = bits[2];
  for (int a = 0; a < 3; ++a) {
    V.box_min[a] = static_cast<int32_t>(bmin[a]);
    V.dim[a] = static_cast<uint32_t>(dims[a]);
  }
  V.nwz = static_cast<uint32_t>((dims[2] + 31) / 32);

  const uint64_t nwords = dims[0] * dims[1] * V.nwz;
  const bool bitmap_ok = nwords < (1ull << 32);  // 32-bit word indices in the kernels
  const uint64_t bitmap_bytes = bitmap_ok ? nwords * 4ull : ~0ull;
  const uint64_t slots = std::max<uint64_t>(8, next_pow2(2 * n));
  const uint64_t hash_bytes = slots * 8ull;

  int layout = layout_pref;
  if (layout == BBS_LAYOUT_AUTO)
    layout = (bitmap_ok && bitmap_bytes <= 2 * hash_bytes) ? BBS_LAYOUT_BITMAP : BBS_LAYOUT_HASH;
  if (layout == BBS_LAYOUT_BITMAP && !bitmap_ok)
    throw Error(BBS_ERR_CAPACITY_EXCEEDED,
                "level " + std::to_string(level) + ": voxel box too large for a bitmap");
  uint64_t bytes = layout == BBS_LAYOUT_BITMAP ? bitmap_bytes : hash_bytes;
  if (bytes > m->memory_cap && layout_pref == BBS_LAYOUT_AUTO) {
    const int other = layout == BBS_LAYOUT_BITMAP ? BBS_LAYOUT_HASH : BBS_LAYOUT_BITMAP;
    const uint64_t ob = other == BBS_LAYOUT_BITMAP ? bitmap_bytes : hash_bytes;
    if (ob <= m->memory_cap) {
      layout = other;
      bytes = ob;
    }
  }
  const uint64_t buckets = layout == BBS_LAYOUT_BITMAP ? nwords * 32ull : slots;
  if (bytes > m->memory_cap)  // voxel_map.hpp:91-95 (same message form)
    throw Error(BBS_ERR_CAPACITY_EXCEEDED,
                "level " + std::to_string(level) + ": bucket table of " + std::to_string(buckets) +
                    " slots exceeds memory cap of " + std::to_string(m->memory_cap) + " bytes");
  V.layout = layout;
  cudaStream_t s = m->stream;
  if (n == 0) {
    V.dim[0] = V.dim[1] = V.dim[2] = 0;  // every probe misses
  } else if (layout == BBS_LAYOUT_BITMAP) {
    uint32_t* words = nullptr;
    BBS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&words), bytes, s));
    BBS_CUDA(cudaMemsetAsync(words, 0, bytes, s));
    V.words = words;
    L.structure = words;
    bitmap_set_kernel<<<grid_for(n), kThreads, 0, s>>>(keys, n, V, words);
    BBS_CUDA(cudaGetLastError());
  } else {
    unsigned long long* sl = nullptr;
    BBS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&sl), bytes, s));
    BBS_CUDA(cudaMemsetAsync(sl, 0xFF, bytes, s));
    const uint64_t nb = slots / 4;
    uint32_t lg = 0;
    while ((1ull << lg) < nb) ++lg;
    V.bucket_mask = nb - 1;
    V.bucket_shift = 64 - lg;
    V.slots = sl;
    L.structure = sl;
    hash_insert_kernel<<<grid_for(n), kThreads, 0, s>>>(keys, n, V, sl);
    BBS_CUDA(cudaGetLastError());
  }
  bbs_level_info& I = L.info;
  I.level = level;
  I.layout = layout;
  I.resolution = V.cell;
  I.occupied_count = n;
  I.bucket_count = buckets;
  I.collision_rate = 0.0;
  I.load_factor = buckets ? static_cast<double>(n) / static_cast<double>(buckets) : 0.0;
  I.bytes = n ? bytes : 0;
  for (int a = 0; a < 3; ++a) {
    I.box_min[a] = V.box_min[a];
    I.box_max[a] = static_cast<int32_t>(bmin[a] + static_cast<int64_t>(dims[a]) - 1);
  }
}

void check_box(int level, const int64_t* lo, const int64_t* hi, uint64_t* dims, uint32_t* bits) {
  uint32_t total = 0;
  for (int a = 0; a < 3; ++a) {
    dims[a] = static_cast<uint64_t>(hi[a] - lo[a] + 1);
    if (lo[a] < INT32_MIN || hi[a] > INT32_MAX || dims[a] >= (1ull << 31))
      throw Error(BBS_ERR_CAPACITY_EXCEEDED,
                  "level " + std::to_string(level) + ": voxel box exceeds 2^31 voxels per axis");
    bits[a] = bits_for(dims[a]);
    total += bits[a];
  }
  if (total > 63)
    throw Error(BBS_ERR_CAPACITY_EXCEEDED,
                "level " + std::to_string(level) + ": voxel box needs " + std::to_string(total) +
                    " key bits (> 63)");
}

}  // namespace

void build_map_from_points(bbs_map* m, const double* xyz, uint64_t n) {
  DeviceGuard g(m->device);
  cudaStream_t s = m->stream;
  cudaEvent_t e0, e1;
  BBS_CUDA(cudaEventCreate(&e0));
  BBS_CUDA(cudaEventCreate(&e1));
  BBS_CUDA(cudaEventRecord(e0, s));
  DevBuf<double> d_xyz(3 * n, s);
  BBS_CUDA(cudaMemcpyAsync(d_xyz.p, xyz, 3 * n * sizeof(double), cudaMemcpyHostToDevice, s));
  DevBuf<int32_t> d_vox(3 * n, s);
  DevBuf<int32_t> d_mm(6, s);
  m->levels.assign(static_cast<size_t>(m->max_level) + 1, bbs_map::Level{});
  m->view.n_levels = m->max_level + 1;
  m->view.r = m->r;
  for (int l = 0; l <= m->max_level; ++l) {
    const double cell = std::ldexp(m->r, l);
    const int32_t init[6] = {INT32_MAX, INT32_MAX, INT32_MAX, INT32_MIN, INT32_MIN, INT32_MIN};
    BBS_CUDA(cudaMemcpyAsync(d_mm.p, init, sizeof(init), cudaMemcpyHostToDevice, s));
    voxelize_kernel<<<grid_for(n), kThreads, 0, s>>>(d_xyz.p, n, cell, d_vox.p, d_mm.p);
    BBS_CUDA(cudaGetLastError());
    int32_t mm[6];
    BBS_CUDA(cudaMemcpyAsync(mm, d_mm.p, sizeof(mm), cudaMemcpyDeviceToHost, s));
    BBS_CUDA(cudaStreamSynchronize(s));
    // inflated box: [min - 1, max] per axis (voxel_map.hpp:197-202)
    int64_t lo[3], hi[3];
    uint64_t dims[3];
    uint32_t bits[3];
    for (int a = 0; a < 3; ++a) {
      lo[a] = static_cast<int64_t>(mm[a]) - 1;
      hi[a] = mm[3 + a];
    }
    check_box(l, lo, hi, dims, bits);
    const int3 bmin = make_int3(static_cast<int32_t>(lo[0]), static_cast<int32_t>(lo[1]),
                                static_cast<int32_t>(lo[2]));
    const int end_bit = static_cast<int>(bits[0] + bits[1] + bits[2]);
    unsigned long long* src = nullptr;
    BBS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&src), n * sizeof(unsigned long long), s));
    pack_kernel<<<grid_for(n), kThreads, 0, s>>>(d_vox.p, n, bmin, bits[1], bits[2], src);
    BBS_CUDA(cudaGetLastError());
    const uint64_t ns = sort_unique(src, n, end_bit, s);
    unsigned long long* inf = nullptr;
    BBS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&inf), 8 * ns * sizeof(unsigned long long), s));
    inflate_kernel<<<grid_for(ns), kThreads, 0, s>>>(src, ns, bits[1], bits[2], inf);
    BBS_CUDA(cudaGetLastError());
    BBS_CUDA(cudaFreeAsync(src, s));
    const uint64_t nu = sort_unique(inf, 8 * ns, end_bit, s);
    finish_level(m, l, inf, nu, lo, dims, bits, m->layout_pref);
  }
  BBS_CUDA(cudaEventRecord(e1, s));
  BBS_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  BBS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  m->build_ms = ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

// One level from n voxel triples already in device memory (LevelMap::from_voxels,
// voxel_map.hpp:72-116: duplicates collapse, membership is the set).
void build_level_from_device_voxels(bbs_map* m, int l, const int32_t* d_vox, uint64_t n) {
  cudaStream_t s = m->stream;
  int64_t lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  uint64_t dims[3] = {1, 1, 1};
  uint32_t bits[3] = {1, 1, 1};
  unsigned long long* keys = nullptr;
  uint64_t nu = 0;
  if (n) {
    DevBuf<int32_t> d_mm(6, s);
    const int32_t init[6] = {INT32_MAX, INT32_MAX, INT32_MAX, INT32_MIN, INT32_MIN, INT32_MIN};
    BBS_CUDA(cudaMemcpyAsync(d_mm.p, init, sizeof(init), cudaMemcpyHostToDevice, s));
    voxel_box_kernel<<<grid_for(n), kThreads, 0, s>>>(d_vox, n, d_mm.p);
    BBS_CUDA(cudaGetLastError());
    int32_t mm[6];
    BBS_CUDA(cudaMemcpyAsync(mm, d_mm.p, sizeof(mm), cudaMemcpyDeviceToHost, s));
    BBS_CUDA(cudaStreamSynchronize(s));
    for (int a = 0; a < 3; ++a) {
      lo[a] = mm[a];
      hi[a] = mm[3 + a];
    }
    check_box(l, lo, hi, dims, bits);
    BBS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&keys), n * sizeof(unsigned long long), s));
    const int3 bmin = make_int3(static_cast<int32_t>(lo[0]), static_cast<int32_t>(lo[1]),
                                static_cast<int32_t>(lo[2]));
    pack_kernel<<<grid_for(n), kThreads, 0, s>>>(d_vox, n, bmin, bits[1], bits[2], keys);
    BBS_CUDA(cudaGetLastError());
    nu = sort_unique(keys, n, static_cast<int>(bits[0] + bits[1] + bits[2]), s);
  }
  finish_level(m, l, keys, nu, lo, dims, bits, m->layout_pref);
}

void begin_levels(bbs_map* m, int n_levels) {
  m->levels.assign(static_cast<size_t>(n_levels), bbs_map::Level{});
  m->view.n_levels = n_levels;
  m->view.r = m->r;
}

void build_map_from_levels(bbs_map* m, const int32_t* const* lv, const uint64_t* counts,
                           int n_levels) {
  DeviceGuard g(m->device);
  cudaStream_t s = m->stream;
  begin_levels(m, n_levels);
  for (int l = 0; l < n_levels; ++l) {
    const uint64_t n = counts[l];
    DevBuf<int32_t> d_vox(3 * std::max<uint64_t>(n, 1), s);
    if (n) BBS_CUDA(cudaMemcpyAsync(d_vox.p, lv[l], 3 * n * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    build_level_from_device_voxels(m, l, d_vox.p, n);
  }
  BBS_CUDA(cudaStreamSynchronize(s));
}

void level_occupied(bbs_map* m, int level, int32_t* xyz, uint64_t cap, uint64_t* count) {
  DeviceGuard g(m->device);
  const bbs_map::Level& L = m->levels[static_cast<size_t>(level)];
  *count = L.n_keys;
  const uint64_t n = std::min<uint64_t>(cap, L.n_keys);
  if (!n || !xyz) return;
  cudaStream_t s = m->stream;
  DevBuf<int32_t> out(3 * n, s);
  const LevelView& V = m->view.level[level];
  unpack_kernel<<<grid_for(n), kThreads, 0, s>>>(
      L.keys, n, make_int3(V.box_min[0], V.box_min[1], V.box_min[2]), L.bits[1], L.bits[2], out.p);
  BBS_CUDA(cudaGetLastError());
  BBS_CUDA(cudaMemcpyAsync(xyz, out.p, 3 * n * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  BBS_CUDA(cudaStreamSynchronize(s));
}

void level_contains(bbs_map* m, int level, const int32_t* xyz, uint64_t n, uint8_t* out) {
  DeviceGuard g(m->device);
  if (!n) return;
  cudaStream_t s = m->stream;
  DevBuf<int32_t> d_in(3 * n, s);
  DevBuf<uint8_t> d_out(n, s);
  BBS_CUDA(cudaMemcpyAsync(d_in.p, xyz, 3 * n * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  contains_kernel<<<grid_for(n), kThreads, 0, s>>>(m->view.level[level], d_in.p, n, d_out.p);
  BBS_CUDA(cudaGetLastError());
  BBS_CUDA(cudaMemcpyAsync(out, d_out.p, n, cudaMemcpyDeviceToHost, s));
  BBS_CUDA(cudaStreamSynchronize(s));
}

void level_score_transform(bbs_map* m, int level, const double* R, const double* t,
                           const double* scan, uint64_t k, int32_t* score) {
  DeviceGuard g(m->device);
  cudaStream_t s = m->stream;
  DevBuf<double> d_rt(12, s);
  DevBuf<double> d_scan(3 * std::max<uint64_t>(k, 1), s);
  DevBuf<int32_t> d_out(1, s);
  double rt[12];
  std::memcpy(rt, R, 9 * sizeof(double));
  std::memcpy(rt + 9, t, 3 * sizeof(double));
  BBS_CUDA(cudaMemcpyAsync(d_rt.p, rt, sizeof(rt), cudaMemcpyHostToDevice, s));
  if (k) BBS_CUDA(cudaMemcpyAsync(d_scan.p, scan, 3 * k * sizeof(double), cudaMemcpyHostToDevice, s));
  BBS_CUDA(cudaMemsetAsync(d_out.p, 0, sizeof(int32_t), s));
  if (k) {
    score_transform_kernel<<<grid_for(k), kThreads, 0, s>>>(m->view.level[level], d_rt.p,
                                                            d_rt.p + 9, d_scan.p, k, d_out.p);
    BBS_CUDA(cudaGetLastError());
  }
  BBS_CUDA(cudaMemcpyAsync(score, d_out.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  BBS_CUDA(cudaStreamSynchronize(s));
}

}  // namespace bbs

bbs_map::~bbs_map() {
  if (device >= 0) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    for (auto* w : ws_pool) bbs::free_workspace(w);
    for (auto& L : levels) {
      if (L.keys) cudaFree(L.keys);
      if (L.structure) cudaFree(L.structure);
    }
    if (own_stream) cudaStreamDestroy(own_stream);
    cudaSetDevice(prev);
  }
}

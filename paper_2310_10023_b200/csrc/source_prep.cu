// source_prep.cu — prepare_source on the device:
// auto_leaf + voxel_grid_downsample (point_cloud.hpp:78-182) and
// max_range (point_cloud.hpp:58-63), pipeline.hpp:25-41.
//
// * count_voxels(leaf) (point_cloud.hpp:115-125): voxel triples of every point
//   (floor(c / leaf) with the x86 int64 conversion: NaN / out of range ->
//   INT64_MIN), sorted on the device (one packed 64-bit radix sort when the
//   triples' box fits 64 bits, else three stable LSD passes), distinct triples
//   counted.  Exact: the count does not depend on any order.
// * auto_leaf's bisection (point_cloud.hpp:137-182) runs on the host with the
//   host libm (sqrt, log) exactly as the reference; only the counts come from
//   the device (one 8-byte read per probe).
// * voxel_grid_downsample: the same sort, then one centroid per voxel in
//   ascending voxel order; each voxel's sum runs over its points in input
//   order (a stable sort).  The reference sums in std::sort's (unstable)
//   order, so a voxel of >= 3 points can differ in the last bits of its
//   centroid; voxel set, count, order, leaf and convergence are exact.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <limits>
#include <vector>

#include "bbs_map_impl.h"
#include "device_common.cuh"

namespace bbs {

namespace {

constexpr int kT = 256;

unsigned grid_n(uint64_t n) {
  return static_cast<unsigned>(std::min<uint64_t>(std::max<uint64_t>((n + kT - 1) / kT, 1), 148ull * 32));
}

template <typename T>
struct DBuf {
  T* p = nullptr;
  cudaStream_t s = nullptr;
  DBuf(size_t n, cudaStream_t st) : s(st) {
    BBS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), std::max<size_t>(n, 1) * sizeof(T), st));
  }
  ~DBuf() {
    if (p) cudaFreeAsync(p, s);
  }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
};

// static_cast<std::int64_t>(std::floor(c / leaf)) with x86 cvttsd2si (64-bit)
__device__ __forceinline__ long long vox64(double c, double leaf) {
  const double f = floor(__ddiv_rn(c, leaf));
  return (f >= -9223372036854775808.0 && f < 9223372036854775808.0) ? static_cast<long long>(f)
                                                                     : LLONG_MIN;
}

// Voxel triples (SoA int64) + per-axis min/max (order-preserving unsigned).
__global__ void vox_keys_kernel(const double* __restrict__ xyz, uint64_t n, double leaf,
                                long long* __restrict__ v, unsigned long long* __restrict__ mm) {
  unsigned long long mn[3] = {~0ull, ~0ull, ~0ull}, mx[3] = {0, 0, 0};
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const long long k = vox64(xyz[3 * i + a], leaf);
      v[a * n + i] = k;
      const unsigned long long u = static_cast<unsigned long long>(k) ^ 0x8000000000000000ull;
      mn[a] = min(mn[a], u);
      mx[a] = max(mx[a], u);
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn[a] = min(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
      mx[a] = max(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&mm[a], mn[a]);
      atomicMax(&mm[3 + a], mx[a]);
    }
  }
}

// Packed key relative to the box (bits per axis sum to <= 64), index payload.
__global__ void pack_keys_kernel(const long long* __restrict__ v, uint64_t n, ulonglong3 lo, uint32_t by,
                                 uint32_t bz, unsigned long long* __restrict__ key, uint32_t* __restrict__ idx) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const unsigned long long ux = (static_cast<unsigned long long>(v[i]) ^ 0x8000000000000000ull) - lo.x;
    const unsigned long long uy = (static_cast<unsigned long long>(v[n + i]) ^ 0x8000000000000000ull) - lo.y;
    const unsigned long long uz = (static_cast<unsigned long long>(v[2 * n + i]) ^ 0x8000000000000000ull) - lo.z;
    const uint32_t sx = by + bz;  // bx + by + bz <= 64, so no set bit is shifted out
    key[i] = (sx >= 64 ? 0ull : ux << sx) | (bz >= 64 ? 0ull : uy << bz) | uz;
    idx[i] = static_cast<uint32_t>(i);
  }
}

// One axis of the LSD passes: the axis value of the point at perm[i].
__global__ void axis_keys_kernel(const long long* __restrict__ v, const uint32_t* __restrict__ perm, uint64_t n,
                                 unsigned long long* __restrict__ key) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    key[i] = static_cast<unsigned long long>(v[perm[i]]) ^ 0x8000000000000000ull;
}

// head[i] = 1 when sorted position i starts a new voxel.
__global__ void heads_kernel(const long long* __restrict__ v, const uint32_t* __restrict__ perm, uint64_t n,
                             uint32_t* __restrict__ head) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    bool h = i == 0;
    if (!h) {
      const uint32_t a = perm[i], b = perm[i - 1];
      h = v[a] != v[b] || v[n + a] != v[n + b] || v[2 * n + a] != v[2 * n + b];
    }
    head[i] = h ? 1u : 0u;
  }
}

// Segment starts from the inclusive head scan (seg id = scan - 1).
__global__ void seg_start_kernel(const uint32_t* __restrict__ head, const uint32_t* __restrict__ incl, uint64_t n,
                                 uint32_t* __restrict__ start) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    if (head[i]) start[incl[i] - 1] = static_cast<uint32_t>(i);
}

// Centroid of each voxel (point_cloud.hpp:95-108): the first point's
// coordinates plus the others in order, divided by the count.
__global__ void centroid_kernel(const double* __restrict__ xyz, const uint32_t* __restrict__ perm,
                                const uint32_t* __restrict__ start, uint32_t n_seg, uint64_t n,
                                double* __restrict__ out) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n_seg; s += gridDim.x * blockDim.x) {
    const uint32_t b = start[s], e = s + 1 < n_seg ? start[s + 1] : static_cast<uint32_t>(n);
    const uint32_t p0 = perm[b];
    double sx = xyz[3 * p0], sy = xyz[3 * p0 + 1], sz = xyz[3 * p0 + 2];
    for (uint32_t j = b + 1; j < e; ++j) {
      const uint32_t p = perm[j];
      sx = __dadd_rn(sx, xyz[3 * p]);
      sy = __dadd_rn(sy, xyz[3 * p + 1]);
      sz = __dadd_rn(sz, xyz[3 * p + 2]);
    }
    const double c = static_cast<double>(e - b);
    out[3 * s] = __ddiv_rn(sx, c);
    out[3 * s + 1] = __ddiv_rn(sy, c);
    out[3 * s + 2] = __ddiv_rn(sz, c);
  }
}

int bits_for_span(unsigned long long span) {  // bits to hold [0, span]
  int b = 0;
  while (b < 64 && (span >> b) != 0) ++b;
  return b;
}

__global__ void iota_kernel(uint32_t* __restrict__ p, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    p[i] = static_cast<uint32_t>(i);
}

size_t sorter_temp_bytes(uint64_t n, cudaStream_t s) {
  size_t a = 0, b = 0;
  cub::DoubleBuffer<unsigned long long> dk(nullptr, nullptr);
  cub::DoubleBuffer<uint32_t> dv(nullptr, nullptr);
  BBS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, a, dk, dv, static_cast<int64_t>(n), 0, 64, s));
  BBS_CUDA(cub::DeviceScan::InclusiveSum(nullptr, b, static_cast<uint32_t*>(nullptr),
                                         static_cast<uint32_t*>(nullptr), static_cast<int64_t>(n), s));
  return std::max(a, b);
}

// The raw cloud on the device and its voxel sort at one leaf.
struct VoxelSorter {
  cudaStream_t s;
  uint64_t n;
  size_t temp_bytes;
  DBuf<double> xyz;
  DBuf<long long> v;
  DBuf<unsigned long long> mm, k0, k1;
  DBuf<uint32_t> i0, i1, head, incl;
  DBuf<unsigned char> temp;
  uint32_t* perm = nullptr;  // sorted order after sort()

  VoxelSorter(const double* host_xyz, uint64_t count, cudaStream_t st)
      : s(st), n(count), temp_bytes(sorter_temp_bytes(count, st)), xyz(3 * count, st), v(3 * count, st),
        mm(6, st), k0(count, st), k1(count, st), i0(count, st), i1(count, st), head(count, st),
        incl(count, st), temp(temp_bytes, st) {
    BBS_CUDA(cudaMemcpyAsync(xyz.p, host_xyz, 3 * n * sizeof(double), cudaMemcpyHostToDevice, s));
  }

  // Sorts the points by voxel triple (stable: ties keep input order) and
  // returns the number of distinct voxels (count_voxels).
  uint64_t sort(double leaf) {
    const unsigned long long init[6] = {~0ull, ~0ull, ~0ull, 0, 0, 0};
    BBS_CUDA(cudaMemcpyAsync(mm.p, init, sizeof(init), cudaMemcpyHostToDevice, s));
    vox_keys_kernel<<<grid_n(n), kT, 0, s>>>(xyz.p, n, leaf, v.p, mm.p);
    BBS_CUDA(cudaGetLastError());
    unsigned long long h[6];
    BBS_CUDA(cudaMemcpyAsync(h, mm.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    BBS_CUDA(cudaStreamSynchronize(s));
    const int bx = bits_for_span(h[3] - h[0]), by = bits_for_span(h[4] - h[1]), bz = bits_for_span(h[5] - h[2]);
    cub::DoubleBuffer<unsigned long long> dk(k0.p, k1.p);
    cub::DoubleBuffer<uint32_t> dv(i0.p, i1.p);
    size_t tb = temp_bytes;
    if (bx + by + bz <= 64) {
      pack_keys_kernel<<<grid_n(n), kT, 0, s>>>(v.p, n, make_ulonglong3(h[0], h[1], h[2]), static_cast<uint32_t>(by),
                                                static_cast<uint32_t>(bz), k0.p, i0.p);
      BBS_CUDA(cudaGetLastError());
      BBS_CUDA(cub::DeviceRadixSort::SortPairs(temp.p, tb, dk, dv, static_cast<int64_t>(n), 0,
                                               std::max(1, bx + by + bz), s));
    } else {
      // three stable LSD passes: z, then y, then x
      iota_kernel<<<grid_n(n), kT, 0, s>>>(dv.Current(), n);
      BBS_CUDA(cudaGetLastError());
      for (int a = 2; a >= 0; --a) {
        axis_keys_kernel<<<grid_n(n), kT, 0, s>>>(v.p + a * n, dv.Current(), n, dk.Current());
        BBS_CUDA(cudaGetLastError());
        BBS_CUDA(cub::DeviceRadixSort::SortPairs(temp.p, tb, dk, dv, static_cast<int64_t>(n), 0, 64, s));
      }
    }
    perm = dv.Current();
    heads_kernel<<<grid_n(n), kT, 0, s>>>(v.p, perm, n, head.p);
    BBS_CUDA(cudaGetLastError());
    BBS_CUDA(cub::DeviceScan::InclusiveSum(temp.p, tb, head.p, incl.p, static_cast<int64_t>(n), s));
    uint32_t count = 0;
    BBS_CUDA(cudaMemcpyAsync(&count, incl.p + (n - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    BBS_CUDA(cudaStreamSynchronize(s));
    return count;
  }

  // voxel_grid_downsample after sort(): centroids in ascending voxel order.
  std::vector<double> centroids(uint64_t count) {
    DBuf<uint32_t> start(count, s);
    DBuf<double> out(3 * count, s);
    seg_start_kernel<<<grid_n(n), kT, 0, s>>>(head.p, incl.p, n, start.p);
    BBS_CUDA(cudaGetLastError());
    centroid_kernel<<<grid_n(count), kT, 0, s>>>(xyz.p, perm, start.p, static_cast<uint32_t>(count), n, out.p);
    BBS_CUDA(cudaGetLastError());
    std::vector<double> h(3 * count);
    BBS_CUDA(cudaMemcpyAsync(h.data(), out.p, h.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    BBS_CUDA(cudaStreamSynchronize(s));
    return h;
  }
};

}  // namespace

// prepare_source, pipeline.hpp:25-41, with auto_leaf (point_cloud.hpp:137-182)
// driving device voxel counts and voxel_grid_downsample on the device.
SourcePrep device_prepare_source(int device, const double* xyz, uint64_t n, uint64_t target,
                                 bool exact_centroids) {
  SourcePrep p;
  if (target > 0 && n > target) {
    if (n >= (1ull << 32)) throw Error(BBS_ERR_TOO_LARGE, "prepare_source: more than 2^32 points");
    DeviceGuard g(device);
    cudaStream_t s;
    BBS_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
      }
    } sg{s};
    VoxelSorter vs(xyz, n, s);
    // auto_leaf, point_cloud.hpp:137-182 (host arithmetic, device counts)
    const std::size_t lo_count = std::max<std::size_t>(1, (target + 1) / 2);
    const std::size_t hi_count = 2 * target;
    const bbs_aabb box = host_bounding_box(xyz, n);
    const double ex = box.max.x - box.min.x, ey = box.max.y - box.min.y, ez = box.max.z - box.min.z;
    const double max_ext = std::max({ex, ey, ez, 1e-9});
    double lo = max_ext / (1 << 24);
    double hi = max_ext;
    double leaf = 0.0;
    bool converged = true, found = false;
    {
      const std::size_t c = vs.sort(lo);
      if (c <= hi_count && (c >= lo_count || c == n)) {
        leaf = lo;
        found = true;
      }
    }
    if (!found) {
      double best_leaf = lo;
      double best_gap = std::numeric_limits<double>::infinity();
      for (int iter = 0; iter < 32 && !found; ++iter) {
        const double mid = std::sqrt(lo * hi);
        const std::size_t c = vs.sort(mid);
        if (c >= lo_count && c <= hi_count) {
          leaf = mid;
          found = true;
          break;
        }
        const double gap = std::abs(std::log(static_cast<double>(std::max<std::size_t>(c, 1))) -
                                    std::log(static_cast<double>(target)));
        if (gap < best_gap) {
          best_gap = gap;
          best_leaf = mid;
        }
        if (c > hi_count)
          lo = mid;
        else
          hi = mid;
      }
      if (!found) {
        leaf = best_leaf;
        converged = false;
      }
    }
    // voxel_grid_downsample, point_cloud.hpp:78-111
    if (!(leaf > 0.0)) throw Error(BBS_ERR_CONFIG, "voxel_grid_downsample: leaf must be > 0");
    if (exact_centroids) {
      // the reference's per-voxel summation order is its introsort's
      // permutation: replayed on the host at the device-found leaf
      p.xyz = host_voxel_grid_downsample(xyz, n, leaf);
    } else {
      const uint64_t count = vs.sort(leaf);
      p.xyz = vs.centroids(count);
    }
    p.leaf = leaf;
    p.converged = converged;
  } else {
    p.xyz.assign(xyz, xyz + 3 * n);  // pipeline.hpp:36-37
  }
  p.d_max = host_max_range(p.xyz.data(), p.xyz.size() / 3);
  return p;
}

}  // namespace bbs

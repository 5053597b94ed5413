// microbench.cu — random 32-byte gather ceiling per memory tier (SURVEY §8d:
// "the tier ceiling must be measured with a random independent 32 B load
// microbenchmark").  A buffer of `bytes` is read in independent random
// 32 B sectors (8 independent streams per thread); the result is the
// sector bandwidth in GB/s (sectors * 32 B / time).  64 MB stays in L2,
// 1 GiB goes to HBM.
#include <cuda_runtime.h>

#include <algorithm>

#include "bbs_internal.h"

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void __launch_bounds__(256) gather32_kernel(const uint4* __restrict__ buf, uint64_t n_sectors,
                                                       uint32_t iters, uint64_t seed,
                                                       unsigned long long* sink) {
  constexpr int S = 8;
  uint64_t st[S];
  const uint64_t tid = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
#pragma unroll
  for (int j = 0; j < S; ++j) st[j] = mix64(seed + tid * S + j);
  uint32_t acc = 0;
  for (uint32_t it = 0; it < iters; ++it) {
    uint4 v[S][2];
#pragma unroll
    for (int j = 0; j < S; ++j) {
      st[j] = mix64(st[j] + 0x9E3779B97F4A7C15ull);
      const uint64_t sct = st[j] % n_sectors;
      v[j][0] = __ldg(buf + 2 * sct);
      v[j][1] = __ldg(buf + 2 * sct + 1);
    }
#pragma unroll
    for (int j = 0; j < S; ++j) acc ^= v[j][0].x ^ v[j][0].w ^ v[j][1].y ^ v[j][1].z;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);  // keeps the loads alive
}

// Shared-memory tier: conflict-free 4-byte reads, the access pattern of the
// root column kernel (the 32 lanes of a warp read 32 distinct banks of a
// staged z-column window).  Per iteration a warp-uniform random base row and
// 8 loads at immediate row offsets, so the loop issues ~2 instructions per
// LDS and the shared-memory pipe (one 128 B wavefront per clock per SM) is
// the limiter.
__global__ void __launch_bounds__(256) smem_gather_kernel(uint32_t iters, uint64_t seed,
                                                          unsigned long long* sink) {
  constexpr int kRows = 384;  // 384 x 32 words = 48 KB
  constexpr int kStride = 7;  // rows between the 8 loads of one iteration
  __shared__ uint32_t buf[kRows * 32];
  for (int i = threadIdx.x; i < kRows * 32; i += blockDim.x) buf[i] = static_cast<uint32_t>(i) * 2654435761u;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  uint32_t st = static_cast<uint32_t>(mix64(seed + blockIdx.x * 1024 + (threadIdx.x >> 5)));
  uint32_t acc = 0;
  for (uint32_t it = 0; it < iters; ++it) {
    st = st * 1664525u + 1013904223u;  // warp-uniform base row
    const uint32_t* p = buf + ((st >> 24) + 1) * 32 + lane;  // rows 1 .. 256 + 7 * 7 < kRows
    uint32_t v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = p[j * kStride * 32];
    acc ^= v[0] ^ v[1] ^ v[2] ^ v[3] ^ v[4] ^ v[5] ^ v[6] ^ v[7];
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

}  // namespace

// Conflict-free shared-memory 4-byte gather ceiling of the whole GPU in GB/s
// (words * 4 B / time; 8 CTAs of 256 threads per SM).
extern "C" int bbs_smem_bench(int32_t device, double* out_gbs) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= device) return BBS_ERR_CUDA;
  cudaSetDevice(device);
  unsigned long long* sink = nullptr;
  if (cudaMalloc(&sink, sizeof(unsigned long long)) != cudaSuccess) return BBS_ERR_CUDA;
  const int blocks = 148 * 4, threads = 256;
  const uint32_t iters = 4096;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  smem_gather_kernel<<<blocks, threads>>>(iters, 1, sink);  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    smem_gather_kernel<<<blocks, threads>>>(iters, 100 + rep, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    best = std::min(best, ms);
  }
  const double words = static_cast<double>(blocks) * threads * iters * 8;
  *out_gbs = words * 4.0 / (best * 1e-3) / 1e9;
  const cudaError_t e = cudaGetLastError();
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  return e == cudaSuccess ? BBS_OK : BBS_ERR_CUDA;
}

extern "C" int bbs_gather_bench(int32_t device, uint64_t bytes, double* out_gbs) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= device) return BBS_ERR_CUDA;
  cudaSetDevice(device);
  uint4* buf = nullptr;
  unsigned long long* sink = nullptr;
  if (cudaMalloc(&buf, bytes) != cudaSuccess) return BBS_ERR_CUDA;
  cudaMalloc(&sink, sizeof(unsigned long long));
  cudaMemset(buf, 0x5A, bytes);
  const uint64_t n_sectors = bytes / 32;
  const int blocks = 148 * 8, threads = 256;
  const uint32_t iters = 64;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  gather32_kernel<<<blocks, threads>>>(buf, n_sectors, iters, 1, sink);  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    gather32_kernel<<<blocks, threads>>>(buf, n_sectors, iters, 100 + rep, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    best = std::min(best, ms);
  }
  const double sectors = static_cast<double>(blocks) * threads * iters * 8;
  *out_gbs = sectors * 32.0 / (best * 1e-3) / 1e9;
  const cudaError_t e = cudaGetLastError();
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(buf);
  cudaFree(sink);
  return e == cudaSuccess ? BBS_OK : BBS_ERR_CUDA;
}

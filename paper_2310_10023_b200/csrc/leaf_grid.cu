// leaf_grid.cu — exhaustive leaf-grid scoring on the device: the reference's
// `oracle_search` (oracle.hpp:29-95), SURVEY §8f row 4.  Every level-0 node
// under the root translation index ranges times the level-0 rotation grid is
// enumerated ON THE DEVICE in the reference's loop order (ix, iy, iz, ir, ip,
// iw; oracle.hpp:80-92), scored by the same batch_evaluate kernels the search
// uses (bit-exact per node), and reduced per block: block max, then an
// order-preserving select of the nodes attaining the running best (the
// reference's drain lambda, oracle.hpp:66-77).  Only the block max (4 B) and
// the argmax nodes cross PCIe.  Host validation lives in capi.cpp
// (bbs_oracle_search), in the reference's order.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <cstdint>
#include <cstring>

#include "bbs_map_impl.h"
#include "kernels.h"

namespace bbs {

namespace {

// leaf index q -> node, iw fastest (oracle.hpp:80-92)
__global__ void leaf_nodes_kernel(LeafGridSpec g, uint64_t first, uint64_t n,
                                  bbs_node* __restrict__ out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t q = first + i;
    const uint64_t iw = q % g.nw;
    q /= g.nw;
    const uint64_t ip = q % g.np;
    q /= g.np;
    const uint64_t ir = q % g.nr;
    q /= g.nr;
    const uint64_t iz = q % g.nz;
    q /= g.nz;
    const uint64_t iy = q % g.ny;
    q /= g.ny;
    bbs_node nd;
    nd.ix = static_cast<int32_t>(g.x_lo + static_cast<int64_t>(q));
    nd.iy = static_cast<int32_t>(g.y_lo + static_cast<int64_t>(iy));
    nd.iz = static_cast<int32_t>(g.z_lo + static_cast<int64_t>(iz));
    nd.iroll = static_cast<int32_t>(ir);
    nd.ipitch = static_cast<int32_t>(ip);
    nd.iyaw = static_cast<int32_t>(iw);
    nd.level = 0;
    nd.score = -1;
    out[i] = nd;
  }
}

__global__ void block_max_kernel(const bbs_node* __restrict__ nodes, uint64_t n,
                                 int32_t* __restrict__ out) {
  int32_t m = -1;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    m = max(m, nodes[i].score);
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

struct ScoreIs {
  int32_t v;
  __device__ __forceinline__ bool operator()(const bbs_node& a) const { return a.score == v; }
};

unsigned grid_for(uint64_t n) {
  return static_cast<unsigned>(std::min<uint64_t>(std::max<uint64_t>((n + 255) / 256, 1), 148ull * 16));
}

}  // namespace

void leaf_grid_search(bbs_map* m, bbs_scan* scan, const bbs_search_config& cfg, double d_max,
                      const LeafGridSpec& g, uint64_t block, int32_t* best_score,
                      std::vector<bbs_node>* argmax) {
  DeviceGuard dg(m->device);
  cudaStream_t s = m->stream;
  const uint64_t total = g.total();
  block = std::max<uint64_t>(1, std::min(block, total));
  // buffers released on every exit path (BBS_CUDA throws)
  struct Bufs {
    cudaStream_t s;
    bbs_node *nodes = nullptr, *sel = nullptr;
    int32_t* small = nullptr;  // [0] block max, [2..3] selected count (u64)
    void* tmp = nullptr;
    int32_t* host = nullptr;
    ~Bufs() {
      for (void* p : {static_cast<void*>(nodes), static_cast<void*>(sel), static_cast<void*>(small), tmp})
        if (p) cudaFreeAsync(p, s);
      cudaStreamSynchronize(s);
      if (host) cudaFreeHost(host);
    }
  } bufs{s};
  size_t tmp_bytes = 0;
  BBS_CUDA(cub::DeviceSelect::If(nullptr, tmp_bytes, bufs.nodes, bufs.sel,
                                 reinterpret_cast<unsigned long long*>(bufs.small), block, ScoreIs{0}, s));
  BBS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&bufs.nodes), block * sizeof(bbs_node), s));
  BBS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&bufs.sel), block * sizeof(bbs_node), s));
  BBS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&bufs.small), 16, s));
  BBS_CUDA(cudaMallocAsync(&bufs.tmp, std::max<size_t>(tmp_bytes, 16), s));
  BBS_CUDA(cudaMallocHost(reinterpret_cast<void**>(&bufs.host), 16));
  bbs_node* const d_nodes = bufs.nodes;
  bbs_node* const d_sel = bufs.sel;
  int32_t* const d_small = bufs.small;
  void* const d_tmp = bufs.tmp;
  int32_t* const h_small = bufs.host;
  unsigned long long* d_nsel = reinterpret_cast<unsigned long long*>(d_small + 2);
  int32_t best = -1;
  argmax->clear();
  // the rotation LUT once for every block (level-0 indices in [0, max_index])
  StreamAllocs al(s);
  const GridView gv = upload_grid(cfg, d_max, nullptr, nullptr, s, al);
  for (uint64_t first = 0; first < total; first += block) {
    const uint64_t n = std::min(block, total - first);
    leaf_nodes_kernel<<<grid_for(n), 256, 0, s>>>(g, first, n, d_nodes);
    BBS_CUDA(cudaGetLastError());
    batch_evaluate_device(m, scan, gv, d_nodes, n, s);
    BBS_CUDA(cudaMemsetAsync(d_small, 0xff, 4, s));  // -1: the reference's initial best
    block_max_kernel<<<grid_for(n), 256, 0, s>>>(d_nodes, n, d_small);
    BBS_CUDA(cudaGetLastError());
    BBS_CUDA(cudaMemcpyAsync(h_small, d_small, 4, cudaMemcpyDeviceToHost, s));
    BBS_CUDA(cudaStreamSynchronize(s));
    const int32_t bm = h_small[0];
    if (bm > best) {  // oracle.hpp:70-73
      best = bm;
      argmax->clear();
    }
    if (bm != best) continue;
    size_t tb = tmp_bytes;
    BBS_CUDA(cub::DeviceSelect::If(d_tmp, tb, d_nodes, d_sel, d_nsel, n, ScoreIs{best}, s));
    BBS_CUDA(cudaMemcpyAsync(h_small + 2, d_nsel, 8, cudaMemcpyDeviceToHost, s));
    BBS_CUDA(cudaStreamSynchronize(s));
    uint64_t nsel = 0;
    std::memcpy(&nsel, h_small + 2, 8);
    if (nsel) {
      const size_t o = argmax->size();
      argmax->resize(o + nsel);
      BBS_CUDA(cudaMemcpyAsync(argmax->data() + o, d_sel, nsel * sizeof(bbs_node), cudaMemcpyDeviceToHost, s));
      BBS_CUDA(cudaStreamSynchronize(s));
    }
  }
  *best_score = best;
}

}  // namespace bbs

// kernels.h — host launchers of the device kernels (score.cu, search.cu).
#pragma once

#include <cuda_runtime.h>

#include "bbs_internal.h"

namespace bbs {

struct ScanView {
  const double* x;
  const double* y;
  const double* z;
  uint32_t k;
};

// Root translation box (initial_nodes, nodes.hpp:60-85) and its shard.
struct BoxParams {
  int32_t level;
  int32_t x0, y0, z0;         // trans_index_range mins
  uint32_t nx, ny, nz;        // counts per axis
  uint32_t nr, np, nw;        // rotation index counts at the root level
  uint32_t rank, world;       // roots with ref index % world == rank
  uint32_t n_tchunks;         // translation chunks per rotation (grid = nrot * n_tchunks)
  uint32_t pad;
  double tmax;                // max |translation index| in the box (fast-path guard)
};

constexpr int kBoxThreads = 256;
constexpr int kBoxTransPerThread = 4;
constexpr int kBoxTransPerCta = kBoxThreads * kBoxTransPerThread;

// Score every root of the box owned by (rank, world) into scores[ref index].
void launch_score_box(const MapView& map, const GridView& grid, const ScanView& scan,
                      const BoxParams& bp, int32_t* scores, cudaStream_t s);

// Score n nodes that come in contiguous same-rotation runs of 8 (the output
// order of branch(), nodes.hpp:103-116).  n is read from *d_n when non-null
// (device-resident count; up to n_max nodes).  scores must be zeroed first
// when n_ptiles > 1.
void launch_score_runs8(const MapView& map, const GridView& grid, const ScanView& scan,
                        const bbs_node* nodes, const uint32_t* d_n, uint32_t n_max,
                        uint32_t n_ptiles, int32_t* scores, cudaStream_t s);

// Score arbitrary nodes in place (node.score), grouping equal rotations on
// the device.  Host-synchronous.
void score_nodes_general(const MapView& map, const GridView& grid, const ScanView& scan,
                         bbs_node* d_nodes, uint64_t n, cudaStream_t s);

// Choose the point-tile split for `runs` runs so the grid fills the chip.
uint32_t choose_ptiles(uint64_t runs, uint32_t k);

}  // namespace bbs

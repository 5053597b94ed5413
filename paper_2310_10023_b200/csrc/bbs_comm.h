// bbs_comm.h — NCCL communicator behind bbs_comm_t (comm.cpp).
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime_api.h>

namespace bbs {

struct Comm {
  void* nccl = nullptr;  // ncclComm_t
  int device = 0, rank = 0, world = 1;
};

void comm_unique_id(uint8_t out[128]);
Comm* comm_create(int device, int rank, int world, const uint8_t id[128]);
void comm_destroy(Comm* c);
// In-place element-wise MAX of n int32 on the device, enqueued on s.
void comm_allreduce_max_i32(Comm* c, int32_t* d, size_t n, cudaStream_t s);
int comm_nccl_version();

}  // namespace bbs

// Kernel-node throughput of T streams each replaying a graph of 64 short
// kernels (the C4 shape: many concurrent searches, ~8 kernels per flush).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o launch_rate launch_rate.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__global__ void tiny(int* p, int spin) {
  // a few microseconds of latency-bound work per CTA
  long long t0 = clock64();
  while (clock64() - t0 < spin) {
  }
  if (threadIdx.x == 0 && p) atomicAdd(p, 1);
}

int main(int argc, char** argv) {
  const int grid = argc > 1 ? atoi(argv[1]) : 148;
  const int spin = argc > 2 ? atoi(argv[2]) : 2000;
  int* d;
  cudaMalloc(&d, 4);
  for (int T : {1, 4, 16, 32}) {
    std::vector<cudaStream_t> st(T);
    std::vector<cudaGraphExec_t> ge(T);
    for (int t = 0; t < T; ++t) {
      cudaStreamCreateWithFlags(&st[t], cudaStreamNonBlocking);
      cudaGraph_t g;
      cudaStreamBeginCapture(st[t], cudaStreamCaptureModeRelaxed);
      for (int k = 0; k < 64; ++k) tiny<<<grid, 256, 0, st[t]>>>(d, spin);
      cudaStreamEndCapture(st[t], &g);
      cudaGraphInstantiate(&ge[t], g, 0);
      cudaGraphDestroy(g);
    }
    const int reps = 20;
    for (int t = 0; t < T; ++t) cudaGraphLaunch(ge[t], st[t]);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, 0);
    cudaDeviceSynchronize();
    for (int r = 0; r < reps; ++r)
      for (int t = 0; t < T; ++t) cudaGraphLaunch(ge[t], st[t]);
    cudaDeviceSynchronize();
    cudaEventRecord(b, 0);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double n = 64.0 * reps * T;
    std::printf("grid %d spin %d streams %2d: %.0f kernels in %.2f ms -> %.2f us per kernel (%.2f us per chain step)\n",
                grid, spin, T, n, ms, 1e3 * ms / n, 1e3 * ms / (64.0 * reps));
    for (int t = 0; t < T; ++t) {
      cudaGraphExecDestroy(ge[t]);
      cudaStreamDestroy(st[t]);
    }
  }
  std::printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

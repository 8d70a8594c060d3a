// microbenchmark: GPU writes / reads of the host leaves' (f, x) spans in mapped
// pinned memory, as k_host_scatter / k_host_gather do (each 896 B span starts
// 32 B into a 64 B line), vs the same spans widened to whole 64 B lines.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int LEAF = 6 * 14 * 14 * 14;
__device__ __forceinline__ int span_src(int f, int x) { return ((f * 14 + x + 3) * 14 + 3) * 14; }

// mode 0: exact spans (112 doubles from span_src); mode 1: the 64 B-aligned hull
__global__ void k_write(double* host, int L, int mode, int write) {
  int per = mode == 0 ? 112 : 120;  // spans start 2 or 6 doubles into a line: hull = 15 lines
  long long total = (long long)L * 48 * per;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    long long sp = i / per;
    int j = (int)(i - sp * per);
    int leaf = (int)(sp / 48), fx = (int)(sp % 48);
    long long off = (long long)leaf * LEAF + span_src(fx >> 3, fx & 7);
    if (mode == 1) {
      off &= ~7LL;  // 64 B aligned start
    }
    if (write) __stcs(host + off + j, (double)j);
    else if (__ldcs(host + off + j) == -1.0) host[0] = 0;
  }
}

int main(int argc, char** argv) {
  int L = argc > 1 ? atoi(argv[1]) : 8192;
  int dev = argc > 2 ? atoi(argv[2]) : 0;
  cudaSetDevice(dev);
  double* h;
  size_t bytes = (size_t)L * LEAF * 8;
  cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
  for (size_t i = 0; i < bytes / 8; i += 512) h[i] = 0;
  double* d;
  cudaHostGetDevicePointer(&d, h, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int write = 0; write < 2; write++)
    for (int mode = 0; mode < 2; mode++)
      for (int grid : {148 * 2, 148 * 8}) {
        float best = 1e9;
        for (int r = 0; r < 5; r++) {
          cudaEventRecord(e0);
          k_write<<<grid, 256>>>(d, L, mode, write);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (ms < best) best = ms;
        }
        double useful = (double)L * 48 * 112 * 8;
        printf("dev %d %s %s grid %d: %.2f ms, %.1f GB/s (useful span bytes)\n", dev, write ? "write" : "read ",
               mode ? "aligned-hull" : "exact-span  ", grid, best, useful / best / 1e6);
      }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

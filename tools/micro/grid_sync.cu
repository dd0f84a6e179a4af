// Micro-benchmark: cost of a cooperative grid-wide barrier on this GPU (cooperative_groups), for
// sizing a persistent PCG kernel.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 grid_sync.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int n, int* out) {
  cg::grid_group g = cg::this_grid();
  int s = 0;
  for (int i = 0; i < n; ++i) {
    s += threadIdx.x;
    g.sync();
  }
  if (s == -1) out[0] = s;
}
int main() {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int* out;
  cudaMalloc(&out, 4);
  for (int threads : {128, 256}) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, threads, 0);
    for (int bps : {1, 2, 4}) {
      if (bps > per) continue;
      int grid = sms * bps, n = 2000;
      void* args[] = {&n, &out};
      cudaLaunchCooperativeKernel((void*)k, grid, threads, args, 0, 0);
      cudaDeviceSynchronize();
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k, grid, threads, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("threads %d blocks/SM %d grid %d: %.3f us per grid sync (%s)\n", threads, bps, grid, 1e3 * ms / n,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}

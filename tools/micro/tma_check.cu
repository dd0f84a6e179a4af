// Micro check of the brick SpMV's TMA usage: 3-D fp64 box loads with negative start coordinates
// (OOB zero fill), boxes larger than the tensor, descriptors in global memory vs kernel parameter.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/tma_check tools/micro/tma_check.cu && /tmp/tma_check
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <bool PARAM>
__global__ void k(const CUtensorMap* gmap, const __grid_constant__ CUtensorMap pmap, int c0, int c1, int c2, int n,
                  double* out) {
  extern __shared__ __align__(128) unsigned char raw[];
  unsigned char* b = raw + ((128u - (sa(raw) & 127u)) & 127u);
  double* xs = (double*)b;
  uint64_t* bar = (uint64_t*)(b + ((n * 8 + 127) / 128) * 128);
  const CUtensorMap* map = PARAM ? &pmap : gmap;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (!PARAM) asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(map) : "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar)), "r"(n * 8) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            sa(xs)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(sa(bar))
        : "memory");
  }
  unsigned done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(sa(bar))
                 : "memory");
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = xs[i];
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const int D0 = 10, D1 = 9, D2 = 8;  // tensor (jj fastest)
  std::vector<double> h(D0 * D1 * D2);
  for (size_t i = 0; i < h.size(); ++i) h[i] = 1.0 + i;
  double *d, *o;
  cudaMalloc(&d, h.size() * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&o, 4096 * 8);
  CUtensorMap *gm;
  cudaMalloc(&gm, sizeof(CUtensorMap));
  struct Case { unsigned b0, b1, b2; int c0, c1, c2; };
  Case cs[] = {{10, 6, 6, 0, 0, 0}, {10, 6, 6, 0, -1, -1}, {10, 6, 6, 2, 0, 0}, {10, 6, 6, -2, 0, 0},
               {10, 6, 6, 1, 0, 0}, {10, 11, 10, 0, -2, -1}, {12, 11, 10, -2, -2, -1}, {10, 6, 6, -1, 0, 0}};
  for (const Case& C : cs) {
    CUtensorMap m;
    cuuint64_t dims[3] = {D0, D1, D2}, str[2] = {D0 * 8, D0 * D1 * 8};
    cuuint32_t box[3] = {C.b0, C.b1, C.b2}, es[3] = {1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaMemcpy(gm, &m, sizeof(m), cudaMemcpyHostToDevice);
    const int n = C.b0 * C.b1 * C.b2;
    for (int param = 0; param < 2; ++param) {
      cudaMemset(o, 0xff, 4096 * 8);
      const int smem = n * 8 + 256 + 128;
      if (param) {
        cudaFuncSetAttribute(k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k<true><<<1, 128, smem>>>(gm, m, C.c0, C.c1, C.c2, n, o);
      } else {
        cudaFuncSetAttribute(k<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k<false><<<1, 128, smem>>>(gm, m, C.c0, C.c1, C.c2, n, o);
      }
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<double> got(n);
      cudaMemcpy(got.data(), o, n * 8, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int z = 0; z < (int)C.b2; ++z)
        for (int y = 0; y < (int)C.b1; ++y)
          for (int x = 0; x < (int)C.b0; ++x) {
            const int gx = x + C.c0, gy = y + C.c1, gz = z + C.c2;
            const double ref = (gx >= 0 && gx < D0 && gy >= 0 && gy < D1 && gz >= 0 && gz < D2) ? h[gx + D0 * (gy + D1 * gz)] : 0.0;
            bad += got[x + C.b0 * (y + C.b1 * z)] != ref;
          }
      printf("box %u %u %u start %d %d %d param=%d: encode=%d err=%s bad=%d\n", C.b0, C.b1, C.b2, C.c0, C.c1, C.c2,
             param, (int)r, cudaGetErrorString(e), bad);
      if (e != cudaSuccess) return 1;  // a sticky error: the remaining cases cannot run
    }
  }
  return 0;
}

// Shared internal definitions of libosm (not part of the public ABI).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "osm.h"

namespace osm {

struct Error : std::runtime_error {
  osm_status status;
  Error(osm_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail(osm_status s, const std::string& m) { throw Error(s, m); }

#define OSM_CUDA(call)                                                                               \
  do {                                                                                               \
    cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess)                                                                           \
      ::osm::fail(OSM_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_) + " @" __FILE__ ":" + \
                                    std::to_string(__LINE__));                                       \
  } while (0)

#define OSM_CHECK_LAUNCH() OSM_CUDA(cudaGetLastError())

constexpr int kWarp = 32;
constexpr int kSlicesPerBlock = 8;                       // warps per hot-path block
constexpr int kRowsPerBlock = kWarp * kSlicesPerBlock;   // 256 rows per block
constexpr int kThreads = kRowsPerBlock;                  // one thread per row in the SpMV kernels
constexpr int kVecTiles = 4;                             // tiles per vector-kernel block (8 rows/thread)

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

#ifdef __CUDACC__
// Block-completion counter bump with release semantics (gpu scope): orders the caller's earlier stores
// (and, being cumulative, the block's stores it observed through a barrier) before the increment,
// without the L1 invalidation of a full fence.  The last block adds the acquire-side fence itself.
__device__ __forceinline__ uint32_t atom_add_release_gpu(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.release.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
#endif
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

}  // namespace osm

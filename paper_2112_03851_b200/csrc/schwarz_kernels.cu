// Hot-path kernels of libosm: batched, masked Jacobi-PCG over every local
// subdomain ("diagonal preconditioner conjugate gradient ...
// addition of vectors (Daxpy), dot product and sparse matrix-vector
// multiplication"), and the Robin interface kernels of the Schwarz iteration
// (SURVEY.md 8(a) a1-a6).
//
// Work decomposition: the concatenated internal rows of all local subdomains are
// cut in blocks of 256 rows (8 SELL-32 slices, one warp each); every block
// belongs to exactly one subdomain.  Per-subdomain scalars live in SubState on
// the device; blocks of converged subdomains exit at once (masking), so one
// launch serves all subdomains whatever their iteration counts.
//
// Reductions are deterministic: warp xor-tree -> 8 warp sums added in order ->
// one partial per block in global memory; the last block of a subdomain to finish
// (threadfence + counter) sums that subdomain's partials in a fixed order.  The
// result depends only on the subdomain's own rows, never on how many subdomains
// or GPUs share the run.
#include "ctx.h"

namespace osm {

namespace {

__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int32_t ld_stream(const int32_t* p) {
  int32_t v;
  asm("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}


__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block sum of N values over NW warps (fixed order); result valid in thread 0.
template <int N, int NW = kSlicesPerBlock>
__device__ __forceinline__ void block_sum(double (&v)[N], double* sm /* NW*N */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = warp_sum(v[i]);
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < N; ++i) sm[warp * N + i] = v[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double s = 0.0;
      for (int w = 0; w < NW; ++w) s += sm[w * N + i];
      v[i] = s;
    }
  }
}

// Thread 0 stores its block partials and bumps the subdomain counter; returns true
// (in every thread) in the last block of the subdomain.
template <int N>
__device__ __forceinline__ bool publish(const double (&v)[N], double* part, int64_t stride, int64_t blk,
                                        uint32_t* cnt, int nblk) {
  __shared__ bool last;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < N; ++i) part[i * stride + blk] = v[i];
    const uint32_t prev = atom_add_release_gpu(cnt, 1u);
    last = (prev == (uint32_t)(nblk - 1));
    if (last) __threadfence();  // acquire side: only the last block pays a full fence
  }
  __syncthreads();
  return last;
}

// Fixed-order sum of one subdomain's block partials; result valid in thread 0.
template <int N, int NW = kSlicesPerBlock>
__device__ __forceinline__ void gather_partials(double (&out)[N], const double* part, int64_t stride, int64_t blk0,
                                                int nblk, double* sm) {
  __threadfence();
#pragma unroll
  for (int i = 0; i < N; ++i) out[i] = 0.0;
  for (int k = threadIdx.x; k < nblk; k += blockDim.x) {
#pragma unroll
    for (int i = 0; i < N; ++i) out[i] += __ldcg(part + i * stride + blk0 + k);
  }
  __syncthreads();
  block_sum<N, NW>(out, sm);
}

// Programmatic dependent launch (sm_90+): wait for the producer grid, then let the
// next kernel in the stream begin launching while this one runs.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---------------------------------------------------------------- SELL-256 row products
// y_row = sum_j A[row, j] x[j] for row threadIdx.x of tile blk, entries in column order
// (sequential per row: deterministic, identical in both variants below).

// Variant 0 (LDG): each thread streams its row's values/columns with non-allocating loads,
// software-pipelined so chunk k+1 is requested before the gathers of chunk k are consumed.
template <int CH>
__device__ __forceinline__ double tile_row_ldg(const SellDev& A, int64_t blk, const double* __restrict__ x) {
  constexpr int T = kRowsPerBlock;
  const int w = A.twidth[blk];
  const int64_t base = A.toff[blk] + threadIdx.x;
  const double* vp = A.val + base;
  const int32_t* cp = A.col + base;
  double s = 0.0;
  double v[CH];
  int32_t c[CH];
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    v[j] = j < w ? ld_stream(vp + T * j) : 0.0;
    c[j] = j < w ? ld_stream(cp + T * j) : 0;
  }
  for (int k = 0; k < w; k += CH) {
    double xv[CH];
#pragma unroll
    for (int j = 0; j < CH; ++j) xv[j] = (k + j < w) ? __ldg(x + c[j]) : 0.0;
    double vn[CH];
    int32_t cn[CH];
    const int kn = k + CH;
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      vn[j] = (kn + j < w) ? ld_stream(vp + T * (int64_t)(kn + j)) : 0.0;
      cn[j] = (kn + j < w) ? ld_stream(cp + T * (int64_t)(kn + j)) : 0;
    }
#pragma unroll
    for (int j = 0; j < CH; ++j)
      if (k + j < w) s = fma(v[j], xv[j], s);
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      v[j] = vn[j];
      c[j] = cn[j];
    }
  }
  return s;
}

// Variant 3 (value-indexed): each entry is one 32-bit word (dictionary index << 16 | 16-bit
// column offset), 4 entries of a row per 16-byte load; the dictionary (tens to thousands of
// distinct values) is read through L1.  The next group's load is issued before the current
// group's gathers are consumed; the main loop has no per-entry predicates (widths are padded to
// a multiple of 4 with zero-valued entries).
__device__ __forceinline__ uint4 ld_stream4(const uint32_t* p) {
  uint4 v;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
      : "l"(p));
  return v;
}
__device__ __forceinline__ double tile_row_vi(const SellDev& A, int64_t blk, const double* __restrict__ x) {
  constexpr int T = kRowsPerBlock;
  const int ng = (A.vtw[blk] + 3) >> 2;
  const uint32_t* gp = A.packed + A.poff[blk] + 4 * threadIdx.x;
  const double* xr = x + blk * T + threadIdx.x;
  double s = 0.0;
  if (ng == 0) return s;
  uint4 e = ld_stream4(gp);
  for (int g = 0; g < ng; ++g) {
    const double x0 = __ldg(xr + (int16_t)(e.x & 0xffffu)), x1 = __ldg(xr + (int16_t)(e.y & 0xffffu));
    const double x2 = __ldg(xr + (int16_t)(e.z & 0xffffu)), x3 = __ldg(xr + (int16_t)(e.w & 0xffffu));
    const double v0 = __ldg(A.dict + (e.x >> 16)), v1 = __ldg(A.dict + (e.y >> 16));
    const double v2 = __ldg(A.dict + (e.z >> 16)), v3 = __ldg(A.dict + (e.w >> 16));
    if (g + 1 < ng) e = ld_stream4(gp + 4 * (int64_t)T * (g + 1));
    s = fma(v0, x0, s);
    s = fma(v1, x1, s);
    s = fma(v2, x2, s);
    s = fma(v3, x3, s);
  }
  return s;
}

// Loads of a tile that touch only static data (the matrix copy, the block -> subdomain map, row codes).
// k_cg_spmv issues them before griddepcontrol.wait, so they overlap the tail of the previous kernel.
struct TilePre {
  int ls = 0;                    // local subdomain of the tile
  int ng = 0;                    // value-indexed: packed groups of the tile
  const uint32_t* gp = nullptr;  // value-indexed: this row's first packed group
  uint4 e = {0u, 0u, 0u, 0u};    // value-indexed: that group
  uint2 e2 = {0u, 0u};           // variant 10: that group's dictionary indices
  int tb = -1;                   // matrix-free: the row's table code (-1: decode the lattice point)
};

template <bool W = false>  // W: wide entries (12-bit index << 20 | 20-bit signed offset)
__device__ __forceinline__ double tile_row_vi_smem(const SellDev& A, int64_t blk, const double* __restrict__ x,
                                                   const double* sdict, const TilePre* pre = nullptr) {
  constexpr int T = kRowsPerBlock;
  int ng;
  const uint32_t* gp;
  uint4 e;
  if (pre) {
    ng = pre->ng;
    gp = pre->gp;
    e = pre->e;
  } else {
    ng = (A.vtw[blk] + 3) >> 2;
    gp = A.packed + A.poff[blk] + 4 * threadIdx.x;
    if (ng > 0) e = ld_stream4(gp);
  }
  const double* xr = x + blk * T + threadIdx.x;
  double s = 0.0;
  if (ng == 0) return s;
  for (int g = 0; g < ng; ++g) {
    double x0, x1, x2, x3, v0, v1, v2, v3;
    if constexpr (W) {
      x0 = __ldg(xr + ((int32_t)(e.x << 12) >> 12));
      x1 = __ldg(xr + ((int32_t)(e.y << 12) >> 12));
      x2 = __ldg(xr + ((int32_t)(e.z << 12) >> 12));
      x3 = __ldg(xr + ((int32_t)(e.w << 12) >> 12));
      v0 = sdict[e.x >> 20];
      v1 = sdict[e.y >> 20];
      v2 = sdict[e.z >> 20];
      v3 = sdict[e.w >> 20];
    } else {
      x0 = __ldg(xr + (int16_t)(e.x & 0xffffu));
      x1 = __ldg(xr + (int16_t)(e.y & 0xffffu));
      x2 = __ldg(xr + (int16_t)(e.z & 0xffffu));
      x3 = __ldg(xr + (int16_t)(e.w & 0xffffu));
      v0 = sdict[e.x >> 16];
      v1 = sdict[e.y >> 16];
      v2 = sdict[e.z >> 16];
      v3 = sdict[e.w >> 16];
    }
    if (g + 1 < ng) e = ld_stream4(gp + 4 * (int64_t)T * (g + 1));
    s = fma(v0, x0, s);
    s = fma(v1, x1, s);
    s = fma(v2, x2, s);
    s = fma(v3, x3, s);
  }
  return s;
}

// Variant 10 (experimental): 3-byte entries.  Per group of 8 entries one 16-byte load of int16 column
// offsets and one 8-byte load of u8 dictionary indices (25 % fewer matrix bytes than variant 6); the
// dictionary (<= 256 slots) is a kernel parameter.  Same entries in the same order as variant 6, so
// the FMA chain is the same (bitwise-identical rows up to the sign of an exact-zero row sum).
__device__ __forceinline__ uint2 ld_stream2u(const uint2* p) {
  uint2 v;
  asm("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ uint4 ld_stream4u(const uint4* p) {
  uint4 v;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
      : "l"(p));
  return v;
}
__device__ __forceinline__ double tile_row_vi3(const SellDev& A, int64_t blk, const double* __restrict__ x,
                                               const double* dict, const TilePre* pre = nullptr) {
  constexpr int T = kRowsPerBlock;
  const int ng = pre ? pre->ng : (A.vtw[blk] + 7) >> 3;
  // the row's group index: from tile_pre's pointer when given (no dependent load after the wait)
  const int64_t b = pre ? reinterpret_cast<const uint4*>(pre->gp) - A.vi3_off : A.vi3_base[blk] + threadIdx.x;
  const double* xr = x + blk * T + threadIdx.x;
  double s = 0.0;
  if (ng == 0) return s;
  uint4 o;
  uint2 ix;
  if (pre) {  // first group loaded before griddepcontrol.wait (tile_pre)
    o = pre->e;
    ix = pre->e2;
  } else {
    o = ld_stream4u(A.vi3_off + b);
    ix = ld_stream2u(A.vi3_idx + b);
  }
  for (int g = 0; g < ng; ++g) {
    const double x0 = __ldg(xr + (int16_t)(o.x & 0xffffu)), x1 = __ldg(xr + (int16_t)(o.x >> 16));
    const double x2 = __ldg(xr + (int16_t)(o.y & 0xffffu)), x3 = __ldg(xr + (int16_t)(o.y >> 16));
    const double v0 = dict[ix.x & 0xffu], v1 = dict[(ix.x >> 8) & 0xffu];
    const double v2 = dict[(ix.x >> 16) & 0xffu], v3 = dict[ix.x >> 24];
    s = fma(v0, x0, s);
    s = fma(v1, x1, s);
    s = fma(v2, x2, s);
    s = fma(v3, x3, s);
    const double x4 = __ldg(xr + (int16_t)(o.z & 0xffffu)), x5 = __ldg(xr + (int16_t)(o.z >> 16));
    const double x6 = __ldg(xr + (int16_t)(o.w & 0xffffu)), x7 = __ldg(xr + (int16_t)(o.w >> 16));
    const uint32_t iy = ix.y;
    if (g + 1 < ng) {
      o = ld_stream4u(A.vi3_off + b + (int64_t)T * (g + 1));
      ix = ld_stream2u(A.vi3_idx + b + (int64_t)T * (g + 1));
    }
    s = fma(dict[iy & 0xffu], x4, s);
    s = fma(dict[(iy >> 8) & 0xffu], x5, s);
    s = fma(dict[(iy >> 16) & 0xffu], x6, s);
    s = fma(dict[iy >> 24], x7, s);
  }
  return s;
}

// Variant 5: matrix-free Kuhn stencil (row order 4, see MfSub).  The row's lattice point, kind
// and parity class follow from its internal index; its table lists (row offset, value) in column
// order, 4 per group, so the sum is the same FMA chain as the SELL variants (bitwise-identical
// iterations).  Table loads are warp-uniform (one broadcast per group); the x gathers of a warp
// are 32 consecutive rows shifted by one offset: coalesced, with no column indices read.
__device__ __forceinline__ double tile_row_mf(const SellDev& A, int64_t blk, const double* __restrict__ x,
                                              const MfConst& P, const TilePre* pre = nullptr) {
  const int64_t ri = blk * kRowsPerBlock + threadIdx.x;
  double s = 0.0;
#ifndef OSM_MF_NOCODE
  if (P.valid && A.mf_code) {  // the row's 1-byte table code instead of its lattice arithmetic
    const int tb = pre && pre->tb >= 0 ? pre->tb : __ldg(A.mf_code + ri);
    if (tb == 0xff) return s;  // dummy row (Dirichlet or padding point): like a SELL padding row
    const double* xr = x + ri;
    asm("" : "+l"(xr));
#pragma unroll 2
    for (int g = P.gbeg[tb]; g < P.gbeg[tb + 1]; ++g) {
      const int4 d = P.delta[g];
      const double x0 = __ldg(xr + d.x), x1 = __ldg(xr + d.y), x2 = __ldg(xr + d.z), x3 = __ldg(xr + d.w);
      s = fma(P.val[4 * g], x0, s);
      s = fma(P.val[4 * g + 1], x1, s);
      s = fma(P.val[4 * g + 2], x2, s);
      s = fma(P.val[4 * g + 3], x3, s);
    }
    return s;
  }
#endif
  const int ls = A.blk_sub[blk];
  const MfSub& M = A.mf_sub[ls];
  const int t = mf_table_of(M, ri - M.row0);
  if (t < 0) return s;  // dummy row (Dirichlet or padding point): like a SELL padding row
  const double* xr = x + ri;
  asm("" : "+l"(xr));  // keep the row pointer opaque: each gather is then one wide IMAD off it
  if (P.valid) {  // tables in the constant bank
    const int tb = P.tabid[t];
#pragma unroll 2
    for (int g = P.gbeg[tb]; g < P.gbeg[tb + 1]; ++g) {
      const int4 d = P.delta[g];
      const double x0 = __ldg(xr + d.x), x1 = __ldg(xr + d.y), x2 = __ldg(xr + d.z), x3 = __ldg(xr + d.w);
      s = fma(P.val[4 * g], x0, s);
      s = fma(P.val[4 * g + 1], x1, s);
      s = fma(P.val[4 * g + 2], x2, s);
      s = fma(P.val[4 * g + 3], x3, s);
    }
    return s;
  }
  const int g0 = A.mf_begin[t] >> 2, g1 = A.mf_begin[t + 1] >> 2;
  const double2* vv = reinterpret_cast<const double2*>(A.mf_val);
  for (int g = g0; g < g1; ++g) {
    const int4 d = A.mf_delta[g];
    const double2 v01 = vv[2 * g], v23 = vv[2 * g + 1];
    const double x0 = __ldg(xr + d.x), x1 = __ldg(xr + d.y), x2 = __ldg(xr + d.z), x3 = __ldg(xr + d.w);
    s = fma(v01.x, x0, s);
    s = fma(v01.y, x1, s);
    s = fma(v23.x, x2, s);
    s = fma(v23.y, x3, s);
  }
  return s;
}

// V = 2: fp64 SELL rows (LDG streams, registers capped at 32: 8 blocks / 64 warps per SM);
// V = 3: value-indexed rows, dictionary through L1; V = 5: matrix-free Kuhn stencil; V = 6/7:
// value-indexed rows (normal / wide entries), dictionary in the constant bank; V = 10: 3-byte entries.
template <int V>
__device__ __forceinline__ TilePre tile_pre(const SellDev& A, const int32_t* __restrict__ blk_sub, int64_t blk,
                                            const MfArg<V>& mf) {
  TilePre t;
  // volatile loads: the compiler must not sink them below the griddepcontrol.wait that follows
  asm volatile("ld.global.s32 %0, [%1];" : "=r"(t.ls) : "l"(blk_sub + blk));
  if constexpr (V == 6 || V == 7) {
    t.ng = (A.vtw[blk] + 3) >> 2;
    t.gp = A.packed + A.poff[blk] + 4 * threadIdx.x;
    if (t.ng > 0)
      asm volatile("ld.global.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(t.e.x), "=r"(t.e.y), "=r"(t.e.z), "=r"(t.e.w)
                   : "l"(t.gp));
  }
  if constexpr (V == 10) {
    t.ng = (A.vtw[blk] + 7) >> 3;
    t.gp = reinterpret_cast<const uint32_t*>(A.vi3_off + A.vi3_base[blk] + threadIdx.x);
    if (t.ng > 0) {
      asm volatile("ld.global.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(t.e.x), "=r"(t.e.y), "=r"(t.e.z), "=r"(t.e.w)
                   : "l"(t.gp));
      asm volatile("ld.global.L1::no_allocate.v2.u32 {%0, %1}, [%2];"
                   : "=r"(t.e2.x), "=r"(t.e2.y)
                   : "l"(A.vi3_idx + A.vi3_base[blk] + threadIdx.x));
    }
  }
  if constexpr (V == 5) {
    if (mf.c.valid && A.mf_code) {
      unsigned short c;
      asm volatile("ld.global.u8 %0, [%1];" : "=h"(c) : "l"(A.mf_code + blk * kRowsPerBlock + threadIdx.x));
      t.tb = c;
    }
  }
  return t;
}

template <int V>
__device__ __forceinline__ double tile_row(const SellDev& A, int64_t blk, const double* __restrict__ x,
                                           const MfArg<V>& mf, const TilePre* pre = nullptr) {
  if constexpr (V == 3) return tile_row_vi(A, blk, x);
  if constexpr (V == 5) return tile_row_mf(A, blk, x, mf.c, pre);
  if constexpr (V == 6) return tile_row_vi_smem<false>(A, blk, x, mf.dict, pre);
  if constexpr (V == 7) return tile_row_vi_smem<true>(A, blk, x, mf.dict, pre);
  if constexpr (V == 10) return tile_row_vi3(A, blk, x, mf.dict, pre);
  return tile_row_ldg<4>(A, blk, x);
}
#define OSM_SPMV_BOUNDS(V) __launch_bounds__(kThreads, 8)

// ---------------------------------------------------------------- PCG kernels

// q = K_s p ; p.q -> alpha = rho / (p.q), for tile blk (one block)
template <int V, int NW>
__device__ __forceinline__ void spmv_tile(const SellDev& A, int64_t blk, const int32_t* __restrict__ blk_sub,
                                          SubState* __restrict__ st, const double* __restrict__ p,
                                          double* __restrict__ q, double* __restrict__ part, int64_t stride,
                                          int32_t* __restrict__ nactive, const MfArg<V>& mf, double* sm,
                                          const TilePre& pre) {
  const int ls = pre.ls;
  if (!st[ls].active) {  // the previous direction kernel has paid the stopped subdomain's x update
    if (threadIdx.x == 0 && blk == st[ls].blk0) st[ls].xpend = 0;
    return;
  }
  const bool has_row = threadIdx.x < kRowsPerBlock;
  const int64_t row = blk * kRowsPerBlock + threadIdx.x;
  const double y = tile_row<V>(A, blk, p, mf, &pre);
  double v[1] = {0.0};
  if (has_row) {
    q[row] = y;
    v[0] = p[row] * y;
  }
  block_sum<1, NW>(v, sm);
  SubState& S = st[ls];
  if (publish<1>(v, part, stride, blk, &S.cnt, S.nblk)) {
    double t[1];
    gather_partials<1, NW>(t, part, stride, S.blk0, S.nblk, sm);
    if (threadIdx.x == 0) {
      const double pq = t[0];
      S.cnt = 0;
      if (!(pq > 0.0) || !isfinite(pq)) {  // breakdown: p = 0 or loss of definiteness
        S.status = 3;
        S.active = 0;
        atomicSub(nactive, 1);
      } else {
        S.alpha = S.rho / pq;
      }
    }
  }
}

template <int V>
__global__ void OSM_SPMV_BOUNDS(V) k_cg_spmv(SellDev A, const int32_t* __restrict__ blk_sub,
                                                      SubState* __restrict__ st, const double* __restrict__ p,
                                                      double* __restrict__ q, double* __restrict__ part,
                                                      int64_t stride, int32_t* __restrict__ nactive,
                                                      const __grid_constant__ MfArg<V> mf, int64_t blk_base) {
  constexpr int NW = kSlicesPerBlock;
  __shared__ double sm[NW * 1];
  const int64_t blk = blockIdx.x + blk_base;
  const TilePre pre = tile_pre<V>(A, blk_sub, blk, mf);  // static data: before the dependency wait
  pdl_enter();
  spmv_tile<V, NW>(A, blk, blk_sub, st, p, q, part, stride, nactive, mf, sm, pre);
}

// r -= alpha q ; z = D^{-1} r ; r.z, r.r ; stop test ||r|| <= tol ||rhs||; beta.  (x += alpha p moves to
// the direction kernel, which reads p anyway: 8 bytes per row per iteration less.)
// Vector blocks: up to kVecTiles tiles (1024 rows) of one subdomain, 128 threads x 8 rows,
// all loads of a thread issued before any use (memory-level parallelism), one reduction
// and one counter update per 1024 rows.
constexpr int kVecThreads = kRowsPerBlock / 2;
// Matrix-free layout (variant 5): D^{-1} of a row pair from the tables via the rows' 1-byte table
// codes (0xff: dummy row) instead of the 8-byte dinv stream.
__device__ __forceinline__ double2 mf_dinv2(uint16_t cc, const MfConst& P) {
  const int c0 = cc & 0xff, c1 = cc >> 8;
  return make_double2(c0 != 0xff ? P.dinv[c0] : 0.0, c1 != 0xff ? P.dinv[c1] : 0.0);
}

// Loads of static vector data (D^{-1}, row codes) that the vector kernels issue before
// griddepcontrol.wait; volatile and coherent, so ptxas keeps them above the wait.
__device__ __forceinline__ double2 ld_pre2(const double* p) {
  double2 v;
  asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ uint16_t ld_pre_u16(const uint8_t* p) {
  uint16_t v;
  asm volatile("ld.global.u16 %0, [%1];" : "=h"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ld_pre_s32(const int32_t* p) {
  int v;
  asm volatile("ld.global.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

template <int MINB, int V>
__global__ void __launch_bounds__(kVecThreads, MINB) k_cg_update(const int32_t* __restrict__ vblk_sub,
                                                           const int32_t* __restrict__ vblk_tile0,
                                                           const int32_t* __restrict__ vblk_ntile,
                                                           SubState* __restrict__ st, double* __restrict__ x,
                                                           double* __restrict__ r, const double* __restrict__ p,
                                                           const double* __restrict__ q,
                                                           const double* __restrict__ dinv, double* __restrict__ part,
                                                           int64_t stride, double tol, int maxit,
                                                           int32_t* __restrict__ nactive, const uint8_t* __restrict__ mcode,
                                                           const __grid_constant__ MfArg<V> mf, int64_t vb_base,
                                                           int split) {
  constexpr bool MF = V == 5;
  __shared__ double sm[(kVecThreads / 32) * 2];
  const int64_t vb = blockIdx.x + vb_base;
  // static data first (block map, D^{-1} or row codes): issued before the dependency wait
  const int ls = ld_pre_s32(vblk_sub + vb);
  const int nt = ld_pre_s32(vblk_ntile + vb);
  const int64_t p0 = (int64_t)ld_pre_s32(vblk_tile0 + vb) * kVecThreads + threadIdx.x;  // row-pair index
  double2 qv[kVecTiles], rv[kVecTiles], dv[kVecTiles];
  bool real[kVecTiles];
  uint16_t cc[kVecTiles];
#pragma unroll
  for (int j = 0; j < kVecTiles; ++j) {
    real[j] = j < nt;
    if (j < nt) {
      if constexpr (MF) cc[j] = ld_pre_u16(mcode + 2 * (p0 + (int64_t)j * kVecThreads));
      else dv[j] = ld_pre2(dinv + 2 * (p0 + (int64_t)j * kVecThreads));
    }
  }
  pdl_enter();
  if (!st[ls].active) return;
  const double a = st[ls].alpha;
#pragma unroll
  for (int j = 0; j < kVecTiles; ++j)
    if (real[j]) {
      const int64_t i2 = p0 + (int64_t)j * kVecThreads;
      qv[j] = reinterpret_cast<const double2*>(q)[i2];
      rv[j] = reinterpret_cast<const double2*>(r)[i2];
    }
  double v[2] = {0.0, 0.0};
#pragma unroll
  for (int j = 0; j < kVecTiles; ++j)
    if (real[j]) {
      const int64_t i2 = p0 + (int64_t)j * kVecThreads;
      rv[j].x = fma(-a, qv[j].x, rv[j].x);
      rv[j].y = fma(-a, qv[j].y, rv[j].y);
      reinterpret_cast<double2*>(r)[i2] = rv[j];
      if constexpr (MF) dv[j] = mf_dinv2(cc[j], mf.c);  // decoded at use: fewer live registers
      const double z0 = dv[j].x * rv[j].x, z1 = dv[j].y * rv[j].y;
      v[0] += rv[j].x * z0 + rv[j].y * z1;
      v[1] += rv[j].x * rv[j].x + rv[j].y * rv[j].y;
    }
  block_sum<2, kVecThreads / 32>(v, sm);
  SubState& S = st[ls];
  if (split) {  // k_cg_update_fin sums the partials: no atomic, the block retires at once
    if (threadIdx.x == 0) {
      part[vb] = v[0];
      part[stride + vb] = v[1];
    }
    return;
  }
  if (publish<2>(v, part, stride, vb, &S.cnt, S.nvblk)) {
    double t[2];
    gather_partials<2, kVecThreads / 32>(t, part, stride, S.vblk0, S.nvblk, sm);
    if (threadIdx.x == 0) {
      S.cnt = 0;
      const double rz = t[0], rr = t[1];
      S.rr = rr;
      S.iters += 1;
      if (sqrt(rr) <= tol * sqrt(S.bb)) {
        S.status = 1;
        S.active = 0;
        S.xpend = 1;
        atomicSub(nactive, 1);
      } else if (S.iters >= maxit) {
        S.status = 2;
        S.active = 0;
        S.xpend = 1;
        atomicSub(nactive, 1);
      } else {
        S.beta = rz / S.rho;
        S.rho = rz;
      }
    }
  }
}

// The update's per-subdomain step without the last-block atomic: one block (kVecThreads threads, the
// update's own gather order, so the sums are bitwise the same) per subdomain of the group sums the
// vector blocks' (r.z, r.r) partials and takes the stop test and beta.
__global__ void __launch_bounds__(kVecThreads) k_cg_update_fin(SubState* __restrict__ st, const double* __restrict__ part,
                                                               int64_t stride, double tol, int maxit,
                                                               int32_t* __restrict__ nactive, int ls0) {
  __shared__ double sm[(kVecThreads / 32) * 2];
  pdl_enter();
  SubState& S = st[ls0 + blockIdx.x];
  if (!S.active) return;
  double t[2];
  gather_partials<2, kVecThreads / 32>(t, part, stride, S.vblk0, S.nvblk, sm);
  if (threadIdx.x == 0) {
    const double rz = t[0], rr = t[1];
    S.rr = rr;
    S.iters += 1;
    if (sqrt(rr) <= tol * sqrt(S.bb)) {
      S.status = 1;
      S.active = 0;
      S.xpend = 1;
      atomicSub(nactive, 1);
    } else if (S.iters >= maxit) {
      S.status = 2;
      S.active = 0;
      S.xpend = 1;
      atomicSub(nactive, 1);
    } else {
      S.beta = rz / S.rho;
      S.rho = rz;
    }
  }
}

// x += alpha p ; p = D^{-1} r + beta p  (vector blocks as k_cg_update).  A subdomain whose PCG stopped in
// this iteration's update (xpend) only gets its x update.
template <int V>
__global__ void __launch_bounds__(kVecThreads) k_cg_dir(const int32_t* __restrict__ vblk_sub,
                                                        const int32_t* __restrict__ vblk_tile0,
                                                        const int32_t* __restrict__ vblk_ntile,
                                                        const SubState* __restrict__ st, const double* __restrict__ r,
                                                        const double* __restrict__ dinv, double* __restrict__ p,
                                                        double* __restrict__ x, const uint8_t* __restrict__ mcode,
                                                        const __grid_constant__ MfArg<V> mf, int64_t vb_base) {
  constexpr bool MF = V == 5;
  const int64_t vb = blockIdx.x + vb_base;
  // static data first (block map, D^{-1} or row codes): issued before the dependency wait
  const int ls = ld_pre_s32(vblk_sub + vb);
  const int nt = ld_pre_s32(vblk_ntile + vb);
  const int64_t p0 = (int64_t)ld_pre_s32(vblk_tile0 + vb) * kVecThreads + threadIdx.x;
  double2 rv[kVecTiles], dv[kVecTiles], pv[kVecTiles], xv[kVecTiles];
  bool real[kVecTiles];
  uint16_t cc[kVecTiles];
#pragma unroll
  for (int j = 0; j < kVecTiles; ++j) {
    real[j] = j < nt;
    if (j < nt) {
      if constexpr (MF) cc[j] = ld_pre_u16(mcode + 2 * (p0 + (int64_t)j * kVecThreads));
      else dv[j] = ld_pre2(dinv + 2 * (p0 + (int64_t)j * kVecThreads));
    }
  }
  pdl_enter();
  const bool act = st[ls].active;
  if (!act && !st[ls].xpend) return;  // stopped in this iteration's update: only x += alpha p is owed
  const double beta = st[ls].beta, a = st[ls].alpha;
#pragma unroll
  for (int j = 0; j < kVecTiles; ++j)
    if (real[j]) {
      const int64_t i2 = p0 + (int64_t)j * kVecThreads;
      pv[j] = reinterpret_cast<const double2*>(p)[i2];
      xv[j] = reinterpret_cast<const double2*>(x)[i2];
      if (act) rv[j] = reinterpret_cast<const double2*>(r)[i2];
    }
#pragma unroll
  for (int j = 0; j < kVecTiles; ++j)
    if (real[j]) {
      const int64_t i2 = p0 + (int64_t)j * kVecThreads;
      xv[j].x = fma(a, pv[j].x, xv[j].x);  // x_{k+1} = x_k + alpha_k p_k (p_k: before the update below)
      xv[j].y = fma(a, pv[j].y, xv[j].y);
      reinterpret_cast<double2*>(x)[i2] = xv[j];
      if (act) {
        if constexpr (MF) dv[j] = mf_dinv2(cc[j], mf.c);  // decoded at use: fewer live registers
        pv[j].x = fma(beta, pv[j].x, dv[j].x * rv[j].x);
        pv[j].y = fma(beta, pv[j].y, dv[j].y * rv[j].y);
        reinterpret_cast<double2*>(p)[i2] = pv[j];
      }
    }
}

// Warm start: rhs = b + P^T lambda ; r = rhs - K_s x ; z = D^{-1} r ; p = z ;
// rho = r.z, ||r||^2, ||rhs||^2 ; zero rhs -> x = 0 after 0 iterations.
template <int V>
__global__ void OSM_SPMV_BOUNDS(V) k_warm(SellDev A, const int32_t* __restrict__ blk_sub,
                                                   SubState* __restrict__ st, const double* __restrict__ x,
                                                   const double* __restrict__ b, const int32_t* __restrict__ islot,
                                                   const double* __restrict__ lam_all, const double* __restrict__ dinv,
                                                   double* __restrict__ r, double* __restrict__ p,
                                                   double* __restrict__ part, int64_t stride, double tol,
                                                   int32_t* __restrict__ nactive, const __grid_constant__ MfArg<V> mf) {
  constexpr int NW = kSlicesPerBlock;
  __shared__ double sm[NW * 3];
  const int64_t blk = blockIdx.x;
  const int ls = blk_sub[blk];
  const int64_t row = blk * kRowsPerBlock + threadIdx.x;
  const double ax = tile_row<V>(A, blk, x, mf);
  double v[3] = {0.0, 0.0, 0.0};
  if (threadIdx.x < kRowsPerBlock) {
    const int sl = islot[row];
    const double rhs = sl >= 0 ? b[row] + lam_all[sl] : b[row];
    const double rv = rhs - ax;
    const double z = dinv[row] * rv;
    r[row] = rv;
    p[row] = z;
    v[0] = rv * z;
    v[1] = rv * rv;
    v[2] = rhs * rhs;
  }
  block_sum<3, NW>(v, sm);
  SubState& S = st[ls];
  if (publish<3>(v, part, stride, blk, &S.cnt, S.nblk)) {
    double t[3];
    gather_partials<3, NW>(t, part, stride, S.blk0, S.nblk, sm);
    if (threadIdx.x == 0) {
      S.cnt = 0;
      S.rho = t[0];
      S.rr = t[1];
      S.bb = t[2];
      S.iters = 0;
      S.xpend = 0;
      S.alpha = 0.0;  // the fused path's first SpMV then keeps x and forms p = fma(0, p, z) = z
      S.beta = 0.0;
      S.zero_rhs = (t[2] == 0.0);
      if (t[2] == 0.0 || sqrt(t[1]) <= tol * sqrt(t[2])) {
        S.status = 1;
        S.active = 0;
      } else {
        S.status = 0;
        S.active = 1;
        atomicAdd(nactive, 1);
      }
    }
  }
}

__global__ void __launch_bounds__(kThreads) k_zero_if(const int32_t* __restrict__ blk_sub,
                                                      const SubState* __restrict__ st, double* __restrict__ x) {
  const int64_t blk = blockIdx.x;
  const int ls = blk_sub[blk];
  if (!st[ls].zero_rhs) return;
  x[blk * kRowsPerBlock + threadIdx.x] = 0.0;
}

// ---------------------------------------------------------------- Schwarz interface kernels

// Robin data to send: g_{s->t} = (A_s + A_t) u_s|Gamma - lambda_s with
// A = p M_Gamma + q S_Gamma (OO0: q = 0); also the trace u_s|Gamma for gluing.  Discrete
// form of PAPER.md:64-71.
__global__ void k_trace(const SideDev* __restrict__ sides, int64_t nG, const int32_t* __restrict__ mrow,
                        const int32_t* __restrict__ mcol, const double* __restrict__ mval,
                        const double* __restrict__ sval, const double* __restrict__ x) {
  const SideDev S = sides[blockIdx.y];
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= nG) return;
  double mu = 0.0;
  for (int j = mrow[g]; j < mrow[g + 1]; ++j)
    mu = fma(fma(S.alpha_sum, mval[j], S.q_sum * sval[j]), x[S.map[mcol[j]]], mu);
  S.out[g] = mu - S.lam[g];
  S.out[nG + g] = x[S.map[g]];
}

// Receiver side: lambda_t <- g_{s->t} ; keep the neighbour's trace.
__global__ void k_accept(const SideDev* __restrict__ sides, int64_t nG) {
  const SideDev S = sides[blockIdx.y];
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= nG) return;
  S.lam[g] = S.in[g];
  S.unbr[g] = S.in[nG + g];
}

// Glued iterate u~: interface copies averaged; zero = 1 builds u~ = 0.
__global__ void __launch_bounds__(kThreads) k_glue(int64_t nrows, const int32_t* __restrict__ islot,
                                                   const double* __restrict__ x, const double* __restrict__ unbr_all,
                                                   int zero, double* __restrict__ ut) {
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row >= nrows) return;
  if (zero) {
    ut[row] = 0.0;
    return;
  }
  const int sl = islot[row];
  ut[row] = sl >= 0 ? 0.5 * (x[row] + unbr_all[sl]) : x[row];
}

// Glued residual, subdomain part: w = b - K_s u~ ; interior rows add w^2 to
// the subdomain's sum, interface rows keep w for the Robin correction and the owner sum.
template <int V>
__global__ void OSM_SPMV_BOUNDS(V) k_resid(SellDev A, const int32_t* __restrict__ blk_sub,
                                                    SubState* __restrict__ st, const double* __restrict__ ut,
                                                    const double* __restrict__ b, const int32_t* __restrict__ islot,
                                                    double* __restrict__ wif_all, double* __restrict__ part,
                                                    int64_t stride, const __grid_constant__ MfArg<V> mf) {
  constexpr int NW = kSlicesPerBlock;
  __shared__ double sm[NW * 1];
  const int64_t blk = blockIdx.x;
  const int ls = blk_sub[blk];
  const int64_t row = blk * kRowsPerBlock + threadIdx.x;
  const double ax = tile_row<V>(A, blk, ut, mf);
  double v[1] = {0.0};
  if (threadIdx.x < kRowsPerBlock) {
    const double w = b[row] - ax;
    const int sl = islot[row];
    if (sl >= 0) wif_all[sl] = w;
    v[0] = sl == -1 ? w * w : 0.0;
  }
  block_sum<1, NW>(v, sm);
  SubState& S = st[ls];
  if (publish<1>(v, part, stride, blk, &S.cnt, S.nblk)) {
    double t[1];
    gather_partials<1, NW>(t, part, stride, S.blk0, S.nblk, sm);
    if (threadIdx.x == 0) {
      S.cnt = 0;
      S.resid = t[0];
    }
  }
}

// Interface rows: w = b - K^N u~ = (b - K_s u~) + A_own u~|Gamma ; publish w in the outbox.
__global__ void k_iface_w(const SideDev* __restrict__ sides, int64_t nG, const int32_t* __restrict__ mrow,
                          const int32_t* __restrict__ mcol, const double* __restrict__ mval,
                          const double* __restrict__ sval, const double* __restrict__ ut) {
  const SideDev S = sides[blockIdx.y];
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= nG) return;
  double mu = 0.0;
  for (int j = mrow[g]; j < mrow[g + 1]; ++j)
    mu = fma(fma(S.alpha_own, mval[j], S.q_own * sval[j]), ut[S.map[mcol[j]]], mu);
  const double w = S.wif[g] + mu;
  S.wif[g] = w;
  S.out[2 * nG + g] = w;
}

// Owner (left slab) of each interface: sum_g (w_s + w_t)^2 over the plane rows.
__global__ void __launch_bounds__(kThreads) k_iface_sum(const SideDev* __restrict__ sides, int64_t nG,
                                                        double* __restrict__ side_part, int64_t side_nblk,
                                                        uint32_t* __restrict__ side_cnt, double* __restrict__ side_sum) {
  __shared__ double sm[kSlicesPerBlock];
  const int k = blockIdx.y;
  const SideDev S = sides[k];
  if (S.which != 0) return;
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double v[1] = {0.0};
  if (g < nG) {
    const double w = S.wif[g] + S.in[2 * nG + g];
    v[0] = w * w;
  }
  block_sum<1>(v, sm);
  if (publish<1>(v, side_part + k * side_nblk, 0, blockIdx.x, side_cnt + k, (int)gridDim.x)) {
    double t[1];
    gather_partials<1>(t, side_part + k * side_nblk, 0, 0, (int)gridDim.x, sm);
    if (threadIdx.x == 0) {
      side_cnt[k] = 0;
      side_sum[k] = t[0];
    }
  }
}

SellDev sell_of(const Ctx& c) {
  return SellDev{c.sell_val,  c.sell_col,   c.sell_soff,  c.sell_swidth,
                 c.vi_packed, c.vi_poff,     c.vi_tw,      c.vi_dict,    (int)c.vi_ndict,
                 c.blk_sub,   c.d_mf_sub,    c.d_mf_begin, reinterpret_cast<const int4*>(c.d_mf_delta),
                 c.d_mf_val,  c.nrows_total,
                 c.h_mf_const && c.h_mf_const->valid ? c.d_mf_code : nullptr,
                 c.vi3_off,    c.vi3_idx,  c.vi3_base};
}

}  // namespace

// The tile-kernel variant (SELL formats) for v; 11 (bricks) is not a tile format: its warm-start and
// residual products use the best SELL format of the same layout.
static int tile_variant_for(const Ctx& c, int v) {
  if (v == 11) v = 10;
  if (v == 10) {  // 3-byte entries
    if (c.vi_packed_ok && c.vi3_ok && c.vi_ndict <= 256) return 10;
    v = 6;
  }
  if (v == 5) {
    if (c.mf_ok) return 5;
    v = 6;
  }
  if (v == 2) return 2;
  // value-indexed family
  if (!c.vi_packed_ok) return 2;
  if (c.vi_wide) return c.vi_ndict <= kCDict ? 7 : 2;  // wide entries: constant-bank kernel only
  if (v == 7) v = 6;
  if (v == 6) return c.vi_ndict <= kCDict ? 6 : 3;
  return 3;
}

int spmv_variant_of(const Ctx& c) {
  if (c.spmv_variant == 11 && c.brick_ok) return 11;
  return tile_variant_for(c, c.spmv_variant);
}

static int tile_variant_of(const Ctx& c) { return tile_variant_for(c, c.spmv_variant); }

template <int V>
static MfArg<V> mf_arg(const Ctx& c) {
  MfArg<V> a{};
  if constexpr (V == 5) {
    if (c.h_mf_const) a.c = *c.h_mf_const;
  }
  if constexpr (V == 6 || V == 7)
    std::copy(c.h_vi_dict.begin(), c.h_vi_dict.begin() + std::min<size_t>(kCDict, c.h_vi_dict.size()), a.dict);
  if constexpr (V == 10)
    std::copy(c.h_vi_dict.begin(), c.h_vi_dict.begin() + std::min<size_t>(256, c.h_vi_dict.size()), a.dict);
  return a;
}

template <int V>
static void warm_v(Ctx& c, double tol) {
  k_warm<V><<<(unsigned)c.nblk_total, kThreads, 0, c.stream>>>(sell_of(c), c.blk_sub, c.st, c.x, c.b, c.islot,
                                                                      c.lam_all, c.dinv, c.r, c.p, c.part,
                                                                      c.nblk_total, tol, c.d_nactive, mf_arg<V>(c));
}

void launch_warm(Ctx& c, double tol, int) {
  timer_begin(c, T_WARM);
  switch (tile_variant_of(c)) {
    case 3: warm_v<3>(c, tol); break;
    case 5: warm_v<5>(c, tol); break;
    case 6: warm_v<6>(c, tol); break;
    case 7: warm_v<7>(c, tol); break;
    case 10: warm_v<10>(c, tol); break;
    default: warm_v<2>(c, tol); break;
  }
  OSM_CHECK_LAUNCH();
  ++c.launches;
  timer_end(c, T_WARM);
}

void launch_zero_if(Ctx& c) {
  k_zero_if<<<(unsigned)c.nblk_total, kThreads, 0, c.stream>>>(c.blk_sub, c.st, c.x);
  OSM_CHECK_LAUNCH();
  ++c.launches;
}

// Stream and block ranges of the group being launched (Ctx::grp_cur; -1: every local subdomain).
static cudaStream_t launch_stream(const Ctx& c) { return c.grp_cur >= 0 ? c.gstream[c.grp_cur] : c.stream; }
static int64_t grp_blk0(const Ctx& c) { return c.grp_cur >= 0 ? c.g_blk0[c.grp_cur] : 0; }
static int64_t grp_nblk(const Ctx& c) { return c.grp_cur >= 0 ? c.g_nblk[c.grp_cur] : c.nblk_total; }
static int64_t grp_vb0(const Ctx& c) { return c.grp_cur >= 0 ? c.g_vb0[c.grp_cur] : 0; }
static int64_t grp_nvb(const Ctx& c) { return c.grp_cur >= 0 ? c.g_nvb[c.grp_cur] : c.nvblk_total; }

template <typename... KArgs, typename... Args>
static void launch_pdl(const Ctx& c, void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem,
                       Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = launch_stream(c);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  OSM_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
}

template <int V>
static void cg_spmv_v(Ctx& c) {
  launch_pdl(c, k_cg_spmv<V>, (unsigned)grp_nblk(c), kThreads, (size_t)0, sell_of(c), (const int32_t*)c.blk_sub, c.st,
             (const double*)c.p, c.q, c.part, c.nblk_total, c.d_nactive, mf_arg<V>(c), grp_blk0(c));
}

void launch_cg_spmv(Ctx& c) {
  timer_begin(c, T_SPMV);
  switch (spmv_variant_of(c)) {
    case 11:
      launch_cg_spmv_brick(c, launch_stream(c), c.grp_cur);
      if (c.brick_kernel > 0) ++c.launches;  // + k_brick_alpha
      break;
    case 3: cg_spmv_v<3>(c); break;
    case 5: cg_spmv_v<5>(c); break;
    case 6: cg_spmv_v<6>(c); break;
    case 7: cg_spmv_v<7>(c); break;
    case 10: cg_spmv_v<10>(c); break;
    default: cg_spmv_v<2>(c); break;
  }
  ++c.launches;
  timer_end(c, T_SPMV);
}

// The vector kernels take D^{-1} from the matrix-free tables (and skip pairs of dummy rows) when
// variant 5 runs with its tables in the constant bank.
static bool mf_vectors(const Ctx& c) {
  const int v = spmv_variant_of(c);
  return (v == 5 || v == 8) && c.h_mf_const && c.h_mf_const->valid && c.d_mf_code;
}

// SELL variants with D^{-1} codes (osm.cu dcode_build): the vector kernels' table path (V = 5) with the
// codes of the distinct D^{-1} values in place of the matrix-free table codes.
static bool dcode_vectors(const Ctx& c) { return !c.h_dcode_tab.empty() && c.d_dcode; }
static MfArg<5> dcode_arg(const Ctx& c) {
  MfArg<5> a{};
  a.c.valid = 1;
  std::copy(c.h_dcode_tab.begin(), c.h_dcode_tab.end(), a.c.dinv);
  return a;
}

template <int MINB, int V>
static void cg_update_v(Ctx& c, double tol, int maxit, const uint8_t* code, const MfArg<V>& mf) {
  launch_pdl(c, k_cg_update<MINB, V>, (unsigned)grp_nvb(c), kVecThreads, (size_t)0, (const int32_t*)c.vblk_sub,
             (const int32_t*)c.vblk_tile0, (const int32_t*)c.vblk_ntile, c.st, c.x, c.r, (const double*)c.p,
             (const double*)c.q, (const double*)c.dinv, c.part_upd, c.nvblk_total, tol, maxit, c.d_nactive, code,
             mf, grp_vb0(c), c.split_update ? 1 : 0);
  if (c.split_update) {
    const int nloc = c.s_end - c.s_begin;
    int s0 = 0, s1 = nloc;
    if (c.grp_cur >= 0) {
      s0 = c.grp_cur * nloc / c.ngroups;
      s1 = (c.grp_cur + 1) * nloc / c.ngroups;
    }
    launch_pdl(c, k_cg_update_fin, (unsigned)(s1 - s0), kVecThreads, (size_t)0, c.st, (const double*)c.part_upd,
               c.nvblk_total, tol, maxit, c.d_nactive, s0);
    ++c.launches;
  }
}

void launch_cg_update(Ctx& c, double tol, int maxit) {
  timer_begin(c, T_UPDATE);
  if (mf_vectors(c))
    cg_update_v<1, 5>(c, tol, maxit, c.d_mf_code, mf_arg<5>(c));
  else if (dcode_vectors(c))
    cg_update_v<1, 5>(c, tol, maxit, c.d_dcode, dcode_arg(c));
  else if (c.update_variant == 1)
    cg_update_v<8, 0>(c, tol, maxit, nullptr, mf_arg<0>(c));
  else
    cg_update_v<1, 0>(c, tol, maxit, nullptr, mf_arg<0>(c));
  ++c.launches;
  timer_end(c, T_UPDATE);
}

template <int V>
static void cg_dir_v(Ctx& c, const uint8_t* code, const MfArg<V>& mf) {
  launch_pdl(c, k_cg_dir<V>, (unsigned)grp_nvb(c), kVecThreads, (size_t)0, (const int32_t*)c.vblk_sub,
             (const int32_t*)c.vblk_tile0, (const int32_t*)c.vblk_ntile, (const SubState*)c.st, (const double*)c.r,
             (const double*)c.dinv, c.p, c.x, code, mf, grp_vb0(c));
}

// The Kuhn brick SpMV carries the direction update (BrickFuse): it needs the D^{-1} codes and the p2
// buffer (brick.cu builds it with the Kuhn kernel).
bool fused_dir(const Ctx& c) {
  return c.fuse_dir && spmv_variant_of(c) == 11 && c.brick_kernel > 0 && c.p2 && dcode_vectors(c) &&
         c.h_dcode_tab.size() <= (size_t)kMfMaxTab;
}

// k_cg_dir once after a batched PCG run of the fused path: x += alpha p for a subdomain that stopped
// in the last update of the run (xpend) with no SpMV after it.  p_k is in Ctx::p (chunks hold an even
// number of iterations); an already paid x has xpend cleared by k_brick_alpha.
void launch_cg_dir_flush(Ctx& c) {
  if (!fused_dir(c)) return;
  c.cg_par = 0;
  timer_begin(c, T_DIR);
  cg_dir_v<5>(c, c.d_dcode, dcode_arg(c));
  ++c.launches;
  timer_end(c, T_DIR);
}

void launch_cg_dir(Ctx& c) {
  if (fused_dir(c)) {  // done by the next SpMV
    c.cg_par ^= 1;
    return;
  }
  timer_begin(c, T_DIR);
  if (mf_vectors(c))
    cg_dir_v<5>(c, c.d_mf_code, mf_arg<5>(c));
  else if (dcode_vectors(c))
    cg_dir_v<5>(c, c.d_dcode, dcode_arg(c));
  else
    cg_dir_v<0>(c, nullptr, mf_arg<0>(c));
  ++c.launches;
  timer_end(c, T_DIR);
}

void launch_trace(Ctx& c) {
  if (c.sides.empty()) return;
  dim3 grid((unsigned)ceil_div(c.nG, 256), (unsigned)c.sides.size());
  k_trace<<<grid, 256, 0, c.stream>>>(c.d_sides, c.nG, c.d_mrow, c.d_mcol, c.d_mval, c.d_sval, c.x);
  OSM_CHECK_LAUNCH();
  ++c.launches;
}

void launch_accept(Ctx& c) {
  if (c.sides.empty()) return;
  dim3 grid((unsigned)ceil_div(c.nG, 256), (unsigned)c.sides.size());
  k_accept<<<grid, 256, 0, c.stream>>>(c.d_sides, c.nG);
  OSM_CHECK_LAUNCH();
  ++c.launches;
}

void launch_glue(Ctx& c, int zero) {
  k_glue<<<(unsigned)ceil_div(c.nrows_total, 256), 256, 0, c.stream>>>(c.nrows_total, c.islot, c.x, c.unbr_all, zero,
                                                                         c.ut);
  OSM_CHECK_LAUNCH();
  ++c.launches;
}

template <int V>
static void resid_v(Ctx& c) {
  k_resid<V><<<(unsigned)c.nblk_total, kThreads, 0, c.stream>>>(
      sell_of(c), c.blk_sub, c.st, c.ut, c.b, c.islot, c.wif_all, c.part, c.nblk_total, mf_arg<V>(c));
}

void launch_resid(Ctx& c) {
  timer_begin(c, T_RESID);
  switch (tile_variant_of(c)) {
    case 3: resid_v<3>(c); break;
    case 5: resid_v<5>(c); break;
    case 6: resid_v<6>(c); break;
    case 7: resid_v<7>(c); break;
    case 10: resid_v<10>(c); break;
    default: resid_v<2>(c); break;
  }
  OSM_CHECK_LAUNCH();
  ++c.launches;
  timer_end(c, T_RESID);
}

void launch_iface_w(Ctx& c) {
  if (c.sides.empty()) return;
  dim3 grid((unsigned)ceil_div(c.nG, 256), (unsigned)c.sides.size());
  k_iface_w<<<grid, 256, 0, c.stream>>>(c.d_sides, c.nG, c.d_mrow, c.d_mcol, c.d_mval, c.d_sval, c.ut);
  OSM_CHECK_LAUNCH();
  ++c.launches;
}

void launch_iface_sum(Ctx& c) {
  if (c.sides.empty()) return;
  dim3 grid((unsigned)c.side_nblk, (unsigned)c.sides.size());
  k_iface_sum<<<grid, kThreads, 0, c.stream>>>(c.d_sides, c.nG, c.side_part, c.side_nblk, c.side_cnt, c.side_sum);
  OSM_CHECK_LAUNCH();
  ++c.launches;
}

}  // namespace osm

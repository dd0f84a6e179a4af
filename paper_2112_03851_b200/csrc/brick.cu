// Brick SpMV (variant 11, row order 6): the PCG product q = K_s p as a shared-memory stencil.
//
// PAPER.md:165-167 ("the coefficient matrices are stored in CSR format ... sparse matrix-vector
// multiplication"): the hot loop's SpMV.  On the Kuhn box mesh every row couples only lattice points
// within +-o of itself (o = element order), so the x gathers of a row-wise CSR/SELL SpMV re-read
// each p value ~27 times through L1/L2 (round-1 measurements: the gathers, not the matrix stream,
// bound variants 6/10).  Here each CTA stages the p values of a lattice brick plus a one-point halo
// in shared memory with TMA (cp.async.bulk.tensor, OOB zero fill = the Dirichlet neighbours), and
// every gather becomes a conflict-free shared-memory load.  The matrix is still streamed from HBM:
// one u8 dictionary index per (row, stencil slot) -- the value-indexed dictionary of vi.cu, <= 256
// slots, in the constant bank -- in the column order of the row, so each row's FMA chain is the
// same sequence as the SELL rows' (bitwise-identical q).
//
// Layout (row order 6, osm.cu assemble): per subdomain, the o^3 lattice parity classes are stored
// one after another; class c is a dense array over its class-local coordinates (jj fastest, then
// ii, then kk), jj = J div o - 1 div o, ii = I div o - I_lo div o, kk = K div o - 1 div o, with the
// jj extent padded to even (16-byte TMA strides; the pad rows are inert zero rows).  A stencil
// neighbour (dI, dJ, dK) of a class-c point is at class-local offset (I + dI) div o - I div o in
// {-1, 0, 1} per axis, in class c' -- so a brick of class-local extent BJ x BI x BK needs, for
// every class, the box extended by one point on each side: one TMA box per class.
//
// Work: one CTA per brick; warps take 32-point chunks of one class box (warp-uniform stencil);
// p.q is reduced per brick (warp tree, block tree, one partial per brick, the last brick of a
// subdomain sums them in brick order and forms alpha = rho / p.q) -- deterministic, independent of
// the number of subdomains or GPUs.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <type_traits>
#include <vector>

#include "ctx.h"
#include "kuhn_slots.h"  // generated at build time by gen_kuhn_slots.cpp

namespace osm {

namespace {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ double warp_sum_b(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Union of the stencil offsets that carry a nonzero (or Robin-fold) value, per class:
// flag[c * 125 + code], code = (dI + 2) + 5 (dJ + 2) + 25 (dK + 2).
__global__ void k_brick_mark(const BrickBuildDev D, const int64_t* __restrict__ toff,
                             const int32_t* __restrict__ twidth, const int32_t* __restrict__ col,
                             const uint16_t* __restrict__ vidx, uint32_t zero_idx, int32_t* __restrict__ flag) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= D.nrows) return;
  const int ls = D.row_sub[r];
  if (ls < 0) return;
  const int32_t lc = D.perm[r];
  if (lc < 0) return;
  const BrickSub& B = D.sub[ls];
  int I, J, K;
  brick_lattice_of(B, lc, I, J, K);
  const int c = brick_class(D.o, I, J, K);
  const int64_t t = r / kRowsPerBlock, l = r % kRowsPerBlock;
  const int w = twidth[t];
  for (int k = 0; k < w; ++k) {
    const int64_t i = toff[t] + (int64_t)kRowsPerBlock * k + l;
    if (vidx[i] == zero_idx) continue;
    const int32_t lc2 = D.perm[col[i]];
    int I2, J2, K2;
    brick_lattice_of(B, lc2, I2, J2, K2);
    const int code = (I2 - I + 2) + 5 * (J2 - J + 2) + 25 * (K2 - K + 2);
    flag[c * 125 + code] = 1;
  }
}

// The u8 index stream: for every real row, its kept entries are matched (in column order) to the
// slots of its class; unmatched slots keep the index of 0.0.  An entry without a slot sets *bad.
__global__ void k_brick_pack(const BrickBuildDev D, const int64_t* __restrict__ toff,
                             const int32_t* __restrict__ twidth, const int32_t* __restrict__ col,
                             const uint16_t* __restrict__ vidx, uint32_t zero_idx,
                             const int16_t* __restrict__ slot_of, uint8_t* __restrict__ stream,
                             int32_t* __restrict__ bad) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= D.nrows) return;
  const int ls = D.row_sub[r];
  if (ls < 0) return;
  const int32_t lc = D.perm[r];
  if (lc < 0) return;
  const BrickSub& B = D.sub[ls];
  int I, J, K;
  brick_lattice_of(B, lc, I, J, K);
  const int c = brick_class(D.o, I, J, K);
  // class-local coordinates -> brick, chunk (il) and lane (jl + 8 kl) in the brick kernel
  const int jj = J / D.o - 1 / D.o, ii = I / D.o - B.I_lo / D.o, kk = K / D.o - 1 / D.o;
  const int bj = jj / D.BJ, bi = ii / D.BI, bk = kk / D.BK;
  const int64_t b = B.brick0 + bj + (int64_t)B.nbj * (bi + (int64_t)B.nbi * bk);
  const int il = ii - bi * D.BI, lane = (jj - bj * D.BJ) + D.BJ * (kk - bk * D.BK);
  const int64_t base = b * D.brick_words + 32 * ((int64_t)D.goff[c] + (int64_t)il * D.ngrp[c]) + lane;
  const int ns = 4 * D.ngrp[c];
  auto at = [&](int j) -> uint8_t& { return stream[4 * (base + 32 * (int64_t)(j >> 2)) + (j & 3)]; };
  for (int j = 0; j < ns; ++j) at(j) = (uint8_t)zero_idx;
  const int64_t tt = r / kRowsPerBlock, l = r % kRowsPerBlock;
  const int w = twidth[tt];
  int last = -1;
  for (int k = 0; k < w; ++k) {
    const int64_t i = toff[tt] + (int64_t)kRowsPerBlock * k + l;
    if (vidx[i] == zero_idx) continue;
    const int32_t lc2 = D.perm[col[i]];
    int I2, J2, K2;
    brick_lattice_of(B, lc2, I2, J2, K2);
    const int code = (I2 - I + 2) + 5 * (J2 - J + 2) + 25 * (K2 - K + 2);
    const int j = slot_of[c * 125 + code];
    if (j < 0 || j <= last) {  // no slot, or out of column order
      atomicAdd(bad, 1);
      return;
    }
    at(j) = (uint8_t)vidx[i];
    last = j;
  }
}

// Row types of the Kuhn layout: one warp per chunk (brick, class, il).  The chunk is uniform when
// every lane whose point is a row holds the same index words (lanes off the class range are never
// stored); out: uni[chunk] and the words of the first row lane (words[chunk][0..ng)).
__global__ void k_brick_chunks(const BrickBuildDev D, const BrickInfo* __restrict__ info,
                               const uint32_t* __restrict__ stream, int BI, int64_t nchunk,
                               uint32_t* __restrict__ words, int32_t* __restrict__ uni) {
  const int64_t ch = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (ch >= nchunk) return;  // whole warps
  const int64_t b = ch / (8 * BI);
  const int r = (int)(ch % (8 * BI)), c = r / BI, il = r % BI;
  const BrickInfo I = info[b];
  const BrickClass& C = D.sub[I.ls].cls[c];
  const int jj = I.bj * D.BJ + (lane & 15), ii = I.bi * BI + il, kk = I.bk * D.BK + (lane >> 4);
  const bool valid = jj >= C.jjlo && jj <= C.jjhi && ii >= C.iilo && ii <= C.iihi && kk >= C.kklo && kk <= C.kkhi;
  const int ng = D.ngrp[c];
  const uint32_t* p = stream + b * D.brick_words + 32 * ((int64_t)D.goff[c] + (int64_t)il * ng) + lane;
  const unsigned vmask = __ballot_sync(0xffffffffu, valid);
  const int src = vmask ? __ffs(vmask) - 1 : 0;
  bool same = true;
  for (int g = 0; g < ng; ++g) {
    const uint32_t w = p[32 * g];
    const uint32_t w0 = __shfl_sync(0xffffffffu, w, src);
    same = same && (!valid || w == w0);
    if (lane == 0) words[ch * 16 + g] = w0;
  }
  const bool all = __all_sync(0xffffffffu, same);
  if (lane == 0) uni[ch] = all ? 1 : 0;
}

// Copies the per-lane words of the non-uniform chunks into the compact stream (one warp per chunk).
__global__ void k_brick_compact(const BrickBuildDev D, const uint32_t* __restrict__ stream, int BI,
                                const int64_t* __restrict__ src_chunk, const int64_t* __restrict__ dst_group,
                                int64_t n, uint32_t* __restrict__ cstream) {
  const int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (k >= n) return;
  const int64_t ch = src_chunk[k];
  const int64_t b = ch / (8 * BI);
  const int r = (int)(ch % (8 * BI)), c = r / BI, il = r % BI;
  const int ng = D.ngrp[c];
  const uint32_t* p = stream + b * D.brick_words + 32 * ((int64_t)D.goff[c] + (int64_t)il * ng) + lane;
  uint32_t* q = cstream + 32 * dst_group[k] + lane;
  for (int g = 0; g < ng; ++g) q[32 * g] = p[32 * g];
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t phase) {
  uint32_t done;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(phase)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_addr(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_addr(bar))
      : "memory");
}


constexpr int kBrickThreads = 256;
constexpr int kMaxDynSmem = 220 * 1024;  // dynamic shared memory budget of a brick CTA (sm_100 opt-in: 227 KB)
constexpr int kMaxSlotGroups = 24;   // slot groups (4 slots) per class: P2 vertex rows need 14

__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

// ---- compile-time geometry of the P2 brick (BJ = 16, BK = 2; class boxes (20, BI + 2, 4))
constexpr int box_stride_of(int BI) { return (20 * (BI + 2) * 4 + 15) / 16 * 16; }
constexpr int jsh_of(int c) { return ((c >> 1) & 1) ? 1 : 0; }  // class box column of jj = -1 (see brick_build)
// byte offset of stencil slot j of class c from the point's own element (kKuhnSlots, gen_kuhn_slots.cpp)
constexpr int kuhn_off(int c, int j, int BI) {
  const int pi = c & 1, pj = (c >> 1) & 1, pk = c >> 2;
  const int dx = kKuhnSlots[c][j][0], dy = kKuhnSlots[c][j][1], dz = kKuhnSlots[c][j][2];
  const int vi = 2 + pi + dx, vj = 2 + pj + dy, vk = 2 + pk + dz;  // floor division of non-negative values
  const int dii = vi / 2 - (2 + pi) / 2, djj = vj / 2 - (2 + pj) / 2, dkk = vk / 2 - (2 + pk) / 2;
  const int cn = (vi % 2) + 2 * ((vj % 2) + 2 * (vk % 2));
  return 8 * ((cn - c) * box_stride_of(BI) + jsh_of(cn) - jsh_of(c) + djj + 20 * (dii + (BI + 2) * dkk));
}
template <int C, int BI>
struct KuhnOffsets {
  static constexpr int n = kKuhnSlotCount[C];
  static constexpr int ng = (n + 3) / 4;
  int v[4 * 16];
  constexpr KuhnOffsets() : v() {
    for (int j = 0; j < 4 * ng; ++j) v[j] = j < n ? kuhn_off(C, j, BI) : 0;
  }
};

// One chunk of class C (32 points at one ii: lane = jl + 16 kl), compile-time slot offsets: each
// slot is one shared-memory load at an immediate offset, a byte extract, a dictionary load and an FMA.
template <int C, int BI>
__device__ __forceinline__ double kuhn_chunk(uint32_t xc, const uint32_t (&w)[16], const double* dict) {
  constexpr KuhnOffsets<C, BI> T{};
  double s = 0.0;
#pragma unroll
  for (int g = 0; g < T.ng; ++g) {
    const uint32_t v = w[g];
    const double x0 = lds_f64(xc + T.v[4 * g]), x1 = lds_f64(xc + T.v[4 * g + 1]);
    const double x2 = lds_f64(xc + T.v[4 * g + 2]), x3 = lds_f64(xc + T.v[4 * g + 3]);
    s = fma(dict[v & 0xffu], x0, s);
    s = fma(dict[(v >> 8) & 0xffu], x1, s);
    s = fma(dict[(v >> 16) & 0xffu], x2, s);
    s = fma(dict[v >> 24], x3, s);
  }
  return s;
}

// Generic chunk: runtime slot offsets (bytes) and group count.
__device__ __forceinline__ double chunk_dot(uint32_t xc, const uint32_t (&w)[16], const int* so, const double* dict,
                                            int ng) {
  double s = 0.0;
#pragma unroll
  for (int g = 0; g < 16; ++g) {
    if (g < ng) {
      const uint32_t v = w[g];
      const double x0 = lds_f64(xc + so[4 * g]), x1 = lds_f64(xc + so[4 * g + 1]);
      const double x2 = lds_f64(xc + so[4 * g + 2]), x3 = lds_f64(xc + so[4 * g + 3]);
      s = fma(dict[v & 0xffu], x0, s);
      s = fma(dict[(v >> 8) & 0xffu], x1, s);
      s = fma(dict[(v >> 16) & 0xffu], x2, s);
      s = fma(dict[v >> 24], x3, s);
    }
  }
  return s;
}

// Generic brick kernel (any order, slots not on the P2 Kuhn lists): one CTA per brick; the p boxes of
// its classes arrive by TMA after the PDL wait; the index stream is read from global memory, the next
// chunk's words in flight while a chunk computes.  Chunks (class c, il) go round robin to the 8 warps,
// with runtime slot offsets and group counts.
template <int NC>
__global__ void __launch_bounds__(kBrickThreads) k_cg_spmv_brick(
    const BrickDev D, const __grid_constant__ BrickArg a, SubState* __restrict__ st, double* __restrict__ q,
    double* __restrict__ part, int32_t* __restrict__ nactive, int64_t b0) {
  extern __shared__ __align__(128) unsigned char bsm_raw[];
  // TMA destinations must be 128-byte aligned in the shared window; the dynamic segment follows the
  // static one, so align by hand (the launch adds 128 bytes)
  unsigned char* bsm = bsm_raw + ((128u - (smem_addr(bsm_raw) & 127u)) & 127u);
  const uint32_t xs_addr = smem_addr(bsm);
  uint64_t* bar = reinterpret_cast<uint64_t*>(bsm + NC * a.box_bytes);
  constexpr int NT = kBrickThreads, NW = NT / 32;
  __shared__ double red[NW];
  __shared__ int flag;
  const int64_t b = b0 + blockIdx.x;
  const BrickInfo bi = D.info[b];  // static: before the dependency wait
  const BrickSub& B = D.sub[bi.ls];
  const int lane = threadIdx.x & 31;
  const int warp = __reduce_max_sync(0xffffffffu, (unsigned)(threadIdx.x >> 5));
  const int BI = a.BI;
  const int nch = NC * BI;
  const uint32_t* ws = D.stream + b * a.brick_words + lane;
  uint32_t wa[16], wb[16];
  auto load_words = [&](uint32_t (&w)[16], int ch) {
    if (ch >= nch) return;
    const int c = ch / BI, il = ch - c * BI;
    const int ng = a.ngrp[c];
    const uint32_t* p = ws + 32 * (a.goff[c] + il * ng);
#pragma unroll
    for (int g = 0; g < 16; ++g)
      if (g < ng) w[g] = __ldg(p + 32 * g);
  };
  load_words(wa, warp);
  // the box barrier is initialised (and the tensor maps prefetched) before the dependency wait, so
  // that both overlap the previous kernel's tail
  if (warp == 0) {
    if (lane == 0) mbar_init(bar, 1);
    if (lane < NC) asm volatile("prefetch.tensormap [%0];" ::"l"(D.tmap + bi.ls * NC + lane) : "memory");
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();  // barrier initialised
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  SubState& S = st[bi.ls];
  if (!S.active) {  // the previous direction kernel has paid the stopped subdomain's x update
    if (threadIdx.x == 0 && b == S.brick0) S.xpend = 0;
    return;
  }
  // one lane of warp 0 per class issues its box (every class's stencil reaches into all 8 boxes, so
  // one barrier covers them); lane 0 arms it before the loads
  if (warp == 0) {
    if (lane == 0) mbar_expect_tx(bar, (uint32_t)(NC * a.box_elems * 8));
    __syncwarp();
    if (lane < NC) {
      const int c = lane;
      const int j0 = bi.bj * 16 - 1, i0 = bi.bi * BI - 1, k0 = bi.bk * 2 - 1;
      const BrickClass& C = B.cls[c];
      // innermost TMA coordinates must be 16-byte aligned (even): the class box starts a.jsh[c] early
      tma_load_3d(reinterpret_cast<double*>(bsm) + c * a.box_stride, D.tmap + bi.ls * NC + c,
                  j0 - C.jjlo - a.jsh[c], i0 - C.iilo, k0 - C.kklo, bar);
    }
  }
  // this lane's point in a class box (BJ = 16, BK = 2: lane = jl + 16 kl), box dims (20, BI + 2, 4)
  const int jl = lane & 15, kl = lane >> 4;
  const uint32_t lane_off = 8u * (uint32_t)((jl + 1) + 20 * (BI + 2) * (kl + 1));
  mbar_wait_parity(bar, 0);
  double pq = 0.0;
  auto compute = [&](const uint32_t (&w)[16], int ch) {
    const int c = ch / BI, il = ch - c * BI;
    const BrickClass& C = B.cls[c];
    const uint32_t xc = xs_addr + 8u * (uint32_t)(c * a.box_stride + a.jsh[c] + 20 * (il + 1)) + lane_off;
    const double s = chunk_dot(xc, w, a.soff + c * 4 * kMaxSlotGroups, a.dict, a.ngrp[c]);
    const int jj = bi.bj * 16 + jl, ii = bi.bi * BI + il, kk = bi.bk * 2 + kl;
    if (jj >= C.jjlo && jj <= C.jjhi && ii >= C.iilo && ii <= C.iihi && kk >= C.kklo && kk <= C.kkhi) {
      const int64_t row =
          B.row0 + C.base + (jj - C.jjlo) + (int64_t)C.nJp * ((ii - C.iilo) + (int64_t)C.nIc * (kk - C.kklo));
      q[row] = s;
      pq = fma(lds_f64(xc), s, pq);
    }
  };
  {
    for (int ch = warp; ch < nch; ch += 2 * NW) {
      load_words(wb, ch + NW);
      compute(wa, ch);
      if (ch + NW >= nch) break;
      load_words(wa, ch + 2 * NW);
      compute(wb, ch + NW);
    }
  }
  // p.q: warp tree, warps in order, one partial per brick; the last brick of the subdomain sums them
  pq = warp_sum_b(pq);
  if (lane == 0) red[warp] = pq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int w = 0; w < NW; ++w) v += red[w];
    part[b] = v;
    __threadfence();
    flag = atomicAdd(&S.cnt, 1u) == (uint32_t)S.nbrick - 1;
  }
  __syncthreads();
  if (!flag) return;
  __threadfence();
  double v = 0.0;  // fixed-order sum of the subdomain's brick partials: strided, then the block tree
  for (int64_t m = threadIdx.x; m < S.nbrick; m += NT) v += __ldcg(part + S.brick0 + m);
  v = warp_sum_b(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double pqs = 0.0;
    for (int w = 0; w < NW; ++w) pqs += red[w];
    S.cnt = 0;
    if (!(pqs > 0.0) || !isfinite(pqs)) {  // breakdown: p = 0 or loss of definiteness
      S.status = 3;
      S.active = 0;
      atomicSub(nactive, 1);
    } else {
      S.alpha = S.rho / pqs;
    }
  }
}

// ---- the P2 Kuhn kernel: one warp per x plane il of the brick (BI warps), each warp running the 8
// classes in a fixed compile-time sequence.  Every class is then a straight line of immediates: the
// stream words of chunk (C, il) at a compile-time offset plus il times a constant, the slot offsets
// as LDS immediates, the row of the result from per-class brick constants staged in shared memory.
// Every warp does the same work (one chunk of each class: the 53 slot groups of the Kuhn stencil), so
// the CTA has no load imbalance, and the next class's index words are two classes in flight.
template <int C>
constexpr int kuhn_ng() {
  return (kKuhnSlotCount[C] + 3) / 4;
}
// The index words of chunk (C, il): a row type's words (the same address in every lane: one
// broadcast transaction) or the chunk's per-lane words in the compact stream.
template <int C>
__device__ __forceinline__ void kuhn_words(uint32_t (&w)[16], const BrickDev& D, int d, int lane) {
  constexpr int ng = kuhn_ng<C>();
  if (d >= 0) {  // a row type: the same ng consecutive words in every lane (broadcast loads)
    const uint32_t* p = D.typetab + 16 * (int64_t)d;
#pragma unroll
    for (int g = 0; g < ng; ++g) w[g] = __ldg(p + g);
  } else {  // per-lane words, lane-interleaved: immediate offsets
    const uint32_t* p = D.cstream + 32 * (int64_t)(-d - 1) + lane;
#pragma unroll
    for (int g = 0; g < ng; ++g) w[g] = __ldg(p + 32 * g);
  }
}
template <int C>
using IC = std::integral_constant<int, C>;

// Dynamic shared memory of k_cg_spmv_kuhn<BI>: the class boxes (128-byte aligned by hand) and the
// mbarrier; the reduction slots are static
constexpr int kuhn_smem_bytes(int BI) { return 8 * box_stride_of(BI) * 8 + 16 + 128; }
// FUSE: the PCG direction update rides on the SpMV (BrickFuse, ctx.h).  After the boxes of p_k land,
// the CTA pays x_{k+1} = x_k + alpha_k p_k on its own rows (p_k from shared memory), then forms
// p_{k+1} = fma(beta_k, p_k, D^{-1} r_{k+1}) in place on every staged point -- the halo too, whose
// values other CTAs form identically -- and the stencil runs on p_{k+1}; own rows of p_{k+1} go to the
// other p buffer.  Bitwise the same x, p and q as k_cg_dir followed by the plain kernel.
template <int BI, bool FUSE>
__device__ __forceinline__ void kuhn_spmv_body(
    const BrickDev& D, const BrickArg& a, SubState* __restrict__ st, double* __restrict__ q,
    double* __restrict__ part, int32_t* __restrict__ nactive, int64_t b0, const BrickFuse& f) {
  constexpr int NC = 8, NW = BI;
  constexpr int kStride = box_stride_of(BI);
  extern __shared__ __align__(128) unsigned char bsm_raw[];
  unsigned char* bsm = bsm_raw + ((128u - (smem_addr(bsm_raw) & 127u)) & 127u);
  const uint32_t xs_addr = smem_addr(bsm);
  uint64_t* bar = reinterpret_cast<uint64_t*>(bsm + NC * kStride * 8);
  __shared__ double red[NW];
  // fused path: per class, the box origin in the class array (jj, ii, kk), nJp, nIc, nKc, first row
  __shared__ int4 fgeo[FUSE ? NC : 1];
  __shared__ int2 fext[FUSE ? NC : 1];
  __shared__ long long fbase[FUSE ? NC : 1];
  const int64_t b = b0 + blockIdx.x;
  const BrickInfo bi = D.info[b];  // static: before the dependency wait
  const BrickSub& B = D.sub[bi.ls];
  const CUtensorMap* tm = (FUSE ? f.tmap : D.tmap) + bi.ls * NC;
  const int lane = threadIdx.x & 31;
  const int w = __reduce_max_sync(0xffffffffu, (unsigned)(threadIdx.x >> 5));  // = il
  // the constants of this warp's 8 chunks (C, il = w): lane C holds class C's (desc, row mask, row
  // offset, kk stride), broadcast by shuffles when the class runs
  const int4 creg = lane < NC ? __ldg(reinterpret_cast<const int4*>(D.chunk) + (b * NC + lane) * BI + w)
                              : make_int4(0, 0, 0, 0);
  auto dsc = [&](int C) { return __shfl_sync(0xffffffffu, creg.x, C); };
  uint32_t W0[16], W1[16];
  uint32_t W2[16];
  kuhn_words<0>(W0, D, dsc(0), lane);  // the stream is static: index words before the wait
  kuhn_words<1>(W1, D, dsc(1), lane);
  const int jl = lane & 15, kl = lane >> 4;
  double* qs = q + B.row0;  // the subdomain's rows
  if (w == 0) {
    if (lane == 0) mbar_init(bar, 1);
    if (lane < NC) asm volatile("prefetch.tensormap [%0];" ::"l"(tm + lane) : "memory");
  }
  if constexpr (FUSE) {
    if (threadIdx.x < NC) {
      const int c = threadIdx.x;
      const BrickClass& C = B.cls[c];
      fgeo[c] = make_int4(bi.bj * 16 - 1 - C.jjlo - jsh_of(c), bi.bi * BI - 1 - C.iilo, bi.bk * 2 - 1 - C.kklo, C.nJp);
      fext[c] = make_int2(C.nIc, C.nKc);
      fbase[c] = B.row0 + C.base;
    }
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();  // barrier initialised
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // the boxes are requested before the subdomain's active flag is read (its load would otherwise sit
  // on every CTA's critical path); a stopped subdomain's CTAs drain them and leave
  if (w == 0) {
    if (lane == 0) mbar_expect_tx(bar, (uint32_t)(NC * a.box_elems * 8));
    __syncwarp();
    if (lane < NC) {
      const int c = lane;
      const BrickClass& C = B.cls[c];
      tma_load_3d(reinterpret_cast<double*>(bsm) + c * kStride, tm + c, bi.bj * 16 - 1 - C.jjlo - jsh_of(c),
                  bi.bi * BI - 1 - C.iilo, bi.bk * 2 - 1 - C.kklo, bar);
    }
  }
  SubState& S = st[bi.ls];
  const uint32_t lane_off = 8u * (uint32_t)((jl + 1) + 20 * (BI + 2) * (kl + 1) + 20 * (w + 1));
  if constexpr (FUSE) {
    const int act = S.active;
    if (!act && !S.xpend) {  // stopped earlier (its x is paid; k_brick_alpha cleared xpend)
      mbar_wait_parity(bar, 0);
      return;
    }
    const double al = S.alpha, be = S.beta;
    mbar_wait_parity(bar, 0);
    // x_{k+1} = x_k + alpha_k p_k on the brick's rows (the update k_cg_dir would have made)
    double* xs = f.x + B.row0;
    double xo[NC];
    int xi[NC];
    uint32_t own = 0;
#pragma unroll
    for (int C = 0; C < NC; ++C) {
      const uint32_t m = (uint32_t)__shfl_sync(0xffffffffu, creg.y, C);
      const int ro = __shfl_sync(0xffffffffu, creg.z, C), nji = __shfl_sync(0xffffffffu, creg.w, C);
      xi[C] = ro + jl + nji * kl;
      if ((m >> lane) & 1u) {
        own |= 1u << C;
        xo[C] = xs[xi[C]];
      }
    }
#pragma unroll
    for (int C = 0; C < NC; ++C)
      if ((own >> C) & 1u)
        xs[xi[C]] = fma(al, lds_f64(xs_addr + 8u * (uint32_t)(C * kStride + jsh_of(C)) + lane_off), xo[C]);
    if (!act) return;  // stopped in the last update: only its x was owed (uniform over the CTA)
    __syncthreads();   // every p_k read above precedes the overwrite below
    // p_{k+1} on every staged point: columns (class, box kk, box jj) of BI + 2 points along ii, jj
    // fastest over the threads (coalesced r and code loads); points outside the class array stay
    // the TMA's zero fill
    double* pb = reinterpret_cast<double*>(bsm);
    constexpr int kCols = NC * 4 * 20;
    for (int col = threadIdx.x; col < kCols; col += 32 * BI) {
      const int c = col / 80, rem = col - 80 * c, ek = rem / 20, ej = rem - 20 * ek;
      const int4 g = fgeo[c];
      const int2 e = fext[c];
      const int gj = g.x + ej, gk = g.z + ek;
      if (gj < 0 || gj >= g.w || gk < 0 || gk >= e.y) continue;
      const int64_t o0 = fbase[c] + gj + (int64_t)g.w * e.x * gk;
      double* pc = pb + c * kStride + ej + 20 * (BI + 2) * ek;
      constexpr int NE = BI + 2, NB = (NE + 1) / 2;  // two batches of loads in flight
#pragma unroll
      for (int e0 = 0; e0 < NE; e0 += NB) {
        double rv[NB];
        uint32_t cv[NB];
#pragma unroll
        for (int u = 0; u < NB; ++u) {
          const int gi = g.y + e0 + u;
          if (e0 + u < NE && gi >= 0 && gi < e.x) {
            const int64_t o = o0 + (int64_t)g.w * gi;
            rv[u] = __ldg(f.r + o);
            cv[u] = __ldg(f.code + o);
          }
        }
#pragma unroll
        for (int u = 0; u < NB; ++u) {
          const int gi = g.y + e0 + u;
          if (e0 + u < NE && gi >= 0 && gi < e.x) {
            const double d = cv[u] != 0xffu ? f.dtab[cv[u]] : 0.0;
            pc[20 * (e0 + u)] = fma(be, pc[20 * (e0 + u)], __dmul_rn(d, rv[u]));
          }
        }
      }
    }
    __syncthreads();
  } else {
    if (!S.active) {  // the previous direction kernel has paid the stopped subdomain's x update
      if (threadIdx.x == 0 && b == S.brick0) S.xpend = 0;
      mbar_wait_parity(bar, 0);  // no CTA leaves with bulk copies into its shared memory in flight
      return;
    }
    mbar_wait_parity(bar, 0);
  }
  double* pns = FUSE ? f.pn + B.row0 : nullptr;
  double pq = 0.0;
  auto run = [&](auto cc, const uint32_t(&Wc)[16]) {
    constexpr int C = decltype(cc)::value;
    const uint32_t xc = xs_addr + 8u * (uint32_t)(C * kStride + jsh_of(C)) + lane_off;
    const double s = kuhn_chunk<C, BI>(xc, Wc, a.dict);
    const uint32_t m = (uint32_t)__shfl_sync(0xffffffffu, creg.y, C);
    const int ro = __shfl_sync(0xffffffffu, creg.z, C), nji = __shfl_sync(0xffffffffu, creg.w, C);
    if ((m >> lane) & 1u) {
      const double pv = lds_f64(xc);
      qs[ro + jl + nji * kl] = s;
      if constexpr (FUSE) pns[ro + jl + nji * kl] = pv;
      pq = fma(pv, s, pq);
    }
  };
  kuhn_words<2>(W2, D, dsc(2), lane);
  run(IC<0>{}, W0);
  kuhn_words<3>(W0, D, dsc(3), lane);
  run(IC<1>{}, W1);
  kuhn_words<4>(W1, D, dsc(4), lane);
  run(IC<2>{}, W2);
  kuhn_words<5>(W2, D, dsc(5), lane);
  run(IC<3>{}, W0);
  kuhn_words<6>(W0, D, dsc(6), lane);
  run(IC<4>{}, W1);
  kuhn_words<7>(W1, D, dsc(7), lane);
  run(IC<5>{}, W2);
  run(IC<6>{}, W0);
  run(IC<7>{}, W1);
  // p.q: warp tree, warps in order, one partial per brick.  Warps 1.. hand their sums to warp 0 over a
  // named barrier (bar.arrive: they exit at once); warp 0 publishes the partial, and in the last brick
  // of the subdomain sums all of them in brick order (strided over its lanes, then the warp tree).
  pq = warp_sum_b(pq);
  if (lane == 0) red[w] = pq;
  __syncthreads();
  if (threadIdx.x == 0) {  // the brick's partial; k_brick_alpha sums them (no atomic on this path)
    double v = 0.0;
    for (int k = 0; k < NW; ++k) v += red[k];
    part[b] = v;
  }
}

// The plain kernel, and the fused one held to the plain one's occupancy (3 CTAs per SM up to BI = 9,
// else 2: the phase-B registers would otherwise cost a CTA per SM).
template <int BI, bool FUSE>
__global__ void __launch_bounds__(32 * BI) k_cg_spmv_kuhn(const BrickDev D, const __grid_constant__ BrickArg a,
                                                          SubState* __restrict__ st, double* __restrict__ q,
                                                          double* __restrict__ part, int32_t* __restrict__ nactive,
                                                          int64_t b0, const __grid_constant__ BrickFuse f) {
  static_assert(!FUSE, "the fused instance is k_cg_spmv_kuhn_fused");
  kuhn_spmv_body<BI, false>(D, a, st, q, part, nactive, b0, f);
}
template <int BI>
__global__ void __launch_bounds__(32 * BI, BI <= 9 ? 3 : 2)
    k_cg_spmv_kuhn_fused(const BrickDev D, const __grid_constant__ BrickArg a, SubState* __restrict__ st,
                         double* __restrict__ q, double* __restrict__ part, int32_t* __restrict__ nactive, int64_t b0,
                         const __grid_constant__ BrickFuse f) {
  kuhn_spmv_body<BI, true>(D, a, st, q, part, nactive, b0, f);
}

// alpha = rho / p.q of each subdomain of a group from its brick partials (brick order: lane-strided
// over the block, then the warp tree, then the warps in order): one block per subdomain, launched
// after the Kuhn kernel (PDL), so the SpMV's CTAs retire without an atomic.
__global__ void __launch_bounds__(256) k_brick_alpha(SubState* __restrict__ st, const double* __restrict__ part,
                                                     int32_t* __restrict__ nactive, int ls0) {
  __shared__ double red[8];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  SubState& S = st[ls0 + blockIdx.x];
  if (!S.active) {  // a stopped subdomain's pending x update has been paid by the SpMV (fused or k_cg_dir)
    if (threadIdx.x == 0) S.xpend = 0;
    return;
  }
  double v = 0.0;
  for (int64_t m = threadIdx.x; m < S.nbrick; m += 256) v += __ldcg(part + S.brick0 + m);
  v = warp_sum_b(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < 8; ++k) t += red[k];
    if (!(t > 0.0) || !isfinite(t)) {  // breakdown: p = 0 or loss of definiteness
      S.status = 3;
      S.active = 0;
      atomicSub(nactive, 1);
    } else {
      S.alpha = S.rho / t;
    }
  }
}

// f(k_cg_spmv_kuhn<BI, FUSE>) for a runtime BI in 1..12
template <int BI, bool FUSE>
constexpr auto kuhn_kernel() {
  if constexpr (FUSE) return k_cg_spmv_kuhn_fused<BI>;
  else return k_cg_spmv_kuhn<BI, false>;
}
template <bool FUSE, class F>
void with_kuhn_kernel(int BI, F&& f) {
  switch (BI) {
    case 1: f(kuhn_kernel<1, FUSE>()); break;
    case 2: f(kuhn_kernel<2, FUSE>()); break;
    case 3: f(kuhn_kernel<3, FUSE>()); break;
    case 4: f(kuhn_kernel<4, FUSE>()); break;
    case 5: f(kuhn_kernel<5, FUSE>()); break;
    case 6: f(kuhn_kernel<6, FUSE>()); break;
    case 7: f(kuhn_kernel<7, FUSE>()); break;
    case 8: f(kuhn_kernel<8, FUSE>()); break;
    case 9: f(kuhn_kernel<9, FUSE>()); break;
    case 10: f(kuhn_kernel<10, FUSE>()); break;
    case 11: f(kuhn_kernel<11, FUSE>()); break;
    case 12: f(kuhn_kernel<12, FUSE>()); break;
    default: fail(OSM_ERR_STATE, "brick: no Kuhn kernel for this BI");
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    OSM_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) fail(OSM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

}  // namespace

void brick_free(Ctx& c) {
  if (c.brick.info) cudaFree(c.brick.info);
  if (c.brick.chunk) cudaFree(c.brick.chunk);
  if (c.brick.typetab) cudaFree(c.brick.typetab);
  if (c.brick.cstream) cudaFree(c.brick.cstream);
  c.brick_cwords = 0;
  c.brick_ntypes = 0;
  c.h_brick_sub_cwords.clear();
  if (c.brick.stream) cudaFree(c.brick.stream);
  if (c.brick.tmap) cudaFree(c.brick.tmap);
  if (c.brick.sub) cudaFree(c.brick.sub);
  if (c.part_brick) cudaFree(c.part_brick);
  c.part_brick = nullptr;
  if (c.p2) cudaFree(c.p2);
  c.p2 = nullptr;
  c.brick = BrickDev{};
  c.brick_ok = false;
  c.brick_total = 0;
  c.h_brick_sub.clear();
}

// Brick geometry of row order 6 (the class arrays are laid out by osm.cu assemble with the same
// rules): per local subdomain and class, the class-local ranges and the array base.
void brick_geometry(const Ctx& c, int ls, BrickSub& B) {
  const Sub& S = c.subs[ls];
  const int o = c.mesh.order;
  const int nc = o * o * o;
  B = BrickSub{};
  B.I_lo = (int)S.g.I_lo;
  B.nI = (int)S.g.nI;
  B.nJ = (int)S.g.nJ;
  B.row0 = S.row0;
  int64_t base = 0;
  for (int cc = 0; cc < nc; ++cc) {
    const int pi = cc % o, pj = (cc / o) % o, pk = cc / (o * o);
    auto range = [&](int lo, int hi, int par, int origin, int& a, int& z) {
      int f = lo;
      while (f <= hi && f % o != par) ++f;
      int l = hi;
      while (l >= lo && l % o != par) --l;
      a = f / o - origin / o;
      z = l / o - origin / o;
    };
    BrickClass& C = B.cls[cc];
    range((int)S.g.I_lo, (int)S.g.I_hi, pi, (int)S.g.I_lo, C.iilo, C.iihi);
    range(1, (int)S.g.Ny - 2, pj, 1, C.jjlo, C.jjhi);
    range(1, (int)S.g.Nz - 2, pk, 1, C.kklo, C.kkhi);
    C.nIc = std::max(0, C.iihi - C.iilo + 1);
    const int nJc = std::max(0, C.jjhi - C.jjlo + 1);
    C.nJp = (nJc + 1) & ~1;
    C.nKc = std::max(0, C.kkhi - C.kklo + 1);
    C.base = base;
    base += (int64_t)C.nJp * C.nIc * C.nKc;
  }
  B.nrows = base;
}

// Builds the brick copy from the assembled (value-indexed) SELL: slot tables, brick map, u8 stream
// and the TMA tensor maps of p.  Needs vi (<= 256 dictionary slots) and row order 6.
void brick_build(Ctx& c, const uint16_t* d_vidx, uint32_t zero_idx) {
  brick_free(c);
  if (c.sort_key != 6 || !c.vi_ok || c.vi_ndict > 256 || !d_vidx) return;
  const int o = c.mesh.order;
  const int nc = o * o * o;
  const int nloc = c.s_end - c.s_begin;
  auto dbg = [&](const char* why) {
    if (std::getenv("OSM_DEBUG")) std::fprintf(stderr, "osm: brick copy not built: %s\n", why);
  };
  int iext = 0;
  std::vector<BrickSub> subs(nloc);
  for (int ls = 0; ls < nloc; ++ls) {
    brick_geometry(c, ls, subs[ls]);
    for (int cc = 0; cc < nc; ++cc) iext = std::max(iext, subs[ls].cls[cc].iihi + 1);
  }
  // per-row subdomain and contract index maps for the build kernels
  std::vector<int32_t> row_sub(c.nrows_total, -1);
  for (int ls = 0; ls < nloc; ++ls)
    for (int64_t k = 0; k < c.subs[ls].npad; ++k) row_sub[c.subs[ls].row0 + k] = ls;
  int32_t *d_row_sub = nullptr, *d_perm = nullptr, *d_flag = nullptr;
  BrickSub* d_sub = nullptr;
  OSM_CUDA(cudaMalloc(&d_row_sub, sizeof(int32_t) * c.nrows_total));
  OSM_CUDA(cudaMemcpy(d_row_sub, row_sub.data(), sizeof(int32_t) * c.nrows_total, cudaMemcpyHostToDevice));
  OSM_CUDA(cudaMalloc(&d_perm, sizeof(int32_t) * c.nrows_total));
  for (int ls = 0; ls < nloc; ++ls)
    OSM_CUDA(cudaMemcpyAsync(d_perm + c.subs[ls].row0, c.subs[ls].perm, sizeof(int32_t) * c.subs[ls].npad,
                             cudaMemcpyDeviceToDevice, c.stream));
  OSM_CUDA(cudaMalloc(&d_sub, sizeof(BrickSub) * std::max(1, nloc)));
  OSM_CUDA(cudaMemcpy(d_sub, subs.data(), sizeof(BrickSub) * nloc, cudaMemcpyHostToDevice));
  BrickBuildDev D{};
  D.o = o;
  D.nrows = c.nrows_total;
  D.row_sub = d_row_sub;
  D.perm = d_perm;
  D.sub = d_sub;
  auto cleanup = [&]() {
    cudaFree(d_flag);
    cudaFree(d_row_sub);
    cudaFree(d_perm);
  };
  // 1. slot lists: union of the kept offsets per class, in column (= (dK, dJ, dI) lexicographic) order
  OSM_CUDA(cudaMalloc(&d_flag, sizeof(int32_t) * 8 * 125));
  OSM_CUDA(cudaMemsetAsync(d_flag, 0, sizeof(int32_t) * 8 * 125, c.stream));
  const unsigned grid = (unsigned)ceil_div(c.nrows_total, 256);
  k_brick_mark<<<grid, 256, 0, c.stream>>>(D, c.sell_soff, c.sell_swidth, c.sell_col, d_vidx, zero_idx, d_flag);
  OSM_CHECK_LAUNCH();
  ++c.launches;
  std::vector<int32_t> flag(8 * 125);
  OSM_CUDA(cudaMemcpyAsync(flag.data(), d_flag, sizeof(int32_t) * flag.size(), cudaMemcpyDeviceToHost, c.stream));
  OSM_CUDA(cudaStreamSynchronize(c.stream));
  struct Slot {
    int cn, dii, djj, dkk;
  };
  std::vector<std::vector<Slot>> slots(nc);
  std::vector<int16_t> slot_of(8 * 125, -1);
  BrickArg& A = c.h_brick_arg;
  A = BrickArg{};
  for (int cc = 0; cc < nc; ++cc) {
    const int pi = cc % o, pj = (cc / o) % o, pk = cc / (o * o);
    for (int dk = -2; dk <= 2; ++dk)  // column order: K slowest, then J, then I
      for (int dj = -2; dj <= 2; ++dj)
        for (int di = -2; di <= 2; ++di) {
          const int code = (di + 2) + 5 * (dj + 2) + 25 * (dk + 2);
          if (!flag[cc * 125 + code]) continue;
          slot_of[cc * 125 + code] = (int16_t)slots[cc].size();
          // neighbour class and class-local offset (floor division by o of non-negative coordinates)
          auto cl = [&](int par, int d, int& nb_par) {
            const int v = o + par + d;  // a representative coordinate of parity par, shifted by d
            nb_par = v % o;
            return v / o - (o + par) / o;
          };
          int qi, qj, qk;
          Slot sl;
          sl.dii = cl(pi, di, qi);
          sl.djj = cl(pj, dj, qj);
          sl.dkk = cl(pk, dk, qk);
          sl.cn = qi + o * (qj + o * qk);
          slots[cc].push_back(sl);
        }
    A.ngrp[cc] = (int)(slots[cc].size() + 3) / 4;
    if (A.ngrp[cc] > 16) {
      dbg("a class has more than 64 stencil slots");
      cleanup();
      cudaFree(d_sub);
      return;
    }
  }
  // P2 with every row's entries on the Kuhn slots of gen_kuhn_slots.cpp: use those slots (a row's
  // missing ones get the index of 0.0) and the kernel with compile-time offsets
  bool kuhn = o == 2 && !std::getenv("OSM_BRICK_GENERIC");
  for (int cc = 0; kuhn && cc < nc; ++cc)
    for (int code = 0; code < 125 && kuhn; ++code) {
      if (slot_of[cc * 125 + code] < 0) continue;
      const int di = code % 5 - 2, dj = (code / 5) % 5 - 2, dk = code / 25 - 2;
      bool found = false;
      for (int j = 0; j < kKuhnSlotCount[cc]; ++j)
        found = found || (kKuhnSlots[cc][j][0] == di && kKuhnSlots[cc][j][1] == dj && kKuhnSlots[cc][j][2] == dk);
      kuhn = found;
    }
  if (kuhn) {
    for (int cc = 0; cc < nc; ++cc) {
      const int pi = cc % o, pj = (cc / o) % o, pk = cc / (o * o);
      slots[cc].clear();
      for (int code = 0; code < 125; ++code) slot_of[cc * 125 + code] = -1;
      for (int j = 0; j < kKuhnSlotCount[cc]; ++j) {
        const int di = kKuhnSlots[cc][j][0], dj = kKuhnSlots[cc][j][1], dk = kKuhnSlots[cc][j][2];
        slot_of[cc * 125 + (di + 2) + 5 * (dj + 2) + 25 * (dk + 2)] = (int16_t)j;
        auto cl = [&](int par, int d, int& nb_par) {
          const int v = o + par + d;
          nb_par = v % o;
          return v / o - (o + par) / o;
        };
        int qi, qj, qk;
        Slot sl;
        sl.dii = cl(pi, di, qi);
        sl.djj = cl(pj, dj, qj);
        sl.dkk = cl(pk, dk, qk);
        sl.cn = qi + o * (qj + o * qk);
        slots[cc].push_back(sl);
      }
      A.ngrp[cc] = (kKuhnSlotCount[cc] + 3) / 4;
    }
  }
  // 2. brick shape: 16 x BI x 2 class-local points (the kernel's lane map is jl + 16 kl); BI is the
  // x extent of the widest slab in chunks of at most 12
  A.BJ = 16;
  A.BK = 2;
  int imax = 12;
  if (const char* e = std::getenv("OSM_BRICK_IMAX")) imax = std::max(1, std::atoi(e));  // tuning
  const int nchunk = (iext + imax - 1) / imax;
  A.BI = (iext + nchunk - 1) / nchunk;
  c.brick_kernel = kuhn && A.BI >= 1 && A.BI <= 12 ? A.BI : 0;  // k_cg_spmv_kuhn<BI> instances
  A.npb = A.BJ * A.BI * A.BK;
  A.box_elems = (A.BJ + 4) * (A.BI + 2) * (A.BK + 2);
  A.box_stride = (int)round_up(A.box_elems, 16);  // 128-byte aligned class boxes
  A.box_bytes = A.box_stride * 8;
  for (int cc = 0; cc < nc; ++cc) {  // class box column of jj = -1: 0 or 1 (even TMA start)
    const int jjlo = subs.empty() ? 0 : subs[0].cls[cc].jjlo;
    A.jsh[cc] = (-1 - jjlo) & 1;
  }
  int goff = 0;
  for (int cc = 0; cc < nc; ++cc) {
    for (size_t j = 0; j < 4 * (size_t)A.ngrp[cc]; ++j) {
      int off = 0;  // padding slots: the own element (times the dictionary's 0.0)
      if (j < slots[cc].size()) {
        const Slot& sl = slots[cc][j];  // byte offset from the point's own element in its class box
        off = 8 * ((sl.cn - cc) * A.box_stride + A.jsh[sl.cn] - A.jsh[cc] + sl.djj +
                   (A.BJ + 4) * (sl.dii + (A.BI + 2) * sl.dkk));
      }
      A.soff[cc * 4 * kBrickMaxGroups + j] = off;
    }
    A.goff[cc] = goff;  // in 32-word groups: class cc's chunk il, slot group g at goff + il ngrp + g
    goff += A.BI * A.ngrp[cc];
  }
  A.brick_words = 32 * (int64_t)goff;
  // 3. brick map (subdomain-major, then kk, ii, jj bricks)
  int64_t nb = 0;
  for (int ls = 0; ls < nloc; ++ls) {
    BrickSub& B = subs[ls];
    int jmax = 0, kmax = 0;
    for (int cc = 0; cc < nc; ++cc) {
      jmax = std::max(jmax, B.cls[cc].jjhi + 1);
      kmax = std::max(kmax, B.cls[cc].kkhi + 1);
    }
    B.nbj = (jmax + A.BJ - 1) / A.BJ;
    B.nbi = (iext + A.BI - 1) / A.BI;
    B.nbk = (kmax + A.BK - 1) / A.BK;
    B.brick0 = nb;
    B.nbrick = (int64_t)B.nbj * B.nbi * B.nbk;
    nb += B.nbrick;
  }
  std::vector<BrickInfo> info(nb);
  for (int ls = 0; ls < nloc; ++ls) {
    const BrickSub& B = subs[ls];
    for (int bk = 0; bk < B.nbk; ++bk)
      for (int bi = 0; bi < B.nbi; ++bi)
        for (int bj = 0; bj < B.nbj; ++bj) {
          BrickInfo& I = info[B.brick0 + bj + (int64_t)B.nbj * (bi + (int64_t)B.nbi * bk)];
          I.ls = ls;
          I.bj = (int16_t)bj;
          I.bi = (int16_t)bi;
          I.bk = (int16_t)bk;
        }
  }
  OSM_CUDA(cudaMemcpy(d_sub, subs.data(), sizeof(BrickSub) * nloc, cudaMemcpyHostToDevice));
  // 4. the u8 index stream (entries whose row has no slot or is out of column order: fall back)
  int16_t* d_slot = nullptr;
  OSM_CUDA(cudaMalloc(&d_slot, sizeof(int16_t) * slot_of.size()));
  OSM_CUDA(cudaMemcpy(d_slot, slot_of.data(), sizeof(int16_t) * slot_of.size(), cudaMemcpyHostToDevice));
  OSM_CUDA(cudaMalloc(&c.brick.stream, sizeof(uint32_t) * std::max<int64_t>(1, nb * A.brick_words)));
  // words of points outside a class's valid range stay "index of 0.0" (never used for output)
  OSM_CUDA(cudaMemsetAsync(c.brick.stream, (int)zero_idx, sizeof(uint32_t) * nb * A.brick_words, c.stream));
  D.BJ = A.BJ;
  D.BI = A.BI;
  D.BK = A.BK;
  D.npb = A.npb;
  D.brick_words = A.brick_words;
  for (int cc = 0; cc < 8; ++cc) {
    D.ngrp[cc] = A.ngrp[cc];
    D.goff[cc] = A.goff[cc];
  }
  int32_t* d_bad = c.d_flags + 3;
  OSM_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int32_t), c.stream));
  k_brick_pack<<<grid, 256, 0, c.stream>>>(D, c.sell_soff, c.sell_swidth, c.sell_col, d_vidx, zero_idx, d_slot,
                                           reinterpret_cast<uint8_t*>(c.brick.stream), d_bad);
  OSM_CHECK_LAUNCH();
  ++c.launches;
  int32_t bad = 0;
  OSM_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(int32_t), cudaMemcpyDeviceToHost, c.stream));
  OSM_CUDA(cudaStreamSynchronize(c.stream));
  OSM_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int32_t), c.stream));
  cudaFree(d_slot);
  cleanup();
  if (bad) {
    dbg("an entry has no slot of its class or is out of column order");
    cudaFree(d_sub);
    cudaFree(c.brick.stream);
    c.brick = BrickDev{};
    return;
  }
  // 5. TMA tensor maps of p: one per (local subdomain, class), dims (nJp, nIc, nKc), jj fastest; with the
  // fused Kuhn kernel (Ctx::fuse_dir) a second set over p2 (the fused direction update's other p buffer, zero-initialised:
  // its padding rows are never written)
  const bool fuse = c.brick_kernel > 0 && c.fuse_dir;  // only the opt-in fused path needs p2
  if (fuse && !c.p2) {
    OSM_CUDA(cudaMalloc(&c.p2, sizeof(double) * std::max<int64_t>(1, c.nrows_total)));
    OSM_CUDA(cudaMemset(c.p2, 0, sizeof(double) * c.nrows_total));
  }
  const int nset = fuse ? 2 : 1;
  std::vector<CUtensorMap> maps((size_t)nset * nloc * nc);
  auto enc = encode_fn();
  for (int set = 0; set < nset; ++set)
  for (int ls = 0; ls < nloc; ++ls)
    for (int cc = 0; cc < nc; ++cc) {
      const BrickClass& C = subs[ls].cls[cc];
      const cuuint64_t dims[3] = {(cuuint64_t)std::max(1, C.nJp), (cuuint64_t)std::max(1, C.nIc),
                                  (cuuint64_t)std::max(1, C.nKc)};
      const cuuint64_t strides[2] = {(cuuint64_t)std::max(2, C.nJp) * 8,
                                     (cuuint64_t)std::max(2, C.nJp) * std::max(1, C.nIc) * 8};
      const cuuint32_t box[3] = {(cuuint32_t)(A.BJ + 4), (cuuint32_t)(A.BI + 2), (cuuint32_t)(A.BK + 2)};
      const cuuint32_t es[3] = {1, 1, 1};
      void* base = (set ? c.p2 : c.p) + subs[ls].row0 + C.base;
      const CUresult r = enc(&maps[((size_t)set * nloc + ls) * nc + cc], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides,
                             box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) fail(OSM_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    }
  OSM_CUDA(cudaMalloc(&c.brick.tmap, sizeof(CUtensorMap) * maps.size()));
  OSM_CUDA(cudaMemcpy(c.brick.tmap, maps.data(), sizeof(CUtensorMap) * maps.size(), cudaMemcpyHostToDevice));
  OSM_CUDA(cudaMalloc(&c.brick.info, sizeof(BrickInfo) * std::max<int64_t>(1, nb)));
  OSM_CUDA(cudaMemcpy(c.brick.info, info.data(), sizeof(BrickInfo) * nb, cudaMemcpyHostToDevice));
  if (c.brick_kernel > 0) {  // per (brick, class, il) chunk constants of the Kuhn kernel
    std::vector<BrickChunk> chunks((size_t)nb * nc * A.BI);
    for (int64_t bb = 0; bb < nb; ++bb) {
      const BrickInfo& I = info[bb];
      const BrickSub& B = subs[I.ls];
      const int j0 = I.bj * A.BJ, i0 = I.bi * A.BI, k0 = I.bk * A.BK;
      for (int cc = 0; cc < nc; ++cc) {
        const BrickClass& C = B.cls[cc];
        for (int il = 0; il < A.BI; ++il) {
          BrickChunk& e = chunks[((size_t)bb * nc + cc) * A.BI + il];
          e = BrickChunk{};
          const int64_t ro =
              C.base + (j0 - C.jjlo) + (int64_t)C.nJp * ((i0 + il - C.iilo) + (int64_t)C.nIc * (k0 - C.kklo));
          if (ro < INT32_MIN || ro > INT32_MAX || (int64_t)C.nJp * C.nIc > INT32_MAX)
            fail(OSM_ERR_STATE, "brick: subdomain too large for 32-bit row offsets");
          e.rowoff = (int32_t)ro;
          e.nJI = C.nJp * C.nIc;
          for (int lane = 0; lane < 32; ++lane) {
            const int jj = j0 + (lane & 15), ii = i0 + il, kk = k0 + (lane >> 4);
            if (jj >= C.jjlo && jj <= C.jjhi && ii >= C.iilo && ii <= C.iihi && kk >= C.kklo && kk <= C.kkhi)
              e.mask |= 1u << lane;
          }
        }
      }
    }
    // row types: chunks whose rows all carry the same index words are stored once (a type table),
    // the others keep their per-lane words in a compact stream (interior chunks are uniform: the
    // stencil of a parity class is translation invariant away from the Dirichlet faces and planes)
    const int64_t nchunk = nb * nc * A.BI;
    uint32_t* d_words = nullptr;
    int32_t* d_uni = nullptr;
    OSM_CUDA(cudaMalloc(&d_words, sizeof(uint32_t) * 16 * std::max<int64_t>(1, nchunk)));
    OSM_CUDA(cudaMalloc(&d_uni, sizeof(int32_t) * std::max<int64_t>(1, nchunk)));
    OSM_CUDA(cudaMemsetAsync(d_words, 0, sizeof(uint32_t) * 16 * std::max<int64_t>(1, nchunk), c.stream));
    k_brick_chunks<<<(unsigned)ceil_div(nchunk * 32, 256), 256, 0, c.stream>>>(D, c.brick.info, c.brick.stream,
                                                                             A.BI, nchunk, d_words, d_uni);
    OSM_CHECK_LAUNCH();
    ++c.launches;
    std::vector<uint32_t> words((size_t)nchunk * 16);
    std::vector<int32_t> uni((size_t)nchunk);
    OSM_CUDA(cudaMemcpyAsync(words.data(), d_words, sizeof(uint32_t) * words.size(), cudaMemcpyDeviceToHost,
                             c.stream));
    OSM_CUDA(cudaMemcpyAsync(uni.data(), d_uni, sizeof(int32_t) * uni.size(), cudaMemcpyDeviceToHost, c.stream));
    OSM_CUDA(cudaStreamSynchronize(c.stream));
    cudaFree(d_words);
    cudaFree(d_uni);
    std::map<std::vector<uint32_t>, int32_t> types;  // key: class, then the class's ng words
    std::vector<uint32_t> typetab;
    std::vector<int32_t> desc((size_t)nchunk);
    std::vector<int64_t> src_chunk, dst_group;
    c.h_brick_sub_cwords.assign(nloc, 0);
    int64_t groups = 0;
    for (int64_t ch = 0; ch < nchunk; ++ch) {
      const int cc = (int)((ch % (nc * A.BI)) / A.BI);
      const int ng = A.ngrp[cc];
      if (uni[ch]) {
        std::vector<uint32_t> key(1 + ng);
        key[0] = (uint32_t)cc;
        std::copy(words.begin() + ch * 16, words.begin() + ch * 16 + ng, key.begin() + 1);
        auto it = types.find(key);
        if (it == types.end()) {
          it = types.emplace(key, (int32_t)types.size()).first;
          typetab.resize(typetab.size() + 16, 0u);
          std::copy(key.begin() + 1, key.end(), typetab.end() - 16);
        }
        desc[ch] = it->second;
      } else {
        src_chunk.push_back(ch);
        dst_group.push_back(groups);
        desc[ch] = (int32_t)(-(groups + 1));
        c.h_brick_sub_cwords[info[ch / (nc * A.BI)].ls] += 32 * (int64_t)ng;
        groups += ng;
        if (groups >= (int64_t)1 << 30) fail(OSM_ERR_STATE, "brick: compact stream too large");
      }
    }
    for (int64_t ch = 0; ch < nchunk; ++ch) chunks[ch].desc = desc[ch];
    OSM_CUDA(cudaMalloc(&c.brick.chunk, sizeof(BrickChunk) * std::max<int64_t>(1, nchunk)));
    OSM_CUDA(cudaMemcpy(c.brick.chunk, chunks.data(), sizeof(BrickChunk) * nchunk, cudaMemcpyHostToDevice));
    OSM_CUDA(cudaMalloc(&c.brick.typetab, sizeof(uint32_t) * std::max<size_t>(16, typetab.size())));
    if (!typetab.empty())
      OSM_CUDA(cudaMemcpy(c.brick.typetab, typetab.data(), sizeof(uint32_t) * typetab.size(), cudaMemcpyHostToDevice));
    OSM_CUDA(cudaMalloc(&c.brick.cstream, sizeof(uint32_t) * 32 * std::max<int64_t>(1, groups)));
    if (!src_chunk.empty()) {
      int64_t *d_src = nullptr, *d_dst = nullptr;
      OSM_CUDA(cudaMalloc(&d_src, sizeof(int64_t) * src_chunk.size()));
      OSM_CUDA(cudaMalloc(&d_dst, sizeof(int64_t) * dst_group.size()));
      OSM_CUDA(cudaMemcpy(d_src, src_chunk.data(), sizeof(int64_t) * src_chunk.size(), cudaMemcpyHostToDevice));
      OSM_CUDA(cudaMemcpy(d_dst, dst_group.data(), sizeof(int64_t) * dst_group.size(), cudaMemcpyHostToDevice));
      const int64_t n = (int64_t)src_chunk.size();
      k_brick_compact<<<(unsigned)ceil_div(n * 32, 256), 256, 0, c.stream>>>(D, c.brick.stream, A.BI, d_src, d_dst, n,
                                                                           c.brick.cstream);
      OSM_CHECK_LAUNCH();
      ++c.launches;
      OSM_CUDA(cudaStreamSynchronize(c.stream));
      cudaFree(d_src);
      cudaFree(d_dst);
    }
    c.brick_cwords = 32 * groups;
    c.brick_ntypes = (int)types.size();

    cudaFree(c.brick.stream);  // the Kuhn kernel reads the type table and the compact stream only
    c.brick.stream = nullptr;
  }
  c.brick.sub = d_sub;
  OSM_CUDA(cudaMalloc(&c.part_brick, sizeof(double) * std::max<int64_t>(1, nb)));
  c.brick_total = nb;
  c.h_brick_sub = subs;
  c.brick_ok = true;
  const int smem = nc * A.box_bytes + 16 + 128;
  if (smem > kMaxDynSmem || kuhn_smem_bytes(12) > kMaxDynSmem)
    fail(OSM_ERR_STATE, "brick: class boxes exceed the shared memory of an SM");
  if (c.brick_kernel > 0)
    for (int cc = 0; cc < nc; ++cc)  // the Kuhn kernel's compile-time stream layout
      if (A.ngrp[cc] != (kKuhnSlotCount[cc] + 3) / 4) fail(OSM_ERR_STATE, "brick: Kuhn slot groups");
  // the opt-in limit is a per-function, process-wide attribute: contexts of other shapes (other
  // ranks of a hub, other problems) share it, so every brick kernel gets the SM maximum (the opt-in
  // limit less its static shared memory) once, not a per-shape value
  static std::mutex attr_mu;
  static bool attr_done[64] = {};  // per device
  {
    std::lock_guard<std::mutex> lk(attr_mu);
    int dev = 0;
    OSM_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) fail(OSM_ERR_STATE, "brick: device ordinal out of range");
    if (!attr_done[dev]) {
      int optin = 0;
      OSM_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
      auto set_max = [&](auto kern) {
        cudaFuncAttributes fa{};
        OSM_CUDA(cudaFuncGetAttributes(&fa, kern));
        OSM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      optin - (int)fa.sharedSizeBytes));
      };
      set_max(k_cg_spmv_brick<8>);
      set_max(k_cg_spmv_brick<1>);
      for (int bi = 1; bi <= 12; ++bi) {
        with_kuhn_kernel<false>(bi, set_max);
        with_kuhn_kernel<true>(bi, set_max);
      }
      attr_done[dev] = true;
    }
  }
  if (std::getenv("OSM_DEBUG"))
    std::fprintf(stderr,
                 "osm: brick copy: %lld bricks, BI %d, kernel %d, %d B shared, %lld stream words/brick, %d row "
                 "types, compact stream %lld words (%.1f %% of the full one)\n",
                 (long long)nb, A.BI, c.brick_kernel, smem, (long long)A.brick_words, c.brick_ntypes,
                 (long long)c.brick_cwords, 100.0 * (double)c.brick_cwords / std::max(1.0, (double)nb * A.brick_words));
}

// One launch over the bricks of the local subdomains of group g (all of them for g < 0), one CTA per
// brick; p.q partials are indexed by the global brick number.
void launch_cg_spmv_brick(Ctx& c, cudaStream_t s, int g) {
  const int nloc = c.s_end - c.s_begin;
  int s0 = 0, s1 = nloc;
  if (g >= 0) {
    s0 = g * nloc / c.ngroups;
    s1 = (g + 1) * nloc / c.ngroups;
  }
  const int64_t b0 = c.h_brick_sub[s0].brick0;
  const int64_t nb = (s1 < nloc ? c.h_brick_sub[s1].brick0 : c.brick_total) - b0;
  if (nb <= 0) return;
  const int nc = c.mesh.order * c.mesh.order * c.mesh.order;
  const size_t smem = (size_t)nc * c.h_brick_arg.box_bytes + 16 + 128;
  c.h_brick_arg.dict_n = (int)std::min<size_t>(256, c.h_vi_dict.size());
  std::copy(c.h_vi_dict.begin(), c.h_vi_dict.begin() + c.h_brick_arg.dict_n, c.h_brick_arg.dict);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)nb);
  cfg.blockDim = dim3(kBrickThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  auto go = [&](auto kern) {
    OSM_CUDA(cudaLaunchKernelEx(&cfg, kern, (const BrickDev)c.brick, c.h_brick_arg, c.st, c.q, c.part_brick,
                                c.d_nactive, b0));
  };
  if (nc != 8) {
    go(k_cg_spmv_brick<1>);
  } else if (c.brick_kernel > 0) {
    cfg.blockDim = dim3(32 * c.brick_kernel);
    cfg.dynamicSmemBytes = kuhn_smem_bytes(c.brick_kernel);
    BrickFuse& F = c.h_brick_fuse;
    auto launch = [&](auto kern) {
      OSM_CUDA(cudaLaunchKernelEx(&cfg, kern, (const BrickDev)c.brick, c.h_brick_arg, c.st, c.q, c.part_brick,
                                  c.d_nactive, b0, F));
    };
    if (fused_dir(c)) {  // p_k in p (parity 0) or p2 (parity 1); p_{k+1} to the other buffer
      F.tmap = c.brick.tmap + (size_t)(c.cg_par & 1) * nloc * nc;
      F.pn = (c.cg_par & 1) ? c.p : c.p2;
      F.x = c.x;
      F.r = c.r;
      F.code = c.d_dcode;
      std::fill(F.dtab, F.dtab + kMfMaxTab, 0.0);
      std::copy(c.h_dcode_tab.begin(), c.h_dcode_tab.end(), F.dtab);
      with_kuhn_kernel<true>(c.brick_kernel, launch);
    } else {
      F = BrickFuse{};
      with_kuhn_kernel<false>(c.brick_kernel, launch);
    }
    cudaLaunchConfig_t ac = cfg;
    ac.gridDim = dim3((unsigned)(s1 - s0));
    ac.blockDim = dim3(256);
    ac.dynamicSmemBytes = 0;
    OSM_CUDA(cudaLaunchKernelEx(&ac, k_brick_alpha, c.st, (const double*)c.part_brick, c.d_nactive, s0));
  } else {
    go(k_cg_spmv_brick<8>);
  }
}

}  // namespace osm

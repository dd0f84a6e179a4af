// Value-indexed SELL-256 (SpMV variant 3): the hot matrix stored as a 16-bit index into a
// per-GPU dictionary of distinct fp64 values plus a 16-bit column offset (col - row, internal
// order), 4 bytes per entry instead of 12.  FE matrices on the structured Kuhn mesh have very
// few distinct values (C3 slab: 87 among 7.0 M entries), so the dictionary stays L1-resident
// and the SpMV streams a third of the bytes.  The values are exact copies: results are bitwise
// identical to the fp64 SELL path.
//
// Robin folding (K_s = K^N + p M + q S on interface rows) gives each distinct
// (side, K^N value, m, s) tuple its own dictionary slot; osm_set_robin/2 only rewrites that
// small dictionary tail.  Entries are (16-bit index, 16-bit offset); when an offset does not fit
// int16 the wide form (12-bit index, 20-bit offset; e.g. C5 with S = 8) is used.  If neither fits
// (more than 65536 / 4096 values, or offsets beyond 2^19) the context stays on the fp64 SELL path.
#include <thrust/binary_search.h>
#include <thrust/device_ptr.h>
#include <thrust/execution_policy.h>
#include <thrust/sort.h>
#include <thrust/unique.h>

#include <algorithm>
#include <map>
#include <tuple>
#include <vector>

#include "ctx.h"

namespace osm {

namespace {

__global__ void k_vi_index(int64_t n, const double* __restrict__ val, const double* __restrict__ dict, int ndict,
                           uint16_t* __restrict__ vidx) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = val[i];
  int lo = 0, hi = ndict;
  while (lo < hi) {  // first dict entry >= v (the entry is present: dict = unique(val))
    const int mid = (lo + hi) / 2;
    if (dict[mid] < v) lo = mid + 1; else hi = mid;
  }
  vidx[i] = (uint16_t)lo;
}

// Largest |col - own internal row| over the SELL (tile t, lane l = row 256 t + l), into *maxoff.
__global__ void k_vi_maxoff(int64_t ntile, const int64_t* __restrict__ toff, const int32_t* __restrict__ twidth,
                            const int32_t* __restrict__ col, int32_t* __restrict__ maxoff) {
  const int64_t t = blockIdx.x;
  if (t >= ntile) return;
  const int64_t row = t * kRowsPerBlock + threadIdx.x;
  const int w = twidth[t];
  const int64_t base = toff[t] + threadIdx.x;
  int64_t m = 0;
  for (int k = 0; k < w; ++k) {
    const int64_t d = (int64_t)col[base + (int64_t)kRowsPerBlock * k] - row;
    m = max(m, d < 0 ? -d : d);
  }
  atomicMax(maxoff, (int32_t)min(m, (int64_t)INT32_MAX));
}

// Packed layout: tile t holds rows 256 t + r; its entries are grouped by 4 (width padded to a
// multiple of 4 with (zero value, offset 0) entries); group g of row r is the uint4 at
// poff[t] + 4 (256 g + r) (in 32-bit words).  Entry = (value index << 16) | (uint16) offset, or in
// the wide form (value index << 20) | (offset & 0xfffff) (12-bit index, 20-bit signed offset).
template <bool W>
__global__ void k_vi_pack(int64_t ntile, const int64_t* __restrict__ toff, const int32_t* __restrict__ twidth,
                          const int32_t* __restrict__ vtw, const int64_t* __restrict__ poff,
                          const uint16_t* __restrict__ vidx, const int32_t* __restrict__ col, uint32_t zero_idx,
                          uint32_t* __restrict__ packed) {
  constexpr int IS = W ? 20 : 16;
  constexpr uint32_t OM = W ? 0xfffffu : 0xffffu;
  const int64_t t = blockIdx.x;
  if (t >= ntile) return;
  const int r = threadIdx.x;
  const int64_t row = t * kRowsPerBlock + r;
  const int w = twidth[t];
  const int w4 = (vtw[t] + 3) & ~3;
  const int64_t base = toff[t] + r;
  int kk = 0;  // kept entries so far (the row's exact zeros and SELL padding are dropped, order kept)
  for (int k = 0; k < w; ++k) {
    const int64_t i = base + (int64_t)kRowsPerBlock * k;
    if (vidx[i] == zero_idx) continue;
    const uint32_t e = ((uint32_t)vidx[i] << IS) | ((uint32_t)(int32_t)(col[i] - row) & OM);
    packed[poff[t] + 4 * ((int64_t)kRowsPerBlock * (kk >> 2) + r) + (kk & 3)] = e;
    ++kk;
  }
  for (; kk < w4; ++kk) packed[poff[t] + 4 * ((int64_t)kRowsPerBlock * (kk >> 2) + r) + (kk & 3)] = zero_idx << IS;
}

// Kept (nonzero-value) entries per row: per-tile maximum (the packed width) and per-subdomain totals.
__global__ void k_vi_kept(int64_t ntile, const int64_t* __restrict__ toff, const int32_t* __restrict__ twidth,
                          const uint16_t* __restrict__ vidx, uint32_t zero_idx, const int32_t* __restrict__ blk_sub,
                          int32_t* __restrict__ vtw, unsigned long long* __restrict__ kept_sub) {
  __shared__ int wmax;
  const int64_t t = blockIdx.x;
  if (t >= ntile) return;
  if (threadIdx.x == 0) wmax = 0;
  __syncthreads();
  const int w = twidth[t];
  const int64_t base = toff[t] + threadIdx.x;
  int kk = 0;
  for (int k = 0; k < w; ++k) kk += vidx[base + (int64_t)kRowsPerBlock * k] != zero_idx;
  atomicMax(&wmax, kk);
  atomicAdd(&kept_sub[blk_sub[t]], (unsigned long long)kk);
  __syncthreads();
  if (threadIdx.x == 0) vtw[t] = wmax;
}

// K^N values back at the Robin fold positions (the dictionary is built from the unfolded matrix).
__global__ void k_vi_unfold(int64_t nfold, const int64_t* __restrict__ pos, const double* __restrict__ kn,
                            double* __restrict__ val) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= nfold || pos[e] < 0) return;
  val[pos[e]] = kn[e];
}

__global__ void k_vi_fold_slots(int64_t nfold, const int64_t* __restrict__ pos, const int32_t* __restrict__ slot,
                                uint16_t* __restrict__ vidx) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= nfold || pos[e] < 0) return;
  vidx[pos[e]] = (uint16_t)slot[e];
}

}  // namespace

// Variant 10 (3-byte entries): regroups the 4-entry packed words (dict index << 16 | uint16 offset) into
// 8-entry groups split in an offset stream and an index stream; entry order within a row is kept,
// the odd tail group is padded with (0.0, offset 0) entries like the packed rows.
__global__ void k_vi3_pack(const int32_t* __restrict__ tw, const int64_t* __restrict__ poff,
                           const uint32_t* __restrict__ packed, const int64_t* __restrict__ base3, uint32_t zero_word,
                           uint4* __restrict__ off3, uint2* __restrict__ idx3) {
  const int64_t t = blockIdx.x;
  const int r = threadIdx.x;
  const int n4 = (tw[t] + 3) >> 2, n8 = (tw[t] + 7) >> 3;
  for (int G = 0; G < n8; ++G) {
    uint32_t w[8];
    for (int h = 0; h < 2; ++h) {
      const int g4 = 2 * G + h;
      uint4 v = make_uint4(zero_word, zero_word, zero_word, zero_word);
      if (g4 < n4) v = *reinterpret_cast<const uint4*>(packed + poff[t] + 4 * ((int64_t)kRowsPerBlock * g4 + r));
      w[4 * h] = v.x;
      w[4 * h + 1] = v.y;
      w[4 * h + 2] = v.z;
      w[4 * h + 3] = v.w;
    }
    uint4 o;
    o.x = (w[0] & 0xffffu) | (w[1] << 16);
    o.y = (w[2] & 0xffffu) | (w[3] << 16);
    o.z = (w[4] & 0xffffu) | (w[5] << 16);
    o.w = (w[6] & 0xffffu) | (w[7] << 16);
    uint2 ix;
    ix.x = (w[0] >> 16) | ((w[1] >> 16) << 8) | ((w[2] >> 16) << 16) | ((w[3] >> 16) << 24);
    ix.y = (w[4] >> 16) | ((w[5] >> 16) << 8) | ((w[6] >> 16) << 16) | ((w[7] >> 16) << 24);
    const int64_t at = base3[t] + (int64_t)kRowsPerBlock * G + r;
    off3[at] = o;
    idx3[at] = ix;
  }
}

static void vi3_free(Ctx& c) {
  if (c.vi3_off) cudaFree(c.vi3_off);
  if (c.vi3_idx) cudaFree(c.vi3_idx);
  if (c.vi3_base) cudaFree(c.vi3_base);
  c.vi3_off = nullptr;
  c.vi3_idx = nullptr;
  c.vi3_base = nullptr;
  c.vi3_ok = false;
  c.vi3_groups = 0;
}

static void vi3_build(Ctx& c, const std::vector<int32_t>& tw, uint32_t zero_idx) {
  vi3_free(c);
  if (c.vi_wide || c.vi_ndict > 256) return;
  std::vector<int64_t> base(c.nblk_total);
  int64_t groups = 0;
  for (int64_t t = 0; t < c.nblk_total; ++t) {
    base[t] = groups;
    groups += (int64_t)((tw[t] + 7) >> 3) * kRowsPerBlock;
  }
  OSM_CUDA(cudaMalloc(&c.vi3_base, sizeof(int64_t) * c.nblk_total));
  OSM_CUDA(cudaMemcpy(c.vi3_base, base.data(), sizeof(int64_t) * c.nblk_total, cudaMemcpyHostToDevice));
  OSM_CUDA(cudaMalloc(&c.vi3_off, sizeof(uint4) * std::max<int64_t>(1, groups)));
  OSM_CUDA(cudaMalloc(&c.vi3_idx, sizeof(uint2) * std::max<int64_t>(1, groups)));
  k_vi3_pack<<<(unsigned)c.nblk_total, kRowsPerBlock, 0, c.stream>>>(c.vi_tw, c.vi_poff, c.vi_packed, c.vi3_base,
                                                                     zero_idx << 16, c.vi3_off, c.vi3_idx);
  OSM_CHECK_LAUNCH();
  ++c.launches;
  OSM_CUDA(cudaStreamSynchronize(c.stream));
  c.vi3_groups = groups;
  c.vi3_ok = true;
}

void vi_free(Ctx& c) {
  vi3_free(c);
  if (c.vi_idx) cudaFree(c.vi_idx);
  if (c.vi_dict) cudaFree(c.vi_dict);
  if (c.vi_packed) cudaFree(c.vi_packed);
  if (c.vi_poff) cudaFree(c.vi_poff);
  if (c.vi_tw) cudaFree(c.vi_tw);
  c.vi_tw = nullptr;
  c.vi_kept.clear();
  c.vi_idx = nullptr;
  c.vi_dict = nullptr;
  c.vi_packed = nullptr;
  c.vi_poff = nullptr;
  c.vi_ok = false;
  c.vi_packed_ok = false;
  c.vi_wide = false;
  c.vi_fold_tuples.clear();
}

// Builds the dictionary, the 16-bit value indices (fold positions -> tuple slots) and the int16
// column offsets from the fp64 SELL arrays.  Fold tuples are keyed by the side kind (0: left slab
// of its interface, 1: right slab) -- shared by every interface, valid while p and q are uniform per
// kind -- or, with per_side, by the individual side.
void vi_build(Ctx& c, bool per_side) {
  vi_free(c);
  const int64_t n = c.sell_total;
  if (n == 0) return;
  // 1. distinct K^N values, from the UNFOLDED matrix: c.sell_val holds K^N + p M + q S on the fold
  // positions once a Robin term has been applied (a per-side rebuild from vi_apply_robin), and those
  // folded values must not enter the base dictionary (the fold positions get tuple slots below)
  double* unf = nullptr;
  OSM_CUDA(cudaMalloc(&unf, sizeof(double) * n));
  OSM_CUDA(cudaMemcpyAsync(unf, c.sell_val, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.stream));
  if (c.nfold) {
    k_vi_unfold<<<(unsigned)ceil_div(c.nfold, 256), 256, 0, c.stream>>>(c.nfold, c.fold_pos, c.fold_kn, unf);
    OSM_CHECK_LAUNCH();
    ++c.launches;
  }
  double* tmp = nullptr;
  OSM_CUDA(cudaMalloc(&tmp, sizeof(double) * (n + 1)));
  OSM_CUDA(cudaMemcpyAsync(tmp, unf, sizeof(double) * n, cudaMemcpyDeviceToDevice, c.stream));
  OSM_CUDA(cudaMemsetAsync(tmp + n, 0, sizeof(double), c.stream));  // 0.0 is always in the dictionary
  thrust::device_ptr<double> tp(tmp);
  thrust::sort(thrust::cuda::par.on(c.stream), tp, tp + n + 1);
  const int64_t nd = thrust::unique(thrust::cuda::par.on(c.stream), tp, tp + n + 1) - tp;
  // 2. fold tuples (side, K^N, m, s) -> slots after the K^N values
  std::vector<int64_t> pos(c.nfold);
  std::vector<double> kn(c.nfold), m(c.nfold), sv(c.nfold);
  std::vector<int32_t> side(c.nfold);
  if (c.nfold) {
    OSM_CUDA(cudaMemcpyAsync(pos.data(), c.fold_pos, sizeof(int64_t) * c.nfold, cudaMemcpyDeviceToHost, c.stream));
    OSM_CUDA(cudaMemcpyAsync(kn.data(), c.fold_kn, sizeof(double) * c.nfold, cudaMemcpyDeviceToHost, c.stream));
    OSM_CUDA(cudaMemcpyAsync(m.data(), c.fold_m, sizeof(double) * c.nfold, cudaMemcpyDeviceToHost, c.stream));
    OSM_CUDA(cudaMemcpyAsync(sv.data(), c.fold_s, sizeof(double) * c.nfold, cudaMemcpyDeviceToHost, c.stream));
    OSM_CUDA(cudaMemcpyAsync(side.data(), c.fold_side, sizeof(int32_t) * c.nfold, cudaMemcpyDeviceToHost, c.stream));
  }
  OSM_CUDA(cudaStreamSynchronize(c.stream));
  std::map<std::tuple<int32_t, double, double, double>, int32_t> tuples;
  std::vector<int32_t> slot(c.nfold, 0);
  for (int64_t e = 0; e < c.nfold; ++e) {
    const int32_t key_side = per_side ? side[e] : c.sides[side[e]].which;
    auto key = std::make_tuple(key_side, kn[e], m[e], sv[e]);
    auto it = tuples.find(key);
    if (it == tuples.end()) it = tuples.emplace(key, (int32_t)(nd + tuples.size())).first;
    slot[e] = it->second;
  }
  const int64_t ndict = nd + (int64_t)tuples.size();
  if (ndict > 65536) {  // too many distinct values: stay on the fp64 SELL path
    cudaFree(tmp);
    cudaFree(unf);
    return;
  }
  c.vi_fold_tuples.assign(tuples.size(), {});
  for (const auto& kv : tuples) {
    auto& T = c.vi_fold_tuples[kv.second - nd];
    T.side = std::get<0>(kv.first);
    T.kn = std::get<1>(kv.first);
    T.m = std::get<2>(kv.first);
    T.s = std::get<3>(kv.first);
  }
  c.vi_ndict = ndict;
  c.vi_nbase = nd;
  OSM_CUDA(cudaMalloc(&c.vi_dict, sizeof(double) * ndict));
  OSM_CUDA(cudaMemcpyAsync(c.vi_dict, tmp, sizeof(double) * nd, cudaMemcpyDeviceToDevice, c.stream));
  // tail starts as K^N (alpha = 0); apply_robin rewrites it
  std::vector<double> tail(tuples.size());
  for (size_t t = 0; t < tail.size(); ++t) tail[t] = c.vi_fold_tuples[t].kn;
  if (!tail.empty())
    OSM_CUDA(cudaMemcpyAsync(c.vi_dict + nd, tail.data(), sizeof(double) * tail.size(), cudaMemcpyHostToDevice,
                             c.stream));
  // 3. indices (from the unfolded K^N SELL values), then fold positions -> tuple slots
  OSM_CUDA(cudaMalloc(&c.vi_idx, sizeof(uint16_t) * n));
  k_vi_index<<<(unsigned)ceil_div(n, 256), 256, 0, c.stream>>>(n, unf, tmp, (int)nd, c.vi_idx);
  OSM_CHECK_LAUNCH();
  ++c.launches;
  if (c.nfold) {
    int32_t* d_slot = nullptr;
    OSM_CUDA(cudaMalloc(&d_slot, sizeof(int32_t) * c.nfold));
    OSM_CUDA(cudaMemcpyAsync(d_slot, slot.data(), sizeof(int32_t) * c.nfold, cudaMemcpyHostToDevice, c.stream));
    k_vi_fold_slots<<<(unsigned)ceil_div(c.nfold, 256), 256, 0, c.stream>>>(c.nfold, c.fold_pos, d_slot, c.vi_idx);
    OSM_CHECK_LAUNCH();
    ++c.launches;
    OSM_CUDA(cudaStreamSynchronize(c.stream));
    cudaFree(d_slot);
  }
  // 4. offset width: 16-bit offsets with 16-bit indices, else 20-bit offsets with 12-bit indices
  OSM_CUDA(cudaMemsetAsync(c.d_flags + 2, 0, sizeof(int32_t), c.stream));
  k_vi_maxoff<<<(unsigned)c.nblk_total, kRowsPerBlock, 0, c.stream>>>(c.nblk_total, c.sell_soff, c.sell_swidth,
                                                                     c.sell_col, c.d_flags + 2);
  OSM_CHECK_LAUNCH();
  ++c.launches;
  int32_t flags[4];
  OSM_CUDA(cudaMemcpyAsync(flags, c.d_flags, sizeof(flags), cudaMemcpyDeviceToHost, c.stream));
  OSM_CUDA(cudaStreamSynchronize(c.stream));
  OSM_CUDA(cudaMemsetAsync(c.d_flags + 2, 0, sizeof(int32_t), c.stream));
  cudaFree(tmp);
  cudaFree(unf);
  const int32_t maxoff = flags[2];
  bool wide = false;
  // index of 0.0 in the sorted dictionary
  std::vector<double> hd(nd);
  OSM_CUDA(cudaMemcpy(hd.data(), c.vi_dict, sizeof(double) * nd, cudaMemcpyDeviceToHost));
  const uint32_t zero_idx = (uint32_t)(std::lower_bound(hd.begin(), hd.end(), 0.0) - hd.begin());
  if (maxoff > 32767) {
    if (maxoff > 524287 || ndict > 4096) {  // neither packed form fits
      if (c.sort_key == 6 && ndict <= 256) {
        // row order 6 (class arrays: a neighbour in another class is a class array away): no packed
        // SELL copy, but the brick copy needs only the dictionary and the per-entry indices
        c.vi_per_side = per_side;
        c.vi_ok = true;
        c.vi_packed_ok = false;
        brick_build(c, c.vi_idx, zero_idx);
        cudaFree(c.vi_idx);
        c.vi_idx = nullptr;
        return;
      }
      vi_free(c);
      return;
    }
    wide = true;
  }
  // 5. packed copy (4 entries of a row per 16-byte load).  Entries whose value is exactly 0.0 -- the
  // Kuhn stencil's structural zeros (~19 % of P2 entries) and the SELL padding -- are
  // dropped: they add exact zeros (+-0) to the row sums, so the iterations stay the same.  Fold
  // positions keep their own dictionary slots and are never dropped.
  const int nloc = c.s_end - c.s_begin;
  unsigned long long* d_kept = nullptr;
  OSM_CUDA(cudaMalloc(&d_kept, sizeof(unsigned long long) * std::max(1, nloc)));
  OSM_CUDA(cudaMemsetAsync(d_kept, 0, sizeof(unsigned long long) * std::max(1, nloc), c.stream));
  OSM_CUDA(cudaMalloc(&c.vi_tw, sizeof(int32_t) * c.nblk_total));
  k_vi_kept<<<(unsigned)c.nblk_total, kRowsPerBlock, 0, c.stream>>>(c.nblk_total, c.sell_soff, c.sell_swidth, c.vi_idx,
                                                                   zero_idx, c.blk_sub, c.vi_tw, d_kept);
  OSM_CHECK_LAUNCH();
  ++c.launches;
  std::vector<int32_t> tw(c.nblk_total);
  std::vector<unsigned long long> kept(std::max(1, nloc));
  OSM_CUDA(cudaMemcpyAsync(tw.data(), c.vi_tw, sizeof(int32_t) * c.nblk_total, cudaMemcpyDeviceToHost, c.stream));
  OSM_CUDA(cudaMemcpyAsync(kept.data(), d_kept, sizeof(unsigned long long) * kept.size(), cudaMemcpyDeviceToHost,
                           c.stream));
  OSM_CUDA(cudaStreamSynchronize(c.stream));
  cudaFree(d_kept);
  c.vi_kept.assign(kept.begin(), kept.begin() + nloc);
  std::vector<int64_t> poff(c.nblk_total);
  int64_t words = 0;
  for (int64_t t = 0; t < c.nblk_total; ++t) {
    poff[t] = words;
    words += (int64_t)((tw[t] + 3) & ~3) * kRowsPerBlock;
  }
  OSM_CUDA(cudaMalloc(&c.vi_poff, sizeof(int64_t) * c.nblk_total));
  OSM_CUDA(cudaMemcpy(c.vi_poff, poff.data(), sizeof(int64_t) * c.nblk_total, cudaMemcpyHostToDevice));
  OSM_CUDA(cudaMalloc(&c.vi_packed, sizeof(uint32_t) * std::max<int64_t>(1, words)));
  if (wide)
    k_vi_pack<true><<<(unsigned)c.nblk_total, kRowsPerBlock, 0, c.stream>>>(
        c.nblk_total, c.sell_soff, c.sell_swidth, c.vi_tw, c.vi_poff, c.vi_idx, c.sell_col, zero_idx, c.vi_packed);
  else
    k_vi_pack<false><<<(unsigned)c.nblk_total, kRowsPerBlock, 0, c.stream>>>(
        c.nblk_total, c.sell_soff, c.sell_swidth, c.vi_tw, c.vi_poff, c.vi_idx, c.sell_col, zero_idx, c.vi_packed);
  OSM_CHECK_LAUNCH();
  ++c.launches;
  OSM_CUDA(cudaStreamSynchronize(c.stream));
  c.vi_words = words;
  c.vi_per_side = per_side;
  c.vi_wide = wide;
  c.vi_ok = true;
  c.vi_packed_ok = true;
  if (c.sort_key == 6) brick_build(c, c.vi_idx, zero_idx);  // the brick copy reads the per-entry indices
  cudaFree(c.vi_idx);
  c.vi_idx = nullptr;
  vi3_build(c, tw, zero_idx);
}

// Dictionary tail for the current Robin coefficients: value = K^N + (p m + q s), rounded exactly
// as k_fold_apply rounds it.
void vi_apply_robin(Ctx& c, const std::vector<double>& p_side, const std::vector<double>& q_side) {
  if (!c.vi_ok || c.vi_fold_tuples.empty()) return;
  // coefficients per tuple key: the side itself, or the side kind when uniform over interfaces
  std::vector<double> pk(2, 0.0), qk(2, 0.0);
  if (!c.vi_per_side) {
    bool seen[2] = {false, false}, uniform = true;
    for (size_t k = 0; k < c.sides.size(); ++k) {
      const int w = c.sides[k].which;
      if (!seen[w]) {
        pk[w] = p_side[k];
        qk[w] = q_side[k];
        seen[w] = true;
      } else if (pk[w] != p_side[k] || qk[w] != q_side[k]) {
        uniform = false;
      }
    }
    if (!uniform) {  // per-interface coefficients: rebuild with per-side slots
      vi_build(c, true);
      if (!c.vi_ok) return;
      vi_apply_robin(c, p_side, q_side);
      return;
    }
  }
  std::vector<double> tail(c.vi_fold_tuples.size());
  for (size_t t = 0; t < tail.size(); ++t) {
    const auto& T = c.vi_fold_tuples[t];
    const double pt = c.vi_per_side ? p_side[T.side] : pk[T.side];
    const double qt = c.vi_per_side ? q_side[T.side] : qk[T.side];
    volatile double a = pt * T.m;  // no contraction: match __dmul_rn / __dadd_rn
    volatile double b = qt * T.s;
    volatile double ab = a + b;
    tail[t] = T.kn + ab;
  }
  OSM_CUDA(cudaMemcpyAsync(c.vi_dict + c.vi_nbase, tail.data(), sizeof(double) * tail.size(), cudaMemcpyHostToDevice,
                           c.stream));
  OSM_CUDA(cudaStreamSynchronize(c.stream));
}

}  // namespace osm

// libosm C ABI and host driver of the optimized Schwarz iteration.
//
// Host side only orchestrates: every arithmetic step of the solve runs in the
// kernels of assemble.cu / schwarz_kernels.cu.  Cross-GPU traffic (interface
// traces, interface-row residuals, per-subdomain residual sums, the solution
// gather) goes through NCCL over NVLink; subdomains that share a GPU exchange
// through device memory inside the interface kernels.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>
#include <string>
#include <tuple>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "ctx.h"

namespace osm {

thread_local std::string g_last_error;

// NVTX ranges (tracing) around the phases of a solve; free when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

#define OSM_NCCL(call)                                                                         \
  do {                                                                                         \
    ncclResult_t r_ = (call);                                                                  \
    if (r_ != ncclSuccess) ::osm::fail(OSM_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

template <class T>
static T* dalloc(int64_t n) {
  void* p = nullptr;
  if (n <= 0) n = 1;
  OSM_CUDA(cudaMalloc(&p, sizeof(T) * (size_t)n));
  return (T*)p;
}
template <class T>
static void dfree(T*& p) {
  if (p) cudaFree((void*)p);
  p = nullptr;
}
template <class T>
static T* dupload(const Ctx& c, const std::vector<T>& h) {
  T* d = dalloc<T>((int64_t)h.size());
  if (!h.empty()) OSM_CUDA(cudaMemcpyAsync(d, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, c.stream));
  return d;
}

// ------------------------------------------------------------------ timers
void timer_begin(Ctx& c, int id) {
  if (!c.timing) return;
  KernelTimer& t = c.timers[id];
  if ((int64_t)t.ev.size() < 2 * (t.used + 1)) {
    for (int k = 0; k < 256; ++k) {
      cudaEvent_t e;
      OSM_CUDA(cudaEventCreate(&e));
      t.ev.push_back(e);
    }
  }
  OSM_CUDA(cudaEventRecord(t.ev[2 * t.used], c.stream));
}
void timer_end(Ctx& c, int id) {
  if (!c.timing) return;
  KernelTimer& t = c.timers[id];
  OSM_CUDA(cudaEventRecord(t.ev[2 * t.used + 1], c.stream));
  t.used++;
}
static void timers_collect(Ctx& c) {
  if (!c.timing) return;
  OSM_CUDA(cudaStreamSynchronize(c.stream));
  for (auto& t : c.timers) {
    for (int64_t i = 0; i < t.used; ++i) {
      float ms = 0.f;
      OSM_CUDA(cudaEventElapsedTime(&ms, t.ev[2 * i], t.ev[2 * i + 1]));
      t.total_ms += ms;
    }
    t.launches += t.used;
    t.used = 0;
  }
}

// ------------------------------------------------------------------ teardown

static void drop_graph(Ctx& c) {
  if (c.cg_graph) cudaGraphExecDestroy(c.cg_graph);
  c.cg_graph = nullptr;
  for (auto& g : c.cg_graph_g) {
    if (g) cudaGraphExecDestroy(g);
    g = nullptr;
  }
}

static void free_assembly(Ctx& c) {
  drop_graph(c);
  brick_free(c);
  batch_free(c);
  vi_free(c);
  for (auto& s : c.subs) {
    dfree(s.rowptr);
    dfree(s.col);
    dfree(s.val);
    dfree(s.perm);
    dfree(s.iperm);
  }
  c.subs.clear();
  for (auto& sd : c.sides) {
    dfree(sd.map_c);
    dfree(sd.map_g);
    dfree(sd.out);
    dfree(sd.inbuf);
  }
  c.sides.clear();
  dfree(c.d_col_begin);
  dfree(c.d_load_begin);
  dfree(c.d_cols);
  dfree(c.d_contribs);
  dfree(c.d_loads);
  dfree(c.d_mrow);
  dfree(c.d_mcol);
  dfree(c.d_mval);
  dfree(c.d_sval);
  dfree(c.sell_val);
  dfree(c.sell_col);
  dfree(c.sell_soff);
  dfree(c.sell_swidth);
  dfree(c.blk_sub);
  dfree(c.vblk_sub);
  dfree(c.vblk_tile0);
  dfree(c.vblk_ntile);
  dfree(c.islot);
  dfree(c.fold_pos);
  dfree(c.fold_m);
  dfree(c.fold_s);
  dfree(c.fold_kn);
  dfree(c.fold_diag_row);
  dfree(c.fold_side);
  dfree(c.x);
  dfree(c.r);
  dfree(c.p);
  dfree(c.q);
  dfree(c.dinv);
  dfree(c.b);
  dfree(c.ut);
  dfree(c.lam_all);
  dfree(c.unbr_all);
  dfree(c.wif_all);
  dfree(c.d_sides);
  dfree(c.part);
  dfree(c.part_upd);
  dfree(c.side_part);
  dfree(c.side_sum);
  dfree(c.side_cnt);
  dfree(c.st);
  dfree(c.phi);
  dfree(c.d_mf_sub);
  dfree(c.d_mf_begin);
  dfree(c.d_mf_delta);
  dfree(c.d_mf_val);
  dfree(c.d_mf_src);
  c.mf_ok = false;
  c.mf_entries = 0;
  delete c.h_mf_const;
  c.h_mf_const = nullptr;
  dfree(c.d_mf_code);
  dfree(c.d_dcode);
  c.h_dcode_tab.clear();
  c.assembled = false;
  c.density_set = false;
}

// ------------------------------------------------------------------ assembly
static SlabGeom slab_geom(const Ctx& c, int s) {
  SlabGeom g{};
  const int o = c.mesh.order;
  g.c0 = c.cstart[s];
  g.c1 = c.cstart[s + 1];
  g.nx = c.mesh.nx;
  g.ny = c.mesh.ny;
  g.nz = c.mesh.nz;
  g.Ny = o * c.mesh.ny + 1;
  g.Nz = o * c.mesh.nz + 1;
  const int64_t Nx = o * c.mesh.nx + 1;
  g.I_lo = std::max<int64_t>(o * g.c0, 1);
  g.I_hi = std::min<int64_t>(o * g.c1, Nx - 2);
  g.nI = g.I_hi - g.I_lo + 1;
  g.nJ = g.Ny - 2;
  g.nK = g.Nz - 2;
  g.order = o;
  return g;
}


// Host copy of the value-indexed dictionary (the variant 6 kernel parameter); captured graphs embed it.
static void vi_sync_host_dict(Ctx& c) {
  c.h_vi_dict.assign(c.vi_ok ? c.vi_ndict : 0, 0.0);
  if (c.vi_ok && c.vi_ndict > 0)
    OSM_CUDA(cudaMemcpy(c.h_vi_dict.data(), c.vi_dict, sizeof(double) * c.vi_ndict, cudaMemcpyDeviceToHost));
  drop_graph(c);
}

static void mf_refresh(Ctx& c) {
  launch_mf_refresh(c);
  OSM_CUDA(cudaMemsetAsync(c.d_flags + 3, 0, sizeof(int32_t), c.stream));
  launch_mf_verify(c, c.d_flags + 3);
  int32_t bad = 0;
  OSM_CUDA(cudaMemcpyAsync(&bad, c.d_flags + 3, sizeof(int32_t), cudaMemcpyDeviceToHost, c.stream));
  OSM_CUDA(cudaStreamSynchronize(c.stream));
  drop_graph(c);  // captured launches embed the kernel-parameter tables
  if (bad) {
    c.mf_ok = false;
    return;
  }
  // deduplicated kernel-parameter copy of the tables
  if (!c.h_mf_const) c.h_mf_const = new MfConst();
  MfConst& P = *c.h_mf_const;
  std::memset(&P, 0, sizeof(MfConst));
  const int ntab = (int)c.h_mf_begin.size() - 1;
  const int nloc = c.s_end - c.s_begin, ncls = c.mesh.order * c.mesh.order * c.mesh.order;
  if (nloc > kMfMaxSub || ncls > 8) return;
  std::vector<double> val(c.mf_entries);
  OSM_CUDA(cudaMemcpy(val.data(), c.d_mf_val, sizeof(double) * c.mf_entries, cudaMemcpyDeviceToHost));
  std::map<std::vector<int64_t>, int> seen;
  int ng = 0, nt = 0;
  P.gbeg[0] = 0;
  for (int t = 0; t < ntab; ++t) {
    std::vector<int64_t> key;
    for (int e = c.h_mf_begin[t]; e < c.h_mf_begin[t + 1]; ++e) {
      int64_t bits;
      std::memcpy(&bits, &val[e], sizeof(bits));
      key.push_back(c.h_mf_delta[e]);
      key.push_back(bits);
    }
    auto it = seen.find(key);
    if (it == seen.end()) {
      // the constant-bank copy keeps only the nonzero values (the Kuhn stencil's exact zeros add +-0
      // to the row sums), in column order, padded to whole groups of 4 with (0, +0.0)
      std::vector<int> keep;
      double diag = 0.0;
      for (int e = c.h_mf_begin[t]; e < c.h_mf_begin[t + 1]; ++e) {
        if (val[e] == 0.0) continue;
        keep.push_back(e);
        if (c.h_mf_delta[e] == 0) diag = val[e];
      }
      const int g = ((int)keep.size() + 3) / 4;
      if (nt >= kMfMaxTab || ng + g > kMfMaxGroups) return;  // too many: global tables
      for (int k = 0; k < 4 * g; ++k) {
        const bool real = k < (int)keep.size();
        (&P.delta[0].x)[4 * ng + k] = real ? c.h_mf_delta[keep[k]] : 0;
        P.val[4 * ng + k] = real ? val[keep[k]] : 0.0;
      }
      P.dinv[nt] = diag > 0.0 ? 1.0 / diag : 0.0;
      ng += g;
      it = seen.emplace(key, nt).first;
      P.gbeg[++nt] = ng;
    }
    P.tabid[t] = (int16_t)it->second;  // t = (ls * 3 + kind) * ncls + class, as mf_table_of
  }
  P.valid = 1;
  // per-row table codes for the vector kernels (D^{-1} from the tables, dummy rows skipped)
  if (nt <= 255) {
    if (!c.d_mf_code) c.d_mf_code = dalloc<uint8_t>(c.nrows_total);
    std::vector<int16_t> tabid(P.tabid, P.tabid + ntab);
    int16_t* d_tabid = dupload(c, tabid);
    launch_mf_codes(c, d_tabid);
    OSM_CUDA(cudaStreamSynchronize(c.stream));
    dfree(d_tabid);
  } else {
    dfree(c.d_mf_code);
  }
}

// D^{-1} codes for the vector kernels of the SELL variants.  On the structured mesh the Robin-folded
// diagonal takes a few distinct values (row kind x parity class), so each row's D^{-1} is replaced by a
// 1-byte index into a table of its distinct bit patterns (the same doubles: iterations stay bitwise).
// More than 255 distinct values: no codes, the 8-byte stream stays.  Rebuilt after every Robin fold.
static void dcode_build(Ctx& c) {
  c.h_dcode_tab.clear();
  if (!c.dcode_on || c.nrows_total == 0 || c.nrows_total % 2) return;
  std::vector<double> dv((size_t)c.nrows_total);
  OSM_CUDA(cudaMemcpy(dv.data(), c.dinv, sizeof(double) * dv.size(), cudaMemcpyDeviceToHost));
  std::map<uint64_t, int> idx;
  std::vector<double> tab;
  std::vector<uint8_t> code(dv.size());
  for (size_t i = 0; i < dv.size(); ++i) {
    uint64_t bits;
    std::memcpy(&bits, &dv[i], 8);
    if (bits == 0) {  // +0.0 (padding rows): 0xff decodes to +0.0
      code[i] = 0xff;
      continue;
    }
    auto it = idx.find(bits);
    if (it == idx.end()) {
      if ((int)tab.size() >= kMfMaxTab) return;  // too many distinct values: keep the stream
      it = idx.emplace(bits, (int)tab.size()).first;
      tab.push_back(dv[i]);
    }
    code[i] = (uint8_t)it->second;
  }
  if (!c.d_dcode) c.d_dcode = dalloc<uint8_t>(c.nrows_total);
  OSM_CUDA(cudaMemcpy(c.d_dcode, code.data(), code.size(), cudaMemcpyHostToDevice));
  c.h_dcode_tab = tab;
}

// Matrix-free Kuhn-stencil tables (SpMV variant 5, row order 4).  For every
// local subdomain, row kind (0 interior, 1 left interface plane, 2 right interface plane) and
// parity class, the longest row of that kind and class is the representative: its CSR columns,
// as lattice offsets, become constant internal offsets (the layout makes them row-independent)
// and its SELL positions the value sources (k_mf_refresh copies the assembled, Robin-folded
// values bitwise).  k_mf_verify then checks every row of the subdomain against its table
// (same entries in the same order, same bits, table entries into dummy rows aside); on any
// mismatch (e.g. slabs too thin for a complete representative) mf_ok drops to false and
// variant 5 falls back to the SELL variants.
static void mf_build(Ctx& c, const std::vector<std::vector<int32_t>>& h_iperm,
                     const std::vector<std::vector<int32_t>>& h_len, const std::vector<int64_t>& h_soff) {
  c.mf_ok = false;
  const int o = c.mesh.order, ncls = o * o * o;
  const int nloc = c.s_end - c.s_begin;
  std::vector<MfSub> msub(nloc);
  std::vector<int32_t> begin(1, 0), delta;
  std::vector<int64_t> src;
  for (int ls = 0; ls < nloc; ++ls) {
    const Sub& S = c.subs[ls];
    MfSub& M = msub[ls];
    const int64_t nIs = (int64_t)o * (S.g.c1 - S.g.c0) + 1;
    const int64_t hI = (nIs + o - 1) / o, hJ = (S.g.Ny + o - 1) / o, hK = (S.g.Nz + o - 1) / o;
    M.row0 = S.row0;
    M.hJ = (int32_t)hJ;
    M.hK = (int32_t)hK;
    M.hJK = (int32_t)(hJ * hK);
    M.hIJK = (int32_t)(hI * hJ * hK);
    M.nIs = (int32_t)nIs;
    M.Ny = (int32_t)S.g.Ny;
    M.Nz = (int32_t)S.g.Nz;
    M.dir_lo = S.g.c0 == 0;
    M.dir_hi = S.g.c1 == c.mesh.nx;
    M.tab0 = ls * 3 * ncls;
    M.o = o;
    M.nclass = ncls;
    M.inv_hIJK = 1.0 / (double)M.hIJK;
    M.inv_hJK = 1.0 / (double)M.hJK;
    M.inv_hJ = 1.0 / (double)M.hJ;
    auto internal_of = [&](int64_t Il, int64_t J, int64_t K) {  // slab-local lattice point (>= 0) -> internal
      const int64_t cl = Il % o + o * (J % o + o * (K % o));
      return cl * M.hIJK + J / o + hJ * (K / o + hK * (Il / o));
    };
    std::vector<int64_t> rep(3 * ncls, -1);
    const auto& len = h_len[ls];
    for (int64_t lc = 0; lc < S.n; ++lc) {
      const int64_t Ig = S.g.I_lo + lc % S.g.nI, t = lc / S.g.nI, J = 1 + t % S.g.nJ, K = 1 + t / S.g.nJ;
      const int64_t Il = Ig - (int64_t)o * S.g.c0;
      const int kind = Il == 0 ? 1 : (Il == nIs - 1 ? 2 : 0);
      const int t2 = kind * ncls + (int)(Il % o + o * (J % o + o * (K % o)));
      if (rep[t2] < 0 || len[lc] > len[rep[t2]]) rep[t2] = lc;
    }
    std::vector<int64_t> rowptr(S.n + 1, 0);
    for (int64_t i = 0; i < S.n; ++i) rowptr[i + 1] = rowptr[i] + len[i];
    for (int t2 = 0; t2 < 3 * ncls; ++t2) {
      if (rep[t2] >= 0) {
        const int64_t lc = rep[t2], nl = len[lc];
        std::vector<int32_t> cols(nl);
        OSM_CUDA(cudaMemcpy(cols.data(), S.col + rowptr[lc], sizeof(int32_t) * nl, cudaMemcpyDeviceToHost));
        const int64_t I0 = S.g.I_lo + lc % S.g.nI, t0 = lc / S.g.nI, J0 = 1 + t0 % S.g.nJ, K0 = 1 + t0 / S.g.nJ;
        const int64_t Il0 = I0 - (int64_t)o * S.g.c0;
        // base point of the same class with coordinates >= 2: offsets of the affine class layout
        const int64_t bI = 2 * o + Il0 % o, bJ = 2 * o + J0 % o, bK = 2 * o + K0 % o;
        const int64_t gr = S.row0 + h_iperm[ls][lc], tile = gr / kRowsPerBlock, lane = gr % kRowsPerBlock;
        for (int64_t j = 0; j < nl; ++j) {
          const int64_t cc = cols[j];
          const int64_t I = S.g.I_lo + cc % S.g.nI, t = cc / S.g.nI, J = 1 + t % S.g.nJ, K = 1 + t / S.g.nJ;
          const int64_t d = internal_of(bI + (I - I0), bJ + (J - J0), bK + (K - K0)) - internal_of(bI, bJ, bK);
          delta.push_back((int32_t)d);
          src.push_back(h_soff[tile] + (int64_t)kRowsPerBlock * j + lane);
        }
        while (delta.size() % 4) {  // pad the table to whole groups of 4 with (0, +0.0)
          delta.push_back(0);
          src.push_back(-1);
        }
      }
      begin.push_back((int32_t)delta.size());
    }
  }
  c.mf_entries = (int64_t)delta.size();
  c.h_mf_begin = begin;
  c.h_mf_delta = delta;
  c.d_mf_sub = dupload(c, msub);
  c.d_mf_begin = dupload(c, begin);
  c.d_mf_delta = dupload(c, delta);
  c.d_mf_src = dupload(c, src);
  c.d_mf_val = dalloc<double>(std::max<int64_t>(4, c.mf_entries));
  c.mf_ok = true;
  mf_refresh(c);
}

static void assemble(Ctx& c) {
  free_assembly(c);
  const int o = c.mesh.order;
  const double h[3] = {c.mesh.lx / c.mesh.nx, c.mesh.ly / c.mesh.ny, c.mesh.lz / c.mesh.nz};
  c.tables = build_stencil_tables(o, h);
  c.d_col_begin = dupload(c, c.tables.col_begin);
  c.d_cols = dupload(c, c.tables.cols);
  c.d_contribs = dupload(c, c.tables.contribs);
  c.d_load_begin = dupload(c, c.tables.load_begin);
  c.d_loads = dupload(c, c.tables.loads);
  interface_mass(o, c.mesh.ny, c.mesh.nz, h[1], h[2], c.h_mrow, c.h_mcol, c.h_mval, c.h_sval);
  c.nG = (int64_t)c.h_mrow.size() - 1;
  c.d_mrow = dupload(c, c.h_mrow);
  c.d_mcol = dupload(c, c.h_mcol);
  c.d_mval = dupload(c, c.h_mval);
  c.d_sval = dupload(c, c.h_sval);
  if (!c.d_flags) c.d_flags = dalloc<int32_t>(4);
  OSM_CUDA(cudaMemsetAsync(c.d_flags, 0, 4 * sizeof(int32_t), c.stream));

  // --- per-subdomain structural CSR of K_s^N (contract order) and SELL layout
  const int nloc = c.s_end - c.s_begin;
  c.subs.resize(nloc);
  std::vector<std::vector<int32_t>> h_perm(nloc);
  std::vector<std::vector<int32_t>> h_iperm(nloc);
  std::vector<std::vector<int32_t>> h_len(nloc);
  std::vector<int64_t> h_soff;
  std::vector<int32_t> h_swidth;
  int64_t row0 = 0, slice0 = 0, sell_off = 0;
  for (int ls = 0; ls < nloc; ++ls) {
    Sub& S = c.subs[ls];
    S.s = c.s_begin + ls;
    S.g = slab_geom(c, S.s);
    S.n = S.g.nI * S.g.nJ * S.g.nK;
    if (S.n >= (int64_t)INT32_MAX) fail(OSM_ERR_INVALID_ARG, "subdomain too large for int32 local indices");
    int32_t* d_len = dalloc<int32_t>(S.n);
    launch_count(c, S, d_len);
    std::vector<int32_t> len(S.n);
    OSM_CUDA(cudaMemcpyAsync(len.data(), d_len, sizeof(int32_t) * S.n, cudaMemcpyDeviceToHost, c.stream));
    OSM_CUDA(cudaStreamSynchronize(c.stream));
    dfree(d_len);
    std::vector<int64_t> rowptr(S.n + 1, 0);
    for (int64_t i = 0; i < S.n; ++i) rowptr[i + 1] = rowptr[i] + len[i];
    S.nnz = rowptr[S.n];
    S.rowptr = dupload(c, rowptr);
    S.col = dalloc<int32_t>(S.nnz);
    S.val = dalloc<double>(S.nnz);
    launch_fill(c, S);

    // SELL-32-sigma: within windows of kSigma rows, sort rows by length (descending, stable)
    const bool mf_layout = c.sort_key == 4;
    const bool brick_layout = c.sort_key == 6;
    const int64_t mf_nIs = (int64_t)o * (S.g.c1 - S.g.c0) + 1;
    const int64_t mf_hI = (mf_nIs + o - 1) / o, mf_hJ = (S.g.Ny + o - 1) / o, mf_hK = (S.g.Nz + o - 1) / o;
    const int64_t mf_rows = (int64_t)o * o * o * mf_hI * mf_hJ * mf_hK;
    BrickSub bsub;
    if (brick_layout) brick_geometry(c, ls, bsub);
    S.npad = round_up(mf_layout ? mf_rows : (brick_layout ? bsub.nrows : S.n), kRowsPerBlock);
    if (S.npad >= (int64_t)INT32_MAX) fail(OSM_ERR_INVALID_ARG, "subdomain too large for int32 local indices");
    h_len[ls] = len;
    S.row0 = row0;
    S.slice0 = slice0;
    S.nslice = S.npad / kWarp;
    S.blk0 = row0 / kRowsPerBlock;
    S.nblk = S.npad / kRowsPerBlock;
    auto& perm = h_perm[ls];
    auto& iperm = h_iperm[ls];
    perm.assign(S.npad, -1);
    iperm.assign(S.n, -1);
    std::vector<int32_t> idx;
    // sigma: fixed by OSM_SIGMA, else the largest power of two (<= 32768) that keeps every column
    // offset col - row of the internal order within int16 (offset <= sigma + stencil reach), so
    // the value-indexed copy can use 16-bit offsets; 32768 when no such sigma >= 1024 exists.
    int64_t sigma = c.sigma;
    if (sigma <= 0) {
      const int64_t reach = 2 * S.g.nI * S.g.nJ + 2 * S.g.nI + 2;
      sigma = 32768;
      while (sigma > 1024 && sigma + reach > 32767) sigma /= 2;
      if (sigma + reach > 32767) sigma = 32768;
    }
    sigma = std::max<int64_t>(kRowsPerBlock, sigma);
    if (mf_layout) {  // class-major lattice layout of MfSub (dummy rows: perm -1)
      const int64_t hJK = mf_hJ * mf_hK, hIJK = mf_hI * hJK;
      for (int64_t li = 0; li < mf_rows; ++li) {
        const int64_t cc = li / hIJK, rem = li % hIJK, ii = rem / hJK, kk = (rem % hJK) / mf_hJ, jj = rem % mf_hJ;
        const int64_t I = o * ii + cc % o, J = o * jj + (cc / o) % o, K = o * kk + cc / (o * o);
        const int64_t Ig = (int64_t)o * S.g.c0 + I;
        if (I >= mf_nIs || Ig < S.g.I_lo || Ig > S.g.I_hi || J < 1 || J > S.g.Ny - 2 || K < 1 || K > S.g.Nz - 2)
          continue;
        const int64_t lc = (Ig - S.g.I_lo) + S.g.nI * ((J - 1) + S.g.nJ * (K - 1));
        perm[li] = (int32_t)lc;
        iperm[lc] = (int32_t)li;
      }
    }
    if (brick_layout) {  // one dense array per parity class (brick.cu); J pad rows: perm -1
      for (int64_t lc = 0; lc < S.n; ++lc) {
        const int64_t I = S.g.I_lo + lc % S.g.nI, t = lc / S.g.nI, J = 1 + t % S.g.nJ, K = 1 + t / S.g.nJ;
        const int cc = brick_class(o, (int)I, (int)J, (int)K);
        const BrickClass& C = bsub.cls[cc];
        const int64_t ii = I / o - S.g.I_lo / o, jj = J / o - 1 / o, kk = K / o - 1 / o;
        const int64_t li = C.base + (jj - C.jjlo) + (int64_t)C.nJp * ((ii - C.iilo) + (int64_t)C.nIc * (kk - C.kklo));
        perm[li] = (int32_t)lc;
        iperm[lc] = (int32_t)li;
      }
    }
    for (int64_t w0 = 0; w0 < (mf_layout || brick_layout ? 0 : S.n); w0 += sigma) {
      const int64_t w1 = std::min<int64_t>(S.n, w0 + sigma);
      idx.resize(w1 - w0);
      std::iota(idx.begin(), idx.end(), (int32_t)w0);
      if (c.sort_key == 0) {  // row length, descending (minimal SELL padding)
        std::stable_sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) { return len[a] > len[b]; });
      } else {  // lattice parity class (then length when sort_key >= 2): same-class rows in spatial order;
                // sort_key 3 also orders a class by (K, I, J) so warps run along the long y axis and
                // their gathers hit consecutive addresses of the neighbour class
        auto key = [&](int32_t i) {
          const int64_t I = S.g.I_lo + i % S.g.nI, t = i / S.g.nI, J = 1 + t % S.g.nJ, K = 1 + t / S.g.nJ;
          const int cls = (int)((I % 2) + 2 * (J % 2) + 4 * (K % 2));
          return std::make_tuple(cls, c.sort_key >= 2 ? -len[i] : 0, c.sort_key == 3 ? K : 0, c.sort_key == 3 ? I : 0,
                                 c.sort_key == 3 ? J : 0);
        };
        std::stable_sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) { return key(a) < key(b); });
      }
      for (int64_t k = 0; k < w1 - w0; ++k) {
        perm[w0 + k] = idx[k];
        iperm[idx[k]] = (int32_t)(w0 + k);
      }
    }
    S.sell_entries = 0;
    for (int64_t t = 0; t < S.nblk; ++t) {  // SELL-256 tiles = hot-path blocks
      int w = 0;
      for (int l = 0; l < kRowsPerBlock; ++l) {
        const int32_t cr = perm[t * kRowsPerBlock + l];
        if (cr >= 0) w = std::max(w, len[cr]);
      }
      h_soff.push_back(sell_off);
      h_swidth.push_back(w);
      sell_off += (int64_t)w * kRowsPerBlock;
      S.sell_entries += (int64_t)w * kRowsPerBlock;
    }
    S.perm = dupload(c, perm);
    S.iperm = dupload(c, iperm);
    row0 += S.npad;
    slice0 += S.nslice;
  }
  c.nrows_total = row0;
  c.nslices_total = slice0;
  c.nblk_total = row0 / kRowsPerBlock;
  c.sell_total = sell_off;
  if (c.nrows_total >= (int64_t)INT32_MAX) fail(OSM_ERR_INVALID_ARG, "too many rows per GPU for int32 columns");
  c.sell_soff = dupload(c, h_soff);
  c.sell_swidth = dupload(c, h_swidth);
  c.sell_val = dalloc<double>(c.sell_total);
  c.sell_col = dalloc<int32_t>(c.sell_total);
  c.x = dalloc<double>(c.nrows_total);
  c.r = dalloc<double>(c.nrows_total);
  c.p = dalloc<double>(c.nrows_total);
  c.q = dalloc<double>(c.nrows_total);
  c.dinv = dalloc<double>(c.nrows_total);
  c.b = dalloc<double>(c.nrows_total);
  c.ut = dalloc<double>(c.nrows_total);
  for (double* v : {c.x, c.r, c.p, c.q, c.dinv, c.b, c.ut})
    OSM_CUDA(cudaMemsetAsync(v, 0, sizeof(double) * c.nrows_total, c.stream));
  for (int ls = 0; ls < nloc; ++ls) launch_sell_build(c, c.subs[ls], nullptr);

  std::vector<int32_t> blk_sub(c.nblk_total);
  for (int ls = 0; ls < nloc; ++ls)
    for (int64_t k = 0; k < c.subs[ls].nblk; ++k) blk_sub[c.subs[ls].blk0 + k] = ls;
  c.blk_sub = dupload(c, blk_sub);
  // tiles per vector block: 4 (8 rows per thread) measured best even for one C3 slab per GPU
  // (tools/slab_probe.py: 23.9 / 24.5 / 26.5 us per PCG iteration with 4 / 2 / 1); OSM_VT overrides
  c.vec_tiles = c.vt_override > 0 ? std::min(kVecTiles, c.vt_override) : kVecTiles;
  {
    std::vector<int32_t> vs, vt, vn;
    for (int ls = 0; ls < nloc; ++ls) {
      Sub& S = c.subs[ls];
      for (int64_t t = 0; t < S.nblk; t += c.vec_tiles) {
        vs.push_back(ls);
        vt.push_back((int32_t)(S.blk0 + t));
        vn.push_back((int32_t)std::min<int64_t>(c.vec_tiles, S.nblk - t));
      }
    }
    c.nvblk_total = (int64_t)vs.size();
    c.vblk_sub = dupload(c, vs);
    c.vblk_tile0 = dupload(c, vt);
    c.vblk_ntile = dupload(c, vn);
  }

  // --- interface sides
  const int64_t nG = c.nG;
  std::vector<int32_t> islot(c.nrows_total, -1);
  for (int ls = 0; ls < nloc; ++ls) {
    const Sub& S = c.subs[ls];
    for (int64_t k = 0; k < S.npad; ++k)
      if (h_perm[ls][k] < 0) islot[S.row0 + k] = -2;
  }
  {
    int sb, se;
    std::vector<PlanSide> plan;
    plan_rank(c.nsub, c.nranks, c.rank, sb, se, plan);
    for (const PlanSide& ps : plan) {
      const int ls = ps.sub - c.s_begin;
      Sub& S = c.subs[ls];
      const int which_plane = ps.which == 1 ? 0 : 1;  // the right slab of an interface owns its left plane
      Side sd;
      sd.sub = ls;
      sd.iface = ps.iface;
      sd.which = ps.which;
      sd.remote = ps.remote != 0 || c.force_remote;
      sd.peer = c.force_remote ? c.rank : ps.peer;
      const int64_t I = which_plane == 0 ? (int64_t)o * S.g.c0 : (int64_t)o * S.g.c1;
      std::vector<int32_t> mc(nG), mg(nG);
      const int k = (int)c.sides.size();
      for (int64_t kk = 0; kk < S.g.nK; ++kk)
        for (int64_t jj = 0; jj < S.g.nJ; ++jj) {
          const int64_t gidx = jj + S.g.nJ * kk;
          const int64_t lc = (I - S.g.I_lo) + S.g.nI * (jj + S.g.nJ * kk);
          mc[gidx] = (int32_t)lc;
          mg[gidx] = (int32_t)(S.row0 + h_iperm[ls][lc]);
          islot[mg[gidx]] = (int32_t)(k * nG + gidx);
        }
      sd.map_c = dupload(c, mc);
      sd.map_g = dupload(c, mg);
      sd.out = dalloc<double>(3 * nG);
      OSM_CUDA(cudaMemsetAsync(sd.out, 0, sizeof(double) * 3 * nG, c.stream));
      if (sd.remote) {
        sd.inbuf = dalloc<double>(3 * nG);
        OSM_CUDA(cudaMemsetAsync(sd.inbuf, 0, sizeof(double) * 3 * nG, c.stream));
      }
      S.side[which_plane] = k;
      c.sides.push_back(sd);
    }
  }
  const int nsides = (int)c.sides.size();
  for (int k = 0; k < nsides; ++k) {
    Side& sd = c.sides[k];
    for (int j = 0; j < nsides; ++j)
      if (j != k && c.sides[j].iface == sd.iface) sd.partner = j;  // -1 when the neighbour is on another rank
  }
  c.islot = dupload(c, islot);
  c.lam_all = dalloc<double>(nsides * nG);
  c.unbr_all = dalloc<double>(nsides * nG);
  c.wif_all = dalloc<double>(nsides * nG);
  for (double* v : {c.lam_all, c.unbr_all, c.wif_all})
    OSM_CUDA(cudaMemsetAsync(v, 0, sizeof(double) * std::max<int64_t>(1, nsides * nG), c.stream));

  // --- Robin fold list: one entry per M_Gamma nonzero per side
  const int64_t mnnz = c.h_mrow.empty() ? 0 : c.h_mrow.back();
  c.nfold = nsides * mnnz;
  c.fold_pos = dalloc<int64_t>(c.nfold);
  c.fold_m = dalloc<double>(c.nfold);
  c.fold_s = dalloc<double>(c.nfold);
  c.fold_kn = dalloc<double>(c.nfold);
  c.fold_diag_row = dalloc<int32_t>(c.nfold);
  c.fold_side = dalloc<int32_t>(c.nfold);
  for (int k = 0; k < nsides; ++k) {
    c.sides[k].fold0 = k * mnnz;
    launch_fold_build(c, c.sides[k], c.subs[c.sides[k].sub]);
  }
  vi_build(c);  // value-indexed hot copy (from the unfolded K^N values)
  vi_sync_host_dict(c);
  if (c.sort_key == 4) mf_build(c, h_iperm, h_len, h_soff);

  // --- reductions and device side table
  c.part = dalloc<double>(3 * c.nblk_total);
  c.part_upd = dalloc<double>(2 * std::max<int64_t>(1, c.nvblk_total));
  c.side_nblk = std::max<int64_t>(1, ceil_div(nG, 256));
  c.side_part = dalloc<double>(std::max(1, nsides) * c.side_nblk);
  c.side_sum = dalloc<double>(std::max(1, nsides));
  c.side_cnt = dalloc<uint32_t>(std::max(1, nsides));
  OSM_CUDA(cudaMemsetAsync(c.side_cnt, 0, sizeof(uint32_t) * std::max(1, nsides), c.stream));
  OSM_CUDA(cudaMemsetAsync(c.side_sum, 0, sizeof(double) * std::max(1, nsides), c.stream));
  c.st = dalloc<SubState>(nloc);
  std::vector<SubState> hst(nloc);
  for (int ls = 0; ls < nloc; ++ls) {
    std::memset(&hst[ls], 0, sizeof(SubState));
    hst[ls].blk0 = c.subs[ls].blk0;
    hst[ls].nblk = (int32_t)c.subs[ls].nblk;
    int64_t v0 = 0;
    for (int j = 0; j < ls; ++j) v0 += ceil_div(c.subs[j].nblk, c.vec_tiles);
    hst[ls].vblk0 = v0;
    hst[ls].nvblk = (int32_t)ceil_div(c.subs[ls].nblk, c.vec_tiles);
    if (c.brick_ok) {
      hst[ls].brick0 = c.h_brick_sub[ls].brick0;
      hst[ls].nbrick = c.h_brick_sub[ls].nbrick;
    }
  }
  OSM_CUDA(cudaMemcpyAsync(c.st, hst.data(), sizeof(SubState) * nloc, cudaMemcpyHostToDevice, c.stream));
  // two subdomain groups for the two-stream PCG (halves of the local subdomains, in block order)
  c.ngroups = 1;
  while (c.ngroups * 2 <= std::min(c.want_groups, nloc)) c.ngroups *= 2;
  // with the tile SpMVs, groups only pay while a group's SpMV is a few waves (C3: ~1 wave); at C5 they
  // thrash L2.  The brick path (the default) gains from them at C5 too (33.3 s with 8 groups against
  // 34.2 s with one, tools/cg_bench.py, r02), so it keeps them.
  if (c.spmv_variant != 11) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
    const int64_t wave = 8LL * sms;  // SpMV blocks resident per wave
    while (c.ngroups > 1 && c.nblk_total / c.ngroups > 8 * wave && !c.groups_forced) c.ngroups /= 2;
  }
  for (int g = 0; g < c.ngroups; ++g) {  // group g = local subdomains [g nloc / G, (g + 1) nloc / G)
    const int s0 = g * nloc / c.ngroups, s1 = (g + 1) * nloc / c.ngroups;
    c.g_blk0[g] = c.subs[s0].blk0;
    c.g_nblk[g] = (s1 < nloc ? c.subs[s1].blk0 : c.nblk_total) - c.subs[s0].blk0;
    c.g_vb0[g] = hst[s0].vblk0;
    c.g_nvb[g] = (s1 < nloc ? hst[s1].vblk0 : c.nvblk_total) - hst[s0].vblk0;
  }
  if (c.h_st) cudaFreeHost(c.h_st);
  OSM_CUDA(cudaMallocHost((void**)&c.h_st, sizeof(SubState) * std::max(1, nloc)));
  if (c.h_side_sum) cudaFreeHost(c.h_side_sum);
  OSM_CUDA(cudaMallocHost((void**)&c.h_side_sum, sizeof(double) * std::max(1, nsides)));
  c.h_sides.assign(nsides, SideDev{});
  for (int k = 0; k < nsides; ++k) {
    const Side& sd = c.sides[k];
    SideDev& D = c.h_sides[k];
    D.map = sd.map_g;
    D.lam = c.lam_all + k * nG;
    D.out = sd.out;
    D.in = sd.remote ? sd.inbuf : c.sides[sd.partner].out;
    D.unbr = c.unbr_all + k * nG;
    D.wif = c.wif_all + k * nG;
    D.alpha_own = D.alpha_sum = 0.0;
    D.sub = sd.sub;
    D.which = sd.which;
    D.slot0 = (int32_t)(k * nG);
  }
  c.d_sides = dalloc<SideDev>(std::max(1, nsides));
  if (nsides)
    OSM_CUDA(cudaMemcpyAsync(c.d_sides, c.h_sides.data(), sizeof(SideDev) * nsides, cudaMemcpyHostToDevice, c.stream));

  int32_t flags[4];
  OSM_CUDA(cudaMemcpyAsync(flags, c.d_flags, sizeof(flags), cudaMemcpyDeviceToHost, c.stream));
  OSM_CUDA(cudaStreamSynchronize(c.stream));
  if (flags[1]) fail(OSM_ERR_INVALID_ARG, "internal: interface mass entry outside the stiffness pattern");
  if (flags[0]) fail(OSM_ERR_PRECOND, "non-positive diagonal entry in K_s^N");
  c.assembled = true;
  c.robin_dirty = true;
  c.density_set = false;
}

// Apply alpha to the SELL values of interface rows (K_s = K_s^N + alpha_s M_Gamma).
static void apply_robin(Ctx& c) {
  if (!c.robin_dirty) return;
  const int nsides = (int)c.sides.size();
  if (nsides == 0) {
    dcode_build(c);
    c.robin_dirty = false;
    return;
  }
  if (!c.robin_set) fail(OSM_ERR_STATE, "osm_set_robin must be called before solving with nsub > 1");
  std::vector<double> a(nsides), qv(nsides);
  for (int k = 0; k < nsides; ++k) {
    const Side& sd = c.sides[k];
    const double al = c.alpha_left[sd.iface], ar = c.alpha_right[sd.iface];
    const double ql = c.q_left[sd.iface], qr = c.q_right[sd.iface];
    a[k] = sd.which == 0 ? al : ar;
    qv[k] = sd.which == 0 ? ql : qr;
    c.h_sides[k].alpha_own = a[k];
    c.h_sides[k].alpha_sum = al + ar;
    c.h_sides[k].q_own = qv[k];
    c.h_sides[k].q_sum = ql + qr;
  }
  double* d_a = dupload(c, a);
  double* d_q = dupload(c, qv);
  OSM_CUDA(cudaMemsetAsync(c.d_flags, 0, 4 * sizeof(int32_t), c.stream));
  launch_fold_apply(c, d_a, d_q);
  if (c.mf_ok) mf_refresh(c);
  OSM_CUDA(cudaMemcpyAsync(c.d_sides, c.h_sides.data(), sizeof(SideDev) * nsides, cudaMemcpyHostToDevice, c.stream));
  int32_t flags[4];
  OSM_CUDA(cudaMemcpyAsync(flags, c.d_flags, sizeof(flags), cudaMemcpyDeviceToHost, c.stream));
  OSM_CUDA(cudaStreamSynchronize(c.stream));
  dfree(d_a);
  dfree(d_q);
  vi_apply_robin(c, a, qv);
  vi_sync_host_dict(c);
  dcode_build(c);
  if (flags[0]) fail(OSM_ERR_PRECOND, "non-positive diagonal entry after the Robin term");
  c.robin_dirty = false;
}

// ------------------------------------------------------------------ exchange
// part 1: [g | u] both directions for every remote side; part 2: the right slab's
// interface-row residual w to the owner (left slab).
static void exchange(Ctx& c, int part) {
  if (!c.tp) return;
  bool any = false;
  for (const Side& sd : c.sides) any = any || sd.remote;
  if (!any && !c.hub) return;  // (hub ranks always meet at the exchange barriers)
  timer_begin(c, T_OUTER_MISC);  // trace exchange, timed on the library stream
  c.tp->exchange(c, part);
  timer_end(c, T_OUTER_MISC);
  for (const Side& sd : c.sides)  // bytes this rank sends (traffic[7])
    if (sd.remote && (part == 1 || sd.which == 1)) c.exch_bytes += (part == 1 ? 16.0 : 8.0) * c.nG;
}

// Per-subdomain values (local, in subdomain order) -> all nsub values on every rank.
static std::vector<double> allgather_sub(Ctx& c, const std::vector<double>& local, int width) {
  if (!c.tp) return local;
  return c.tp->allgather_host(c, local, width);
}

// Glued residual pipeline: sum over global free rows of (f - K u~)^2,
// each interface row counted once (owned by the left slab).  zero = 1 gives ||f||^2.
static double glued_residual2(Ctx& c, int zero, std::vector<int32_t>* iters_out) {
  launch_glue(c, zero);
  launch_resid(c);
  launch_iface_w(c);
  exchange(c, 2);
  launch_iface_sum(c);
  const int nloc = c.s_end - c.s_begin;
  const int nsides = (int)c.sides.size();
  OSM_CUDA(cudaMemcpyAsync(c.h_st, c.st, sizeof(SubState) * nloc, cudaMemcpyDeviceToHost, c.stream));
  if (nsides)
    OSM_CUDA(cudaMemcpyAsync(c.h_side_sum, c.side_sum, sizeof(double) * nsides, cudaMemcpyDeviceToHost, c.stream));
  OSM_CUDA(cudaStreamSynchronize(c.stream));
  std::vector<double> loc(2 * nloc);
  for (int ls = 0; ls < nloc; ++ls) {
    double v = c.h_st[ls].resid;
    const int k = c.subs[ls].side[1];
    if (k >= 0) v += c.h_side_sum[k];
    loc[2 * ls] = v;
    loc[2 * ls + 1] = (double)c.h_st[ls].iters + 1e6 * (c.h_st[ls].status == 2);
  }
  std::vector<double> all = allgather_sub(c, loc, 2);
  double tot = 0.0;
  for (int s = 0; s < c.nsub; ++s) tot += all[2 * s];
  if (iters_out) {
    iters_out->resize(c.nsub);
    for (int s = 0; s < c.nsub; ++s) (*iters_out)[s] = (int32_t)all[2 * s + 1];
  }
  return tot;
}

double fnorm2_of(Ctx& c) { return glued_residual2(c, 1, nullptr); }

// ------------------------------------------------------------------ solve
static constexpr int kCgChunk = 8;  // PCG iterations per enqueued chunk

// One chunk of kCgChunk batched PCG iterations: replayed from a CUDA graph (kernels
// chained by programmatic dependent launch) unless per-launch timing is on.
// One chunk of kCgChunk PCG iterations of group g on its stream, from a captured graph.
static void enqueue_group_chunk(Ctx& c, int g, double tol, int maxit) {
  if (!c.cg_graph_g[g] || c.graph_tol != tol || c.graph_maxit != maxit) {
    if (c.cg_graph_g[g]) cudaGraphExecDestroy(c.cg_graph_g[g]);
    c.cg_graph_g[g] = nullptr;
    const int64_t l0 = c.launches;
    cudaGraph_t gr = nullptr;
    c.grp_cur = g;
    OSM_CUDA(cudaStreamBeginCapture(c.gstream[g], cudaStreamCaptureModeThreadLocal));
    try {
      c.cg_par = 0;
      for (int it = 0; it < kCgChunk; ++it) {
        launch_cg_spmv(c);
        launch_cg_update(c, tol, maxit);
        launch_cg_dir(c);
      }
    } catch (...) {
      c.grp_cur = -1;
      cudaStreamEndCapture(c.gstream[g], &gr);
      if (gr) cudaGraphDestroy(gr);
      throw;
    }
    c.grp_cur = -1;
    OSM_CUDA(cudaStreamEndCapture(c.gstream[g], &gr));
    const cudaError_t e = cudaGraphInstantiate(&c.cg_graph_g[g], gr, 0);
    cudaGraphDestroy(gr);
    c.cg_graph_launches_g[g] = c.launches - l0;
    c.launches = l0;
    if (e != cudaSuccess) fail(OSM_ERR_CUDA, "graph instantiation failed");
  }
  OSM_CUDA(cudaGraphLaunch(c.cg_graph_g[g], c.gstream[g]));
  c.launches += c.cg_graph_launches_g[g];
}

static bool group_streams(const Ctx& c) { return c.ngroups > 1 && !c.timing && c.use_graph; }

static void enqueue_cg_chunk(Ctx& c, double tol, int maxit) {
  if (group_streams(c)) {
    for (int g = 0; g < c.ngroups; ++g) enqueue_group_chunk(c, g, tol, maxit);
    c.graph_tol = tol;
    c.graph_maxit = maxit;
    return;
  }
  if (c.timing || !c.use_graph) {
    c.cg_par = 0;
    for (int it = 0; it < kCgChunk; ++it) {
      launch_cg_spmv(c);
      launch_cg_update(c, tol, maxit);
      launch_cg_dir(c);
    }
    return;
  }
  if (!c.cg_graph || c.graph_tol != tol || c.graph_maxit != maxit) {
    drop_graph(c);
    const int64_t l0 = c.launches;
    cudaGraph_t g = nullptr;
    OSM_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
    try {
      c.cg_par = 0;
      for (int it = 0; it < kCgChunk; ++it) {
        launch_cg_spmv(c);
        launch_cg_update(c, tol, maxit);
        launch_cg_dir(c);
      }
    } catch (...) {
      cudaStreamEndCapture(c.stream, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    OSM_CUDA(cudaStreamEndCapture(c.stream, &g));
    const cudaError_t e = cudaGraphInstantiate(&c.cg_graph, g, 0);
    cudaGraphDestroy(g);
    c.cg_graph_launches = c.launches - l0;
    c.launches = l0;
    if (e != cudaSuccess) {  // graphs unavailable: plain stream launches (same kernels)
      cudaGetLastError();
      c.cg_graph = nullptr;
      c.use_graph = false;
      enqueue_cg_chunk(c, tol, maxit);
      return;
    }
    c.graph_tol = tol;
    c.graph_maxit = maxit;
  }
  OSM_CUDA(cudaGraphLaunch(c.cg_graph, c.stream));
  c.launches += c.cg_graph_launches;
}

static osm_status solve(Ctx& c, const osm_solve_opts& o, osm_report* rep) {
  NvtxRange nv_solve("osm_solve");
  if (!c.assembled) fail(OSM_ERR_STATE, "osm_assemble must precede osm_solve");
  if (!c.density_set) fail(OSM_ERR_STATE, "osm_upload_density must precede osm_solve");
  if (o.max_outer < 1 || o.max_inner < 1 || !(o.tol_outer > 0) || !(o.tol_inner > 0))
    fail(OSM_ERR_INVALID_ARG, "bad solve options");
  const auto t0 = std::chrono::steady_clock::now();
  apply_robin(c);
  const int64_t nGs = (int64_t)c.sides.size() * c.nG;
  c.fnorm2 = glued_residual2(c, 1, nullptr);
  const double fnorm = std::sqrt(c.fnorm2);
  OSM_CUDA(cudaMemsetAsync(c.x, 0, sizeof(double) * c.nrows_total, c.stream));
  if (nGs) {
    OSM_CUDA(cudaMemsetAsync(c.lam_all, 0, sizeof(double) * nGs, c.stream));
    OSM_CUDA(cudaMemsetAsync(c.unbr_all, 0, sizeof(double) * nGs, c.stream));
  }
  c.hist.clear();
  c.exch_bytes = 0;
  c.inner.clear();
  int status = OSM_NOT_CONVERGED;
  int grow = 0;
  int64_t inner_total = 0;
  int inner_maxed = 0;
  for (int n = 1; n <= o.max_outer; ++n) {
    NvtxRange nv_outer("schwarz_iteration");
    if (!o.warm_start) OSM_CUDA(cudaMemsetAsync(c.x, 0, sizeof(double) * c.nrows_total, c.stream));
    OSM_CUDA(cudaMemsetAsync(c.d_nactive, 0, sizeof(int32_t), c.stream));
    launch_warm(c, o.tol_inner, o.warm_start);
    launch_zero_if(c);
    OSM_CUDA(cudaMemcpyAsync(&c.h_nactive[0], c.d_nactive, sizeof(int32_t), cudaMemcpyDeviceToHost, c.stream));
    OSM_CUDA(cudaStreamSynchronize(c.stream));
    if (c.h_nactive[0] > 0) {
      NvtxRange nv_pcg("batched_pcg");
      // batched masked PCG: enqueue chunks; poll the active count one chunk behind.  With subdomain
      // groups, the group streams fork from the library stream; group 0's stream joins the others
      // after every chunk (the active count covers all) and the library stream joins at the end.
      const bool grp = group_streams(c);
      cudaStream_t ps = c.stream;
      if (grp) {
        OSM_CUDA(cudaEventRecord(c.ev_fork, c.stream));
        for (int g = 0; g < c.ngroups; ++g) OSM_CUDA(cudaStreamWaitEvent(c.gstream[g], c.ev_fork, 0));
        ps = c.gstream[0];
      }
      int ch = 0;
      for (;; ++ch) {
        enqueue_cg_chunk(c, o.tol_inner, o.max_inner);
        for (int g = 1; grp && g < c.ngroups; ++g) {
          OSM_CUDA(cudaEventRecord(c.ev_join[g], c.gstream[g]));
          OSM_CUDA(cudaStreamWaitEvent(ps, c.ev_join[g], 0));
        }
        OSM_CUDA(cudaMemcpyAsync(&c.h_nactive[ch & 1], c.d_nactive, sizeof(int32_t), cudaMemcpyDeviceToHost, ps));
        OSM_CUDA(cudaEventRecord(c.ev_chunk[ch & 1], ps));
        if (ch > 0) {
          OSM_CUDA(cudaEventSynchronize(c.ev_chunk[(ch - 1) & 1]));
          if (c.h_nactive[(ch - 1) & 1] == 0) break;
        }
        if ((int64_t)ch * kCgChunk > (int64_t)o.max_inner + 2 * kCgChunk) break;  // safety net
      }
      if (grp) OSM_CUDA(cudaStreamWaitEvent(c.stream, c.ev_chunk[ch & 1], 0));
      launch_cg_dir_flush(c);  // fused path: an x update still owed after the last SpMV
    }
    {
      NvtxRange nv_x("trace_exchange");
      launch_trace(c);
      exchange(c, 1);
      launch_accept(c);
    }
    NvtxRange nv_r("glued_residual");
    std::vector<int32_t> its;
    const double r2 = glued_residual2(c, 0, &its);
    const double h = fnorm > 0 ? std::sqrt(r2) / fnorm : std::sqrt(r2);
    c.hist.push_back(h);
    for (int s = 0; s < c.nsub; ++s) {
      int32_t k = its[s];
      if (k >= 1000000) {
        ++inner_maxed;
        k -= 1000000;
      }
      c.inner.push_back((s >= c.s_begin && s < c.s_end) ? k : -1);
      inner_total += k;
    }
    if (c.hist.size() >= 2 && c.hist[c.hist.size() - 1] > c.hist[c.hist.size() - 2]) ++grow; else grow = 0;
    if (!std::isfinite(h)) {
      status = OSM_ERR_DIVERGED;
      break;
    }
    if (h <= o.tol_outer) {
      status = OSM_OK;
      break;
    }
    if (o.diverge_window > 0 && grow >= o.diverge_window) {
      status = OSM_ERR_DIVERGED;
      break;
    }
  }
  timers_collect(c);
  // traffic model: algorithmic bytes per CG iteration per subdomain x its iterations
  for (double& t : c.traffic) t = 0;
  c.traffic[7] = c.exch_bytes;
  const int nloc = c.s_end - c.s_begin;
  const int sv = spmv_variant_of(c);
  const bool vi = sv == 3 || sv == 6 || sv == 7 || sv == 10, mf = sv == 5, br = sv == 11;
  for (int ls = 0; ls < nloc; ++ls) {
    const Sub& S = c.subs[ls];
    int64_t its = 0;
    for (size_t k = S.s; k < c.inner.size(); k += c.nsub) its += std::max(0, c.inner[k]);
    // SpMV bytes in the format launched: fp64 SELL 12 B/entry (+ CSR-equivalent 4 B/row),
    // value-indexed 4 B/entry (index + offset; the dictionary is on chip), or matrix-free 0 B/entry
    // (tables in the constant bank); vectors p, q 16 B/row
    const double kept = ls < (int)c.vi_kept.size() ? (double)c.vi_kept[ls] : (double)S.nnz;
    // (variant 5 reads a 1-byte table code per row)
    // (variant 11: its u8 index stream, 1 byte per (class-box point, slot), padding included; with
    // the Kuhn kernel the per-lane words of the non-uniform chunks and one descriptor per chunk)
    const double mat = mf ? (c.d_mf_code ? (double)S.npad : 0.0)
                     : br ? (c.brick_kernel > 0
                                 // Kuhn kernel: compact per-lane words + one descriptor per chunk (the
                                 // row-type table is a few KB, cached)
                                 ? 4.0 * (double)c.h_brick_sub_cwords[ls] +
                                       4.0 * 8.0 * c.h_brick_arg.BI * (double)c.h_brick_sub[ls].nbrick
                                 : 4.0 * (double)c.h_brick_arg.brick_words * (double)c.h_brick_sub[ls].nbrick)
                          : (vi ? (sv == 10 ? 3.0 : 4.0) * kept : 12.0 * S.nnz + 4.0 * (S.n + 1));
    c.traffic[0] += (double)its * (mat + 16.0 * S.n);
    c.traffic[6] += (double)its * (12.0 * S.nnz + 4.0 * (S.n + 1) + 16.0 * S.n);  // CSR-equivalent
    // D^-1 as an 8-byte stream, or as a 1-byte code (table codes of variant 5, dcode_build otherwise)
    const bool coded = mf ? c.d_mf_code != nullptr : !c.h_dcode_tab.empty();
    const double db = coded ? 1.0 : 8.0;
    c.traffic[1] += (double)its * (24.0 + db) * S.n;  // update: read r, q, D^-1; write r
    if (fused_dir(c))  // the SpMV reads r, D^-1 (codes) and x, writes x and p_{k+1}
      c.traffic[0] += (double)its * (32.0 + db) * S.n;
    else
      c.traffic[2] += (double)its * (40.0 + db) * S.n;  // direction: read r, D^-1, p, x; write p, x
    c.traffic[3] += (double)(S.sell_entries - S.nnz);
    c.traffic[4] += (double)S.nnz;
    c.traffic[5] += (double)S.n;
  }
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (rep) {
    rep->outer_iters = (int)c.hist.size();
    rep->converged = status == OSM_OK;
    rep->h_final = c.hist.empty() ? 0.0 : c.hist.back();
    rep->seconds = secs;
    rep->inner_total = inner_total;
    rep->inner_maxed = inner_maxed;
  }
  return (osm_status)status;
}

}  // namespace osm

// ================================================================== C ABI
using namespace osm;

struct osm_ctx {
  Ctx c;
};

#define OSM_API_BEGIN try {
#define OSM_API_END                                 \
  }                                                 \
  catch (const Error& e) {                          \
    g_last_error = e.what();                        \
    hub_poison_current();                           \
    return e.status;                                \
  }                                                 \
  catch (const std::exception& e) {                 \
    g_last_error = e.what();                        \
    hub_poison_current();                           \
    return OSM_ERR_CUDA;                            \
  }                                                 \
  catch (...) {                                     \
    g_last_error = "unknown error";                 \
    hub_poison_current();                           \
    return OSM_ERR_CUDA;                            \
  }

static Ctx& ctx_of(osm_ctx* c) {
  hub_set_current(nullptr);  // set again by the collective calls (solve, solution, gravity)
  if (!c) fail(OSM_ERR_INVALID_ARG, "NULL context");
  OSM_CUDA(cudaSetDevice(c->c.device));
  return c->c;
}

extern "C" {

int osm_abi_version(void) { return OSM_ABI_VERSION; }

const char* osm_last_error(void) { return g_last_error.c_str(); }

osm_status osm_nccl_unique_id(void* uid128) {
  OSM_API_BEGIN
  if (!uid128) fail(OSM_ERR_INVALID_ARG, "NULL uid buffer");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  OSM_NCCL(ncclGetUniqueId(&id));
  std::memcpy(uid128, &id, sizeof(id));
  return OSM_OK;
  OSM_API_END
}

osm_status osm_create(const osm_mesh_desc* mesh, const osm_dist_desc* dist, osm_ctx** out) {
  OSM_API_BEGIN
  if (!mesh || !out) fail(OSM_ERR_INVALID_ARG, "NULL argument");
  *out = nullptr;
  const osm_mesh_desc& m = *mesh;
  if (m.nx <= 0 || m.ny <= 0 || m.nz <= 0 || !(m.lx > 0) || !(m.ly > 0) || !(m.lz > 0))
    fail(OSM_ERR_INVALID_ARG, "cell counts and extents must be positive");
  if (m.order != 1 && m.order != 2) fail(OSM_ERR_INVALID_ARG, "order must be 1 or 2");
  if (m.order * m.nx + 1 < 3 || m.order * m.ny + 1 < 3 || m.order * m.nz + 1 < 3)
    fail(OSM_ERR_GRID_TOO_SMALL, "fewer than 3 lattice points on an axis: no interior");
  osm_dist_desc d{0, 1, 0, nullptr, nullptr, nullptr};
  if (dist) d = *dist;
  if (d.nranks < 1 || d.rank < 0 || d.rank >= d.nranks) fail(OSM_ERR_INVALID_ARG, "bad rank/nranks");
  if (d.nranks > 1 && !d.nccl_uid && !d.hub) fail(OSM_ERR_INVALID_ARG, "nccl_uid or hub required when nranks > 1");
  if (d.nccl_uid && d.hub) fail(OSM_ERR_INVALID_ARG, "nccl_uid and hub are exclusive");
  auto* h = new osm_ctx();
  Ctx& c = h->c;
  try {
    c.mesh = m;
    c.rank = d.rank;
    c.nranks = d.nranks;
    c.device = d.device;
    OSM_CUDA(cudaSetDevice(c.device));
    if (d.stream) {
      c.stream = (cudaStream_t)d.stream;
    } else {
      OSM_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
      c.own_stream = true;
    }
    OSM_CUDA(cudaMallocHost((void**)&c.h_nactive, 2 * sizeof(int32_t)));
    c.d_nactive = dalloc<int32_t>(1);
    OSM_CUDA(cudaEventCreateWithFlags(&c.ev_chunk[0], cudaEventDisableTiming));
    OSM_CUDA(cudaEventCreateWithFlags(&c.ev_chunk[1], cudaEventDisableTiming));
    OSM_CUDA(cudaEventCreateWithFlags(&c.ev_fork, cudaEventDisableTiming));
    for (auto& e : c.ev_join) OSM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& gs : c.gstream) OSM_CUDA(cudaStreamCreateWithFlags(&gs, cudaStreamNonBlocking));
    if (const char* e = std::getenv("OSM_GROUPS")) {
      c.want_groups = std::max(1, std::atoi(e));
      c.groups_forced = true;
    }
    if (const char* e = std::getenv("OSM_VT")) c.vt_override = std::atoi(e);
    if (const char* e = std::getenv("OSM_SIGMA")) c.sigma = std::atoi(e);
    if (const char* e = std::getenv("OSM_NO_GRAPH")) c.use_graph = std::atoi(e) == 0;
    if (const char* e = std::getenv("OSM_SPMV")) c.spmv_variant = std::atoi(e);
    if (const char* e = std::getenv("OSM_UPD")) c.update_variant = std::atoi(e);
    if (const char* e = std::getenv("OSM_SPLIT_UPD")) c.split_update = std::atoi(e) != 0;
    if (const char* e = std::getenv("OSM_SORT")) c.sort_key = std::atoi(e);
    if (const char* e = std::getenv("OSM_DCODE")) c.dcode_on = std::atoi(e) != 0;
    if (const char* e = std::getenv("OSM_FUSE_DIR")) c.fuse_dir = std::atoi(e) != 0;
    c.timers.resize(T_COUNT);
    const char* names[T_COUNT] = {"cg_spmv", "cg_update", "cg_dir", "warm_spmv", "resid_spmv", "exchange"};
    for (int i = 0; i < T_COUNT; ++i) c.timers[i].name = names[i];
    if (const char* e = std::getenv("OSM_FORCE_REMOTE")) c.force_remote = std::atoi(e) != 0 && c.nranks == 1;
    if (d.hub) {
      c.hub = d.hub;
      c.tp = make_hub_transport(c, d.hub);
    } else if (c.nranks > 1) {
      c.tp = make_nccl_transport(c, d.nccl_uid, false);
    } else if (c.force_remote) {  // debug: a 1-rank communicator so the NCCL path runs on one GPU
      c.tp = make_nccl_transport(c, nullptr, true);
    }
  } catch (...) {
    osm_destroy(h);
    throw;
  }
  *out = h;
  return OSM_OK;
  OSM_API_END
}

void osm_destroy(osm_ctx* h) {
  if (!h) return;
  Ctx& c = h->c;
  cudaSetDevice(c.device);
  if (c.stream) cudaStreamSynchronize(c.stream);
  try {
    free_assembly(c);
  } catch (...) {
  }
  dfree(c.drho);
  dfree(c.d_gz);
  dfree(c.d_nactive);
  dfree(c.d_flags);
  if (c.h_nactive) cudaFreeHost(c.h_nactive);
  if (c.h_st) cudaFreeHost(c.h_st);
  if (c.h_side_sum) cudaFreeHost(c.h_side_sum);
  for (auto& e : c.ev_chunk)
    if (e) cudaEventDestroy(e);
  if (c.ev_fork) cudaEventDestroy(c.ev_fork);
  for (auto& e : c.ev_join)
    if (e) cudaEventDestroy(e);
  for (auto& gs : c.gstream)
    if (gs) cudaStreamDestroy(gs);
  for (auto& t : c.timers)
    for (auto& e : t.ev) cudaEventDestroy(e);
  delete c.tp;
  c.tp = nullptr;
  if (c.own_stream && c.stream) cudaStreamDestroy(c.stream);
  delete h;
}

osm_status osm_decompose(osm_ctx* h, int nsub) {
  OSM_API_BEGIN
  Ctx& c = ctx_of(h);
  if (nsub < 1 || nsub > c.mesh.nx || nsub % c.nranks != 0)
    fail(OSM_ERR_INVALID_ARG, "need 1 <= nsub <= nx and nsub % nranks == 0");
  free_assembly(c);
  c.nsub = nsub;
  c.cstart = partition_x(c.mesh.nx, nsub);
  {
    std::vector<PlanSide> plan;
    plan_rank(nsub, c.nranks, c.rank, c.s_begin, c.s_end, plan);
  }
  c.robin_set = nsub == 1;
  c.alpha_left.assign(nsub > 1 ? nsub - 1 : 0, 0.0);
  c.alpha_right.assign(nsub > 1 ? nsub - 1 : 0, 0.0);
  c.q_left.assign(nsub > 1 ? nsub - 1 : 0, 0.0);
  c.q_right.assign(nsub > 1 ? nsub - 1 : 0, 0.0);
  return OSM_OK;
  OSM_API_END
}

static void set_robin(Ctx& c, const double* al, const double* ql, const double* ar, const double* qr) {
  if (c.nsub < 1) fail(OSM_ERR_STATE, "osm_decompose must precede osm_set_robin");
  const int ni = c.nsub - 1;
  if (ni > 0 && (!al || !ar)) fail(OSM_ERR_INVALID_ARG, "NULL alpha array");
  for (int i = 0; i < ni; ++i) {
    const double pl = al[i], pr = ar[i], l = ql ? ql[i] : 0.0, r = qr ? qr[i] : 0.0;
    for (double v : {pl, pr, l, r})
      if (!(v >= 0) || !std::isfinite(v)) fail(OSM_ERR_ILL_POSED, "Robin coefficients must be finite and >= 0");
    if (pl == 0 && pr == 0 && l == 0 && r == 0) fail(OSM_ERR_ILL_POSED, "zero transmission on both sides of an interface");
    if (pl == 0 && pr == 0) fail(OSM_ERR_ILL_POSED, "p = 0 on both sides of an interface");
  }
  c.alpha_left.assign(al, al + ni);
  c.alpha_right.assign(ar, ar + ni);
  c.q_left.assign(ni, 0.0);
  c.q_right.assign(ni, 0.0);
  if (ql) c.q_left.assign(ql, ql + ni);
  if (qr) c.q_right.assign(qr, qr + ni);
  c.robin_set = true;
  c.robin_dirty = true;
}

osm_status osm_set_robin(osm_ctx* h, const double* al, const double* ar) {
  OSM_API_BEGIN
  set_robin(ctx_of(h), al, nullptr, ar, nullptr);
  return OSM_OK;
  OSM_API_END
}

osm_status osm_set_robin2(osm_ctx* h, const double* pl, const double* ql, const double* pr, const double* qr) {
  OSM_API_BEGIN
  if (!ql || !qr) fail(OSM_ERR_INVALID_ARG, "NULL q array");
  set_robin(ctx_of(h), pl, ql, pr, qr);
  return OSM_OK;
  OSM_API_END
}

osm_status osm_assemble(osm_ctx* h) {
  OSM_API_BEGIN
  Ctx& c = ctx_of(h);
  if (c.nsub < 1) fail(OSM_ERR_STATE, "osm_decompose must precede osm_assemble");
  assemble(c);
  return OSM_OK;
  OSM_API_END
}

static void upload_density(Ctx& c, const double* drho, bool device, double G) {
  if (!c.assembled) fail(OSM_ERR_STATE, "osm_assemble must precede osm_upload_density");
  if (!drho) fail(OSM_ERR_INVALID_ARG, "NULL density");
  if (!std::isfinite(G)) fail(OSM_ERR_INVALID_ARG, "G must be finite");
  const int64_t ncell = c.mesh.nx * c.mesh.ny * c.mesh.nz;
  if (!c.drho) c.drho = dalloc<double>(ncell);
  OSM_CUDA(cudaMemcpyAsync(c.drho, drho, sizeof(double) * ncell,
                           device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c.stream));
  c.G = G;
  const double fourpiG = 4.0 * M_PI * G;
  for (const Sub& S : c.subs) launch_load(c, S, fourpiG);
  if (!device) OSM_CUDA(cudaStreamSynchronize(c.stream));  // the caller may free its host buffer
  c.density_set = true;
}

osm_status osm_upload_load_vector(osm_ctx* h, const double* b_free, int64_t n) {
  OSM_API_BEGIN
  Ctx& c = ctx_of(h);
  if (!c.assembled) fail(OSM_ERR_STATE, "osm_assemble must precede osm_upload_load_vector");
  const int o = c.mesh.order;
  const int64_t N = (o * c.mesh.nx - 1) * (o * c.mesh.ny - 1) * (o * c.mesh.nz - 1);
  if (!b_free || n != N) fail(OSM_ERR_INVALID_ARG, "load vector must hold the global free DOFs");
  double* d = dalloc<double>(N);
  OSM_CUDA(cudaMemcpyAsync(d, b_free, sizeof(double) * N, cudaMemcpyHostToDevice, c.stream));
  for (const Sub& S : c.subs) launch_load_free(c, S, d);
  OSM_CUDA(cudaStreamSynchronize(c.stream));
  dfree(d);
  c.density_set = true;
  return OSM_OK;
  OSM_API_END
}

osm_status osm_upload_density(osm_ctx* h, const double* drho, double G) {
  OSM_API_BEGIN
  upload_density(ctx_of(h), drho, false, G);
  return OSM_OK;
  OSM_API_END
}

osm_status osm_upload_density_device(osm_ctx* h, const double* drho, double G) {
  OSM_API_BEGIN
  upload_density(ctx_of(h), drho, true, G);
  return OSM_OK;
  OSM_API_END
}

osm_status osm_solve(osm_ctx* h, const osm_solve_opts* o, osm_report* rep) {
  OSM_API_BEGIN
  Ctx& c = ctx_of(h);
  hub_set_current(c.hub);  // [collective]: a failure here releases the other hub ranks
  if (!o) fail(OSM_ERR_INVALID_ARG, "NULL options");
  return solve(c, *o, rep);
  OSM_API_END
}

osm_status osm_get_history(osm_ctx* h, double* out, int cap, int* n) {
  OSM_API_BEGIN
  Ctx& c = ctx_of(h);
  if (!n) fail(OSM_ERR_INVALID_ARG, "NULL size");
  *n = (int)c.hist.size();
  if (out) std::copy(c.hist.begin(), c.hist.begin() + std::min<int>(cap, (int)c.hist.size()), out);
  return OSM_OK;
  OSM_API_END
}

osm_status osm_get_inner_iters(osm_ctx* h, int32_t* its, int cap_outer, int* n_outer) {
  OSM_API_BEGIN
  Ctx& c = ctx_of(h);
  if (!n_outer) fail(OSM_ERR_INVALID_ARG, "NULL size");
  *n_outer = (int)c.hist.size();
  if (its) {
    const size_t m = std::min<size_t>((size_t)cap_outer * c.nsub, c.inner.size());
    std::copy(c.inner.begin(), c.inner.begin() + m, its);
  }
  return OSM_OK;
  OSM_API_END
}

// Glued Phi of the last solve on the full lattice into c.phi (on rank 0 after the reduce).
static void gather_phi(Ctx& c, int64_t N) {
  if (!c.assembled) fail(OSM_ERR_STATE, "nothing solved");
  if (!c.phi) c.phi = dalloc<double>(N);
  OSM_CUDA(cudaMemsetAsync(c.phi, 0, sizeof(double) * N, c.stream));
  for (const Sub& S : c.subs) launch_scatter_phi(c, S, c.nranks > 1 ? 1 : 0);
  if (c.nranks > 1) c.tp->reduce_phi(c, c.phi, N);
}

osm_status osm_get_solution(osm_ctx* h, double* phi, int64_t* n) {
  OSM_API_BEGIN
  Ctx& c = ctx_of(h);
  hub_set_current(c.hub);  // [collective]: a failure here releases the other hub ranks
  if (!n) fail(OSM_ERR_INVALID_ARG, "NULL size");
  const int o = c.mesh.order;
  const int64_t N = (o * c.mesh.nx + 1) * (o * c.mesh.ny + 1) * (o * c.mesh.nz + 1);
  if (!phi && c.rank == 0) {
    *n = N;
    return OSM_OK;
  }
  if (c.rank == 0 && *n < N) fail(OSM_ERR_INVALID_ARG, "solution buffer too small");
  gather_phi(c, N);
  if (c.rank == 0 && phi)
    OSM_CUDA(cudaMemcpyAsync(phi, c.phi, sizeof(double) * N, cudaMemcpyDeviceToHost, c.stream));
  OSM_CUDA(cudaStreamSynchronize(c.stream));
  *n = N;
  return OSM_OK;
  OSM_API_END
}

osm_status osm_gravity_z(osm_ctx* h, double z0, double* gz, int64_t* n) {
  OSM_API_BEGIN
  Ctx& c = ctx_of(h);
  hub_set_current(c.hub);  // [collective]: a failure here releases the other hub ranks
  if (!n) fail(OSM_ERR_INVALID_ARG, "NULL size");
  const int64_t M = c.mesh.nx * c.mesh.ny;
  if (!gz && c.rank == 0) {
    *n = M;
    return OSM_OK;
  }
  if (!(z0 >= 0) || !(z0 <= c.mesh.lz)) fail(OSM_ERR_INVALID_ARG, "z0 outside [0, lz]");
  if (c.rank == 0 && *n < M) fail(OSM_ERR_INVALID_ARG, "buffer too small");
  const int o = c.mesh.order;
  const int64_t N = (o * c.mesh.nx + 1) * (o * c.mesh.ny + 1) * (o * c.mesh.nz + 1);
  gather_phi(c, N);
  if (c.rank == 0) {
    if (!c.d_gz) c.d_gz = dalloc<double>(M);  // persistent (freed with the context)
    gravity_z(c, z0, c.d_gz);
    OSM_CUDA(cudaMemcpyAsync(gz, c.d_gz, sizeof(double) * M, cudaMemcpyDeviceToHost, c.stream));
  }
  OSM_CUDA(cudaStreamSynchronize(c.stream));
  *n = M;
  return OSM_OK;
  OSM_API_END
}

static const Sub& local_sub(const Ctx& c, int s) {
  if (!c.assembled) fail(OSM_ERR_STATE, "not assembled");
  if (s < c.s_begin || s >= c.s_end) fail(OSM_ERR_INVALID_ARG, "subdomain not owned by this rank");
  return c.subs[s - c.s_begin];
}

osm_status osm_get_local_solution(osm_ctx* h, int s, double* u, int64_t* n) {
  OSM_API_BEGIN
  Ctx& c = ctx_of(h);
  if (!n) fail(OSM_ERR_INVALID_ARG, "NULL size");
  const Sub& S = local_sub(c, s);
  if (!u) {
    *n = S.n;
    return OSM_OK;
  }
  if (*n < S.n) fail(OSM_ERR_INVALID_ARG, "buffer too small");
  double* d = dalloc<double>(S.n);
  launch_gather_local(c, S, d);
  OSM_CUDA(cudaMemcpyAsync(u, d, sizeof(double) * S.n, cudaMemcpyDeviceToHost, c.stream));
  OSM_CUDA(cudaStreamSynchronize(c.stream));
  dfree(d);
  *n = S.n;
  return OSM_OK;
  OSM_API_END
}

static int find_side(const Ctx& c, int iface, int side) {
  if (iface < 0 || iface >= c.nsub - 1 || (side != 0 && side != 1)) fail(OSM_ERR_INVALID_ARG, "bad interface/side");
  for (size_t k = 0; k < c.sides.size(); ++k)
    if (c.sides[k].iface == iface && c.sides[k].which == side) return (int)k;
  fail(OSM_ERR_INVALID_ARG, "interface side not owned by this rank");
}

osm_status osm_get_trace(osm_ctx* h, int iface, int side, double* lam, int64_t* n) {
  OSM_API_BEGIN
  Ctx& c = ctx_of(h);
  if (!n) fail(OSM_ERR_INVALID_ARG, "NULL size");
  const int k = find_side(c, iface, side);
  if (!lam) {
    *n = c.nG;
    return OSM_OK;
  }
  if (*n < c.nG) fail(OSM_ERR_INVALID_ARG, "buffer too small");
  OSM_CUDA(cudaMemcpyAsync(lam, c.lam_all + k * c.nG, sizeof(double) * c.nG, cudaMemcpyDeviceToHost, c.stream));
  OSM_CUDA(cudaStreamSynchronize(c.stream));
  *n = c.nG;
  return OSM_OK;
  OSM_API_END
}

osm_status osm_get_csr(osm_ctx* h, int s, int64_t* rowptr, int32_t* col, double* val, int64_t* nrows, int64_t* nnz) {
  OSM_API_BEGIN
  Ctx& c = ctx_of(h);
  if (!nrows || !nnz) fail(OSM_ERR_INVALID_ARG, "NULL size");
  const Sub& S = local_sub(c, s);
  if (rowptr) {
    if (*nrows < S.n || *nnz < S.nnz) fail(OSM_ERR_INVALID_ARG, "buffer too small");
    OSM_CUDA(cudaMemcpyAsync(rowptr, S.rowptr, sizeof(int64_t) * (S.n + 1), cudaMemcpyDeviceToHost, c.stream));
    if (col) OSM_CUDA(cudaMemcpyAsync(col, S.col, sizeof(int32_t) * S.nnz, cudaMemcpyDeviceToHost, c.stream));
    if (val) OSM_CUDA(cudaMemcpyAsync(val, S.val, sizeof(double) * S.nnz, cudaMemcpyDeviceToHost, c.stream));
    OSM_CUDA(cudaStreamSynchronize(c.stream));
  }
  *nrows = S.n;
  *nnz = S.nnz;
  return OSM_OK;
  OSM_API_END
}

osm_status osm_get_interface_map(osm_ctx* h, int iface, int side, int32_t* idx, int64_t* n) {
  OSM_API_BEGIN
  Ctx& c = ctx_of(h);
  if (!n) fail(OSM_ERR_INVALID_ARG, "NULL size");
  const int k = find_side(c, iface, side);
  if (idx) {
    if (*n < c.nG) fail(OSM_ERR_INVALID_ARG, "buffer too small");
    OSM_CUDA(cudaMemcpyAsync(idx, c.sides[k].map_c, sizeof(int32_t) * c.nG, cudaMemcpyDeviceToHost, c.stream));
    OSM_CUDA(cudaStreamSynchronize(c.stream));
  }
  *n = c.nG;
  return OSM_OK;
  OSM_API_END
}

osm_status osm_get_interface_mass(osm_ctx* h, int64_t* rowptr, int32_t* col, double* val, int64_t* nrows,
                                  int64_t* nnz) {
  OSM_API_BEGIN
  Ctx& c = ctx_of(h);
  if (!nrows || !nnz) fail(OSM_ERR_INVALID_ARG, "NULL size");
  if (!c.assembled) fail(OSM_ERR_STATE, "not assembled");
  const int64_t m = c.h_mrow.back();
  if (rowptr) {
    if (*nrows < c.nG || *nnz < m) fail(OSM_ERR_INVALID_ARG, "buffer too small");
    for (int64_t i = 0; i <= c.nG; ++i) rowptr[i] = c.h_mrow[i];
    if (col) std::copy(c.h_mcol.begin(), c.h_mcol.end(), col);
    if (val) std::copy(c.h_mval.begin(), c.h_mval.end(), val);
  }
  *nrows = c.nG;
  *nnz = m;
  return OSM_OK;
  OSM_API_END
}

osm_status osm_get_interface_stiffness(osm_ctx* h, double* val, int64_t* nnz) {
  OSM_API_BEGIN
  Ctx& c = ctx_of(h);
  if (!nnz) fail(OSM_ERR_INVALID_ARG, "NULL size");
  if (!c.assembled) fail(OSM_ERR_STATE, "not assembled");
  if (val) {
    if (*nnz < (int64_t)c.h_sval.size()) fail(OSM_ERR_INVALID_ARG, "buffer too small");
    std::copy(c.h_sval.begin(), c.h_sval.end(), val);
  }
  *nnz = (int64_t)c.h_sval.size();
  return OSM_OK;
  OSM_API_END
}

osm_status osm_set_kernel_timing(osm_ctx* h, int enable) {
  OSM_API_BEGIN
  Ctx& c = ctx_of(h);
  c.timing = enable != 0;
  for (auto& t : c.timers) {
    t.used = 0;
    t.total_ms = 0;
    t.launches = 0;
  }
  return OSM_OK;
  OSM_API_END
}

osm_status osm_get_kernel_timing(osm_ctx* h, osm_kernel_time* out, int cap, int* n) {
  OSM_API_BEGIN
  Ctx& c = ctx_of(h);
  if (!n) fail(OSM_ERR_INVALID_ARG, "NULL size");
  *n = (int)c.timers.size();
  if (out)
    for (int i = 0; i < std::min(cap, *n); ++i) {
      std::memset(out[i].name, 0, sizeof(out[i].name));
      std::strncpy(out[i].name, c.timers[i].name.c_str(), sizeof(out[i].name) - 1);
      out[i].launches = c.timers[i].launches;
      out[i].total_ms = c.timers[i].total_ms;
    }
  return OSM_OK;
  OSM_API_END
}

osm_status osm_plan(int64_t nx, int nsub, int nranks, int rank, int* s_begin, int* s_end, osm_plan_side* sides,
                     int cap, int* nsides) {
  OSM_API_BEGIN
  if (!s_begin || !s_end || !nsides) fail(OSM_ERR_INVALID_ARG, "NULL output");
  if (nranks < 1 || rank < 0 || rank >= nranks || nsub < 1 || nsub > nx || nsub % nranks != 0)
    fail(OSM_ERR_INVALID_ARG, "need 1 <= nsub <= nx, nsub % nranks == 0, 0 <= rank < nranks");
  std::vector<PlanSide> plan;
  plan_rank(nsub, nranks, rank, *s_begin, *s_end, plan);
  *nsides = (int)plan.size();
  if (sides)
    for (int k = 0; k < std::min(cap, *nsides); ++k) {
      sides[k].iface = plan[k].iface;
      sides[k].side = plan[k].which;
      sides[k].sub = plan[k].sub;
      sides[k].remote = plan[k].remote;
      sides[k].peer = plan[k].peer;
    }
  return OSM_OK;
  OSM_API_END
}

osm_status osm_solve_batch(osm_ctx* h, int B, const double* alphas, const osm_solve_opts* o, osm_batch_report* rep) {
  OSM_API_BEGIN
  Ctx& c = ctx_of(h);
  if (!o) fail(OSM_ERR_INVALID_ARG, "NULL options");
  if (B < 1 || B > 64) fail(OSM_ERR_INVALID_ARG, "need 1 <= B <= 64");
  const int ni = c.nsub - 1;
  std::vector<double> pq((size_t)B * 4 * std::max(ni, 0), 0.0);  // OO0: q = 0
  if (ni > 0 && !alphas) fail(OSM_ERR_INVALID_ARG, "NULL alphas");
  for (int b = 0; b < B; ++b)
    for (int i = 0; i < ni; ++i) {
      pq[(b * 4 + 0) * ni + i] = alphas[(b * 2 + 0) * ni + i];
      pq[(b * 4 + 2) * ni + i] = alphas[(b * 2 + 1) * ni + i];
    }
  return solve_batch(c, B, pq.data(), *o, rep);
  OSM_API_END
}

osm_status osm_cmaes_batch_optimize(osm_ctx* h, osm_cmaes* es, int gens, const double* z, int n_outer, int k0,
                                    int max_iter, double ftol, double* costs, int* gens_done) {
  OSM_API_BEGIN
  Ctx& c = ctx_of(h);
  if (!es || !z || !gens_done) fail(OSM_ERR_INVALID_ARG, "NULL argument");
  if (gens < 1 || k0 < 1 || n_outer <= k0) fail(OSM_ERR_INVALID_ARG, "need gens >= 1 and 1 <= k0 < n_outer");
  if (c.nsub < 2) fail(OSM_ERR_STATE, "the alpha search needs at least one interface");
  // dimension and population from the handle: 1 (symmetric log alpha) or 2 (log alpha_left, log alpha_right)
  int n = 0, lam = 0;
  osm_cmaes_dims(es, &n, &lam);
  if (n < 1 || n > 2) fail(OSM_ERR_INVALID_ARG, "the alpha search has 1 or 2 variables");
  if (lam > 64) fail(OSM_ERR_INVALID_ARG, "population > 64 (the batched solver's limit)");
  const int ni = c.nsub - 1;
  std::vector<double> x((size_t)lam * n), al((size_t)lam * 2 * ni), f(lam);
  osm_solve_opts o{1e-300, n_outer, 1e-10, 20000, 1, 0};
  osm_batch_report rep{};
  *gens_done = 0;
  for (int g = 0; g < gens; ++g) {
    osm_status st = osm_cmaes_ask(es, z + (size_t)g * lam * n, x.data());
    if (st != OSM_OK) return st;
    for (int b = 0; b < lam; ++b) {
      const double a_l = std::exp(x[(size_t)b * n]), a_r = std::exp(x[(size_t)b * n + n - 1]);
      for (int i = 0; i < ni; ++i) {
        al[((size_t)b * 2 + 0) * ni + i] = a_l;
        al[((size_t)b * 2 + 1) * ni + i] = a_r;
      }
    }
    std::vector<double> pq((size_t)lam * 4 * ni, 0.0);  // OO0: q = 0
    for (int b = 0; b < lam; ++b)
      for (int i = 0; i < ni; ++i) {
        pq[(b * 4 + 0) * ni + i] = al[((size_t)b * 2 + 0) * ni + i];
        pq[(b * 4 + 2) * ni + i] = al[((size_t)b * 2 + 1) * ni + i];
      }
    solve_batch(c, lam, pq.data(), o, &rep);
    for (int b = 0; b < lam; ++b) {
      // empirical contraction (DESIGN R6): (h(N) / h(k0))^(1 / (N - k0)); 1 if unusable
      int nh = 0;
      batch_history(c, b, nullptr, 0, &nh);
      std::vector<double> hv(nh);
      batch_history(c, b, hv.data(), nh, &nh);
      double cost = 1.0;
      if ((int)hv.size() >= n_outer && hv[k0 - 1] > 0 && std::isfinite(hv[n_outer - 1]))
        cost = std::pow(hv[n_outer - 1] / hv[k0 - 1], 1.0 / (n_outer - k0));
      f[b] = cost;
      if (costs) costs[(size_t)g * lam + b] = cost;
    }
    st = osm_cmaes_tell(es, f.data());
    if (st != OSM_OK) return st;
    *gens_done = g + 1;
    int stop = 0;
    osm_cmaes_should_stop(es, max_iter, ftol, &stop);
    if (stop) break;
  }
  return OSM_OK;
  OSM_API_END
}

osm_status osm_solve_batch2(osm_ctx* h, int B, const double* pq, const osm_solve_opts* o, osm_batch_report* rep) {
  OSM_API_BEGIN
  Ctx& c = ctx_of(h);
  if (!o) fail(OSM_ERR_INVALID_ARG, "NULL options");
  return solve_batch(c, B, pq, *o, rep);
  OSM_API_END
}

osm_status osm_get_batch_history(osm_ctx* h, int b, double* hist, int cap, int* n) {
  OSM_API_BEGIN
  Ctx& c = ctx_of(h);
  if (!n) fail(OSM_ERR_INVALID_ARG, "NULL size");
  batch_history(c, b, hist, cap, n);
  return OSM_OK;
  OSM_API_END
}

osm_status osm_get_batch_inner_iters(osm_ctx* h, int b, int32_t* its, int cap, int* n) {
  OSM_API_BEGIN
  Ctx& c = ctx_of(h);
  if (!n) fail(OSM_ERR_INVALID_ARG, "NULL size");
  batch_inner(c, b, its, cap, n);
  return OSM_OK;
  OSM_API_END
}

osm_status osm_get_batch_local_solution(osm_ctx* h, int b, int s, double* u, int64_t* n) {
  OSM_API_BEGIN
  Ctx& c = ctx_of(h);
  if (!n) fail(OSM_ERR_INVALID_ARG, "NULL size");
  batch_local_solution(c, b, s, u, n);
  return OSM_OK;
  OSM_API_END
}

osm_status osm_set_spmv_variant(osm_ctx* h, int v, int* active) {
  OSM_API_BEGIN
  Ctx& c = ctx_of(h);
  if (v != 2 && v != 3 && v != 5 && v != 6 && v != 7 && v != 10 && v != 11)
    fail(OSM_ERR_INVALID_ARG, "SpMV variant must be one of 2, 3, 5, 6, 7, 10, 11");
  c.spmv_variant = v;
  drop_graph(c);  // captured launches embed the old kernel
  if (active) *active = spmv_variant_of(c);
  return OSM_OK;
  OSM_API_END
}

osm_status osm_set_row_order(osm_ctx* h, int order) {
  OSM_API_BEGIN
  Ctx& c = ctx_of(h);
  if (order < 0 || order > 6 || order == 5) fail(OSM_ERR_INVALID_ARG, "row order must be 0..4 or 6");
  if (c.assembled) fail(OSM_ERR_STATE, "osm_set_row_order must precede osm_assemble");
  c.sort_key = order;
  return OSM_OK;
  OSM_API_END
}

osm_status osm_get_launch_count(osm_ctx* h, int64_t* n) {
  OSM_API_BEGIN
  Ctx& c = ctx_of(h);
  if (!n) fail(OSM_ERR_INVALID_ARG, "NULL output");
  *n = c.launches;
  return OSM_OK;
  OSM_API_END
}

osm_status osm_get_traffic_model(osm_ctx* h, double* out, int n) {
  OSM_API_BEGIN
  Ctx& c = ctx_of(h);
  if (!out) fail(OSM_ERR_INVALID_ARG, "NULL output");
  for (int i = 0; i < std::min(n, 8); ++i) out[i] = c.traffic[i];
  return OSM_OK;
  OSM_API_END
}

}  // extern "C"

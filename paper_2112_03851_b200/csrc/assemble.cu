// Device-side setup of libosm: structural CSR assembly of K_s^N from the
// per-parity-class stencil tables, the load vector of 4 pi G drho, the SELL-32
// hot-path copy, and the Robin fold list.  (8(c) steps 2-8.)
//
// One thread per row: a row (lattice point P of class r = P mod o) visits the
// table's column offsets dQ in column order and, for each, sums the element
// contributions K_e[t][a][b] of the tets (cell P div o + dc, tet t) that lie in
// the slab, in element order (cell id ascending, then tet), exactly as a
// sequential element-by-element assembly would.  A column exists when the
// point P + dQ is a free point of the slab and at least one of its tets lies in
// the slab -- the structural pattern, independent of rounding.
#include "ctx.h"

namespace osm {

namespace {

__device__ __forceinline__ void lattice_of(const SlabGeom& g, int64_t i, int64_t& I, int64_t& J, int64_t& K) {
  I = g.I_lo + i % g.nI;
  const int64_t t = i / g.nI;
  J = 1 + t % g.nJ;
  K = 1 + t / g.nJ;
}

__device__ __forceinline__ bool cell_in_slab(const SlabGeom& g, int64_t cx, int64_t cy, int64_t cz) {
  return cx >= g.c0 && cx < g.c1 && cy >= 0 && cy < g.ny && cz >= 0 && cz < g.nz;
}

__device__ __forceinline__ int64_t local_of(const SlabGeom& g, int64_t I, int64_t J, int64_t K) {
  if (I < g.I_lo || I > g.I_hi || J < 1 || J > g.Ny - 2 || K < 1 || K > g.Nz - 2) return -1;
  return (I - g.I_lo) + g.nI * ((J - 1) + g.nJ * (K - 1));
}

template <bool kFill>
__global__ void k_assemble(SlabGeom g, int64_t n, StencilDev T, int32_t* __restrict__ rowlen,
                           const int64_t* __restrict__ rowptr, int32_t* __restrict__ col, double* __restrict__ val) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t I, J, K;
  lattice_of(g, i, I, J, K);
  const int o = g.order;
  const int rx = (int)(I % o), ry = (int)(J % o), rz = (int)(K % o);
  const int cls = rx + o * (ry + o * rz);
  const int64_t qx = (I - rx) / o, qy = (J - ry) / o, qz = (K - rz) / o;
  int cnt = 0;
  int64_t pos = kFill ? rowptr[i] : 0;
  for (int e = T.col_begin[cls]; e < T.col_begin[cls + 1]; ++e) {
    const StencilCol sc = T.cols[e];
    const int64_t jc = local_of(g, I + sc.dx, J + sc.dy, K + sc.dz);
    if (jc < 0) continue;
    double s = 0.0;
    bool any = false;
    for (int k = sc.c0; k < sc.c1; ++k) {
      const StiffContrib cb = T.contribs[k];
      if (cell_in_slab(g, qx + cb.dcx, qy + cb.dcy, qz + cb.dcz)) {
        s = __dadd_rn(s, cb.val);
        any = true;
      }
    }
    if (!any) continue;
    if (kFill) {
      col[pos] = (int32_t)jc;
      val[pos] = s;
      ++pos;
    } else {
      ++cnt;
    }
  }
  if (!kFill) rowlen[i] = cnt;
}

// Load b_i = sum_T f_T int_T phi_i with f_T = 4 pi G drho_cell, written in
// internal order.
__global__ void k_load(SlabGeom g, int64_t n, StencilDev T, const double* __restrict__ drho, double fourpiG,
                       const int32_t* __restrict__ iperm, int64_t row0, double* __restrict__ b) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t I, J, K;
  lattice_of(g, i, I, J, K);
  const int o = g.order;
  const int rx = (int)(I % o), ry = (int)(J % o), rz = (int)(K % o);
  const int cls = rx + o * (ry + o * rz);
  const int64_t qx = (I - rx) / o, qy = (J - ry) / o, qz = (K - rz) / o;
  double s = 0.0;
  for (int e = T.load_begin[cls]; e < T.load_begin[cls + 1]; ++e) {
    const LoadContrib L = T.loads[e];
    const int64_t cx = qx + L.dcx, cy = qy + L.dcy, cz = qz + L.dcz;
    if (!cell_in_slab(g, cx, cy, cz)) continue;
    const double f = __dmul_rn(fourpiG, drho[cx + g.nx * (cy + g.ny * cz)]);
    s = __dadd_rn(s, __dmul_rn(f, L.w));
  }
  b[row0 + iperm[i]] = s;
}

// Load from a global free-DOF vector (osm_upload_load_vector): b_s = b_free at the slab's points,
// halved on the slab's interface planes (the two duplicates of an interface row share the load,
// so b_s + b_t = b_free there and the glued system is the monolithic one).
__global__ void k_load_free(SlabGeom g, int64_t n, int64_t Nx, const double* __restrict__ bfree,
                            const int32_t* __restrict__ iperm, int64_t row0, double* __restrict__ b) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t I, J, K;
  lattice_of(g, i, I, J, K);
  const int64_t gi = (I - 1) + (Nx - 2) * ((J - 1) + (g.Ny - 2) * (K - 1));
  const bool iface = (g.c0 > 0 && I == g.order * g.c0) || (g.c1 < g.nx && I == g.order * g.c1);
  b[row0 + iperm[i]] = iface ? 0.5 * bfree[gi] : bfree[gi];
}

// Copy contract CSR rows into SELL-256 tiles (column-major over the tile), remapping
// columns to internal concatenated indices; padding = (val 0, col = own row).  Also dinv from K^N.
__global__ void k_sell_build(int64_t npad, int64_t row0, int64_t blk0, const int32_t* __restrict__ perm,
                             const int32_t* __restrict__ iperm, const int64_t* __restrict__ rowptr,
                             const int32_t* __restrict__ ccol, const double* __restrict__ cval,
                             const int64_t* __restrict__ soff, const int32_t* __restrict__ swidth,
                             double* __restrict__ sval, int32_t* __restrict__ scol, double* __restrict__ dinv,
                             int32_t* __restrict__ flags) {
  const int64_t ri = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (ri >= npad) return;
  const int64_t tile = blk0 + ri / kRowsPerBlock;
  const int lane = (int)(ri % kRowsPerBlock);
  const int64_t off = soff[tile] + lane;
  const int w = swidth[tile];
  const int64_t grow = row0 + ri;
  const int c = perm[ri];
  constexpr int64_t T = kRowsPerBlock;
  if (c < 0) {
    for (int k = 0; k < w; ++k) {
      scol[off + T * k] = (int32_t)grow;
      sval[off + T * k] = 0.0;
    }
    dinv[grow] = 0.0;
    return;
  }
  const int64_t beg = rowptr[c];
  const int len = (int)(rowptr[c + 1] - beg);
  double d = 0.0;
  bool found = false;
  for (int k = 0; k < w; ++k) {
    if (k < len) {
      const int cc = ccol[beg + k];
      scol[off + T * k] = (int32_t)(row0 + iperm[cc]);
      sval[off + T * k] = cval[beg + k];
      if (cc == c) {
        d = cval[beg + k];
        found = true;
      }
    } else {
      scol[off + T * k] = (int32_t)grow;
      sval[off + T * k] = 0.0;
    }
  }
  if (!found || !(d > 0.0)) atomicOr(flags, 1);
  dinv[grow] = (found && d > 0.0) ? 1.0 / d : 0.0;
}

// For each M_Gamma entry (g, g2) of a side: the SELL position of K_s entry (map[g], map[g2]).
__global__ void k_fold_build(int64_t nG, const int32_t* __restrict__ map_c, const int32_t* __restrict__ mrow,
                             const int32_t* __restrict__ mcol, const double* __restrict__ mval,
                             const double* __restrict__ sval, double* __restrict__ fold_s,
                             const int64_t* __restrict__ rowptr, const int32_t* __restrict__ ccol,
                             const double* __restrict__ cval, const int32_t* __restrict__ iperm, int64_t row0,
                             int64_t blk0, const int64_t* __restrict__ soff, int64_t fold0, int side_idx,
                             int64_t* __restrict__ fold_pos, double* __restrict__ fold_m, double* __restrict__ fold_kn,
                             int32_t* __restrict__ fold_diag_row, int32_t* __restrict__ fold_side,
                             int32_t* __restrict__ flags) {
  const int64_t gi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gi >= nG) return;
  const int c = map_c[gi];
  const int ri = iperm[c];
  const int64_t tile = blk0 + ri / kRowsPerBlock;
  const int lane = ri % kRowsPerBlock;
  const int64_t beg = rowptr[c], end = rowptr[c + 1];
  for (int j = mrow[gi]; j < mrow[gi + 1]; ++j) {
    const int cc = map_c[mcol[j]];
    int64_t lo = beg, hi = end;  // binary search in the sorted row
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (ccol[mid] < cc) lo = mid + 1; else hi = mid;
    }
    const int64_t e = fold0 + j;
    if (lo >= end || ccol[lo] != cc) {
      atomicOr(flags, 2);
      fold_pos[e] = -1;
      continue;
    }
    fold_pos[e] = soff[tile] + (int64_t)kRowsPerBlock * (lo - beg) + lane;
    fold_m[e] = mval[j];
    fold_s[e] = sval[j];
    fold_kn[e] = cval[lo];
    fold_diag_row[e] = (cc == c) ? (int32_t)(row0 + ri) : -1;
    fold_side[e] = side_idx;
  }
}

// K_s = K_s^N + (p_s M_Gamma + q_s S_Gamma) on the interface rows (OO2
// PAPER.md:78), and the Jacobi diagonal of the Robin-augmented rows.
__global__ void k_fold_apply(int64_t nfold, const double* __restrict__ alpha_side, const double* __restrict__ q_side,
                             const int64_t* __restrict__ pos, const double* __restrict__ m,
                             const double* __restrict__ sv, const double* __restrict__ kn,
                             const int32_t* __restrict__ diag_row, const int32_t* __restrict__ side,
                             double* __restrict__ sval, double* __restrict__ dinv, int32_t* __restrict__ flags) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= nfold) return;
  const int64_t p = pos[e];
  if (p < 0) return;
  const double a = __dadd_rn(__dmul_rn(alpha_side[side[e]], m[e]), __dmul_rn(q_side[side[e]], sv[e]));
  const double v = __dadd_rn(kn[e], a);
  sval[p] = v;
  const int dr = diag_row[e];
  if (dr >= 0) {
    if (!(v > 0.0)) atomicOr(flags, 1);
    dinv[dr] = v > 0.0 ? 1.0 / v : 0.0;
  }
}

__global__ void k_scatter_phi(SlabGeom g, int64_t npad, int64_t row0, const int32_t* __restrict__ perm,
                              const double* __restrict__ ut, int only_owned, double* __restrict__ phi) {
  const int64_t ri = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (ri >= npad) return;
  const int c = perm[ri];
  if (c < 0) return;
  int64_t I, J, K;
  lattice_of(g, c, I, J, K);
  if (only_owned && g.c0 > 0 && I == g.order * g.c0) return;  // left plane belongs to the left slab
  const int64_t Nx = g.order * g.nx + 1;
  phi[I + Nx * (J + g.Ny * K)] = ut[row0 + ri];
}

__global__ void k_gather_local(int64_t npad, int64_t row0, const int32_t* __restrict__ perm,
                               const double* __restrict__ x, double* __restrict__ out) {
  const int64_t ri = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (ri >= npad) return;
  const int c = perm[ri];
  if (c >= 0) out[c] = x[row0 + ri];
}

inline int grid_for(int64_t n, int threads = 256) { return (int)ceil_div(n > 0 ? n : 1, threads); }

StencilDev tables_of(const Ctx& c) {
  return StencilDev{c.d_col_begin, c.d_cols, c.d_contribs, c.d_load_begin, c.d_loads, c.mesh.order};
}

}  // namespace

void launch_count(const Ctx& c, const Sub& s, int32_t* rowlen) {
  k_assemble<false><<<grid_for(s.n), 256, 0, c.stream>>>(s.g, s.n, tables_of(c), rowlen, nullptr, nullptr, nullptr);
  OSM_CHECK_LAUNCH();
  ++c.launches;
}

void launch_fill(const Ctx& c, const Sub& s) {
  k_assemble<true><<<grid_for(s.n), 256, 0, c.stream>>>(s.g, s.n, tables_of(c), nullptr, s.rowptr, s.col, s.val);
  OSM_CHECK_LAUNCH();
  ++c.launches;
}

void launch_sell_build(const Ctx& c, const Sub& s, const int32_t*) {
  k_sell_build<<<grid_for(s.npad), 256, 0, c.stream>>>(s.npad, s.row0, s.blk0, s.perm, s.iperm, s.rowptr, s.col,
                                                      s.val, c.sell_soff, c.sell_swidth, c.sell_val, c.sell_col,
                                                      c.dinv, c.d_flags);
  OSM_CHECK_LAUNCH();
  ++c.launches;
}

void launch_fold_build(const Ctx& c, const Side& sd, const Sub& s) {
  const int side_idx = (int)(&sd - c.sides.data());
  k_fold_build<<<grid_for(c.nG), 256, 0, c.stream>>>(c.nG, sd.map_c, c.d_mrow, c.d_mcol, c.d_mval, c.d_sval,
                                                    c.fold_s, s.rowptr, s.col,
                                                    s.val, s.iperm, s.row0, s.blk0, c.sell_soff, sd.fold0, side_idx,
                                                    c.fold_pos, c.fold_m, c.fold_kn, c.fold_diag_row, c.fold_side,
                                                    c.d_flags);
  OSM_CHECK_LAUNCH();
  ++c.launches;
}

void launch_fold_apply(const Ctx& c, const double* d_alpha_side, const double* d_q_side) {
  if (c.nfold == 0) return;
  k_fold_apply<<<grid_for(c.nfold), 256, 0, c.stream>>>(c.nfold, d_alpha_side, d_q_side, c.fold_pos, c.fold_m,
                                                       c.fold_s, c.fold_kn,
                                                       c.fold_diag_row, c.fold_side, c.sell_val, c.dinv, c.d_flags);
  OSM_CHECK_LAUNCH();
  ++c.launches;
}

void launch_load(const Ctx& c, const Sub& s, double fourpiG) {
  k_load<<<grid_for(s.n), 256, 0, c.stream>>>(s.g, s.n, tables_of(c), c.drho, fourpiG, s.iperm, s.row0, c.b);
  OSM_CHECK_LAUNCH();
  ++c.launches;
}

void launch_load_free(const Ctx& c, const Sub& s, const double* d_bfree) {
  k_load_free<<<grid_for(s.n), 256, 0, c.stream>>>(s.g, s.n, c.mesh.order * c.mesh.nx + 1, d_bfree, s.iperm, s.row0,
                                                  c.b);
  OSM_CHECK_LAUNCH();
  ++c.launches;
}

void launch_scatter_phi(const Ctx& c, const Sub& s, int only_owned) {
  k_scatter_phi<<<grid_for(s.npad), 256, 0, c.stream>>>(s.g, s.npad, s.row0, s.perm, c.ut, only_owned, c.phi);
  OSM_CHECK_LAUNCH();
  ++c.launches;
}

void launch_gather_local(const Ctx& c, const Sub& s, double* out_contract) {
  k_gather_local<<<grid_for(s.npad), 256, 0, c.stream>>>(s.npad, s.row0, s.perm, c.x, out_contract);
  OSM_CHECK_LAUNCH();
  ++c.launches;
}


namespace {
__global__ void k_mf_refresh(int64_t n, const int64_t* __restrict__ src, const double* __restrict__ sval,
                             double* __restrict__ val) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) val[i] = src[i] >= 0 ? sval[src[i]] : 0.0;
}
}  // namespace

namespace {
// Every real row's SELL entries (padding (+0.0, own row) excluded) must equal, in order and
// bitwise, its table's entries whose target is not a dummy row (islot -2).
__global__ void k_mf_verify(int64_t nrows, const int32_t* __restrict__ blk_sub, const MfSub* __restrict__ msub,
                            const int32_t* __restrict__ mf_begin, const int32_t* __restrict__ mf_delta,
                            const double* __restrict__ mf_val, const int64_t* __restrict__ soff,
                            const int32_t* __restrict__ swidth, const double* __restrict__ sval,
                            const int32_t* __restrict__ scol, const int32_t* __restrict__ islot,
                            int32_t* __restrict__ bad) {
  const int64_t ri = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (ri >= nrows) return;
  const int64_t blk = ri / kRowsPerBlock;
  const int lane = (int)(ri % kRowsPerBlock);
  const MfSub M = msub[blk_sub[blk]];
  const int t = mf_table_of(M, ri - M.row0);
  const int w = swidth[blk];
  const int64_t base = soff[blk] + lane;
  int e = t >= 0 ? mf_begin[t] : 0;
  const int e1 = t >= 0 ? mf_begin[t + 1] : 0;
  for (int k = 0; k < w; ++k) {
    const double v = sval[base + (int64_t)kRowsPerBlock * k];
    const int64_t cidx = scol[base + (int64_t)kRowsPerBlock * k];
    if (cidx == ri && v == 0.0 && !signbit(v)) continue;  // SELL padding (a real diagonal is > 0)
    while (e < e1 && (mf_val[e] == 0.0 && mf_delta[e] == 0 ? true : islot[ri + mf_delta[e]] == -2) &&
           !(ri + mf_delta[e] == cidx && mf_val[e] == v))
      ++e;  // table padding, or an entry into a dummy row (multiplies an exact zero)
    if (e >= e1 || ri + mf_delta[e] != cidx ||
        __double_as_longlong(mf_val[e]) != __double_as_longlong(v)) {
      atomicOr(bad, 1);
      return;
    }
    ++e;
  }
  for (; e < e1; ++e)  // leftovers must be padding or point into dummy rows
    if (!(mf_val[e] == 0.0 && mf_delta[e] == 0) && islot[ri + mf_delta[e]] != -2) {
      atomicOr(bad, 1);
      return;
    }
}
}  // namespace

namespace {
__global__ void k_mf_codes(int64_t nrows, const int32_t* __restrict__ blk_sub, const MfSub* __restrict__ msub,
                           const int16_t* __restrict__ tabid, uint8_t* __restrict__ code) {
  const int64_t ri = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (ri >= nrows) return;
  const MfSub& M = msub[blk_sub[ri / kRowsPerBlock]];
  const int t = mf_table_of(M, ri - M.row0);
  code[ri] = t >= 0 ? (uint8_t)tabid[t] : (uint8_t)0xff;
}
}  // namespace

void launch_mf_codes(const Ctx& c, const int16_t* d_tabid) {
  k_mf_codes<<<(unsigned)ceil_div(c.nrows_total, 256), 256, 0, c.stream>>>(c.nrows_total, c.blk_sub, c.d_mf_sub,
                                                                          d_tabid, c.d_mf_code);
  OSM_CHECK_LAUNCH();
  ++c.launches;
}

void launch_mf_verify(const Ctx& c, int32_t* d_bad) {
  if (!c.mf_ok) return;
  k_mf_verify<<<(unsigned)ceil_div(c.nrows_total, 256), 256, 0, c.stream>>>(
      c.nrows_total, c.blk_sub, c.d_mf_sub, c.d_mf_begin, c.d_mf_delta, c.d_mf_val, c.sell_soff, c.sell_swidth,
      c.sell_val, c.sell_col, c.islot, d_bad);
  OSM_CHECK_LAUNCH();
  ++c.launches;
}

void launch_mf_refresh(const Ctx& c) {
  if (!c.mf_ok || c.mf_entries == 0) return;
  k_mf_refresh<<<(unsigned)ceil_div(c.mf_entries, 256), 256, 0, c.stream>>>(c.mf_entries, c.d_mf_src, c.sell_val,
                                                                           c.d_mf_val);
  OSM_CHECK_LAUNCH();
  ++c.launches;
}

}  // namespace osm

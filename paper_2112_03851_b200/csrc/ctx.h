// Internal context of libosm: per-GPU subdomain store, interface sides and the
// launchers of the device kernels (assemble.cu, schwarz_kernels.cu).
#pragma once
#include <cuda.h>
#include <nccl.h>

#include <string>
#include <vector>

#include "common.h"
#include "lattice.h"
#include "transport.h"

namespace osm {

// Free-point box of one x-slab in lattice coordinates.
struct SlabGeom {
  int64_t c0, c1;          // cells [c0, c1) in x
  int64_t nx, ny, nz;      // global cell counts
  int64_t Ny, Nz;          // lattice points in y, z
  int64_t I_lo, I_hi;      // inclusive free I range
  int64_t nI, nJ, nK;      // free box extents
  int order;
};

// Device view of the stencil tables.
struct StencilDev {
  const int32_t* col_begin;
  const StencilCol* cols;
  const StiffContrib* contribs;
  const int32_t* load_begin;
  const LoadContrib* loads;
  int order;
};

// SELL-256 matrix over the concatenated internal rows of every local subdomain.
// Tile t (= hot-path block t) holds internal rows [256t, 256t+256); entry j of its
// row l sits at toff[t] + 256 j + l (column major over the tile), so entries
// [j0, j1) of the whole tile are one contiguous range (bulk-copy friendly);
// padding entries have val 0, col = own row.
// Matrix-free Kuhn-stencil view of one local subdomain (SpMV variant 5, row order 4).
// Internal layout: the slab's whole lattice box [o c0, o c1] x [0, Ny) x [0, Nz), split into the
// o^3 parity classes c = rx + o (ry + o rz); class c is the sub-lattice (ii, jj, kk) -> point
// (o ii + rx, o jj + ry, o kk + rz), stored at internal local index c hIJK + jj + hJ (kk + hK ii)
// (y fastest, x slowest).  Dirichlet and out-of-box points are inert dummy rows (zero vectors), so
// a row's neighbour through stencil entry e sits at a constant offset delta_e for every row of
// its (kind, class): no column indices and no boundary masks.
struct MfSub {
  int64_t row0;       // first internal row of the subdomain
  int32_t hJ, hK;     // sub-lattice extents in y, z
  int32_t hJK, hIJK;  // hJ hK, hI hJ hK
  int32_t nIs;        // lattice points of the slab in x (o (c1 - c0) + 1)
  int32_t Ny, Nz;     // lattice points in y, z
  int32_t dir_lo;     // 1: the slab's x = first plane is the Dirichlet boundary (first slab)
  int32_t dir_hi;     // 1: the slab's last plane is the Dirichlet boundary (last slab)
  int32_t tab0;       // table index of (kind 0, class 0); table t = tab0 + kind nclass + c
  int32_t o, nclass;
  double inv_hIJK, inv_hJK, inv_hJ;  // reciprocals for the row decode (exact-corrected division)
};

// n / d for 0 <= n < 2^31 via a double reciprocal and one correction step (the quotient estimate is
// within 1 of the truth): ~6 instructions instead of a ~25-instruction integer division.
__device__ __forceinline__ int mf_div(int n, int d, double inv, int& r) {
  int q = (int)((double)n * inv);
  r = n - q * d;
  if (r < 0) {
    --q;
    r += d;
  } else if (r >= d) {
    ++q;
    r -= d;
  }
  return q;
}

// Table of internal local row li of a subdomain (-1: dummy row), see MfSub.
__device__ __forceinline__ int mf_table_of(const MfSub& M, int64_t li) {
  if (li >= (int64_t)M.nclass * M.hIJK) return -1;
  int rem, r2, jj;
  const int cl = mf_div((int)li, M.hIJK, M.inv_hIJK, rem);
  const int ii = mf_div(rem, M.hJK, M.inv_hJK, r2);
  const int kk = mf_div(r2, M.hJ, M.inv_hJ, jj);
  int rx = 0, ry = 0, rz = 0, o = 1;
  if (M.o == 2) {
    rx = cl & 1;
    ry = (cl >> 1) & 1;
    rz = cl >> 2;
    o = 2;
  }
  const int I = o * ii + rx, J = o * jj + ry, K = o * kk + rz;
  if (I >= M.nIs || J < 1 || J > M.Ny - 2 || K < 1 || K > M.Nz - 2 || (M.dir_lo && I == 0) ||
      (M.dir_hi && I == M.nIs - 1))
    return -1;
  const int kind = I == 0 ? 1 : (I == M.nIs - 1 ? 2 : 0);
  return M.tab0 + kind * M.nclass + cl;
}

// The matrix-free tables as a kernel parameter (constant bank): table values and offsets are
// read through the constant cache (uniform broadcast), not the L1/TEX load path, which the x
// gathers need.  Tables are deduplicated across subdomains; used when they fit.
constexpr int kMfMaxSub = 16, kMfMaxTab = 128, kMfMaxGroups = 560;
struct MfConst {
  int32_t valid;
  int16_t tabid[kMfMaxSub * 3 * 8];  // (local subdomain, kind, class) -> deduplicated table
  int32_t gbeg[kMfMaxTab + 1];       // group range [gbeg[t], gbeg[t+1]) of a table
  int4 delta[kMfMaxGroups];
  double val[4 * kMfMaxGroups];
  double dinv[kMfMaxTab];            // 1 / (Robin-folded) diagonal of a table, as k_sell_build / k_fold_apply
};
template <int V>
struct MfArg {
  int32_t unused;
};
template <>
struct MfArg<5> {
  MfConst c;
};
// Variant 6: the value-indexed dictionary in the constant bank (kernel parameter) instead of
// shared memory (variant 4).
constexpr int kCDict = 2048;
template <>
struct MfArg<6> {
  double dict[kCDict];
};
template <>
struct MfArg<7> {  // variant 6 on the wide (20-bit offset) entries
  double dict[kCDict];
};
template <>
struct MfArg<10> {  // variant 10: 3-byte entries, at most 256 dictionary slots
  double dict[256];
};
struct SellDev {
  const double* val;
  const int32_t* col;
  const int64_t* toff;
  const int32_t* twidth;
  const uint32_t* packed;  // value-indexed copy (variant 3): (dict index << 16) | (uint16)(col - row),
  const int64_t* poff;     //   4 entries of a row per uint4 (see vi.cu); per-tile word offsets
  const int32_t* vtw;      //   per-tile packed widths (exact zeros dropped)
  const double* dict;      // distinct values
  int ndict;
  // matrix-free view (variant 5): kinds 0 interior, 1 left interface plane, 2 right interface plane
  const int32_t* blk_sub;   // block -> local subdomain
  const MfSub* mf_sub;      // per local subdomain
  const int32_t* mf_begin;  // table t = entries [mf_begin[t], mf_begin[t+1]), padded to a multiple of 4
  const int4* mf_delta;     // 4 row offsets per group
  const double* mf_val;     // values (exact copies of the assembled, Robin-folded SELL entries)
  int64_t nrows;            // rows of the concatenated vectors (bulk-copy bounds)
  const uint8_t* mf_code;   // per row: deduplicated table id of the constant-bank tables, 0xff dummy row
  const uint4* vi3_off;     // variant 10: 8 int16 offsets per group
  const uint2* vi3_idx;     //   8 u8 dictionary indices per group
  const int64_t* vi3_base;  //   per tile: first group slot
};

// ---- brick SpMV (variant 11, row order 6; brick.cu)
// One lattice parity class of one local subdomain: class-local ranges (inclusive) and its dense array
// (jj fastest, padded to nJp; then ii; then kk) at internal row row0 + base.
struct BrickClass {
  int32_t iilo, iihi, jjlo, jjhi, kklo, kkhi;
  int32_t nIc, nJp, nKc;
  int64_t base;
};
struct BrickSub {
  BrickClass cls[8];
  int64_t row0;              // first internal row of the subdomain
  int64_t nrows;             // class-array rows (before the padding to 256)
  int32_t I_lo, nI, nJ;      // contract geometry (lattice of a contract local index)
  int32_t nbj, nbi, nbk;     // bricks along jj, ii, kk
  int64_t brick0, nbrick;    // the subdomain's bricks (global brick index on this GPU)
};
struct BrickInfo {
  int32_t ls;
  int16_t bj, bi, bk, pad;
};
// Per (brick, class, il) chunk of the Kuhn kernel: desc >= 0 a row-type id (every row of the chunk has
// the same index words: typetab[desc][0..ng)), < 0 -(g + 1) with the chunk's per-lane words at
// cstream[32 g + 32 k + lane], k < ng; mask bit lane: the lane's point (jl = lane & 15, kl = lane >> 4)
// is a row; its row is the subdomain's row0 + rowoff + jl + nJI kl.
struct alignas(16) BrickChunk {
  int32_t desc;
  uint32_t mask;
  int32_t rowoff;
  int32_t nJI;
};
struct BrickDev {
  BrickInfo* info = nullptr;
  BrickChunk* chunk = nullptr;   // [brick][class][il] (Kuhn kernel)
  BrickSub* sub = nullptr;
  uint32_t* stream = nullptr;    // u8 dictionary indices, 4 slots per word
  CUtensorMap* tmap = nullptr;   // (local subdomain, class) TMA maps of p
  uint32_t* typetab = nullptr;   // [ntypes][16]
  uint32_t* cstream = nullptr;   // per-lane words of the non-uniform chunks
};
constexpr int kBrickMaxGroups = 24;
// Kernel parameter (constant bank): brick shape, per-class slot groups and shared-memory offsets of
// the slots (relative to the point's own element), the dictionary.
struct BrickArg {
  int32_t BJ, BI, BK, npb;            // brick extents (class-local points) and points per class box
  int32_t box_elems, box_stride, box_bytes;
  int32_t stage_bytes;                // one stage of the persistent kernel: p boxes + index stream
  int32_t dict_n;
  int64_t brick_words;                // stream words per brick
  int32_t ngrp[8], goff[8];           // slot groups per class, first group of the class in a brick
  int32_t jsh[8];                     // class box column of jj = -1 (0 or 1: even TMA start)
  int32_t soff[8 * 4 * kBrickMaxGroups];
  double dict[256];
};
// The PCG direction update fused into the Kuhn SpMV (brick.cu, Ctx::fuse_dir): the kernel of iteration
// k+1 forms p_{k+1} = D^{-1} r_{k+1} + beta_k p_k on its staged boxes (halo included) and pays
// x_{k+1} = x_k + alpha_k p_k on its own rows, so k_cg_dir does not run; p alternates between Ctx::p
// and Ctx::p2 (neighbouring CTAs still read p_k while a CTA writes p_{k+1}).
struct BrickFuse {
  const CUtensorMap* tmap;  // TMA maps of p_k (the buffer read in this iteration)
  double* pn;               // p_{k+1} (the other buffer)
  double* x;
  const double* r;
  const uint8_t* code;      // D^{-1} codes (osm.cu dcode_build; 0xff = +0.0)
  double dtab[kMfMaxTab];
};
// Build-time view (brick.cu).
struct BrickBuildDev {
  int o;
  int64_t nrows;
  const int32_t* row_sub;  // internal row -> local subdomain (-1: none)
  const int32_t* perm;     // internal row -> contract local (-1: pad / dummy)
  const BrickSub* sub;
  int32_t BJ, BI, BK, npb;
  int64_t brick_words;
  int32_t ngrp[8], goff[8];
};
__host__ __device__ inline void brick_lattice_of(const BrickSub& B, int32_t lc, int& I, int& J, int& K) {
  I = B.I_lo + lc % B.nI;
  const int32_t t = lc / B.nI;
  J = 1 + t % B.nJ;
  K = 1 + t / B.nJ;
}
__host__ __device__ inline int brick_class(int o, int I, int J, int K) { return (I % o) + o * ((J % o) + o * (K % o)); }

// Per-subdomain device scalars of the batched PCG / Schwarz kernels.
struct SubState {
  double rho;      // r.z
  double alpha;    // CG step
  double beta;     // CG direction factor
  double bb;       // ||rhs||^2
  double rr;       // ||r||^2
  double resid;    // interior part of sum (f - K u~)^2 for this subdomain
  int64_t blk0;    // first block (256 rows) of the subdomain
  int32_t nblk;    // number of blocks
  int64_t vblk0;   // first vector block (up to kVecTiles tiles) of the subdomain
  int32_t nvblk;   // number of vector blocks
  int32_t active;  // PCG still running
  int32_t iters;   // PCG iterations of the current inner solve
  int32_t status;  // 0 running, 1 converged, 2 max_inner, 3 breakdown
  int32_t zero_rhs;
  uint32_t cnt;    // last-block counter
  int32_t xpend;   // the PCG stopped in this iteration's update: the direction kernel still owes x += alpha p
  int64_t brick0;  // brick SpMV (variant 11): first brick and bricks of the subdomain
  int64_t nbrick;
};

// Device view of one interface side (grid.y of the interface kernels).
struct SideDev {
  const int32_t* map;  // internal (concatenated) row of each plane point
  double* lam;         // lambda_{s,Gamma}
  double* out;         // outbox [g | u | w] (3 nG)
  const double* in;    // partner outbox (local) or receive buffer (remote) [g | u | w]
  double* unbr;        // neighbour trace u_t|Gamma (for gluing)
  double* wif;         // residual (f - K^N u~) at this side's plane rows
  double alpha_own, alpha_sum;  // p of this side, p_s + p_t
  double q_own, q_sum;          // OO2 tangential coefficients (0 for OO0)
  int32_t sub;         // local subdomain index
  int32_t which;       // 0: this slab is the left slab of the interface (its right plane), 1: right slab
  int32_t slot0;       // first islot index of the side (= side * nG)
  int32_t pad;
};

struct Sub {
  int s = -1;  // global subdomain id
  SlabGeom g{};
  int64_t n = 0;                 // local rows (contract)
  int64_t row0 = 0, npad = 0;    // internal range in the concatenated vectors
  int64_t slice0 = 0, nslice = 0;
  int64_t blk0 = 0, nblk = 0;
  int64_t nnz = 0;               // structural nnz of K_s^N
  int64_t sell_entries = 0;      // including padding
  int64_t* rowptr = nullptr;     // contract CSR of K_s^N (device)
  int32_t* col = nullptr;
  double* val = nullptr;
  int32_t* perm = nullptr;       // internal local -> contract local (device, npad, -1 for pad)
  int32_t* iperm = nullptr;      // contract local -> internal local (device, n)
  int side[2] = {-1, -1};        // [0] left plane, [1] right plane (indices into Ctx::sides)
};

struct Side {
  int iface = -1, which = 0, sub = -1;
  bool remote = false;
  int peer = -1;                  // rank of the neighbour
  int partner = -1;               // local side index of the neighbour side (local only)
  int32_t* map_c = nullptr;       // contract local rows (device, nG)
  int32_t* map_g = nullptr;       // internal concatenated rows (device, nG)
  double* out = nullptr;          // outbox (device, 3 nG)
  double* inbuf = nullptr;        // receive buffer (remote only, device, 3 nG)
  int64_t fold0 = 0;              // first Robin fold entry
};

struct KernelTimer {
  std::string name;
  std::vector<cudaEvent_t> ev;  // start/end pairs
  int64_t used = 0;
  double total_ms = 0;
  int64_t launches = 0;
};

struct BatchBuf;

struct Ctx {
  // configuration
  osm_mesh_desc mesh{};
  int rank = 0, nranks = 1, device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  Transport* tp = nullptr;  // inter-rank transport (NCCL or the in-process hub); null for one rank
  osm_hub* hub = nullptr;
  int nsub = 0;
  std::vector<int64_t> cstart;  // slab cell starts
  int s_begin = 0, s_end = 0;   // local subdomains [s_begin, s_end)
  std::vector<double> alpha_left, alpha_right;  // p^(1), p^(2) per interface
  std::vector<double> q_left, q_right;          // q^(1), q^(2) per interface (OO2; 0 = OO0)
  bool robin_set = false, assembled = false, density_set = false;
  bool robin_dirty = true;
  double G = 6.672e-11;

  // stencil tables (device)
  StencilTables tables;
  int32_t *d_col_begin = nullptr, *d_load_begin = nullptr;
  StencilCol* d_cols = nullptr;
  StiffContrib* d_contribs = nullptr;
  LoadContrib* d_loads = nullptr;

  // interface mass (host + device), plane-point order
  int64_t nG = 0;
  std::vector<int32_t> h_mrow, h_mcol;
  std::vector<double> h_mval, h_sval;
  int32_t *d_mrow = nullptr, *d_mcol = nullptr;
  double* d_mval = nullptr;
  double* d_sval = nullptr;  // S_Gamma values aligned with M_Gamma

  // subdomains and sides
  std::vector<Sub> subs;
  std::vector<Side> sides;
  int64_t nrows_total = 0, nslices_total = 0, nblk_total = 0, sell_total = 0;

  // SELL matrix (device)
  double* sell_val = nullptr;
  int32_t* sell_col = nullptr;
  int64_t* sell_soff = nullptr;
  int32_t* sell_swidth = nullptr;
  int32_t* blk_sub = nullptr;  // block -> local subdomain
  int32_t* vblk_sub = nullptr;    // vector block -> local subdomain
  int32_t* vblk_tile0 = nullptr;  // vector block -> first tile
  int32_t* vblk_ntile = nullptr;  // vector block -> tiles (<= kVecTiles)
  int64_t nvblk_total = 0;
  int32_t* islot = nullptr;    // per internal row: -2 pad, -1 interior, >= 0 interface slot

  // Robin fold list (device): sell position, M value, K^N value, diag row (-1 if off-diagonal)
  int64_t nfold = 0;
  int64_t* fold_pos = nullptr;
  double* fold_m = nullptr;
  double* fold_s = nullptr;
  double* fold_kn = nullptr;
  int32_t* fold_diag_row = nullptr;
  int32_t* fold_side = nullptr;

  // vectors (device, nrows_total)
  double *x = nullptr, *r = nullptr, *p = nullptr, *q = nullptr, *dinv = nullptr, *b = nullptr, *ut = nullptr;
  double* drho = nullptr;  // cell density (device, nx ny nz)
  double* d_gz = nullptr;  // gravity-anomaly output (device, nx ny; rank 0)
  // interface arrays (device, nsides * nG)
  double *lam_all = nullptr, *unbr_all = nullptr, *wif_all = nullptr;
  SideDev* d_sides = nullptr;
  std::vector<SideDev> h_sides;
  // reductions
  double* part = nullptr;  // 3 * nblk_total block partials (SpMV / warm / residual kernels)
  double* part_upd = nullptr;  // 2 * nvblk_total vector-block partials (update kernel; separate so that
                               // two subdomain groups' SpMV and update can run concurrently)
  double* side_part = nullptr;  // per side block partials
  double* side_sum = nullptr;   // per side result
  uint32_t* side_cnt = nullptr;
  int64_t side_nblk = 0;
  SubState* st = nullptr;       // per local subdomain
  int32_t* d_nactive = nullptr;
  int32_t* d_flags = nullptr;   // [0] precond failure, [1] fold miss, [2] vi offset overflow, [3] mf mismatch
  // host staging (pinned)
  int32_t* h_nactive = nullptr;  // 2 slots
  SubState* h_st = nullptr;
  double* h_side_sum = nullptr;
  cudaEvent_t ev_chunk[2] = {nullptr, nullptr};

  // full-lattice output buffer (device)
  double* phi = nullptr;

  // last solve results
  std::vector<double> hist;
  std::vector<int32_t> inner;  // [outer][nsub]
  double fnorm2 = 0;

  // Two-stream PCG: the local subdomains split into two groups whose chunk graphs run on their own
  // streams, so one group's kernels fill the other's wave tails (iterations are unchanged: every
  // subdomain's arithmetic is the same).  grp_cur selects the group a launcher works on (-1: all).
  static constexpr int kMaxGroups = 8;
  int ngroups = 1;
  int grp_cur = -1;
  cudaStream_t gstream[kMaxGroups] = {};
  cudaEvent_t ev_fork = nullptr, ev_join[kMaxGroups] = {};
  cudaGraphExec_t cg_graph_g[kMaxGroups] = {};
  int64_t cg_graph_launches_g[kMaxGroups] = {};  // kernels in one replay of cg_graph_g[g] / cg_graph
  int64_t cg_graph_launches = 0;
  int64_t g_blk0[kMaxGroups] = {}, g_nblk[kMaxGroups] = {}, g_vb0[kMaxGroups] = {}, g_nvb[kMaxGroups] = {};
  int vec_tiles = kVecTiles;  // tiles per vector block (update/dir kernels), chosen at assembly
  int vt_override = 0;         // OSM_VT
  bool groups_forced = false;  // OSM_GROUPS given: no size-based reduction
  int want_groups = 8;  // OSM_GROUPS = 1, 2, 4 or 8 (capped by the local subdomain count)

  // CUDA graph of one chunk of PCG iterations (spmv, update, dir) x kCgChunk, with PDL edges
  cudaGraphExec_t cg_graph = nullptr;
  double graph_tol = -1;
  int graph_maxit = -1;
  bool use_graph = true;
  bool force_remote = false;  // debug: every side goes through NCCL (peer = own rank), see osm_create
  bool split_update = true;  // k_cg_update + k_cg_update_fin (no last-block atomic); OSM_SPLIT_UPD=0: one kernel
  int update_variant = 0;  // 0: k_cg_update at 96 regs, 1: capped for 8 blocks/SM
  int sort_key = 6;  // 6 (default): brick layout of the brick SpMV (variant 11): per subdomain, one dense
                    // array per lattice parity class (brick.cu); else the SELL row order inside sigma
                    // windows: 0 length desc, 1 parity class, 2 class then length,
                    // 3 class, length, then (K, I, J) with J fastest; 4: the matrix-free
                    // class-major lattice layout of MfSub (whole subdomain, dummy rows included)
  int sigma = 0;  // SELL sorting window (rows); 0 = automatic (see assemble)
  int spmv_variant = 11;  // SpMV variant (falls back when its format does not apply, spmv_variant_of):
                          // 2: fp64 SELL rows (LDG streams, 32 registers, 8 blocks/SM);
                          // 3: value-indexed SELL (packed 16-bit index + offset, dictionary through L1);
                          // 5: matrix-free Kuhn stencil (row order 4 only; else as 6);
                          // 6: 3 with the dictionary in the constant bank; 7: 6 on wide entries (chosen
                          // automatically when offsets need 20 bits);
                          // 10: 6 with 3-byte entries (int16 offset + u8 index streams; <= 256 slots);
                          // 11 (default): brick copy (row order 6: TMA-staged p bricks, u8 index stream
                          // per (row, stencil slot)); else as 10

  // matrix-free Kuhn-stencil tables (row order 4, SpMV variant 5; osm.cu mf_build)
  bool mf_ok = false;
  MfSub* d_mf_sub = nullptr;
  int32_t* d_mf_begin = nullptr;
  int32_t* d_mf_delta = nullptr;  // int4 groups
  double* d_mf_val = nullptr;
  int64_t* d_mf_src = nullptr;    // SELL position of each table value (-1: padding)
  int64_t mf_entries = 0;         // including padding
  std::vector<int32_t> h_mf_begin, h_mf_delta;
  MfConst* h_mf_const = nullptr;  // host copy of the kernel-parameter tables (valid = 0: global tables)
  uint8_t* d_mf_code = nullptr;   // per internal row: deduplicated table id, 0xff dummy (vector kernels)
  // D^{-1} codes (osm.cu dcode_build): per row a 1-byte index into the distinct D^{-1} values (0xff:
  // +0.0, padding rows), so the SELL-path vector kernels read 1 byte instead of 8 per row
  bool dcode_on = true;           // OSM_DCODE=0 keeps the 8-byte D^{-1} stream
  uint8_t* d_dcode = nullptr;
  std::vector<double> h_dcode_tab;  // empty: codes not built (too many distinct values)

  // brick SpMV (variant 11, row order 6; brick.cu)
  bool brick_ok = false;
  BrickDev brick;
  BrickArg h_brick_arg{};
  std::vector<BrickSub> h_brick_sub;
  int64_t brick_total = 0;
  int64_t brick_cwords = 0;     // words of the compact stream (non-uniform chunks)
  std::vector<int64_t> h_brick_sub_cwords;  // per local subdomain
  int brick_ntypes = 0;
  int brick_kernel = 0;          // 1..12: the P2 Kuhn kernel k_cg_spmv_kuhn<BI>; 0: the generic brick kernel
  double* part_brick = nullptr;  // one p.q partial per brick
  // direction update fused into the Kuhn SpMV (BrickFuse; OSM_FUSE_DIR=0: k_cg_dir runs)
  bool fuse_dir = false;  // measured slower: opt-in
  double* p2 = nullptr;          // the second p buffer of the fused path
  int cg_par = 0;                // PCG iteration parity within a chunk: p_k in p (0) or p2 (1)
  BrickFuse h_brick_fuse{};      // the fused kernel's parameter (host copy, rebuilt per launch)

  // value-indexed SELL (vi.cu)
  bool vi_ok = false;         // dictionary and fold tuples built (the brick copy needs only these)
  bool vi_packed_ok = false;  // the packed value-indexed SELL copy exists (variants 3/6/7)
  bool vi_per_side = false;  // fold slots per interface side (else per side kind)
  uint16_t* vi_idx = nullptr;
  bool vi_wide = false;  // entries (12-bit index << 20) | 20-bit offset (else 16 | 16)
  double* vi_dict = nullptr;
  uint32_t* vi_packed = nullptr;
  int64_t* vi_poff = nullptr;
  int32_t* vi_tw = nullptr;          // per tile: packed width (kept entries of the longest row)
  std::vector<int64_t> vi_kept;      // per local subdomain: kept (nonzero-value) entries
  int64_t vi_words = 0;
  int64_t vi_ndict = 0, vi_nbase = 0;
  struct FoldTuple {
    int32_t side;
    double kn, m, s;
  };
  std::vector<FoldTuple> vi_fold_tuples;
  std::vector<double> h_vi_dict;  // host copy of the dictionary (variant 6 kernel parameter)
  // variant 10 (experimental): 3-byte entries, 8 per group: int16 offsets (uint4) + u8 dictionary
  // indices (uint2) in two streams; group G of row r of tile t at vi3_base[t] + 256 G + r
  bool vi3_ok = false;
  uint4* vi3_off = nullptr;
  uint2* vi3_idx = nullptr;
  int64_t* vi3_base = nullptr;
  int64_t vi3_groups = 0;

  // instrumentation
  bool timing = false;
  std::vector<KernelTimer> timers;

  // batched-alpha solver (batch.cu), built lazily on the first osm_solve_batch
  BatchBuf* batch = nullptr;
  int64_t* batch_sub_blk0 = nullptr;
  int32_t* batch_sub_nblk = nullptr;

  // traffic model of the last solve
  double traffic[8] = {0};
  double exch_bytes = 0;  // NCCL exchange bytes sent in the current solve
  mutable int64_t launches = 0;  // kernel launches issued by this context
};

// ---- launchers (assemble.cu)
void launch_count(const Ctx& c, const Sub& s, int32_t* rowlen);
void launch_fill(const Ctx& c, const Sub& s);
void launch_sell_build(const Ctx& c, const Sub& s, const int32_t* d_slice_width_local);
void launch_fold_build(const Ctx& c, const Side& sd, const Sub& s);
void launch_fold_apply(const Ctx& c, const double* d_alpha_side, const double* d_q_side);
void launch_load(const Ctx& c, const Sub& s, double fourpiG);
void launch_load_free(const Ctx& c, const Sub& s, const double* d_bfree);
void launch_scatter_phi(const Ctx& c, const Sub& s, int only_owned);
void launch_gather_local(const Ctx& c, const Sub& s, double* out_contract);
void launch_mf_refresh(const Ctx& c);  // matrix-free table values <- assembled (folded) SELL values
void launch_mf_verify(const Ctx& c, int32_t* d_bad);  // every row of every subdomain vs its table
void launch_mf_codes(const Ctx& c, const int16_t* d_tabid);  // per-row table codes (d_mf_code)

// ---- launchers (schwarz_kernels.cu)
void launch_warm(Ctx& c, double tol, int warm);
void launch_zero_if(Ctx& c);
void launch_cg_spmv(Ctx& c);
void launch_cg_update(Ctx& c, double tol, int maxit);
void launch_cg_dir(Ctx& c);
void launch_trace(Ctx& c);
void launch_accept(Ctx& c);
void launch_glue(Ctx& c, int zero);
void launch_resid(Ctx& c);
void launch_iface_w(Ctx& c);
void launch_iface_sum(Ctx& c);

// ---- batched alpha (batch.cu)
osm_status solve_batch(Ctx& c, int B, const double* pq, const osm_solve_opts& o, osm_batch_report* rep);
void batch_history(const Ctx& c, int b, double* h, int cap, int* n);
void batch_inner(const Ctx& c, int b, int32_t* its, int cap, int* n);
void batch_local_solution(Ctx& c, int b, int s, double* u, int64_t* n);
void batch_free(Ctx& c);
double fnorm2_of(Ctx& c);  // ||f||^2 of the glued global system (osm.cu)

void gravity_z(Ctx& c, double z0, double* d_out);  // gravity.cu (uses c.phi)
void vi_build(Ctx& c, bool per_side = false);
void vi_free(Ctx& c);
void vi_apply_robin(Ctx& c, const std::vector<double>& p_side, const std::vector<double>& q_side);
void brick_build(Ctx& c, const uint16_t* d_vidx, uint32_t zero_idx);  // brick.cu (row order 6)
void brick_free(Ctx& c);
void brick_geometry(const Ctx& c, int ls, BrickSub& B);
void launch_cg_spmv_brick(Ctx& c, cudaStream_t s, int g);
bool fused_dir(const Ctx& c);  // schwarz_kernels.cu: the Kuhn SpMV carries the direction update
void launch_cg_dir_flush(Ctx& c);
int spmv_variant_of(const Ctx& c);  // the variant actually launched (3 falls back to 2 without vi)

// timing helpers (osm.cu)
void timer_begin(Ctx& c, int id);
void timer_end(Ctx& c, int id);
enum TimerId { T_SPMV = 0, T_UPDATE, T_DIR, T_WARM, T_RESID, T_OUTER_MISC /* NCCL exchange */, T_COUNT };

}  // namespace osm

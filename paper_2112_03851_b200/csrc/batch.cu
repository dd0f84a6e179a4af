// Batched-alpha optimized Schwarz (BASELINE config C4): B candidate
// Robin parameter sets solved simultaneously on one GPU, sharing the Neumann matrices K_s^N.
//
// Each batched PCG iteration reads every K_s^N entry ONCE and applies it to all B
// candidates: vectors are stored [row][candidate] (candidate fastest, stride KB = 32 when
// B <= 32, else 64), one warp per matrix row, lane l owns candidates KB/32 l + j, so a column
// gather is a single coalesced KB*8-byte row of the candidate block.  The candidate-specific Robin
// term alpha_b M_Gamma (OO0) is applied on the fly on interface rows, and
// the Jacobi diagonal of K_b = K^N + alpha_b M_Gamma is formed on the fly, so no per-
// candidate matrix is ever stored.  Every candidate follows exactly the recurrence of the
// single-candidate path (osm_solve) and of the oracle (Jacobi schedule, warm-started
// Jacobi-PCG, glued residual); converged candidates are frozen.
//
// Scope: one rank (C4 runs on one B200); subdomains of that rank are batched together.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "ctx.h"

namespace osm {

constexpr int kBmax = 64;   // largest candidate stride (buffers are sized for it)
constexpr int kRB = 128;    // rows per batched block
constexpr int kBT = 256;    // threads per batched block

struct BState {
  double rho, alpha, beta, bb, rr, resid;
  int32_t active, iters, status, zero_rhs;
};

struct BatchDev {
  // concatenated contract CSR of K^N over local subdomains
  const int64_t* rowptr;
  const int32_t* col;
  const double* val;
  const double* dkn;        // K^N diagonal
  const int32_t* islot;     // per row: -1 interior, else side * nG + g
  const double* b;          // load (contract order)
  const int32_t* blk_sub;   // block -> local subdomain
  const int64_t* blk_row0;  // block -> first row
  const int32_t* blk_nrow;  // block -> rows in block
  const int32_t* mapg;      // [nsides * nG] concatenated contract row of plane point
  const int32_t* mrow;
  const int32_t* mcol;
  const int32_t* mcolg;      // [nsides][nnzM] contract row of each M_Gamma column, per side
  const double* mval;
  const double* sval;       // S_Gamma values (OO2), aligned with mval
  const double* mdiag;      // [nG]
  const double* sdiag;      // [nG]
  const double* alpha_own;  // p of the side, [nsides][KB]
  const double* alpha_sum;  // p_s + p_t, [nsides][KB]
  const double* q_own;      // q of the side (OO2), [nsides][KB]
  const double* q_sum;      // q_s + q_t, [nsides][KB]
  const int32_t* side_which;   // [nsides]
  const int32_t* side_partner; // [nsides]
  const int32_t* cand_active;  // [KB]
  int64_t nG, nnzM;
  int nsides;
};

struct BatchBuf {
  int B = 0;
  int KB = kBmax;               // candidate stride of the last solve (32 or 64)
  int64_t nrows = 0, nblk = 0, nnz = 0;
  int64_t* rowptr = nullptr;
  int32_t* col = nullptr;
  double* val = nullptr;
  double *dkn = nullptr, *b = nullptr;
  int32_t* islot = nullptr;
  int32_t *blk_sub = nullptr, *blk_nrow = nullptr;
  int64_t* blk_row0 = nullptr;
  int32_t* mapg = nullptr;
  int32_t* mcolg = nullptr;
  double *mdiag = nullptr, *sdiag = nullptr;
  double *alpha_own = nullptr, *alpha_sum = nullptr, *q_own = nullptr, *q_sum = nullptr;
  int32_t *side_which = nullptr, *side_partner = nullptr, *cand_active = nullptr;
  double *x = nullptr, *r = nullptr, *p = nullptr, *q = nullptr, *ut = nullptr;
  double *lam = nullptr, *unbr = nullptr, *wif = nullptr, *out = nullptr;
  BState* st = nullptr;
  uint32_t* cnt = nullptr;
  int32_t* nact = nullptr;      // per local subdomain: active candidates (CG)
  int32_t* d_nactive = nullptr; // total active (s, b)
  double* part = nullptr;       // [nblk][3][KB] (SpMM kernels)
  double* part_v = nullptr;     // [nblk][2][KB] (vector kernel; separate so subdomain groups overlap)
  std::vector<int64_t> sblk0_h; // first block of each local subdomain
  int64_t nblk_h = 0;
  double* side_sum = nullptr;   // [nsides][KB]
  std::vector<int64_t> rc0;     // contract row offset of each local subdomain
  // results
  std::vector<std::vector<double>> hist;  // [b][n]
  std::vector<std::vector<int32_t>> inner;  // [b][n * nsub + s]
};

namespace {

// dinv of K_b = K^N + p_b M + q_b S on the fly (rounded like the single path's fold)
template <int KB>
__device__ __forceinline__ double dinv_b(const BatchDev& D, int64_t row, int sl, int b) {
  double d = D.dkn[row];
  if (sl >= 0) {
    const int k = sl / (int)D.nG, g = sl % (int)D.nG;
    d = __dadd_rn(d, __dadd_rn(__dmul_rn(D.alpha_own[k * KB + b], D.mdiag[g]), __dmul_rn(D.q_own[k * KB + b], D.sdiag[g])));
  }
  return d > 0.0 ? 1.0 / d : 0.0;
}

// Block partials [blk][NP][KB] (thread t < KB of the block holds candidate t's sums in sm);
// returns true in the last block of the subdomain.
template <int KB>
__device__ __forceinline__ bool bpublish(double* part, int64_t blk, int NP, const double* sm, uint32_t* cnt,
                                         int nblk_sub) {
  __shared__ bool last;
  for (int i = threadIdx.x; i < NP * KB; i += blockDim.x) part[blk * NP * KB + i] = sm[i];
  __syncthreads();
  if (threadIdx.x == 0) {  // release is cumulative: it orders the block's stores seen through the barrier
    const uint32_t prev = atom_add_release_gpu(cnt, 1u);
    last = prev == (uint32_t)(nblk_sub - 1);
    if (last) __threadfence();
  }
  __syncthreads();
  return last;
}

// Fixed-order sum of the subdomain's block partials, by the whole (last) block: thread
// (g, c) = (tid / KB, tid % KB) sums blocks g, g + G, ... of candidate c (many loads in
// flight per thread), then the G group sums are added in order.  out[k KB + c] = total.
template <int KB, int NP>
__device__ __forceinline__ void bgather_block(const double* part, int64_t blk0, int nblk_sub, double* scratch,
                                              double* out) {
  constexpr int G = kBT / KB;
  __threadfence();
  const int c = threadIdx.x % KB, g = threadIdx.x / KB;
  double s[NP];
#pragma unroll
  for (int k = 0; k < NP; ++k) s[k] = 0.0;
#pragma unroll 4
  for (int j = g; j < nblk_sub; j += G)
#pragma unroll
    for (int k = 0; k < NP; ++k) s[k] += __ldcg(part + (blk0 + j) * NP * KB + k * KB + c);
#pragma unroll
  for (int k = 0; k < NP; ++k) scratch[(g * NP + k) * KB + c] = s[k];
  __syncthreads();
  if (threadIdx.x < NP * KB) {
    const int k = threadIdx.x / KB, cc = threadIdx.x % KB;
    double t = 0.0;
    for (int gg = 0; gg < G; ++gg) t += scratch[(gg * NP + k) * KB + cc];
    out[threadIdx.x] = t;
  }
  __syncthreads();
}

enum { MODE_CG = 0, MODE_WARM = 1, MODE_RESID = 2 };

// One warp per row (see below).  Per-candidate dot partials
// reduced over the block's warps in a fixed order.
template <int MODE, int KB>
__global__ void __launch_bounds__(kBT, 3) kb_spmm(BatchDev D, BState* __restrict__ st, uint32_t* __restrict__ cnt,
                                               const int32_t* __restrict__ nact, const int64_t* __restrict__ sub_blk0,
                                               const int32_t* __restrict__ sub_nblk, const double* __restrict__ X,
                                               double* __restrict__ Y, double* __restrict__ R, double* __restrict__ P,
                                               const double* __restrict__ lam, double* __restrict__ wif,
                                               double* __restrict__ part, double tol, int32_t* __restrict__ nactive,
                                               int64_t blk_base = 0) {
  constexpr int NP = MODE == MODE_WARM ? 3 : 1;
  __shared__ double wsum[kBT / 32][NP][KB];
  __shared__ double sm[NP * KB];
  const int64_t blk = blockIdx.x + blk_base;
  const int ls = D.blk_sub[blk];
  if (MODE == MODE_CG && nact[ls] == 0) return;
  // One warp per row, split in two half-warps h = lane / 16: half h takes the row's nonzeros
  // h, h+2, h+4, ...; lane t = lane % 16 owns the CPT = KB/16 contiguous candidates
  // [CPT t, CPT t + CPT), so every gather is one coalesced KB*8-byte row in 16-byte loads
  // and each warp instruction serves two nonzeros.  The kernel is latency and issue bound:
  // the next row's rowptr and first 32 (val, col) pairs are fetched while the current row's
  // gathers are in flight, GU steps of gathers are issued back to back, and lanes past the
  // row end carry (val, col) = (0, 0) so no step is predicated.  The two half sums are
  // combined by one xor shuffle; the epilogue gives candidate CPT t + CPE h + e to half h.
  constexpr int CPT = KB / 16;
  constexpr int CPE = CPT / 2;
  constexpr int GU = CPT == 2 ? 8 : 4;  // steps (2 nonzeros each) in flight
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int hf = lane >> 4, t16 = lane & 15;
  const int cb = CPT * t16;            // first gathered candidate of this lane
  const int eb = CPT * t16 + CPE * hf; // first epilogue candidate of this lane
  bool act[CPE];
#pragma unroll
  for (int e = 0; e < CPE; ++e)
    act[e] = MODE == MODE_CG ? (bool)st[ls * KB + eb + e].active : (bool)D.cand_active[eb + e];
  double acc[CPE][NP];
#pragma unroll
  for (int e = 0; e < CPE; ++e)
#pragma unroll
    for (int k = 0; k < NP; ++k) acc[e][k] = 0.0;
  auto gather = [&](const double* rowp, double (&v)[CPT]) {
    const double2* q = reinterpret_cast<const double2*>(rowp + cb);
#pragma unroll
    for (int h = 0; h < CPT / 2; ++h) {
      const double2 w = q[h];
      v[2 * h] = w.x;
      v[2 * h + 1] = w.y;
    }
  };
  // y += sum over the chunk's nonzeros (lane-held (v, c), zero past the end) of v X[c]
  auto chunk = [&](double v, int c, int m, double (&y)[CPT]) {
#pragma unroll 1
    for (int j0 = 0; j0 < m; j0 += 2 * GU) {
      double xv[GU][CPT];
#pragma unroll
      for (int u = 0; u < GU; ++u) gather(X + (int64_t)__shfl_sync(0xffffffffu, c, j0 + 2 * u + hf) * KB, xv[u]);
#pragma unroll
      for (int u = 0; u < GU; ++u) {
        const double vj = __shfl_sync(0xffffffffu, v, j0 + 2 * u + hf);
#pragma unroll
        for (int j = 0; j < CPT; ++j) y[j] = fma(vj, xv[u][j], y[j]);
      }
    }
  };
  auto halves = [&](double (&y)[CPT], double (&ye)[CPE]) {  // full sums of the epilogue candidates
#pragma unroll
    for (int j = 0; j < CPT; ++j) y[j] += __shfl_xor_sync(0xffffffffu, y[j], 16);
#pragma unroll
    for (int e = 0; e < CPE; ++e) ye[e] = hf ? y[CPE + e] : y[e];
  };
  const int64_t row0 = D.blk_row0[blk];
  const int nrow = D.blk_nrow[blk];
  int64_t nbeg = 0, nend = 0;  // prefetch state of the warp's next row
  double nv = 0.0;
  int nc = 0;
  auto fetch = [&](int rr) {
    if (rr < nrow) {
      nbeg = D.rowptr[row0 + rr];
      nend = D.rowptr[row0 + rr + 1];
      nv = 0.0;
      nc = 0;
      if (nbeg + lane < nend) {
        nv = D.val[nbeg + lane];
        nc = D.col[nbeg + lane];
      }
    }
  };
  fetch(warp);
  for (int rr = warp; rr < nrow; rr += kBT / 32) {
    const int64_t row = row0 + rr;
    const int64_t beg = nbeg, end = nend;
    const double v0 = nv;
    const int c0 = nc;
    const int sl = D.islot[row];
    const int64_t er = row * KB;
    double pv[CPE];
    if (MODE == MODE_CG) {
#pragma unroll
      for (int e = 0; e < CPE; ++e) pv[e] = X[er + eb + e];
    }
    fetch(rr + kBT / 32);
    double y[CPT];
#pragma unroll
    for (int j = 0; j < CPT; ++j) y[j] = 0.0;
    chunk(v0, c0, end - beg < 32 ? (int)(end - beg) : 32, y);
    for (int64_t k0 = beg + 32; k0 < end; k0 += 32) {  // rows longer than 32
      double v = 0.0;
      int c = 0;
      if (k0 + lane < end) {
        v = D.val[k0 + lane];
        c = D.col[k0 + lane];
      }
      chunk(v, c, end - k0 < 32 ? (int)(end - k0) : 32, y);
    }
    double ye[CPE];
    halves(y, ye);
    if (MODE != MODE_RESID && sl >= 0) {  // + (p_b M_Gamma + q_b S_Gamma) X on the interface rows
      const int side = sl / (int)D.nG, g = sl % (int)D.nG;
      const int mb = D.mrow[g], me = D.mrow[g + 1];  // at most 19 entries: one chunk
      double mv = 0.0, sv = 0.0;
      int cr = 0;
      if (mb + lane < me) {
        mv = D.mval[mb + lane];
        sv = D.sval[mb + lane];
        cr = D.mcolg[(int64_t)side * D.nnzM + mb + lane];
      }
      double mm[CPT], ss[CPT], me2[CPE], se2[CPE];
#pragma unroll
      for (int j = 0; j < CPT; ++j) mm[j] = ss[j] = 0.0;
      chunk(mv, cr, me - mb, mm);
      chunk(sv, cr, me - mb, ss);
      halves(mm, me2);
      halves(ss, se2);
#pragma unroll
      for (int e = 0; e < CPE; ++e)
        ye[e] += fma(D.alpha_own[side * KB + eb + e], me2[e], D.q_own[side * KB + eb + e] * se2[e]);
    }
    if (MODE == MODE_CG) {
#pragma unroll
      for (int e = 0; e < CPE; ++e) {
        Y[er + eb + e] = ye[e];
        if (act[e]) acc[e][0] += pv[e] * ye[e];
      }
    } else if (MODE == MODE_WARM) {
      const double bv = D.b[row];
#pragma unroll
      for (int e = 0; e < CPE; ++e) {
        const int bj = eb + e;
        const double rhs = sl >= 0 ? bv + lam[(int64_t)sl * KB + bj] : bv;
        const double rj = rhs - ye[e];
        const double zj = dinv_b<KB>(D, row, sl, bj) * rj;
        if (act[e]) {
          R[er + bj] = rj;
          P[er + bj] = zj;
          acc[e][0] += rj * zj;
          acc[e][1] += rj * rj;
          acc[e][2] += rhs * rhs;
        }
      }
    } else {  // MODE_RESID: w = b - K^N u~
      const double bv = D.b[row];
#pragma unroll
      for (int e = 0; e < CPE; ++e) {
        const double w = bv - ye[e];
        if (sl >= 0) {
          wif[(int64_t)sl * KB + eb + e] = w;
        } else if (act[e]) {
          acc[e][0] += w * w;
        }
      }
    }
  }
#pragma unroll
  for (int e = 0; e < CPE; ++e)
#pragma unroll
    for (int k = 0; k < NP; ++k) wsum[warp][k][eb + e] = acc[e][k];
  __syncthreads();
  for (int i = threadIdx.x; i < NP * KB; i += kBT) {
    double s = 0.0;
    for (int w = 0; w < kBT / 32; ++w) s += wsum[w][i / KB][i % KB];
    sm[i] = s;
  }
  __syncthreads();
  const int64_t sb0 = sub_blk0[ls];
  const int snb = sub_nblk[ls];
  if (bpublish<KB>(part, blk, NP, sm, cnt + ls, snb)) {
    const int t = threadIdx.x;
    bgather_block<KB, NP>(part, sb0, snb, &wsum[0][0][0], sm);
    double tot[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) tot[k] = t < KB ? sm[k * KB + t] : 0.0;
    if (t < KB) {
      BState& S = st[ls * KB + t];
      if (MODE == MODE_CG) {
        if (S.active) {
          if (!(tot[0] > 0.0) || !isfinite(tot[0])) {
            S.status = 3;
            S.active = 0;
            atomicSub(nactive, 1);
            atomicSub((int32_t*)&nact[ls], 1);
          } else {
            S.alpha = S.rho / tot[0];
          }
        }
      } else if (MODE == MODE_WARM) {
        if (D.cand_active[t]) {
          S.rho = tot[0];
          S.rr = tot[1];
          S.bb = tot[2];
          S.iters = 0;
          S.zero_rhs = tot[2] == 0.0;
          if (tot[2] == 0.0 || sqrt(tot[1]) <= tol * sqrt(tot[2])) {
            S.status = 1;
            S.active = 0;
          } else {
            S.status = 0;
            S.active = 1;
            atomicAdd(nactive, 1);
            atomicAdd((int32_t*)&nact[ls], 1);
          }
        } else {
          S.active = 0;
        }
      } else {
        S.resid = tot[0];
      }
    }
    if (t == 0) cnt[ls] = 0;
  }
}

// x += alpha p ; r -= alpha q ; z = D_b^{-1} r ; r.z, r.r ; stop test ; beta.  mode 1: p = z + beta p.
template <int MODE, int KB>
__global__ void __launch_bounds__(kBT) kb_vec(BatchDev D, BState* __restrict__ st, uint32_t* __restrict__ cnt,
                                              int32_t* __restrict__ nact, const int64_t* __restrict__ sub_blk0,
                                              const int32_t* __restrict__ sub_nblk, double* __restrict__ x,
                                              double* __restrict__ r, double* __restrict__ p,
                                              const double* __restrict__ q, double* __restrict__ part, double tol,
                                              int maxit, int32_t* __restrict__ nactive, int64_t blk_base) {
  __shared__ double red[kBT / KB][2][KB];
  __shared__ double sm[2 * KB];
  const int64_t blk = blockIdx.x + blk_base;
  const int ls = D.blk_sub[blk];
  if (nact[ls] == 0) return;
  const int b = threadIdx.x % KB, rg = threadIdx.x / KB;
  const BState S0 = st[ls * KB + b];
  const bool act = S0.active;
  const int64_t row0 = D.blk_row0[blk];
  const int nrow = D.blk_nrow[blk];
  double a0 = 0.0, a1 = 0.0;
  if (act) {
#pragma unroll 4
    for (int rr = rg; rr < nrow; rr += kBT / KB) {
      const int64_t row = row0 + rr;
      const int64_t e = row * KB + b;
      const int sl = D.islot[row];
      const double di = dinv_b<KB>(D, row, sl, b);
      if (MODE == 0) {
        const double xv = fma(S0.alpha, p[e], x[e]);
        const double rv = fma(-S0.alpha, q[e], r[e]);
        x[e] = xv;
        r[e] = rv;
        a0 += rv * (di * rv);
        a1 += rv * rv;
      } else {
        p[e] = fma(S0.beta, p[e], di * r[e]);
      }
    }
  }
  if (MODE == 1) return;
  red[rg][0][b] = a0;
  red[rg][1][b] = a1;
  __syncthreads();
  if (threadIdx.x < 2 * KB) {
    const int k = threadIdx.x / KB, t = threadIdx.x % KB;
    double s = 0.0;
    for (int g = 0; g < kBT / KB; ++g) s += red[g][k][t];
    sm[threadIdx.x] = s;
  }
  __syncthreads();
  const int64_t sb0 = sub_blk0[ls];
  const int snb = sub_nblk[ls];
  if (bpublish<KB>(part, blk, 2, sm, cnt + ls, snb)) {
    const int t = threadIdx.x;
    bgather_block<KB, 2>(part, sb0, snb, &red[0][0][0], sm);
    if (t < KB) {
      const double rz = sm[t], rr = sm[KB + t];
      BState& S = st[ls * KB + t];
      if (S.active) {
        S.rr = rr;
        S.iters += 1;
        if (sqrt(rr) <= tol * sqrt(S.bb)) {
          S.status = 1;
          S.active = 0;
          atomicSub(nactive, 1);
          atomicSub(&nact[ls], 1);
        } else if (S.iters >= maxit) {
          S.status = 2;
          S.active = 0;
          atomicSub(nactive, 1);
          atomicSub(&nact[ls], 1);
        } else {
          S.beta = rz / S.rho;
          S.rho = rz;
        }
      }
    }
    if (t == 0) cnt[ls] = 0;
  }
}

template <int KB>
__global__ void kb_zero_if(BatchDev D, const BState* __restrict__ st, double* __restrict__ x) {
  const int64_t blk = blockIdx.x;
  const int ls = D.blk_sub[blk];
  const int b = threadIdx.x % KB, rg = threadIdx.x / KB;
  if (!D.cand_active[b] || !st[ls * KB + b].zero_rhs) return;
  for (int rr = rg; rr < D.blk_nrow[blk]; rr += kBT / KB) x[(D.blk_row0[blk] + rr) * KB + b] = 0.0;
}

// Robin data out of every side: g = (alpha_s + alpha_t) M u|Gamma - lambda, and u|Gamma.
template <int KB>
__global__ void kb_trace(BatchDev D, const double* __restrict__ x, const double* __restrict__ lam,
                         double* __restrict__ out) {
  const int k = blockIdx.y;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= D.nG * KB) return;
  const int64_t g = i / KB;
  const int b = (int)(i % KB);
  if (!D.cand_active[b]) return;
  const double ps = D.alpha_sum[k * KB + b], qs = D.q_sum[k * KB + b];
  double mu = 0.0;
  for (int j = D.mrow[g]; j < D.mrow[g + 1]; ++j)
    mu = fma(fma(ps, D.mval[j], qs * D.sval[j]), x[(int64_t)D.mcolg[k * D.nnzM + j] * KB + b], mu);
  double* o = out + (int64_t)k * 3 * D.nG * KB;
  o[i] = mu - lam[(int64_t)k * D.nG * KB + i];
  o[D.nG * KB + i] = x[(int64_t)D.mapg[k * D.nG + g] * KB + b];
}

template <int KB>
__global__ void kb_accept(BatchDev D, const double* __restrict__ out, double* __restrict__ lam,
                          double* __restrict__ unbr) {
  const int k = blockIdx.y;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= D.nG * KB) return;
  if (!D.cand_active[i % KB]) return;
  const double* in = out + (int64_t)D.side_partner[k] * 3 * D.nG * KB;
  lam[(int64_t)k * D.nG * KB + i] = in[i];
  unbr[(int64_t)k * D.nG * KB + i] = in[D.nG * KB + i];
}

template <int KB>
__global__ void kb_glue(BatchDev D, int64_t nrows, const double* __restrict__ x, const double* __restrict__ unbr,
                        double* __restrict__ ut) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nrows * KB) return;
  const int64_t row = i / KB;
  const int sl = D.islot[row];
  ut[i] = sl >= 0 ? 0.5 * (x[i] + unbr[(int64_t)sl * KB + i % KB]) : x[i];
}

// Owner side (left slab) of every interface: sum_g (w_s + w_t)^2 per candidate; one block per side.
template <int KB>
__global__ void __launch_bounds__(kBT) kb_iface_sum(BatchDev D, const double* __restrict__ wif,
                                                    double* __restrict__ side_sum) {
  __shared__ double red[kBT / KB][KB];
  const int k = blockIdx.x;
  const int b = threadIdx.x % KB, rg = threadIdx.x / KB;
  if (D.side_which[k] != 0) return;
  const int pk = D.side_partner[k];
  double s = 0.0;
  for (int64_t g = rg; g < D.nG; g += kBT / KB) {
    const double w = wif[((int64_t)k * D.nG + g) * KB + b] + wif[((int64_t)pk * D.nG + g) * KB + b];
    s += w * w;
  }
  red[rg][b] = s;
  __syncthreads();
  if (threadIdx.x < KB) {
    double t = 0.0;
    for (int g = 0; g < kBT / KB; ++g) t += red[g][threadIdx.x];
    side_sum[k * KB + threadIdx.x] = t;
  }
}

__global__ void kb_gather_b(int64_t npad, int64_t row0, const int32_t* __restrict__ perm, const double* __restrict__ bi,
                            int64_t rc0, double* __restrict__ bc) {
  const int64_t ri = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (ri >= npad) return;
  const int c = perm[ri];
  if (c >= 0) bc[rc0 + c] = bi[row0 + ri];
}

template <int KB>
__global__ void kb_extract(int64_t n, int64_t rc0, int b, const double* __restrict__ x, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = x[(rc0 + i) * KB + b];
}

int64_t nG_nnz(const Ctx& c) { return c.nG ? (int64_t)c.h_mrow[c.nG] : 0; }

template <class T>
T* balloc(int64_t n) {
  void* p = nullptr;
  OSM_CUDA(cudaMalloc(&p, sizeof(T) * (size_t)std::max<int64_t>(1, n)));
  return (T*)p;
}

}  // namespace

void batch_free(Ctx& c) {
  BatchBuf* B = c.batch;
  if (!B) return;
  void* ptrs[] = {B->rowptr, B->col, B->val, B->dkn, B->b, B->islot, B->blk_sub, B->blk_nrow, B->blk_row0, B->mapg, B->mcolg,
                  B->mdiag, B->sdiag, B->q_own, B->q_sum, B->alpha_own, B->alpha_sum, B->side_which, B->side_partner, B->cand_active, B->x, B->r,
                  B->p, B->q, B->ut, B->lam, B->unbr, B->wif, B->out, B->st, B->cnt, B->nact, B->d_nactive,
                  B->part, B->part_v, B->side_sum};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete B;
  c.batch = nullptr;
  if (c.batch_sub_blk0) cudaFree(c.batch_sub_blk0);
  if (c.batch_sub_nblk) cudaFree(c.batch_sub_nblk);
  c.batch_sub_blk0 = nullptr;
  c.batch_sub_nblk = nullptr;
}

static void batch_setup(Ctx& c) {
  if (c.batch) return;
  auto* B = new BatchBuf();
  c.batch = B;
  const int nloc = c.s_end - c.s_begin;
  // Concatenated contract CSR of K^N over the local subdomains, without its exact-zero entries (the
  // Kuhn stencil's structural zeros, ~19 % of P2 entries: they add +-0 to every candidate's row sum).
  int64_t nrows = 0;
  B->rc0.resize(nloc + 1);
  for (int ls = 0; ls < nloc; ++ls) {
    B->rc0[ls] = nrows;
    nrows += c.subs[ls].n;
  }
  B->rc0[nloc] = nrows;
  B->nrows = nrows;
  std::vector<int64_t> hrp(1, 0);
  std::vector<int32_t> hcol;
  std::vector<double> hval, hdkn(nrows, 0.0);
  for (int ls = 0; ls < nloc; ++ls) {
    const Sub& S = c.subs[ls];
    std::vector<int64_t> rp(S.n + 1);
    std::vector<int32_t> cl(S.nnz);
    std::vector<double> vl(S.nnz);
    OSM_CUDA(cudaMemcpy(rp.data(), S.rowptr, sizeof(int64_t) * (S.n + 1), cudaMemcpyDeviceToHost));
    OSM_CUDA(cudaMemcpy(cl.data(), S.col, sizeof(int32_t) * S.nnz, cudaMemcpyDeviceToHost));
    OSM_CUDA(cudaMemcpy(vl.data(), S.val, sizeof(double) * S.nnz, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < S.n; ++i) {
      for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
        if (cl[k] == i) hdkn[B->rc0[ls] + i] = vl[k];
        if (vl[k] == 0.0) continue;
        hcol.push_back((int32_t)(B->rc0[ls] + cl[k]));
        hval.push_back(vl[k]);
      }
      hrp.push_back((int64_t)hcol.size());
    }
  }
  B->nnz = (int64_t)hcol.size();
  auto upload = [&](const auto& v, auto*& d) {
    using T = typename std::decay<decltype(v)>::type::value_type;
    d = balloc<T>((int64_t)v.size());
    OSM_CUDA(cudaMemcpy(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
  };
  upload(hrp, B->rowptr);
  upload(hcol, B->col);
  upload(hval, B->val);
  upload(hdkn, B->dkn);
  B->b = balloc<double>(nrows);
  // blocks of kRB rows, never straddling subdomains
  std::vector<int32_t> bsub, bnrow;
  std::vector<int64_t> brow0, sblk0;
  std::vector<int32_t> snblk;
  int64_t rb = kRB;
  if (const char* e = std::getenv("OSM_BATCH_RB")) rb = std::max(64, std::atoi(e));  // experiment knob
  for (int ls = 0; ls < nloc; ++ls) {
    sblk0.push_back((int64_t)bsub.size());
    const int64_t n = c.subs[ls].n;
    int cnt = 0;
    for (int64_t r0 = 0; r0 < n; r0 += rb) {
      bsub.push_back(ls);
      brow0.push_back(B->rc0[ls] + r0);
      bnrow.push_back((int32_t)std::min<int64_t>(rb, n - r0));
      ++cnt;
    }
    snblk.push_back(cnt);
  }
  B->nblk = (int64_t)bsub.size();
  auto up = [&](auto& v, auto*& d) {
    using T = typename std::decay<decltype(v)>::type::value_type;
    d = balloc<T>((int64_t)v.size());
    OSM_CUDA(cudaMemcpyAsync(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, c.stream));
  };
  up(bsub, B->blk_sub);
  up(bnrow, B->blk_nrow);
  up(brow0, B->blk_row0);
  int64_t* d_sblk0 = nullptr;
  int32_t* d_snblk = nullptr;
  up(sblk0, d_sblk0);
  up(snblk, d_snblk);
  c.batch_sub_blk0 = d_sblk0;
  c.batch_sub_nblk = d_snblk;
  // interface slots in contract order and side tables
  const int nsides = (int)c.sides.size();
  const int64_t nG = c.nG;
  std::vector<int32_t> islot(nrows, -1), mapg((size_t)std::max<int64_t>(1, nsides * nG)), which(std::max(1, nsides)),
      partner(std::max(1, nsides));
  for (int k = 0; k < nsides; ++k) {
    const Side& sd = c.sides[k];
    std::vector<int32_t> mc(nG);
    OSM_CUDA(cudaMemcpy(mc.data(), sd.map_c, sizeof(int32_t) * nG, cudaMemcpyDeviceToHost));
    for (int64_t g = 0; g < nG; ++g) {
      mapg[k * nG + g] = (int32_t)(B->rc0[sd.sub] + mc[g]);
      islot[B->rc0[sd.sub] + mc[g]] = (int32_t)(k * nG + g);
    }
    which[k] = sd.which;
    partner[k] = sd.partner;
  }
  up(islot, B->islot);
  up(mapg, B->mapg);
  {
    const int64_t nm = nG_nnz(c);
    std::vector<int32_t> mcg((size_t)std::max<int64_t>(1, nsides * nm));
    for (int k = 0; k < nsides; ++k)
      for (int64_t j = 0; j < nm; ++j) mcg[k * nm + j] = mapg[k * nG + c.h_mcol[j]];
    up(mcg, B->mcolg);
  }
  up(which, B->side_which);
  up(partner, B->side_partner);
  std::vector<double> md(std::max<int64_t>(1, nG), 0.0), sd(std::max<int64_t>(1, nG), 0.0);
  for (int64_t g = 0; g < nG; ++g)
    for (int j = c.h_mrow[g]; j < c.h_mrow[g + 1]; ++j)
      if (c.h_mcol[j] == g) {
        md[g] = c.h_mval[j];
        sd[g] = c.h_sval[j];
      }
  up(md, B->mdiag);
  up(sd, B->sdiag);
  B->alpha_own = balloc<double>(std::max(1, nsides) * kBmax);
  B->alpha_sum = balloc<double>(std::max(1, nsides) * kBmax);
  B->q_own = balloc<double>(std::max(1, nsides) * kBmax);
  B->q_sum = balloc<double>(std::max(1, nsides) * kBmax);
  B->cand_active = balloc<int32_t>(kBmax);
  const int64_t nv = nrows * kBmax;
  B->x = balloc<double>(nv);
  B->r = balloc<double>(nv);
  B->p = balloc<double>(nv);
  B->q = balloc<double>(nv);
  B->ut = balloc<double>(nv);
  const int64_t ns = std::max<int64_t>(1, nsides * nG * kBmax);
  B->lam = balloc<double>(ns);
  B->unbr = balloc<double>(ns);
  B->wif = balloc<double>(ns);
  B->out = balloc<double>(3 * ns);
  B->st = balloc<BState>(nloc * kBmax);
  B->cnt = balloc<uint32_t>(nloc);
  B->nact = balloc<int32_t>(nloc);
  B->d_nactive = balloc<int32_t>(1);
  B->part = balloc<double>(B->nblk * 3 * kBmax);
  B->part_v = balloc<double>(B->nblk * 2 * kBmax);
  B->sblk0_h = sblk0;
  B->nblk_h = B->nblk;
  B->side_sum = balloc<double>(std::max(1, nsides) * kBmax);
  for (double* v : {B->x, B->r, B->p, B->q, B->ut}) OSM_CUDA(cudaMemsetAsync(v, 0, sizeof(double) * nv, c.stream));
  OSM_CUDA(cudaMemsetAsync(B->cnt, 0, sizeof(uint32_t) * nloc, c.stream));
  OSM_CUDA(cudaMemsetAsync(B->st, 0, sizeof(BState) * nloc * kBmax, c.stream));
  OSM_CUDA(cudaMemsetAsync(B->side_sum, 0, sizeof(double) * std::max(1, nsides) * kBmax, c.stream));
  OSM_CUDA(cudaStreamSynchronize(c.stream));
}

static BatchDev batch_view(const Ctx& c) {
  const BatchBuf* B = c.batch;
  BatchDev D{};
  D.rowptr = B->rowptr;
  D.col = B->col;
  D.val = B->val;
  D.dkn = B->dkn;
  D.islot = B->islot;
  D.b = B->b;
  D.blk_sub = B->blk_sub;
  D.blk_row0 = B->blk_row0;
  D.blk_nrow = B->blk_nrow;
  D.mapg = B->mapg;
  D.mrow = c.d_mrow;
  D.mcol = c.d_mcol;
  D.mcolg = B->mcolg;
  D.nnzM = nG_nnz(c);
  D.mval = c.d_mval;
  D.sval = c.d_sval;
  D.mdiag = B->mdiag;
  D.sdiag = B->sdiag;
  D.alpha_own = B->alpha_own;
  D.alpha_sum = B->alpha_sum;
  D.q_own = B->q_own;
  D.q_sum = B->q_sum;
  D.side_which = B->side_which;
  D.side_partner = B->side_partner;
  D.cand_active = B->cand_active;
  D.nG = c.nG;
  D.nsides = (int)c.sides.size();
  return D;
}

template <int KB>
static osm_status solve_batch_kb(Ctx& c, int nB, const double* pq, const osm_solve_opts& o, osm_batch_report* rep,
                                 std::chrono::steady_clock::time_point t0);

osm_status solve_batch(Ctx& c, int nB, const double* pq, const osm_solve_opts& o, osm_batch_report* rep) {
  if (!c.assembled || !c.density_set) fail(OSM_ERR_STATE, "assemble and upload a density before osm_solve_batch");
  if (c.nranks != 1) fail(OSM_ERR_INVALID_ARG, "osm_solve_batch runs on a single rank");
  if (nB < 1 || nB > kBmax) fail(OSM_ERR_INVALID_ARG, "need 1 <= B <= 64");
  if (c.nsub > 1 && !pq) fail(OSM_ERR_INVALID_ARG, "NULL coefficients");
  const int ni = c.nsub - 1;
  // pq: [b][4][iface] = p_left, q_left, p_right, q_right
  for (int i = 0; i < nB * 4 * ni; ++i)
    if (!(pq[i] >= 0) || !std::isfinite(pq[i])) fail(OSM_ERR_ILL_POSED, "coefficients must be finite and >= 0");
  for (int bb = 0; bb < nB; ++bb)
    for (int i = 0; i < ni; ++i)
      if (pq[(bb * 4 + 0) * ni + i] == 0 && pq[(bb * 4 + 2) * ni + i] == 0)
        fail(OSM_ERR_ILL_POSED, "p = 0 on both sides of an interface");
  const auto t0 = std::chrono::steady_clock::now();
  batch_setup(c);
  // Candidate stride: 32 halves every gather and vector stream when the population fits.
  if (nB <= 32) return solve_batch_kb<32>(c, nB, pq, o, rep, t0);
  return solve_batch_kb<64>(c, nB, pq, o, rep, t0);
}

template <int KB>
static osm_status solve_batch_kb(Ctx& c, int nB, const double* pq, const osm_solve_opts& o, osm_batch_report* rep,
                                 std::chrono::steady_clock::time_point t0) {
  const int ni = c.nsub - 1;
  BatchBuf* B = c.batch;
  B->KB = KB;
  const int nloc = c.s_end - c.s_begin;
  const int nsides = (int)c.sides.size();
  const int64_t nG = c.nG;
  // alpha per side per candidate
  std::vector<double> aown(std::max(1, nsides) * KB, 0.0), asum(std::max(1, nsides) * KB, 0.0);
  std::vector<double> qown(std::max(1, nsides) * KB, 0.0), qsum(std::max(1, nsides) * KB, 0.0);
  for (int k = 0; k < nsides; ++k)
    for (int bb = 0; bb < nB; ++bb) {
      const int i = c.sides[k].iface;
      const double pl = pq[(bb * 4 + 0) * ni + i], ql = pq[(bb * 4 + 1) * ni + i];
      const double pr = pq[(bb * 4 + 2) * ni + i], qr = pq[(bb * 4 + 3) * ni + i];
      aown[k * KB + bb] = c.sides[k].which == 0 ? pl : pr;
      qown[k * KB + bb] = c.sides[k].which == 0 ? ql : qr;
      asum[k * KB + bb] = pl + pr;
      qsum[k * KB + bb] = ql + qr;
    }
  OSM_CUDA(cudaMemcpyAsync(B->alpha_own, aown.data(), sizeof(double) * aown.size(), cudaMemcpyHostToDevice, c.stream));
  OSM_CUDA(cudaMemcpyAsync(B->alpha_sum, asum.data(), sizeof(double) * asum.size(), cudaMemcpyHostToDevice, c.stream));
  OSM_CUDA(cudaMemcpyAsync(B->q_own, qown.data(), sizeof(double) * qown.size(), cudaMemcpyHostToDevice, c.stream));
  OSM_CUDA(cudaMemcpyAsync(B->q_sum, qsum.data(), sizeof(double) * qsum.size(), cudaMemcpyHostToDevice, c.stream));
  // load vector in contract order (from the single-candidate internal b)
  for (int ls = 0; ls < nloc; ++ls) {
    const Sub& S = c.subs[ls];
    kb_gather_b<<<(unsigned)ceil_div(S.npad, 256), 256, 0, c.stream>>>(S.npad, S.row0, S.perm, c.b, B->rc0[ls], B->b);
    OSM_CHECK_LAUNCH();
    ++c.launches;
  }
  const double fnorm2 = fnorm2_of(c);
  const double fnorm = std::sqrt(fnorm2);
  const int64_t nv = B->nrows * KB;
  OSM_CUDA(cudaMemsetAsync(B->x, 0, sizeof(double) * nv, c.stream));
  if (nsides) OSM_CUDA(cudaMemsetAsync(B->lam, 0, sizeof(double) * nsides * nG * KB, c.stream));
  if (nsides) OSM_CUDA(cudaMemsetAsync(B->unbr, 0, sizeof(double) * nsides * nG * KB, c.stream));
  std::vector<int32_t> cand(KB, 0);
  for (int bb = 0; bb < nB; ++bb) cand[bb] = 1;
  B->B = nB;
  B->hist.assign(nB, {});
  B->inner.assign(nB, {});
  std::vector<BState> hst(nloc * KB);
  std::vector<double> hside(std::max(1, nsides) * KB);
  BatchDev D = batch_view(c);
  const unsigned nblk = (unsigned)B->nblk;
  const dim3 gI((unsigned)ceil_div(nG * KB, 256), (unsigned)std::max(1, nsides));
  int64_t inner_total = 0;
  int n_conv = 0, outer_max = 0;
  constexpr int kChunk = 8;
  for (int n = 1; n <= o.max_outer; ++n) {
    OSM_CUDA(cudaMemcpyAsync(B->cand_active, cand.data(), sizeof(int32_t) * KB, cudaMemcpyHostToDevice, c.stream));
    if (!o.warm_start) OSM_CUDA(cudaMemsetAsync(B->x, 0, sizeof(double) * nv, c.stream));
    OSM_CUDA(cudaMemsetAsync(B->d_nactive, 0, sizeof(int32_t), c.stream));
    OSM_CUDA(cudaMemsetAsync(B->nact, 0, sizeof(int32_t) * nloc, c.stream));
    kb_spmm<MODE_WARM, KB><<<nblk, kBT, 0, c.stream>>>(D, B->st, B->cnt, B->nact, c.batch_sub_blk0, c.batch_sub_nblk, B->x,
                                                   nullptr, B->r, B->p, B->lam, nullptr, B->part, o.tol_inner,
                                                   B->d_nactive);
    kb_zero_if<KB><<<nblk, kBT, 0, c.stream>>>(D, B->st, B->x);
    OSM_CHECK_LAUNCH();
    c.launches += 2;
    OSM_CUDA(cudaMemcpyAsync(&c.h_nactive[0], B->d_nactive, sizeof(int32_t), cudaMemcpyDeviceToHost, c.stream));
    OSM_CUDA(cudaStreamSynchronize(c.stream));
    if (c.h_nactive[0] > 0) {
      // subdomain groups on the library's group streams (as osm_solve): one group's kernels fill the
      // others' wave tails; the first group's stream joins the rest after every chunk
      const int G = std::min(std::min(c.want_groups, nloc), Ctx::kMaxGroups);
      cudaStream_t ps = c.stream;
      if (G > 1) {
        OSM_CUDA(cudaEventRecord(c.ev_fork, c.stream));
        for (int g = 0; g < G; ++g) OSM_CUDA(cudaStreamWaitEvent(c.gstream[g], c.ev_fork, 0));
        ps = c.gstream[0];
      }
      int ch = 0;
      for (;; ++ch) {
        for (int g = 0; g < G; ++g) {
          const int s0 = g * nloc / G, s1 = (g + 1) * nloc / G;
          const int64_t b0 = B->sblk0_h[s0], b1 = s1 < nloc ? B->sblk0_h[s1] : B->nblk_h;
          const unsigned gb = (unsigned)(b1 - b0);
          cudaStream_t gs = G > 1 ? c.gstream[g] : c.stream;
          for (int it = 0; it < kChunk; ++it) {
            kb_spmm<MODE_CG, KB><<<gb, kBT, 0, gs>>>(D, B->st, B->cnt, B->nact, c.batch_sub_blk0, c.batch_sub_nblk,
                                                     B->p, B->q, nullptr, nullptr, nullptr, nullptr, B->part,
                                                     o.tol_inner, B->d_nactive, b0);
            kb_vec<0, KB><<<gb, kBT, 0, gs>>>(D, B->st, B->cnt, B->nact, c.batch_sub_blk0, c.batch_sub_nblk, B->x,
                                              B->r, B->p, B->q, B->part_v, o.tol_inner, o.max_inner, B->d_nactive, b0);
            kb_vec<1, KB><<<gb, kBT, 0, gs>>>(D, B->st, B->cnt, B->nact, c.batch_sub_blk0, c.batch_sub_nblk, B->x,
                                              B->r, B->p, B->q, B->part_v, o.tol_inner, o.max_inner, B->d_nactive, b0);
          }
          if (G > 1 && g > 0) {
            OSM_CUDA(cudaEventRecord(c.ev_join[g], gs));
            OSM_CUDA(cudaStreamWaitEvent(ps, c.ev_join[g], 0));
          }
        }
        OSM_CHECK_LAUNCH();
        c.launches += 3 * kChunk * G;
        OSM_CUDA(cudaMemcpyAsync(&c.h_nactive[ch & 1], B->d_nactive, sizeof(int32_t), cudaMemcpyDeviceToHost, ps));
        OSM_CUDA(cudaEventRecord(c.ev_chunk[ch & 1], ps));
        if (ch > 0) {
          OSM_CUDA(cudaEventSynchronize(c.ev_chunk[(ch - 1) & 1]));
          if (c.h_nactive[(ch - 1) & 1] == 0) break;
        }
        if ((int64_t)ch * kChunk > (int64_t)o.max_inner + 2 * kChunk) break;
      }
      if (G > 1) OSM_CUDA(cudaStreamWaitEvent(c.stream, c.ev_chunk[ch & 1], 0));
    }
    if (nsides) {
      kb_trace<KB><<<gI, 256, 0, c.stream>>>(D, B->x, B->lam, B->out);
      kb_accept<KB><<<gI, 256, 0, c.stream>>>(D, B->out, B->lam, B->unbr);
      c.launches += 2;
    }
    kb_glue<KB><<<(unsigned)ceil_div(nv, 256), 256, 0, c.stream>>>(D, B->nrows, B->x, B->unbr, B->ut);
    kb_spmm<MODE_RESID, KB><<<nblk, kBT, 0, c.stream>>>(D, B->st, B->cnt, B->nact, c.batch_sub_blk0, c.batch_sub_nblk,
                                                    B->ut, nullptr, nullptr, nullptr, nullptr, B->wif, B->part,
                                                    o.tol_inner, B->d_nactive);
    c.launches += 2;
    if (nsides) {
      kb_iface_sum<KB><<<(unsigned)nsides, kBT, 0, c.stream>>>(D, B->wif, B->side_sum);
      ++c.launches;
    }
    OSM_CHECK_LAUNCH();
    OSM_CUDA(cudaMemcpyAsync(hst.data(), B->st, sizeof(BState) * nloc * KB, cudaMemcpyDeviceToHost, c.stream));
    if (nsides)
      OSM_CUDA(cudaMemcpyAsync(hside.data(), B->side_sum, sizeof(double) * nsides * KB, cudaMemcpyDeviceToHost,
                               c.stream));
    OSM_CUDA(cudaStreamSynchronize(c.stream));
    bool any = false;
    for (int bb = 0; bb < nB; ++bb) {
      if (!cand[bb]) continue;
      double r2 = 0.0;
      for (int ls = 0; ls < nloc; ++ls) {
        double v = hst[ls * KB + bb].resid;
        const int k = c.subs[ls].side[1];
        if (k >= 0) v += hside[k * KB + bb];
        r2 += v;
      }
      const double h = fnorm > 0 ? std::sqrt(r2) / fnorm : std::sqrt(r2);
      B->hist[bb].push_back(h);
      for (int ls = 0; ls < nloc; ++ls) {
        B->inner[bb].push_back(hst[ls * KB + bb].iters);
        inner_total += hst[ls * KB + bb].iters;
      }
      outer_max = std::max(outer_max, n);
      if (h <= o.tol_outer) {
        cand[bb] = 0;
        ++n_conv;
      } else if (!std::isfinite(h)) {
        cand[bb] = 0;
      } else {
        any = true;
      }
    }
    if (!any) break;
  }
  if (rep) {
    rep->B = nB;
    rep->outer_max = outer_max;
    rep->n_converged = n_conv;
    rep->inner_total = inner_total;
    rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  return OSM_OK;
}

void batch_history(const Ctx& c, int b, double* h, int cap, int* n) {
  if (!c.batch || b < 0 || b >= c.batch->B) fail(OSM_ERR_INVALID_ARG, "no such candidate");
  const auto& v = c.batch->hist[b];
  *n = (int)v.size();
  if (h) std::copy(v.begin(), v.begin() + std::min<int>(cap, (int)v.size()), h);
}

void batch_inner(const Ctx& c, int b, int32_t* its, int cap, int* n) {
  if (!c.batch || b < 0 || b >= c.batch->B) fail(OSM_ERR_INVALID_ARG, "no such candidate");
  const auto& v = c.batch->inner[b];
  *n = (int)v.size();
  if (its) std::copy(v.begin(), v.begin() + std::min<int>(cap, (int)v.size()), its);
}

void batch_local_solution(Ctx& c, int b, int s, double* u, int64_t* n) {
  if (!c.batch || b < 0 || b >= c.batch->B) fail(OSM_ERR_INVALID_ARG, "no such candidate");
  if (s < c.s_begin || s >= c.s_end) fail(OSM_ERR_INVALID_ARG, "subdomain not owned by this rank");
  const int ls = s - c.s_begin;
  const int64_t ns = c.subs[ls].n;
  if (!u) {
    *n = ns;
    return;
  }
  if (*n < ns) fail(OSM_ERR_INVALID_ARG, "buffer too small");
  double* d = balloc<double>(ns);
  if (c.batch->KB == 32)
    kb_extract<32><<<(unsigned)ceil_div(ns, 256), 256, 0, c.stream>>>(ns, c.batch->rc0[ls], b, c.batch->x, d);
  else
    kb_extract<64><<<(unsigned)ceil_div(ns, 256), 256, 0, c.stream>>>(ns, c.batch->rc0[ls], b, c.batch->x, d);
  OSM_CHECK_LAUNCH();
  ++c.launches;
  OSM_CUDA(cudaMemcpyAsync(u, d, sizeof(double) * ns, cudaMemcpyDeviceToHost, c.stream));
  OSM_CUDA(cudaStreamSynchronize(c.stream));
  cudaFree(d);
  *n = ns;
}

}  // namespace osm

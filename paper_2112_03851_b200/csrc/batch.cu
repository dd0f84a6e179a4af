// Batched-alpha optimized Schwarz (BASELINE config C4): B candidate
// Robin parameter sets solved simultaneously on one GPU, sharing the Neumann matrices K_s^N.
//
// Each batched PCG iteration reads every K_s^N entry ONCE and applies it to all B
// candidates: vectors are stored [row][candidate] (candidate fastest, stride kB = 64),
// one warp per matrix row, lane l owns candidates 2l and 2l+1, so a column gather is a
// single coalesced 512-byte row of the candidate block.  The candidate-specific Robin
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
#include <cstring>
#include <vector>

#include "ctx.h"

namespace osm {

constexpr int kB = 64;      // candidate stride
constexpr int kRB = 512;    // rows per batched block
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
  const double* mval;
  const double* sval;       // S_Gamma values (OO2), aligned with mval
  const double* mdiag;      // [nG]
  const double* sdiag;      // [nG]
  const double* alpha_own;  // p of the side, [nsides][kB]
  const double* alpha_sum;  // p_s + p_t, [nsides][kB]
  const double* q_own;      // q of the side (OO2), [nsides][kB]
  const double* q_sum;      // q_s + q_t, [nsides][kB]
  const int32_t* side_which;   // [nsides]
  const int32_t* side_partner; // [nsides]
  const int32_t* cand_active;  // [kB]
  int64_t nG;
  int nsides;
};

struct BatchBuf {
  int B = 0;
  int64_t nrows = 0, nblk = 0, nnz = 0;
  int64_t* rowptr = nullptr;
  int32_t* col = nullptr;
  double* val = nullptr;
  double *dkn = nullptr, *b = nullptr;
  int32_t* islot = nullptr;
  int32_t *blk_sub = nullptr, *blk_nrow = nullptr;
  int64_t* blk_row0 = nullptr;
  int32_t* mapg = nullptr;
  double *mdiag = nullptr, *sdiag = nullptr;
  double *alpha_own = nullptr, *alpha_sum = nullptr, *q_own = nullptr, *q_sum = nullptr;
  int32_t *side_which = nullptr, *side_partner = nullptr, *cand_active = nullptr;
  double *x = nullptr, *r = nullptr, *p = nullptr, *q = nullptr, *ut = nullptr;
  double *lam = nullptr, *unbr = nullptr, *wif = nullptr, *out = nullptr;
  BState* st = nullptr;
  uint32_t* cnt = nullptr;
  int32_t* nact = nullptr;      // per local subdomain: active candidates (CG)
  int32_t* d_nactive = nullptr; // total active (s, b)
  double* part = nullptr;       // [nblk][3][kB]
  double* side_sum = nullptr;   // [nsides][kB]
  std::vector<int64_t> rc0;     // contract row offset of each local subdomain
  // results
  std::vector<std::vector<double>> hist;  // [b][n]
  std::vector<std::vector<int32_t>> inner;  // [b][n * nsub + s]
};

namespace {

// dinv of K_b = K^N + p_b M + q_b S on the fly (rounded like the single path's fold)
__device__ __forceinline__ double dinv_b(const BatchDev& D, int64_t row, int sl, int b) {
  double d = D.dkn[row];
  if (sl >= 0) {
    const int k = sl / (int)D.nG, g = sl % (int)D.nG;
    d = __dadd_rn(d, __dadd_rn(__dmul_rn(D.alpha_own[k * kB + b], D.mdiag[g]), __dmul_rn(D.q_own[k * kB + b], D.sdiag[g])));
  }
  return d > 0.0 ? 1.0 / d : 0.0;
}

// Block partials [blk][NP][kB] (thread t < kB of the block holds candidate t's sums in sm);
// returns true in the last block of the subdomain.
__device__ __forceinline__ bool bpublish(double* part, int64_t blk, int NP, const double* sm, uint32_t* cnt,
                                         int nblk_sub) {
  __shared__ bool last;
  for (int i = threadIdx.x; i < NP * kB; i += blockDim.x) part[blk * NP * kB + i] = sm[i];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t prev = atomicAdd(cnt, 1u);
    last = prev == (uint32_t)(nblk_sub - 1);
  }
  __syncthreads();
  return last;
}

// fixed-order sum over the subdomain's blocks, candidate t = threadIdx.x < kB
__device__ __forceinline__ double bgather(const double* part, int64_t blk0, int nblk_sub, int NP, int k, int t) {
  __threadfence();
  double s = 0.0;
  for (int j = 0; j < nblk_sub; ++j) s += __ldcg(part + (blk0 + j) * NP * kB + k * kB + t);
  return s;
}

enum { MODE_CG = 0, MODE_WARM = 1, MODE_RESID = 2 };

// One warp per row, lanes own candidates (2 lane, 2 lane + 1).  Per-candidate dot partials
// reduced over the block's warps in a fixed order.
template <int MODE>
__global__ void __launch_bounds__(kBT) kb_spmm(BatchDev D, BState* __restrict__ st, uint32_t* __restrict__ cnt,
                                               const int32_t* __restrict__ nact, const int64_t* __restrict__ sub_blk0,
                                               const int32_t* __restrict__ sub_nblk, const double* __restrict__ X,
                                               double* __restrict__ Y, double* __restrict__ R, double* __restrict__ P,
                                               const double* __restrict__ lam, double* __restrict__ wif,
                                               double* __restrict__ part, double tol, int32_t* __restrict__ nactive) {
  constexpr int NP = MODE == MODE_WARM ? 3 : 1;
  __shared__ double wsum[kBT / 32][NP][kB];
  __shared__ double sm[NP * kB];
  const int64_t blk = blockIdx.x;
  const int ls = D.blk_sub[blk];
  if (MODE == MODE_CG && nact[ls] == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b0 = 2 * lane, b1 = 2 * lane + 1;
  bool act0, act1;
  if (MODE == MODE_CG) {
    act0 = st[ls * kB + b0].active;
    act1 = st[ls * kB + b1].active;
  } else {
    act0 = D.cand_active[b0];
    act1 = D.cand_active[b1];
  }
  double acc0[NP], acc1[NP];
#pragma unroll
  for (int k = 0; k < NP; ++k) acc0[k] = acc1[k] = 0.0;
  const int64_t row0 = D.blk_row0[blk];
  const int nrow = D.blk_nrow[blk];
  for (int rr = warp; rr < nrow; rr += kBT / 32) {
    const int64_t row = row0 + rr;
    const int64_t beg = D.rowptr[row], end = D.rowptr[row + 1];
    double y0 = 0.0, y1 = 0.0;
    for (int64_t k0 = beg; k0 < end; k0 += 32) {
      const int64_t k = k0 + lane;
      double v = 0.0;
      int c = 0;
      if (k < end) {
        v = D.val[k];
        c = D.col[k];
      }
      const int m = end - k0 < 32 ? (int)(end - k0) : 32;
      for (int j = 0; j < m; ++j) {
        const double vj = __shfl_sync(0xffffffffu, v, j);
        const int cj = __shfl_sync(0xffffffffu, c, j);
        const double2 xv = reinterpret_cast<const double2*>(X + (int64_t)cj * kB)[lane];
        y0 = fma(vj, xv.x, y0);
        y1 = fma(vj, xv.y, y1);
      }
    }
    const int sl = D.islot[row];
    if (MODE != MODE_RESID && sl >= 0) {  // + (p_b M_Gamma + q_b S_Gamma) X on the interface rows
      const int side = sl / (int)D.nG, g = sl % (int)D.nG;
      const double p0 = D.alpha_own[side * kB + b0], p1 = D.alpha_own[side * kB + b1];
      const double q0 = D.q_own[side * kB + b0], q1 = D.q_own[side * kB + b1];
      double m0 = 0.0, m1 = 0.0;
      for (int j = D.mrow[g]; j < D.mrow[g + 1]; ++j) {
        const double mv = D.mval[j], sv = D.sval[j];
        const int64_t cr = D.mapg[side * D.nG + D.mcol[j]];
        const double2 xv = reinterpret_cast<const double2*>(X + cr * kB)[lane];
        m0 = fma(fma(p0, mv, q0 * sv), xv.x, m0);
        m1 = fma(fma(p1, mv, q1 * sv), xv.y, m1);
      }
      y0 += m0;
      y1 += m1;
    }
    const int64_t e = row * kB;
    if (MODE == MODE_CG) {
      const double2 pv = reinterpret_cast<const double2*>(X + e)[lane];
      double2 out;
      out.x = y0;
      out.y = y1;
      reinterpret_cast<double2*>(Y + e)[lane] = out;
      if (act0) acc0[0] += pv.x * y0;
      if (act1) acc1[0] += pv.y * y1;
    } else if (MODE == MODE_WARM) {
      const double bv = D.b[row];
      double rhs0 = bv, rhs1 = bv;
      if (sl >= 0) {
        const double2 lv = reinterpret_cast<const double2*>(lam + (int64_t)sl * kB)[lane];
        rhs0 = bv + lv.x;
        rhs1 = bv + lv.y;
      }
      const double r0 = rhs0 - y0, r1 = rhs1 - y1;
      const double z0 = dinv_b(D, row, sl, b0) * r0, z1 = dinv_b(D, row, sl, b1) * r1;
      if (act0) {
        R[e + b0] = r0;
        P[e + b0] = z0;
        acc0[0] += r0 * z0;
        acc0[1] += r0 * r0;
        acc0[2] += rhs0 * rhs0;
      }
      if (act1) {
        R[e + b1] = r1;
        P[e + b1] = z1;
        acc1[0] += r1 * z1;
        acc1[1] += r1 * r1;
        acc1[2] += rhs1 * rhs1;
      }
    } else {  // MODE_RESID: w = b - K^N u~
      const double bv = D.b[row];
      const double w0 = bv - y0, w1 = bv - y1;
      if (sl >= 0) {
        double2 wv;
        wv.x = w0;
        wv.y = w1;
        reinterpret_cast<double2*>(wif + (int64_t)sl * kB)[lane] = wv;
      } else {
        if (act0) acc0[0] += w0 * w0;
        if (act1) acc1[0] += w1 * w1;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    wsum[warp][k][b0] = acc0[k];
    wsum[warp][k][b1] = acc1[k];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NP * kB; i += kBT) {
    double s = 0.0;
    for (int w = 0; w < kBT / 32; ++w) s += wsum[w][i / kB][i % kB];
    sm[i] = s;
  }
  __syncthreads();
  const int64_t sb0 = sub_blk0[ls];
  const int snb = sub_nblk[ls];
  if (bpublish(part, blk, NP, sm, cnt + ls, snb)) {
    const int t = threadIdx.x;
    double tot[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) tot[k] = t < kB ? bgather(part, sb0, snb, NP, k, t) : 0.0;
    if (t < kB) {
      BState& S = st[ls * kB + t];
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
template <int MODE>
__global__ void __launch_bounds__(kBT) kb_vec(BatchDev D, BState* __restrict__ st, uint32_t* __restrict__ cnt,
                                              int32_t* __restrict__ nact, const int64_t* __restrict__ sub_blk0,
                                              const int32_t* __restrict__ sub_nblk, double* __restrict__ x,
                                              double* __restrict__ r, double* __restrict__ p,
                                              const double* __restrict__ q, double* __restrict__ part, double tol,
                                              int maxit, int32_t* __restrict__ nactive) {
  __shared__ double red[kBT / kB][2][kB];
  __shared__ double sm[2 * kB];
  const int64_t blk = blockIdx.x;
  const int ls = D.blk_sub[blk];
  if (nact[ls] == 0) return;
  const int b = threadIdx.x % kB, rg = threadIdx.x / kB;
  const BState S0 = st[ls * kB + b];
  const bool act = S0.active;
  const int64_t row0 = D.blk_row0[blk];
  const int nrow = D.blk_nrow[blk];
  double a0 = 0.0, a1 = 0.0;
  if (act) {
    for (int rr = rg; rr < nrow; rr += kBT / kB) {
      const int64_t row = row0 + rr;
      const int64_t e = row * kB + b;
      const int sl = D.islot[row];
      const double di = dinv_b(D, row, sl, b);
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
  if (threadIdx.x < 2 * kB) {
    const int k = threadIdx.x / kB, t = threadIdx.x % kB;
    double s = 0.0;
    for (int g = 0; g < kBT / kB; ++g) s += red[g][k][t];
    sm[threadIdx.x] = s;
  }
  __syncthreads();
  const int64_t sb0 = sub_blk0[ls];
  const int snb = sub_nblk[ls];
  if (bpublish(part, blk, 2, sm, cnt + ls, snb)) {
    const int t = threadIdx.x;
    if (t < kB) {
      const double rz = bgather(part, sb0, snb, 2, 0, t), rr = bgather(part, sb0, snb, 2, 1, t);
      BState& S = st[ls * kB + t];
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

__global__ void kb_zero_if(BatchDev D, const BState* __restrict__ st, double* __restrict__ x) {
  const int64_t blk = blockIdx.x;
  const int ls = D.blk_sub[blk];
  const int b = threadIdx.x % kB, rg = threadIdx.x / kB;
  if (!D.cand_active[b] || !st[ls * kB + b].zero_rhs) return;
  for (int rr = rg; rr < D.blk_nrow[blk]; rr += kBT / kB) x[(D.blk_row0[blk] + rr) * kB + b] = 0.0;
}

// Robin data out of every side: g = (alpha_s + alpha_t) M u|Gamma - lambda, and u|Gamma.
__global__ void kb_trace(BatchDev D, const double* __restrict__ x, const double* __restrict__ lam,
                         double* __restrict__ out) {
  const int k = blockIdx.y;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= D.nG * kB) return;
  const int64_t g = i / kB;
  const int b = (int)(i % kB);
  if (!D.cand_active[b]) return;
  const double ps = D.alpha_sum[k * kB + b], qs = D.q_sum[k * kB + b];
  double mu = 0.0;
  for (int j = D.mrow[g]; j < D.mrow[g + 1]; ++j)
    mu = fma(fma(ps, D.mval[j], qs * D.sval[j]), x[(int64_t)D.mapg[k * D.nG + D.mcol[j]] * kB + b], mu);
  double* o = out + (int64_t)k * 3 * D.nG * kB;
  o[i] = mu - lam[(int64_t)k * D.nG * kB + i];
  o[D.nG * kB + i] = x[(int64_t)D.mapg[k * D.nG + g] * kB + b];
}

__global__ void kb_accept(BatchDev D, const double* __restrict__ out, double* __restrict__ lam,
                          double* __restrict__ unbr) {
  const int k = blockIdx.y;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= D.nG * kB) return;
  if (!D.cand_active[i % kB]) return;
  const double* in = out + (int64_t)D.side_partner[k] * 3 * D.nG * kB;
  lam[(int64_t)k * D.nG * kB + i] = in[i];
  unbr[(int64_t)k * D.nG * kB + i] = in[D.nG * kB + i];
}

__global__ void kb_glue(BatchDev D, int64_t nrows, const double* __restrict__ x, const double* __restrict__ unbr,
                        double* __restrict__ ut) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nrows * kB) return;
  const int64_t row = i / kB;
  const int sl = D.islot[row];
  ut[i] = sl >= 0 ? 0.5 * (x[i] + unbr[(int64_t)sl * kB + i % kB]) : x[i];
}

// Owner side (left slab) of every interface: sum_g (w_s + w_t)^2 per candidate; one block per side.
__global__ void __launch_bounds__(kBT) kb_iface_sum(BatchDev D, const double* __restrict__ wif,
                                                    double* __restrict__ side_sum) {
  __shared__ double red[kBT / kB][kB];
  const int k = blockIdx.x;
  const int b = threadIdx.x % kB, rg = threadIdx.x / kB;
  if (D.side_which[k] != 0) return;
  const int pk = D.side_partner[k];
  double s = 0.0;
  for (int64_t g = rg; g < D.nG; g += kBT / kB) {
    const double w = wif[((int64_t)k * D.nG + g) * kB + b] + wif[((int64_t)pk * D.nG + g) * kB + b];
    s += w * w;
  }
  red[rg][b] = s;
  __syncthreads();
  if (threadIdx.x < kB) {
    double t = 0.0;
    for (int g = 0; g < kBT / kB; ++g) t += red[g][threadIdx.x];
    side_sum[k * kB + threadIdx.x] = t;
  }
}

__global__ void kb_concat_csr(int64_t n, int64_t rc0, int64_t nnz0, const int64_t* __restrict__ rp,
                              const int32_t* __restrict__ col, int64_t nnz, int64_t* __restrict__ rowptr,
                              int32_t* __restrict__ colg, double* __restrict__ dkn, const double* __restrict__ val) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < nnz) colg[nnz0 + i] = (int32_t)(rc0 + col[i]);
  if (i <= n) rowptr[rc0 + i] = nnz0 + rp[i];
  if (i < n) {
    double d = 0.0;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
      if (col[k] == i) d = val[k];
    dkn[rc0 + i] = d;
  }
}

__global__ void kb_gather_b(int64_t npad, int64_t row0, const int32_t* __restrict__ perm, const double* __restrict__ bi,
                            int64_t rc0, double* __restrict__ bc) {
  const int64_t ri = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (ri >= npad) return;
  const int c = perm[ri];
  if (c >= 0) bc[rc0 + c] = bi[row0 + ri];
}

__global__ void kb_extract(int64_t n, int64_t rc0, int b, const double* __restrict__ x, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = x[(rc0 + i) * kB + b];
}

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
  void* ptrs[] = {B->rowptr, B->col, B->val, B->dkn, B->b, B->islot, B->blk_sub, B->blk_nrow, B->blk_row0, B->mapg,
                  B->mdiag, B->sdiag, B->q_own, B->q_sum, B->alpha_own, B->alpha_sum, B->side_which, B->side_partner, B->cand_active, B->x, B->r,
                  B->p, B->q, B->ut, B->lam, B->unbr, B->wif, B->out, B->st, B->cnt, B->nact, B->d_nactive,
                  B->part, B->side_sum};
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
  int64_t nrows = 0, nnz = 0;
  B->rc0.resize(nloc + 1);
  for (int ls = 0; ls < nloc; ++ls) {
    B->rc0[ls] = nrows;
    nrows += c.subs[ls].n;
    nnz += c.subs[ls].nnz;
  }
  B->rc0[nloc] = nrows;
  B->nrows = nrows;
  B->nnz = nnz;
  B->rowptr = balloc<int64_t>(nrows + 1);
  B->col = balloc<int32_t>(nnz);
  B->val = balloc<double>(nnz);
  B->dkn = balloc<double>(nrows);
  B->b = balloc<double>(nrows);
  int64_t nnz0 = 0;
  for (int ls = 0; ls < nloc; ++ls) {
    const Sub& S = c.subs[ls];
    OSM_CUDA(cudaMemcpyAsync(B->val + nnz0, S.val, sizeof(double) * S.nnz, cudaMemcpyDeviceToDevice, c.stream));
    const int64_t m = std::max<int64_t>(S.nnz, S.n + 1);
    kb_concat_csr<<<(unsigned)ceil_div(m, 256), 256, 0, c.stream>>>(S.n, B->rc0[ls], nnz0, S.rowptr, S.col, S.nnz,
                                                                    B->rowptr, B->col, B->dkn, S.val);
    OSM_CHECK_LAUNCH();
    ++c.launches;
    nnz0 += S.nnz;
  }
  // blocks of kRB rows, never straddling subdomains
  std::vector<int32_t> bsub, bnrow;
  std::vector<int64_t> brow0, sblk0;
  std::vector<int32_t> snblk;
  for (int ls = 0; ls < nloc; ++ls) {
    sblk0.push_back((int64_t)bsub.size());
    const int64_t n = c.subs[ls].n;
    int cnt = 0;
    for (int64_t r0 = 0; r0 < n; r0 += kRB) {
      bsub.push_back(ls);
      brow0.push_back(B->rc0[ls] + r0);
      bnrow.push_back((int32_t)std::min<int64_t>(kRB, n - r0));
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
  B->alpha_own = balloc<double>(std::max(1, nsides) * kB);
  B->alpha_sum = balloc<double>(std::max(1, nsides) * kB);
  B->q_own = balloc<double>(std::max(1, nsides) * kB);
  B->q_sum = balloc<double>(std::max(1, nsides) * kB);
  B->cand_active = balloc<int32_t>(kB);
  const int64_t nv = nrows * kB;
  B->x = balloc<double>(nv);
  B->r = balloc<double>(nv);
  B->p = balloc<double>(nv);
  B->q = balloc<double>(nv);
  B->ut = balloc<double>(nv);
  const int64_t ns = std::max<int64_t>(1, nsides * nG * kB);
  B->lam = balloc<double>(ns);
  B->unbr = balloc<double>(ns);
  B->wif = balloc<double>(ns);
  B->out = balloc<double>(3 * ns);
  B->st = balloc<BState>(nloc * kB);
  B->cnt = balloc<uint32_t>(nloc);
  B->nact = balloc<int32_t>(nloc);
  B->d_nactive = balloc<int32_t>(1);
  B->part = balloc<double>(B->nblk * 3 * kB);
  B->side_sum = balloc<double>(std::max(1, nsides) * kB);
  for (double* v : {B->x, B->r, B->p, B->q, B->ut}) OSM_CUDA(cudaMemsetAsync(v, 0, sizeof(double) * nv, c.stream));
  OSM_CUDA(cudaMemsetAsync(B->cnt, 0, sizeof(uint32_t) * nloc, c.stream));
  OSM_CUDA(cudaMemsetAsync(B->st, 0, sizeof(BState) * nloc * kB, c.stream));
  OSM_CUDA(cudaMemsetAsync(B->side_sum, 0, sizeof(double) * std::max(1, nsides) * kB, c.stream));
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

osm_status solve_batch(Ctx& c, int nB, const double* pq, const osm_solve_opts& o, osm_batch_report* rep) {
  if (!c.assembled || !c.density_set) fail(OSM_ERR_STATE, "assemble and upload a density before osm_solve_batch");
  if (c.nranks != 1) fail(OSM_ERR_INVALID_ARG, "osm_solve_batch runs on a single rank");
  if (nB < 1 || nB > kB) fail(OSM_ERR_INVALID_ARG, "need 1 <= B <= 64");
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
  BatchBuf* B = c.batch;
  const int nloc = c.s_end - c.s_begin;
  const int nsides = (int)c.sides.size();
  const int64_t nG = c.nG;
  // alpha per side per candidate
  std::vector<double> aown(std::max(1, nsides) * kB, 0.0), asum(std::max(1, nsides) * kB, 0.0);
  std::vector<double> qown(std::max(1, nsides) * kB, 0.0), qsum(std::max(1, nsides) * kB, 0.0);
  for (int k = 0; k < nsides; ++k)
    for (int bb = 0; bb < nB; ++bb) {
      const int i = c.sides[k].iface;
      const double pl = pq[(bb * 4 + 0) * ni + i], ql = pq[(bb * 4 + 1) * ni + i];
      const double pr = pq[(bb * 4 + 2) * ni + i], qr = pq[(bb * 4 + 3) * ni + i];
      aown[k * kB + bb] = c.sides[k].which == 0 ? pl : pr;
      qown[k * kB + bb] = c.sides[k].which == 0 ? ql : qr;
      asum[k * kB + bb] = pl + pr;
      qsum[k * kB + bb] = ql + qr;
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
  const int64_t nv = B->nrows * kB;
  OSM_CUDA(cudaMemsetAsync(B->x, 0, sizeof(double) * nv, c.stream));
  if (nsides) OSM_CUDA(cudaMemsetAsync(B->lam, 0, sizeof(double) * nsides * nG * kB, c.stream));
  if (nsides) OSM_CUDA(cudaMemsetAsync(B->unbr, 0, sizeof(double) * nsides * nG * kB, c.stream));
  std::vector<int32_t> cand(kB, 0);
  for (int bb = 0; bb < nB; ++bb) cand[bb] = 1;
  B->B = nB;
  B->hist.assign(nB, {});
  B->inner.assign(nB, {});
  std::vector<BState> hst(nloc * kB);
  std::vector<double> hside(std::max(1, nsides) * kB);
  BatchDev D = batch_view(c);
  const unsigned nblk = (unsigned)B->nblk;
  const dim3 gI((unsigned)ceil_div(nG * kB, 256), (unsigned)std::max(1, nsides));
  int64_t inner_total = 0;
  int n_conv = 0, outer_max = 0;
  constexpr int kChunkB = 8;
  for (int n = 1; n <= o.max_outer; ++n) {
    OSM_CUDA(cudaMemcpyAsync(B->cand_active, cand.data(), sizeof(int32_t) * kB, cudaMemcpyHostToDevice, c.stream));
    if (!o.warm_start) OSM_CUDA(cudaMemsetAsync(B->x, 0, sizeof(double) * nv, c.stream));
    OSM_CUDA(cudaMemsetAsync(B->d_nactive, 0, sizeof(int32_t), c.stream));
    OSM_CUDA(cudaMemsetAsync(B->nact, 0, sizeof(int32_t) * nloc, c.stream));
    kb_spmm<MODE_WARM><<<nblk, kBT, 0, c.stream>>>(D, B->st, B->cnt, B->nact, c.batch_sub_blk0, c.batch_sub_nblk, B->x,
                                                   nullptr, B->r, B->p, B->lam, nullptr, B->part, o.tol_inner,
                                                   B->d_nactive);
    kb_zero_if<<<nblk, kBT, 0, c.stream>>>(D, B->st, B->x);
    OSM_CHECK_LAUNCH();
    c.launches += 2;
    OSM_CUDA(cudaMemcpyAsync(&c.h_nactive[0], B->d_nactive, sizeof(int32_t), cudaMemcpyDeviceToHost, c.stream));
    OSM_CUDA(cudaStreamSynchronize(c.stream));
    if (c.h_nactive[0] > 0) {
      for (int ch = 0;; ++ch) {
        for (int it = 0; it < kChunkB; ++it) {
          kb_spmm<MODE_CG><<<nblk, kBT, 0, c.stream>>>(D, B->st, B->cnt, B->nact, c.batch_sub_blk0, c.batch_sub_nblk,
                                                       B->p, B->q, nullptr, nullptr, nullptr, nullptr, B->part,
                                                       o.tol_inner, B->d_nactive);
          kb_vec<0><<<nblk, kBT, 0, c.stream>>>(D, B->st, B->cnt, B->nact, c.batch_sub_blk0, c.batch_sub_nblk, B->x,
                                                B->r, B->p, B->q, B->part, o.tol_inner, o.max_inner, B->d_nactive);
          kb_vec<1><<<nblk, kBT, 0, c.stream>>>(D, B->st, B->cnt, B->nact, c.batch_sub_blk0, c.batch_sub_nblk, B->x,
                                                B->r, B->p, B->q, B->part, o.tol_inner, o.max_inner, B->d_nactive);
        }
        OSM_CHECK_LAUNCH();
        c.launches += 3 * kChunkB;
        OSM_CUDA(cudaMemcpyAsync(&c.h_nactive[ch & 1], B->d_nactive, sizeof(int32_t), cudaMemcpyDeviceToHost,
                                 c.stream));
        OSM_CUDA(cudaEventRecord(c.ev_chunk[ch & 1], c.stream));
        if (ch > 0) {
          OSM_CUDA(cudaEventSynchronize(c.ev_chunk[(ch - 1) & 1]));
          if (c.h_nactive[(ch - 1) & 1] == 0) break;
        }
        if ((int64_t)ch * kChunkB > (int64_t)o.max_inner + 2 * kChunkB) break;
      }
    }
    if (nsides) {
      kb_trace<<<gI, 256, 0, c.stream>>>(D, B->x, B->lam, B->out);
      kb_accept<<<gI, 256, 0, c.stream>>>(D, B->out, B->lam, B->unbr);
      c.launches += 2;
    }
    kb_glue<<<(unsigned)ceil_div(nv, 256), 256, 0, c.stream>>>(D, B->nrows, B->x, B->unbr, B->ut);
    kb_spmm<MODE_RESID><<<nblk, kBT, 0, c.stream>>>(D, B->st, B->cnt, B->nact, c.batch_sub_blk0, c.batch_sub_nblk,
                                                    B->ut, nullptr, nullptr, nullptr, nullptr, B->wif, B->part,
                                                    o.tol_inner, B->d_nactive);
    c.launches += 2;
    if (nsides) {
      kb_iface_sum<<<(unsigned)nsides, kBT, 0, c.stream>>>(D, B->wif, B->side_sum);
      ++c.launches;
    }
    OSM_CHECK_LAUNCH();
    OSM_CUDA(cudaMemcpyAsync(hst.data(), B->st, sizeof(BState) * nloc * kB, cudaMemcpyDeviceToHost, c.stream));
    if (nsides)
      OSM_CUDA(cudaMemcpyAsync(hside.data(), B->side_sum, sizeof(double) * nsides * kB, cudaMemcpyDeviceToHost,
                               c.stream));
    OSM_CUDA(cudaStreamSynchronize(c.stream));
    bool any = false;
    for (int bb = 0; bb < nB; ++bb) {
      if (!cand[bb]) continue;
      double r2 = 0.0;
      for (int ls = 0; ls < nloc; ++ls) {
        double v = hst[ls * kB + bb].resid;
        const int k = c.subs[ls].side[1];
        if (k >= 0) v += hside[k * kB + bb];
        r2 += v;
      }
      const double h = fnorm > 0 ? std::sqrt(r2) / fnorm : std::sqrt(r2);
      B->hist[bb].push_back(h);
      for (int ls = 0; ls < nloc; ++ls) {
        B->inner[bb].push_back(hst[ls * kB + bb].iters);
        inner_total += hst[ls * kB + bb].iters;
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
  kb_extract<<<(unsigned)ceil_div(ns, 256), 256, 0, c.stream>>>(ns, c.batch->rc0[ls], b, c.batch->x, d);
  OSM_CHECK_LAUNCH();
  ++c.launches;
  OSM_CUDA(cudaMemcpyAsync(u, d, sizeof(double) * ns, cudaMemcpyDeviceToHost, c.stream));
  OSM_CUDA(cudaStreamSynchronize(c.stream));
  cudaFree(d);
  *n = ns;
}

}  // namespace osm

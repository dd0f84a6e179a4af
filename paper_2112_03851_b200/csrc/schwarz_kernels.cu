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
    __threadfence();
    const uint32_t prev = atomicAdd(cnt, 1u);
    last = (prev == (uint32_t)(nblk - 1));
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

// y_row = sum_j A[row, j] x[j] for the lane's row of a SELL-32 slice, entries in
// column order (sequential per row, deterministic).  Software-pipelined: the
// value/column chunk k+1 is requested before the gathers of chunk k are consumed,
// so every warp keeps two chunks of streaming loads in flight.  The slice width
// is warp-uniform, so the tail predicates never diverge.
template <int CH>
__device__ __forceinline__ double sell_row(const SellDev& A, int64_t slice, int lane, const double* __restrict__ x) {
  const int w = A.swidth[slice];
  const int64_t base = A.soff[slice] + lane;
  const double* vp = A.val + base;
  const int32_t* cp = A.col + base;
  double s = 0.0;
  double v[CH];
  int32_t c[CH];
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    v[j] = j < w ? ld_stream(vp + 32 * j) : 0.0;
    c[j] = j < w ? ld_stream(cp + 32 * j) : 0;
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
      vn[j] = (kn + j < w) ? ld_stream(vp + 32 * (kn + j)) : 0.0;
      cn[j] = (kn + j < w) ? ld_stream(cp + 32 * (kn + j)) : 0;
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

constexpr int kChunk = 4;

// ---------------------------------------------------------------- PCG kernels

// q = K_s p ; p.q -> alpha = rho / (p.q)
__global__ void __launch_bounds__(kThreads) k_cg_spmv(SellDev A, const int32_t* __restrict__ blk_sub,
                                                      SubState* __restrict__ st, const double* __restrict__ p,
                                                      double* __restrict__ q, double* __restrict__ part,
                                                      int64_t stride, int32_t* __restrict__ nactive) {
  __shared__ double sm[kSlicesPerBlock * 1];
  pdl_enter();
  const int64_t blk = blockIdx.x;
  const int ls = blk_sub[blk];
  if (!st[ls].active) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t slice = blk * kSlicesPerBlock + warp;
  const int64_t row = slice * kWarp + lane;
  const double y = sell_row<kChunk>(A, slice, lane, p);
  q[row] = y;
  double v[1] = {p[row] * y};
  block_sum<1>(v, sm);
  SubState& S = st[ls];
  if (publish<1>(v, part, stride, blk, &S.cnt, S.nblk)) {
    double t[1];
    gather_partials<1>(t, part, stride, S.blk0, S.nblk, sm);
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

// x += alpha p ; r -= alpha q ; z = D^{-1} r ; r.z, r.r ; stop test ||r|| <= tol ||rhs||; beta.
// 128 threads x 2 rows (16-byte loads) per 256-row block.
constexpr int kVecThreads = kRowsPerBlock / 2;
__global__ void __launch_bounds__(kVecThreads) k_cg_update(const int32_t* __restrict__ blk_sub, SubState* __restrict__ st,
                                                           double* __restrict__ x, double* __restrict__ r,
                                                           const double* __restrict__ p, const double* __restrict__ q,
                                                           const double* __restrict__ dinv, double* __restrict__ part,
                                                           int64_t stride, double tol, int maxit,
                                                           int32_t* __restrict__ nactive) {
  __shared__ double sm[(kVecThreads / 32) * 2];
  pdl_enter();
  const int64_t blk = blockIdx.x;
  const int ls = blk_sub[blk];
  if (!st[ls].active) return;
  const int64_t i2 = blk * kVecThreads + threadIdx.x;  // index of the row pair
  const double a = st[ls].alpha;
  const double2 pv = reinterpret_cast<const double2*>(p)[i2];
  const double2 qv = reinterpret_cast<const double2*>(q)[i2];
  double2 xv = reinterpret_cast<const double2*>(x)[i2];
  double2 rv = reinterpret_cast<const double2*>(r)[i2];
  const double2 dv = reinterpret_cast<const double2*>(dinv)[i2];
  xv.x = fma(a, pv.x, xv.x);
  xv.y = fma(a, pv.y, xv.y);
  rv.x = fma(-a, qv.x, rv.x);
  rv.y = fma(-a, qv.y, rv.y);
  reinterpret_cast<double2*>(x)[i2] = xv;
  reinterpret_cast<double2*>(r)[i2] = rv;
  const double z0 = dv.x * rv.x, z1 = dv.y * rv.y;
  double v[2] = {rv.x * z0 + rv.y * z1, rv.x * rv.x + rv.y * rv.y};
  block_sum<2, kVecThreads / 32>(v, sm);
  SubState& S = st[ls];
  if (publish<2>(v, part, stride, blk, &S.cnt, S.nblk)) {
    double t[2];
    gather_partials<2, kVecThreads / 32>(t, part, stride, S.blk0, S.nblk, sm);
    if (threadIdx.x == 0) {
      S.cnt = 0;
      const double rz = t[0], rr = t[1];
      S.rr = rr;
      S.iters += 1;
      if (sqrt(rr) <= tol * sqrt(S.bb)) {
        S.status = 1;
        S.active = 0;
        atomicSub(nactive, 1);
      } else if (S.iters >= maxit) {
        S.status = 2;
        S.active = 0;
        atomicSub(nactive, 1);
      } else {
        S.beta = rz / S.rho;
        S.rho = rz;
      }
    }
  }
}

// p = D^{-1} r + beta p  (128 threads x 2 rows per 256-row block)
__global__ void __launch_bounds__(kVecThreads) k_cg_dir(const int32_t* __restrict__ blk_sub,
                                                        const SubState* __restrict__ st, const double* __restrict__ r,
                                                        const double* __restrict__ dinv, double* __restrict__ p) {
  pdl_enter();
  const int64_t blk = blockIdx.x;
  const int ls = blk_sub[blk];
  if (!st[ls].active) return;
  const int64_t i2 = blk * kVecThreads + threadIdx.x;
  const double beta = st[ls].beta;
  const double2 rv = reinterpret_cast<const double2*>(r)[i2];
  const double2 dv = reinterpret_cast<const double2*>(dinv)[i2];
  double2 pv = reinterpret_cast<const double2*>(p)[i2];
  pv.x = fma(beta, pv.x, dv.x * rv.x);
  pv.y = fma(beta, pv.y, dv.y * rv.y);
  reinterpret_cast<double2*>(p)[i2] = pv;
}

// Warm start: rhs = b + P^T lambda ; r = rhs - K_s x ; z = D^{-1} r ; p = z ;
// rho = r.z, ||r||^2, ||rhs||^2 ; zero rhs -> x = 0 after 0 iterations.
__global__ void __launch_bounds__(kThreads) k_warm(SellDev A, const int32_t* __restrict__ blk_sub,
                                                   SubState* __restrict__ st, const double* __restrict__ x,
                                                   const double* __restrict__ b, const int32_t* __restrict__ islot,
                                                   const double* __restrict__ lam_all, const double* __restrict__ dinv,
                                                   double* __restrict__ r, double* __restrict__ p,
                                                   double* __restrict__ part, int64_t stride, double tol,
                                                   int32_t* __restrict__ nactive) {
  __shared__ double sm[kSlicesPerBlock * 3];
  const int64_t blk = blockIdx.x;
  const int ls = blk_sub[blk];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t slice = blk * kSlicesPerBlock + warp;
  const int64_t row = slice * kWarp + lane;
  const double ax = sell_row<kChunk>(A, slice, lane, x);
  const int sl = islot[row];
  const double rhs = sl >= 0 ? b[row] + lam_all[sl] : b[row];
  const double rv = rhs - ax;
  const double z = dinv[row] * rv;
  r[row] = rv;
  p[row] = z;
  double v[3] = {rv * z, rv * rv, rhs * rhs};
  block_sum<3>(v, sm);
  SubState& S = st[ls];
  if (publish<3>(v, part, stride, blk, &S.cnt, S.nblk)) {
    double t[3];
    gather_partials<3>(t, part, stride, S.blk0, S.nblk, sm);
    if (threadIdx.x == 0) {
      S.cnt = 0;
      S.rho = t[0];
      S.rr = t[1];
      S.bb = t[2];
      S.iters = 0;
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

// Robin data to send: g_{s->t} = (alpha_s + alpha_t) M_Gamma u_s|Gamma - lambda_s ;
// also the trace u_s|Gamma for gluing.  Discrete form of PAPER.md:64-71.
__global__ void k_trace(const SideDev* __restrict__ sides, int64_t nG, const int32_t* __restrict__ mrow,
                        const int32_t* __restrict__ mcol, const double* __restrict__ mval,
                        const double* __restrict__ x) {
  const SideDev S = sides[blockIdx.y];
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= nG) return;
  double mu = 0.0;
  for (int j = mrow[g]; j < mrow[g + 1]; ++j) mu = fma(mval[j], x[S.map[mcol[j]]], mu);
  S.out[g] = S.alpha_sum * mu - S.lam[g];
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
__global__ void __launch_bounds__(kThreads) k_resid(SellDev A, const int32_t* __restrict__ blk_sub,
                                                    SubState* __restrict__ st, const double* __restrict__ ut,
                                                    const double* __restrict__ b, const int32_t* __restrict__ islot,
                                                    double* __restrict__ wif_all, double* __restrict__ part,
                                                    int64_t stride) {
  __shared__ double sm[kSlicesPerBlock * 1];
  const int64_t blk = blockIdx.x;
  const int ls = blk_sub[blk];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t slice = blk * kSlicesPerBlock + warp;
  const int64_t row = slice * kWarp + lane;
  const double w = b[row] - sell_row<kChunk>(A, slice, lane, ut);
  const int sl = islot[row];
  if (sl >= 0) wif_all[sl] = w;
  double v[1] = {sl == -1 ? w * w : 0.0};
  block_sum<1>(v, sm);
  SubState& S = st[ls];
  if (publish<1>(v, part, stride, blk, &S.cnt, S.nblk)) {
    double t[1];
    gather_partials<1>(t, part, stride, S.blk0, S.nblk, sm);
    if (threadIdx.x == 0) {
      S.cnt = 0;
      S.resid = t[0];
    }
  }
}

// Interface rows: w = b - K^N u~ = (b - K_s u~) + alpha_own M u~|Gamma ; publish w in the outbox.
__global__ void k_iface_w(const SideDev* __restrict__ sides, int64_t nG, const int32_t* __restrict__ mrow,
                          const int32_t* __restrict__ mcol, const double* __restrict__ mval,
                          const double* __restrict__ ut) {
  const SideDev S = sides[blockIdx.y];
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= nG) return;
  double mu = 0.0;
  for (int j = mrow[g]; j < mrow[g + 1]; ++j) mu = fma(mval[j], ut[S.map[mcol[j]]], mu);
  const double w = fma(S.alpha_own, mu, S.wif[g]);
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

SellDev sell_of(const Ctx& c) { return SellDev{c.sell_val, c.sell_col, c.sell_soff, c.sell_swidth}; }

}  // namespace

void launch_warm(Ctx& c, double tol, int) {
  timer_begin(c, T_WARM);
  k_warm<<<(unsigned)c.nblk_total, kThreads, 0, c.stream>>>(sell_of(c), c.blk_sub, c.st, c.x, c.b, c.islot, c.lam_all,
                                                            c.dinv, c.r, c.p, c.part, c.nblk_total, tol, c.d_nactive);
  OSM_CHECK_LAUNCH();
  ++c.launches;
  timer_end(c, T_WARM);
}

void launch_zero_if(Ctx& c) {
  k_zero_if<<<(unsigned)c.nblk_total, kThreads, 0, c.stream>>>(c.blk_sub, c.st, c.x);
  OSM_CHECK_LAUNCH();
  ++c.launches;
}

template <typename... KArgs, typename... Args>
static void launch_pdl(const Ctx& c, void (*kern)(KArgs...), unsigned grid, unsigned block, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = c.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  OSM_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
}

void launch_cg_spmv(Ctx& c) {
  timer_begin(c, T_SPMV);
  launch_pdl(c, k_cg_spmv, (unsigned)c.nblk_total, kThreads, sell_of(c), (const int32_t*)c.blk_sub, c.st,
             (const double*)c.p, c.q, c.part, c.nblk_total, c.d_nactive);
  ++c.launches;
  timer_end(c, T_SPMV);
}

void launch_cg_update(Ctx& c, double tol, int maxit) {
  timer_begin(c, T_UPDATE);
  launch_pdl(c, k_cg_update, (unsigned)c.nblk_total, kVecThreads, (const int32_t*)c.blk_sub, c.st, c.x, c.r,
             (const double*)c.p, (const double*)c.q, (const double*)c.dinv, c.part, c.nblk_total, tol, maxit,
             c.d_nactive);
  ++c.launches;
  timer_end(c, T_UPDATE);
}

void launch_cg_dir(Ctx& c) {
  timer_begin(c, T_DIR);
  launch_pdl(c, k_cg_dir, (unsigned)c.nblk_total, kVecThreads, (const int32_t*)c.blk_sub, (const SubState*)c.st,
             (const double*)c.r, (const double*)c.dinv, c.p);
  ++c.launches;
  timer_end(c, T_DIR);
}

void launch_trace(Ctx& c) {
  if (c.sides.empty()) return;
  dim3 grid((unsigned)ceil_div(c.nG, 256), (unsigned)c.sides.size());
  k_trace<<<grid, 256, 0, c.stream>>>(c.d_sides, c.nG, c.d_mrow, c.d_mcol, c.d_mval, c.x);
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

void launch_resid(Ctx& c) {
  timer_begin(c, T_RESID);
  k_resid<<<(unsigned)c.nblk_total, kThreads, 0, c.stream>>>(sell_of(c), c.blk_sub, c.st, c.ut, c.b, c.islot,
                                                             c.wif_all, c.part, c.nblk_total);
  OSM_CHECK_LAUNCH();
  ++c.launches;
  timer_end(c, T_RESID);
}

void launch_iface_w(Ctx& c) {
  if (c.sides.empty()) return;
  dim3 grid((unsigned)ceil_div(c.nG, 256), (unsigned)c.sides.size());
  k_iface_w<<<grid, 256, 0, c.stream>>>(c.d_sides, c.nG, c.d_mrow, c.d_mcol, c.d_mval, c.ut);
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

/*
 * osm.h -- C ABI of the B200-native optimized-Schwarz gravimetry solver.
 *
 * Method: arXiv 2112.03851 ("stochastic-based optimized Schwarz method for the
 * gravimetry equation on GPU clusters").  The library solves
 *     -Delta Phi = 4 pi G drho  in a box,  Phi = 0 on the boundary
 * ("Delta Phi = -4 pi G delta rho", "homogeneous
 * Dirichlet condition") with P1/P2 tetrahedral finite elements on a Kuhn box
 * mesh ("high order finite element"; reading SURVEY.md 8(c) Q1/Q2),
 * partitioned into x-slabs ("partionned in the x-direction"), by the
 * non-overlapping Schwarz iteration with Robin transmission,
 * each subdomain solved by Jacobi-preconditioned CG to eps = 1e-10
 * (PAPER.md:165).  Everything on the solve path runs in this library's CUDA
 * kernels (sm_100a); there is no CPU fallback.
 *
 * Conventions shared by every call:
 *  - All floating point is IEEE fp64.  All arrays are plain C arrays.
 *  - "host" pointers are ordinary CPU memory; "device" pointers are CUDA device
 *    memory on the context's device.  The caller owns every buffer it passes;
 *    the library copies what it needs before returning (inputs) or writes into
 *    the caller's buffer (outputs).  The context owns all of its device memory
 *    and its NCCL communicator.
 *  - Lattice ordering: points of the (o*nx+1) x (o*ny+1) x (o*nz+1) lattice
 *    (o = element order) have id = I + Nx*(J + Ny*K), x fastest.  Cells are
 *    ordered the same way (ci + nx*(cj + ny*ck)).
 *  - Subdomain s is the x-slab of cells [c_s, c_{s+1}) (widths differ by <= 1,
 *    remainder to the left).  Its local unknowns are its free
 *    lattice points (interface planes duplicated in both neighbours), numbered
 *    x fastest over the slab ("contract order").  Interface i lies between
 *    slabs i and i+1; side 0 = the left slab, side 1 = the right slab.
 *  - Every call returns an osm_status.  On failure the call has no partial
 *    effect on results previously read back, and osm_last_error() returns a
 *    thread-local message.  No C++ exception crosses this boundary.
 *  - Output-size queries: where noted, passing NULL for the output buffer
 *    writes the required element count to the size argument and returns OSM_OK.
 *  - Collective calls (marked [collective]) must be made by every rank of the
 *    communicator in the same order.
 */
#ifndef OSM_H_
#define OSM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OSM_ABI_VERSION 2

typedef enum osm_status {
  OSM_OK = 0,
  OSM_ERR_INVALID_ARG = 1,    /* a count/extent <= 0, size mismatch, bad index, NULL where required */
  OSM_ERR_GRID_TOO_SMALL = 2, /* fewer than 3 lattice points per axis: no interior */
  OSM_ERR_ILL_POSED = 3,      /* Robin alpha < 0, or alpha = 0 on both sides of an interface */
  OSM_ERR_PRECOND = 4,        /* a diagonal entry <= 0: Jacobi preconditioner undefined */
  OSM_NOT_CONVERGED = 5,      /* max_outer reached; report and iterate stay readable */
  OSM_ERR_DIVERGED = 6,       /* h(n) grew for diverge_window consecutive iterations */
  OSM_ERR_CUDA = 7,           /* a CUDA runtime error (message has the CUDA error string) */
  OSM_ERR_NCCL = 8,           /* an NCCL error */
  OSM_ERR_STATE = 9           /* call out of order (e.g. solve before assemble) */
} osm_status;

typedef struct osm_ctx osm_ctx;

/* Box mesh: nx*ny*nz hexahedral cells on [0,lx]x[0,ly]x[0,lz] (metres), each
 * split into the 6 Kuhn tetrahedra sharing the (0,0,0)-(1,1,1) diagonal;
 * order = 1 (P1) or 2 (P2) Lagrange elements. */
typedef struct osm_mesh_desc {
  int64_t nx, ny, nz;
  double lx, ly, lz;
  int order;
} osm_mesh_desc;

/* In-process transport (PAPER.md:157-158 one subdomain block per processor): the
 * ranks are host threads of ONE process, each driving its own context (on the same or on different
 * devices).  The trace exchange, the residual allgather and the Phi reduce become device-to-device
 * copies ordered by CUDA events, with host barriers between the phases; no kernel waits on another
 * rank's kernel.  It runs every nranks > 1 code path of the library without NCCL (tests, and
 * single-process multi-GPU use).  Create one hub for nranks ranks, pass it in osm_dist_desc.hub of
 * every rank's osm_create (made from its own thread), and make every collective call from the rank's
 * own thread.  A rank whose collective call fails releases the others (they return OSM_ERR_STATE);
 * a barrier that waits 600 s fails the same way.  Destroy the hub after every context attached to it. */
typedef struct osm_hub osm_hub;
osm_status osm_hub_create(int nranks, osm_hub** out);
void osm_hub_destroy(osm_hub* hub);

/* Distribution: this process is `rank` of `nranks` (one process per GPU),
 * driving CUDA device `device`.  nccl_uid: 128-byte ncclUniqueId made by
 * osm_nccl_unique_id() on rank 0 and broadcast by the caller (e.g. with
 * torch.distributed); NULL when nranks == 1 or when hub is given.  hub: an
 * osm_hub (in-process ranks) instead of NCCL; NULL otherwise.  stream: a
 * cudaStream_t to run on, or NULL for a library-owned stream.  (ABI 2 added hub.) */
typedef struct osm_dist_desc {
  int rank, nranks, device;
  const void* nccl_uid;
  void* stream;
  osm_hub* hub;
} osm_dist_desc;

/* Solve options.  tol_outer: stop when h(n) = ||f - K u~||_2/||f||_2 <= tol_outer
 * (PAPER.md:215 uses 1e-6; BASELINE metric 1e-8).  tol_inner: PCG stops when the
 * recursive residual ||r||_2 <= tol_inner * ||rhs||_2 (1e-10).
 * warm_start: start each inner solve from the previous outer iterate.
 * diverge_window: DIVERGED after this many consecutive growing h(n) (0 = off). */
typedef struct osm_solve_opts {
  double tol_outer;
  int max_outer;
  double tol_inner;
  int max_inner;
  int warm_start;
  int diverge_window;
} osm_solve_opts;

typedef struct osm_report {
  int outer_iters;     /* N: outer iterations performed */
  int converged;       /* 1 if h(N) <= tol_outer */
  double h_final;      /* h(N) */
  double seconds;      /* wall time of the solve (host clock around the device work) */
  int64_t inner_total; /* sum over outer iterations and subdomains of PCG iterations (all ranks) */
  int inner_maxed;     /* number of (n, s) inner solves that hit max_inner */
} osm_report;

/* Per-kernel device timing (CUDA events on the library stream), accumulated
 * while osm_set_kernel_timing(ctx, 1) is on. */
typedef struct osm_kernel_time {
  char name[32];
  int64_t launches;
  double total_ms;
} osm_kernel_time;

int osm_abi_version(void);
const char* osm_last_error(void);

/* Writes a fresh 128-byte ncclUniqueId to uid128 (host).  Call on rank 0 only. */
osm_status osm_nccl_unique_id(void* uid128);

/* [collective] Creates a context.  INVALID_ARG if a count/extent <= 0, order not
 * in {1,2}, rank/nranks inconsistent; GRID_TOO_SMALL if o*n+1 < 3 on an axis. */
osm_status osm_create(const osm_mesh_desc* mesh, const osm_dist_desc* dist, osm_ctx** out);
void osm_destroy(osm_ctx* ctx);

/* Splits the box into nsub x-slabs; slab s goes to rank floor(s*nranks/nsub).
 * INVALID_ARG if nsub < 1, nsub > nx, or nsub % nranks != 0.  Invalidates assembly. */
osm_status osm_decompose(osm_ctx* ctx, int nsub);

/* Robin parameters (OO0: A^(s) = alpha_s, weak form alpha_s M_Gamma; PAPER.md:77-79,
 * SURVEY Q8).  alpha_left[i] is used by the slab left of interface i (side 0),
 * alpha_right[i] by the slab right of it (side 1); nsub-1 host values each.
 * ILL_POSED if any alpha < 0 or both alphas of an interface are 0.  May be
 * called between solves; the Robin term is re-applied on the device. */
osm_status osm_set_robin(osm_ctx* ctx, const double* alpha_left, const double* alpha_right);

/* OO2 transmission ("A^(s) := p^(s) + q^(s) d^2_tau", optimized in Table 1
 * rows oo2_*; sign reading SURVEY Q25: symbol Lambda = p + q k^2, i.e. the operator
 * p - q d^2_tau, weak form int_Gamma p u v + q grad_tau u . grad_tau v = p M_Gamma + q S_Gamma).
 * p_left[i], q_left[i]: side 0 (slab left of interface i); p_right, q_right: side 1.
 * ILL_POSED if any coefficient < 0 or p = 0 on both sides.  osm_set_robin == q = 0. */
osm_status osm_set_robin2(osm_ctx* ctx, const double* p_left, const double* q_left, const double* p_right,
                          const double* q_right);

/* [device work] Builds, per local subdomain: the Neumann stiffness K_s^N
 * (structural pattern, Dirichlet rows/cols removed), the interface mass
 * M_Gamma, interface maps, the SELL-32 hot-path copy and the Jacobi diagonal.
 * PRECOND if a diagonal <= 0. */
osm_status osm_assemble(osm_ctx* ctx);

/* Density anomaly drho[nx*ny*nz] (kg/m^3, cell-wise constant, x fastest; host
 * pointer) and the gravity constant G (6.672e-11).  The load is
 * f = 4 pi G drho, integrated exactly per tet.  Requires osm_assemble. */
osm_status osm_upload_density(osm_ctx* ctx, const double* drho, double G);
/* Same, from a device pointer (nx*ny*nz doubles on the context's device). */
osm_status osm_upload_density_device(osm_ctx* ctx, const double* drho_dev, double G);

/* Load vector given directly in global free-DOF order (lattice ids increasing, Dirichlet points
 * removed; n = (o nx - 1)(o ny - 1)(o nz - 1) host doubles), instead of a density (SURVEY 8(b)
 * "escape hatch").  Each slab takes b_free at its points, halved on its interface planes (the two
 * slab copies of an interface row share it), so the glued system is K u = b_free.
 * INVALID_ARG on a size mismatch; STATE before osm_assemble. */
osm_status osm_upload_load_vector(osm_ctx* ctx, const double* b_free, int64_t n);

/* [collective] Runs the Schwarz iteration from u^0 = lambda^0 = 0.  Returns OK,
 * NOT_CONVERGED (max_outer reached), DIVERGED, or an error.  report may be NULL. */
osm_status osm_solve(osm_ctx* ctx, const osm_solve_opts* opts, osm_report* report);

/* Batched-alpha solve (BASELINE config C4): B <= 64 candidate Robin
 * parameter sets solved simultaneously, sharing K_s^N (each matrix entry is read once per
 * batched PCG iteration for all candidates; alpha_b M_Gamma is applied on the fly).
 * alphas: host array [b][side][iface], i.e. alphas[(b*2 + side)*(nsub-1) + i], side 0 =
 * the slab left of interface i.  Every candidate runs exactly the osm_solve iteration and
 * stops at its own h_b(n) <= tol_outer or max_outer (PAPER.md:95 population of 25 fits).
 * Single rank only (INVALID_ARG otherwise).  ILL_POSED as osm_set_robin. */
typedef struct osm_batch_report {
  int B;               /* candidates */
  int outer_max;       /* largest outer count over candidates */
  int n_converged;     /* candidates with h_b <= tol_outer */
  int64_t inner_total; /* PCG iterations summed over candidates, outer iterations, subdomains */
  double seconds;
} osm_batch_report;
osm_status osm_solve_batch(osm_ctx* ctx, int B, const double* alphas, const osm_solve_opts* opts,
                           osm_batch_report* report);
/* OO2 batch: pq host array [b][4][iface]: (p_left, q_left, p_right, q_right) of interface i,
 * i.e. pq[(b*4 + j)*(nsub-1) + i]; A_b = p M_Gamma + q S_Gamma per side (as osm_set_robin2). */
osm_status osm_solve_batch2(osm_ctx* ctx, int B, const double* pq, const osm_solve_opts* opts,
                            osm_batch_report* report);
/* h_b(1..N_b) of candidate b of the last batched solve.  h == NULL: *n = N_b. */
osm_status osm_get_batch_history(osm_ctx* ctx, int b, double* h, int cap, int* n);
/* PCG iterations [n][s] (local subdomains) of candidate b.  its == NULL: *n = N_b * nsub_local. */
osm_status osm_get_batch_inner_iters(osm_ctx* ctx, int b, int32_t* its, int cap, int* n);
/* Candidate b's final u_s (contract order, host).  u == NULL: *n = n_s. */
osm_status osm_get_batch_local_solution(osm_ctx* ctx, int b, int s, double* u, int64_t* n);

/* h(1..N) of the last solve (every rank holds it).  h == NULL: *n = N. */
osm_status osm_get_history(osm_ctx* ctx, double* h, int cap, int* n);
/* PCG iterations its[n*nsub + s] of the last solve, for the subdomains of this
 * rank (-1 for subdomains of other ranks).  its == NULL: *n_outer = N. */
osm_status osm_get_inner_iters(osm_ctx* ctx, int32_t* its, int cap_outer, int* n_outer);

/* [collective] Phi of the last solve on the full lattice (Nx*Ny*Nz host doubles,
 * x fastest, Dirichlet points 0, interface points averaged between the two slab
 * copies).  Gathered to rank 0; other ranks may pass NULL.  phi == NULL on
 * rank 0: *n = Nx*Ny*Nz. */
osm_status osm_get_solution(osm_ctx* ctx, double* phi, int64_t* n);
/* [collective] Gravity anomaly of the last solve:
 * g_z = -dPhi_h/dz (m/s^2, z up, positive for excess mass below) of the glued FE potential on the
 * plane z = z0 (0 <= z0 <= lz) at the cell-centre columns (x_c, y_c), nx*ny host doubles, x fastest,
 * evaluated exactly in the Kuhn tet containing the point (ties between tets: lower axis first).
 * Rank 0 receives it; gz == NULL on rank 0: *n = nx*ny. */
osm_status osm_gravity_z(osm_ctx* ctx, double z0, double* gz, int64_t* n);
/* Local subdomain iterate u_s (contract order, host).  u == NULL: *n = n_s. */
osm_status osm_get_local_solution(osm_ctx* ctx, int s, double* u, int64_t* n);
/* lambda_{s,Gamma} of interface `iface`, side 0/1 (owner rank only; host). */
osm_status osm_get_trace(osm_ctx* ctx, int iface, int side, double* lam, int64_t* n);

/* Parity dumps (owner rank only, host buffers).  K_s^N in canonical CSR
 * (columns ascending, explicit structural zeros kept, SURVEY
 * Q17), contract order.  rowptr == NULL: writes *nrows and *nnz only. */
osm_status osm_get_csr(osm_ctx* ctx, int s, int64_t* rowptr, int32_t* col, double* val, int64_t* nrows,
                       int64_t* nnz);
/* Interface map of interface `iface`, side 0 (left slab) or 1 (right slab): the
 * local contract index of each plane point, plane points ordered j fastest then
 * k (interior points only).  idx == NULL: *n = n_Gamma. */
osm_status osm_get_interface_map(osm_ctx* ctx, int iface, int side, int32_t* idx, int64_t* n);
/* The interface mass matrix M_Gamma (n_Gamma rows, plane-point order, CSR). */
osm_status osm_get_interface_mass(osm_ctx* ctx, int64_t* rowptr, int32_t* col, double* val, int64_t* nrows,
                                  int64_t* nnz);

/* S_Gamma values (the OO2 tangential stiffness), aligned with osm_get_interface_mass's pattern.
 * val == NULL: *nnz only. */
osm_status osm_get_interface_stiffness(osm_ctx* ctx, double* val, int64_t* nnz);

/* Device-timing instrumentation: events around every launch of the named
 * kernels, on the library stream.  Reset on enable. */
osm_status osm_set_kernel_timing(osm_ctx* ctx, int enable);
osm_status osm_get_kernel_timing(osm_ctx* ctx, osm_kernel_time* out, int cap, int* n);

/* Algorithmic HBM bytes of one PCG iteration of local subdomain-set work,
 * summed over this rank's subdomains weighted by their inner iteration counts in
 * the last solve: out[0] = SpMV kernel bytes (in the format of the
 * SpMV variant that ran), out[1] = update kernel bytes, out[2] = direction kernel bytes,
 * out[3] = SELL padding entries, out[4] = structural nnz (local), out[5] = local rows,
 * out[6] = SpMV bytes of the CSR-equivalent fp64 format (12 nnz + 4 (n+1) + 16 n), out[7] = bytes
 * this rank sent through NCCL in the interface exchanges of the last solve. n <= 8.  With timing
 * on, osm_get_kernel_timing also reports "exchange": the NCCL exchange calls on the stream. */
osm_status osm_get_traffic_model(osm_ctx* ctx, double* out, int n);

/* Host-only distribution plan (no GPU needed): subdomains [s_begin, s_end) of `rank`, and
 * its interface sides in the order the library uses them.  Per Schwarz iteration the
 * library exchanges, for every remote side: [g | u] (2 n_Gamma doubles) both ways with
 * `peer`; then the right slab of the interface (side 1) sends its interface-row
 * residual (n_Gamma doubles) to the left slab (side 0), which owns those rows of h(n);
 * then an allgather of one residual partial per subdomain (summed in subdomain order).
 * n_Gamma = (o ny - 1)(o nz - 1).  INVALID_ARG as osm_decompose. */
typedef struct osm_plan_side {
  int iface;  /* interface i, between slabs i and i+1 */
  int side;   /* 0: owner slab is the left slab (its right plane), 1: the right slab */
  int sub;    /* owning subdomain */
  int remote; /* neighbour slab on another rank */
  int peer;   /* rank of the neighbour slab */
} osm_plan_side;
osm_status osm_plan(int64_t nx, int nsub, int nranks, int rank, int* s_begin, int* s_end, osm_plan_side* sides,
                    int cap, int* nsides);

/* SpMV implementation of the PCG kernels (the local solves' sparse
 * matrix-vector product).  Every variant stores the assembled K_s = K_s^N + p M_Gamma + q S_Gamma
 * (values copied exactly, never recomputed) and forms each row's sum in the row's column order, so
 * the variants of one row order give the same q; the p.q reduction order differs between the tile
 * variants (per 256-row tile) and the brick variant (per brick):
 *   2  fp64 SELL-256 (value + int32 column per entry);
 *   3  value-indexed SELL: 16-bit dictionary index + 16-bit column offset per entry, dictionary
 *      through L1;  6 = 3 with the dictionary in the constant bank (<= 2048 distinct values);
 *   7  6 on wide entries (12-bit index, 20-bit offset), chosen automatically when offsets need it;
 *   10 3-byte entries: an int16 offset stream and a u8 dictionary-index stream (<= 256 values);
 *   11 (default) brick copy: needs row order 6; the p values of a lattice brick are staged in
 *      shared memory by TMA and the matrix is a u8 dictionary-index stream, one byte per (row,
 *      stencil slot) with the slots in column order (<= 256 values);
 *   5  matrix-free Kuhn stencil: per-(class, row kind) tables built from
 *      and verified against the assembled rows; needs row order 4.
 * A variant whose format does not apply falls back: 11 -> 10 -> 6 -> 3 -> 2, 5 -> 6.  *active
 * (may be NULL) receives the variant that will actually run.  INVALID_ARG for other values. */
osm_status osm_set_spmv_variant(osm_ctx* ctx, int variant, int* active);

/* Internal row order of the GPU copy (a permutation private to the library; results are
 * independent of it up to reduction order).  6 (default): the brick layout of variant 11, per
 * subdomain one dense array per lattice parity class (class-local jj fastest, then ii, then kk).
 * 0 SELL rows by length in sigma windows; 1 by parity class; 2 class then length; 3 class,
 * length, then lattice (K, I, J); 4 the class-major lattice layout of the matrix-free variant:
 * every lattice point of the slab box has a row, the Dirichlet points being inert zero rows
 * (+4..12 % rows).  Must precede osm_assemble (STATE after it); INVALID_ARG outside 0..4 and 6. */
osm_status osm_set_row_order(osm_ctx* ctx, int order);

/* Number of this library's kernel launches on the context's stream since
 * creation (every kernel of setup, solve and readback). */
osm_status osm_get_launch_count(osm_ctx* ctx, int64_t* n);

/* ---- Transmission-coefficient optimisation (host only, no GPU needed) ----
 * Fourier convergence rate of the two-subdomain OSM on R^2, f = 0: with
 * Lambda_s(k) = p_s + q_s k^2 (sign reading SURVEY Q25),
 *   rho(k) = |(Lambda_1 - k)/(Lambda_1 + k)| |(Lambda_2 - k)/(Lambda_2 + k)|.
 * osm_rate_max: max over nsamp geometric samples of [kmin, kmax] (PAPER.md:82 cost), and its argmax.
 * osm_rate_curve: rho at n given frequencies (Fig. "Fourier convergence rate"). */
osm_status osm_rate_max(double p1, double q1, double p2, double q2, double kmin, double kmax, int nsamp, double* rho,
                        double* kargmax);
osm_status osm_rate_curve(double p1, double q1, double p2, double q2, const double* k, int n, double* rho);

/* CMA-ES (population lambda = 25 in the paper).  Standard
 * (mu/mu_w, lambda) updates with cumulative step-size adaptation and rank-one + rank-mu covariance
 * adaptation.  ask: the caller supplies lambda x n standard normal draws z (row-major) and gets
 * x_k = m + sigma C^{1/2} z_k (symmetric square root).  tell: lambda costs (non-finite = worst; ties
 * broken by sample index).  should_stop: 1 = max_iter reached, 2 = spread of the best cost over the
 * last 10 + ceil(30 n / lambda) generations < ftol (7200 / 5e-11), 3 = sigma sqrt(max
 * eig C) < 1e-14.  The handle owns its state; osm_cmaes_destroy frees it. */
typedef struct osm_cmaes osm_cmaes;
osm_status osm_cmaes_create(int n, int lambda, const double* mean, double sigma0, osm_cmaes** out);
void osm_cmaes_destroy(osm_cmaes* es);
osm_status osm_cmaes_ask(osm_cmaes* es, const double* z, double* x);
osm_status osm_cmaes_tell(osm_cmaes* es, const double* f);
osm_status osm_cmaes_state(osm_cmaes* es, double* mean, double* sigma, double* cov, double* best_x, double* best_f,
                           int* generation);
osm_status osm_cmaes_should_stop(osm_cmaes* es, int max_iter, double ftol, int* stop);
/* Dimension n and population lambda of the handle (0 for NULL). */
void osm_cmaes_dims(const osm_cmaes* es, int* n, int* lambda);

/* [collective] CMA-ES over the batched-alpha solver (population
 * lambda = 25 at P:95, stopping rule P:171): es must have n = 1 (x = log alpha, both sides) or n = 2
 * (x = (log alpha_left, log alpha_right)), lambda <= 64, and was made by osm_cmaes_create.  Each
 * generation g asks lambda candidates from the caller's standard normals z[g][lambda][n] (host), solves
 * all of them in ONE batched solve (osm_solve_batch semantics: OO0, every interface the same pair,
 * n_outer outer iterations, tol_inner 1e-10, warm start) and tells es the costs
 * cost_b = (h_b(n_outer) / h_b(k0))^(1/(n_outer - k0)) (the empirical contraction, SURVEY 8(d) C4;
 * 1 when a history is unusable).  costs[g][lambda] (host, may be NULL) receives them.  Stops after gens
 * generations or when osm_cmaes_should_stop(es, max_iter, ftol) says so; *gens_done = generations run.
 * INVALID_ARG on bad sizes; STATE without interfaces. */
osm_status osm_cmaes_batch_optimize(osm_ctx* ctx, osm_cmaes* es, int gens, const double* z, int n_outer, int k0,
                                    int max_iter, double ftol, double* costs, int* gens_done);

#ifdef __cplusplus
}
#endif
#endif /* OSM_H_ */

/*
 * msp.h — C-ABI of the B200-native MSP-GMRES SOLVE phase (libmsp.so).
 *
 * Method: Zhao, Zhang, Feng, Shu, "An Improved Multi-Stage Preconditioner on GPUs
 * for Compositional Reservoir Simulation", arXiv 2208.08594 (= PAPER.md; "P:n" is
 * PAPER.md line n).  Restarted GMRES(m) right-preconditioned by the
 * multi-stage preconditioner of Eq. 21 / Alg. 1: a pressure stage
 * Π_P B_P W^T (B_P = UA-AMG V-cycle with NPAIR aggregation, PGS-MC smoothing over the
 * adjacency-graph coloring of Alg. 2-4, direct coarsest solve)
 * followed by the block smoother R = BILU(0) on the full block system.
 * Hierarchy setup is host C++ (timed separately); every SOLVE-phase step runs in
 * hand-written sm_100a CUDA kernels.  Readings of paper gaps: DESIGN.md §3.
 *
 * Conventions for every entry point:
 *  - Return value is an msp_status.  On any status other than MSP_OK / MSP_ENOCONV
 *    the outputs are unspecified and msp_last_error(handle) (or msp_last_error(NULL)
 *    when no handle exists yet) gives the stage name and the offending row/cell.
 *  - The caller owns every array it passes.  msp_setup deep-copies A; no caller
 *    pointer is retained after a call returns.
 *  - A handle is single-owner and not re-entrant; distinct handles are independent.
 *  - All GPU work of every call is ordered after prior work on the caller's stream (the
 *    `cuda_stream` of msp_setup, changeable by msp_set_stream; 0 = legacy default
 *    stream) and the call returns after it has completed.
 *  - A handle whose (re)SETUP failed (msp_update rebuild) is unusable: compute calls
 *    return MSP_EINVAL until an msp_update rebuild succeeds.  The previous
 *    preconditioner is not kept.
 *  - Sizes are element counts unless stated.  FP64 everywhere (R9).
 */
#ifndef MSP_H_
#define MSP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MSP_OK = 0,
  MSP_EINVAL = 1,      /* bad shape / unsorted or duplicate column / block != nc+1 / bad pointer */
  MSP_ESINGULAR = 2,   /* zero A_PP diagonal, singular N-N block (decoupling), singular BILU pivot
                          block or singular coarsest matrix; index in msp_last_error */
  MSP_ENOCONV = 3,     /* maxit reached: x, history and final residual are still valid */
  MSP_EBREAKDOWN = 4,  /* happy breakdown (h_{j+1,j} < 1e-14 ||b||, an invariant Krylov space)
                          with the true residual still above tol: restarting cannot help;
                          x, history and final residual are valid */
  MSP_ESTALL = 5,      /* AMG coarsening stalled above coarsest_max_dof on a non-diagonal level */
  MSP_ECUDA = 6,       /* CUDA runtime / cuSOLVER error (message in msp_last_error) */
  MSP_ENCCL = 7,       /* NCCL error (distributed entry points) */
  MSP_ENOMEM = 8       /* device allocation failed */
} msp_status;

/* Block-sparse Jacobian A_RR of Eq. 20 in BSR form.
 *  n_cells rows/columns of b x b blocks, b = block = nc + 1 (unknown 0 is the
 *  pressure P, unknowns 1..nc are N_1..N_nc).
 *  row_ptr[n_cells+1] (row_ptr[0] = 0), col_idx[nnzb] strictly ascending per row,
 *  values[nnzb*b*b]: each block ROW-major.  Every row must store its diagonal block.
 *  device = -1: host pointers; >= 0: pointers live on that CUDA device. */
typedef struct {
  int64_t n_cells;
  int32_t block;
  const int32_t* row_ptr;
  const int32_t* col_idx;
  const double* values;
  int32_t device;
} msp_bsr;

/* Device allocation callback (e.g. the PyTorch caching allocator).  NULL = cudaMalloc.
 * `stream` is the caller's stream (msp_setup / msp_set_stream): the library's own stream
 * waits on it before using the memory, and the library synchronises its stream before
 * every free, so a stream-keyed caching allocator may reuse blocks across handles. */
typedef void* (*msp_alloc_fn)(size_t bytes, void* stream, void* ctx);
typedef void (*msp_free_fn)(void* ptr, void* ctx);

/* Solver configuration.  msp_config_default() fills the paper's / DESIGN.md's values. */
typedef struct {
  int32_t coarsest_max_dof;  /* 10000: "degree of freedom of the coarsest space" */
  int32_t max_levels;        /* 20, including the coarsest */
  int32_t pre_sweeps;        /* 1 PGS-MC pre-sweep, colors 1..g (R6) */
  int32_t post_sweeps;       /* 1 PGS-MC post-sweep, colors g..1 (R6) */
  int32_t pair_passes;       /* 2 NPAIR passes per level (R3) */
  int32_t decoupling;        /* 0 NONE (W = Π_P), 1 QI, 2 TI (default, R4) */
  int32_t bilu_order;        /* 0 RB (Alg. 2/3 cell colors), 1 ABMC1 (default, R5) */
  int32_t stages;            /* 2 = P,R (north_star, default); 3 = N,P,R (full Eq. 21) */
  int32_t orth;              /* GMRES Arnoldi orthogonalisation: 2 DCGS2 (default, R14: CGS2's
                                basis with the re-orthogonalisation delayed by one step, two
                                passes over the basis per step instead of three); 0 CGS2 (R8);
                                1 MGS */
  int32_t use_graphs;        /* 1: replay each Arnoldi step as a CUDA graph (default) */
  int32_t use_coop;          /* must be 0 (a cooperative persistent V-cycle existed in round 1 and
                                measured slower than graph replay: removed; 1 -> MSP_EINVAL) */
  int32_t smoother;          /* AMG smoother (NEXT-4, reading R13): 0 PGS-MC (Alg. 4,
                                default), 1 PJAC-NO (Jacobi), 2 PGS-NO (hybrid Jacobi/GS:
                                natural-order chunks of gs_chunk rows, GS inside a chunk) */
  int32_t gs_chunk;          /* PGS-NO chunk size K (default 32) */
  msp_alloc_fn alloc;        /* optional device allocator */
  msp_free_fn free_fn;
  void* alloc_ctx;
  int32_t coarse_mode;       /* distributed handles: 0 (default) levels >= 1 and the
                                coarsest replicated on every rank (allgather of the level-1
                                right-hand side); 1 ROOT: agglomerated onto rank 0, which runs them
                                and broadcasts the level-1 correction (north_star's "coarse levels
                                are agglomerated onto one GPU"; bit-identical iterates) */
  int32_t bilu_local;        /* distributed handles: 0 (default) BILU(0) of the whole matrix (the
                                single-GPU preconditioner; halo exchanges after every color
                                phase); 1 rank-local BILU: couplings between cells of different
                                ranks removed before the factorization (block Jacobi across the
                                slabs; no exchange in the substitutions; the preconditioner then
                                depends on the partition).  Single-GPU handles: must be 0. */
  int32_t dist_levels;       /* distributed handles (NEXT-3): AMG levels 1..dist_levels are
                                partitioned like level 0 (a level-l row lives on the owner of
                                its lowest-index member; general ghost lists per level, a halo
                                per color in the sweeps, member / parent halos for the
                                restriction / prolongation) and only the levels below run
                                replicated (or on rank 0, coarse_mode 1).  0 (default): levels
                                >= 1 replicated; clamped to the number of smoothed levels - 1.
                                Bit-identical iterates for every value.  Single-GPU: ignored. */
} msp_config;

typedef struct msp_handle msp_handle;

typedef struct {
  int32_t setup_calls;       /* SETUP executions (ASMSP SetupCalls) */
  int32_t reuse_calls;       /* msp_update calls that reused the preconditioner */
  double setup_seconds;      /* host setup + upload, cumulative (wall clock) */
  double last_setup_seconds;
  double solve_seconds;      /* cumulative device time of msp_solve (CUDA events) */
  int32_t levels;            /* AMG smoothing levels L (coarsest is level L) */
  int32_t n_coarsest;
  int32_t bilu_colors;       /* block colors g_B of the BILU ordering */
  int32_t level_n[24];       /* rows per level 0..L */
  int64_t level_nnz[24];
  int32_t level_colors[24];  /* PGS-MC colors per smoothing level */
  int64_t device_bytes;      /* device memory held by the handle */
  int32_t kernels_per_iter;  /* kernel launches of one Arnoldi step */
  int32_t fused_a8;          /* always 0 (the a8-in-BILU fusion measured slower and was removed) */
} msp_stats;

void msp_config_default(msp_config* cfg);

/* SETUP (Alg. 1 preamble; §8(a) S1-S4): decoupling weights W and A_PP = W^T A Π_P,
 * PGS-MC coloring per AMG level (Alg. 2/3 on Eq. 23's graph), NPAIR aggregation and
 * Galerkin A_{l+1} = P^T A_l P, coarsest dense inverse, ABMC ordering, BILU(0)
 * factorization; upload.  nc = number of components (block must equal nc+1).
 * cfg NULL = defaults.  On success *out owns all device memory of the solver. */
msp_status msp_setup(const msp_bsr* A, int nc, const msp_config* cfg, void* cuda_stream,
                     msp_handle** out);

/* ASMSP: for Newton step iota with matrix A_new, rebuild the
 * preconditioner iff iota == 1, last_iterations > mu, or the size changed
 * (Remark 2); otherwise keep all stage operators and only replace A's values
 * used by SpMV and the Alg. 1 residuals.  *did_setup = 1 if rebuilt. */
msp_status msp_update(msp_handle* h, const msp_bsr* A_new, int iota, int last_iterations, int mu,
                      int* did_setup);

/* SOLVE: restarted right-preconditioned GMRES(restart) to ||b-Ax||/||b|| <= tol.
 * b[n*block], x[n*block] in the caller's natural cell order, cell-interleaved
 * (unknown 0 = pressure).  Host or device pointers (detected); x is read as x0 and
 * overwritten with the solution.  *iterations = Arnoldi steps.  resid_hist
 * (caller-owned HOST buffer, may be NULL) receives |gamma_{j+1}|/||b|| per Arnoldi
 * step and the true relative residual at each cycle end, truncated at hist_cap. */
msp_status msp_solve(msp_handle* h, const double* b, double* x, double tol, int restart, int maxit,
                     int* iterations, double* final_rel_res, double* resid_hist, int hist_cap,
                     int* hist_len);

/* One MSP application w = B g (Alg. 1 with w = 0 on entry), natural order; host or
 * device pointers.  For parity tests. */
msp_status msp_apply(msp_handle* h, const double* g, double* w);

msp_status msp_get_stats(const msp_handle* h, msp_stats* out);
const char* msp_last_error(const msp_handle* h);
void msp_destroy(msp_handle* h);

/* ---- Kernel-level entry points (parity tests and bench; device pointers, internal
 * order of the handle) ---- */

/* y = A x with the handle's BSR (a2, K1); vectors in the handle's internal (ABMC) cell
 * order, length n*block, device pointers. */
msp_status msp_spmv(msp_handle* h, const double* x, double* y);
/* One PGS-MC sweep (Alg. 4) on AMG level l: b, x of length level_n[l] in natural level
 * order (device); ascending != 0 -> colors 1..g, else g..1. */
msp_status msp_pgs_sweep(msp_handle* h, int level, const double* b, double* x, int ascending);
/* One V-cycle B_P r (natural level-0 = cell order, device). */
msp_status msp_vcycle(msp_handle* h, const double* r, double* x);
/* R r: BILU(0) forward/backward substitution (natural order, device). */
msp_status msp_bilu_apply(msp_handle* h, const double* r, double* x);
/* BILU(0) factors held by the handle (R5), for parity tests: F_out (HOST, nnzb*b*b doubles,
 * caller-allocated) receives row-major blocks in the caller's natural entry order: the L
 * and U blocks of the factorization, and D~_i^-1 in the diagonal slots.  Single-GPU
 * handles only (MSP_EINVAL otherwise). */
msp_status msp_bilu_factors(msp_handle* h, double* F_out);
/* ---- Single steps of the hot path, for the per-kernel parity tests (device pointers,
 * single-GPU handles; each call returns after its work completed).  Each runs the same
 * kernel the solve runs for that step. ---- */
/* a3 (R4; Π_P^T of Alg. 1 line 4, with the decoupling weights): rp = W^T g.
 * g: n_cells*block doubles, natural cell order; rp: n_cells doubles, natural cell order. */
msp_status msp_restrict_pressure(msp_handle* h, const double* g, double* rp);
/* a5 (UA-AMG residual + restriction): bc = P_l^T (b - A_l x) on smoothing level l.
 * b, x: level_n[l] doubles in the level's natural row numbering (the oracle's); bc:
 * level_n[l+1] doubles in level l+1's natural numbering (aggregate creation order). */
msp_status msp_residual_restrict(msp_handle* h, int level, const double* b, const double* x, double* bc);
/* a7 (prolongation + correction): x += P_l e; e: level_n[l+1], x: level_n[l]
 * (in/out), natural numberings as above. */
msp_status msp_prolong(msp_handle* h, int level, const double* e, double* x);
/* a8 (Alg. 1 line 5, with w = Π_P x_p): r = g - A Π_P x_p, reading only the pressure
 * column of each block.  g, r: n_cells*block; xp: n_cells; natural cell order. */
msp_status msp_pcol_residual(msp_handle* h, const double* g, const double* xp, double* r);
/* a9 halves (Alg. 1 line 6; BILU(0) in ABMC order, R5): forward y = L^-1 r (all
 * block colors ascending), backward x = U^-1 y (all colors descending, D~^-1 applied).
 * Natural cell order, n_cells*block doubles. */
msp_status msp_bilu_forward(msp_handle* h, const double* r, double* y);
msp_status msp_bilu_backward(msp_handle* h, const double* y, double* x);
/* a10 (Arnoldi orthogonalisation pass): out[i] = V_i^T w for i < k <= 32 with the
 * multi-vector dot kernel.  V: k vectors of n_cells*block doubles, consecutive (device);
 * w: device; out: HOST, k doubles. */
msp_status msp_multidot(msp_handle* h, int k, const double* V, const double* w, double* out);
/* Test hook: replace the handle's BILU factors by F (HOST, nnzb*block*block doubles,
 * natural entry order, row-major blocks, D~_i^-1 in the diagonal slots -- the layout of
 * msp_bilu_factors), e.g. with integer-valued factors for bit-exact substitution tests. */
msp_status msp_bilu_set_factors(msp_handle* h, const double* F);
/* SETUP step S1 as the handle computed it (NEXT-2: on the GPU unless MSP_HOST_SETUP=1):
 * W[n_cells*block] decoupling weights and App[nnzb] the A_PP values in the caller's
 * natural entry order (pattern = A's), both HOST buffers; *on_gpu = 1 if computed on the
 * GPU.  For the bit-exact parity tests against the host setup and the oracle. */
msp_status msp_get_s1(const msp_handle* h, double* W, double* App, int32_t* on_gpu);
/* The caller's stream: every entry point orders the handle's work after the work queued
 * on it (default: the stream given to msp_setup; 0 = legacy default stream). */
msp_status msp_set_stream(msp_handle* h, void* cuda_stream);

/* Times `reps` launches of one hot-path piece on the handle's stream with CUDA events,
 * flushing L2 before each launch by READING a 256 MB buffer (clean lines: no write-back of
 * unrelated dirty data inside the timed launch).  Returns the mean device
 * milliseconds per launch and the ALGORITHMIC bytes per launch (compulsory
 * traffic, each vector counted once).  kind: 0 a2 BSR SpMV; 1 a4 level-0 PGS-MC sweep
 * (all colors, descending = full work per color); 2 a8 pressure-column residual;
 * 3 a9 BILU(0) apply (all colors); 4 a10 CGS2 pass A (dot) over 16 basis vectors;
 * 5 a6 coarsest dense-inverse GEMV; 6 one whole MSP application; 7 one V-cycle B_P;
 * 8 BILU apply; 9 one whole Arnoldi step (j = 15); 10 the CGS2 of step 15 (55 vectors);
 * 11/12 Arnoldi step / CGS2 at j = 25; 13 a9 + SpMV; 14 MSP application + SpMV;
 * 15 SpMV + orthogonalisation of step 15; 16 + l (0 <= l <= L, L = the number of
 * smoothed AMG levels): the V-cycle from level l down (l = L: the coarsest solve alone), so
 * the time spent AT level l is T(16 + l) - T(17 + l) (bytes = 0 for kinds 6-9, 11, 13-15, >= 16; kind 12 counts DCGS2 only).
 * kind | 0x100: no L2 flush (warm caches).  Each piece is captured once into a CUDA graph and replayed (as in the solve); the first replay is a warm-up.
 * Scratch contents of the handle are overwritten. */
msp_status msp_time_kernel(msp_handle* h, int kind, int reps, double* ms_per_launch,
                           double* bytes_per_launch);
/* Number of CUDA kernels launched by the handle so far (graph replays counted per kernel). */
int64_t msp_kernel_launches(const msp_handle* h);
/* Internal cell order: order[p] = natural cell at position p (host buffer n_cells). */
msp_status msp_get_order(const msp_handle* h, int32_t* order);

/* ---- Host-setup introspection (no GPU needed): runs setup steps S1-S4 on the host
 * only and exposes the integer structures and Galerkin values for bit-exact parity
 * against the oracle. ---- */
typedef struct msp_host_setup msp_host_setup;
msp_status msp_host_setup_run(const msp_bsr* A, int nc, const msp_config* cfg,
                              msp_host_setup** out);
/* sizes: out[0]=levels L, out[1]=n_coarsest, out[2]=coarse_diag, out[3]=bilu colors */
msp_status msp_host_setup_info(const msp_host_setup* s, int32_t* out4);
/* level l (0..L; l == L is the coarsest): n, nnz, colors */
msp_status msp_host_setup_level_dims(const msp_host_setup* s, int level, int32_t* n, int64_t* nnz,
                                     int32_t* ncolors);
/* level CSR in NATURAL level numbering (ptr[n+1], col[nnz], val[nnz]) */
msp_status msp_host_setup_level_csr(const msp_host_setup* s, int level, int32_t* ptr, int32_t* col,
                                    double* val);
/* color of each row (natural numbering), smoothing levels only */
msp_status msp_host_setup_level_colors(const msp_host_setup* s, int level, int32_t* color);
/* composite aggregate of each row of level l (l < L) */
msp_status msp_host_setup_level_agg(const msp_host_setup* s, int level, int32_t* agg);
/* decoupling weights W[n*block] and BILU cell order[n] */
msp_status msp_host_setup_weights(const msp_host_setup* s, double* W);
msp_status msp_host_setup_order(const msp_host_setup* s, int32_t* order);
void msp_host_setup_free(msp_host_setup* s);

/* ---- Multi-GPU: z-slab row partition, NCCL halo + allreduce ---- */
/* Distributed SETUP on rank `rank` of `nranks` (one process per GPU).  A_global_host:
 * the whole matrix on every rank (every rank runs the same deterministic host setup, so
 * the preconditioner equals the single-GPU one); owner[n_cells] = rank of every cell
 * (e.g. z-slabs from msp_partition_owner), NULL = contiguous index ranges.  Every ABMC
 * block / level-1 aggregate is assigned whole to the owner of its lowest-index cell.
 * Each rank keeps its rows plus ghost cells; halos (ncclSend/ncclRecv) follow every
 * level-0 PGS-MC color and every BILU color phase, dot products use ncclAllReduce and
 * the replicated coarse levels receive the level-1 right-hand side by ncclAllGather.
 * nccl_unique_id: 128 bytes from msp_nccl_unique_id() on rank 0, broadcast by the
 * caller.  Supports stages=2, 1 pre/post sweep, ABMC1 order.  Afterwards msp_solve /
 * msp_update / msp_apply take this rank's owned cells (ascending natural cell id, see
 * msp_dist_owned_cells); all ranks must call them collectively. */
msp_status msp_nccl_unique_id(void* id128);
msp_status msp_setup_dist(const msp_bsr* A_global_host, int nc, const msp_config* cfg, const int32_t* owner,
                          const void* nccl_unique_id, int rank, int nranks, void* cuda_stream,
                          msp_handle** out);
int32_t msp_dist_n_owned(const msp_handle* h);
msp_status msp_dist_owned_cells(const msp_handle* h, int32_t* cells);
/* Test harness of the distributed path on ONE GPU: nranks virtual ranks as host threads,
 * each with its own handle and stream; halos/collectives are device copies ordered by
 * CUDA events (no kernel waits on another).  b, x: global natural order (x in: x0, out:
 * solution).  rank_info (optional, 4*nranks): n_own, n_ghost, level-0 rows, level-0
 * ghosts per rank. */
msp_status msp_loopback_solve(const msp_bsr* A, int nc, const msp_config* cfg, const int32_t* owner, int nranks,
                              const double* b, double* x, double tol, int restart, int maxit,
                              int* iterations, double* final_rel_res, int32_t* rank_info);
/* Host-side partition plan (no GPU): owner rank of each cell for `nranks` z-slabs of
 * an nx*ny*nz grid (cell c = i + nx*(j + ny*k)), aggregate-owner rule (cells follow
 * the owner of the lowest-index cell of their level-1 aggregate). */
msp_status msp_partition_owner(const msp_host_setup* s, int nx, int ny, int nz, int nranks,
                               int32_t* owner);
/* Host-only halo plan of the cell space for `rank` (what msp_setup_dist builds; no GPU):
 * owned_cells[n_own] natural ids in local order, ghost_cells[n_ghost] natural ids in
 * receive order (grouped by source rank, then BILU color); send_cells (natural ids, size
 * <= n*nranks) in send order per destination rank with offsets send_ptr[nranks+1];
 * recv_ptr[nranks+1] ghost offsets per source rank.  owner NULL = index ranges. */
msp_status msp_dist_plan(const msp_host_setup* s, const int32_t* owner, int rank, int nranks, int32_t* n_own,
                         int32_t* owned_cells, int32_t* n_ghost, int32_t* ghost_cells, int32_t* send_ptr,
                         int32_t* send_cells, int32_t* recv_ptr);
/* Host-only plan of a PARTITIONED AMG level (msp_config.dist_levels, SURVEY §8(e)
 * "distribute levels 1..k"; no GPU): for `rank` of `nranks` (cell owners as msp_dist_plan),
 * level 1 <= level < number of smoothed levels.  Serialised into buf (int32, capacity cap;
 * *len = required length; buf NULL: length only), natural row ids of the level throughout:
 *   n_own, n_gx, n_gp, n_gm, owned rows (global row order), matrix ghosts, parent ghosts,
 *   member ghosts (each in receive order: peer-major, then global row order), then for every
 *   peer q = 0..nranks-1: [count, rows sent to q for its matrix ghosts], [count, parent
 *   ghosts sent], [count, member ghosts sent] (send order = the peer's receive order), then
 *   the level's row count m, the owner of every row (m) and the global (color-major) row
 *   index of every row (m). */
msp_status msp_dist_level_plan(const msp_host_setup* s, const int32_t* owner, int rank, int nranks, int level,
                               int32_t* buf, int64_t cap, int64_t* len);

#ifdef __cplusplus
}
#endif
#endif /* MSP_H_ */

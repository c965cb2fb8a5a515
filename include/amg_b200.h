/*
 * amg_b200.h — C ABI of the B200-native solve path of arXiv 2511.21268 (D'Ambra, Durastante,
 * Filippone, "Parallel matching-based AMG preconditioners for elliptic equations discretized by
 * IgA"): fp64 PCG on the IgA Poisson stiffness system K u = F, preconditioned by one V-cycle of a
 * compatible-weighted-matching AMG hierarchy with Chebyshev-accelerated ℓ1-Jacobi smoothing.
 *
 * Citations "P:Lnnn" are lines of the paper text; "c.N" are the readings listed in
 * DESIGN.md §3 (taken from SURVEY.md §8(c)).
 *
 * Conventions for every entry point:
 *   - All functions return amg_status.  No C++ exception crosses the ABI.  On a non-OK status the
 *     thread-local message from amg_last_error() says what failed; output arguments are then
 *     unspecified unless stated otherwise.
 *   - Input arrays are BORROWED for the duration of the call (copied when kept).  Every output the
 *     library allocates is released by the matching amg_*_free / amg_free.
 *   - Matrices are CSR, 0-based, int64 row pointers, int32 columns sorted strictly ascending in each
 *     row, fp64 values (amg_csr).
 *   - A hierarchy handle may be used by one host thread at a time.
 *   - There is no CPU fallback: solve-phase entry points need a CUDA device (sm_100a) and return
 *     AMG_ENODEV / AMG_ECUDA without one.
 */
#ifndef AMG_B200_H
#define AMG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    AMG_OK = 0,
    AMG_NOT_CONVERGED = 1, /* outputs valid; iters == maxit and relres > rtol                  */
    AMG_EINVAL = -1,       /* bad argument (NULL, size mismatch, unsupported option)            */
    AMG_ENOMEM = -2,       /* host or device allocation failed                                  */
    AMG_ECUDA = -3,        /* CUDA runtime error (message has the CUDA error string)            */
    AMG_ENCCL = -4,        /* NCCL error (multi-GPU)                                            */
    AMG_ENOTSPD = -5,      /* d̂_i <= 0, missing diagonal, pᵀKp <= 0 or rᵀz <= 0 (CG breakdown)  */
    AMG_ENODEV = -6        /* no usable CUDA device                                             */
} amg_status;

/* Host CSR matrix (n_rows x n_cols, nnz entries). */
typedef struct {
    int64_t n_rows, n_cols, nnz;
    int64_t *row_ptr; /* n_rows + 1 */
    int32_t *col;     /* nnz, strictly ascending within a row */
    double *val;      /* nnz */
} amg_csr;

/* ---------------------------------------------------------------------------------------------
 * Problem generator: tensor-product B-spline Poisson stiffness (eq:matrix_and_vector_
 * values P:L646-650) on the unit square (dim 2) or cube (dim 3) with n_elem uniform elements per
 * direction, degree `degree`, maximal regularity C^{p-1}.
 *
 * DOFs on Dirichlet sides are eliminated.  Side s (1..2*dim) is Dirichlet iff bit s-1
 * of dirichlet_sides is set; sides are 1:x=0 2:x=1 3:y=0 4:y=1 5:z=0 6:z=1; the paper's cube uses
 * sides 1,2,3 = 0x7.  Free DOFs are numbered lexicographically, x fastest (c.1).
 * K is assembled as the Kronecker sum of 1-D tables computed by (p+1)-point Gauss quadrature in
 * binary128 and rounded once (c.3, Remark P:L570-573), in the canonical order of DESIGN.md §3 (c.4).
 *
 * rhs = 0: F = load of the manufactured solution u* = sin(πx) sin(πy/2) [cos(πz)] (c.5);
 * rhs = 1: F = 0;
 * rhs = 2: the paper's own cube data (dim 3, Dirichlet sides 1,2,3 only):
 *          f = −e^{x+z} sin y, g_D = e^{x+z} sin y by one L2 projection onto the Dirichlet faces' trace
 *          space, Neumann g_N on sides 4-6; F = (source + Neumann load)_free − K_fD u_D (lifting).
 * Outputs: *K (free with amg_csr_free) and *F (length K->n_rows, free with amg_free).
 * Errors: AMG_EINVAL for dim ∉ {2,3}, degree ∉ [1,8], n_elem < 1, sides out of range, or more
 * than 2^31-1 free DOFs; AMG_ENOMEM.
 *
 * geometry = 1: the thick quarter ring of the paper (dim 3 only): inner radius 1, outer
 *          radius 2, height 1, exact NURBS circle, B-spline solution space (non-isoparametric, §3.3
 *          P:L592-605).  x = (1+u)c_x(v), y = (1+u)c_y(v), z = w; sides 1: u=0, 2: u=1, 3: v=0 (y=0),
 *          4: v=1 (x=0), 5: w=0, 6: w=1.  Since JᵀJ = diag(1, r²|c'|², 1), K = A_u⊗B_v⊗M_w +
 *          C_u⊗D_v⊗M_w + E_u⊗B_v⊗K_w with r- and |c'|-weighted 1-D tables (binary128 Gauss, rounded
 *          once), entry ((A·B)·M + (C·D)·M) + (E·B)·K.  rhs = 1: F = 0; rhs = 2: the paper's ring data
 *          (u = e^x sin(xy) cos z, f and g_N of eq:Lshapedcoeff; g_D by one L2 projection
 *          onto sides 1-3; source by (p+1)³ Gauss points through the map).
 *
 * geometry = 2: the three-patch thick L-shape (multipatch gluing P:L575-583; readings
 *          N4.a/N4.b of DESIGN.md §3; dim 3, dirichlet_sides must be 0x7 and is otherwise unused):
 *          patches A = [0,1]³, B = [1,2]×[0,1]², C = [0,1]×[1,2]×[0,1], each the unit-cube space of
 *          degree p on n³ elements, interface functions identified (C⁰).  Control lattice
 *          0 ≤ x, y ≤ 2m−2, 0 ≤ z ≤ m−1 without x, y ≥ m (m = n+p); Dirichlet faces x=0, y=0, x=2, y=2,
 *          z=0, z=1; Neumann faces y=1 (on B) and x=1 (on C).  Free DOFs lexicographic, x fastest
 *          (sizes: Table 2b).  Entries: Σ over the patches holding both functions, in order A, B, C,
 *          of the cube entry.  rhs = 0: F_i = ∫ φ_i (f = 1, homogeneous data); rhs = 1: F = 0;
 *          rhs = 2: the paper's L-shape data (u = e^x sin(xy) cos z, its f, g_N on the
 *          two Neumann faces, g_D by one joint L2 projection onto the glued Dirichlet faces, lifting;
 *          fp64 (p+1)-point Gauss).
 */
typedef struct {
    int dim;
    int degree;
    int n_elem;
    uint32_t dirichlet_sides;
    int rhs;
    int geometry; /* 0 unit square / cube, 1 thick quarter ring (dim 3), 2 three-patch L-shape (dim 3) */
} amg_iga_desc;

amg_status amg_iga_poisson(const amg_iga_desc *desc, amg_csr **K, double **F);

/* The rounded integer-knot (h = 1) 1-D tables M̂_ab = ∫N_aN_b, K̂_ab = ∫N'_aN'_b (c.3) in band
 * storage: mhat[a*(2p+1) + (b-a+p)], a = 0..n+p-1 (caller allocates (n+p)*(2p+1) doubles each;
 * entries with b outside 0..n+p-1 are 0).  For bitwise checks against exact rationals. */
amg_status amg_iga_tables(int degree, int n_elem, double *mhat, double *khat);

void amg_csr_free(amg_csr *K);
void amg_free(void *p);

/* ---------------------------------------------------------------------------------------------
 * Hierarchy parameters (defaults from amg_params_default; meaning in DESIGN.md §3).
 */
typedef struct {
    int agg_steps;          /* pairwise matchings per level: 3 -> aggregates of size <= 8 */
    int smooth_prolong;     /* 1: P̄ = (I − ω D_f⁻¹K_f) P; 0: tentative P            */
    double match_threshold; /* edge eligible iff c_ij > threshold (1.0, c.8)                          */
    double filter_theta;    /* strength filter for the prolongator smoothing matrix (0.01, c.12);
                               0 = literal (I − ωD⁻¹K)P                                                */
    int cheb_degree;        /* Chebyshev degree m = SpMVs per smoothing (p=3→8, 4→12, 5→14, 6→16; p=2→4) */
    int coarse_sweeps;      /* ℓ1-Jacobi sweeps on the coarsest level (30)                */
    int64_t coarse_size;    /* coarsest when N_l <= coarse_size (50)                 */
    int max_levels;         /* 20                                                                 */
    int format;             /* device matrix format: 0 auto (K_l and P̄_l with >= 2e6 non-zeros whose
                               column offsets (>= 16 bits, <= 24) and distinct-value indices fit one
                               32-bit word, <= 50 % slice padding, sampled row-to-row locality and, for
                               rows longer than 64 entries, <= 8192 distinct values: SELL-VI, a fixed rule; every
                               other operator: CSR rows padded to 8 with the
                               kernel, column and value source autotuned), 1 CSR warp-per-row,
                               2 SELL-32 (row per lane), 3 TMA-staged CSR, 4 CSR with 16-bit column
                               offsets (register core), 5 CSR with 16-bit column offsets (TMA-staged
                               values), 6 SELL-VI (row per lane, column offset + value index in one
                               32-bit word per entry) for every K_l, P̄_l, R_l that admits it, any size */
    int host_only;          /* 1: build the hierarchy on the host only (export/inspection; no CUDA call) */
    int num_threads;        /* host setup threads (OpenMP); 0 = runtime default                     */
    int krylov;             /* outer solver: 0 = PCG (c.19); 1 = flexible CG, Notay's FCG(1)
                               ("the flexible variant of the CG"): α = pᵀr/pᵀq, β = −zᵀq_prev/pᵀq_prev */
    int coarse_solver;      /* coarsest level: 0 = coarse_sweeps ℓ1-Jacobi sweeps (§4); 1 = CG
                               preconditioned by one weighted-Jacobi sweep (D = diag K_L) to coarse_tol
                               or coarse_maxit iterations (§5.1; a nonlinear preconditioner:
                               use krylov = 1) */
    double coarse_tol;      /* 1e-4 */
    int coarse_maxit;       /* 30 */
} amg_params;

/* Defaults for spline degree p (sets cheb_degree from the table above). EINVAL for p ∉ [1,8]. */
amg_status amg_params_default(amg_params *prm, int spline_degree);

/* Device allocator hook (e.g. PyTorch's caching allocator).  Unset -> cudaMalloc/cudaFree.
 * alloc returns NULL on failure.  Must be set before amg_setup; applies to hierarchies created after. */
typedef void *(*amg_alloc_fn)(size_t bytes, int device, void *cuda_stream);
typedef void (*amg_free_fn)(void *ptr, size_t bytes, int device, void *cuda_stream);
amg_status amg_set_allocator(amg_alloc_fn alloc, amg_free_fn free_fn);

/* Host threads (OpenMP) of this process's later library calls: generator, setup, share export/import,
 * device uploads (amg_params.num_threads overrides it inside amg_setup).  Launchers such as torchrun
 * set OMP_NUM_THREADS=1 per process; the shared setup gives rank 0 every core for the host setup and
 * each rank its share of the cores for its device setup.  AMG_EINVAL if n < 1. */
amg_status amg_set_num_threads(int n);

/* Multi-GPU descriptor: one process per GPU.  NULL or nranks == 1 -> single GPU `device`
 * (NULL -> the current device). */
typedef struct {
    int rank, nranks;
    unsigned char nccl_id[128]; /* ncclUniqueId from rank 0, broadcast by the caller */
    int device;
} amg_dist;

typedef struct amg_hierarchy amg_hierarchy; /* opaque, library-owned */

/* Rank 0 creates the NCCL unique id (128 bytes) and broadcasts it to the other ranks (e.g. with
 * torch.distributed) before they call amg_setup with amg_dist.  AMG_ENCCL on failure. */
amg_status amg_nccl_unique_id(unsigned char id[128]);

/* Multi-GPU row ownership: every level is split into contiguous row blocks balanced by
 * nnz; levels with nnz <= 7e6 (env AMG_REPLICATE_NNZ) and the coarsest are replicated on all ranks.
 * With nranks > 1, the F and u passed to amg_pcg_solve are this rank's rows [row_begin, row_end) of
 * level 0 (global numbering); every rank builds the same global hierarchy on the host from the same
 * full K (or receives its share of it: amg_share_export below).  Returns [0, N_0) on one GPU.  Host
 * information: also valid for host_only setups. */
amg_status amg_local_rows(amg_hierarchy *H, int64_t *row_begin, int64_t *row_end);

/* Builds the hierarchy of K on the host (deterministic; bitwise reproducible; c.6-c.15) and, unless
 * prm->host_only, uploads it to the device.  K is borrowed (copied).  K must be square, symmetric
 * and have a positive diagonal (else AMG_ENOTSPD).  prm NULL -> amg_params_default(·, 2).
 * *H is released with amg_hierarchy_free. */
amg_status amg_setup(const amg_csr *K, const amg_params *prm, const amg_dist *dist, amg_hierarchy **H);

/* amg_setup without the copy of K: the hierarchy takes K's three arrays over (they must come from the
 * library, e.g. amg_iga_poisson, i.e. be malloc'd) and K itself is released with amg_csr_free — in
 * every case, also on error; the caller must not touch K afterwards.  For the largest workloads, whose
 * K₀ alone is tens of GB (C5 at 4 GPUs: 94 GB of host RAM): it saves one copy of K at the setup's
 * peak.  Same parameters, results (bitwise) and errors as amg_setup. */
amg_status amg_setup_take(amg_csr *K, const amg_params *prm, const amg_dist *dist, amg_hierarchy **H);

/* PCG (c.19) preconditioned by one V-cycle per iteration (c.18).
 * F, u: DEVICE pointers (fp64, N = K->n_rows); u holds the initial guess on entry and the solution on
 * exit.  Stops when ‖r_k‖₂ <= rtol·‖F‖₂ (recurrence residual) or k == maxit; iteration count = number
 * of K·p products.  F == 0 -> u = 0, *iters = 0.  cuda_stream: cudaStream_t (NULL = legacy default).
 * resid_history: nullable host array of length maxit+1, receives ‖r_k‖/‖F‖.
 * The iterations run as ONE CUDA graph launch with a conditional WHILE node whose controller kernel
 * takes the stopping test on the device (env AMG_DEVICE_LOOP=0: one graph per iteration and the test
 * on the host; bitwise the same results).  The call returns when the solve is complete.
 * Returns AMG_OK, AMG_NOT_CONVERGED, AMG_ENOTSPD (breakdown), AMG_ECUDA, AMG_EINVAL. */
amg_status amg_pcg_solve(amg_hierarchy *H, const double *F, double *u, double rtol, int maxit,
                         void *cuda_stream, int *iters, double *relres, double *resid_history);

/* Same as amg_pcg_solve with HOST F and u (copied to / from the device inside the call). */
amg_status amg_pcg_solve_host(amg_hierarchy *H, const double *F, double *u, double rtol, int maxit,
                              void *cuda_stream, int *iters, double *relres, double *resid_history);

/* One V-cycle z = V(r) (c.18) on DEVICE vectors of length N_0. */
amg_status amg_vcycle(amg_hierarchy *H, const double *r, double *z, void *cuda_stream);

/* y = A x on the device for A = K_l (op 0), P̄_l (op 1, x has N_{l+1} entries) or R_l = P̄_lᵀ (op 2).
 * x must be 16-byte aligned (the windowed SELL-VI layout stages it with bulk copies; AMG_EINVAL
 * otherwise) and readable up to the next 16-byte boundary past its end. */
amg_status amg_level_apply(amg_hierarchy *H, int level, int op, const double *x, double *y,
                           void *cuda_stream);

/* Hierarchy summary; arrays sized >= max_levels (nullable).  nnz_P[l] = nnz(P̄_l) (0 on the
 * coarsest).  opc = Σ nnz(K_l)/nnz(K_0). */
amg_status amg_hierarchy_info(const amg_hierarchy *H, int64_t *n_levels, int64_t *N, int64_t *nnz,
                              int64_t *nnz_P, double *opc);

/* Host copies of level l's K_l, P̄_l (NULL on the coarsest), composite aggregate map (fine row ->
 * coarse index; NULL on the coarsest), ℓ1 diagonal d̂_l and ω_l.  Any output pointer may be NULL.
 * Free with amg_csr_free / amg_free. */
amg_status amg_hierarchy_export(const amg_hierarchy *H, int level, amg_csr **K_l, amg_csr **P_l,
                                int32_t **aggregate_of, double **dhat, double *omega);

/* Kernel timing of the dominant kernel (the fused Chebyshev step on level 0), recorded with CUDA
 * events on the launching stream while enabled.  bytes_per_launch is the ALGORITHMIC byte count of
 * one launch: the level-0 operator's alg_bytes in the format it is stored in (amg_op_config.alg_bytes:
 * 4 B per stored entry + table + row bases + slice offsets for SELL-VI; 8 B value + the column source
 * + 8 B row pointers per row for CSR) plus the epilogue's 56·N_0 vector bytes. */
typedef struct {
    int64_t launches;
    double total_ms;
    double bytes_per_launch;
    int64_t kernels_launched; /* all library kernels launched since the counter was reset */
} amg_kernel_stats;
amg_status amg_set_profiling(amg_hierarchy *H, int enable); /* enable resets the counters */
amg_status amg_get_kernel_stats(amg_hierarchy *H, amg_kernel_stats *st);

/* Device kernel chosen for operator op (0 K_l, 1 P̄_l, 2 R_l) of level l: layout (0 padded CSR,
 * 1 SELL-32, 2 SELL-VI: row per lane, column offset + value index in one 32-bit word per entry,
 * 3 windowed SELL-VI (single GPU): the multiplied vector's window of each block of 8 slices staged in
 * shared memory by TMA, window position + value index per word; its `kernel` = windows staged per CTA,
 * 1 or 2), kernel (CSR layouts: bit 0: 0 register-batched warp-per-row CSR, 1 TMA-staged CSR; bit 1: column
 * source, 0 int32 columns, 1 16-bit column offsets from a per-row base; bit 2: register core with an L2
 * bulk prefetch of the next row; bit 3: value source, 0 streamed fp64 values, 1 value index into the
 * operator's table of distinct values — CSR-VI, register core only), rows per warp group G, pairs per
 * lane per round trip U, stored entries (with padding), the autotuned y = A·x time in microseconds (0
 * if the heuristic choice was kept), the bytes one application streams for the operator in that format
 * (8 B per value, or the value index bytes + 8 B per distinct value, for the nnz entries + the column
 * data actually stored + 8 B row pointers; vectors excluded), nnz, the number of distinct values in
 * the value table (0: no value index built) and the bytes of one value index (2: packed with the 16-bit
 * column offset into one 32-bit word; 4; 0: none).  AMG_EINVAL for a bad level/op. */
typedef struct {
    int layout, kernel, G, U;
    int64_t stored;
    double tuned_us;
    double alg_bytes;
    int64_t nnz;
    int64_t n_values;
    int value_index_bytes;
    int sellvi_parts;       /* SELL-VI: quad-range parts (1, 2, 4; one warp each) of the 32-row slices of
                               the last round of work items, so that round is short (env
                               AMG_SELLVI_PARTS=k forces 2^k parts on every slice); the rows of a split
                               slice sum their parts' chains in part order.  0 other layouts */
    int offset_bits;        /* SELL-VI: column-offset bits of an entry word (16..24); windowed SELL-VI:
                               window-position bits; 0 other layouts */
} amg_op_config;
amg_status amg_operator_config(amg_hierarchy *H, int level, int op, amg_op_config *cfg);
/* Force the kernel configuration of one CSR-layout operator (experiments and the kernel-equivalence
 * tests): kernel as in the amg_op_config struct: bit 1 needs the 16-bit encoding (formats 0, 3, 4, 5, and
 * only where every row spans < 65536 columns); bit 0 = TMA needs rows padded to 8 and U <= 4; bit 2
 * (prefetch) needs the register core and rows padded to 8; bit 3 (value index) needs the register core
 * and a value table (built at setup for format 0 operators with >= 2e6 stored entries, >= 4 entries per
 * distinct value and <= 2^21 distinct values, unless env AMG_VALUE_INDEX=0); a SELL-VI operator
 * (layout 2) takes kernel 0, G 32 and U in {1, 2, 4} only, a windowed one (layout 3) kernel 1 or 2 (windows
 * staged per CTA), G 32 and U in {1, 2, 4}; G in {1,2,4,8,32}, U in {2,4,6,8}.  Every configuration
 * sums each row in the same order, so results are bitwise unchanged.  Drops captured PCG graphs.
 * AMG_EINVAL for a bad level/op or an unavailable configuration. */
amg_status amg_operator_set_config(amg_hierarchy *H, int level, int op, int kernel, int G, int U);

/* Per-level time breakdown of the V-cycles run since the last call (experiments): exclusive device
 * milliseconds per V-cycle of every level — its smoothing, residual, transfers and halo / lock-step
 * waits, without the coarser levels.  Recorded only for hierarchies created with the environment
 * AMG_PROF_LEVELS=1 and AMG_GRAPHS=0 (else zeros).  Resets the accumulation.  nlevels: the level count. */
amg_status amg_get_level_times(amg_hierarchy *H, double *ms_per_vcycle, int nmax, int *nlevels);

/* Host view of this rank's share of operator op (0 K_l, 1 P̄_l, 2 R_l) on level l, for hierarchies
 * set up with an amg_dist of nranks > 1 (host_only or not).  Local column indices keep the global
 * order: ghost[0..n_ghost-1] holds the ghost columns' global ids ascending, the first n_ghost_lo of them
 * (owned by lower ranks) have local indices g − n_ghost_lo (negative), owned global column
 * col_begin + j has local index j, and upper ghost g ≥ n_ghost_lo has col_end − col_begin + g − n_ghost_lo.
 * Ghost values are received from rank q for ghost positions recv_off[q] .. recv_off[q]+recv_count[q];
 * this rank sends the owned entries send_idx[send_off[q] .. send_off[q]+send_count[q]) (local indices)
 * to rank q.  All arrays are library-owned and valid until amg_hierarchy_free.  replicated = 1: the
 * level is held whole by every rank (no view).  AMG_EINVAL if the hierarchy is not distributed or
 * level/op is bad. */
typedef struct {
    int nranks, replicated, full_cols;
    int64_t row_begin, row_end, col_begin, col_end, n_ghost, n_ghost_lo;
    const int64_t *ghost;
    const int32_t *send_count, *send_off, *send_idx, *recv_count, *recv_off;
    amg_csr local;
} amg_dist_view;
amg_status amg_dist_view_get(const amg_hierarchy *H, int level, int op, amg_dist_view *view);

/* Shared setup for one process per GPU (the host hierarchy is built once, not once per
 * rank).  One process calls amg_setup on the full K with prm->host_only = 1 and dist = NULL, then
 * amg_share_export once per rank: *share receives a malloc'd blob (free with amg_free) of *bytes bytes
 * holding everything rank `rank` of an nranks-GPU run needs — the row bounds of every level, its local
 * operators and halo plans on the distributed levels (the same plan amg_setup with that amg_dist would
 * build), the replicated levels whole, every level's size, nnz, ω and ℓ1 diagonal.  The caller moves
 * the blob to that rank (e.g. torch.distributed).  AMG_EINVAL for a bad rank/nranks or a hierarchy
 * itself built from a share; AMG_ENOMEM.
 * Each rank then calls amg_setup_from_share with its blob and its amg_dist, whose rank/nranks must match the
 * export (NULL dist = rank 0 of 1): the result behaves like amg_setup's for that rank — same device
 * state, same kernels, bitwise the same solve — except that amg_hierarchy_export is unavailable
 * (AMG_EINVAL: the global operators are not held).  host_only = 1 skips the device part (for
 * amg_dist_view_get / amg_hierarchy_info); with host_only = 0 the host copies of this rank's operators
 * are freed once the device holds them (amg_dist_view_get then returns AMG_EINVAL; amg_hierarchy_info and
 * amg_local_rows keep working).  The blob is borrowed (copied); AMG_EINVAL on a truncated or corrupt
 * blob. */
amg_status amg_share_export(const amg_hierarchy *H, int rank, int nranks, void **share, int64_t *bytes);
amg_status amg_setup_from_share(const void *share, int64_t bytes, const amg_dist *dist, int host_only,
                                amg_hierarchy **H);
/* amg_setup_from_share that takes the blob over: it is freed (std::free) as soon as it is imported —
 * in every case, also on error — so a rank does not hold the blob and its imported copy through the
 * device setup.  The blob must come from amg_malloc (or amg_share_export). */
amg_status amg_setup_from_share_take(void *share, int64_t bytes, const amg_dist *dist, int host_only,
                                     amg_hierarchy **H);
/* Host allocation the library may free (receive buffers for amg_setup_from_share_take); NULL on failure. */
void *amg_malloc(int64_t bytes);

void amg_hierarchy_free(amg_hierarchy *H);

/* Thread-local description of the last non-OK status ("" if none). */
const char *amg_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* AMG_B200_H */

/* walklap.h — C ABI of the B200 walk-based Laplacian library (libwalklap.so).
 *
 * Implements the data-parallel hot path of arXiv 2601.11338 (F. Arrigo, F. Durastante,
 * "Walk based Laplacians for Modeling Diffusion on Complex Networks"):
 *   * total communicability t = φ_θ(A,c) 1              ("a single evaluation")
 *   * Laplacian action 𝕃_θ(c) V = diag(t) V - φ_θ(A,c) V  (eq:weighted_laplacian)
 *   * matrix-function action φ_θ(A,c) V                  (Prop. pro:whe-we-converge)
 *   * diffusion exp(-τ 𝕃_θ) x0 for a sweep of τ
 * where φ_θ(A,c) = Σ_k c_k q_k(A), q_k the backtrack-downweighted walk counts of eq:qrec
 * with θ = 1 - μ: θ = 1 all walks, θ = 0 nonbacktracking (eq:Br).
 * Every action is evaluated by polynomial Krylov (Arnoldi) on the 2n x 2n companion
 * operator Z = [[O, I], [μ(μI - D), A]] (eq:Zdef) started from [q_1 v; q_2 v]; the small
 * projected function f_1(H_k) (eq:fs with s = 1) is evaluated on the device.
 *
 * Conventions (all entry points):
 *  - Return WL_OK (0) on success.  On failure a thread-local message is available from
 *    wl_last_error().  Argument errors are detected synchronously before anything is enqueued.
 *  - Pointers documented as "device" must be CUDA device (or managed) memory on the operator's
 *    device; "host" pointers are ordinary host memory.  The caller owns every buffer it passes.
 *  - Work is stream-ordered on `stream` (a cudaStream_t passed as void*; NULL = legacy default
 *    stream) and asynchronous unless stated: results are valid after the stream is synchronized.
 *  - Dense blocks are row-major: element (row r, column c) of a block with leading dimension ld
 *    lives at ptr[r * ld + c]; ld >= number of columns.
 *  - Multi-GPU: every rank calls the same functions collectively with its own contiguous row range
 *    (from wl_partition); inputs and outputs are row-distributed the same way.
 *  - Handles are opaque and owned by the library until the matching *_destroy.
 */
#ifndef WALKLAP_H
#define WALKLAP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  WL_OK = 0,
  WL_EINVAL = 1,      /* bad argument: θ ∉ [0,1], b < 1, ld < columns, null pointer, sizes */
  WL_EGRAPH = 2,      /* CSR not simple/symmetric-compatible: unsorted row_ptr, column out of range,
                         self loop or duplicate entry (simple graphs only) */
  WL_EDIVERGE = 3,    /* resolvent with α·ρ ≥ 1: the series of Prop. pro:whe-we-converge diverges
                         (Remark P:390-392); CG solver: 𝒜_θ(α) not positive definite */
  WL_ENOCONV = 4,     /* CG solver: a column did not reach cg_tol within cg_maxit; Krylov: the a-posteriori
                         estimate exceeded opts.tol (reported by wl_wait).  Best iterate written. */
  WL_ENOMEM = 5,      /* device allocation failed */
  WL_ECUDA = 6,       /* CUDA runtime error (message has the CUDA error string) */
  WL_ENCCL = 7,       /* NCCL error */
  WL_EUNSUPPORTED = 8 /* size/feature outside this build (e.g. local nnz >= 2^31) */
} wl_status;

typedef enum {
  WL_WALK = 0, /* all walks: θ = 1 (μ = 0), 𝕃(f) = diag(f(A)1) - f(A), eq:f-laplacian */
  WL_NBT = 1,  /* nonbacktracking: θ = 0 (μ = 1), p_k of eq:Br */
  WL_BTDW = 2  /* backtrack-downweighted: θ ∈ [0,1] given explicitly */
} wl_variant;

typedef enum {
  WL_F_EXP = 0,       /* c_k = β^k / k!  (f = exp(βx); inverse temperature β) */
  WL_F_RESOLVENT = 1, /* c_k = α^k       (f = (1 - αx)^{-1}) */
  WL_F_SERIES = 2     /* explicit c_0..c_{K}, zero beyond (Def. def:transformedlaplacian) */
} wl_fkind;

/* Walk weights {c_k} of Def. def:BDTW-Laplacian.  `coeffs` (host, ncoeffs entries) is read only
 * for WL_F_SERIES and copied by wl_operator_create. */
typedef struct {
  int32_t kind;         /* wl_fkind */
  double param;         /* β (WL_F_EXP) or α (WL_F_RESOLVENT) */
  const double* coeffs; /* host; WL_F_SERIES only */
  int32_t ncoeffs;      /* 1..64; WL_F_SERIES only */
  double scale;         /* multiplies 𝕃 (wl_apply, wl_diffuse); 0 means 1.  The paper's eq:katz-based-
                           walk-laplacian uses (1-α²); Fig. 4b was produced with (1-α), i.e. scale =
                           1/(1+α) (reading R5).  φ, t and the Markov chain are not scaled. */
} wl_walkfun;

/* Options; initialise with wl_opts_default(). */
typedef struct {
  int32_t krylov_dim;   /* Arnoldi steps k per action (default 30; 1..64) */
  int32_t reorth;       /* Arnoldi orthogonalisation of the 2n-long Krylov basis of Z:
                           2 = TOAR (default; two-level orthogonal Arnoldi): the basis is stored as [U g; U f]
                           over k+2 n-vectors U (the halves of all Krylov vectors of Z share one
                           n-dimensional space, eq:qrec), one dot pass + one update pass over U per
                           step, coefficient-space Gram-Schmidt twice;
                           1 = DCGS2 on the 2n-vectors (second pass delayed and fused with the next
                           step's projection);  0 = single classical Gram-Schmidt pass */
  int32_t max_cols;     /* columns per internal Krylov batch (default 32; 1..32) */
  double breakdown_tol; /* lucky breakdown when ||w_{j+1}|| <= tol * ||Z q_j|| (default 1e-12) */
  double rho_bound;     /* optional upper bound on ρ(Z_θ) (e.g. ρ(A), which bounds it since
                           0 <= q_k <= A^k): a resolvent with α * rho_bound >= 1 is rejected with
                           WL_EDIVERGE (Prop. pro:whe-we-converge).  0 = no check (default). */
  int32_t relabel;      /* 1 (default): relabel the local rows by decreasing degree internally
                           (gather locality); results are returned in the caller's row order */
  int32_t solver;       /* WL_SOLVER_KRYLOV (default): polynomial Krylov on Z for every f.
                           WL_SOLVER_CG (resolvent only, α > 0): φ_θ = (1-μ²α²) 𝒜_θ(α)^{-1} with the
                           deformed Laplacian 𝒜_θ(α) = (1-μ²α²)I - αA + μα²D (eq:deformed at μ = 1,
                           P:436-441), solved by Jacobi-preconditioned conjugate gradients (§4.2 P:545-551;
                           SPD when α ρ(Z_θ) < 1, Prop. prop:CGworks).  Actions then synchronize the
                           stream every cg_check iterations; a non-SPD system returns WL_EDIVERGE and
                           columns not converged after cg_maxit return WL_ENOCONV (best iterate written). */
  double cg_tol;        /* relative residual ||b - 𝒜x|| <= cg_tol ||b|| per column (default 1e-9) */
  int32_t cg_maxit;     /* iteration cap (default 1000) */
  int32_t cg_check;     /* convergence is read back every cg_check iterations (default 8) */
  double tol;           /* a-posteriori Krylov check (reading R11): when > 0, every action estimates
                           ||u|| h_{k+1,k} |e_k^T f_1(H_k) e_1| relative to ||u|| ||f_1(H_k) e_1|| per column;
                           an estimate above tol sets a sticky WL_ENOCONV that wl_wait reports (the
                           result is still written).  0 = no check (default). */
  int32_t halo_overlap; /* multi-rank only: 1 (default) splits the local CSR into A_loc (local columns)
                           and A_halo (halo columns) so A_loc's SpMM runs while the halo exchange is
                           in flight on a second stream; 0 exchanges first, then runs
                           one SpMM over the full local CSR */
  int32_t lanczos;      /* 1 (default, with reorth = 2): Krylov batches whose columns are all θ = 1 (μ = 0, the
                           all-walk operator, where q_k = A^k) run the symmetric three-term Lanczos
                           recurrence on A from A v ("Lanczos (for A = Aᵀ)") instead of TOAR on Z:
                           three n-block passes per step instead of two passes over the whole basis */
  int32_t krylov_adaptive; /* 1 (requires tol > 0; TOAR path): stop the Arnoldi process early, after the
                           first step k' >= 6 (checked every 2 steps) at which the a-posteriori estimate of
                           `tol` is below tol for every column of the batch (reading R11); krylov_dim is
                           then the cap.  Each check synchronizes the stream (not CUDA-graph capturable).
                           0 (default): always krylov_dim steps */
  int32_t fp32;         /* 1 (reorth = 2, Krylov solver): the fp32 mode of the north star (parity 1e-4): the
                           n-vectors of each TOAR batch — the basis U, the SpMM operand and output — are
                           stored in float, halving the bytes of the Gram passes and of the SpMM gathers;
                           every sum (SpMM rows, dot products, basis updates, combine) and all projected
                           work stay double, inputs and results are double, and t (create) is computed
                           in double.  θ = 1 batches run Lanczos on float vectors likewise.  0 (default): double */
} wl_opts;

typedef enum { WL_SOLVER_KRYLOV = 0, WL_SOLVER_CG = 1 } wl_solver;

typedef struct wl_comm wl_comm;
typedef struct wl_operator wl_operator;
typedef struct wl_workspace wl_workspace;
typedef void* wl_stream; /* cudaStream_t */

void wl_opts_default(wl_opts* opts);
const char* wl_last_error(void);
const char* wl_version(void);
/* Number of CUDA kernels this library has launched in the calling process (monotone counter). */
int64_t wl_launch_count(void);

/* ---- multi-GPU plumbing (NCCL over NVLink; one process per GPU) --------------------------- */
/* Rank 0 creates a 128-byte NCCL unique id (host buffer `out128`) and broadcasts it. */
wl_status wl_nccl_unique_id(void* out128);
/* Collective over `nranks` processes; binds `device`.  comm = NULL everywhere means 1 GPU. */
wl_status wl_comm_create(int32_t nranks, int32_t rank, const void* id128, int32_t device,
                         wl_comm** out);
void wl_comm_destroy(wl_comm* comm);

/* Loopback transport (testing the row-partitioned path on ONE device; SURVEY §4 "simulated
 * exchange"): a group of nranks ranks living in one process, each driven by its own host thread and
 * its own stream.  Every rank calls wl_comm_create_loopback(group, rank, device) and then uses the
 * comm exactly like an NCCL one; halo exchanges become device-to-device copies between the ranks'
 * buffers and allreduces a fixed-order device sum, both stream-ordered like NCCL.  Collective calls
 * block the calling host thread until every rank has joined (a rendezvous, up to the group timeout,
 * default 600 s, after which the group is broken and every collective returns WL_ENCCL).
 * The group must outlive its comms.  1 <= nranks <= 64. */
typedef struct wl_loopback wl_loopback;
wl_status wl_loopback_create(int32_t nranks, wl_loopback** out);
wl_status wl_loopback_set_timeout(wl_loopback* group, double seconds);
void wl_loopback_destroy(wl_loopback* group);
wl_status wl_comm_create_loopback(wl_loopback* group, int32_t rank, int32_t device, wl_comm** out);

/* nnz-balanced contiguous row partition (host, bit-exact integer arithmetic):
 * bounds[0] = 0, bounds[nranks] = n, bounds[p] = smallest r with row_ptr[r] >= ceil(p*nnz/nranks)
 * (clamped to be nondecreasing).  row_ptr: host, n+1 entries.  bounds_out: host, nranks+1. */
wl_status wl_partition(int64_t n, const int64_t* row_ptr, int32_t nranks, int64_t* bounds_out);

/* Host-only halo plan of rank `rank` under the row partition `bounds` (nranks+1 entries), the
 * plan wl_operator_create builds before its internal relabelling; needs no GPU.
 *   col_local_out  : nnz_local int32 — owned column g -> g - bounds[rank]; every other column ->
 *                    n_local + h, h its index in halo_ids_out
 *   halo_ids_out   : capacity nnz_local int64 — sorted distinct global ids of the non-owned
 *                    columns (grouped by owner, partitions being contiguous); *n_halo_out entries
 *   recv_count_out : nranks int64 (may be NULL) — halo rows owned by each rank
 * Validates the CSR like wl_operator_create (WL_EGRAPH). */
wl_status wl_halo_plan(int64_t n_global, int32_t nranks, const int64_t* bounds, int32_t rank,
                       const int64_t* row_ptr_local, const int32_t* col_idx_local, int32_t* col_local_out,
                       int64_t* halo_ids_out, int64_t* n_halo_out, int64_t* recv_count_out);

/* ---- operator --------------------------------------------------------------------------------
 * Builds the operator for rows [row_begin, row_end) of an n_global-node simple graph and
 * computes + caches t_θ = φ_θ(A,c) 1 for every requested θ (step a8; synchronous on return).
 *   row_ptr_local : host, (row_end-row_begin)+1 entries, global nnz offsets of the local rows
 *                   (row_ptr_local[0] need not be 0)
 *   col_idx_local : host, global column ids of those rows (sorted per row, no self loops/dups)
 *   variant       : WL_WALK / WL_NBT force θ = 1 / θ = 0 and require n_theta == 1;
 *                   WL_BTDW takes thetas[0..n_theta) ∈ [0,1] (host)
 *   n_theta       : 1..32 downweighting values evaluated together (a θ sweep); an action on a
 *                   b-column block V returns n_theta*b columns (see wl_apply)
 *   f, opts       : walk weights and options (copied)
 * The CSR is copied to device memory; host arrays may be freed on return.  WL_EGRAPH on
 * malformed CSR; WL_EDIVERGE for a resolvent with α * opts->rho_bound >= 1. */
wl_status wl_operator_create(wl_comm* comm, int64_t n_global, int64_t row_begin, int64_t row_end,
                             const int64_t* row_ptr_local, const int32_t* col_idx_local,
                             int32_t variant, int32_t n_theta, const double* thetas,
                             const wl_walkfun* f, const wl_opts* opts, wl_stream stream,
                             wl_operator** out);
void wl_operator_destroy(wl_operator* op);
/* Local sizes: n_local rows, nnz_local, halo rows, number of θ values. Any pointer may be NULL. */
wl_status wl_operator_info(const wl_operator* op, int64_t* n_local, int64_t* nnz_local,
                           int64_t* n_halo, int32_t* n_theta);
/* Rows of this rank's internal (relabelled) order that carry Krylov data: the rows after them are isolated (no
 * nonzeros, referenced by no row of any rank), and every Krylov vector built from A v vanishes there (q_k(A) v = 0
 * for k >= 1; P:76-88 simple graphs), so the Krylov batches store and stream only the first *n_active rows;
 * their outputs on the isolated rows are c_0 v (φ) and 0 (𝕃; t = c_0 there).  *n_active = n_local without
 * relabelling (opts.relabel = 0) or when an empty row is referenced (non-symmetric input).  WL_EINVAL on NULL. */
wl_status wl_operator_active_rows(const wl_operator* op, int64_t* n_active);
/* Copies t_θ = φ_θ 1 (device, n_local x n_theta, ld ldt >= n_theta) — the "diagonal shift". */
wl_status wl_operator_diag_shift(const wl_operator* op, double* t_dev, int64_t ldt,
                                 wl_stream stream);

/* Workspace for actions on up to max_b input columns (device memory is allocated here: the
 * Krylov basis takes (k+5) * n_local * min(32, n_theta*max_b) doubles with TOAR, (k+2) * 2 * n_local *
 * min(32, n_theta*max_b) with DCGS2). */
wl_status wl_workspace_create(const wl_operator* op, int32_t max_b, wl_workspace** out);
void wl_workspace_destroy(wl_workspace* ws);
/* Counters of a workspace (host): cg_iterations = CG iterations executed by actions on it so far
 * (per solve, the largest count over its columns; WL_SOLVER_CG only); krylov_steps / krylov_batches =
 * Arnoldi steps taken and Krylov batches run by the TOAR path (their ratio is the mean k' under
 * opts.krylov_adaptive).  Any pointer may be NULL. */
wl_status wl_workspace_stats(const wl_workspace* ws, int64_t* cg_iterations, int64_t* krylov_steps,
                             int64_t* krylov_batches);

/* ---- actions (step a3-a7) -------------------------------------------------------------------
 * V  : device, n_local x b, leading dimension ldv >= b
 * LV : device, n_local x (n_theta*b), ldlv >= n_theta*b;
 *      column i*b + c receives 𝕃_{θ_i} V[:, c]  (wl_apply) or φ_{θ_i} V[:, c] (wl_phi_apply).
 * V and LV must not overlap.  1 <= b <= max_b of the workspace.  Asynchronous on `stream`. */
wl_status wl_apply(const wl_operator* op, int32_t b, const double* V, int64_t ldv, double* LV,
                   int64_t ldlv, wl_workspace* ws, wl_stream stream);
wl_status wl_phi_apply(const wl_operator* op, int32_t b, const double* V, int64_t ldv,
                       double* LV, int64_t ldlv, wl_workspace* ws, wl_stream stream);
/* Same as wl_apply with HOST buffers (pinned or pageable): copies V to the device, applies, and
 * copies the result back inside the call; synchronous (returns after LV is written). */
wl_status wl_apply_host(const wl_operator* op, int32_t b, const double* V_host, int64_t ldv,
                        double* LV_host, int64_t ldlv, wl_workspace* ws, wl_stream stream);

/* ---- diffusion (step a9) --------------------------------------------------------------------
 * X[:, s] = exp(-tau[s] 𝕃_{θ_i}) x0 for s < nt, i = theta_index, by an outer Lanczos process of
 * dimension k_out on the symmetric 𝕃 (each step one wl_apply) with full reorthogonalisation,
 * then X = ||x0|| Q_out exp(-tau T) e_1 (dense exponential of the k_out x k_out tridiagonal T).
 *   tau : host, nt >= 1 values >= 0;   x0 : device, n_local;   X : device, n_local x nt (ldx).
 * 2 <= k_out <= 128.  Asynchronous on `stream`. */
wl_status wl_diffuse(const wl_operator* op, int32_t theta_index, int32_t nt, const double* tau,
                     const double* x0, double* X, int64_t ldx, int32_t k_out, wl_workspace* ws,
                     wl_stream stream);

/* ---- average return probability (Alg. 1 XNysTrace-exp) -----------
 * p_out[s] ≈ p̂_0(t_s) = (1/n) tr exp(-t_s 𝕃_{θ_i}) (eq:average_return_probabilities) and
 * e_out[s] its error estimate, for i = theta_index:
 *   1. V_1 R_0 = Ω (Cholesky QR, twice); block Arnoldi with every pole at ∞ (reading R16: the
 *      polynomial block Krylov space span{Ω, 𝕃Ω, …, 𝕃^{k-1}Ω}; each step one batched wl_apply on M
 *      columns and block classical Gram–Schmidt applied twice, with cuBLAS DGEMMs and an NCCL
 *      allreduce of the Gram blocks across ranks);
 *   2. H_k = V_kᵀ 𝕃 V_k (kM x kM) = Q Λ Qᵀ on the host;
 *   3. for every t: Y(t) = (1/n) V_k exp(-t H_k) V_kᵀ Ω and XNysTrace(Y(t), Ω) (reading R17), both in
 *      the kM-dimensional coordinates of V_k.
 * Omega: device, n_local x M (ld ldo >= M), user row order: the iid isotropic probes (e.g. Gaussian)
 *        ω_1..ω_M; rows of all ranks together form the global probe block.
 * times: host, nt >= 1 values >= 0.  p_out, e_out: host, nt values (identical on every rank).
 * 1 <= M <= the workspace's column batch (wl_workspace_create max_b and opts.max_cols);
 * 1 <= k and k*M <= min(1024, n_global).  Synchronous.  WL_ENOCONV if the block Krylov space is
 * exhausted (k*M above the dimension it can reach) or an eigen/Cholesky step fails. */
wl_status wl_xnystrace_exp(const wl_operator* op, int32_t theta_index, int32_t M, const double* Omega,
                           int64_t ldo, int32_t k, int32_t nt, const double* times, double* p_out,
                           double* e_out, wl_workspace* ws, wl_stream stream);

/* ---- the RATIONAL block Krylov variant of Alg. 1 ------------------
 * Same estimate as wl_xnystrace_exp, on the block rational Krylov space of eq:block-rational-Krylov with
 * the given poles and the reduced pencil (𝓗_k, 𝒦_k) of the block rational Arnoldi
 * decomposition 𝔏 V_{k+1} 𝒦_k = V_{k+1} 𝓗_k, Y(t) = (1/n) V_k exp(−t Ĥ_k K̂_k⁻¹) V_kᵀ Ω:
 *   poles_re/poles_im (host, npoles >= 0): ξ_j = +inf (pole at ∞), a real number (poles_im = 0), or
 *     a + ib with b > 0 standing for the conjugate pair {ξ, ξ̄} (the basis is kept real: the pair adds
 *     the real and imaginary parts of (𝔏 − ξI)⁻¹u, 2M columns).  A final pole at ∞ is appended (reading
 *     R18), which makes Ĥ_k K̂_k⁻¹ = V_kᵀ 𝔏 V_k.  Each finite pole costs one shifted solve
 *     (𝔏 − ξI)X = u by MINRES to relative residual inner_tol (at most inner_maxit iterations; the paper
 *     used GMRES at 1e-6), one batched Laplacian action per iteration (two for a pair).
 *   The basis dimension M(1 + Σ_j m_j) − M (m_j = 2 for a pair, else 1, plus the final ∞) must be
 *     <= min(1024, n_global).  inner_iters (host, may be NULL) receives Σ over poles of the largest
 *     MINRES iteration count over the M columns.
 * WL_ENOCONV when a shifted solve misses inner_tol, the basis becomes rank deficient, or a small
 * eigen/Cholesky step fails.  Synchronous. */
wl_status wl_xnystrace_exp_rational(const wl_operator* op, int32_t theta_index, int32_t M, const double* Omega,
                                    int64_t ldo, int32_t npoles, const double* poles_re, const double* poles_im,
                                    double inner_tol, int32_t inner_maxit, int32_t nt, const double* times,
                                    double* p_out, double* e_out, int64_t* inner_iters, wl_workspace* ws,
                                    wl_stream stream);
/* Poles of the AAA rational approximation of exp(−x) on [0, xmax] (Alg. 1 line 3, P:595, P:623-625;
 * AAA = Nakatsukasa–Sète–Trefethen, the paper's [MR3805855]): samples {0} ∪ xmax·10^linspace(−10, 0, 2000),
 * relative tolerance tol, at most 30 support points; Froissart doublets (|residue| < 1e-13) and poles on
 * [0, xmax] are dropped; one representative (Im > 0) per conjugate pair; sorted by (|Im|, Re) (reading
 * R18).  re/im: host arrays of capacity cap; *npoles receives the count (WL_EINVAL if above cap). */
wl_status wl_aaa_exp_poles(double xmax, double tol, int32_t cap, double* re, double* im, int32_t* npoles);
/* Gershgorin bound 2·scale·max_i t'_i >= ρ(𝕃_θ) (Prop. pro:still-again-an-mmatrix), the ρ(𝔏) estimate of
 * Alg. 1 line 3 (host output; collective over the ranks). */
wl_status wl_laplacian_bound(const wl_operator* op, int32_t theta_index, double* bound);

/* The host steps behind it, exported for testing (host buffers, synchronous):
 * wl_symmetric_eig: A (n x n row-major symmetric) is overwritten by its eigenvectors (column i of A =
 *   eigenvector i), lam (n) receives the eigenvalues; method 0 = Householder tridiagonalisation +
 *   implicit QL (the one wl_xnystrace_exp uses), 1 = cyclic Jacobi.
 * wl_xnystrace_curve: XNysTrace (reading R17) of Y(t) = (1/n) Q diag(e^{-t lam}) W for every t, in
 *   the coordinates of an orthonormal basis: lam (d) the eigenvalues of the projected 𝕃, W (d x M
 *   row-major) the probes in its eigen-coordinates, n the global dimension (for 1/n and the shift). */
wl_status wl_symmetric_eig(int32_t n, double* A, double* lam, int32_t method);
wl_status wl_xnystrace_curve(int32_t d, int32_t M, double n, const double* lam, const double* W, int32_t nt,
                             const double* times, double* p_out, double* e_out);

/* ---- discrete-time diffusion: Markov chain (eq:let_there_be_markov P:506-533)
 * P = I - D^{-1} 𝕃_θ with D = diag(t_θ), t_θ = φ_θ 1 (reading R6: "a single evaluation of
 * the underlying matrix function"; Fig. 1's stationary bars are t/Σt), i.e. P = diag(t)^{-1} φ_θ,
 * row-stochastic with stationary distribution π = t/Σt (see wl_operator_diag_shift).  Evolves
 * p_{k+1} = p_k P (row vectors) from p0 for θ value theta_index: each step is one φ_θ action on
 * p_k / t (φ symmetric).  p0 : device, n_local (user row order, p0 1 = 1 over all ranks);
 * P : device, n_local x nsteps (ldp >= nsteps), column k receives p_{k+1}.  Requires t > 0
 * (true for exp and resolvent weights, c_0 = 1).  Asynchronous on `stream`. */
wl_status wl_markov(const wl_operator* op, int32_t theta_index, int32_t nsteps, const double* p0, double* P,
                    int64_t ldp, wl_workspace* ws, wl_stream stream);

/* ---- spectral radius (helper for β = 1/ρ(A); convergence checks, Prop. pro:whe-we-converge)
 * ρ(A) of the operator's graph by k steps of Lanczos on A (full reorthogonalisation) started from
 * the all-ones vector (positive overlap with the Perron vector of the nonnegative symmetric A);
 * returns the largest eigenvalue of the k x k tridiagonal (a lower bound converging to ρ(A)).
 * Synchronous.  2 <= k <= 128. */
wl_status wl_spectral_radius(const wl_operator* op, int32_t k, double* rho_out, wl_stream stream);

/* ---- ρ(Z_θ) (Prop. pro:whe-we-converge P:317-322, §5.3 α scaling P:1490)
 * Spectral radius of the companion operator Z_θ = [[O, I], [μ(μI - D), A]] (eq:Zdef) of θ value
 * theta_index: k steps of Arnoldi (CGS2) on Z from a positive pseudo-random vector (hash of the
 * row index; [1; 1] itself is an eigenvector of Z_1), then the largest
 * modulus among the eigenvalues of the k_eff x k_eff Hessenberg matrix (Francis double-shift QR on
 * the host).  Ritz values converge to the extremal eigenvalues; for θ = 0 Z is the Ihara-Bass
 * linearisation of the nonbacktracking matrix, whose spectral radius is a real eigenvalue.
 * Synchronous.  2 <= k <= 128.  WL_ENOCONV if the small QR iteration fails. */
wl_status wl_spectral_radius_z(const wl_operator* op, int32_t theta_index, int32_t k, double* rho_out,
                               wl_stream stream);
/* The host eigenvalue routine behind it, exported for testing: H (host) n x n row-major upper
 * Hessenberg (entries below the subdiagonal ignored); wr/wi (host, n) receive real/imaginary parts. */
wl_status wl_hessenberg_eigvals(int32_t n, const double* H, double* wr, double* wi);

/* ---- live per-kernel timing (benchmarking) ----------------------------------------------------
 * When enabled, every kernel launch scope is bracketed by CUDA events on its stream (small
 * overhead).  wl_profile_collect() synchronizes on the recorded events, aggregates elapsed time
 * per kernel name and clears the session; wl_profile_get(i) reads entry i < wl_profile_count().
 * `name` points to library-owned storage valid until the next collect. */
void wl_profile_enable(int32_t on);
wl_status wl_profile_collect(void);
int32_t wl_profile_count(void);
wl_status wl_profile_get(int32_t i, const char** name, double* total_ms, int64_t* launches);

/* Synchronizes `stream` and returns the first asynchronous error recorded on `op` (or WL_OK): CUDA
 * errors, and WL_ENOCONV when an action's a-posteriori Krylov estimate exceeded opts.tol (the flag is
 * cleared by the call). */
wl_status wl_wait(const wl_operator* op, wl_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* WALKLAP_H */

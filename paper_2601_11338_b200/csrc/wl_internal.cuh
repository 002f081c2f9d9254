// wl_internal.cuh — shared declarations of the walklap CUDA library (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include "walklap.h"
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace wl {

// ---------------------------------------------------------------- errors / launch accounting
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
void cuda_check(cudaError_t e, const char* what, const char* file, int line);
#define WL_CUDA(x) ::wl::cuda_check((x), #x, __FILE__, __LINE__)
void note_launch(const char* name);  // increments the process-wide launch counter
// Scoped launch accounting: counts the launch and, when profiling is enabled (wl_profile_enable),
// brackets the launch(es) in this scope with CUDA events on stream `s`, accumulated per name.
struct LaunchScope {
  int slot = -1;
  cudaStream_t s;
  LaunchScope(const char* name, cudaStream_t st);
  ~LaunchScope();
};
#define WL_LAUNCH(name) ::wl::LaunchScope wl_launch_scope_(name, s)

// NVTX range over a host scope (Krylov phases: seeds, Arnoldi step, f(H) + combine, shifted solve, ...);
// header-only NVTX3, a no-op unless a profiler is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name);
  ~NvtxRange();
};
#define WL_NVTX_CAT2(a, b) a##b
#define WL_NVTX_CAT(a, b) WL_NVTX_CAT2(a, b)
#define WL_NVTX(name) ::wl::NvtxRange WL_NVTX_CAT(wl_nvtx_, __LINE__)(name)

// ---------------------------------------------------------------- C ABI error plumbing
// Every extern "C" entry point runs its body through guarded(): a thrown Error becomes its
// wl_status and the thread-local message returned by wl_last_error().
wl_status set_last_error(int code, const std::string& m);
template <class F>
wl_status guarded(F&& f) {
  try {
    f();
    return WL_OK;
  } catch (const Error& e) {
    return set_last_error(e.code, e.what());
  } catch (const std::bad_alloc&) {
    return set_last_error(WL_ENOMEM, "host allocation failed");
  } catch (const std::exception& e) {
    return set_last_error(WL_EINVAL, e.what());
  }
}

int num_sms();  // SMs of the current device (cached per device)
// Gathered blocks of B > 1 columns (spmv.cu 256-bit lanes): a lane loads 32 bytes, so the loaded part of a row is
// pad_vec(B) = 4⌈B/4⌉ doubles; the row STRIDE pad_cols(B) is the next power of two (4, 8, 16, 32 doubles), so no
// row straddles a 128-byte line (B = 11: 3 sectors at a 128-byte stride — one L1 wavefront per gathered row
// instead of 1.5 at a 96-byte stride).  Columns in [B, pad_vec(B)) are zero; beyond are never read.
__host__ __device__ inline int pad_vec(int B) { return B <= 1 ? B : (B + 3) / 4 * 4; }
__host__ __device__ inline int pad_cols(int B) {
  if (B <= 1) return B;
  int p = 4;
  while (p < B) p *= 2;
  return p;
}
// the same for a storage type T (opts.fp32: a 32-byte lane is 8 floats, rows padded to 8 ⌈B/8⌉ loaded floats at
// a power-of-two stride >= 8; B = 11: 2 sectors at a 64-byte stride)
template <class T>
__host__ __device__ inline int pad_vec_t(int B) {
  constexpr int L = 32 / (int)sizeof(T);
  return B <= 1 ? B : (B + L - 1) / L * L;
}
template <class T>
__host__ __device__ inline int pad_cols_t(int B) {
  if (B <= 1) return B;
  int p = 32 / (int)sizeof(T);
  while (p < B) p *= 2;
  return p;
}

constexpr int kMaxCols = 32;    // columns per Krylov batch (B)
constexpr int kMaxKrylov = 64;  // Arnoldi steps per action
constexpr int kMaxSmallN = 130; // largest dense matrix of the projected-function kernels

// ---------------------------------------------------------------- degree-binned Z-SpMV
// out[r][c] = scale[c] * ( Σ_{z in row r} y[col[z]][c] + (g0[c] + g1[c] * deg(r)) * x[r][c] )
// Gathers y rows (ld ldy) for local columns < n_loc, halo rows (ld ldh) for columns >= n_loc.
#ifndef WL_SMALL_MAX
#define WL_SMALL_MAX 32
#endif
#ifndef WL_HUB_CHUNK
#define WL_HUB_CHUNK 4096
#endif
#ifndef WL_MEDIUM_MAX
#define WL_MEDIUM_MAX WL_HUB_CHUNK
#endif
constexpr int kSmallMax = WL_SMALL_MAX;    // rows with deg <= 32: lane group per row (batched, 32 rows a warp)
constexpr int kMediumMax = WL_MEDIUM_MAX;  // rows with deg <= kMediumMax: one warp per row
constexpr int kHubChunk = WL_HUB_CHUNK;    // longer rows: split into chunks of kHubChunk nonzeros
struct SpmvArgs {
  const int32_t* rowptr;  // n_loc + 1, local offsets
  const int32_t* col;     // nnz, local ids (halo ids >= n_loc)
  int32_t n_loc;
  const int32_t* small_rows; int n_small;
  int small_first;                   // small rows are ids [small_first, small_first + n_small), or -1
  int n_iso;                         // the last n_iso of them have no nonzeros (out = scale (g0 + g1 d) x)
  const int32_t* medium_rows; int n_medium;
  int medium_first;                  // medium rows are ids [medium_first, medium_first + n_medium), or -1
  const int4* chunks; int n_chunks;  // (row, z0, z1, first chunk index of that row)
  double* chunk_part;                // n_chunks * B partial sums (scratch)
  unsigned int* row_ticket;          // n_chunks, zero between launches
  int nblk_small, nblk_medium;       // filled by spmv()
  const double* y; int64_t ldy;
  const double* yh; int64_t ldh;   // halo rows (multi-rank), n_halo of them
  int64_t n_halo;
  const double* x; int64_t ldx;   // may be null (no diagonal term)
  double* out; int64_t ldo;
  const double* g0; const double* g1; const double* scale;  // device, B entries (null = 0,0,1)
  const int32_t* degptr;             // row pointer giving d_i for the γ term (null: this CSR's rowptr)
  const int32_t* out_row;            // output row of CSR row i (null: i); not with the batched small rows
  int accumulate;                    // out += scale * Σ (no diagonal term): the A_halo part
  int hot_rows;                      // > 0: L2 evict_last hints for gathered rows < hot_rows (degree-sorted)
  int med_sub;                       // filled by spmv(): lanes per medium row when a row is one lane wide (0: a warp)
  int med_rpw;                       // filled by spmv(): medium rows per warp when a row is several lanes wide
  int B;
  const int* active;                 // optional (CG): the launch does nothing when *active == 0
  int f32;                           // 1: y, yh, x and out hold float (opts.fp32 TOAR batches)
  int64_t row_limit;                 // > 0: rows >= row_limit (isolated, the tail of the contiguous small range) are
                                     // not written
};
void spmv(const SpmvArgs& a, cudaStream_t s);

// ---------------------------------------------------------------- Gram-Schmidt passes
int gram_grid(int64_t elems, int B);  // upper bound on the CTAs of a dot pass (partial buffer sizing)

// DCGS2: delayed classical Gram-Schmidt (one reduction per Arnoldi step).  Step j holds the
// finalised orthonormal q_0..q_{j-1} (Q) and p_j (P): once orthogonalised, unnormalised.
//   pass A (dcgs2_dots):   a_i = q_i.p_j, b_i = q_i.w (i < j), α = p_j.p_j, β = p_j.w, γ = w.w,
//                          w = Z p_j; sums layout [a_0 b_0 a_1 b_1 ... α β γ] x B (w null: b=β=γ=0)
//   pass B (dcgs2_update): q_j = cq_p p_j + Σ cq_i q_i  (into Qout, which must not alias P),
//                          p_{j+1} = cp_w w + cp_p p_j + Σ cp_i q_i  (into Pnext)
// Basis vectors are addressed through a pointer table (slot i -> vector), passed by value.
constexpr int kMaxVecSlots = 130;  // basis slots a pass can address: k+2 <= 66 inner, k_out+1 <= 129 outer
struct VecPtrs {
  const double* p[kMaxVecSlots];
};
struct Dcgs2Args {
  VecPtrs Q; int nq;                  // q_0 .. q_{nq-1}
  int64_t len; int B;
  const double* P;                    // p_j
  const double* wa; int64_t split; const double* wb;   // w two-source (wa null: no w)
  double* Qout;                       // pass B: q_j
  double* Pnext;                      // pass B: p_{j+1}
  const double* coef_v;               // pass B: [cq_i, cp_i] interleaved per vector, x B
  const double* coef_s;               // pass B: [cq_p, cp_p, cp_w] x B
  int accumulate;                     // pass B vector tiles after the first: add to Qout / Pnext
  double* partials; double* sums_out;
  int grid;
  int f32;                            // 1: P, w and Q hold float (opts.fp32; pass A only), sums in double
};
void reduce_partials(const double* partials, int nout, int G, double* sums_out, cudaStream_t s);

// TOAR basis update (dcgs2.cu): out_o = coef_y[o] y + Σ_i coef_u[o][i] U_i, o < nout <= 3.
// coef_u layout [(o * coef_ld + i) * B + c].  Outputs must not alias y or U.
struct ToarArgs {
  VecPtrs U; int m;
  int64_t len; int B;
  const double* y;
  double* out[3]; int nout;
  int64_t out_ld[3];                  // row stride of output o (0 = B); > B only without tiling (m <= 32)
  const double* coef_y;
  const double* coef_u; int coef_ld;
  int accumulate;
  int f32;                            // 1: y, U and the outputs hold float (opts.fp32), combinations in double
};
void toar_update(ToarArgs a, cudaStream_t s);
// TOAR coefficient bookkeeping (toar.cu), one thread per Krylov column
size_t toar_state_doubles(int K);
// sums: reduced dot-pass outputs ([k*B + c]); or, with partials != null, the unreduced per-CTA partials
// ([(k*B + c)*G + cta]) that the kernel reduces itself (single GPU: one launch fewer per step)
void toar_coeffs(const double* sums, const double* partials, int G, int j, int final_pass, int B, int K, double btol,
                 double* H, double* n0, int* keff, double* state, size_t stride, double* coef_y, double* coef_u,
                 int coef_ld, cudaStream_t s);
void toar_combine_coef(const double* comb, int B, int K, const int* keff, const double* state, size_t stride,
                       double* combU, cudaStream_t s);
// returns the grid of the (single) launch: with sums_out == null the partials ([output][CTA]) are left
// for the consumer to reduce (single launch, nq <= 32)
int dcgs2_dots(Dcgs2Args a, cudaStream_t s);
void dcgs2_update(Dcgs2Args a, cudaStream_t s);
void dcgs2_coeffs(const double* sums, int j, int B, int K, double btol, int final_pass, int reorth, double* H,
                  double* ref, double* n0, int* keff, double* coef_v, double* coef_s, cudaStream_t s);

// ---------------------------------------------------------------- resolvent by PCG (cg.cu)
struct CgArgs {
  int64_t n; int B;
  const int32_t* rowptr;       // degrees for the Jacobi preconditioner
  const double* cs;            // per column constants (cg_setup)
  const double* b;             // right-hand sides, n x B
  double *x, *r, *p, *q;       // n x B each
  double* partials; double* sums;
  double* sc;                  // per column scalars: rz, alpha, beta, active
  double* bb;                  // per column ||b||^2
  int* iters;                  // per column iteration counts
  int* flags;                  // [0] bit 0: not positive definite; [1] active columns
};
void cg_setup(const double* mu, double alpha, double tol, int gstart, int b, int B, double* cs, double* g0,
              double* g1, double* scale, int* vcol, int* tcol, cudaStream_t s);
void cg_init(CgArgs a, cudaStream_t s);
void cg_dot(CgArgs a, cudaStream_t s);
void cg_update(CgArgs a, cudaStream_t s);
void cg_direction(CgArgs a, cudaStream_t s);
void cg_scalar(int which, const CgArgs& a, cudaStream_t s);         // after reduce (+ allreduce)
void cg_reduce(int which, const CgArgs& a, cudaStream_t s);         // partials -> sums
void cg_reduce_scalar(int which, const CgArgs& a, cudaStream_t s);  // single GPU: both in one CTA
void cg_combine(int mode, double lscale, const double* x, int64_t n, int B, const double* cs, const double* V, int64_t ldv,
                const int* vcol, double c0, const double* tprime, int64_t ldt, const int* tcol, double* out,
                int64_t ldo, const int32_t* perm, cudaStream_t s,
                int64_t nx = -1);  // rows >= nx (>= 0): not solved (isolated rows), φ v = v there

// ---------------------------------------------------------------- shifted solves by MINRES (minres.cu)
// (𝔏 − ξI) X = U for the n × B block U, ξ = shift_re + i shift_im; complex shifts solve the real
// symmetric 2n form, vectors then hold [real n × B | imaginary n × B] (offset n * B).
struct MinresArgs {
  int64_t n; int B;
  int cplx;                       // shift_im != 0
  double shift_re, shift_im, tol;
  const double* u;                // right-hand side (n x B, real)
  double *v, *vp, *w1, *w2, *x;   // Lanczos vectors, MINRES directions, solution
  double* p;                      // in: 𝔏 v (both halves); out: S v
  double* partials; double* sums; double* sc;
  int* nactive;                   // device: columns not yet converged
  int presummed;                  // scalar phase: a.sums already reduced (multi-rank allreduce)
};
size_t minres_scalar_doubles(int B);
int minres_grid(int64_t n, int B);
// phases: 0 ‖u‖² partials, 1 init vectors, 2 S v + α partials, 3 v̂ + ‖v̂‖² partials, 4 w, x, v update
void minres_vec(int phase, const MinresArgs& a, cudaStream_t s);
// which: 0 after phase 0, 1 after phase 2, 2 after phase 3
void minres_scalar(int which, const MinresArgs& a, cudaStream_t s);

// ---------------------------------------------------------------- μ = 0 Lanczos (lanczos.cu)
int lanczos_grid(int64_t n, int B);
// phase 0: partials of Σ x²; 1: Σ x·y; 2: x = x − α y − β qm with partials of ‖x‖²; 3: x *= scale (and, with
// xp, its row-padded copy xp with ld ldp for the SpMM's 32-byte lane gathers)
void lanczos_vec(int phase, double* x, const double* y, const double* qm, int64_t n, int B, const double* sc,
                 double* partials, cudaStream_t s, double* xp = nullptr, int64_t ldp = 0,
                 bool f32 = false);  // f32: x, y, qm, xp hold float (opts.fp32), sums double
// which 0: β_0 = ‖u‖ (n0, scale); 1: α_j; 2: β_{j+1} (H, scale, breakdown -> keff)
void lanczos_scalar(int which, int j, int64_t n, int presummed, const double* partials, double* sums, int B, int K,
                    double btol, double* sc, double* H, double* n0, int* keff, cudaStream_t s);

// ---------------------------------------------------------------- small dense functions
// Per column c (problem), m = keff[c]: y_c = f_1(H_m) e_1 for the Arnoldi matrix H.
// kind 3 (outer diffusion): problem p uses column 0's H and computes exp(-tau[p] H_m) e_1;
// output comb[p*(K+1) + i] = n0 * y_i * s_i.
struct SmallFArgs {
  const double* H; int ldh_col;   // H of column c at H + c*(K+1)*K, entry (i,j) at [j*(K+1)+i]
  int K;
  const int* keff;
  int kind; double param; const double* coeffs; int ncoeffs;
  const double* n0;  // ||u|| per column
  const double* s;   // basis scales s[i*B + c]
  double* comb;      // out: comb[i*B + c] = n0 * y_i * s_i
  double* scratch;   // per problem 9 * kMaxSmallN^2 doubles
  int B;             // columns of H/s/n0 (problems for kinds 0-2)
  const double* tau; // kind 3 only: nprob values
  int nprob;         // kind 3 only
  double* err;       // optional (kinds 0-2): relative a-posteriori error estimate per column
};
void small_f(const SmallFArgs& a, cudaStream_t s);

// ---------------------------------------------------------------- elementwise / misc kernels
// Vb[r*B + j] = V[r*ldv + vcol[j]]   (j < B); V null => ones
void batch_inputs(const double* V, int64_t ldv, int B, int64_t n, double* Vb, const int* vcol,
                  const int32_t* perm, cudaStream_t s);
void seed_expand(const double* s1, const double* s2, const double* v, int b, const int32_t* rowptr, const double* g1s,
                 const int* vcol, int B, int64_t n, double* t0, double* b0, cudaStream_t s, bool f32 = false);
void setup_chunk(const double* mu, int gstart, int b, int B, double* g0z, double* g1z, double* g0s,
                 double* g1s, int* vcol, int* tcol, cudaStream_t s);
// combine: mode 0 = φV (c0 V + Σ comb_i Q_i,top), 1 = 𝕃V (lscale (t'⊙V - Σ comb_i Q_i,top)),
//          2 = t' (Σ comb_i Q_i,top) for V = 1
// V column of batch column c is vcol[c]; t' column is tcol[c]; internal row r is user row
// perm[r] (modes 0/1 read V and write out in user order; mode 2 writes t' in internal order).
void combine(int mode, double lscale, const VecPtrs& Q, int nvec, int64_t n, int B,
             const double* comb, const double* V, int64_t ldv, const int* vcol, double c0,
             const double* tprime, int64_t ldt, const int* tcol, double* out, int64_t ldo,
             const int32_t* perm, cudaStream_t s, bool f32 = false,  // f32: Q holds float
             int64_t nq = -1);  // rows >= nq (>= 0) have no basis entries (isolated rows): the sum is 0 there
void pack_rows(const double* src, int64_t lds, const int32_t* idx, int64_t cnt, int B, double* dst,
               cudaStream_t s);
// dst[r * ldd + c] = src[r * lds + c] for c < B (other columns of dst untouched), r < n
void repack_rows(const double* src, int64_t lds, int64_t n, int B, double* dst, int64_t ldd, cudaStream_t s);
// the same between storage types (double -> float, float -> float); columns [B, zpad) of dst rows are zeroed
void repack_rows_t(const void* src, bool src_f32, int64_t lds, int64_t n, int B, void* dst, bool dst_f32, int64_t ldd,
                   int zpad, cudaStream_t s);
void pack_rows_f32(const float* src, int64_t lds, const int32_t* idx, int64_t cnt, int B, float* dst, cudaStream_t s);
void fill(double* p, int64_t n, double v, cudaStream_t s);
// sticky convergence flag: flag[0] |= 1 and flag[1] = max estimate (as bits) when err[c] > tol
void krylov_check(const double* err, int B, double tol, int* flag, cudaStream_t s);
// out[c] = min(keff[c], m) (c < B) and flag[0] = 0: the probe of the adaptive Krylov stop
void clamp_keff(const int* keff, int m, int B, int* out, int* flag, cudaStream_t s);
void fill_hash(double* p, int64_t n, uint64_t seed, int64_t i0, cudaStream_t s);  // 0.5 + U[0,1)
void gather_col(const double* src, int64_t lds, const int32_t* perm, int64_t n, double* dst, cudaStream_t s);
void scatter_col(const double* src, const int32_t* perm, int64_t n, double* dst, int64_t ldd, cudaStream_t s);
void markov_scale(const double* p, const double* tprime, int64_t ldt, int tcol, double c0, int64_t n, double* v,
                  cudaStream_t s);

// eigenvalues of a small real upper Hessenberg matrix (host; eig.cu). H row-major n x n, overwritten.
bool hessenberg_eigvals(std::vector<double>& H, int n, std::vector<double>& wr, std::vector<double>& wi);

// XNysTrace-exp host side (trace.cu)
bool sym_eig_jacobi(std::vector<double>& A, int d, std::vector<double>& lam, std::vector<double>& Q);
bool sym_eig_tridiag_ql(std::vector<double>& A, int d, std::vector<double>& lam);
bool xnystrace_curve(const std::vector<double>& lam, const std::vector<double>& W, int d, int M, double n,
                     const double* times, int nt, double* p_out, double* e_out);

// outer Lanczos helpers (diffusion)
void lanczos_combine(const double* Q, int64_t stride, int m, int64_t n, const double* Y, int nt,
                     double scale, double* X, int64_t ldx, const int32_t* perm, cudaStream_t s);

// ---------------------------------------------------------------- block products (block.cu)
// C (p x q col-major, ld p) = X[:, :p]ᵀ Y[:, :q] over n rows (row-major X ld ldx, Y ld ldy), q <= 64;
// partials: block_gram_partials(n, p) doubles of scratch.  Deterministic (fixed row split, CTA order).
size_t block_gram_partials(int64_t n, int p);
void block_gram(int p, int q, int64_t n, const double* X, int64_t ldx, const double* Y, int64_t ldy, double* C,
                double* partials, cudaStream_t s);
// Y[:, :q] = beta Y + alpha X[:, :p] C  (C p x q col-major, ld p; Y not read when beta == 0), q <= 64
void block_axpy(int p, int q, int64_t n, double alpha, const double* X, int64_t ldx, const double* C, double beta,
                double* Y, int64_t ldy, cudaStream_t s);

// ---------------------------------------------------------------- collectives (comm.cu)
constexpr int kMaxRanks = 64;
struct SumSrc {
  const double* p[kMaxRanks];
};
// dst[i] = Σ_{r < P} src.p[r][i], summed in rank order (the loopback allreduce)
void sum_ranks(const SumSrc& src, int P, int64_t count, double* dst, cudaStream_t s);
struct Xfer {
  void* ptr;     // device
  size_t bytes;
  int peer;
};
void comm_allreduce(wl_comm* c, double* buf, size_t count, cudaStream_t s);
void comm_sendrecv(wl_comm* c, const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs, cudaStream_t s);
void comm_alltoallv_host(wl_comm* c, const std::vector<std::vector<int64_t>>& send,
                         std::vector<std::vector<int64_t>>& recv, cudaStream_t s);
void comm_allgather_host(wl_comm* c, const std::vector<int64_t>& mine, std::vector<std::vector<int64_t>>& all,
                         cudaStream_t s);
void comm_barrier_host(wl_comm* c);

}  // namespace wl

// Communicator: NCCL (one process per GPU) or a loopback group (P ranks in one process on one device).
struct wl_loopback;
struct wl_comm {
  void* nccl = nullptr;        // ncclComm_t
  wl_loopback* lb = nullptr;   // loopback transport when set
  int nranks = 1, rank = 0, device = 0;
  cudaEvent_t ev_ready = nullptr, ev_done = nullptr;  // loopback rendezvous events
  double* scratch = nullptr;                           // loopback allreduce sums
  size_t scratch_n = 0;
};

// engine.cu — host orchestration of the walk-Laplacian Krylov path and the C ABI (walklap.h).
//
// One "action" on a chunk of B <= 32 columns (column c = (θ index, input column)) is
// (SURVEY §8(a) a3-a7):
//   a3  u = [A v ; A(Av) - μ d⊙v]                          two SpMM launches (θ-independent: over b columns)
//   a4  for j < k: w = Z q_j  (bottom half only)           spmv (degree-binned, fused recurrence)
//   a5            orthogonalise against the basis           TOAR (default): dcgs2_dots + toar_coeffs +
//                                                           toar_update; DCGS2: dcgs2_dots/coeffs/update
//   a6  y = f_1(H_k) e_1 on the device                     small_f
//   a7  φv = c_0 v + ||u|| [I O] Q_k y ;  𝕃v = t'⊙v - (φv - c_0 v)    combine
// with t' = φ1 - c_0 1 cached at operator creation (a8).  Multi-GPU: the SpMM input rows owned
// by other ranks are exchanged (grouped ncclSend/ncclRecv) before each SpMM and every Gram
// reduction is summed with ncclAllReduce, so H is bit-identical on every rank.
#include "walklap.h"
#include "wl_internal.cuh"

#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

namespace wl {

static std::atomic<int64_t> g_launches{0};
void note_launch(const char*) { g_launches.fetch_add(1, std::memory_order_relaxed); }

// ---- live per-kernel timing (bench.py): CUDA events around every launch scope ----------------
struct ProfRec {
  std::string name;
  cudaEvent_t a, b;
};
static std::mutex g_prof_mtx;
static bool g_prof_on = false;
static std::vector<ProfRec> g_prof;          // events of the current session
static std::vector<cudaEvent_t> g_prof_pool;  // recycled events
static std::vector<std::pair<std::string, std::pair<double, int64_t>>> g_prof_result;

static cudaEvent_t prof_event() {
  if (!g_prof_pool.empty()) {
    cudaEvent_t e = g_prof_pool.back();
    g_prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  WL_CUDA(cudaEventCreate(&e));
  return e;
}

LaunchScope::LaunchScope(const char* name, cudaStream_t st) : s(st) {
  if (!name) return;  // disabled scope
  note_launch(name);
  if (!g_prof_on) return;
  std::lock_guard<std::mutex> lk(g_prof_mtx);
  ProfRec r{name, prof_event(), prof_event()};
  WL_CUDA(cudaEventRecord(r.a, s));
  slot = (int)g_prof.size();
  g_prof.push_back(r);
}

LaunchScope::~LaunchScope() {
  if (slot < 0) return;
  std::lock_guard<std::mutex> lk(g_prof_mtx);
  cudaEventRecord(g_prof[slot].b, s);
}

thread_local std::string g_last_error;

wl_status set_last_error(int code, const std::string& m) {
  g_last_error = m;
  return (wl_status)code;
}

int num_sms() {
  static std::mutex mtx;
  static std::map<int, int> cache;
  int dev = 0;
  WL_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mtx);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int sms = 0;
  WL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  cache[dev] = sms;
  return sms;
}

NvtxRange::NvtxRange(const char* name) { nvtxRangePushA(name); }
NvtxRange::~NvtxRange() { nvtxRangePop(); }

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e == cudaSuccess) return;
  const std::string msg = std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                          std::to_string(line) + ")";
  if (e == cudaErrorMemoryAllocation) throw Error(WL_ENOMEM, msg);
  throw Error(WL_ECUDA, msg);
}

template <class T>
struct DArr {
  T* p = nullptr;
  size_t n = 0;
  DArr() = default;
  DArr(const DArr&) = delete;
  DArr& operator=(const DArr&) = delete;
  ~DArr() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    if (count <= n && p) return;
    release();
    if (count == 0) return;
    WL_CUDA(cudaMalloc(&p, sizeof(T) * count));
    n = count;
  }
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) WL_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// One CSR operand of the SpMM with its degree bins (spmv.cu): small rows (deg <= kSmallMax),
// medium rows (deg <= kMediumMax) and hub-row chunks; out_row maps row i of this CSR to the output
// row it updates (null = identity).
struct CsrPart {
  DArr<int32_t> rowptr, col, small_rows, medium_rows, out_row;
  DArr<int4> chunks;
  int32_t n_rows = 0;
  int64_t nnz = 0;
  int n_small = 0, n_medium = 0, n_chunks = 0;
  int small_first = -1;  // small rows form the contiguous id range [small_first, +n_small), or -1
  int medium_first = -1; // medium rows form the contiguous id range [medium_first, +n_medium), or -1
  int n_iso = 0;          // the last n_iso rows of that range have no nonzeros

  void upload(const std::vector<int32_t>& rp, const std::vector<int32_t>& col_h, const std::vector<int32_t>* rows) {
    n_rows = (int32_t)rp.size() - 1;
    nnz = rp.back();
    std::vector<int32_t> sm, md;
    std::vector<int4> ch;
    for (int64_t r = 0; r < n_rows; ++r) {
      const int32_t d = rp[r + 1] - rp[r];
      if (d <= kSmallMax) sm.push_back((int32_t)r);
      else if (d <= kMediumMax) md.push_back((int32_t)r);
      else {
        const int first = (int)ch.size();
        for (int32_t z = rp[r]; z < rp[r + 1]; z += kHubChunk)
          ch.push_back(make_int4((int)r, z, std::min(z + kHubChunk, rp[r + 1]), first));
      }
    }
    n_small = (int)sm.size();
    n_medium = (int)md.size();
    // the batched small-row kernel needs contiguous ids and writes rows in place (no out_row)
    small_first = (!rows && !sm.empty() && sm.back() - sm.front() + 1 == (int32_t)sm.size()) ? sm.front() : -1;
    // (the degree-sorted relabelling makes both ranges contiguous: the kernels then skip the row-list load)
    medium_first = (!md.empty() && md.back() - md.front() + 1 == (int32_t)md.size()) ? md.front() : -1;
    // trailing rows of that range without nonzeros (isolated vertices sort last): a plain stream kernel
    n_iso = 0;
    if (small_first >= 0)
      for (int64_t r = small_first + n_small - 1; r >= small_first && rp[r + 1] == rp[r]; --r) ++n_iso;
    n_chunks = (int)ch.size();
    small_rows.alloc(std::max<size_t>(1, sm.size()));
    medium_rows.alloc(std::max<size_t>(1, md.size()));
    chunks.alloc(std::max<size_t>(1, ch.size()));
    if (!sm.empty()) WL_CUDA(cudaMemcpy(small_rows.p, sm.data(), 4 * sm.size(), cudaMemcpyHostToDevice));
    if (!md.empty()) WL_CUDA(cudaMemcpy(medium_rows.p, md.data(), 4 * md.size(), cudaMemcpyHostToDevice));
    if (!ch.empty()) WL_CUDA(cudaMemcpy(chunks.p, ch.data(), sizeof(int4) * ch.size(), cudaMemcpyHostToDevice));
    rowptr.alloc(n_rows + 1);
    col.alloc(std::max<int64_t>(nnz, 1));
    WL_CUDA(cudaMemcpy(rowptr.p, rp.data(), sizeof(int32_t) * (n_rows + 1), cudaMemcpyHostToDevice));
    if (nnz) WL_CUDA(cudaMemcpy(col.p, col_h.data(), sizeof(int32_t) * nnz, cudaMemcpyHostToDevice));
    if (rows) {
      out_row.alloc(std::max<size_t>(1, rows->size()));
      if (!rows->empty()) WL_CUDA(cudaMemcpy(out_row.p, rows->data(), 4 * rows->size(), cudaMemcpyHostToDevice));
    }
  }
};

}  // namespace wl

using wl::DArr;
using wl::Error;

struct wl_operator {
  int device = 0;
  wl_comm* comm = nullptr;
  int nranks = 1, rank = 0;
  int64_t n_global = 0, row_begin = 0, row_end = 0;
  int32_t n_loc = 0, nnz_loc = 0;
  // rows [n_act, n_loc) of the internal order are isolated (no nonzeros, referenced by no row of any rank): every
  // Krylov vector built from A v vanishes there (q_k(A) v = 0 for k >= 1, R13), so the Krylov batches store and
  // stream only the first n_act rows; their outputs there are c_0 v (φ) and t' v = 0 (𝕃)
  int64_t n_act = 0;
  // SpMM operand: A (all local rows; with split, only their local columns) and, with split, Ah (the
  // rows that reference halo columns, only those columns) — the A_loc / A_halo split of SURVEY §8(e):
  // A's SpMM runs while the halo is in flight, Ah's adds the halo terms after it arrived.
  wl::CsrPart A, Ah;
  bool split = false;
  DArr<int32_t> rowptr_full;  // split only: row pointer of the full local rows (degrees d_i)
  const int32_t* degrp() const { return split ? rowptr_full.p : A.rowptr.p; }
  // halo plan (rows exchanged per SpMM; counts in rows)
  int64_t n_halo = 0, n_send = 0;
  std::vector<int64_t> send_cnt, send_displ, recv_cnt, recv_displ;
  DArr<int32_t> send_idx;
  // walk weights / parameters
  int n_theta = 1;
  std::vector<double> theta, mu;
  DArr<double> mu_dev;
  int fkind = WL_F_EXP;
  double fparam = 1.0, c0 = 1.0;
  double lscale = 1.0;  // multiplies 𝕃 (wl_walkfun.scale)
  mutable DArr<int> kstat;  // sticky a-posteriori Krylov check (opts.tol): [bits, pad, max estimate (2 ints)]
  std::vector<double> coeffs;
  DArr<double> coeffs_dev;
  wl_opts opts{};
  DArr<double> tprime;  // n_loc x n_theta, internal row order: t - c_0 (φ1 minus its identity term)
  DArr<int32_t> perm;   // internal row -> user row (degree-sorted relabelling); empty = identity
  // buffers of the spectral-radius estimates (0: ρ(A), 1: ρ(Z_θ)), kept between calls: a fresh workspace per
  // call cost a cudaMalloc/cudaFree of k+3 outer vectors (~10 GB for ρ(Z) on C4) each time
  mutable struct wl_workspace* est_ws[2] = {nullptr, nullptr};
};

struct wl_workspace {
  const wl_operator* op = nullptr;
  int max_b = 1, Bmax = 1, K = 30;
  DArr<double> basis, S, Vb, halo_send, halo_recv;
  DArr<double> partials, sums1, sums2, sums3;
  DArr<unsigned int> ticket;
  DArr<double> H, s_all, n0, comb, scratch, ref, coef_v, coef_s;
  DArr<int> keff, vcol, tcol;
  DArr<double> colp;  // g0z, g1z, g0s, g1s (kMaxCols each)
  DArr<double> chunk_part;
  DArr<unsigned int> row_ticket;
  // multi-rank: the halo exchange runs on its own stream, overlapping the local SpMM
  cudaStream_t cstream = nullptr;
  cudaEvent_t ev_pack = nullptr, ev_halo = nullptr;
  // conjugate-gradient solver state (cg.cu): per column constants, scalars, |b|², iterations, flags
  DArr<double> cg_cs, cg_sc, cg_bb;
  DArr<int> cg_iters, cg_flags;
  int* cg_flags_host = nullptr;  // pinned: 2 flags + kMaxCols iteration counts
  int64_t cg_iterations = 0;     // executed CG iterations (max over the columns of each solve), cumulative
  int64_t krylov_steps = 0, krylov_batches = 0;  // Arnoldi steps taken / Krylov batches run (adaptive stop)
  int k_last = 0;                                 // steps of the previous batch (first adaptive probe)
  DArr<int> kprobe;              // adaptive stop: probe dimensions per column + flag (4 ints)
  DArr<double> kcomb;            // adaptive stop: the probe's f_1(H_m)e_1 (discarded)
  int* kflag_host = nullptr;
  DArr<double> mk_p, mk_v;       // Markov chain: current distribution and p / t (internal order)
  DArr<double> kerr;             // a-posteriori Krylov error estimates per column (opts.tol > 0)
  DArr<double> seed;             // TOAR shared seeds: v, A v, A(Av) over the b input columns
  DArr<int> vid;                 // 0, 1, ..., kMaxCols-1
  DArr<double> toar_state, toar_cy, toar_cu, toar_comb;  // TOAR (toar.cu): per-column state, update coefficients
  DArr<double> xg;               // TOAR: the SpMM's gathered block with rows padded to pad_cols(B) (zero phantoms)
  DArr<double> seed32;           // TOAR, opts.fp32: A v and A(Av) - μ d v in double before rounding (2 n x B)
  // host-buffer entry point
  DArr<double> hV, hLV;
  // diffusion (outer Lanczos)
  int kout_alloc = 0;
  DArr<double> oQ, ow, oH, on0, oref, osums1, ocoef_v, ocoef_s, otau, oY, oscratch;
  DArr<int> okeff;
  // XNysTrace-exp (wl_xnystrace_exp): block basis, block, temp block, Gram blocks, Gram partials (block.cu)
  DArr<double> trV, trW, trW2, trC, trR, trPart;
  // rational XNysTrace-exp: continuation block, MINRES vectors (v, v_prev, w1, w2, x, p; 2 halves each)
  DArr<double> rkU, mrV;
  DArr<double> mr_sc, mr_sums;
  DArr<int> mr_nact;
  int* mr_nact_host = nullptr;
  ~wl_workspace() {
    if (cstream) cudaStreamDestroy(cstream);
    if (ev_pack) cudaEventDestroy(ev_pack);
    if (ev_halo) cudaEventDestroy(ev_halo);
    if (cg_flags_host) cudaFreeHost(cg_flags_host);
    if (mr_nact_host) cudaFreeHost(mr_nact_host);
    if (kflag_host) cudaFreeHost(kflag_host);
  }
};

namespace wl {
namespace {

inline cudaStream_t S_(wl_stream s) { return reinterpret_cast<cudaStream_t>(s); }
inline bool multi(const wl_operator* op) { return op->comm && op->comm->nranks > 1; }

void allreduce(const wl_operator* op, double* buf, size_t count, cudaStream_t s) {
  if (!multi(op)) return;
  comm_allreduce(op->comm, buf, count, s);
}

// Rows of `src` (n_loc x B, ld lds) that other ranks reference are packed and exchanged into
// ws->halo_recv (n_halo x B), ordered by owner rank then global id (comm.cu: grouped NCCL
// send/recv, or device copies in a loopback group).
// f32: src and the halo buffers hold float (opts.fp32 TOAR batches).
void halo_post(const wl_operator* op, wl_workspace* ws, const double* src, int64_t lds, int w, bool f32,
               cudaStream_t pack_stream, cudaStream_t xfer_stream, cudaEvent_t ev) {
  if (f32) pack_rows_f32(reinterpret_cast<const float*>(src), lds, op->send_idx.p, op->n_send, w,
                         reinterpret_cast<float*>(ws->halo_send.p), pack_stream);
  else pack_rows(src, lds, op->send_idx.p, op->n_send, w, ws->halo_send.p, pack_stream);
  if (ev) {
    WL_CUDA(cudaEventRecord(ev, pack_stream));
    WL_CUDA(cudaStreamWaitEvent(xfer_stream, ev, 0));
  }
  const size_t esz = f32 ? sizeof(float) : sizeof(double);
  char* sb = reinterpret_cast<char*>(ws->halo_send.p);
  char* rb = reinterpret_cast<char*>(ws->halo_recv.p);
  std::vector<Xfer> sends, recvs;
  for (int p = 0; p < op->nranks; ++p) {
    if (p == op->rank) continue;
    if (op->send_cnt[p] > 0) sends.push_back({sb + esz * op->send_displ[p] * w, esz * op->send_cnt[p] * w, p});
    if (op->recv_cnt[p] > 0) recvs.push_back({rb + esz * op->recv_displ[p] * w, esz * op->recv_cnt[p] * w, p});
  }
  comm_sendrecv(op->comm, sends, recvs, xfer_stream);
}
void halo_exchange(const wl_operator* op, wl_workspace* ws, const double* src, int64_t lds, int B,
                   cudaStream_t s, bool f32 = false) {
  if (!multi(op)) return;
  WL_NVTX("halo_exchange");
  halo_post(op, ws, src, lds, B, f32, s, s, nullptr);
}

// One SpMM launch over CSR part `part` of the operator (see wl_operator::A / Ah).
void spmv_part(const wl_operator* op, wl_workspace* ws, const CsrPart& part, bool halo_part, const double* y,
               int64_t ldy, const double* x, const double* g0, const double* g1, const double* scale, double* out,
               int B, cudaStream_t s, const int* active, bool f32, int64_t rows) {
  SpmvArgs a{};
  a.active = active;
  a.f32 = f32 ? 1 : 0;
  a.row_limit = rows;
  a.rowptr = part.rowptr.p;
  a.col = part.col.p;
  a.n_loc = op->n_loc;
  a.small_rows = part.small_rows.p;
  a.n_small = part.n_small;
  a.small_first = part.small_first;
  a.medium_first = part.medium_first;
  a.n_iso = part.n_iso;
  a.medium_rows = part.medium_rows.p;
  a.n_medium = part.n_medium;
  a.chunks = part.chunks.p;
  a.n_chunks = part.n_chunks;
  a.chunk_part = ws->chunk_part.p;
  a.row_ticket = ws->row_ticket.p;
  a.out_row = part.out_row.p;
  a.y = y;
  a.ldy = ldy;
  // halo rows: the full CSR without split, or the Ah part with it
  const bool with_halo = multi(op) && op->n_halo > 0 && (halo_part || !op->split);
  a.yh = with_halo ? ws->halo_recv.p : nullptr;
  a.ldh = ldy;  // halo rows are packed with the gathered block's row width
  a.n_halo = op->n_halo;
  a.ldx = B;
  a.out = out;
  a.ldo = B;
  a.B = B;
  if (halo_part) {  // out += scale * Σ_halo y: no diagonal term
    a.accumulate = 1;
    a.scale = scale;
  } else {
    a.x = x;
    a.g0 = g0;
    a.g1 = g1;
    a.scale = scale;
    a.degptr = op->split ? op->rowptr_full.p : nullptr;  // γ = μ(μ - d) needs the full degree
  }
  spmv(a, s);
}

// Z-SpMM out = scale ⊙ (A y + (g0 + g1 d) ⊙ x) with y in this rank's rows (n_loc x B, ld ldy >= B: the
// gathered block may be padded to a row width the wide-lane gathers can load, spmv.cu).
// Multi-rank: the rows of y that peers reference are exchanged first (whole padded rows); with the
// A_loc / A_halo split (opts.halo_overlap) the exchange runs on the workspace's comm stream while
// A_loc's SpMM runs, and A_halo's SpMM adds the halo terms once it has arrived.
// f32: y, x and out hold float (opts.fp32 TOAR batches; element strides).  rows > 0: only output rows < rows are
// written (the Krylov batches' active rows; the isolated rows beyond are never gathered)
void do_spmv(const wl_operator* op, wl_workspace* ws, const double* y, int64_t ldy, const double* x,
             const double* g0, const double* g1, const double* scale, double* out, int B,
             cudaStream_t s, const int* active = nullptr, bool f32 = false, int64_t rows = 0) {
  if (!multi(op) || !op->split) {
    halo_exchange(op, ws, y, ldy, (int)ldy, s, f32);
    spmv_part(op, ws, op->A, false, y, ldy, x, g0, g1, scale, out, B, s, active, f32, rows);
    return;
  }
  halo_post(op, ws, y, ldy, (int)ldy, f32, s, ws->cstream, ws->ev_pack);
  WL_CUDA(cudaEventRecord(ws->ev_halo, ws->cstream));
  spmv_part(op, ws, op->A, false, y, ldy, x, g0, g1, scale, out, B, s, active, f32, rows);
  WL_CUDA(cudaStreamWaitEvent(s, ws->ev_halo, 0));
  spmv_part(op, ws, op->Ah, true, y, ldy, x, g0, g1, scale, out, B, s, active, f32, rows);
}

// halo buffers, comm stream and events of a workspace (multi-rank)
void ws_comm_init(const wl_operator* op, wl_workspace* ws, int B) {
  if (op->n_halo > 0 && ws->halo_recv.n < (size_t)op->n_halo * B) ws->halo_recv.alloc((size_t)op->n_halo * B);
  if (op->n_send > 0 && ws->halo_send.n < (size_t)op->n_send * B) ws->halo_send.alloc((size_t)op->n_send * B);
  if (op->split && !ws->cstream) {
    WL_CUDA(cudaStreamCreateWithFlags(&ws->cstream, cudaStreamNonBlocking));
    WL_CUDA(cudaEventCreateWithFlags(&ws->ev_pack, cudaEventDisableTiming));
    WL_CUDA(cudaEventCreateWithFlags(&ws->ev_halo, cudaEventDisableTiming));
  }
}

// Scratch of the hub-row chunks (partials + tickets) for B columns.
void spmv_scratch(const wl_operator* op, wl_workspace* ws, int B) {
  ws_comm_init(op, ws, B);
  const int nch = std::max(op->A.n_chunks, op->Ah.n_chunks);  // the two parts run one after the other
  if (nch == 0) return;
  // a chunk's partial row holds W * VW <= 32 values (every lane slot of its group, either storage type)
  if (ws->chunk_part.n < (size_t)nch * kMaxCols) ws->chunk_part.alloc((size_t)nch * kMaxCols);
  if (ws->row_ticket.n < (size_t)nch) {
    ws->row_ticket.alloc(nch);
    WL_CUDA(cudaMemset(ws->row_ticket.p, 0, sizeof(unsigned int) * nch));
  }
}

// One Krylov action on global output columns [gstart, gstart + B) of the n_theta*b block;
// `out` points at column gstart.  mode: 0 = φV, 1 = 𝕃V, 2 = t' (V = ones).
// user_order: V / out rows are in the caller's order (gathered / scattered through op->perm);
// false for the internal-order vectors of the outer diffusion Lanczos.
void krylov_chunk(const wl_operator* op, wl_workspace* ws, int mode, const double* V, int64_t ldv, int b,
                  int gstart, int B, double* out, int64_t ldo, cudaStream_t s, bool user_order) {
  WL_NVTX("krylov_batch_dcgs2");
  const int32_t* perm = user_order ? op->perm.p : nullptr;
  const int64_t n = op->n_loc;
  const int K = ws->K;
  // Z-vector halves hold n_pad >= n rows, n_pad * B even (a zero phantom row when n and B are
  // both odd): every half starts 16-byte aligned for the bulk copies of the DCGS2 passes.
  const int64_t n_pad = n + ((n * B) & 1);
  const int64_t L = 2 * n_pad;
  const int64_t vstride = L * B;
  double* g0z = ws->colp.p;
  double* g1z = g0z + kMaxCols;
  double* g0s = g1z + kMaxCols;
  double* g1s = g0s + kMaxCols;
  setup_chunk(op->mu_dev.p, gstart, b, B, g0z, g1z, g0s, g1s, ws->vcol.p, ws->tcol.p, s);
  batch_inputs(V, ldv, B, n, ws->Vb.p, ws->vcol.p, perm, s);
  double* Q0 = ws->basis.p;
  // a3: seeds q_1 v = A v (top) and q_2 v = A(Av) - μ d⊙v (bottom)   (eq:qrec seeds)
  do_spmv(op, ws, ws->Vb.p, B, nullptr, nullptr, nullptr, nullptr, Q0, B, s);
  do_spmv(op, ws, Q0, B, ws->Vb.p, g0s, g1s, nullptr, Q0 + n_pad * B, B, s);
  if (n_pad > n) {  // phantom rows of the seed vector and of S stay zero; the passes keep them so
    fill(Q0 + n * B, B, 0.0, s);
    fill(Q0 + (n_pad + n) * B, B, 0.0, s);
    fill(ws->S.p + n * B, B, 0.0, s);
  }
  // a5: Arnoldi with delayed classical Gram-Schmidt (DCGS2): per step one SpMM, one fused dot
  // pass (single reduction / allreduce) and one fused two-output update pass.
  WL_CUDA(cudaMemsetAsync(ws->H.p, 0, sizeof(double) * B * (K + 1) * K, s));
  // Basis slots: vector slot i -> buffer; slot K+1 is the spare that receives q_j, after which the
  // buffers of slots j and K+1 swap (q_j never overwrites p_j while pass B still reads it).
  VecPtrs slot{};
  for (int i = 0; i < K + 2; ++i) slot.p[i] = ws->basis.p + (int64_t)i * vstride;
  Dcgs2Args d{};
  d.len = L;
  d.B = B;
  d.partials = ws->partials.p;
  d.sums_out = ws->sums1.p;
  d.coef_v = ws->coef_v.p;
  d.coef_s = ws->coef_s.p;
  const double btol = op->opts.breakdown_tol;
  for (int j = 0; j < K; ++j) {
    double* Pj = const_cast<double*>(slot.p[j]);
    // a4: S = A Pj_bot + μ(μ - d) Pj_top — bottom half of Z p_j; its top half is Pj_bot
    do_spmv(op, ws, Pj + n_pad * B, B, Pj, g0z, g1z, nullptr, ws->S.p, B, s);
    d.Q = slot;
    d.nq = j;
    d.P = Pj;
    d.wa = Pj + n_pad * B;
    d.split = n_pad;
    d.wb = ws->S.p;
    dcgs2_dots(d, s);
    allreduce(op, ws->sums1.p, (size_t)(2 * j + 3) * B, s);
    dcgs2_coeffs(ws->sums1.p, j, B, K, btol, 0, op->opts.reorth, ws->H.p, ws->ref.p, ws->n0.p, ws->keff.p,
                 ws->coef_v.p, ws->coef_s.p, s);
    d.Qout = const_cast<double*>(slot.p[K + 1]);
    d.Pnext = const_cast<double*>(slot.p[j + 1]);
    d.accumulate = 0;
    dcgs2_update(d, s);
    std::swap(slot.p[j], slot.p[K + 1]);
  }
  {  // delayed reorthogonalisation of p_K completes column K-1 of H
    d.Q = slot;
    d.nq = K;
    d.P = slot.p[K];
    d.wa = nullptr;
    d.wb = nullptr;
    d.split = n_pad;
    dcgs2_dots(d, s);
    allreduce(op, ws->sums1.p, (size_t)(2 * K + 3) * B, s);
    dcgs2_coeffs(ws->sums1.p, K, B, K, btol, 1, op->opts.reorth, ws->H.p, ws->ref.p, ws->n0.p, ws->keff.p,
                 ws->coef_v.p, ws->coef_s.p, s);
  }
  // a6: y = f_1(H_k) e_1 per column; comb_i = ||u|| y_i  (q_i stored normalised)
  SmallFArgs f{};
  f.H = ws->H.p;
  f.K = K;
  f.keff = ws->keff.p;
  f.kind = op->fkind;
  f.param = op->fparam;
  f.coeffs = op->coeffs_dev.p;
  f.ncoeffs = (int)op->coeffs.size();
  f.n0 = ws->n0.p;
  f.s = nullptr;
  f.comb = ws->comb.p;
  f.scratch = ws->scratch.p;
  f.B = B;
  f.err = op->opts.tol > 0.0 ? ws->kerr.p : nullptr;
  small_f(f, s);
  if (op->opts.tol > 0.0) krylov_check(ws->kerr.p, B, op->opts.tol, op->kstat.p, s);
  // a7: combine (top halves of the basis)
  combine(mode, op->lscale, slot, K, n, B, ws->comb.p, V, ldv, ws->vcol.p, op->c0,
          op->tprime.p, op->n_theta, ws->tcol.p, out, ldo, perm, s);
}


// TOAR Arnoldi on Z (opts.reorth == 2; toar.cu): the 2n-long basis is q_i = [U g_i; U f_i] over K+2
// n-vectors U, so each step runs one dot pass and one three-output update pass over U (n-vectors)
// instead of DCGS2's two passes over 2n-vectors.  Same seeds, SpMM, f(H) and combine as krylov_chunk.
void toar_chunk(const wl_operator* op, wl_workspace* ws, int mode, const double* V, int64_t ldv, int b, int gstart,
                int B, double* out, int64_t ldo, cudaStream_t s, bool user_order) {
  WL_NVTX("krylov_batch_toar");
  const int32_t* perm = user_order ? op->perm.p : nullptr;
  const int64_t n = op->n_act;  // the rows the Krylov vectors live on (isolated rows beyond: §6)
  const int K = ws->K;
  // opts.fp32: the n-vectors of the batch (U, x, z, y and the gathered block) hold float; the seeds, every sum and
  // the coefficient work stay double.  t' (mode 2, at create) is always computed in double.
  const bool f32 = op->opts.fp32 && mode != 2;
  const size_t esz = f32 ? sizeof(float) : sizeof(double);
  // bulk copies move whole 16-byte pieces: the element count of a vector is padded with zero phantom rows
  int64_t n_pad = n;
  while ((n_pad * B * (int64_t)esz) % 16) ++n_pad;
  const int64_t vs = n_pad * B;
  auto vec = [&](int64_t i) -> double* {  // vector slot i of the basis allocation, in the storage type
    return f32 ? reinterpret_cast<double*>(reinterpret_cast<float*>(ws->basis.p) + i * vs) : ws->basis.p + i * vs;
  };
  auto zero_rows = [&](double* v, int64_t r0, int64_t r1) {  // rows [r0, r1) of an n_pad x B vector
    if (r1 > r0)
      WL_CUDA(cudaMemsetAsync(reinterpret_cast<char*>(v) + (size_t)r0 * B * esz, 0, (size_t)(r1 - r0) * B * esz, s));
  };
  double* g0z = ws->colp.p;
  double* g1z = g0z + kMaxCols;
  double* g0s = g1z + kMaxCols;
  double* g1s = g0s + kMaxCols;
  setup_chunk(op->mu_dev.p, gstart, b, B, g0z, g1z, g0s, g1s, ws->vcol.p, ws->tcol.p, s);
  VecPtrs U{};
  for (int i = 0; i < K + 2; ++i) U.p[i] = vec(i);
  double* xb = vec(K + 2);
  double* zb = vec(K + 3);
  double* yb = vec(K + 4);
  double* U0 = const_cast<double*>(U.p[0]);
  // a3 seeds: t0 = A v -> U_0, b0 = A t0 - μ d⊙v -> x   (eq:qrec seeds); q̂_0 = [t0; b0]
  if (b < B && gstart % b == 0 && B % b == 0) {
    // A v and A(Av) do not depend on θ: two SpMMs over the b input columns, expanded to the B columns
    double* vs_ = ws->seed.p;
    double* s1 = vs_ + (n + 1) * b;
    double* s2 = s1 + (n + 1) * b;
    batch_inputs(V, ldv, b, n, vs_, ws->vid.p, perm, s);
    do_spmv(op, ws, vs_, b, nullptr, nullptr, nullptr, nullptr, s1, b, s, nullptr, false, n);
    do_spmv(op, ws, s1, b, nullptr, nullptr, nullptr, nullptr, s2, b, s, nullptr, false, n);
    seed_expand(s1, s2, vs_, b, op->degrp(), g1s, ws->vcol.p, B, n, U0, xb, s, f32);
  } else if (!f32) {
    batch_inputs(V, ldv, B, n, ws->Vb.p, ws->vcol.p, perm, s);
    do_spmv(op, ws, ws->Vb.p, B, nullptr, nullptr, nullptr, nullptr, U0, B, s, nullptr, false, n);
    do_spmv(op, ws, U0, B, ws->Vb.p, g0s, g1s, nullptr, xb, B, s, nullptr, false, n);
  } else {  // fp32: the seeds in double, then rounded once
    double* t1 = ws->seed32.p;
    double* t2 = t1 + (n + 1) * B;
    batch_inputs(V, ldv, B, n, ws->Vb.p, ws->vcol.p, perm, s);
    do_spmv(op, ws, ws->Vb.p, B, nullptr, nullptr, nullptr, nullptr, t1, B, s, nullptr, false, n);
    do_spmv(op, ws, t1, B, ws->Vb.p, g0s, g1s, nullptr, t2, B, s, nullptr, false, n);
    repack_rows_t(t1, false, B, n, B, U0, true, B, 0, s);
    repack_rows_t(t2, false, B, n, B, xb, true, B, 0, s);
  }
  zero_rows(U0, n, n_pad);
  zero_rows(xb, n, n_pad);
  zero_rows(yb, n, n_pad);
  WL_CUDA(cudaMemsetAsync(ws->H.p, 0, sizeof(double) * B * (K + 1) * K, s));
  const size_t stride = toar_state_doubles(K);
  const int ld = K + 3;
  const double btol = op->opts.breakdown_tol;
  Dcgs2Args d{};
  d.len = n_pad;
  d.B = B;
  d.split = n_pad;
  d.partials = ws->partials.p;
  d.sums_out = ws->sums1.p;
  d.Q = U;
  d.f32 = f32 ? 1 : 0;
  ToarArgs t{};
  t.U = U;
  t.len = n_pad;
  t.B = B;
  t.f32 = f32 ? 1 : 0;
  t.coef_y = ws->toar_cy.p;
  t.coef_u = ws->toar_cu.p;
  t.coef_ld = ld;
  // one GPU, <= 32 basis vectors per dot pass: toar_coeffs reduces the dot pass's partials itself;
  // otherwise the pass reduces them and NCCL allreduces the sums across ranks
  const bool fuse = !multi(op) && K + 1 <= 32;
  int G = 0;
  auto dots = [&](int count) {
    d.sums_out = fuse ? nullptr : ws->sums1.p;
    G = dcgs2_dots(d, s);
    if (!fuse) allreduce(op, ws->sums1.p, (size_t)count, s);
  };
  auto coeffs = [&](int j, int final_pass) {
    toar_coeffs(ws->sums1.p, fuse ? ws->partials.p : nullptr, G, j, final_pass, B, K, btol, ws->H.p, ws->n0.p,
                ws->keff.p, ws->toar_state.p, stride, ws->toar_cy.p, ws->toar_cu.p, ld, s);
  };
  // seed step: Gram of (t0, b0), u_1 = (b0 - proj)/ν
  d.nq = 0;
  d.P = U0;
  d.wa = xb;
  dots(3 * B);
  coeffs(-1, 0);
  t.m = 1;
  t.y = xb;
  t.out[0] = const_cast<double*>(U.p[1]);
  t.nout = 1;
  toar_update(t, s);
  // The SpMM gathers rows of x.  With B not a multiple of 4 they are kept in a second block xg whose
  // rows are padded to ldg = 4 ceil(B/4) doubles (zero phantom columns), so every gathered row is
  // whole 32-byte pieces for the 256-bit lane loads (spmv.cu): the update pass writes x there
  // directly; the seed's x is repacked once.  (Tiled update passes, K + 1 > 32, keep ld B.)
  const int64_t ldg = ws->xg.p ? (f32 ? pad_cols_t<float>(B) : pad_cols(B)) : B;
  const bool padx = ldg != B && K + 1 <= 32;
  double* xg = padx ? ws->xg.p : xb;
  if (padx) repack_rows_t(xb, f32, B, n, B, xg, f32, ldg, f32 ? pad_vec_t<float>(B) : pad_vec(B), s);
  const double* xin = xg;  // bottom half of the vector the next SpMM applies Z to
  const int64_t ldx_in = padx ? ldg : B;
  const double* zin = U0;  // its top half
  // opts.krylov_adaptive: after step j (j + 1 >= 6, every 2 steps) the a-posteriori estimate of smallf.cu is
  // evaluated on the final H columns 0..j-1 (m = j); once every column is below opts.tol the basis stops
  // at k' = j + 1 steps (the final pass completes column j).  One host synchronisation per probe.
  const bool adaptive = op->opts.krylov_adaptive && op->opts.tol > 0.0;
  int kstop = K;
  if (adaptive) {
    ws->kprobe.alloc(kMaxCols + 4);
    ws->kcomb.alloc((size_t)(K + 1) * B);
    if (!ws->kflag_host) WL_CUDA(cudaMallocHost(&ws->kflag_host, 4 * sizeof(int)));
  }
  for (int j = 0; j < K; ++j) {
    WL_NVTX("arnoldi_step");
    const int m = j + 2;
    // a4: y = A x + μ(μ - d)⊙z  (bottom half of Z [z; x])
    do_spmv(op, ws, xin, ldx_in, zin, g0z, g1z, nullptr, yb, B, s, nullptr, f32, n);
    // a5: one dot pass (Gram row of the newest U vector, U^T y, |y|^2) and one update pass
    d.nq = m - 1;
    d.P = U.p[m - 1];
    d.wa = yb;
    dots((2 * (m - 1) + 3) * B);
    coeffs(j, 0);
    t.m = m;
    t.y = yb;
    t.out[0] = const_cast<double*>(U.p[m]);
    t.out[1] = xg;
    t.out_ld[1] = ldx_in;
    t.out[2] = zb;
    t.nout = 3;
    toar_update(t, s);
    t.out_ld[1] = 0;
    xin = xg;
    zin = zb;
    // first probe: 2 steps before the previous batch's stop (repeated actions — a diffusion sweep, CG-free
    // trace steps — converge alike), never before k' = 6; then every 2 steps
    const int kfirst = std::max(6, ws->k_last - 2);
    if (adaptive && j + 1 < K && j + 1 >= kfirst && (j + 1 - kfirst) % 2 == 0) {
      int* kp = ws->kprobe.p;
      int* flag = kp + kMaxCols;
      clamp_keff(ws->keff.p, j, B, kp, flag, s);
      SmallFArgs f{};
      f.H = ws->H.p;
      f.K = K;
      f.keff = kp;
      f.kind = op->fkind;
      f.param = op->fparam;
      f.coeffs = op->coeffs_dev.p;
      f.ncoeffs = (int)op->coeffs.size();
      f.n0 = ws->n0.p;
      f.comb = ws->kcomb.p;
      f.scratch = ws->scratch.p;
      f.B = B;
      f.err = ws->kerr.p;
      small_f(f, s);
      krylov_check(ws->kerr.p, B, op->opts.tol, flag, s);
      WL_CUDA(cudaMemcpyAsync(ws->kflag_host, flag, 4 * sizeof(int), cudaMemcpyDeviceToHost, s));
      WL_CUDA(cudaStreamSynchronize(s));
      static const bool dbg = getenv("WL_DEBUG_ADAPTIVE") != nullptr;
      if (dbg) {
        double est;
        std::memcpy(&est, ws->kflag_host + 2, sizeof(est));
        fprintf(stderr, "[adaptive] step %d probe m=%d flag=%d max_est=%.3e (k_last %d)\n", j + 1, j, ws->kflag_host[0], est,
                ws->k_last);
      }
      if ((ws->kflag_host[0] & 1) == 0) {
        kstop = j + 1;
        break;
      }
    }
  }
  ws->krylov_steps += kstop;
  ws->krylov_batches += 1;
  ws->k_last = kstop;
  d.nq = kstop + 1;  // Gram row of the last U vector completes H column kstop-1
  d.P = U.p[kstop + 1];
  d.wa = nullptr;
  dots((2 * (kstop + 1) + 3) * B);
  coeffs(kstop, 1);
  WL_NVTX("f_of_H_and_combine");
  // a6: y = f_1(H_k) e_1 per column; a7: combine top halves U (Σ_i comb_i g_i)
  SmallFArgs f{};
  f.H = ws->H.p;
  f.K = K;
  f.keff = ws->keff.p;
  f.kind = op->fkind;
  f.param = op->fparam;
  f.coeffs = op->coeffs_dev.p;
  f.ncoeffs = (int)op->coeffs.size();
  f.n0 = ws->n0.p;
  f.s = nullptr;
  f.comb = ws->comb.p;
  f.scratch = ws->scratch.p;
  f.B = B;
  f.err = op->opts.tol > 0.0 ? ws->kerr.p : nullptr;
  small_f(f, s);
  if (op->opts.tol > 0.0) krylov_check(ws->kerr.p, B, op->opts.tol, op->kstat.p, s);
  toar_combine_coef(ws->comb.p, B, K, ws->keff.p, ws->toar_state.p, stride, ws->toar_comb.p, s);
  combine(mode, op->lscale, U, kstop + 2, op->n_loc, B, ws->toar_comb.p, V, ldv, ws->vcol.p, op->c0, op->tprime.p,
          op->n_theta, ws->tcol.p, out, ldo, perm, s, f32, n);
}

// μ = 0 (θ = 1) chunks: symmetric Lanczos on A from u = A v (lanczos.cu; "Lanczos (for A = Aᵀ)"):
// φ v = c_0 v + ‖u‖ Q_k f_1(T_k) e_1 with the same f_1, small_f and combine as the companion path.
void lanczos_chunk(const wl_operator* op, wl_workspace* ws, int mode, const double* V, int64_t ldv, int b,
                   int gstart, int B, double* out, int64_t ldo, cudaStream_t s, bool user_order) {
  WL_NVTX("krylov_batch_lanczos");
  const int32_t* perm = user_order ? op->perm.p : nullptr;
  const int64_t n = op->n_act;  // the rows the Krylov vectors live on (isolated rows beyond: §6)
  const int K = ws->K;
  const bool f32 = op->opts.fp32 && mode != 2;  // float storage of the Lanczos vectors (R21); t' stays double
  const int64_t vs = (n + 1) * B;  // elements per vector (floats fill half of a double slot)
  double* g0z = ws->colp.p;
  double* g1z = g0z + kMaxCols;
  double* g0s = g1z + kMaxCols;
  double* g1s = g0s + kMaxCols;
  setup_chunk(op->mu_dev.p, gstart, b, B, g0z, g1z, g0s, g1s, ws->vcol.p, ws->tcol.p, s);
  VecPtrs Q{};
  for (int i = 0; i <= K; ++i)
    Q.p[i] = f32 ? reinterpret_cast<const double*>(reinterpret_cast<float*>(ws->basis.p) + (int64_t)i * vs)
                 : ws->basis.p + (int64_t)i * vs;
  batch_inputs(V, ldv, B, n, ws->Vb.p, ws->vcol.p, perm, s);
  const int G = lanczos_grid(n, B);
  const size_t need = (size_t)G * B;
  if (ws->partials.n < need) ws->partials.alloc(need);
  double* sc = ws->cg_sc.p;  // 4 slots per column: [β_j, α_j, scale, active]
  const double btol = op->opts.breakdown_tol;
  const int pres = multi(op) ? 1 : 0;
  auto scalar = [&](int which, int j) {
    if (pres) {
      reduce_partials(ws->partials.p, B, G, ws->sums1.p, s);
      allreduce(op, ws->sums1.p, (size_t)B, s);
    }
    lanczos_scalar(which, j, n, pres, ws->partials.p, ws->sums1.p, B, K, btol, sc, ws->H.p, ws->n0.p, ws->keff.p, s);
  };
  WL_CUDA(cudaMemsetAsync(ws->H.p, 0, sizeof(double) * B * (K + 1) * K, s));
  double* q0 = const_cast<double*>(Q.p[0]);
  // the SpMM gathers q_j from a row-padded copy (32-byte lanes, §7) written by the scaling pass
  const int pc = f32 ? pad_cols_t<float>(B) : pad_cols(B);
  double* xg = ws->xg.p && pc != B ? ws->xg.p : nullptr;
  const int64_t ldg = xg ? pc : B;
  if (!f32) {
    do_spmv(op, ws, ws->Vb.p, B, nullptr, nullptr, nullptr, nullptr, q0, B, s, nullptr, false, n);  // u = A v (a3, μ = 0)
  } else {  // u = A v in double (v is double), rounded once
    do_spmv(op, ws, ws->Vb.p, B, nullptr, nullptr, nullptr, nullptr, ws->seed32.p, B, s, nullptr, false, n);
    repack_rows_t(ws->seed32.p, false, B, n, B, q0, true, B, 0, s);
  }
  lanczos_vec(0, q0, nullptr, nullptr, n, B, sc, ws->partials.p, s, nullptr, 0, f32);
  scalar(0, 0);
  lanczos_vec(3, q0, nullptr, nullptr, n, B, sc, ws->partials.p, s, xg, ldg, f32);   // q_0 = u / ‖u‖
  for (int j = 0; j < K; ++j) {
    double* qj = const_cast<double*>(Q.p[j]);
    double* w = const_cast<double*>(Q.p[j + 1]);
    do_spmv(op, ws, xg ? xg : qj, ldg, nullptr, nullptr, nullptr, nullptr, w, B, s, nullptr, f32, n);  // w' = A q_j
    lanczos_vec(1, qj, w, nullptr, n, B, sc, ws->partials.p, s, nullptr, 0, f32);
    scalar(1, j);                                                                 // α_j
    lanczos_vec(2, w, qj, j > 0 ? Q.p[j - 1] : nullptr, n, B, sc, ws->partials.p, s, nullptr, 0, f32);
    scalar(2, j);                                                                 // β_{j+1}
    lanczos_vec(3, w, nullptr, nullptr, n, B, sc, ws->partials.p, s, xg, ldg, f32);   // q_{j+1}
  }
  SmallFArgs f{};
  f.H = ws->H.p;
  f.K = K;
  f.keff = ws->keff.p;
  f.kind = op->fkind;
  f.param = op->fparam;
  f.coeffs = op->coeffs_dev.p;
  f.ncoeffs = (int)op->coeffs.size();
  f.n0 = ws->n0.p;
  f.s = nullptr;
  f.comb = ws->comb.p;
  f.scratch = ws->scratch.p;
  f.B = B;
  f.err = op->opts.tol > 0.0 ? ws->kerr.p : nullptr;
  small_f(f, s);
  if (op->opts.tol > 0.0) krylov_check(ws->kerr.p, B, op->opts.tol, op->kstat.p, s);
  combine(mode, op->lscale, Q, K, op->n_loc, B, ws->comb.p, V, ldv, ws->vcol.p, op->c0, op->tprime.p, op->n_theta,
          ws->tcol.p, out, ldo, perm, s, f32, n);
}

// Resolvent action by Jacobi-preconditioned CG on the deformed Laplacian (cg.cu; opts.solver ==
// WL_SOLVER_CG): x = 𝒜_θ(α)^{-1} V per column, then φ V = (1-μ²α²) x.  Vector roles reuse the
// Krylov basis memory: x, r, p, q.  Synchronizes every opts.cg_check iterations.
void cg_chunk(const wl_operator* op, wl_workspace* ws, int mode, const double* V, int64_t ldv, int b, int gstart,
              int B, double* out, int64_t ldo, cudaStream_t s, bool user_order) {
  WL_NVTX("cg_solve");
  const int32_t* perm = user_order ? op->perm.p : nullptr;
  // the isolated tail (R13) decouples: 𝒜 = (1 - μ²α²) I there, solved in closed form by cg_combine
  const int64_t n = op->n_act;
  double* g0 = ws->colp.p;
  double* g1 = g0 + kMaxCols;
  double* scale = g1 + kMaxCols;
  cg_setup(op->mu_dev.p, op->fparam, op->opts.cg_tol, gstart, b, B, ws->cg_cs.p, g0, g1, scale, ws->vcol.p,
           ws->tcol.p, s);
  batch_inputs(V, ldv, B, n, ws->Vb.p, ws->vcol.p, perm, s);
  CgArgs a{};
  a.n = n;
  a.B = B;
  a.rowptr = op->degrp();
  a.cs = ws->cg_cs.p;
  a.b = ws->Vb.p;
  a.x = ws->basis.p;
  a.r = a.x + n * B;
  a.p = a.r + n * B;
  a.q = a.p + n * B;
  a.partials = ws->partials.p;
  a.sums = ws->sums1.p;
  a.sc = ws->cg_sc.p;
  a.bb = ws->cg_bb.p;
  a.iters = ws->cg_iters.p;
  a.flags = ws->cg_flags.p;
  WL_CUDA(cudaMemsetAsync(ws->cg_flags.p, 0, 2 * sizeof(int), s));
  // reductions: one fused reduce+scalar CTA on one GPU; reduce -> NCCL allreduce -> scalar across GPUs
  auto reduce_scalar = [&](int which) {
    if (!multi(op)) return cg_reduce_scalar(which, a, s);
    cg_reduce(which, a, s);
    allreduce(op, a.sums, (size_t)(which == 1 ? 1 : 2) * B, s);
    cg_scalar(which, a, s);
  };
  cg_init(a, s);
  reduce_scalar(0);
  bool done = false;
  for (int it = 0; it < op->opts.cg_maxit && !done; ++it) {
    do_spmv(op, ws, a.p, B, a.p, g0, g1, scale, a.q, B, s, a.flags + 1, false, n);  // q = 𝒜 p
    cg_dot(a, s);
    reduce_scalar(1);
    cg_update(a, s);
    reduce_scalar(2);
    cg_direction(a, s);
    if ((it + 1) % op->opts.cg_check == 0 || it + 1 == op->opts.cg_maxit) {
      WL_CUDA(cudaMemcpyAsync(ws->cg_flags_host, ws->cg_flags.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
      WL_CUDA(cudaStreamSynchronize(s));
      if (ws->cg_flags_host[0] & 1) throw Error(WL_EDIVERGE, "CG: deformed Laplacian not positive definite (α ρ(Z_θ) >= 1?)");
      done = ws->cg_flags_host[1] == 0;
    }
  }
  cg_combine(mode, op->lscale, a.x, op->n_loc, B, ws->cg_cs.p, V, ldv, ws->vcol.p, op->c0, op->tprime.p, op->n_theta,
             ws->tcol.p, out, ldo, perm, s, n);
  WL_CUDA(cudaMemcpyAsync(ws->cg_flags_host + 2, ws->cg_iters.p, B * sizeof(int), cudaMemcpyDeviceToHost, s));
  WL_CUDA(cudaStreamSynchronize(s));
  ws->cg_iterations += *std::max_element(ws->cg_flags_host + 2, ws->cg_flags_host + 2 + B);
  if (!done) throw Error(WL_ENOCONV, "CG: residual above cg_tol after cg_maxit iterations (best iterate written)");
}

void run_chunk(const wl_operator* op, wl_workspace* ws, int mode, const double* V, int64_t ldv, int b, int gstart,
               int B, double* out, int64_t ldo, cudaStream_t s, bool user_order = true) {
  // every column θ = 1 (μ = 0): Lanczos on A
  bool walk = op->opts.reorth == 2 && op->opts.lanczos;
  for (int c = 0; c < B && walk; ++c) walk = op->mu[(gstart + c) / b] == 0.0;
  if (op->opts.solver == WL_SOLVER_CG) cg_chunk(op, ws, mode, V, ldv, b, gstart, B, out, ldo, s, user_order);
  else if (walk) lanczos_chunk(op, ws, mode, V, ldv, b, gstart, B, out, ldo, s, user_order);
  else if (op->opts.reorth == 2) toar_chunk(op, ws, mode, V, ldv, b, gstart, B, out, ldo, s, user_order);
  else krylov_chunk(op, ws, mode, V, ldv, b, gstart, B, out, ldo, s, user_order);
}

void run_action(const wl_operator* op, wl_workspace* ws, int mode, const double* V, int64_t ldv, int b,
                double* out, int64_t ldo, cudaStream_t s) {
  const int G = op->n_theta * b;
  for (int g0 = 0; g0 < G; g0 += ws->Bmax) {
    const int B = std::min(ws->Bmax, G - g0);
    run_chunk(op, ws, mode, V, ldv, b, g0, B, out + g0, ldo, s);
  }
}

void workspace_alloc(wl_workspace* ws, const wl_operator* op, int max_b) {
  ws->op = op;
  ws->max_b = max_b;
  ws->K = op->opts.krylov_dim;
  ws->Bmax = std::max(1, std::min({op->opts.max_cols, kMaxCols, op->n_theta * max_b}));
  const int64_t n = op->n_loc;
  const int B = ws->Bmax, K = ws->K;
  if (op->opts.solver == WL_SOLVER_CG) ws->basis.alloc((size_t)4 * (n + 1) * B);  // x, r, p, q
  else if (op->opts.reorth == 2) ws->basis.alloc((size_t)(K + 5) * (n + 1) * B);  // TOAR: U (K+2), x, z, y
  else ws->basis.alloc((size_t)(K + 2) * 2 * (n + 1) * B);  // halves padded by <= 1 phantom row
  ws->S.alloc((size_t)(n + 1) * B);
  ws->Vb.alloc((size_t)n * B);
  if (op->n_halo > 0) ws->halo_recv.alloc((size_t)op->n_halo * pad_cols(B));  // padded gathered rows
  if (op->n_send > 0) ws->halo_send.alloc((size_t)op->n_send * pad_cols(B));
  const int grid = gram_grid(2 * n * B, B);
  ws->partials.alloc((size_t)grid * (2 * K + 5) * B);
  ws->ref.alloc(B);
  ws->coef_v.alloc((size_t)2 * (K + 1) * B);
  ws->coef_s.alloc((size_t)3 * B);
  ws->sums1.alloc((size_t)(2 * K + 5) * B);
  ws->sums2.alloc((size_t)(K + 2) * B);
  ws->sums3.alloc((size_t)(K + 2) * B);
  ws->ticket.alloc(1);
  WL_CUDA(cudaMemset(ws->ticket.p, 0, sizeof(unsigned int)));
  ws->H.alloc((size_t)B * (K + 1) * K);
  WL_CUDA(cudaMemset(ws->H.p, 0, sizeof(double) * B * (K + 1) * K));
  ws->s_all.alloc((size_t)(K + 1) * B);
  ws->n0.alloc(B);
  ws->comb.alloc((size_t)(K + 1) * B);
  ws->scratch.alloc((size_t)B * 9 * kMaxSmallN * kMaxSmallN);
  ws->keff.alloc(B);
  ws->vcol.alloc(kMaxCols);
  ws->tcol.alloc(kMaxCols);
  ws->colp.alloc(4 * kMaxCols);
  ws->cg_cs.alloc(8 * kMaxCols);
  ws->kerr.alloc(kMaxCols);
  ws->cg_sc.alloc(4 * kMaxCols);
  ws->cg_bb.alloc(kMaxCols);
  ws->cg_iters.alloc(kMaxCols);
  ws->cg_flags.alloc(2);
  if (op->opts.reorth == 2) {
    ws->toar_state.alloc(toar_state_doubles(K) * B);
    ws->toar_cy.alloc((size_t)3 * B);
    ws->toar_cu.alloc((size_t)3 * (K + 3) * B);
    ws->toar_comb.alloc((size_t)(K + 2) * B);
    if (pad_cols(B) != B || (op->opts.fp32 && pad_cols_t<float>(B) != B)) {  // phantom columns stay zero
      // rows: n plus the phantom rows of either storage (<= 3); float rows take half the bytes of a double row
      const size_t dbl = (size_t)(n + 4) * std::max(pad_cols(B), (pad_cols_t<float>(B) + 1) / 2);
      ws->xg.alloc(dbl);
      WL_CUDA(cudaMemset(ws->xg.p, 0, sizeof(double) * dbl));
    }
    if (op->opts.fp32) ws->seed32.alloc((size_t)2 * (n + 1) * B);  // fp64 seeds before rounding to float
    ws->seed.alloc((size_t)3 * (n + 1) * std::max(1, std::min(max_b, kMaxCols)));
    std::vector<int> id(kMaxCols);
    std::iota(id.begin(), id.end(), 0);
    ws->vid.alloc(kMaxCols);
    WL_CUDA(cudaMemcpy(ws->vid.p, id.data(), sizeof(int) * kMaxCols, cudaMemcpyHostToDevice));
  }
  if (!ws->cg_flags_host) WL_CUDA(cudaMallocHost(&ws->cg_flags_host, (2 + kMaxCols) * sizeof(int)));
  spmv_scratch(op, ws, B);
  WL_CUDA(cudaDeviceSynchronize());
}

// Column renumbering of a row block [row_begin, row_end): owned column g -> g - row_begin, other
// columns -> n + (index of g in the sorted, deduplicated halo list).  Validates the CSR
// (in-range, no self loops, strictly increasing columns per row: simple graphs).
void halo_plan_host(int64_t n_global, int64_t row_begin, int64_t row_end, const int64_t* rp_in,
                    const int32_t* ci_in, std::vector<int32_t>& col, std::vector<int64_t>& remote) {
  const int64_t n = row_end - row_begin;
  const int64_t base = rp_in[0];
  const int64_t nnz = rp_in[n] - base;
  col.assign((size_t)nnz, 0);
  remote.clear();
  for (int64_t r = 0; r < n; ++r) {
    const int64_t grow = row_begin + r;
    if (rp_in[r + 1] < rp_in[r]) throw Error(WL_EGRAPH, "row_ptr not nondecreasing");
    for (int64_t z = rp_in[r] - base; z < rp_in[r + 1] - base; ++z) {
      const int64_t cg = ci_in[z];
      if (cg < 0 || cg >= n_global) throw Error(WL_EGRAPH, "column id out of range");
      if (cg == grow) throw Error(WL_EGRAPH, "self loop (graphs must be simple, P:76)");
      if (z > rp_in[r] - base && cg <= ci_in[z - 1]) throw Error(WL_EGRAPH, "columns not strictly increasing in a row");
      if (cg < row_begin || cg >= row_end) remote.push_back(cg);
    }
  }
  std::sort(remote.begin(), remote.end());
  remote.erase(std::unique(remote.begin(), remote.end()), remote.end());
  for (int64_t z = 0; z < nnz; ++z) {
    const int64_t cg = ci_in[z];
    if (cg >= row_begin && cg < row_end) col[z] = (int32_t)(cg - row_begin);
    else col[z] = (int32_t)(n + (std::lower_bound(remote.begin(), remote.end(), cg) - remote.begin()));
  }
}

void build_operator(wl_operator* op, const int64_t* rp_in, const int32_t* ci_in, cudaStream_t s) {
  const int64_t n = op->n_loc;
  const int64_t base = rp_in[0];
  const int64_t nnz = rp_in[n] - base;
  if (nnz < 0) throw Error(WL_EGRAPH, "row_ptr decreases");
  if (nnz >= INT32_MAX || n >= INT32_MAX) throw Error(WL_EUNSUPPORTED, "local nnz or rows >= 2^31");
  op->nnz_loc = (int32_t)nnz;
  std::vector<int32_t> rp((size_t)n + 1);
  for (int64_t i = 0; i <= n; ++i) {
    const int64_t v = rp_in[i] - base;
    if (v < 0 || v > nnz || (i > 0 && v < rp[i - 1])) throw Error(WL_EGRAPH, "row_ptr not nondecreasing");
    rp[i] = (int32_t)v;
  }
  // gather all ranks' row ranges
  std::vector<int64_t> bounds(op->nranks + 1, 0);
  if (multi(op)) {
    std::vector<std::vector<int64_t>> all;
    comm_allgather_host(op->comm, {op->row_begin, op->row_end}, all, s);
    for (int p = 0; p < op->nranks; ++p) {
      if (all[p][0] != (p == 0 ? 0 : all[p - 1][1])) throw Error(WL_EINVAL, "row ranges not contiguous by rank");
      bounds[p] = all[p][0];
      bounds[p + 1] = all[p][1];
    }
    if (bounds[op->nranks] != op->n_global) throw Error(WL_EINVAL, "row ranges do not cover n_global");
  } else {
    bounds[0] = 0;
    bounds[1] = op->n_global;
  }
  // validate columns, renumber them (local ids, then halo ids n + h) and collect the halo
  std::vector<int32_t> col((size_t)nnz);
  std::vector<int64_t> remote;
  halo_plan_host(op->n_global, op->row_begin, op->row_end, rp_in, ci_in, col, remote);
  op->n_halo = (int64_t)remote.size();
  // A_loc / A_halo split: only with peers to exchange with
  op->split = multi(op) && op->opts.halo_overlap && op->n_halo > 0;
  // Degree-sorted relabelling of the local rows: internal row r' holds user row perm[r'], rows
  // in decreasing degree (ties by id).  The hot gather set (high-degree rows, i.e. the columns
  // most nonzeros point to) becomes a dense, L2-resident prefix of every gathered block instead
  // of being scattered across random ids.  Halo ids (>= n) are unchanged; inputs are gathered and
  // outputs scattered through perm at the boundary (batch_inputs / combine).  With the split the
  // key is the LOCAL degree: the number of local nonzeros that gather the row, and the row length
  // the local SpMM's bins see.
  // Rows without nonzeros sort last (key -1 with the split, whose local degree is 0 for halo-only rows too).
  std::vector<int32_t> key((size_t)n);
  for (int64_t r = 0; r < n; ++r) {
    key[r] = rp[r + 1] - rp[r];
    if (op->split) {
      for (int32_t z = rp[r]; z < rp[r + 1]; ++z) key[r] -= col[z] >= n;
      if (rp[r + 1] == rp[r]) key[r] = -1;
    }
  }
  std::vector<int32_t> newid;
  if (op->opts.relabel) {
    std::vector<int32_t> perm((size_t)n);
    std::iota(perm.begin(), perm.end(), 0);
    std::stable_sort(perm.begin(), perm.end(), [&](int32_t x, int32_t y) { return key[x] > key[y]; });
    newid.assign((size_t)n, 0);
    for (int64_t k = 0; k < n; ++k) newid[perm[k]] = (int32_t)k;
    std::vector<int32_t> rp2((size_t)n + 1, 0), col2((size_t)nnz);
    for (int64_t k = 0; k < n; ++k) rp2[k + 1] = rp2[k] + (rp[perm[k] + 1] - rp[perm[k]]);
    for (int64_t k = 0; k < n; ++k) {
      const int32_t src = rp[perm[k]], dst = rp2[k], d = rp[perm[k] + 1] - src;
      for (int32_t t = 0; t < d; ++t) {
        const int32_t cl = col[src + t];
        col2[dst + t] = cl < n ? newid[cl] : cl;
      }
    }
    rp.swap(rp2);
    col.swap(col2);
    op->perm.alloc(std::max<int64_t>(1, n));
    if (n) WL_CUDA(cudaMemcpy(op->perm.p, perm.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice));
  }
  // isolated tail: with the relabelling the empty rows are the last ones; they are isolated when no local row
  // references them (a symmetric graph never does; checked) and no peer requests them (checked below)
  op->n_act = n;
  if (op->opts.relabel) {
    int64_t na = n;
    while (na > 0 && rp[na] == rp[na - 1]) --na;
    bool referenced = false;
    for (int64_t z = 0; z < nnz && !referenced; ++z) referenced = col[z] >= na && col[z] < n;
    if (!referenced) op->n_act = na;
  }
  if (!op->split) {
    op->A.upload(rp, col, nullptr);
  } else {
    // A_loc: every row, its local columns; A_halo: the rows with halo columns, those columns
    std::vector<int32_t> rpl((size_t)n + 1, 0), cl, rph(1, 0), ch, hrows;
    cl.reserve((size_t)nnz);
    for (int64_t r = 0; r < n; ++r) {
      int32_t nh = 0;
      for (int32_t z = rp[r]; z < rp[r + 1]; ++z) {
        if (col[z] < n) cl.push_back(col[z]);
        else { ch.push_back(col[z]); ++nh; }
      }
      rpl[r + 1] = (int32_t)cl.size();
      if (nh) {
        hrows.push_back((int32_t)r);
        rph.push_back((int32_t)ch.size());
      }
    }
    op->A.upload(rpl, cl, nullptr);
    op->Ah.upload(rph, ch, &hrows);
    op->rowptr_full.alloc(n + 1);
    WL_CUDA(cudaMemcpy(op->rowptr_full.p, rp.data(), sizeof(int32_t) * (n + 1), cudaMemcpyHostToDevice));
  }
  // halo plan: how many rows I need from each owner, then the ids (owners pack them)
  const int P = op->nranks;
  op->recv_cnt.assign(P, 0);
  op->recv_displ.assign(P, 0);
  op->send_cnt.assign(P, 0);
  op->send_displ.assign(P, 0);
  if (multi(op)) {
    // requests grouped by owner (remote is sorted and partitions are contiguous)
    std::vector<std::vector<int64_t>> need(P), give;
    for (int64_t id : remote) {
      const int owner = (int)(std::upper_bound(bounds.begin(), bounds.end(), id) - bounds.begin()) - 1;
      need[owner].push_back(id);
    }
    for (int p = 0; p < P; ++p) op->recv_cnt[p] = (int64_t)need[p].size();
    for (int p = 1; p < P; ++p) op->recv_displ[p] = op->recv_displ[p - 1] + op->recv_cnt[p - 1];
    comm_alltoallv_host(op->comm, need, give, s);
    for (int p = 0; p < P; ++p) op->send_cnt[p] = (int64_t)give[p].size();
    for (int p = 1; p < P; ++p) op->send_displ[p] = op->send_displ[p - 1] + op->send_cnt[p - 1];
    op->n_send = op->send_displ[P - 1] + op->send_cnt[P - 1];
    // owners pack the requested rows in request order; ids -> internal (relabelled) local rows
    std::vector<int32_t> idx((size_t)op->n_send);
    for (int p = 0, k = 0; p < P; ++p)
      for (int64_t g : give[p]) {
        if (g < op->row_begin || g >= op->row_end) throw Error(WL_EGRAPH, "halo request for a row not owned");
        idx[k] = (int32_t)(g - op->row_begin);
        if (!newid.empty()) idx[k] = newid[idx[k]];
        if (idx[k] >= op->n_act) op->n_act = n;  // an "isolated" row a peer references: not isolated
        ++k;
      }
    op->send_idx.alloc(std::max<int64_t>(1, op->n_send));
    if (op->n_send) WL_CUDA(cudaMemcpy(op->send_idx.p, idx.data(), sizeof(int32_t) * op->n_send, cudaMemcpyHostToDevice));
  } else if (op->n_halo) {
    throw Error(WL_EGRAPH, "column outside [row_begin,row_end) without a communicator");
  }
}


// Outer basis vectors are padded to an even length (16-byte aligned rows for the bulk-copy
// Gram kernels); the pad entries are zero and never written.
inline int64_t outer_stride(const wl_operator* op) { return std::max<int64_t>(2, op->n_loc + (op->n_loc & 1)); }

// Outer Arnoldi with CGS2 on unit-stride n-vectors (B = 1), basis ws->oQ (vector 0 preset by the
// caller), Hessenberg ws->oH (layout (m+1) x m), scales ws->os, ||P_0|| in ws->on0.
// `apply(P̃_j, out)` writes the operator applied to the UNNORMALISED basis vector P̃_j.
template <class Apply>
void outer_arnoldi(const wl_operator* op, wl_workspace* ws, int m, Apply&& apply, cudaStream_t s, int64_t len = 0) {
  // Arnoldi with DCGS2 on the bulk-copy ring passes (B = 1): q_i in order at oQ + i*n (normalised),
  // the pending once-orthogonalised p_j alternates between the two buffers after slot m.
  const int64_t n = len ? len : outer_stride(op);
  WL_CUDA(cudaMemsetAsync(ws->oH.p, 0, sizeof(double) * (m + 1) * m, s));
  VecPtrs Q{};
  for (int i = 0; i <= m; ++i) Q.p[i] = ws->oQ.p + (int64_t)i * n;
  double* P[2] = {ws->oQ.p + (int64_t)(m + 1) * n, ws->oQ.p + (int64_t)(m + 2) * n};
  WL_CUDA(cudaMemcpyAsync(P[0], ws->oQ.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));  // p_0 = x0
  Dcgs2Args d{};
  d.Q = Q;
  d.len = n;
  d.B = 1;
  d.split = n;
  d.partials = ws->partials.p;
  d.sums_out = ws->osums1.p;
  d.coef_v = ws->ocoef_v.p;
  d.coef_s = ws->ocoef_s.p;
  const double btol = op->opts.breakdown_tol;
  int cur = 0;
  for (int j = 0; j < m; ++j) {
    apply(P[cur], ws->ow.p);  // w = Op p_j
    d.nq = j;
    d.P = P[cur];
    d.wa = ws->ow.p;
    d.wb = nullptr;
    dcgs2_dots(d, s);
    allreduce(op, ws->osums1.p, (size_t)(2 * j + 3), s);
    dcgs2_coeffs(ws->osums1.p, j, 1, m, btol, 0, 1, ws->oH.p, ws->oref.p, ws->on0.p, ws->okeff.p, ws->ocoef_v.p,
                 ws->ocoef_s.p, s);
    d.Qout = const_cast<double*>(Q.p[j]);
    d.Pnext = P[cur ^ 1];
    d.accumulate = 0;
    dcgs2_update(d, s);
    cur ^= 1;
  }
  d.nq = m;  // delayed reorthogonalisation of p_m completes column m-1 of H
  d.P = P[cur];
  d.wa = nullptr;
  d.wb = nullptr;
  dcgs2_dots(d, s);
  allreduce(op, ws->osums1.p, (size_t)(2 * m + 3), s);
  dcgs2_coeffs(ws->osums1.p, m, 1, m, btol, 1, 1, ws->oH.p, ws->oref.p, ws->on0.p, ws->okeff.p, ws->ocoef_v.p,
               ws->ocoef_s.p, s);
}


void outer_alloc(const wl_operator* op, wl_workspace* ws, int m, int nt, int64_t len = 0) {
  const int64_t np = len ? len : outer_stride(op);
  if (ws->kout_alloc >= m && ws->otau.n >= (size_t)nt) return;
  ws->oQ.alloc((size_t)(m + 3) * np);  // q_0..q_m, then the two pending-vector buffers
  ws->ow.alloc((size_t)np);
  WL_CUDA(cudaMemset(ws->oQ.p, 0, sizeof(double) * (m + 3) * np));
  WL_CUDA(cudaMemset(ws->ow.p, 0, sizeof(double) * np));
  ws->oH.alloc((size_t)(m + 1) * m);
  ws->on0.alloc(1);
  ws->okeff.alloc(1);
  ws->oref.alloc(1);
  ws->osums1.alloc((size_t)2 * m + 5);
  ws->ocoef_v.alloc((size_t)2 * (m + 1));
  ws->ocoef_s.alloc(3);
  ws->otau.alloc(std::max(1, nt));
  ws->oY.alloc((size_t)std::max(1, nt) * (m + 1));
  ws->oscratch.alloc((size_t)std::max(1, nt) * 9 * kMaxSmallN * kMaxSmallN);
  ws->kout_alloc = m;
  const size_t need = (size_t)gram_grid(np, 1) * (m + 2);
  if (ws->partials.n < need) ws->partials.alloc(need);
  if (!ws->ticket.p) {
    ws->ticket.alloc(1);
    WL_CUDA(cudaMemset(ws->ticket.p, 0, sizeof(unsigned int)));
  }
}

// Largest eigenvalue of the symmetric tridiagonal (a, b) by bisection on Sturm counts.
double tridiag_max_eig(const std::vector<double>& a, const std::vector<double>& b) {
  const int m = (int)a.size();
  double lo = 1e300, hi = -1e300;
  for (int i = 0; i < m; ++i) {  // Gershgorin interval
    const double r = (i > 0 ? std::fabs(b[i - 1]) : 0.0) + (i + 1 < m ? std::fabs(b[i]) : 0.0);
    lo = std::min(lo, a[i] - r);
    hi = std::max(hi, a[i] + r);
  }
  auto count_below = [&](double x) {  // number of eigenvalues < x
    int c = 0;
    double d = 1.0;
    for (int i = 0; i < m; ++i) {
      d = a[i] - x - (i > 0 ? b[i - 1] * b[i - 1] / d : 0.0);
      if (d == 0.0) d = -1e-300;
      if (d < 0) ++c;
    }
    return c;
  };
  for (int it = 0; it < 200 && hi - lo > 1e-15 * std::max(1.0, std::fabs(hi)); ++it) {
    const double mid = 0.5 * (lo + hi);
    if (count_below(mid) >= m) hi = mid;  // all eigenvalues below mid
    else lo = mid;
  }
  return hi;
}

void check_block(const void* p, int64_t ld, int64_t cols, const char* what) {
  if (!p) throw Error(WL_EINVAL, std::string(what) + " is NULL");
  if (ld < cols) throw Error(WL_EINVAL, std::string(what) + ": leading dimension < columns");
}

}  // namespace
}  // namespace wl

using namespace wl;

extern "C" {

const char* wl_last_error(void) { return g_last_error.c_str(); }
const char* wl_version(void) { return "walklap-b200 0.1 (sm_100a)"; }
int64_t wl_launch_count(void) { return g_launches.load(); }

void wl_opts_default(wl_opts* o) {
  if (!o) return;
  o->krylov_dim = 30;
  o->reorth = 2;
  o->max_cols = 32;
  o->breakdown_tol = 1e-12;
  o->rho_bound = 0.0;
  o->relabel = 1;
  o->solver = WL_SOLVER_KRYLOV;
  o->cg_tol = 1e-9;
  o->cg_maxit = 1000;
  o->cg_check = 8;
  o->tol = 0.0;
  o->halo_overlap = 1;
  o->lanczos = 1;
  o->krylov_adaptive = 0;
  o->fp32 = 0;
}

wl_status wl_partition(int64_t n, const int64_t* row_ptr, int32_t nranks, int64_t* bounds) {
  return guarded([&] {
    if (n < 0 || !row_ptr || !bounds || nranks < 1) throw Error(WL_EINVAL, "bad partition args");
    const int64_t nnz = row_ptr[n] - row_ptr[0];
    bounds[0] = 0;
    for (int p = 1; p < nranks; ++p) {
      const int64_t target = row_ptr[0] + (p * nnz + nranks - 1) / nranks;  // ceil(p nnz / P)
      int64_t r = std::lower_bound(row_ptr, row_ptr + n + 1, target) - row_ptr;
      r = std::min(std::max(r, bounds[p - 1]), n);
      bounds[p] = r;
    }
    bounds[nranks] = n;
  });
}

wl_status wl_halo_plan(int64_t n_global, int32_t nranks, const int64_t* bounds, int32_t rank,
                       const int64_t* row_ptr_local, const int32_t* col_idx_local, int32_t* col_local_out,
                       int64_t* halo_ids_out, int64_t* n_halo_out, int64_t* recv_count_out) {
  return guarded([&] {
    if (!bounds || !row_ptr_local || nranks < 1 || rank < 0 || rank >= nranks || !n_halo_out)
      throw Error(WL_EINVAL, "bad halo plan args");
    const int64_t rb = bounds[rank], re = bounds[rank + 1];
    if (rb < 0 || re < rb || re > n_global) throw Error(WL_EINVAL, "bad bounds");
    const int64_t nnz = row_ptr_local[re - rb] - row_ptr_local[0];
    if (nnz > 0 && (!col_idx_local || !col_local_out || !halo_ids_out)) throw Error(WL_EINVAL, "NULL arrays");
    std::vector<int32_t> col;
    std::vector<int64_t> remote;
    halo_plan_host(n_global, rb, re, row_ptr_local, col_idx_local, col, remote);
    if (nnz > 0) std::memcpy(col_local_out, col.data(), sizeof(int32_t) * col.size());
    if (!remote.empty()) std::memcpy(halo_ids_out, remote.data(), sizeof(int64_t) * remote.size());
    *n_halo_out = (int64_t)remote.size();
    if (recv_count_out) {
      for (int p = 0; p < nranks; ++p) recv_count_out[p] = 0;
      for (int64_t id : remote) {
        const int owner = (int)(std::upper_bound(bounds, bounds + nranks + 1, id) - bounds) - 1;
        recv_count_out[owner]++;
      }
    }
  });
}

wl_status wl_operator_create(wl_comm* comm, int64_t n_global, int64_t row_begin, int64_t row_end,
                             const int64_t* row_ptr_local, const int32_t* col_idx_local, int32_t variant,
                             int32_t n_theta, const double* thetas, const wl_walkfun* f,
                             const wl_opts* opts, wl_stream stream, wl_operator** out) {
  return guarded([&] {
    if (!out || !row_ptr_local || !f) throw Error(WL_EINVAL, "NULL argument");
    if (n_global < 1 || row_begin < 0 || row_end < row_begin || row_end > n_global)
      throw Error(WL_EINVAL, "bad row range");
    if (row_ptr_local[row_end - row_begin] > row_ptr_local[0] && !col_idx_local)
      throw Error(WL_EINVAL, "col_idx is NULL");
    auto op = std::make_unique<wl_operator>();
    op->comm = comm;
    if (comm) {
      op->nranks = comm->nranks;
      op->rank = comm->rank;
      op->device = comm->device;
    } else {
      WL_CUDA(cudaGetDevice(&op->device));
      if (row_begin != 0 || row_end != n_global) throw Error(WL_EINVAL, "single GPU operator must own all rows");
    }
    DeviceGuard dg(op->device);
    op->n_global = n_global;
    op->row_begin = row_begin;
    op->row_end = row_end;
    if (row_end - row_begin >= INT32_MAX) throw Error(WL_EUNSUPPORTED, "local rows >= 2^31");
    op->n_loc = (int32_t)(row_end - row_begin);
    if (opts) op->opts = *opts;
    else wl_opts_default(&op->opts);
    if (op->opts.krylov_dim < 1 || op->opts.krylov_dim > kMaxKrylov) throw Error(WL_EINVAL, "krylov_dim must be in [1, 64]");
    if (op->opts.max_cols < 1 || op->opts.max_cols > kMaxCols) throw Error(WL_EINVAL, "max_cols must be in [1, 32]");
    if (!(op->opts.breakdown_tol >= 0.0)) throw Error(WL_EINVAL, "breakdown_tol < 0");
    if (op->opts.solver != WL_SOLVER_KRYLOV && op->opts.solver != WL_SOLVER_CG) throw Error(WL_EINVAL, "unknown solver");
    if (op->opts.reorth < 0 || op->opts.reorth > 2) throw Error(WL_EINVAL, "reorth must be 0, 1 or 2");
    if (!(op->opts.tol >= 0.0)) throw Error(WL_EINVAL, "tol must be >= 0");
    if (op->opts.fp32 && (op->opts.reorth != 2 || op->opts.solver != WL_SOLVER_KRYLOV))
      throw Error(WL_EINVAL, "fp32 needs reorth = 2 (TOAR) and the Krylov solver");
    op->kstat.alloc(4);
    WL_CUDA(cudaMemset(op->kstat.p, 0, 4 * sizeof(int)));
    if (op->opts.solver == WL_SOLVER_CG) {
      if (f->kind != WL_F_RESOLVENT || !(f->param > 0.0))
        throw Error(WL_EINVAL, "WL_SOLVER_CG needs the resolvent with α > 0");
      if (!(op->opts.cg_tol > 0.0) || op->opts.cg_maxit < 1 || op->opts.cg_check < 1)
        throw Error(WL_EINVAL, "cg_tol > 0, cg_maxit >= 1, cg_check >= 1 required");
    }
    // θ values (θ = 1 - μ)
    if (variant == WL_WALK || variant == WL_NBT) {
      if (n_theta != 1) throw Error(WL_EINVAL, "WL_WALK/WL_NBT take exactly one θ");
      op->theta = {variant == WL_WALK ? 1.0 : 0.0};
    } else if (variant == WL_BTDW) {
      if (n_theta < 1 || n_theta > kMaxCols || !thetas) throw Error(WL_EINVAL, "n_theta must be in [1, 32]");
      for (int i = 0; i < n_theta; ++i) {
        if (!(thetas[i] >= 0.0 && thetas[i] <= 1.0)) throw Error(WL_EINVAL, "θ must be in [0, 1]");
        op->theta.push_back(thetas[i]);
      }
    } else {
      throw Error(WL_EINVAL, "unknown variant");
    }
    op->n_theta = (int)op->theta.size();
    for (double t : op->theta) op->mu.push_back(1.0 - t);
    // walk weights
    op->fkind = f->kind;
    op->fparam = f->param;
    op->lscale = f->scale != 0.0 ? f->scale : 1.0;
    if (f->kind == WL_F_EXP) {
      op->c0 = 1.0;
    } else if (f->kind == WL_F_RESOLVENT) {
      op->c0 = 1.0;
      if (op->opts.rho_bound > 0.0 && std::fabs(f->param) * op->opts.rho_bound >= 1.0)
        throw Error(WL_EDIVERGE, "resolvent: α ρ >= 1, series diverges (Prop. pro:whe-we-converge)");
    } else if (f->kind == WL_F_SERIES) {
      if (!f->coeffs || f->ncoeffs < 1 || f->ncoeffs > 64) throw Error(WL_EINVAL, "series needs 1..64 coefficients");
      op->coeffs.assign(f->coeffs, f->coeffs + f->ncoeffs);
      op->c0 = op->coeffs[0];
    } else {
      throw Error(WL_EINVAL, "unknown walk-function kind");
    }
    cudaStream_t s = S_(stream);
    op->mu_dev.alloc(op->n_theta);
    WL_CUDA(cudaMemcpy(op->mu_dev.p, op->mu.data(), sizeof(double) * op->n_theta, cudaMemcpyHostToDevice));
    if (!op->coeffs.empty()) {
      op->coeffs_dev.alloc(op->coeffs.size());
      WL_CUDA(cudaMemcpy(op->coeffs_dev.p, op->coeffs.data(), sizeof(double) * op->coeffs.size(),
                         cudaMemcpyHostToDevice));
    }
    build_operator(op.get(), row_ptr_local, col_idx_local, s);
    // a8: t' = φ_θ 1 - c_0 1 for every θ (one batched Krylov action on V = 1)
    op->tprime.alloc((size_t)std::max<int64_t>(1, op->n_loc) * op->n_theta);
    {
      wl_workspace ws;
      workspace_alloc(&ws, op.get(), 1);
      run_action(op.get(), &ws, 2, nullptr, 1, 1, op->tprime.p, op->n_theta, s);
      WL_CUDA(cudaStreamSynchronize(s));
      WL_CUDA(cudaMemset(op->kstat.p, 0, 4 * sizeof(int)));  // opts.tol reports on actions, not on t
    }
    *out = op.release();
  });
}

void wl_operator_destroy(wl_operator* op) {
  if (!op) return;
  DeviceGuard dg(op->device);
  WL_CUDA(cudaDeviceSynchronize());
  delete op->est_ws[0];
  delete op->est_ws[1];
  delete op;
}

wl_status wl_workspace_stats(const wl_workspace* ws, int64_t* cg_iterations, int64_t* krylov_steps,
                             int64_t* krylov_batches) {
  return guarded([&] {
    if (!ws) throw Error(WL_EINVAL, "ws is NULL");
    if (cg_iterations) *cg_iterations = ws->cg_iterations;
    if (krylov_steps) *krylov_steps = ws->krylov_steps;
    if (krylov_batches) *krylov_batches = ws->krylov_batches;
  });
}

wl_status wl_operator_info(const wl_operator* op, int64_t* n_local, int64_t* nnz_local, int64_t* n_halo,
                           int32_t* n_theta) {
  return guarded([&] {
    if (!op) throw Error(WL_EINVAL, "op is NULL");
    if (n_local) *n_local = op->n_loc;
    if (nnz_local) *nnz_local = op->nnz_loc;
    if (n_halo) *n_halo = op->n_halo;
    if (n_theta) *n_theta = op->n_theta;
  });
}

wl_status wl_operator_active_rows(const wl_operator* op, int64_t* n_active) {
  return guarded([&] {
    if (!op || !n_active) throw Error(WL_EINVAL, "NULL argument");
    *n_active = op->n_act;
  });
}

wl_status wl_operator_diag_shift(const wl_operator* op, double* t_dev, int64_t ldt, wl_stream stream) {
  return guarded([&] {
    if (!op) throw Error(WL_EINVAL, "op is NULL");
    check_block(t_dev, ldt, op->n_theta, "t_dev");
    DeviceGuard dg(op->device);
    // t = t' + c_0
    const int nt = op->n_theta;
    std::vector<double> host((size_t)op->n_loc * nt);
    WL_CUDA(cudaMemcpyAsync(host.data(), op->tprime.p, sizeof(double) * host.size(), cudaMemcpyDeviceToHost, S_(stream)));
    WL_CUDA(cudaStreamSynchronize(S_(stream)));
    for (auto& v : host) v += op->c0;
    if (op->perm.p) {  // internal -> user row order
      std::vector<int32_t> perm((size_t)op->n_loc);
      WL_CUDA(cudaMemcpy(perm.data(), op->perm.p, sizeof(int32_t) * op->n_loc, cudaMemcpyDeviceToHost));
      std::vector<double> u(host.size());
      for (int64_t r = 0; r < op->n_loc; ++r)
        for (int i = 0; i < nt; ++i) u[(size_t)perm[r] * nt + i] = host[(size_t)r * nt + i];
      host.swap(u);
    }
    WL_CUDA(cudaMemcpy2DAsync(t_dev, sizeof(double) * ldt, host.data(), sizeof(double) * nt, sizeof(double) * nt,
                              op->n_loc, cudaMemcpyHostToDevice, S_(stream)));
    WL_CUDA(cudaStreamSynchronize(S_(stream)));
  });
}

wl_status wl_workspace_create(const wl_operator* op, int32_t max_b, wl_workspace** out) {
  return guarded([&] {
    if (!op || !out || max_b < 1) throw Error(WL_EINVAL, "bad workspace args");
    DeviceGuard dg(op->device);
    auto ws = std::make_unique<wl_workspace>();
    workspace_alloc(ws.get(), op, max_b);
    *out = ws.release();
  });
}

void wl_workspace_destroy(wl_workspace* ws) {
  if (!ws) return;
  DeviceGuard dg(ws->op->device);
  cudaDeviceSynchronize();
  delete ws;
}

static wl_status apply_common(int mode, const wl_operator* op, int32_t b, const double* V, int64_t ldv, double* LV,
                              int64_t ldlv, wl_workspace* ws, wl_stream stream) {
  return guarded([&] {
    if (!op || !ws || ws->op != op) throw Error(WL_EINVAL, "operator/workspace mismatch");
    if (b < 1 || b > ws->max_b) throw Error(WL_EINVAL, "b out of [1, max_b]");
    if (op->n_loc > 0) {
      check_block(V, ldv, b, "V");
      check_block(LV, ldlv, (int64_t)op->n_theta * b, "LV");
    }
    DeviceGuard dg(op->device);
    run_action(op, ws, mode, V, ldv, b, LV, ldlv, S_(stream));
  });
}

wl_status wl_apply(const wl_operator* op, int32_t b, const double* V, int64_t ldv, double* LV, int64_t ldlv,
                   wl_workspace* ws, wl_stream stream) {
  return apply_common(1, op, b, V, ldv, LV, ldlv, ws, stream);
}

wl_status wl_phi_apply(const wl_operator* op, int32_t b, const double* V, int64_t ldv, double* LV, int64_t ldlv,
                       wl_workspace* ws, wl_stream stream) {
  return apply_common(0, op, b, V, ldv, LV, ldlv, ws, stream);
}

wl_status wl_apply_host(const wl_operator* op, int32_t b, const double* Vh, int64_t ldv, double* LVh,
                        int64_t ldlv, wl_workspace* ws, wl_stream stream) {
  return guarded([&] {
    if (!op || !ws || ws->op != op) throw Error(WL_EINVAL, "operator/workspace mismatch");
    if (b < 1 || b > ws->max_b) throw Error(WL_EINVAL, "b out of [1, max_b]");
    const int64_t n = op->n_loc;
    const int64_t G = (int64_t)op->n_theta * b;
    check_block(Vh, ldv, b, "V_host");
    check_block(LVh, ldlv, G, "LV_host");
    DeviceGuard dg(op->device);
    cudaStream_t s = S_(stream);
    ws->hV.alloc((size_t)std::max<int64_t>(1, n * b));
    ws->hLV.alloc((size_t)std::max<int64_t>(1, n * G));
    // contiguous blocks go as one linear copy (a pitched copy of 1e7 short rows runs at a fraction of the link)
    if (ldv == b) WL_CUDA(cudaMemcpyAsync(ws->hV.p, Vh, sizeof(double) * n * b, cudaMemcpyHostToDevice, s));
    else WL_CUDA(cudaMemcpy2DAsync(ws->hV.p, sizeof(double) * b, Vh, sizeof(double) * ldv, sizeof(double) * b, n,
                                   cudaMemcpyHostToDevice, s));
    run_action(op, ws, 1, ws->hV.p, b, b, ws->hLV.p, G, s);
    if (ldlv == G) WL_CUDA(cudaMemcpyAsync(LVh, ws->hLV.p, sizeof(double) * n * G, cudaMemcpyDeviceToHost, s));
    else WL_CUDA(cudaMemcpy2DAsync(LVh, sizeof(double) * ldlv, ws->hLV.p, sizeof(double) * G, sizeof(double) * G, n,
                                   cudaMemcpyDeviceToHost, s));
    WL_CUDA(cudaStreamSynchronize(s));
  });
}

wl_status wl_diffuse(const wl_operator* op, int32_t theta_index, int32_t nt, const double* tau, const double* x0,
                     double* X, int64_t ldx, int32_t k_out, wl_workspace* ws, wl_stream stream) {
  return guarded([&] {
    if (!op || !ws || ws->op != op) throw Error(WL_EINVAL, "operator/workspace mismatch");
    if (theta_index < 0 || theta_index >= op->n_theta) throw Error(WL_EINVAL, "theta_index out of range");
    if (nt < 1 || !tau) throw Error(WL_EINVAL, "need nt >= 1 times");
    if (k_out < 2 || k_out > 128) throw Error(WL_EINVAL, "k_out must be in [2, 128]");
    for (int i = 0; i < nt; ++i)
      if (!(tau[i] >= 0.0)) throw Error(WL_EINVAL, "times must be >= 0");
    if (op->n_loc > 0) {
      check_block(x0, 1, 1, "x0");
      check_block(X, ldx, nt, "X");
    }
    DeviceGuard dg(op->device);
    cudaStream_t s = S_(stream);
    const int64_t n = op->n_loc;
    const int m = k_out;
    outer_alloc(op, ws, m, nt);
    WL_CUDA(cudaMemcpyAsync(ws->otau.p, tau, sizeof(double) * nt, cudaMemcpyHostToDevice, s));
    if (op->perm.p) pack_rows(x0, 1, op->perm.p, n, 1, ws->oQ.p, s);  // user -> internal order
    else WL_CUDA(cudaMemcpyAsync(ws->oQ.p, x0, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    // outer Arnoldi (= Lanczos with full reorthogonalisation: 𝕃 symmetric, Prop. pro:still-again-an-mmatrix)
    outer_arnoldi(op, ws, m, [&](const double* Pj, double* out) {
      run_chunk(op, ws, 1, Pj, 1, 1, theta_index, 1, out, 1, s, false);  // inner action 𝕃 P̃_j
    }, s);
    SmallFArgs f{};
    f.H = ws->oH.p;
    f.K = m;
    f.keff = ws->okeff.p;
    f.kind = 3;
    f.n0 = ws->on0.p;
    f.s = nullptr;  // q_i stored normalised
    f.comb = ws->oY.p;
    f.scratch = ws->oscratch.p;
    f.B = 1;
    f.tau = ws->otau.p;
    f.nprob = nt;
    small_f(f, s);
    // m + 1 = the row stride of Y (small_f kind 3); slot m is never written (zero) and its weight is 0
    lanczos_combine(ws->oQ.p, outer_stride(op), m + 1, n, ws->oY.p, nt, 1.0, X, ldx, op->perm.p, s);
  });
}

wl_status wl_spectral_radius(const wl_operator* op, int32_t k, double* rho_out, wl_stream stream) {
  return guarded([&] {
    if (!op || !rho_out) throw Error(WL_EINVAL, "NULL argument");
    if (k < 2 || k > 128) throw Error(WL_EINVAL, "k must be in [2, 128]");
    DeviceGuard dg(op->device);
    cudaStream_t s = S_(stream);
    if (!op->est_ws[0]) op->est_ws[0] = new wl_workspace;
    wl_workspace& ws = *op->est_ws[0];
    ws.op = op;
    outer_alloc(op, &ws, k, 1);
    spmv_scratch(op, &ws, 1);
    fill(ws.oQ.p, op->n_loc, 1.0, s);
    outer_arnoldi(op, &ws, k, [&](const double* Pj, double* out) {
      do_spmv(op, &ws, Pj, 1, nullptr, nullptr, nullptr, nullptr, out, 1, s);  // A P̃_j
    }, s);
    std::vector<double> H((size_t)(k + 1) * k);
    int keff = 0;
    WL_CUDA(cudaMemcpyAsync(H.data(), ws.oH.p, sizeof(double) * H.size(), cudaMemcpyDeviceToHost, s));
    WL_CUDA(cudaMemcpyAsync(&keff, ws.okeff.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    WL_CUDA(cudaStreamSynchronize(s));
    if (keff <= 0) { *rho_out = 0.0; return; }
    std::vector<double> a(keff), b(std::max(0, keff - 1));
    for (int i = 0; i < keff; ++i) a[i] = H[(size_t)i * (k + 1) + i];
    for (int i = 0; i + 1 < keff; ++i) b[i] = H[(size_t)i * (k + 1) + i + 1];
    *rho_out = tridiag_max_eig(a, b);
  });
}

wl_status wl_spectral_radius_z(const wl_operator* op, int32_t theta_index, int32_t k, double* rho_out,
                               wl_stream stream) {
  return guarded([&] {
    if (!op || !rho_out) throw Error(WL_EINVAL, "NULL argument");
    if (k < 2 || k > 128) throw Error(WL_EINVAL, "k must be in [2, 128]");
    if (theta_index < 0 || theta_index >= op->n_theta) throw Error(WL_EINVAL, "theta_index out of range");
    DeviceGuard dg(op->device);
    cudaStream_t s = S_(stream);
    if (!op->est_ws[1]) op->est_ws[1] = new wl_workspace;
    wl_workspace& ws = *op->est_ws[1];
    ws.op = op;
    const int64_t np = outer_stride(op), len = 2 * np;  // Z vector = [top np ; bottom np], pad rows stay 0
    outer_alloc(op, &ws, k, 1, len);
    spmv_scratch(op, &ws, 1);
    ws.colp.alloc(4 * kMaxCols);
    ws.vcol.alloc(kMaxCols);
    ws.tcol.alloc(kMaxCols);
    double* g0z = ws.colp.p;
    double* g1z = g0z + kMaxCols;
    setup_chunk(op->mu_dev.p, theta_index, 1, 1, g0z, g1z, g0z + 2 * kMaxCols, g0z + 3 * kMaxCols, ws.vcol.p,
                ws.tcol.p, s);
    // positive pseudo-random start vector (structured ones can be eigenvectors: Z_1 [1; 1] = [1; 1])
    fill_hash(ws.oQ.p, op->n_loc, 0x5EEDull, 2 * op->row_begin, s);
    fill_hash(ws.oQ.p + np, op->n_loc, 0x5EEDull, 2 * op->row_begin + op->n_loc, s);
    outer_arnoldi(op, &ws, k, [&](const double* Pj, double* out) {
      // Z (x; y) = (y; A y + μ(μ - d) x)   (eq:Zdef)
      WL_CUDA(cudaMemcpyAsync(out, Pj + np, sizeof(double) * np, cudaMemcpyDeviceToDevice, s));
      do_spmv(op, &ws, Pj + np, 1, Pj, g0z, g1z, nullptr, out + np, 1, s);
    }, s, len);
    std::vector<double> H((size_t)(k + 1) * k);
    int keff = 0;
    WL_CUDA(cudaMemcpyAsync(H.data(), ws.oH.p, sizeof(double) * H.size(), cudaMemcpyDeviceToHost, s));
    WL_CUDA(cudaMemcpyAsync(&keff, ws.okeff.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    WL_CUDA(cudaStreamSynchronize(s));
    if (keff <= 0) { *rho_out = 0.0; return; }
    std::vector<double> Hm((size_t)keff * keff, 0.0), wr, wi;
    for (int j = 0; j < keff; ++j)
      for (int i = 0; i <= std::min(j + 1, keff - 1); ++i) Hm[(size_t)i * keff + j] = H[(size_t)j * (k + 1) + i];
    if (!hessenberg_eigvals(Hm, keff, wr, wi)) throw Error(WL_ENOCONV, "Hessenberg QR did not converge");
    double r = 0.0;
    for (int i = 0; i < keff; ++i) r = std::max(r, std::hypot(wr[i], wi[i]));
    *rho_out = r;
  });
}

wl_status wl_markov(const wl_operator* op, int32_t theta_index, int32_t nsteps, const double* p0, double* P,
                    int64_t ldp, wl_workspace* ws, wl_stream stream) {
  return guarded([&] {
    if (!op || !ws || ws->op != op) throw Error(WL_EINVAL, "operator/workspace mismatch");
    if (theta_index < 0 || theta_index >= op->n_theta) throw Error(WL_EINVAL, "theta_index out of range");
    if (nsteps < 1) throw Error(WL_EINVAL, "nsteps must be >= 1");
    if (op->n_loc > 0) {
      check_block(p0, 1, 1, "p0");
      check_block(P, ldp, nsteps, "P");
    }
    DeviceGuard dg(op->device);
    cudaStream_t s = S_(stream);
    const int64_t n = op->n_loc;
    ws->mk_p.alloc((size_t)std::max<int64_t>(1, n));
    ws->mk_v.alloc((size_t)std::max<int64_t>(1, n));
    gather_col(p0, 1, op->perm.p, n, ws->mk_p.p, s);  // user -> internal order
    for (int k = 0; k < nsteps; ++k) {
      // p_{k+1}^T = P^T p_k^T = φ (p_k / t)   (P = diag(t)^{-1} φ, φ symmetric)
      markov_scale(ws->mk_p.p, op->tprime.p, op->n_theta, theta_index, op->c0, n, ws->mk_v.p, s);
      run_chunk(op, ws, 0, ws->mk_v.p, 1, 1, theta_index, 1, ws->mk_p.p, 1, s, false);
      scatter_col(ws->mk_p.p, op->perm.p, n, P + k, ldp, s);
    }
  });
}

wl_status wl_hessenberg_eigvals(int32_t n, const double* H, double* wr, double* wi) {
  return guarded([&] {
    if (n < 1 || !H || !wr || !wi) throw Error(WL_EINVAL, "bad arguments");
    std::vector<double> a(H, H + (size_t)n * n), r, i;
    if (!hessenberg_eigvals(a, n, r, i)) throw Error(WL_ENOCONV, "Hessenberg QR did not converge");
    std::copy(r.begin(), r.end(), wr);
    std::copy(i.begin(), i.end(), wi);
  });
}

namespace wl {
namespace {
// Column-major views of the row-major n x cols blocks the engine uses (block.cu): gram: C (p x q, col-major,
// ld p) = X[:, :p]ᵀ Y[:, :q];  axpy_block: Y[:, :q] = beta Y + alpha X[:, :p] C, C p x q col-major (ld p).
void gram(wl_workspace* ws, int p, int q, int64_t n, const double* X, int64_t ldx, const double* Y, int64_t ldy,
          double* C, cudaStream_t s) {
  ws->trPart.alloc(block_gram_partials(n, p));
  block_gram(p, q, n, X, ldx, Y, ldy, C, ws->trPart.p, s);
}
void axpy_block(int p, int q, int64_t n, double alpha, const double* X, int64_t ldx, const double* C, double beta,
                double* Y, int64_t ldy, cudaStream_t s) {
  block_axpy(p, q, n, alpha, X, ldx, C, beta, Y, ldy, s);
}

// dst (ld lddst) R = src (n x m, ld m) by Cholesky QR applied twice (Gram by block.cu + allreduce, the
// m x m Cholesky and triangular inverse on the host); R (m x m upper, col-major) returned.  W2 is
// n x m scratch.  Throws WL_ENOCONV when the block is numerically rank deficient.
void chol_qr2(const wl_operator* op, wl_workspace* ws, const double* src, int m, int64_t n, double* W2, double* Rd,
              double* dst, int64_t lddst, std::vector<double>& R, cudaStream_t s) {
  std::vector<double> Rt((size_t)m * m, 0.0), G((size_t)m * m);
  for (int i = 0; i < m; ++i) Rt[(size_t)i * m + i] = 1.0;
  for (int pass = 0; pass < 2; ++pass) {
    const double* in = pass == 0 ? src : W2;
    gram(ws, m, m, n, in, m, in, m, Rd, s);
    allreduce(op, Rd, (size_t)m * m, s);
    WL_CUDA(cudaMemcpyAsync(G.data(), Rd, sizeof(double) * m * m, cudaMemcpyDeviceToHost, s));
    WL_CUDA(cudaStreamSynchronize(s));
    std::vector<double> U((size_t)m * m, 0.0), Ui((size_t)m * m, 0.0);  // G = Uᵀ U, col-major
    for (int j = 0; j < m; ++j)
      for (int i = 0; i <= j; ++i) {
        double v = G[(size_t)j * m + i];
        for (int q = 0; q < i; ++q) v -= U[(size_t)i * m + q] * U[(size_t)j * m + q];
        if (i == j) {
          if (!(v > 1e-28 * std::max(1.0, G[0]))) throw Error(WL_ENOCONV, "block rational Krylov space exhausted (rank-deficient block)");
          U[(size_t)j * m + j] = std::sqrt(v);
        } else {
          U[(size_t)j * m + i] = v / U[(size_t)i * m + i];
        }
      }
    for (int j = 0; j < m; ++j) {
      Ui[(size_t)j * m + j] = 1.0 / U[(size_t)j * m + j];
      for (int i = j - 1; i >= 0; --i) {
        double v = 0.0;
        for (int q = i + 1; q <= j; ++q) v += U[(size_t)q * m + i] * Ui[(size_t)j * m + q];
        Ui[(size_t)j * m + i] = -v / U[(size_t)i * m + i];
      }
    }
    WL_CUDA(cudaMemcpyAsync(Rd, Ui.data(), sizeof(double) * m * m, cudaMemcpyHostToDevice, s));
    axpy_block(m, m, n, 1.0, in, m, Rd, 0.0, pass == 0 ? W2 : dst, pass == 0 ? m : lddst, s);
    std::vector<double> T((size_t)m * m, 0.0);  // Rt <- U Rt
    for (int c = 0; c < m; ++c)
      for (int r = 0; r < m; ++r) {
        double v = 0.0;
        for (int q = r; q < m; ++q) v += U[(size_t)q * m + r] * Rt[(size_t)c * m + q];
        T[(size_t)c * m + r] = v;
      }
    Rt.swap(T);
    WL_CUDA(cudaStreamSynchronize(s));  // the host Ui buffer is reused by the next pass
  }
  R = Rt;
}

// X (n x B, ld B, internal order) = (𝔏 − ξI)⁻¹ U by MINRES (minres.cu), 𝔏 = 𝕃_θ (wl_apply's operator,
// one batched action per iteration on the real and the imaginary half).  Complex ξ: X holds
// [Re x | Im x] as two n x B blocks.  Returns the largest iteration count over the columns.
int shifted_solve(const wl_operator* op, wl_workspace* ws, int theta_index, const double* U, int B, double xre,
                  double xim, double tol, int maxit, double* X, cudaStream_t s) {
  WL_NVTX("minres_shifted_solve");
  const int64_t n = op->n_loc;
  const int64_t nb = std::max<int64_t>(1, n) * B;
  const bool cplx = xim != 0.0;
  ws->mrV.alloc((size_t)12 * nb);
  ws->mr_sc.alloc(minres_scalar_doubles(kMaxCols));
  ws->mr_sums.alloc(kMaxCols);
  ws->mr_nact.alloc(1);
  if (!ws->mr_nact_host) WL_CUDA(cudaMallocHost(&ws->mr_nact_host, sizeof(int)));
  const size_t need = (size_t)minres_grid(n, B) * B;
  if (ws->partials.n < need) ws->partials.alloc(need);
  MinresArgs a{};
  a.n = n;
  a.B = B;
  a.cplx = cplx;
  a.shift_re = xre;
  a.shift_im = xim;
  a.tol = tol;
  a.u = U;
  a.v = ws->mrV.p;
  a.vp = a.v + 2 * nb;
  a.w1 = a.vp + 2 * nb;
  a.w2 = a.w1 + 2 * nb;
  a.p = a.w2 + 2 * nb;
  a.x = X;
  a.partials = ws->partials.p;
  a.sums = ws->mr_sums.p;
  a.sc = ws->mr_sc.p;
  a.nactive = ws->mr_nact.p;
  a.presummed = multi(op) ? 1 : 0;
  auto reduce = [&](int which) {
    if (multi(op)) {
      reduce_partials(a.partials, B, minres_grid(n, B), a.sums, s);
      allreduce(op, a.sums, (size_t)B, s);
    }
    minres_scalar(which, a, s);
  };
  minres_vec(0, a, s);
  reduce(0);
  minres_vec(1, a, s);
  const int check = 4;
  for (int it = 0; it < maxit; ++it) {
    // p = 𝔏 v on both halves: the whole Laplacian action per half (internal row order)
    run_chunk(op, ws, 1, a.v, B, B, theta_index * B, B, a.p, B, s, false);
    if (cplx) run_chunk(op, ws, 1, a.v + nb, B, B, theta_index * B, B, a.p + nb, B, s, false);
    minres_vec(2, a, s);
    reduce(1);
    minres_vec(3, a, s);
    reduce(2);
    minres_vec(4, a, s);
    std::swap(a.v, a.vp);   // v_{j+1} was written over v̂ in the v_prev buffer
    std::swap(a.w1, a.w2);  // w_j was written over w_{j-2}
    if ((it + 1) % check == 0 || it + 1 == maxit) {
      WL_CUDA(cudaMemcpyAsync(ws->mr_nact_host, a.nactive, sizeof(int), cudaMemcpyDeviceToHost, s));
      WL_CUDA(cudaStreamSynchronize(s));
      if (*ws->mr_nact_host == 0) break;
    }
  }
  std::vector<double> sc(minres_scalar_doubles(B));
  WL_CUDA(cudaMemcpyAsync(sc.data(), a.sc, sizeof(double) * sc.size(), cudaMemcpyDeviceToHost, s));
  WL_CUDA(cudaStreamSynchronize(s));
  int iters = 0;
  bool conv = true;
  const int kS = (int)(minres_scalar_doubles(1));
  for (int c = 0; c < B; ++c) {
    iters = std::max(iters, (int)sc[(size_t)c * kS + 15]);
    conv &= sc[(size_t)c * kS + 9] == 0.0;
  }
  if (!conv) throw Error(WL_ENOCONV, "MINRES: shifted solve above inner_tol after inner_maxit iterations");
  return iters;
}

}  // namespace
}  // namespace wl

// Block Arnoldi with poles at ∞ (reading R16) on 𝔏 = 𝕃_{θ_i}, then XNysTrace in the projected space.
wl_status wl_xnystrace_exp(const wl_operator* op, int32_t theta_index, int32_t M, const double* Omega,
                           int64_t ldo, int32_t k, int32_t nt, const double* times, double* p_out, double* e_out,
                           wl_workspace* ws, wl_stream stream) {
  return guarded([&] {
    if (!op || !ws || ws->op != op) throw Error(WL_EINVAL, "operator/workspace mismatch");
    if (theta_index < 0 || theta_index >= op->n_theta) throw Error(WL_EINVAL, "theta_index out of range");
    if (M < 1 || M > ws->Bmax) throw Error(WL_EINVAL, "M must be in [1, workspace column batch]");
    if (k < 1 || (int64_t)k * M > std::min<int64_t>(1024, op->n_global))
      throw Error(WL_EINVAL, "need 1 <= k and k*M <= min(1024, n)");
    if (nt < 1 || !times || !p_out || !e_out) throw Error(WL_EINVAL, "bad output arguments");
    for (int i = 0; i < nt; ++i)
      if (!(times[i] >= 0.0)) throw Error(WL_EINVAL, "times must be >= 0");
    if (op->n_loc > 0) check_block(Omega, ldo, M, "Omega");
    DeviceGuard dg(op->device);
    cudaStream_t s = S_(stream);
    const int64_t n = op->n_loc;
    const int P = (k + 1) * M, d = k * M;
    // buffers live in the workspace (grown on demand, reused across calls)
    DArr<double>&V = ws->trV, &Wb = ws->trW, &W2 = ws->trW2, &Cd = ws->trC, &Rd = ws->trR;
    V.alloc(std::max<int64_t>(1, n) * P);
    Wb.alloc(std::max<int64_t>(1, n) * M);
    W2.alloc(std::max<int64_t>(1, n) * M);
    Cd.alloc((size_t)P * M);
    Rd.alloc((size_t)M * M);
    std::vector<double> H((size_t)d * d, 0.0), R0((size_t)M * M), Ch((size_t)P * M), G((size_t)M * M);
    // Ω in internal row order
    if (n > 0) {
      if (op->perm.p) pack_rows(Omega, ldo, op->perm.p, n, M, Wb.p, s);
      else WL_CUDA(cudaMemcpy2DAsync(Wb.p, sizeof(double) * M, Omega, sizeof(double) * ldo, sizeof(double) * M, n,
                                     cudaMemcpyDeviceToDevice, s));
    }
    // dst (ld P) R = Wb (ld M) by Cholesky QR applied twice; R (M x M upper, col-major) returned
    auto cholqr = [&](double* dst, std::vector<double>& R) {
      std::vector<double> Rt((size_t)M * M, 0.0);
      for (int i = 0; i < M; ++i) Rt[(size_t)i * M + i] = 1.0;
      for (int pass = 0; pass < 2; ++pass) {
        const double* src = pass == 0 ? Wb.p : W2.p;
        gram(ws, M, M, n, src, M, src, M, Rd.p, s);
        allreduce(op, Rd.p, (size_t)M * M, s);
        WL_CUDA(cudaMemcpyAsync(G.data(), Rd.p, sizeof(double) * M * M, cudaMemcpyDeviceToHost, s));
        WL_CUDA(cudaStreamSynchronize(s));
        // G = Uᵀ U (U upper, col-major): Cholesky
        std::vector<double> U((size_t)M * M, 0.0), Ui((size_t)M * M, 0.0);
        for (int j = 0; j < M; ++j) {
          for (int i = 0; i <= j; ++i) {
            double v = G[(size_t)j * M + i];
            for (int q = 0; q < i; ++q) v -= U[(size_t)i * M + q] * U[(size_t)j * M + q];
            if (i == j) {
              if (!(v > 1e-28 * std::max(1.0, G[0]))) throw Error(WL_ENOCONV, "block Krylov space exhausted (k*M too large for this graph)");
              U[(size_t)j * M + j] = std::sqrt(v);
            } else {
              U[(size_t)j * M + i] = v / U[(size_t)i * M + i];
            }
          }
        }
        // U⁻¹ (upper) by back substitution, column by column
        for (int j = 0; j < M; ++j) {
          Ui[(size_t)j * M + j] = 1.0 / U[(size_t)j * M + j];
          for (int i = j - 1; i >= 0; --i) {
            double v = 0.0;
            for (int q = i + 1; q <= j; ++q) v += U[(size_t)q * M + i] * Ui[(size_t)j * M + q];
            Ui[(size_t)j * M + i] = -v / U[(size_t)i * M + i];
          }
        }
        WL_CUDA(cudaMemcpyAsync(Rd.p, Ui.data(), sizeof(double) * M * M, cudaMemcpyHostToDevice, s));
        // out = src U⁻¹  (Uinv is M x M col-major: exactly the "C" operand of axpy_block)
        double* out = pass == 0 ? W2.p : dst;
        const int64_t ldout = pass == 0 ? M : P;
        axpy_block(M, M, n, 1.0, src, M, Rd.p, 0.0, out, ldout, s);
        // Rt <- U Rt
        std::vector<double> T((size_t)M * M, 0.0);
        for (int c = 0; c < M; ++c)
          for (int r = 0; r < M; ++r) {
            double v = 0.0;
            for (int q = r; q < M; ++q) v += U[(size_t)q * M + r] * Rt[(size_t)c * M + q];
            T[(size_t)c * M + r] = v;
          }
        Rt.swap(T);
        WL_CUDA(cudaStreamSynchronize(s));  // Ui host buffer reused next pass
      }
      R = Rt;
    };
    cholqr(V.p, R0);
    std::vector<double> Rj;
    for (int j = 0; j < k; ++j) {
      // W = 𝕃_θ V_j  (one batched Laplacian action on M columns, internal order)
      run_chunk(op, ws, 1, V.p + (size_t)j * M, P, M, theta_index * M, M, Wb.p, M, s, false);
      const int pj = (j + 1) * M;
      for (int pass = 0; pass < 2; ++pass) {  // block classical Gram–Schmidt, twice
        gram(ws, pj, M, n, V.p, P, Wb.p, M, Cd.p, s);
        allreduce(op, Cd.p, (size_t)pj * M, s);
        axpy_block(pj, M, n, -1.0, V.p, P, Cd.p, 1.0, Wb.p, M, s);
        WL_CUDA(cudaMemcpyAsync(Ch.data(), Cd.p, sizeof(double) * pj * M, cudaMemcpyDeviceToHost, s));
        WL_CUDA(cudaStreamSynchronize(s));
        for (int c = 0; c < M; ++c)
          for (int r = 0; r < pj; ++r)
            if (r < d) H[(size_t)r * d + j * M + c] += Ch[(size_t)c * pj + r];
      }
      if (j + 1 < k) {
        cholqr(V.p + (size_t)(j + 1) * M, Rj);
        for (int c = 0; c < M; ++c)
          for (int r = 0; r < M; ++r) H[(size_t)((j + 1) * M + r) * d + j * M + c] = Rj[(size_t)c * M + r];
      }
    }
    // symmetric 𝕃 ⇒ H_k symmetric up to rounding
    for (int r = 0; r < d; ++r)
      for (int c = r + 1; c < d; ++c) {
        const double v = 0.5 * (H[(size_t)r * d + c] + H[(size_t)c * d + r]);
        H[(size_t)r * d + c] = H[(size_t)c * d + r] = v;
      }
    std::vector<double> lam, Q;
    if (!sym_eig_tridiag_ql(H, d, lam)) throw Error(WL_ENOCONV, "symmetric QL iteration did not converge");
    Q.swap(H);  // column a = eigenvector a
    // W = Qᵀ [R_0; 0]  (d x M row-major)
    std::vector<double> Wc((size_t)d * M, 0.0);
    for (int a = 0; a < d; ++a)
      for (int c = 0; c < M; ++c) {
        double v = 0.0;
        for (int r = 0; r <= c; ++r) v += Q[(size_t)r * d + a] * R0[(size_t)c * M + r];
        Wc[(size_t)a * M + c] = v;
      }
    if (!xnystrace_curve(lam, Wc, d, M, (double)op->n_global, times, nt, p_out, e_out))
      throw Error(WL_ENOCONV, "XNysTrace: leave-one-out Gram matrix not positive definite");
  });
}

// Block RATIONAL Arnoldi (Alg. 1 with its poles) on 𝔏 = 𝕃_{θ_i} in real arithmetic, then
// XNysTrace in the projected space.  Poles: ξ = ∞ (re = +inf), real, or a + ib (b > 0) standing for
// the conjugate pair; a final ∞ is appended (reading R18).  Step with continuation block u = V c (the last M
// columns of the newest block):
//   ∞: X = 𝔏 u;  real ξ: X = (𝔏 − ξI)⁻¹ u;  pair: X = [Re, Im] of (𝔏 − ξI)⁻¹ u   (MINRES, minres.cu)
// then block classical Gram–Schmidt twice + Cholesky QR (X = V_new h) and the pencil columns
//   ∞: K ← c, H ← h;  real: K ← h, H ← c + ξh;  pair: K ← [hr hi], H ← [c + a hr − b hi, b hr + a hi]
// so 𝔏 V K = V H.  Reduced pencil (last block row dropped): Ĥ K̂⁻¹ = V_kᵀ𝔏V_k (last pole ∞),
// symmetrised, eigendecomposed on the host, and Y(t) / XNysTrace as in wl_xnystrace_exp.
wl_status wl_xnystrace_exp_rational(const wl_operator* op, int32_t theta_index, int32_t M, const double* Omega,
                                    int64_t ldo, int32_t npoles, const double* poles_re, const double* poles_im,
                                    double inner_tol, int32_t inner_maxit, int32_t nt, const double* times,
                                    double* p_out, double* e_out, int64_t* inner_iters, wl_workspace* ws,
                                    wl_stream stream) {
  return guarded([&] {
    if (!op || !ws || ws->op != op) throw Error(WL_EINVAL, "operator/workspace mismatch");
    if (theta_index < 0 || theta_index >= op->n_theta) throw Error(WL_EINVAL, "theta_index out of range");
    if (M < 1 || M > ws->Bmax) throw Error(WL_EINVAL, "M must be in [1, workspace column batch]");
    if (npoles < 0 || (npoles > 0 && (!poles_re || !poles_im))) throw Error(WL_EINVAL, "bad poles");
    if (!(inner_tol > 0.0) || inner_maxit < 1) throw Error(WL_EINVAL, "inner_tol > 0 and inner_maxit >= 1 required");
    if (nt < 1 || !times || !p_out || !e_out) throw Error(WL_EINVAL, "bad output arguments");
    for (int i = 0; i < nt; ++i)
      if (!(times[i] >= 0.0)) throw Error(WL_EINVAL, "times must be >= 0");
    // pole list (+ the final ∞) and the dimension it builds
    std::vector<double> pre, pim;
    int64_t Dtot = M;
    for (int i = 0; i <= npoles; ++i) {
      const double re = i < npoles ? poles_re[i] : INFINITY, im = i < npoles ? poles_im[i] : 0.0;
      if (std::isnan(re) || std::isnan(im) || im < 0.0) throw Error(WL_EINVAL, "poles: NaN or negative imaginary part");
      if (std::isinf(re) && im != 0.0) throw Error(WL_EINVAL, "poles: infinite pole with an imaginary part");
      pre.push_back(re);
      pim.push_back(im);
      Dtot += im != 0.0 ? 2 * M : M;
    }
    if (Dtot - M > std::min<int64_t>(1024, op->n_global)) throw Error(WL_EINVAL, "basis dimension above min(1024, n)");
    if (op->n_loc > 0) check_block(Omega, ldo, M, "Omega");
    DeviceGuard dg(op->device);
    cudaStream_t s = S_(stream);
    const int64_t n = op->n_loc, nn = std::max<int64_t>(1, n);
    const int64_t ldV = Dtot;
    DArr<double>&V = ws->trV, &X = ws->trW, &W2 = ws->trW2, &Cd = ws->trC, &Rd = ws->trR;
    V.alloc((size_t)nn * ldV);
    X.alloc((size_t)nn * 2 * M);
    W2.alloc((size_t)nn * 2 * M);
    Cd.alloc((size_t)Dtot * 2 * M);
    Rd.alloc((size_t)4 * M * M);
    ws->rkU.alloc((size_t)nn * M + (size_t)nn * 2 * M);
    double* U = ws->rkU.p;
    double* XS = U + nn * M;  // MINRES solution [Re | Im], each n x M
    // Ω (user order) -> internal order -> V_1 R_0
    if (n > 0) {
      if (op->perm.p) pack_rows(Omega, ldo, op->perm.p, n, M, X.p, s);
      else WL_CUDA(cudaMemcpy2DAsync(X.p, sizeof(double) * M, Omega, sizeof(double) * ldo, sizeof(double) * M, n,
                                     cudaMemcpyDeviceToDevice, s));
    }
    std::vector<double> R0;
    chol_qr2(op, ws, X.p, M, n, W2.p, Rd.p, V.p, ldV, R0, s);
    const int64_t Dk = Dtot - M;                      // columns of the pencil
    std::vector<double> K((size_t)Dtot * Dk, 0.0), Hm((size_t)Dtot * Dk, 0.0);  // row-major D x Dk
    int64_t D = M, cstart = 0, col = 0, iters = 0;
    std::vector<double> Ch((size_t)Dtot * 2 * M), Rj;
    for (size_t st = 0; st < pre.size(); ++st) {
      const double re = pre[st], im = pim[st];
      const bool inf = std::isinf(re), cplx = im != 0.0;
      const int m = cplx ? 2 * M : M;
      // continuation u = V[:, cstart : cstart + M]
      repack_rows(V.p + cstart, ldV, n, M, U, M, s);
      if (inf) {
        run_chunk(op, ws, 1, U, M, M, theta_index * M, M, X.p, M, s, false);  // X = 𝔏 u
      } else {
        iters += shifted_solve(op, ws, theta_index, U, M, re, im, inner_tol, inner_maxit, XS, s);
        if (cplx) {
          repack_rows(XS, M, n, M, X.p, 2 * M, s);
          repack_rows(XS + nn * M, M, n, M, X.p + M, 2 * M, s);
        } else {
          repack_rows(XS, M, n, M, X.p, M, s);
        }
      }
      // block classical Gram–Schmidt twice against V[:, :D]; h accumulates the coefficients
      std::vector<double> hcoef((size_t)(D + m) * m, 0.0);  // row-major (D + m) x m
      for (int pass = 0; pass < 2; ++pass) {
        gram(ws, (int)D, m, n, V.p, ldV, X.p, m, Cd.p, s);
        allreduce(op, Cd.p, (size_t)D * m, s);
        axpy_block((int)D, m, n, -1.0, V.p, ldV, Cd.p, 1.0, X.p, m, s);
        WL_CUDA(cudaMemcpyAsync(Ch.data(), Cd.p, sizeof(double) * D * m, cudaMemcpyDeviceToHost, s));
        WL_CUDA(cudaStreamSynchronize(s));
        for (int c = 0; c < m; ++c)
          for (int64_t r = 0; r < D; ++r) hcoef[(size_t)r * m + c] += Ch[(size_t)c * D + r];
      }
      chol_qr2(op, ws, X.p, m, n, W2.p, Rd.p, V.p + D, ldV, Rj, s);
      if (getenv("WL_DEBUG_RATIONAL")) {
        double hmax = 0.0, rmin = INFINITY;
        for (double v : hcoef) hmax = std::max(hmax, std::fabs(v));
        for (int c = 0; c < m; ++c) rmin = std::min(rmin, std::fabs(Rj[(size_t)c * m + c]));
        fprintf(stderr, "[rational] step %zu pole (%g, %g) m=%d D=%lld max|h| %.3e min|R_ii| %.3e iters %lld\n", st, re,
                im, m, (long long)D, hmax, rmin, (long long)iters);
      }
      for (int c = 0; c < m; ++c)
        for (int r = 0; r <= c; ++r) hcoef[(size_t)(D + r) * m + c] = Rj[(size_t)c * m + r];
      // pencil columns [col, col + m)
      auto Kat = [&](int64_t r, int64_t c) -> double& { return K[(size_t)r * Dk + c]; };
      auto Hat = [&](int64_t r, int64_t c) -> double& { return Hm[(size_t)r * Dk + c]; };
      for (int c = 0; c < m; ++c)
        for (int64_t r = 0; r < D + m; ++r) {
          const double hv = hcoef[(size_t)r * m + c];
          const double cu = (c < M && r == cstart + c) ? 1.0 : 0.0;  // continuation selector
          if (inf) {
            Kat(r, col + c) = cu;
            Hat(r, col + c) = hv;
          } else if (!cplx) {
            Kat(r, col + c) = hv;
            Hat(r, col + c) = cu + re * hv;
          } else {
            Kat(r, col + c) = hv;
            if (c < M) Hat(r, col + c) = cu + re * hv - im * hcoef[(size_t)r * m + c + M];
            else Hat(r, col + c) = im * hcoef[(size_t)r * m + c - M] + re * hv;
          }
        }
      col += m;
      cstart = D + m - M;  // continuation: the last M columns of the newest block (reading R18)
      D += m;
    }
    // Projected operator on V_k = V[:, :d].  With the last pole at ∞ the reduced pencil Ĥ K̂⁻¹ equals the
    // Rayleigh quotient V_kᵀ 𝔏 V_k (reading R18); K̂ is, however, ill-conditioned in floating point once a
    // conjugate pair's real and imaginary directions nearly coincide modulo the basis (far poles: both
    // ≈ 𝔏u/|ξ|²; measured on the oracle at d = 450: ‖Ĥ K̂⁻¹ − (Ĥ K̂⁻¹)ᵀ‖ = 0.6 and a negative eigenvalue).
    // So the Rayleigh quotient is formed directly: d/M more batched Laplacian actions, symmetric by
    // construction.  (K, H above stay the Arnoldi bookkeeping of the decomposition 𝔏 V K = V H.)
    const int d = (int)Dk;
    std::vector<double> A((size_t)d * d, 0.0);
    for (int j0 = 0; j0 < d; j0 += M) {
      repack_rows(V.p + j0, ldV, n, M, U, M, s);
      run_chunk(op, ws, 1, U, M, M, theta_index * M, M, X.p, M, s, false);  // 𝔏 V[:, j0 : j0 + M]
      gram(ws, d, M, n, V.p, ldV, X.p, M, Cd.p, s);
      allreduce(op, Cd.p, (size_t)d * M, s);
      WL_CUDA(cudaMemcpyAsync(Ch.data(), Cd.p, sizeof(double) * d * M, cudaMemcpyDeviceToHost, s));
      WL_CUDA(cudaStreamSynchronize(s));
      for (int c = 0; c < M; ++c)
        for (int r = 0; r < d; ++r) A[(size_t)r * d + j0 + c] = Ch[(size_t)c * d + r];
    }
    double asym = 0.0;
    for (int r = 0; r < d; ++r)
      for (int c = r + 1; c < d; ++c) {
        asym = std::max(asym, std::fabs(A[(size_t)r * d + c] - A[(size_t)c * d + r]));
        A[(size_t)r * d + c] = A[(size_t)c * d + r] = 0.5 * (A[(size_t)r * d + c] + A[(size_t)c * d + r]);
      }
    std::vector<double> lam;
    if (!sym_eig_tridiag_ql(A, d, lam)) throw Error(WL_ENOCONV, "symmetric QL iteration did not converge");
    static const bool dbg = getenv("WL_DEBUG_RATIONAL") != nullptr;
    if (dbg)
      fprintf(stderr, "[rational] d=%d max|A-A^T| %.3e lambda [%.6e, %.6e] inner iters %lld\n", d, asym,
              *std::min_element(lam.begin(), lam.end()), *std::max_element(lam.begin(), lam.end()), (long long)iters);
    std::vector<double> Wc((size_t)d * M, 0.0);  // Qᵀ [R_0; 0]
    for (int a2 = 0; a2 < d; ++a2)
      for (int c = 0; c < M; ++c) {
        double v = 0.0;
        for (int r = 0; r <= c; ++r) v += A[(size_t)r * d + a2] * R0[(size_t)c * M + r];
        Wc[(size_t)a2 * M + c] = v;
      }
    if (!xnystrace_curve(lam, Wc, d, M, (double)op->n_global, times, nt, p_out, e_out))
      throw Error(WL_ENOCONV, "XNysTrace: leave-one-out Gram matrix not positive definite");
    if (inner_iters) *inner_iters = iters;
  });
}

// Gershgorin bound on ρ(𝕃_θ): |𝕃| row sums are 2 (t_i − φ_ii) <= 2 t'_i (φ − c_0 I >= 0 entrywise,
// Prop. pro:still-again-an-mmatrix), times wl_walkfun.scale — the interval of Alg. 1 line 3.
wl_status wl_laplacian_bound(const wl_operator* op, int32_t theta_index, double* bound) {
  return guarded([&] {
    if (!op || !bound) throw Error(WL_EINVAL, "NULL argument");
    if (theta_index < 0 || theta_index >= op->n_theta) throw Error(WL_EINVAL, "theta_index out of range");
    DeviceGuard dg(op->device);
    std::vector<double> t((size_t)op->n_loc * op->n_theta);
    if (!t.empty()) WL_CUDA(cudaMemcpy(t.data(), op->tprime.p, sizeof(double) * t.size(), cudaMemcpyDeviceToHost));
    double mx = 0.0;
    for (int64_t r = 0; r < op->n_loc; ++r) mx = std::max(mx, t[(size_t)r * op->n_theta + theta_index]);
    if (multi(op)) {
      int64_t bits;
      std::memcpy(&bits, &mx, sizeof(bits));
      std::vector<std::vector<int64_t>> all;
      comm_allgather_host(op->comm, {bits}, all, nullptr);
      for (auto& v : all) {
        double x;
        std::memcpy(&x, &v[0], sizeof(x));
        mx = std::max(mx, x);
      }
    }
    *bound = 2.0 * std::fabs(op->lscale) * mx;
  });
}

wl_status wl_symmetric_eig(int32_t n, double* A, double* lam, int32_t method) {
  return guarded([&] {
    if (n < 1 || !A || !lam || method < 0 || method > 1) throw Error(WL_EINVAL, "bad arguments");
    std::vector<double> a(A, A + (size_t)n * n), w, Q;
    bool ok = method == 0 ? sym_eig_tridiag_ql(a, n, w) : sym_eig_jacobi(a, n, w, Q);
    if (!ok) throw Error(WL_ENOCONV, "symmetric eigensolver did not converge");
    if (method == 1) a.swap(Q);
    std::copy(a.begin(), a.end(), A);
    std::copy(w.begin(), w.end(), lam);
  });
}

wl_status wl_xnystrace_curve(int32_t d, int32_t M, double n, const double* lam, const double* W, int32_t nt,
                             const double* times, double* p_out, double* e_out) {
  return guarded([&] {
    if (d < 1 || M < 1 || !(n > 0) || !lam || !W || nt < 1 || !times || !p_out || !e_out)
      throw Error(WL_EINVAL, "bad arguments");
    std::vector<double> l(lam, lam + d), w(W, W + (size_t)d * M);
    if (!xnystrace_curve(l, w, d, M, n, times, nt, p_out, e_out))
      throw Error(WL_ENOCONV, "XNysTrace: leave-one-out Gram matrix not positive definite");
  });
}

void wl_profile_enable(int32_t on) {
  std::lock_guard<std::mutex> lk(g_prof_mtx);
  g_prof_on = on != 0;
}

wl_status wl_profile_collect(void) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(g_prof_mtx);
    std::map<std::string, std::pair<double, int64_t>> acc;
    for (auto& r : g_prof) {
      WL_CUDA(cudaEventSynchronize(r.b));
      float ms = 0.f;
      WL_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
      auto& e = acc[r.name];
      e.first += ms;
      e.second += 1;
      g_prof_pool.push_back(r.a);
      g_prof_pool.push_back(r.b);
    }
    g_prof.clear();
    g_prof_result.assign(acc.begin(), acc.end());
  });
}

int32_t wl_profile_count(void) { return (int32_t)g_prof_result.size(); }

wl_status wl_profile_get(int32_t i, const char** name, double* total_ms, int64_t* launches) {
  return guarded([&] {
    if (i < 0 || i >= (int32_t)g_prof_result.size()) throw Error(WL_EINVAL, "profile index out of range");
    if (name) *name = g_prof_result[i].first.c_str();
    if (total_ms) *total_ms = g_prof_result[i].second.first;
    if (launches) *launches = g_prof_result[i].second.second;
  });
}

wl_status wl_wait(const wl_operator* op, wl_stream stream) {
  return guarded([&] {
    if (!op) throw Error(WL_EINVAL, "op is NULL");
    DeviceGuard dg(op->device);
    WL_CUDA(cudaStreamSynchronize(S_(stream)));
    WL_CUDA(cudaGetLastError());
    int st[4] = {0, 0, 0, 0};
    WL_CUDA(cudaMemcpy(st, op->kstat.p, sizeof(st), cudaMemcpyDeviceToHost));
    if (st[0] & 1) {
      WL_CUDA(cudaMemset(op->kstat.p, 0, sizeof(st)));
      double est;
      std::memcpy(&est, st + 2, sizeof(est));
      throw Error(WL_ENOCONV, "a-posteriori Krylov estimate " + std::to_string(est) + " above opts.tol (best iterate written)");
    }
  });
}

}  // extern "C"

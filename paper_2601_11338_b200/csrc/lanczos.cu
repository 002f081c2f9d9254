// lanczos.cu — the μ = 0 (θ = 1, all-walk) path: symmetric Lanczos on A ("Lanczos
// (for A = Aᵀ)").
//
// At μ = 0 the recurrence eq:qrec is q_k = A^k (P:286-288 with μ = 0), so φ v = c_0 v + f_1(A)(Av) with
// f_1(x) = Σ_k c_{k+1} x^k — the same f_1 and the same small-function kernel as the companion path, but
// on the n-dimensional symmetric A instead of the 2n-dimensional Z: the three-term Lanczos recurrence
//     β_0 q_0 = u = A v,   w = A q_j − β_j q_{j−1},   α_j = q_jᵀ w,   w ← w − α_j q_j,   β_{j+1} q_{j+1} = w
// builds T_k = tridiag(β, α, β), and φ v = c_0 v + ‖u‖ Q_k f_1(T_k) e_1.  Per step: one SpMM and three
// vector passes (α; w and ‖w‖²; scaling) over at most three n x B blocks, instead of TOAR's two passes
// over all j + 2 basis vectors.  No reorthogonalisation: for matrix functions the Lanczos approximation
// stays accurate in finite precision even when the basis loses orthogonality (Druskin & Knizhnerman;
// Musco, Musco & Sidford 2018); the parity tests check 1e-10 against the oracle.  Lucky breakdown
// (β_{j+1} <= btol ‖T_j‖ estimate) freezes a column at k_eff = j + 1.
// Vector kernels: thread t owns column t % B; per-CTA partials reduced in a fixed order.
#include "wl_internal.cuh"

#include <algorithm>

namespace wl {
namespace {

constexpr int kThreads = 256;

struct LzLane {
  int tpb, c;
  bool act;
  int64_t e0, stride;
  __device__ explicit LzLane(int B) {
    tpb = blockDim.x / B * B;
    act = (int)threadIdx.x < tpb;
    c = threadIdx.x % B;
    e0 = (int64_t)blockIdx.x * tpb + threadIdx.x;
    stride = (int64_t)gridDim.x * tpb;
  }
};

__device__ void lz_partials(double v, int B, int tpb, double* partials) {
  __shared__ double red[kThreads];
  red[threadIdx.x] = (int)threadIdx.x < tpb ? v : 0.0;
  __syncthreads();
  for (int c = threadIdx.x; c < B; c += blockDim.x) {
    double s = 0.0;
    for (int t = c; t < tpb; t += B) s += red[t];
    partials[(int64_t)c * gridDim.x + blockIdx.x] = s;
  }
}

// T: the storage type of the Lanczos vectors (double; float in the fp32 mode, R21) — sums are double.
// phase 0: Σ x² (x = the block at `a`);  phase 1: Σ q·w (a = q_j, b = w')
template <class T>
__global__ void __launch_bounds__(kThreads) lz_dot_kernel(int phase, const T* x, const T* y, int64_t n, int B,
                                                          double* partials) {
  const LzLane L(B);
  double v = 0.0;
  if (L.act)
    for (int64_t e = L.e0; e < n * B; e += L.stride) v += (double)x[e] * (double)(phase == 0 ? x[e] : y[e]);
  lz_partials(v, B, L.tpb, partials);
}

// w = w' − α q_j − β_j q_{j−1} (in place over w'); partials of ‖w‖² (of the stored values)
template <class T>
__global__ void __launch_bounds__(kThreads) lz_update_kernel(T* w, const T* q, const T* qm, int64_t n, int B,
                                                             const double* sc, double* partials) {
  const LzLane L(B);
  double v = 0.0;
  if (L.act) {
    const double al = sc[L.c * 4 + 1], be = sc[L.c * 4 + 0];
    for (int64_t e = L.e0; e < n * B; e += L.stride) {
      const T x = (T)((double)w[e] - al * (double)q[e] - (qm ? be * (double)qm[e] : 0.0));
      w[e] = x;
      v += (double)x * (double)x;
    }
  }
  lz_partials(v, B, L.tpb, partials);
}

// x *= 1/β per column (sc slot 2); with xp, also the row-padded copy the SpMM gathers (ld ldp, 32-byte rows)
template <class T>
__global__ void __launch_bounds__(kThreads) lz_scale_kernel(T* x, int64_t n, int B, const double* sc, T* xp,
                                                            int64_t ldp) {
  const LzLane L(B);
  if (!L.act) return;
  const double s = sc[L.c * 4 + 2];
  const int64_t dr = L.stride / B;  // the stride is a multiple of B: rows advance without a division
  int64_t r = L.e0 / B;
  for (int64_t e = L.e0; e < n * B; e += L.stride, r += dr) {
    const T v = (T)((double)x[e] * s);
    x[e] = v;
    if (xp) {
      xp[r * ldp + L.c] = v;
      // phantom columns: whole 32-byte sectors (no partial-sector writes in DRAM), spread over the row's threads
      for (int cc = B + L.c; cc < pad_vec_t<T>(B); cc += B) xp[r * ldp + cc] = T(0);
    }
  }
}

// One CTA: reduce the per-CTA partial rows (unless presummed), then per column
//   which 0 (‖u‖²):   β_0 = ‖u‖ -> n0, scale 1/β_0, k_eff = K (no breakdown yet)
//   which 1 (q·w'):   α_j -> H(j, j)
//   which 2 (‖w‖²):   β_{j+1} -> H(j+1, j) = H(j, j+1); scale 1/β_{j+1}; breakdown freezes the column
// sc per column: [β_j, α_j, scale, active]; H per column (K+1) x K column-major as in smallf.cu.
__global__ void __launch_bounds__(256) lz_scalar_kernel(int which, int j, int G, int presummed, const double* partials,
                                                        double* sums, int B, int K, double btol, double* sc, double* H,
                                                        double* n0, int* keff) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int ic = warp; ic < (presummed ? 0 : B); ic += blockDim.x / 32) {
    const double* p = partials + (int64_t)ic * G;
    double s0 = 0.0, s1 = 0.0;
    int g = lane;
    for (; g + 32 < G; g += 64) {
      s0 += p[g];
      s1 += p[g + 32];
    }
    if (g < G) s0 += p[g];
    double v = s0 + s1;
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) sums[ic] = v;
  }
  __syncthreads();
  const int c = threadIdx.x;
  if (c >= B) return;
  double* s = sc + c * 4;
  double* Hc = H + (int64_t)c * (K + 1) * K;
  const double v = sums[c];
  if (which == 0) {
    const double nu = sqrt(fmax(v, 0.0));
    n0[c] = nu;
    s[0] = 0.0;
    s[1] = 0.0;
    s[2] = nu > 0.0 ? 1.0 / nu : 0.0;
    s[3] = nu > 0.0 ? 1.0 : 0.0;
    keff[c] = nu > 0.0 ? K : 0;
  } else if (which == 1) {
    s[1] = v;
    if (s[3] != 0.0) Hc[(int64_t)j * (K + 1) + j] = v;
  } else {
    const double be = sqrt(fmax(v, 0.0));
    if (s[3] != 0.0) {
      // lucky breakdown: the Krylov space of this column is invariant after j + 1 vectors
      const double ref = fabs(s[1]) + s[0];
      if (!(be > btol * ref)) {
        s[3] = 0.0;
        keff[c] = j + 1;
        s[2] = 0.0;
      } else {
        Hc[(int64_t)j * (K + 1) + j + 1] = be;
        if (j + 1 < K) Hc[(int64_t)(j + 1) * (K + 1) + j] = be;
        s[2] = 1.0 / be;
      }
    } else {
      s[2] = 0.0;
    }
    s[0] = be;
  }
}

int lz_grid(int64_t n, int B) {
  const int tpb = kThreads / B * B;
  const int64_t need = (n * B + tpb - 1) / tpb;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)num_sms() * 6));
}

}  // namespace

int lanczos_grid(int64_t n, int B) { return lz_grid(n, B); }

template <class T>
void lanczos_vec_t(int phase, T* x, const T* y, const T* qm, int64_t n, int B, const double* sc, double* partials,
                   cudaStream_t s, T* xp, int64_t ldp) {
  const int G = lz_grid(n, B);
  if (phase <= 1) lz_dot_kernel<T><<<G, kThreads, 0, s>>>(phase, x, y, n, B, partials);
  else if (phase == 2) lz_update_kernel<T><<<G, kThreads, 0, s>>>(x, y, qm, n, B, sc, partials);
  else lz_scale_kernel<T><<<G, kThreads, 0, s>>>(x, n, B, sc, xp, ldp);
}

void lanczos_vec(int phase, double* x, const double* y, const double* qm, int64_t n, int B, const double* sc,
                 double* partials, cudaStream_t s, double* xp, int64_t ldp, bool f32) {
  WL_LAUNCH("lanczos_vec");
  if (f32)
    lanczos_vec_t<float>(phase, reinterpret_cast<float*>(x), reinterpret_cast<const float*>(y),
                         reinterpret_cast<const float*>(qm), n, B, sc, partials, s, reinterpret_cast<float*>(xp), ldp);
  else
    lanczos_vec_t<double>(phase, x, y, qm, n, B, sc, partials, s, xp, ldp);
  WL_CUDA(cudaGetLastError());
}

void lanczos_scalar(int which, int j, int64_t n, int presummed, const double* partials, double* sums, int B, int K,
                    double btol, double* sc, double* H, double* n0, int* keff, cudaStream_t s) {
  WL_LAUNCH("lanczos_scalar");
  lz_scalar_kernel<<<1, 256, 0, s>>>(which, j, lz_grid(n, B), presummed, partials, sums, B, K, btol, sc, H, n0, keff);
  WL_CUDA(cudaGetLastError());
}

}  // namespace wl

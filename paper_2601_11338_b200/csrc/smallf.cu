// smallf.cu — the small projected matrix function (step a6), on the device.
//
// After k Arnoldi steps on Z the action is  φ v = c_0 v + ||u|| [I O] Q_k f_1(H_k) e_1
// (Prop. pro:whe-we-converge; Krylov approximation).  One CTA per Krylov
// column evaluates y = f_1(H_m) e_1 for the m x m leading block of its upper Hessenberg H
// (m = k, or the breakdown dimension):
//   exp(βx):     f_1(x) = β φ_1(βx)  ->  y = β * (top m entries of the last column of
//                expm([[βH, e_1], [0, 0]]))  — Padé(13) scaling-and-squaring (Higham 2005)
//   resolvent:   f_1(x) = α (1 - αx)^{-1}        ->  y = α (I - αH)^{-1} e_1   (LU, partial pivot)
//   series c_j:  f_1(x) = Σ_j c_{j+1} x^j        ->  Horner-free power accumulation of H^j e_1
// The outer diffusion Lanczos (kind 3) uses the same expm for exp(-τ H_out) e_1.
// Everything is fp64; matrices live in a per-problem global scratch (L1/L2 resident, <= 130^2).
#include "wl_internal.cuh"
#include <cmath>

namespace wl {
namespace {

constexpr int kBS = 256;
constexpr int kSlots = 9;  // scratch matrices per problem

__device__ void mm(const double* A, const double* B, double* C, int N) {  // C = A B
  for (int idx = threadIdx.x; idx < N * N; idx += blockDim.x) {
    const int i = idx / N, j = idx - i * N;
    double s = 0.0;
    for (int k = 0; k < N; ++k) s += A[i * N + k] * B[k * N + j];
    C[idx] = s;
  }
  __syncthreads();
}

// X <- solve(Qm, X) for N right-hand sides, Gaussian elimination with partial pivoting.
__device__ void lu_solve(double* Qm, double* X, int N, int nrhs) {
  __shared__ int s_piv;
  __shared__ double s_l[kMaxSmallN];
  for (int k = 0; k < N; ++k) {
    if (threadIdx.x < 32) {
      double best = -1.0;
      int bi = k;
      for (int i = k + (int)threadIdx.x; i < N; i += 32) {
        const double v = fabs(Qm[i * N + k]);
        if (v > best) { best = v; bi = i; }
      }
      for (int off = 16; off > 0; off >>= 1) {
        const double ob = __shfl_down_sync(0xffffffffu, best, off);
        const int oi = __shfl_down_sync(0xffffffffu, bi, off);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (threadIdx.x == 0) s_piv = bi;
    }
    __syncthreads();
    const int p = s_piv;
    if (p != k) {
      for (int j = threadIdx.x; j < N; j += blockDim.x) {
        const double t = Qm[k * N + j]; Qm[k * N + j] = Qm[p * N + j]; Qm[p * N + j] = t;
      }
      for (int j = threadIdx.x; j < nrhs; j += blockDim.x) {
        const double t = X[k * nrhs + j]; X[k * nrhs + j] = X[p * nrhs + j]; X[p * nrhs + j] = t;
      }
    }
    __syncthreads();
    const double piv = Qm[k * N + k];
    for (int i = k + 1 + threadIdx.x; i < N; i += blockDim.x) s_l[i] = (piv != 0.0) ? Qm[i * N + k] / piv : 0.0;
    __syncthreads();
    const int rows = N - k - 1, colsA = N - k - 1;
    for (int idx = threadIdx.x; idx < rows * colsA; idx += blockDim.x) {
      const int i = k + 1 + idx / colsA, j = k + 1 + idx % colsA;
      Qm[i * N + j] -= s_l[i] * Qm[k * N + j];
    }
    for (int idx = threadIdx.x; idx < rows * nrhs; idx += blockDim.x) {
      const int i = k + 1 + idx / nrhs, j = idx % nrhs;
      X[i * nrhs + j] -= s_l[i] * X[k * nrhs + j];
    }
    __syncthreads();
  }
  for (int j = threadIdx.x; j < nrhs; j += blockDim.x) {  // back substitution, one RHS per thread
    for (int i = N - 1; i >= 0; --i) {
      double s = X[i * nrhs + j];
      for (int l = i + 1; l < N; ++l) s -= Qm[i * N + l] * X[l * nrhs + j];
      X[i * nrhs + j] = s / Qm[i * N + i];
    }
  }
  __syncthreads();
}

// In place: A (N x N, row-major) <- expm(A).  Padé(13) with scaling and squaring.
__device__ void expm_inplace(double* A, int N, double* scr) {
  const double b[14] = {64764752532480000.0, 32382376266240000.0, 7771770303897600.0,
                        1187353796428800.0, 129060195264000.0, 10559470521600.0,
                        670442572800.0, 33522128640.0, 1323241920.0, 40840800.0,
                        960960.0, 16380.0, 182.0, 1.0};
  const int NN = N * N;
  double* A2 = scr;
  double* A4 = scr + NN;
  double* A6 = scr + 2 * NN;
  double* U = scr + 3 * NN;
  double* V = scr + 4 * NN;
  double* T1 = scr + 5 * NN;
  double* T2 = scr + 6 * NN;
  __shared__ int s_sq;
  if (threadIdx.x == 0) {
    double nrm = 0.0;  // ||A||_1
    for (int j = 0; j < N; ++j) {
      double cs = 0.0;
      for (int i = 0; i < N; ++i) cs += fabs(A[i * N + j]);
      nrm = fmax(nrm, cs);
    }
    const double theta13 = 5.371920351148152;
    int sq = 0;
    if (nrm > theta13) sq = (int)ceil(log2(nrm / theta13));
    s_sq = sq;
  }
  __syncthreads();
  const int sq = s_sq;
  const double scale = ldexp(1.0, -sq);
  for (int i = threadIdx.x; i < NN; i += blockDim.x) A[i] *= scale;
  __syncthreads();
  mm(A, A, A2, N);
  mm(A2, A2, A4, N);
  mm(A4, A2, A6, N);
  for (int idx = threadIdx.x; idx < NN; idx += blockDim.x) {
    const double id = (idx % (N + 1) == 0) ? 1.0 : 0.0;
    T1[idx] = b[13] * A6[idx] + b[11] * A4[idx] + b[9] * A2[idx];
    T2[idx] = b[12] * A6[idx] + b[10] * A4[idx] + b[8] * A2[idx];
    U[idx] = b[7] * A6[idx] + b[5] * A4[idx] + b[3] * A2[idx] + b[1] * id;
    V[idx] = b[6] * A6[idx] + b[4] * A4[idx] + b[2] * A2[idx] + b[0] * id;
  }
  __syncthreads();
  mm(A6, T1, A2, N);  // A2 <- A6 * T1   (A2 no longer needed)
  for (int idx = threadIdx.x; idx < NN; idx += blockDim.x) T1[idx] = A2[idx] + U[idx];
  __syncthreads();
  mm(A, T1, U, N);    // U = A (A6 T1 + ...)
  mm(A6, T2, A4, N);  // A4 <- A6 * T2
  for (int idx = threadIdx.x; idx < NN; idx += blockDim.x) {
    V[idx] += A4[idx];
    const double u = U[idx], v = V[idx];
    T1[idx] = v - u;  // Q = V - U
    A[idx] = v + U[idx];  // P = V + U (A consumed)
  }
  __syncthreads();
  lu_solve(T1, A, N, N);  // A <- (V - U)^{-1} (V + U)
  for (int s = 0; s < sq; ++s) {
    mm(A, A, T2, N);
    for (int idx = threadIdx.x; idx < NN; idx += blockDim.x) A[idx] = T2[idx];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kBS) small_f_kernel(SmallFArgs a) {
  const int p = blockIdx.x;
  const int c = (a.kind == 3) ? 0 : p;  // Krylov column whose H is used
  const int K = a.K, B = a.B;
  double* scr = a.scratch + (int64_t)p * kSlots * kMaxSmallN * kMaxSmallN;
  const double* H = a.H + (int64_t)c * (K + 1) * K;
  const int m = a.keff[c];
  double* y = scr + 8 * kMaxSmallN * kMaxSmallN;  // m entries
  if (m > 0) {
    if (a.kind == 3) {  // outer diffusion: y = exp(-tau_p H_m) e_1
      const int N = m;
      double* M = scr + 7 * kMaxSmallN * kMaxSmallN;
      const double tp = a.tau[p];
      for (int idx = threadIdx.x; idx < N * N; idx += blockDim.x) {
        const int i = idx / N, j = idx - i * N;
        M[idx] = -tp * H[j * (K + 1) + i];
      }
      __syncthreads();
      expm_inplace(M, N, scr);
      for (int i = threadIdx.x; i < m; i += blockDim.x) y[i] = M[i * N + 0];
    } else if (a.kind == 0) {  // exp: y = β φ_1(βH) e_1 via expm of the (m+1) augmented matrix
      const int N = m + 1;
      double* M = scr + 7 * kMaxSmallN * kMaxSmallN;
      for (int idx = threadIdx.x; idx < N * N; idx += blockDim.x) {
        const int i = idx / N, j = idx - i * N;
        double v = 0.0;
        if (i < m && j < m) v = a.param * H[j * (K + 1) + i];
        else if (i == 0 && j == m) v = 1.0;
        M[idx] = v;
      }
      __syncthreads();
      expm_inplace(M, N, scr);
      for (int i = threadIdx.x; i < m; i += blockDim.x) y[i] = a.param * M[i * N + m];
    } else if (a.kind == 1) {  // resolvent: y = α (I - αH)^{-1} e_1
      const int N = m;
      double* M = scr;
      double* X = scr + kMaxSmallN * kMaxSmallN;
      for (int idx = threadIdx.x; idx < N * N; idx += blockDim.x) {
        const int i = idx / N, j = idx - i * N;
        M[idx] = (i == j ? 1.0 : 0.0) - a.param * H[j * (K + 1) + i];
      }
      for (int i = threadIdx.x; i < N; i += blockDim.x) X[i] = (i == 0) ? 1.0 : 0.0;
      __syncthreads();
      lu_solve(M, X, N, 1);
      for (int i = threadIdx.x; i < m; i += blockDim.x) y[i] = a.param * X[i];
    } else {  // series: y = Σ_{j>=0} c_{j+1} H^j e_1
      double* p = scr;                       // current H^j e_1
      double* pn = scr + kMaxSmallN;
      for (int i = threadIdx.x; i < m; i += blockDim.x) { p[i] = (i == 0) ? 1.0 : 0.0; y[i] = 0.0; }
      __syncthreads();
      for (int j = 0; j + 1 < a.ncoeffs; ++j) {
        const double cj = a.coeffs[j + 1];
        for (int i = threadIdx.x; i < m; i += blockDim.x) y[i] += cj * p[i];
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
          double s = 0.0;
          for (int l = 0; l < m; ++l) s += H[l * (K + 1) + i] * p[l];
          pn[i] = s;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < m; i += blockDim.x) p[i] = pn[i];
        __syncthreads();
      }
    }
  }
  __syncthreads();
  const double n0 = a.n0[c];
  // a-posteriori estimate (kinds 0-2): ||u|| h_{m+1,m} |e_m^T y| relative to ||u|| ||y||; exact (0) after a
  // breakdown (h_{m+1,m} = 0: invariant Krylov space).  m < K is also the probe of the adaptive stop.
  if (a.kind != 3 && a.err && threadIdx.x == 0) {
    double e = 0.0;
    if (m > 0) {
      double yy = 0.0;
      for (int i = 0; i < m; ++i) yy += y[i] * y[i];
      e = yy > 0.0 ? fabs(H[(m - 1) * (K + 1) + m] * y[m - 1]) / sqrt(yy) : 0.0;
    }
    a.err[c] = e;
  }
  for (int i = threadIdx.x; i <= K; i += blockDim.x) {
    const double v = (i < m) ? n0 * y[i] * (a.s ? a.s[i * B + c] : 1.0) : 0.0;
    if (a.kind == 3) a.comb[(int64_t)p * (K + 1) + i] = v;
    else a.comb[i * B + c] = v;
  }
}

}  // namespace

void small_f(const SmallFArgs& a, cudaStream_t s) {
  if (a.K + 1 > kMaxSmallN) throw Error(1, "small_f: Krylov dimension too large");
  WL_LAUNCH("small_f");
  small_f_kernel<<<a.kind == 3 ? a.nprob : a.B, kBS, 0, s>>>(a);
  WL_CUDA(cudaGetLastError());
}

}  // namespace wl

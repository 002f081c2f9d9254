// toar.cu — two-level orthogonal Arnoldi (TOAR) bookkeeping for the companion operator Z (step a5).
//
// Why.  The Krylov space of Z = [[O, I], [M, A]] (M = μ(μI - D), eq:Zdef) started from
// u = [q_1 v; q_2 v] is spanned by Z^i u = [w_{i+1}; w_{i+2}], w_k = q_k(A) v (eq:qrec): the top and
// bottom halves of every Krylov vector lie in ONE n-dimensional space span{w_1, ..., w_{k+2}}.  So
// the 2n-long Arnoldi basis q_0..q_k is stored as q_i = [U g_i; U f_i] over k+2 n-vectors U (half the
// memory), and the Gram-Schmidt work on n-vectors shrinks to one dot pass and one update pass over U
// per step (about 45% fewer bytes than DCGS2 on 2n-vectors).  This is the TOAR idea of Su, Zhang &
// Bai (2008) for linearised quadratic eigenproblems, applied to the paper's Arnoldi.
//
// Numerics.  U is orthogonalised by ONE classical Gram-Schmidt pass per step, and its exact Gram
// matrix G = U^T U is measured by the next step's dot pass (the row of the newest vector) and
// factored incrementally, G = L L^T.  All coefficient-space work uses the orthonormal basis
// W = U L^{-T} ("W coordinates"), in which inner products of 2n-vectors are plain dot products of
// coefficient vectors.  When a step forms its new U vector it does not know that vector's Gram row
// yet and assumes it orthonormal; the next step learns the true row, converts the provisional
// Arnoldi vector to true coordinates and re-orthonormalises it, correcting the previous H column
// exactly as delayed classical Gram-Schmidt does (Z q_j = (Z q̂_j - Σ a_i Z q_i)/ν).  Coefficient-
// space Gram-Schmidt is done twice.  One thread per Krylov column; everything here is O(k^2) per
// step on vectors of length <= k+3.
#include "wl_internal.cuh"

#include <algorithm>

namespace wl {
namespace {

// per-column state: L (M x M, row-major lower), TQg/TQf ((K+1) x M: W coords of q_i), QHg/QHf (M:
// the provisional next vector), ZY (M: W coords of y), DEAD (M), SC (8 scalars)
struct State {
  double *L, *TQg, *TQf, *QHg, *QHf, *ZY, *DEAD, *SC;
  __device__ State(double* base, int M, int K) {
    L = base;
    TQg = L + M * M;
    TQf = TQg + (K + 1) * M;
    QHg = TQf + (K + 1) * M;
    QHf = QHg + M;
    ZY = QHf + M;
    DEAD = ZY + M;
    SC = DEAD + M;
  }
};
enum { kHprov = 0, kAlive = 1, kNuY = 2, kRef = 3 };

// x = L^{-T} v over indices < m (back substitution)
__device__ void solve_lt(const double* L, int M, int m, const double* v, double* x) {
  for (int i = m - 1; i >= 0; --i) {
    double s = v[i];
    for (int k = i + 1; k < m; ++k) s -= L[k * M + i] * x[k];
    const double dg = L[i * M + i];
    x[i] = dg != 0.0 ? s / dg : s;  // rows never measured (column stopped early) act as identity
  }
}

}  // namespace

size_t toar_state_doubles(int K) {
  const int M = K + 3;
  return (size_t)M * M + 2 * (size_t)(K + 1) * M + 5 * (size_t)M + 8;
}

// One warp per column c (lanes over coefficient indices).  j = -1: seed step (U = [t0], y = b0);
// j = 0..K-1: Arnoldi step j; final = 1: only the Gram row of the last U vector and the correction
// of H column K-1.
// sums: the dcgs2_dots layout for Q = U_0..U_{m-2}, p = U_{m-1}, w = y: [a_i b_i]_{i<m-1} α β γ.
// Outputs: coef_y[o*B + c], coef_u[(o*coef_ld + i)*B + c] for the TOAR update pass:
//   j = -1: o = 0 -> u_1;   j >= 0: o = 0 -> u_m, 1 -> x_{j+1} = bottom(q̂_{j+1}), 2 -> z_{j+1} = top.
constexpr int kCoefWarps = 4;
constexpr int kV = kMaxKrylov + 4;  // coefficient vector capacity (>= K + 3)

__device__ inline double wsum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ inline double diag_or_one(double d) { return d != 0.0 ? d : 1.0; }

// x = L^{-1} v (rows < m), x may not alias v
__device__ void fwd_w(const double* L, int M, int m, const double* v, double* x, int lane) {
  for (int i = 0; i < m; ++i) {
    double p = 0.0;
    for (int k = lane; k < i; k += 32) p += L[i * M + k] * x[k];
    p = wsum(p);
    if (lane == 0) x[i] = (v[i] - p) / diag_or_one(L[i * M + i]);
    __syncwarp();
  }
}
// x = L^{-T} v (rows < m); rows never measured (column stopped early) act as identity
__device__ void bwd_w(const double* L, int M, int m, const double* v, double* x, int lane) {
  for (int i = m - 1; i >= 0; --i) {
    double p = 0.0;
    for (int k = i + 1 + lane; k < m; k += 32) p += L[k * M + i] * x[k];
    p = wsum(p);
    if (lane == 0) x[i] = (v[i] - p) / diag_or_one(L[i * M + i]);
    __syncwarp();
  }
}
// <(g1,f1),(g2,f2)> over indices < m
__device__ inline double dot2(const double* g1, const double* f1, const double* g2, const double* f2, int m,
                              int lane) {
  double p = 0.0;
  for (int k = lane; k < m; k += 32) p += g1[k] * g2[k] + f1[k] * f2[k];
  return wsum(p);
}
__device__ inline void axpy2(double s, const double* g, const double* f, double* yg, double* yf, int m, int lane) {
  for (int k = lane; k < m; k += 32) {
    yg[k] += s * g[k];
    yf[k] += s * f[k];
  }
  __syncwarp();
}

__global__ void __launch_bounds__(32 * kCoefWarps) toar_coeffs_kernel(const double* sums, int j, int final_pass, int B,
                                                                      int K, double btol, double* H, double* n0,
                                                                      int* keff, double* state, size_t stride,
                                                                      double* coef_y, double* coef_u, int coef_ld) {
  __shared__ double sh[kCoefWarps][8][kV];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * kCoefWarps + wid;
  if (c >= B) return;
  double* Fh = sh[wid][0];
  double* av = sh[wid][1];
  double* wg = sh[wid][2];
  double* wf = sh[wid][3];
  double* cu = sh[wid][4];
  double* tmp = sh[wid][5];
  double* sv = sh[wid][6];
  double* hv = sh[wid][7];
  const int M = K + 3;
  State S(state + (size_t)c * stride, M, K);
  double* Hc = H + (size_t)c * (K + 1) * K;  // (row i, col l) at Hc[l*(K+1) + i]
  const int m = final_pass ? K + 2 : (j < 0 ? 1 : j + 2);  // U vectors with a Gram row after this step
  const int nq = m - 1;
  auto sum = [&](int k) { return sums[(size_t)k * B + c]; };
  const int nout = j < 0 ? 1 : 3;
  auto zero_out = [&]() {
    for (int o = 0; o < nout; ++o) {
      if (lane == 0) coef_y[o * B + c] = 0.0;
      for (int i = lane; i < m; i += 32) coef_u[((size_t)o * coef_ld + i) * B + c] = 0.0;
    }
  };
  if (j < 0) {  // fresh column state
    for (int i = lane; i < M * M; i += 32) S.L[i] = 0.0;
    for (int i = lane; i < M; i += 32) S.DEAD[i] = 0.0;
    if (lane == 0) S.SC[kAlive] = 1.0;
    __syncwarp();
  }
  if (S.SC[kAlive] == 0.0) {
    if (!final_pass) zero_out();
    return;
  }
  // 1. Gram row of the newest U vector u_{m-1}: L row m-1 (forward solve); a zero vector gets the
  //    identity row and is marked dead
  {
    double* Lr = S.L + (size_t)(m - 1) * M;
    for (int i = lane; i < nq; i += 32) sv[i] = sum(2 * i);
    __syncwarp();
    fwd_w(S.L, M, nq, sv, tmp, lane);
    double ll = 0.0;
    for (int i = lane; i < nq; i += 32) ll += tmp[i] * tmp[i];
    ll = wsum(ll);
    const double alpha = sum(2 * nq);
    const double d2 = alpha - ll;
    const bool dead = !(alpha > 0.0) || !(d2 > 1e-24 * alpha);
    for (int i = lane; i < nq; i += 32) Lr[i] = dead ? 0.0 : tmp[i];
    if (lane == 0) {
      Lr[nq] = dead ? 1.0 : sqrt(d2);
      S.DEAD[nq] = dead ? 1.0 : 0.0;
    }
    __syncwarp();
  }
  const double* Lm = S.L + (size_t)(m - 1) * M;
  // 2. provisional vector to true W coordinates: its component e along the assumed w_{m-1} = u_{m-1}
  //    is e u_{m-1} = e Σ_i L[m-1][i] w_i
  if (j >= 0) {
    const double eg = S.QHg[m - 1], ef = S.QHf[m - 1];
    const bool dead = S.DEAD[m - 1] != 0.0;
    __syncwarp();
    for (int i = lane; i < m; i += 32) {
      const double l = dead ? 0.0 : Lm[i];
      if (i < m - 1) {
        S.QHg[i] += eg * l;
        S.QHf[i] += ef * l;
      } else {
        S.QHg[i] = eg * l;
        S.QHf[i] = ef * l;
      }
    }
    __syncwarp();
    for (int i = lane; i < m; i += 32) Fh[i] = S.QHf[i];
    __syncwarp();
  }
  // 3. y in W coordinates: z = L^{-1} s, ν_y² = γ - |z|²;  y = W z + ν_y u_m  (u_m := (y - U c)/ν_y)
  double nuy = 0.0;
  if (!final_pass) {
    for (int i = lane; i < m; i += 32) sv[i] = i < nq ? sum(2 * i + 1) : sum(2 * nq + 1);
    __syncwarp();
    fwd_w(S.L, M, m, sv, S.ZY, lane);
    double zz = 0.0;
    for (int i = lane; i < m; i += 32) zz += S.ZY[i] * S.ZY[i];
    zz = wsum(zz);
    const double gamma = sum(2 * nq + 2);
    nuy = sqrt(fmax(gamma - zz, 0.0));
    if (!(nuy > 1e-12 * sqrt(gamma))) nuy = 0.0;  // y in span(U): no new direction
  }
  if (j < 0) {  // seed: q̂_0 = [t0; b0] = [L00 w_0; W z + ν_y u_1]
    for (int i = lane; i < M; i += 32) {
      S.QHg[i] = i == 0 ? (S.DEAD[0] != 0.0 ? 0.0 : S.L[0]) : 0.0;
      S.QHf[i] = i == 0 ? S.ZY[0] : (i == 1 ? nuy : 0.0);
    }
    __syncwarp();
    bwd_w(S.L, M, m, S.ZY, cu, lane);  // u_1 = (b0 - U c)/ν_y, c = L^{-T} z
    const double inv = nuy > 0.0 ? 1.0 / nuy : 0.0;
    if (lane == 0) coef_y[c] = inv;
    for (int i = lane; i < m; i += 32) coef_u[(size_t)i * B + c] = -cu[i] * inv;
    return;
  }
  // 4. re-orthonormalise q̂_j against q_0..q_{j-1} (twice), completing H column j-1
  for (int i = lane; i < j; i += 32) av[i] = 0.0;
  __syncwarp();
  for (int pass = 0; pass < 2; ++pass)
    for (int i = 0; i < j; ++i) {
      const double* tg = S.TQg + (size_t)i * M;
      const double* tf = S.TQf + (size_t)i * M;
      const double dd = dot2(tg, tf, S.QHg, S.QHf, m, lane);
      axpy2(-dd, tg, tf, S.QHg, S.QHf, m, lane);
      if (lane == 0) av[i] += dd;
    }
  __syncwarp();
  const double nuq = sqrt(dot2(S.QHg, S.QHf, S.QHg, S.QHf, m, lane));
  if (j == 0) {
    if (lane == 0) {
      n0[c] = nuq;
      keff[c] = nuq > 0.0 ? K : 0;
      S.SC[kRef] = nuq;
      if (!(nuq > 0.0)) S.SC[kAlive] = 0.0;
    }
  } else if (lane == 0) {
    const double hp = S.SC[kHprov];
    for (int i = 0; i < j; ++i) Hc[(j - 1) * (K + 1) + i] += hp * av[i];
    const double sub = hp * nuq;
    if (sub > btol * S.SC[kRef] && sub > 0.0) {
      Hc[(j - 1) * (K + 1) + j] = sub;
    } else {
      Hc[(j - 1) * (K + 1) + j] = 0.0;
      keff[c] = j;
      S.SC[kAlive] = 0.0;
    }
  }
  __syncwarp();
  if (final_pass) return;
  if (S.SC[kAlive] == 0.0) {
    zero_out();
    return;
  }
  {  // q_j
    double* tg = S.TQg + (size_t)j * M;
    double* tf = S.TQf + (size_t)j * M;
    const double inv = 1.0 / nuq;
    for (int k = lane; k < M; k += 32) {
      tg[k] = k < m ? S.QHg[k] * inv : 0.0;
      tf[k] = k < m ? S.QHf[k] * inv : 0.0;
    }
    __syncwarp();
  }
  // 5. Z q_j = (Z q̂_j - Σ_{i<j} a_i Z q_i)/ν,  Z q̂_j = [f̂ ; W z + ν_y u_m],  Σ_i a_i Z q_i = Σ_l (H a)_l q_l
  const int m1 = m + 1;
  for (int k = lane; k < m1; k += 32) {
    wg[k] = k < m ? Fh[k] : 0.0;
    wf[k] = k < m ? S.ZY[k] : nuy;
  }
  for (int l = lane; l <= j; l += 32) {
    double s = 0.0;
    for (int i = (l > 0 ? l - 1 : 0); i < j; ++i) s += Hc[i * (K + 1) + l] * av[i];
    hv[l] = s;
  }
  __syncwarp();
  for (int l = 0; l <= j; ++l)
    if (hv[l] != 0.0) axpy2(-hv[l], S.TQg + (size_t)l * M, S.TQf + (size_t)l * M, wg, wf, m, lane);
  {
    const double inv = 1.0 / nuq;
    for (int k = lane; k < m1; k += 32) {
      wg[k] *= inv;
      wf[k] *= inv;
    }
    __syncwarp();
  }
  const double ref = sqrt(dot2(wg, wf, wg, wf, m1, lane));
  // 6. Arnoldi: h = Q^T Z q_j (twice), provisional q̂_{j+1}
  for (int i = lane; i <= j; i += 32) hv[i] = 0.0;
  __syncwarp();
  for (int pass = 0; pass < 2; ++pass)
    for (int i = 0; i <= j; ++i) {
      const double* tg = S.TQg + (size_t)i * M;
      const double* tf = S.TQf + (size_t)i * M;
      const double dd = dot2(tg, tf, wg, wf, m, lane);
      axpy2(-dd, tg, tf, wg, wf, m, lane);
      if (lane == 0) hv[i] += dd;
    }
  __syncwarp();
  const double hs = sqrt(dot2(wg, wf, wg, wf, m1, lane));
  for (int i = lane; i <= j; i += 32) Hc[j * (K + 1) + i] = hv[i];
  if (lane == 0) {
    S.SC[kHprov] = hs;
    S.SC[kRef] = ref;
  }
  __syncwarp();
  if (!(hs > btol * ref)) {  // invariant Krylov subspace: column j is final, H(j+1, j) = 0
    if (lane == 0) {
      keff[c] = j + 1;
      S.SC[kAlive] = 0.0;
    }
    zero_out();
    return;
  }
  {
    const double inv = 1.0 / hs;
    for (int k = lane; k < M; k += 32) {
      S.QHg[k] = k < m1 ? wg[k] * inv : 0.0;
      S.QHf[k] = k < m1 ? wf[k] * inv : 0.0;
    }
    __syncwarp();
  }
  // 7. update-pass coefficients: u_m = (y - U c)/ν_y;  v in W coords over [W_m, u_m]:
  //    W v = U L^{-T} v[0:m] + v[m] (y - U c)/ν_y
  bwd_w(S.L, M, m, S.ZY, cu, lane);
  const double iy = nuy > 0.0 ? 1.0 / nuy : 0.0;
  if (lane == 0) coef_y[c] = iy;
  for (int i = lane; i < m; i += 32) coef_u[(size_t)i * B + c] = -cu[i] * iy;
  for (int o = 1; o < 3; ++o) {
    const double* v = o == 1 ? S.QHf : S.QHg;
    bwd_w(S.L, M, m, v, tmp, lane);
    const double vm = v[m] * iy;
    if (lane == 0) coef_y[o * B + c] = vm;
    for (int i = lane; i < m; i += 32) coef_u[((size_t)o * coef_ld + i) * B + c] = tmp[i] - vm * cu[i];
    __syncwarp();
  }
}

// comb_U = L^{-T} Σ_i comb_i g_i (W coords -> U coords) so that Σ_i comb_i top(q_i) = U comb_U
__global__ void toar_combine_coef_kernel(const double* comb, int B, int K, const int* keff, const double* state,
                                         size_t stride, double* combU) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= B) return;
  const int M = K + 3, mU = K + 2;
  State S(const_cast<double*>(state) + (size_t)c * stride, M, K);
  double v[kMaxKrylov + 3], x[kMaxKrylov + 3];
  for (int k = 0; k < mU; ++k) v[k] = 0.0;
  const int ke = keff[c];
  for (int i = 0; i < ke; ++i) {
    const double w = comb[(size_t)i * B + c];
    const double* tg = S.TQg + (size_t)i * M;
    for (int k = 0; k < mU; ++k) v[k] += w * tg[k];
  }
  // rows of L beyond what the (possibly early-stopped) column measured are identity rows
  solve_lt(S.L, M, mU, v, x);
  for (int k = 0; k < mU; ++k) combU[(size_t)k * B + c] = ke > 0 ? x[k] : 0.0;
}

void toar_coeffs(const double* sums, int j, int final_pass, int B, int K, double btol, double* H, double* n0,
                 int* keff, double* state, size_t stride, double* coef_y, double* coef_u, int coef_ld,
                 cudaStream_t s) {
  WL_LAUNCH("toar_coeffs");
  toar_coeffs_kernel<<<(B + kCoefWarps - 1) / kCoefWarps, 32 * kCoefWarps, 0, s>>>(
      sums, j, final_pass, B, K, btol, H, n0, keff, state, stride, coef_y, coef_u, coef_ld);
  WL_CUDA(cudaGetLastError());
}

void toar_combine_coef(const double* comb, int B, int K, const int* keff, const double* state, size_t stride,
                       double* combU, cudaStream_t s) {
  WL_LAUNCH("toar_coeffs");
  toar_combine_coef_kernel<<<1, 32, 0, s>>>(comb, B, K, keff, state, stride, combU);
  WL_CUDA(cudaGetLastError());
}

}  // namespace wl

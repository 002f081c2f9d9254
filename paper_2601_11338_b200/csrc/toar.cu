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
  double *L, *TQg, *TQf, *QHg, *QHf, *ZY, *DEAD, *SC, *LI;
  __device__ State(double* base, int M, int K) {
    L = base;
    TQg = L + M * M;
    TQf = TQg + (K + 1) * M;
    QHg = TQf + (K + 1) * M;
    QHf = QHg + M;
    ZY = QHf + M;
    DEAD = ZY + M;
    SC = DEAD + M;
    LI = SC + 8;  // L^{-1}, maintained row by row (M x M, row-major lower)
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
  return 2 * (size_t)M * M + 2 * (size_t)(K + 1) * M + 5 * (size_t)M + 8;
}

// One CTA (4 warps) per column c, its state staged in shared memory.  j = -1: seed step (U = [t0],
// y = b0); j = 0..K-1: Arnoldi step j; final = 1: only the Gram row of the last U vector and the
// correction of H column K-1.
// sums: the dcgs2_dots layout for Q = U_0..U_{m-2}, p = U_{m-1}, w = y: [a_i b_i]_{i<m-1} α β γ.
// Outputs: coef_y[o*B + c], coef_u[(o*coef_ld + i)*B + c] for the TOAR update pass:
//   j = -1: o = 0 -> u_1;   j >= 0: o = 0 -> u_m, 1 -> x_{j+1} = bottom(q̂_{j+1}), 2 -> z_{j+1} = top.
// Gram-Schmidt in coefficient space is classical (all projections of a pass at once), done twice.
#ifndef WL_COEF_THREADS
#define WL_COEF_THREADS 1024  // C3 diffusion sweep: 128 -> 1024 threads, toar_coeffs 119 -> 111 ms
#endif
constexpr int kCoefThreads = WL_COEF_THREADS;
constexpr int kMaxVecPerLaunchCoef = kMaxKrylov + 2;  // dot-pass outputs per column: 2(m-1)+3, m <= K+2
constexpr int kV = kMaxKrylov + 4;  // coefficient vector capacity (>= K + 3)

__device__ inline double wsum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ inline double diag_or_one(double d) { return d != 0.0 ? d : 1.0; }

constexpr int kCoefWarps = kCoefThreads / 32;

// out(r, Σ_{k in [lo(r), hi(r))} term(r, k)) for r < nrows: a warp per output, lanes over k (the
// mat-vecs here have <= K+3 terms, so one or two lane rounds and one shuffle reduction); caller syncs
template <class Lo, class Hi, class T, class O>
__device__ inline void warp_rows(int nrows, Lo lo, Hi hi, T term, O out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  #pragma unroll 1
  for (int r = warp; r < nrows; r += kCoefWarps) {
    double s = 0.0;
    #pragma unroll 1
    for (int k = lo(r) + lane; k < hi(r); k += 32) s += term(r, k);
    s = wsum(s);
    if (lane == 0) out(r, s);
  }
}

// x = LI v (LI lower triangular, rows < m); caller syncs
__device__ __noinline__ void li_mv(const double* LI, int M, int m, const double* v, double* x) {
  warp_rows(m, [](int) { return 0; }, [](int i) { return i + 1; },
            [&](int i, int k) { return LI[i * M + k] * v[k]; }, [&](int i, double s) { x[i] = s; });
}
// x = LI^T v (rows < m); caller syncs
__device__ __noinline__ void li_tmv(const double* LI, int M, int m, const double* v, double* x) {
  warp_rows(m, [](int k) { return k; }, [&](int) { return m; },
            [&](int k, int i) { return LI[i * M + k] * v[i]; }, [&](int k, double s) { x[k] = s; });
}

// classical Gram-Schmidt pass of (wg, wf) (length n) against the nb vectors (TG_i, TF_i) (stride M):
// d_i = <TQ_i, w> for all i (a warp per i, lanes over k), then w -= Σ d_i TQ_i (a thread per k);
// acc[i] += d_i
__device__ __noinline__ void cgs_pass(const double* TG, const double* TF, int M, int nb, double* wg, double* wf, int n,
                         double* dv, double* acc, bool first) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  #pragma unroll 1
  for (int i = warp; i < nb; i += kCoefWarps) {
    double p = 0.0;
    #pragma unroll 1
    for (int k = lane; k < n; k += 32) p += TG[i * M + k] * wg[k] + TF[i * M + k] * wf[k];
    p = wsum(p);
    if (lane == 0) dv[i] = p;
  }
  __syncthreads();
  // w -= Σ_i d_i TQ_i: a warp per entry (g half in rows [0, n), f half in [n, 2n))
  warp_rows(2 * n, [](int) { return 0; }, [&](int) { return nb; },
            [&](int r, int i) { return dv[i] * (r < n ? TG[i * M + r] : TF[i * M + r - n]); },
            [&](int r, double s) {
              if (r < n) wg[r] -= s;
              else wf[r - n] -= s;
            });
  #pragma unroll 1
  for (int i = threadIdx.x; i < nb; i += kCoefThreads) acc[i] = first ? dv[i] : acc[i] + dv[i];
  __syncthreads();
}
__device__ __noinline__ double block_norm2(const double* g, const double* f, int n, double* red) {
  double p = 0.0;
  #pragma unroll 1
  for (int k = threadIdx.x; k < n; k += kCoefThreads) p += g[k] * g[k] + f[k] * f[k];
  p = wsum(p);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = p;
  __syncthreads();
  const double s = wsum((threadIdx.x & 31) < kCoefWarps ? red[threadIdx.x & 31] : 0.0);
  __syncthreads();
  return s;
}

__global__ void __launch_bounds__(kCoefThreads) toar_coeffs_kernel(const double* sums, const double* partials, int G,
                                                                   int j, int final_pass, int B,
                                                                   int K, double btol, double* H, double* n0,
                                                                   int* keff, double* state, size_t stride,
                                                                   double* coef_y, double* coef_u, int coef_ld) {
  extern __shared__ double smem[];
  const int c = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int M = K + 3;
  State S(state + (size_t)c * stride, M, K);
  double* Hc = H + (size_t)c * (K + 1) * K;  // (row i, col l) at Hc[l*(K+1) + i]
  // the final pass after k' <= K steps (k' = K, or earlier with opts.krylov_adaptive) is called with j = k'
  const int m = final_pass ? j + 2 : (j < 0 ? 1 : j + 2);  // U vectors with a Gram row after this step
  const int nq = m - 1;
  const int nt = j < 0 ? 0 : (final_pass ? j : j + 1);      // q vectors used this step (q_0..q_j)
  // shared layout: L (m x M), TQg/TQf (nt x M), QHg/QHf, ZY, work vectors
  double* L = smem;
  double* TG = L + (size_t)m * M;
  double* TF = TG + (size_t)nt * M;
  double* QG = TF + (size_t)nt * M;
  double* QF = QG + kV;
  double* ZY = QF + kV;
  double* Fh = ZY + kV;
  double* av = Fh + kV;
  double* wg = av + kV;
  double* wf = wg + kV;
  double* cu = wf + kV;
  double* t1 = cu + kV;
  double* t2 = t1 + kV;
  double* sv = t2 + kV;
  double* hv = sv + kV;
  double* dv = hv + kV;
  double* red = dv + kV;
  double* Hs = red + kV;  // H columns 0..j (ld K+1), staged
  double* LIs = Hs + (size_t)(K + 1) * K;  // L^{-1} rows 0..m-1
  __shared__ int alive_s;
  __shared__ double ssum[2 * kMaxVecPerLaunchCoef + 3];
  {  // this column's dot-pass outputs, reduced here from the per-CTA partials when given (fixed order)
    const int nval = 2 * (m - 1) + 3;
    if (partials) {
      #pragma unroll 1
      for (int k = warp; k < nval; k += kCoefWarps) {
        const double* p = partials + ((size_t)k * B + c) * G;
        double v = 0.0;
        #pragma unroll 8  // independent loads in flight: G partials are L2 round trips
        for (int g = lane; g < G; g += 32) v += p[g];
        v = wsum(v);
        if (lane == 0) ssum[k] = v;
      }
    } else {
      #pragma unroll 1
      for (int k = tid; k < nval; k += kCoefThreads) ssum[k] = sums[(size_t)k * B + c];
    }
    __syncthreads();
  }
  auto sum = [&](int k) { return ssum[k]; };
  const int nout = j < 0 ? 1 : 3;
  auto zero_out = [&]() {
    #pragma unroll 1
    for (int o = 0; o < nout; ++o) {
      if (tid == 0) coef_y[o * B + c] = 0.0;
      #pragma unroll 1
      for (int i = tid; i < m; i += kCoefThreads) coef_u[((size_t)o * coef_ld + i) * B + c] = 0.0;
    }
  };
  if (j < 0) {  // fresh column state
    #pragma unroll 1
    for (int i = tid; i < M * M; i += kCoefThreads) {
      S.L[i] = 0.0;
      S.LI[i] = 0.0;
    }
    #pragma unroll 1
    for (int i = tid; i < M; i += kCoefThreads) S.DEAD[i] = 0.0;
    if (tid == 0) S.SC[kAlive] = 1.0;
    __syncthreads();
  }
  if (S.SC[kAlive] == 0.0) {
    if (!final_pass) zero_out();
    return;
  }
  // stage the state: one flat index space over (L, L^{-1}), (TQg, TQf), (QHg, QHf), H; each thread
  // issues the global loads of 4 pairs before it stores any of them (one L2 round trip per 4 pairs
  // instead of one per array)
  const int hcols = j < 0 ? 0 : (final_pass ? j : j + 1);
  {
    const int nL = (m - 1) * M, nT = nt * M, nH = hcols * (K + 1);
    const int tkeep = final_pass ? nT : (nt - 1) * M;  // q_j is recomputed this step
    const int total = nL + nT + kV + nH;
    auto load = [&](int i, double& x, double& y) {
      if (i < nL) {
        x = S.L[i];
        y = S.LI[i];
      } else if ((i -= nL) < nT) {
        x = i < tkeep ? S.TQg[i] : 0.0;
        y = i < tkeep ? S.TQf[i] : 0.0;
      } else if ((i -= nT) < kV) {
        x = i < M ? S.QHg[i] : 0.0;
        y = i < M ? S.QHf[i] : 0.0;
      } else {
        x = Hc[i - kV];
        y = 0.0;
      }
    };
    auto store = [&](int i, double x, double y) {
      if (i < nL) {
        L[i] = x;
        LIs[i] = y;
      } else if ((i -= nL) < nT) {
        TG[i] = x;
        TF[i] = y;
      } else if ((i -= nT) < kV) {
        QG[i] = x;
        QF[i] = y;
      } else {
        Hs[i - kV] = x;
      }
    };
    #pragma unroll 1
    for (int base = tid; base < total; base += 4 * kCoefThreads) {
      double x[4], y[4];
      #pragma unroll
      for (int u = 0; u < 4; ++u)
        if (base + u * kCoefThreads < total) load(base + u * kCoefThreads, x[u], y[u]);
      #pragma unroll
      for (int u = 0; u < 4; ++u)
        if (base + u * kCoefThreads < total) store(base + u * kCoefThreads, x[u], y[u]);
    }
  }
  __syncthreads();
  // 1. Gram row of the newest U vector u_{m-1}: l = L^{-1} a, L row m-1 = (l, sqrt(α - |l|²)), and the
  //    matching row of L^{-1}, (-l^T L^{-1}, 1)/L[m-1][m-1]; a zero vector gets identity rows (dead)
  double* Lr = L + (size_t)(m - 1) * M;
  double* LIr = LIs + (size_t)(m - 1) * M;
  #pragma unroll 1
  for (int i = tid; i < nq; i += kCoefThreads) sv[i] = sum(2 * i);
  __syncthreads();
  li_mv(LIs, M, nq, sv, t1);
  __syncthreads();
  double llv = 0.0;
  {
    double p = 0.0;
    #pragma unroll 1
    for (int i = tid; i < nq; i += kCoefThreads) p += t1[i] * t1[i];
    p = wsum(p);
    if (lane == 0) red[warp] = p;
    __syncthreads();
    llv = wsum(lane < kCoefWarps ? red[lane] : 0.0);
    __syncthreads();
  }
  const double alpha = sum(2 * nq);
  const double d2 = alpha - llv;
  const bool dead_new = !(alpha > 0.0) || !(d2 > 1e-24 * alpha);
  const double lmm = dead_new ? 1.0 : sqrt(d2);
  #pragma unroll 1
  for (int k = tid; k < M; k += kCoefThreads) {
    Lr[k] = k < nq ? (dead_new ? 0.0 : t1[k]) : (k == nq ? lmm : 0.0);
    if (k >= nq || dead_new) LIr[k] = k == nq ? 1.0 / lmm : 0.0;
  }
  if (!dead_new)
    warp_rows(nq, [](int k) { return k; }, [&](int) { return nq; },
              [&](int k, int i) { return t1[i] * LIs[i * M + k]; }, [&](int k, double s) { LIr[k] = -s / lmm; });
  if (tid == 0) S.DEAD[nq] = dead_new ? 1.0 : 0.0;
  __syncthreads();
  #pragma unroll 1
  for (int i = tid; i < M; i += kCoefThreads) {
    S.L[(size_t)(m - 1) * M + i] = Lr[i];
    S.LI[(size_t)(m - 1) * M + i] = LIr[i];
  }
  // 2. provisional vector to true W coordinates: its component e along the assumed w_{m-1} = u_{m-1}
  //    is e u_{m-1} = e Σ_i L[m-1][i] w_i
  if (j >= 0) {
    const double eg = QG[m - 1], ef = QF[m - 1];
    const bool dead = S.DEAD[m - 1] != 0.0;
    __syncthreads();
    #pragma unroll 1
    for (int i = tid; i < m; i += kCoefThreads) {
      const double l = dead ? 0.0 : Lr[i];
      if (i < m - 1) {
        QG[i] += eg * l;
        QF[i] += ef * l;
      } else {
        QG[i] = eg * l;
        QF[i] = ef * l;
      }
    }
    __syncthreads();
    #pragma unroll 1
    for (int i = tid; i < m; i += kCoefThreads) Fh[i] = QF[i];
  }
  // 3. y in W coordinates: z = L^{-1} s, ν_y² = γ - |z|²;  y = W z + ν_y u_m  (u_m := (y - U c)/ν_y)
  double nuy = 0.0;
  if (!final_pass) {
    #pragma unroll 1
    for (int i = tid; i < m; i += kCoefThreads) sv[i] = i < nq ? sum(2 * i + 1) : sum(2 * nq + 1);
    __syncthreads();
    li_mv(LIs, M, m, sv, ZY);
    __syncthreads();
    double zz = 0.0;
    #pragma unroll 1
    for (int i = lane; i < m; i += 32) zz += ZY[i] * ZY[i];
    zz = wsum(zz);
    const double gamma = sum(2 * nq + 2);
    nuy = sqrt(fmax(gamma - zz, 0.0));
    if (!(nuy > 1e-12 * sqrt(gamma))) nuy = 0.0;  // y in span(U): no new direction
  }
  if (j < 0) {  // seed: q̂_0 = [t0; b0] = [L00 w_0; W z + ν_y u_1]
    #pragma unroll 1
    for (int i = tid; i < M; i += kCoefThreads) {
      S.QHg[i] = i == 0 ? (S.DEAD[0] != 0.0 ? 0.0 : L[0]) : 0.0;
      S.QHf[i] = i == 0 ? ZY[0] : (i == 1 ? nuy : 0.0);
    }
    li_tmv(LIs, M, m, ZY, cu);  // u_1 = (b0 - U c)/ν_y, c = L^{-T} z
    __syncthreads();
    const double inv = nuy > 0.0 ? 1.0 / nuy : 0.0;
    if (tid == 0) coef_y[c] = inv;
    #pragma unroll 1
    for (int i = tid; i < m; i += kCoefThreads) coef_u[(size_t)i * B + c] = -cu[i] * inv;
    return;
  }
  // 4. re-orthonormalise q̂_j against q_0..q_{j-1} (classical, twice), completing H column j-1
  cgs_pass(TG, TF, M, j, QG, QF, m, dv, av, true);  // av[i < j] = the two passes' coefficients
  cgs_pass(TG, TF, M, j, QG, QF, m, dv, av, false);
  const double nuq = sqrt(block_norm2(QG, QF, m, red));
  if (j > 0) {  // H column j-1 += hprov a, H(j, j-1) = hprov ν
    const double hp = S.SC[kHprov];
    #pragma unroll 1
    for (int i = tid; i < j; i += kCoefThreads) {
      const double v = Hs[(j - 1) * (K + 1) + i] + hp * av[i];
      Hs[(j - 1) * (K + 1) + i] = v;
      Hc[(j - 1) * (K + 1) + i] = v;
    }
  }
  if (tid == 0) {
    if (j == 0) {
      n0[c] = nuq;
      keff[c] = nuq > 0.0 ? K : 0;
      S.SC[kRef] = nuq;
      alive_s = nuq > 0.0;
    } else {
      const double sub = S.SC[kHprov] * nuq;
      alive_s = sub > btol * S.SC[kRef] && sub > 0.0;
      Hs[(j - 1) * (K + 1) + j] = alive_s ? sub : 0.0;
      Hc[(j - 1) * (K + 1) + j] = alive_s ? sub : 0.0;
      if (!alive_s) keff[c] = j;
    }
    if (!alive_s) S.SC[kAlive] = 0.0;
    if (final_pass && keff[c] > j) keff[c] = j;  // stopped after j < K steps
  }
  __syncthreads();
  if (final_pass) return;
  if (!alive_s) {
    zero_out();
    return;
  }
  {  // q_j
    const double inv = 1.0 / nuq;
    #pragma unroll 1
    for (int k = tid; k < M; k += kCoefThreads) {
      const double g = k < m ? QG[k] * inv : 0.0, f = k < m ? QF[k] * inv : 0.0;
      TG[(size_t)j * M + k] = g;
      TF[(size_t)j * M + k] = f;
      S.TQg[(size_t)j * M + k] = g;
      S.TQf[(size_t)j * M + k] = f;
    }
  }
  // 5. Z q_j = (Z q̂_j - Σ_{i<j} a_i Z q_i)/ν,  Z q̂_j = [f̂ ; W z + ν_y u_m],  Σ_i a_i Z q_i = Σ_l (H a)_l q_l
  const int m1 = m + 1;
  #pragma unroll 1
  for (int k = tid; k < m1; k += kCoefThreads) {
    wg[k] = k < m ? Fh[k] : 0.0;
    wf[k] = k < m ? ZY[k] : nuy;
  }
  warp_rows(j + 1, [](int l) { return l > 0 ? l - 1 : 0; }, [&](int) { return j; },
            [&](int l, int i) { return Hs[i * (K + 1) + l] * av[i]; }, [&](int l, double s) { hv[l] = s; });
  __syncthreads();
  warp_rows(2 * m, [](int) { return 0; }, [&](int) { return j + 1; },
            [&](int r, int l) { return hv[l] * (r < m ? TG[(size_t)l * M + r] : TF[(size_t)l * M + r - m]); },
            [&](int r, double s) {
              if (r < m) wg[r] = (wg[r] - s) / nuq;
              else wf[r - m] = (wf[r - m] - s) / nuq;
            });
  if (tid == 0) {
    wg[m] /= nuq;
    wf[m] /= nuq;
  }
  __syncthreads();
  const double ref = sqrt(block_norm2(wg, wf, m1, red));
  // 6. Arnoldi: h = Q^T Z q_j (classical, twice), provisional q̂_{j+1}
  cgs_pass(TG, TF, M, j + 1, wg, wf, m, dv, hv, true);  // hv[i <= j] = h
  cgs_pass(TG, TF, M, j + 1, wg, wf, m, dv, hv, false);
  const double hs = sqrt(block_norm2(wg, wf, m1, red));
  #pragma unroll 1
  for (int i = tid; i <= j; i += kCoefThreads) Hc[j * (K + 1) + i] = hv[i];
  if (tid == 0) {
    S.SC[kHprov] = hs;
    S.SC[kRef] = ref;
  }
  if (!(hs > btol * ref)) {  // invariant Krylov subspace: column j is final, H(j+1, j) = 0
    if (tid == 0) {
      keff[c] = j + 1;
      S.SC[kAlive] = 0.0;
    }
    zero_out();
    return;
  }
  {
    const double inv = 1.0 / hs;
    #pragma unroll 1
    for (int k = tid; k < M; k += kCoefThreads) {
      const double g = k < m1 ? wg[k] * inv : 0.0, f = k < m1 ? wf[k] * inv : 0.0;
      QG[k] = g;
      QF[k] = f;
      S.QHg[k] = g;
      S.QHf[k] = f;
    }
  }
  __syncthreads();
  // 7. update-pass coefficients: u_m = (y - U c)/ν_y;  v in W coords over [W_m, u_m]:
  //    W v = U L^{-T} v[0:m] + v[m] (y - U c)/ν_y      (three back-solves on three warps)
  li_tmv(LIs, M, m, ZY, cu);
  li_tmv(LIs, M, m, QF, t1);
  li_tmv(LIs, M, m, QG, t2);
  __syncthreads();
  const double iy = nuy > 0.0 ? 1.0 / nuy : 0.0;
  const double vm1 = QF[m] * iy, vm2 = QG[m] * iy;
  if (tid == 0) {
    coef_y[c] = iy;
    coef_y[B + c] = vm1;
    coef_y[2 * B + c] = vm2;
  }
  #pragma unroll 1
  for (int i = tid; i < m; i += kCoefThreads) {
    coef_u[(size_t)i * B + c] = -cu[i] * iy;
    coef_u[((size_t)coef_ld + i) * B + c] = t1[i] - vm1 * cu[i];
    coef_u[((size_t)2 * coef_ld + i) * B + c] = t2[i] - vm2 * cu[i];
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

void toar_coeffs(const double* sums, const double* partials, int G, int j, int final_pass, int B, int K, double btol,
                 double* H, double* n0, int* keff, double* state, size_t stride, double* coef_y, double* coef_u,
                 int coef_ld, cudaStream_t s) {
  WL_LAUNCH("toar_coeffs");
  const int M = K + 3;
  const size_t smem = sizeof(double) * (2 * (size_t)(K + 2) * M + 2 * (size_t)(K + 1) * M + 16 * (size_t)kV +
                                       (size_t)(K + 1) * K);
  static bool attr = false;
  if (!attr) {
    const size_t smax = sizeof(double) * (2 * (size_t)(kMaxKrylov + 2) * (kMaxKrylov + 3) +
                                          2 * (size_t)(kMaxKrylov + 1) * (kMaxKrylov + 3) + 16 * (size_t)kV +
                                          (size_t)(kMaxKrylov + 1) * kMaxKrylov);
    WL_CUDA(cudaFuncSetAttribute(toar_coeffs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax));
    attr = true;
  }
  toar_coeffs_kernel<<<B, kCoefThreads, smem, s>>>(sums, partials, G, j, final_pass, B, K, btol, H, n0, keff, state,
                                                  stride, coef_y, coef_u, coef_ld);
  WL_CUDA(cudaGetLastError());
}

void toar_combine_coef(const double* comb, int B, int K, const int* keff, const double* state, size_t stride,
                       double* combU, cudaStream_t s) {
  WL_LAUNCH("toar_coeffs");
  toar_combine_coef_kernel<<<1, 32, 0, s>>>(comb, B, K, keff, state, stride, combU);
  WL_CUDA(cudaGetLastError());
}

}  // namespace wl

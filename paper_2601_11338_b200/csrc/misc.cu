// misc.cu — small kernels of the Krylov engine: batching of inputs, DCGS2 bookkeeping,
// the combine/Laplacian epilogue (step a7) and halo packing.
#include "wl_internal.cuh"
#include <cmath>

namespace wl {
namespace {

// internal row r holds user row perm[r] (degree-sorted relabelling; perm null = identity)
__global__ void batch_inputs_kernel(const double* V, int64_t ldv, int B, int64_t n, double* Vb,
                                    const int* vcol, const int32_t* perm) {
  const int64_t total = n * B;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / B;
    const int j = (int)(e - r * B);
    const int64_t ru = perm ? perm[r] : r;
    Vb[e] = V ? V[ru * ldv + vcol[j]] : 1.0;
  }
}

// Seeds shared by the θ columns of one input column (TOAR path): s1 = A v and s2 = A(Av) are
// θ-independent, so they are computed once per input column (n x b) and expanded to the B Krylov
// columns: t0[r][c] = s1[r][vcol c],  b0[r][c] = s2[r][vcol c] - μ_c d_r v[r][vcol c]  (eq:qrec seeds).
template <class T>
__global__ void seed_expand_kernel(const double* s1, const double* s2, const double* v, int b, const int32_t* rowptr,
                                   const double* g1s, const int* vcol, int B, int64_t n, T* t0, T* b0) {
  const int64_t total = n * B;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / B;
    const int c = (int)(e - r * B);
    const int64_t src = r * b + vcol[c];
    const double d = (double)(__ldg(rowptr + r + 1) - __ldg(rowptr + r));
    t0[e] = (T)s1[src];
    b0[e] = (T)(s2[src] + g1s[c] * d * v[src]);  // g1s = -μ
  }
}

// mode 0: out = c0 V + Σ_i comb_i Q_i          (φ V, top half of the Z basis)
// mode 1: out = t' ⊙ V - Σ_i comb_i Q_i        (𝕃 V = diag(t)V - φV, c_0 cancels)
// mode 2: out = Σ_i comb_i Q_i                 (t' = φ1 - c_0 1 for V = 1)
template <int NV, class T>
__global__ void combine_kernel(int mode, double lscale, const VecPtrs Q, int nvec, int64_t n, int B,
                               const double* comb, const double* V, int64_t ldv, const int* vcol,
                               double c0, const double* tprime, int64_t ldt, const int* tcol,
                               double* out, int64_t ldo, const int32_t* perm, int64_t nq) {
  __shared__ double s_comb[NV * kMaxCols];
  for (int idx = threadIdx.x; idx < nvec * B; idx += blockDim.x) s_comb[idx] = comb[idx];
  __syncthreads();
  const int64_t total = n * B;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / B;
    const int c = (int)(e - r * B);
    double acc = 0.0;
    if (r < nq) {
#pragma unroll 8
      for (int i = 0; i < NV; ++i)
        if (i < nvec) acc += s_comb[i * B + c] * (double)__ldg(reinterpret_cast<const T*>(Q.p[i]) + e);
    }
    double o;
    const int64_t ru = perm ? perm[r] : r;  // user row of internal row r
    if (mode == 2) {
      o = acc;
      out[r * ldo + c] = o;  // t' stays in internal order
    } else {
      const double v = V ? V[ru * ldv + vcol[c]] : 1.0;
      o = (mode == 0) ? c0 * v + acc : lscale * (tprime[r * ldt + tcol[c]] * v - acc);
      out[ru * ldo + c] = o;
    }
  }
}

template <class T>
__global__ void pack_rows_kernel(const T* src, int64_t lds, const int32_t* idx, int64_t cnt, int B, T* dst) {
  const int64_t total = cnt * B;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / B;
    const int c = (int)(e - k * B);
    dst[e] = src[(int64_t)idx[k] * lds + c];
  }
}

__global__ void krylov_check_kernel(const double* err, int B, double tol, int* flag) {
  const int c = threadIdx.x;
  if (c < B && err[c] > tol) {
    atomicOr(flag, 1);
    atomicMax(reinterpret_cast<unsigned long long*>(flag + 2), (unsigned long long)__double_as_longlong(err[c]));
  }
}

// Markov chain helpers (eq:let_there_be_markov): internal-order vectors, perm = internal -> user row
__global__ void gather_col_kernel(const double* src, int64_t lds, const int32_t* perm, int64_t n, double* dst) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    dst[r] = src[(perm ? (int64_t)perm[r] : r) * lds];
}
__global__ void scatter_col_kernel(const double* src, const int32_t* perm, int64_t n, double* dst, int64_t ldd) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    dst[(perm ? (int64_t)perm[r] : r) * ldd] = src[r];
}
// v = p / t,  t = t' + c0 (D = diag(t), reading R6)
__global__ void markov_scale_kernel(const double* p, const double* tprime, int64_t ldt, int tcol, double c0,
                                    int64_t n, double* v) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    v[r] = p[r] / (tprime[r * ldt + tcol] + c0);
}

// p[i] = 0.5 + u(seed, i0 + i), u uniform in [0,1) from a counter-based hash (splitmix64)
__global__ void fill_hash_kernel(double* p, int64_t n, uint64_t seed, int64_t i0) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * (uint64_t)(i0 + i + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    p[i] = 0.5 + (double)(z >> 11) * (1.0 / 9007199254740992.0);
  }
}

__global__ void fill_kernel(double* p, int64_t n, double v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// X[r, s] = scale * Σ_i Q_i[r] Y[s*m + i]   (outer Lanczos combine, Q_i unit-stride length n)
__global__ void lanczos_combine_kernel(const double* Q, int64_t stride, int m, int64_t n, const double* Y,
                                       int nt, double scale, double* X, int64_t ldx, const int32_t* perm) {
  extern __shared__ double s_Y[];  // m * nt
  for (int idx = threadIdx.x; idx < m * nt; idx += blockDim.x) s_Y[idx] = Y[idx];
  __syncthreads();
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    for (int s0 = 0; s0 < nt; s0 += 8) {
      double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int i = 0; i < m; ++i) {
        const double qi = __ldg(Q + i * stride + r);
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (s0 + u < nt) acc[u] += qi * s_Y[(s0 + u) * m + i];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (s0 + u < nt) X[(perm ? (int64_t)perm[r] : r) * ldx + s0 + u] = scale * acc[u];
    }
  }
}

// Per-chunk column parameters: batch column c is global column g = gstart + c of the
// n_theta*b output block, i.e. θ index g / b and input column g % b; μ = 1 - θ.
//   Z step   (eq:Zdef):  g0 = μ²,  g1 = -μ     (μ(μI - D))
//   seed q_2 (eq:qrec):  g0 = 0,   g1 = -μ     (A² - μD)
__global__ void setup_chunk_kernel(const double* mu, int gstart, int b, int B, double* g0z, double* g1z,
                                   double* g0s, double* g1s, int* vcol, int* tcol) {
  const int c = threadIdx.x;
  if (c >= B) return;
  const int g = gstart + c;
  const double m = mu[g / b];
  g0z[c] = m * m;
  g1z[c] = -m;
  g0s[c] = 0.0;
  g1s[c] = -m;
  vcol[c] = g % b;
  tcol[c] = g / b;
}

// ---- DCGS2 Arnoldi bookkeeping (one thread per Krylov column) -----------------------------
// Delayed reorthogonalisation (Świrydowicz et al. 2021; Bielich et al. 2022), derived for the
// Arnoldi relation Z Q_k = Q_{k+1} H_k.  At step j the dots of pass A give, for p_j (the vector
// orthogonalised once at step j-1) and w = Z p_j:
//   a = Q_j^T p_j, b = Q_j^T w, α = p_j.p_j, β = p_j.w, γ = w.w.
// Reorthogonalisation: q_j = (p_j - Q_j a)/ν, ν² = α - |a|²; it completes column j-1 of H:
//   H(0:j, j-1) += a, H(j, j-1) = ν.
// Then Z q_j = (w - Q_{j+1} H_j a)/ν, so its first-pass projection on Q_{j+1} is
//   h = ([b ; (β - a.b)/ν] - H_j a)/ν   (stored as the provisional column j of H)
// and p_{j+1} = Z q_j - Q_{j+1} h = (w - Q_{j+1} Q_{j+1}^T w)/ν
//            = w/ν - (r_j/ν) p_j - Q_j (r_{0:j} - a r_j/ν),  r = Q_{j+1}^T w/ν = [b/ν ; (β - a.b)/ν²].
// Pass B coefficients: q_j = cq_p p_j + Σ cq_i q_i, p_{j+1} = cp_w w + cp_p p_j + Σ cp_i q_i.
// Breakdown (invariant Krylov space): ν <= btol ||Z q_{j-1}||  ->  keff = j, column zeroed after.
// reorth = 0 drops the delayed correction (a := 0): single classical Gram-Schmidt.
__global__ void dcgs2_coeffs_kernel(const double* sums, int j, int B, int K, double btol, int final_pass,
                                    int reorth, double* H, double* ref, double* n0, int* keff, double* coef_v,
                                    double* coef_s) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= B) return;
  double* Hc = H + (int64_t)c * (K + 1) * K;  // (row i, col l) at Hc[l*(K+1) + i]
  auto S = [&](int k) {  // a_i entries (even k < 2j) vanish without reorthogonalisation
    return (!reorth && k < 2 * j && (k & 1) == 0) ? 0.0 : sums[(int64_t)k * B + c];
  };
  const double alpha = S(2 * j), beta = S(2 * j + 1), gamma = S(2 * j + 2);
  bool alive;
  double nu;
  if (j == 0) {
    nu = sqrt(alpha);
    alive = nu > 0.0;
    n0[c] = nu;
    keff[c] = alive ? K : 0;
  } else {
    alive = keff[c] == K;
    double aa = 0.0;
    for (int i = 0; i < j; ++i) aa += S(2 * i) * S(2 * i);
    nu = sqrt(fmax(alpha - aa, 0.0));
    if (alive) {
      for (int i = 0; i < j; ++i) Hc[(j - 1) * (K + 1) + i] += S(2 * i);
      if (nu > btol * ref[c] && nu > 0.0) {
        Hc[(j - 1) * (K + 1) + j] = nu;
      } else {
        Hc[(j - 1) * (K + 1) + j] = 0.0;
        keff[c] = j;
        alive = false;
      }
    }
  }
  const int nq = j;
  auto zero = [&]() {
    for (int i = 0; i < nq; ++i) {
      coef_v[(2 * i) * B + c] = 0.0;
      coef_v[(2 * i + 1) * B + c] = 0.0;
    }
    coef_s[c] = 0.0;
    coef_s[B + c] = 0.0;
    coef_s[2 * B + c] = 0.0;
  };
  if (final_pass) return;
  if (!alive) {
    zero();
    return;
  }
  // (H_j a)_i for i <= j, H_j = columns 0..j-1 (rows 0..j)
  double Ha[kMaxKrylov + 1];
  double ab = 0.0;
  for (int i = 0; i <= j; ++i) Ha[i] = 0.0;
  for (int l = 0; l < j; ++l) {
    const double al = S(2 * l);
    ab += al * S(2 * l + 1);
    for (int i = 0; i <= l + 1 && i <= j; ++i) Ha[i] += Hc[l * (K + 1) + i] * al;
  }
  const double inv = 1.0 / nu;
  const double qw = (beta - ab) * inv;
  double* hcol = Hc + (int64_t)j * (K + 1);
  for (int i = 0; i <= j; ++i)  // provisional column j (completed by step j+1's correction)
    if (j < K) hcol[i] = ((i < j ? S(2 * i + 1) : qw) - Ha[i]) * inv;
  // r = H_j a/ν + h = Q_{j+1}^T w / ν = [b/ν ; qw/ν]:  p_{j+1} = (w - Q_{j+1} Q_{j+1}^T w)/ν
  const double rj = qw * inv;
  for (int i = 0; i < j; ++i) {
    const double ai = S(2 * i);
    coef_v[(2 * i) * B + c] = -ai * inv;
    coef_v[(2 * i + 1) * B + c] = -(S(2 * i + 1) * inv - ai * rj * inv);
  }
  coef_s[c] = inv;
  coef_s[B + c] = -rj * inv;
  coef_s[2 * B + c] = inv;
  ref[c] = sqrt(gamma) * inv;
}

inline int grid_for(int64_t total, int bs = 256) {
  int64_t g = (total + bs - 1) / bs;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)num_sms() * 8));
}

// loopback allreduce: dst = Σ_r src_r in rank order (bitwise identical on every rank)
__global__ void sum_ranks_kernel(const SumSrc src, int P, int64_t count, double* dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    double v = src.p[0][i];
    for (int r = 1; r < P; ++r) v += src.p[r][i];
    dst[i] = v;
  }
}

}  // namespace

void batch_inputs(const double* V, int64_t ldv, int B, int64_t n, double* Vb, const int* vcol,
                  const int32_t* perm, cudaStream_t s) {
  WL_LAUNCH("batch_inputs");
  batch_inputs_kernel<<<grid_for(n * B), 256, 0, s>>>(V, ldv, B, n, Vb, vcol, perm);
  WL_CUDA(cudaGetLastError());
}

void seed_expand(const double* s1, const double* s2, const double* v, int b, const int32_t* rowptr, const double* g1s,
                 const int* vcol, int B, int64_t n, double* t0, double* b0, cudaStream_t s, bool f32) {
  WL_LAUNCH("batch_inputs");
  if (f32)
    seed_expand_kernel<float><<<grid_for(n * B), 256, 0, s>>>(s1, s2, v, b, rowptr, g1s, vcol, B, n,
                                                              reinterpret_cast<float*>(t0), reinterpret_cast<float*>(b0));
  else
    seed_expand_kernel<double><<<grid_for(n * B), 256, 0, s>>>(s1, s2, v, b, rowptr, g1s, vcol, B, n, t0, b0);
  WL_CUDA(cudaGetLastError());
}

void setup_chunk(const double* mu, int gstart, int b, int B, double* g0z, double* g1z, double* g0s,
                 double* g1s, int* vcol, int* tcol, cudaStream_t s) {
  WL_LAUNCH("setup_chunk");
  setup_chunk_kernel<<<1, 32, 0, s>>>(mu, gstart, b, B, g0z, g1z, g0s, g1s, vcol, tcol);
  WL_CUDA(cudaGetLastError());
}

void combine(int mode, double lscale, const VecPtrs& Q, int nvec, int64_t n, int B,
                 const double* comb, const double* V, int64_t ldv, const int* vcol, double c0,
                 const double* tprime, int64_t ldt, const int* tcol, double* out, int64_t ldo,
                 const int32_t* perm, cudaStream_t s, bool f32, int64_t nq) {
  WL_LAUNCH("combine");
  if (nq < 0) nq = n;
  const int g = grid_for(n * B);
#define WL_COMBINE(NV, T) \
  combine_kernel<NV, T><<<g, 256, 0, s>>>(mode, lscale, Q, nvec, n, B, comb, V, ldv, vcol, c0, tprime, ldt, tcol, out, ldo, perm, nq)
  if (f32) {
    if (nvec <= 16) WL_COMBINE(16, float);
    else if (nvec <= 32) WL_COMBINE(32, float);
    else WL_COMBINE(kMaxKrylov + 2, float);
  } else {
    if (nvec <= 16) WL_COMBINE(16, double);
    else if (nvec <= 32) WL_COMBINE(32, double);
    else WL_COMBINE(kMaxKrylov + 2, double);
  }
#undef WL_COMBINE
  WL_CUDA(cudaGetLastError());
}

namespace {
template <class Ti, class To>
__global__ void repack_rows_kernel(const Ti* src, int64_t lds, int64_t n, int B, To* dst, int64_t ldd, int zpad) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * B; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / B;
    const int c = (int)(e - r * B);
    dst[r * ldd + c] = (To)src[r * lds + c];
    if (c == B - 1)
      for (int cc = B; cc < zpad; ++cc) dst[r * ldd + cc] = To(0);
  }
}
}  // namespace

void repack_rows(const double* src, int64_t lds, int64_t n, int B, double* dst, int64_t ldd, cudaStream_t s) {
  if (n <= 0) return;
  WL_LAUNCH("repack_rows");
  repack_rows_kernel<double, double><<<grid_for(n * B), 256, 0, s>>>(src, lds, n, B, dst, ldd, 0);
  WL_CUDA(cudaGetLastError());
}

void repack_rows_t(const void* src, bool src_f32, int64_t lds, int64_t n, int B, void* dst, bool dst_f32, int64_t ldd,
                   int zpad, cudaStream_t s) {
  if (n <= 0) return;
  WL_LAUNCH("repack_rows");
  const int g = grid_for(n * B);
  if (src_f32 && dst_f32)
    repack_rows_kernel<float, float><<<g, 256, 0, s>>>((const float*)src, lds, n, B, (float*)dst, ldd, zpad);
  else if (!src_f32 && dst_f32)
    repack_rows_kernel<double, float><<<g, 256, 0, s>>>((const double*)src, lds, n, B, (float*)dst, ldd, zpad);
  else if (!src_f32 && !dst_f32)
    repack_rows_kernel<double, double><<<g, 256, 0, s>>>((const double*)src, lds, n, B, (double*)dst, ldd, zpad);
  else
    throw Error(1, "repack_rows_t: float -> double not used");
  WL_CUDA(cudaGetLastError());
}

void sum_ranks(const SumSrc& src, int P, int64_t count, double* dst, cudaStream_t s) {
  if (count <= 0) return;
  WL_LAUNCH("allreduce_sum");
  sum_ranks_kernel<<<grid_for(count), 256, 0, s>>>(src, P, count, dst);
  WL_CUDA(cudaGetLastError());
}

void pack_rows(const double* src, int64_t lds, const int32_t* idx, int64_t cnt, int B, double* dst,
               cudaStream_t s) {
  if (cnt <= 0) return;
  WL_LAUNCH("pack_rows");
  pack_rows_kernel<double><<<grid_for(cnt * B), 256, 0, s>>>(src, lds, idx, cnt, B, dst);
  WL_CUDA(cudaGetLastError());
}

void pack_rows_f32(const float* src, int64_t lds, const int32_t* idx, int64_t cnt, int B, float* dst, cudaStream_t s) {
  if (cnt <= 0) return;
  WL_LAUNCH("pack_rows");
  pack_rows_kernel<float><<<grid_for(cnt * B), 256, 0, s>>>(src, lds, idx, cnt, B, dst);
  WL_CUDA(cudaGetLastError());
}

namespace {
__global__ void clamp_keff_kernel(const int* keff, int m, int B, int* out, int* flag) {
  const int c = threadIdx.x;
  if (c < B) out[c] = min(keff[c], m);
  if (c < 4) flag[c] = 0;
}
}  // namespace

void clamp_keff(const int* keff, int m, int B, int* out, int* flag, cudaStream_t s) {
  WL_LAUNCH("krylov_check");
  clamp_keff_kernel<<<1, 32, 0, s>>>(keff, m, B, out, flag);
  WL_CUDA(cudaGetLastError());
}

void krylov_check(const double* err, int B, double tol, int* flag, cudaStream_t s) {
  WL_LAUNCH("krylov_check");
  krylov_check_kernel<<<1, 32, 0, s>>>(err, B, tol, flag);
  WL_CUDA(cudaGetLastError());
}

void gather_col(const double* src, int64_t lds, const int32_t* perm, int64_t n, double* dst, cudaStream_t s) {
  WL_LAUNCH("markov_vec");
  if (n <= 0) return;
  gather_col_kernel<<<grid_for(n), 256, 0, s>>>(src, lds, perm, n, dst);
  WL_CUDA(cudaGetLastError());
}

void scatter_col(const double* src, const int32_t* perm, int64_t n, double* dst, int64_t ldd, cudaStream_t s) {
  WL_LAUNCH("markov_vec");
  if (n <= 0) return;
  scatter_col_kernel<<<grid_for(n), 256, 0, s>>>(src, perm, n, dst, ldd);
  WL_CUDA(cudaGetLastError());
}

void markov_scale(const double* p, const double* tprime, int64_t ldt, int tcol, double c0, int64_t n, double* v,
                  cudaStream_t s) {
  WL_LAUNCH("markov_vec");
  if (n <= 0) return;
  markov_scale_kernel<<<grid_for(n), 256, 0, s>>>(p, tprime, ldt, tcol, c0, n, v);
  WL_CUDA(cudaGetLastError());
}

void fill_hash(double* p, int64_t n, uint64_t seed, int64_t i0, cudaStream_t s) {
  WL_LAUNCH("fill");
  if (n <= 0) return;
  fill_hash_kernel<<<grid_for(n), 256, 0, s>>>(p, n, seed, i0);
  WL_CUDA(cudaGetLastError());
}

void fill(double* p, int64_t n, double v, cudaStream_t s) {
  if (n <= 0) return;
  WL_LAUNCH("fill");
  fill_kernel<<<grid_for(n), 256, 0, s>>>(p, n, v);
  WL_CUDA(cudaGetLastError());
}

void lanczos_combine(const double* Q, int64_t stride, int m, int64_t n, const double* Y, int nt,
                     double scale, double* X, int64_t ldx, const int32_t* perm, cudaStream_t s) {
  WL_LAUNCH("lanczos_combine");
  const size_t smem = sizeof(double) * (size_t)m * nt;
  if (smem > 200 * 1024) throw Error(1, "lanczos_combine: k_out * nt too large");
  if (smem > 48 * 1024)
    WL_CUDA(cudaFuncSetAttribute(lanczos_combine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
  lanczos_combine_kernel<<<grid_for(n), 256, smem, s>>>(Q, stride, m, n, Y, nt, scale, X, ldx, perm);
  WL_CUDA(cudaGetLastError());
}

void dcgs2_coeffs(const double* sums, int j, int B, int K, double btol, int final_pass, int reorth, double* H,
                  double* ref, double* n0, int* keff, double* coef_v, double* coef_s, cudaStream_t s) {
  WL_LAUNCH("dcgs2_coeffs");
  dcgs2_coeffs_kernel<<<1, 32, 0, s>>>(sums, j, B, K, btol, final_pass, reorth, H, ref, n0, keff, coef_v,
                                       coef_s);
  WL_CUDA(cudaGetLastError());
}

}  // namespace wl

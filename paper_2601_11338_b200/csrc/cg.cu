// cg.cu — resolvent Laplacian by preconditioned conjugate gradients.
//
// For the resolvent weights c_k = α^k the operator has the closed form (derived from eq:qrec; at
// μ = 1 it is eq:deformed)
//     φ_θ = (1 - μ²α²) 𝒜_θ(α)^{-1},   𝒜_θ(α) = (1 - μ²α²) I - α A + μα² D,
// so 𝕃_θ V = diag(φ_θ 1) V - φ_θ V needs solves with the deformed Laplacian 𝒜_θ(α), which is SPD
// when α ρ(Z_θ) < 1 (Prop. prop:CGworks).  The paper solves them by CG with an AMG preconditioner
// (§4.2, §5.3, tol 1e-9); here Jacobi (diag 𝒜 = (1 - μ²α²) + μα² d_i).
// The product 𝒜 p is the SpMM kernel of spmv.cu with per-column (g0, g1, scale) = (-(1-μ²α²)/α,
// -μα, -α):  scale (A p + (g0 + g1 d) p) = 𝒜 p.
//
// B columns (θ, input-column pairs) iterate together; each column has its own scalars and stops
// (α_k = 0) once ||r|| <= tol ||b||.  Vector kernels: thread t of a block owns column t % B
// (threads per block and the grid stride are multiples of B); per-CTA partial sums are reduced
// by reduce_partials (gram.cu) in a fixed order: deterministic.
#include "wl_internal.cuh"

#include <algorithm>

namespace wl {
namespace {

constexpr int kThreads = 256;
constexpr int kSlots = 4;  // scalar slots per column: rz, alpha, beta, active

// per-column constants: cs[c*8 + k], k: 0 d0 = 1-μ²α², 1 d1 = μα², 2 g0, 3 g1, 4 scale, 5 tol²
__global__ void cg_setup_kernel(const double* mu, double alpha, double tol, int gstart, int b, int B, double* cs,
                                double* g0, double* g1, double* scale, int* vcol, int* tcol) {
  const int c = threadIdx.x;
  if (c >= B) return;
  const int g = gstart + c;
  const double m = mu[g / b];
  const double d0 = 1.0 - m * m * alpha * alpha, d1 = m * alpha * alpha;
  cs[c * 8 + 0] = d0;
  cs[c * 8 + 1] = d1;
  cs[c * 8 + 5] = tol * tol;
  g0[c] = -d0 / alpha;
  g1[c] = -m * alpha;
  scale[c] = -alpha;
  vcol[c] = g % b;
  tcol[c] = g / b;
}

struct Lane {
  int tpb, c;
  bool act;
  int64_t e0, stride;
  __device__ Lane(int B) {
    tpb = blockDim.x / B * B;
    act = (int)threadIdx.x < tpb;
    c = threadIdx.x % B;
    e0 = (int64_t)blockIdx.x * tpb + threadIdx.x;
    stride = (int64_t)gridDim.x * tpb;
  }
};

// block sums of NV per-thread values by column -> partials[(v*B + c) * grid + block]
template <int NV>
__device__ void block_partials(const double (&v)[NV], int B, int tpb, double* partials) {
  __shared__ double red[NV][kThreads];
#pragma unroll
  for (int k = 0; k < NV; ++k) red[k][threadIdx.x] = (int)threadIdx.x < tpb ? v[k] : 0.0;
  __syncthreads();
  for (int idx = threadIdx.x; idx < NV * B; idx += blockDim.x) {
    const int k = idx / B, c = idx - k * B;
    double s = 0.0;
    for (int t = c; t < tpb; t += B) s += red[k][t];
    partials[(int64_t)idx * gridDim.x + blockIdx.x] = s;
  }
}

__device__ inline double dinv(const int32_t* rowptr, int64_t row, const double* cs, int c) {
  const double d = (double)(__ldg(rowptr + row + 1) - __ldg(rowptr + row));
  return 1.0 / (cs[c * 8 + 0] + cs[c * 8 + 1] * d);
}

// x = 0, r = b, p = z = M^{-1} r;  sums: [r.z, b.b]
__global__ void __launch_bounds__(kThreads) cg_init_kernel(CgArgs a) {
  const Lane L(a.B);
  double v[2] = {0.0, 0.0};
  const int64_t N = a.n * a.B;
  if (L.act)
    for (int64_t e = L.e0; e < N; e += L.stride) {
      const double bv = a.b[e];
      const double z = bv * dinv(a.rowptr, e / a.B, a.cs, L.c);
      a.x[e] = 0.0;
      a.r[e] = bv;
      a.p[e] = z;
      v[0] += bv * z;
      v[1] += bv * bv;
    }
  block_partials<2>(v, a.B, L.tpb, a.partials);
}

// sums: [p.q]
__global__ void __launch_bounds__(kThreads) cg_dot_kernel(CgArgs a) {
  if (a.flags[1] == 0) return;  // every column converged: the rest of the check interval is empty
  const Lane L(a.B);
  double v[1] = {0.0};
  const int64_t N = a.n * a.B;
  if (L.act)
    for (int64_t e = L.e0; e < N; e += L.stride) v[0] += a.p[e] * a.q[e];
  block_partials<1>(v, a.B, L.tpb, a.partials);
}

// x += α p, r -= α q;  sums: [r.z, r.r] with z = M^{-1} r
__global__ void __launch_bounds__(kThreads) cg_update_kernel(CgArgs a) {
  if (a.flags[1] == 0) return;
  const Lane L(a.B);
  double v[2] = {0.0, 0.0};
  const int64_t N = a.n * a.B;
  if (L.act) {
    const double al = a.sc[L.c * kSlots + 1];
    for (int64_t e = L.e0; e < N; e += L.stride) {
      const double r = a.r[e] - al * a.q[e];
      a.x[e] += al * a.p[e];
      a.r[e] = r;
      v[0] += r * r * dinv(a.rowptr, e / a.B, a.cs, L.c);
      v[1] += r * r;
    }
  }
  block_partials<2>(v, a.B, L.tpb, a.partials);
}

// p = M^{-1} r + β p
__global__ void __launch_bounds__(kThreads) cg_direction_kernel(CgArgs a) {
  if (a.flags[1] == 0) return;
  const Lane L(a.B);
  const int64_t N = a.n * a.B;
  if (!L.act) return;
  const double be = a.sc[L.c * kSlots + 2];
  for (int64_t e = L.e0; e < N; e += L.stride)
    a.p[e] = a.r[e] * dinv(a.rowptr, e / a.B, a.cs, L.c) + be * a.p[e];
}

// scalar steps, one thread per column.
//   which 0 (after init):   rz = sums[0], bb = sums[1]; active = bb > 0
//   which 1 (after dot):    α = active ? rz / pq : 0 (pq <= 0: not SPD -> diverged flag)
//   which 2 (after update): β = rz_new / rz, rz = rz_new; converged when r.r <= tol² b.b
__device__ void scalar_step(int which, const double* sums, int B, double* sc, double* bb, const double* cs,
                            int* iters, int* flags) {
  const int c = threadIdx.x;
  if (c < B) {
    double* s = sc + c * kSlots;
    if (which == 0) {
      s[0] = sums[c];
      bb[c] = sums[B + c];
      s[3] = bb[c] > 0.0 ? 1.0 : 0.0;
      s[1] = 0.0;
      s[2] = 0.0;
      iters[c] = 0;
    } else if (which == 1) {
      const double pq = sums[c];
      s[1] = 0.0;
      if (s[3] != 0.0) {
        if (!(pq > 0.0)) {
          atomicOr(flags, 1);  // 𝒜 not positive definite on this Krylov space
          s[3] = 0.0;
        } else {
          s[1] = s[0] / pq;
        }
      }
    } else {
      s[2] = 0.0;
      if (s[3] != 0.0) {
        const double rz = sums[c], rr = sums[B + c];
        s[2] = rz / s[0];
        s[0] = rz;
        iters[c] += 1;
        if (rr <= cs[c * 8 + 5] * bb[c]) s[3] = 0.0;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // number of still-active columns: read by the vector kernels and the host check
    int act = 0;
    for (int k = 0; k < B; ++k) act += sc[k * kSlots + 3] != 0.0;
    flags[1] = act;
  }
}

// scalar steps, one thread per column.
//   which 0 (after init):   rz = sums[0], bb = sums[1]; active = bb > 0
//   which 1 (after dot):    α = active ? rz / pq : 0 (pq <= 0: not SPD -> diverged flag)
//   which 2 (after update): β = rz_new / rz, rz = rz_new; converged when r.r <= tol² b.b
__global__ void cg_scalar_kernel(int which, const double* sums, int B, double* sc, double* bb, const double* cs,
                                 int* iters, int* flags) {
  if (which != 0 && flags[1] == 0) return;
  scalar_step(which, sums, B, sc, bb, cs, iters, flags);
}

// single-GPU fusion of reduce_partials + cg_scalar: one CTA sums the <= 64 partial rows (warp per
// row, lanes over the CTAs, fixed shuffle tree) and then takes the scalar step.
__global__ void __launch_bounds__(256) cg_reduce_scalar_kernel(int which, int nout, int G, CgArgs a) {
  if (which != 0 && a.flags[1] == 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int ic = warp; ic < nout; ic += blockDim.x / 32) {
    const double* p = a.partials + (int64_t)ic * G;
    double s0 = 0.0, s1 = 0.0;
    int g = lane;
    for (; g + 32 < G; g += 64) {
      s0 += p[g];
      s1 += p[g + 32];
    }
    if (g < G) s0 += p[g];
    double v = s0 + s1;
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) a.sums[ic] = v;
  }
  __syncthreads();
  scalar_step(which, a.sums, a.B, a.sc, a.bb, a.cs, a.iters, a.flags);
}

// out (user order) from the solution x = 𝒜^{-1} b:  φ b = (1-μ²α²) x
//   mode 0: out = φ V;  mode 1: out = (t' + c0) ⊙ V - φ V;  mode 2 (V = 1): t' = φ 1 - c0 (internal order)
__global__ void cg_combine_kernel(int mode, double lscale, const double* x, int64_t n, int B, const double* cs, const double* V,
                                  int64_t ldv, const int* vcol, double c0, const double* tprime, int64_t ldt,
                                  const int* tcol, double* out, int64_t ldo, const int32_t* perm, int64_t nx) {
  const int64_t N = n * B;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < N; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / B;
    const int c = (int)(e - r * B);
    const int64_t ru = perm ? perm[r] : r;
    const double v = V ? V[ru * ldv + vcol[c]] : 1.0;
    // rows >= nx (isolated: 𝒜 = (1 - μ²α²) I there) were not solved: φ v = (1 - μ²α²) v / (1 - μ²α²) = v
    const double ph = r < nx ? cs[c * 8 + 0] * x[e] : v;
    if (mode == 2) {
      out[r * ldo + c] = ph - c0;
      continue;
    }
    out[ru * ldo + c] = mode == 0 ? ph : lscale * ((tprime[r * ldt + tcol[c]] + c0) * v - ph);
  }
}

int vec_grid(int64_t n, int B) {
  const int tpb = kThreads / B * B;
  const int64_t need = (n * B + tpb - 1) / tpb;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)num_sms() * 6));
}

}  // namespace

void cg_setup(const double* mu, double alpha, double tol, int gstart, int b, int B, double* cs, double* g0,
              double* g1, double* scale, int* vcol, int* tcol, cudaStream_t s) {
  WL_LAUNCH("cg_setup");
  cg_setup_kernel<<<1, 32, 0, s>>>(mu, alpha, tol, gstart, b, B, cs, g0, g1, scale, vcol, tcol);
  WL_CUDA(cudaGetLastError());
}

int cg_grid(int64_t n, int B) { return vec_grid(n, B); }

void cg_init(CgArgs a, cudaStream_t s) {
  WL_LAUNCH("cg_vec");
  cg_init_kernel<<<vec_grid(a.n, a.B), kThreads, 0, s>>>(a);
  WL_CUDA(cudaGetLastError());
}

void cg_dot(CgArgs a, cudaStream_t s) {
  WL_LAUNCH("cg_vec");
  cg_dot_kernel<<<vec_grid(a.n, a.B), kThreads, 0, s>>>(a);
  WL_CUDA(cudaGetLastError());
}

void cg_update(CgArgs a, cudaStream_t s) {
  WL_LAUNCH("cg_vec");
  cg_update_kernel<<<vec_grid(a.n, a.B), kThreads, 0, s>>>(a);
  WL_CUDA(cudaGetLastError());
}

void cg_reduce_scalar(int which, const CgArgs& a, cudaStream_t s) {
  WL_LAUNCH("cg_scalar");
  const int nout = (which == 1 ? 1 : 2) * a.B;
  cg_reduce_scalar_kernel<<<1, 256, 0, s>>>(which, nout, vec_grid(a.n, a.B), a);
  WL_CUDA(cudaGetLastError());
}

void cg_reduce(int which, const CgArgs& a, cudaStream_t s) {
  WL_LAUNCH("cg_scalar");
  reduce_partials(a.partials, (which == 1 ? 1 : 2) * a.B, vec_grid(a.n, a.B), a.sums, s);
}

void cg_direction(CgArgs a, cudaStream_t s) {
  WL_LAUNCH("cg_vec");
  cg_direction_kernel<<<vec_grid(a.n, a.B), kThreads, 0, s>>>(a);
  WL_CUDA(cudaGetLastError());
}

void cg_scalar(int which, const CgArgs& a, cudaStream_t s) {
  WL_LAUNCH("cg_scalar");
  cg_scalar_kernel<<<1, 32, 0, s>>>(which, a.sums, a.B, a.sc, a.bb, a.cs, a.iters, a.flags);

  WL_CUDA(cudaGetLastError());
}

void cg_combine(int mode, double lscale, const double* x, int64_t n, int B, const double* cs, const double* V, int64_t ldv,
                const int* vcol, double c0, const double* tprime, int64_t ldt, const int* tcol, double* out,
                int64_t ldo, const int32_t* perm, cudaStream_t s, int64_t nx) {
  if (nx < 0) nx = n;
  WL_LAUNCH("cg_combine");
  const int64_t N = n * B;
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>((N + 255) / 256, (int64_t)num_sms() * 8));
  cg_combine_kernel<<<g, 256, 0, s>>>(mode, lscale, x, n, B, cs, V, ldv, vcol, c0, tprime, ldt, tcol, out, ldo, perm, nx);
  WL_CUDA(cudaGetLastError());
}

}  // namespace wl

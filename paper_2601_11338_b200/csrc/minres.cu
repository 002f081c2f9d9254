// minres.cu — shifted solves (𝔏 − ξI) X = U of the block rational Krylov method.
//
// Alg. 1 (alg:trace_estimation) builds a block rational Krylov space; "the construction of
// the basis vectors requires the solution of linear systems with matrix μ_k 𝔏 − ν_k I ... we only have
// access to routines that allow us to perform the matrix-vector product ... we can rely again on the
// use of a Krylov-type method for the solution of linear systems" (the paper used GMRES,
// tol 1e-6).  𝔏 = 𝕃_θ is symmetric (Prop. pro:still-again-an-mmatrix), so MINRES applies:
//   * real ξ:          S = 𝔏 − ξI (symmetric, indefinite when ξ lies in the spectrum's range)
//   * ξ = a + ib:      (𝔏 − ξI)(x_r + i x_i) = u in real form, second row negated to make it symmetric:
//                          S = [[𝔏 − aI,  bI], [bI, −(𝔏 − aI)]],  S [x_r; x_i] = [u; 0]
// MINRES (Paige–Saunders; the recurrence of van der Vorst, Iterative Krylov Methods §6.4):
//   Lanczos:  α_j = v_jᵀ S v_j,  v̂ = S v_j − α_j v_j − β_j v_{j−1},  β_{j+1} = ‖v̂‖
//   QR:       δ = γ_j α_j − γ_{j−1} σ_j β_j,  ρ1 = √(δ² + β_{j+1}²),  ρ2 = σ_j α_j + γ_{j−1} γ_j β_j,
//             ρ3 = σ_{j−1} β_j,  γ_{j+1} = δ/ρ1,  σ_{j+1} = β_{j+1}/ρ1
//   update:   w_j = (v_j − ρ3 w_{j−2} − ρ2 w_{j−1})/ρ1,  x_j = x_{j−1} + γ_{j+1} η w_j,
//             ‖r_j‖ = |σ_{j+1}| ‖r_{j−1}‖,  η ← −σ_{j+1} η
// Every column of the n × M block has its own scalars and stops at ‖r‖ <= tol ‖u‖.  The product S v is
// one batched Laplacian action (the whole hot path: Krylov on Z + combine) on the real and imaginary
// halves, done by the engine; the kernels here form S v from it and run the recurrence.  Vector
// kernels: thread t owns column t % M; per-CTA partial sums are reduced in a fixed order.
#include "wl_internal.cuh"

#include <algorithm>

namespace wl {
namespace {

constexpr int kThreads = 256;

struct MrLane {
  int tpb, c;
  bool act;
  int64_t e0, stride;
  __device__ explicit MrLane(int B) {
    tpb = blockDim.x / B * B;
    act = (int)threadIdx.x < tpb;
    c = threadIdx.x % B;
    e0 = (int64_t)blockIdx.x * tpb + threadIdx.x;
    stride = (int64_t)gridDim.x * tpb;
  }
};

// block sums of NV per-thread values by column -> partials[(v*B + c) * grid + block]
template <int NV>
__device__ void mr_partials(const double (&v)[NV], int B, int tpb, double* partials) {
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

// scalar slots per column (MinresArgs::sc): 0 β_j, 1 α_j, 2 γ_{j-1}, 3 γ_j, 4 σ_{j-1}, 5 σ_j, 6 η,
// 7 ‖r‖, 8 ‖u‖, 9 active, 10 ρ1, 11 ρ2, 12 ρ3, 13 x coefficient γ_{j+1} η, 14 1/β_{j+1}, 15 iterations
constexpr int kS = 16;

// sums: ‖u‖² (the right-hand side is [u; 0])
__global__ void __launch_bounds__(kThreads) mr_norm_kernel(MinresArgs a) {
  const MrLane L(a.B);
  double v[1] = {0.0};
  const int64_t N = a.n * a.B;
  if (L.act)
    for (int64_t e = L.e0; e < N; e += L.stride) v[0] += a.u[e] * a.u[e];
  mr_partials<1>(v, a.B, L.tpb, a.partials);
}

// v = u / ‖u‖, v_prev = w1 = w2 = x = 0 (real and imaginary halves)
__global__ void __launch_bounds__(kThreads) mr_init_kernel(MinresArgs a) {
  const MrLane L(a.B);
  if (!L.act) return;
  const double s = a.sc[L.c * kS + 8] > 0.0 ? 1.0 / a.sc[L.c * kS + 8] : 0.0;
  const int64_t N = a.n * a.B;
  for (int64_t e = L.e0; e < N; e += L.stride) {
    a.v[e] = a.u[e] * s;
    a.vp[e] = a.w1[e] = a.w2[e] = a.x[e] = 0.0;
    if (a.cplx) a.v[N + e] = a.vp[N + e] = a.w1[N + e] = a.w2[N + e] = a.x[N + e] = 0.0;
  }
}

// p (holding 𝔏 v on entry) <- S v;  sums: α = vᵀ S v
__global__ void __launch_bounds__(kThreads) mr_alpha_kernel(MinresArgs a) {
  if (*a.nactive == 0) return;
  const MrLane L(a.B);
  double v[1] = {0.0};
  const int64_t N = a.n * a.B;
  if (L.act) {
    const double sa = a.shift_re, sb = a.shift_im;
    for (int64_t e = L.e0; e < N; e += L.stride) {
      if (a.cplx) {
        const double vr = a.v[e], vi = a.v[N + e];
        const double top = a.p[e] - sa * vr + sb * vi;
        const double bot = sb * vr - a.p[N + e] + sa * vi;
        a.p[e] = top;
        a.p[N + e] = bot;
        v[0] += vr * top + vi * bot;
      } else {
        const double vr = a.v[e];
        const double top = a.p[e] - sa * vr;
        a.p[e] = top;
        v[0] += vr * top;
      }
    }
  }
  mr_partials<1>(v, a.B, L.tpb, a.partials);
}

// v̂ = S v − α v − β v_prev, written over v_prev;  sums: ‖v̂‖²
__global__ void __launch_bounds__(kThreads) mr_lanczos_kernel(MinresArgs a) {
  if (*a.nactive == 0) return;
  const MrLane L(a.B);
  double v[1] = {0.0};
  const int64_t N = a.n * a.B * (a.cplx ? 2 : 1);
  if (L.act) {
    const double al = a.sc[L.c * kS + 1], be = a.sc[L.c * kS + 0];
    for (int64_t e = L.e0; e < N; e += L.stride) {
      const double h = a.p[e] - al * a.v[e] - be * a.vp[e];
      a.vp[e] = h;
      v[0] += h * h;
    }
  }
  mr_partials<1>(v, a.B, L.tpb, a.partials);
}

// w_j = (v_j − ρ3 w_{j−2} − ρ2 w_{j−1}) / ρ1 over w_{j−2};  x += γ_{j+1} η w_j;  v_{j+1} = v̂ / β_{j+1} over v̂
__global__ void __launch_bounds__(kThreads) mr_update_kernel(MinresArgs a) {
  if (*a.nactive == 0) return;
  const MrLane L(a.B);
  if (!L.act) return;
  const double* s = a.sc + L.c * kS;
  if (s[9] == 0.0 && s[13] == 0.0) return;  // converged before this iteration: x stays
  const double r1 = 1.0 / s[10], r2 = s[11], r3 = s[12], xc = s[13], ib = s[14];
  const int64_t N = a.n * a.B * (a.cplx ? 2 : 1);
  for (int64_t e = L.e0; e < N; e += L.stride) {
    const double w = (a.v[e] - r3 * a.w2[e] - r2 * a.w1[e]) * r1;
    a.w2[e] = w;
    a.x[e] += xc * w;
    a.vp[e] *= ib;
  }
}

// one CTA: reduce the partial rows (warp per row, fixed order), then the scalar step of every column
//   which 0: ‖u‖ -> β_1 = η = ‖r‖ = ‖u‖, γ = 1, σ = 0, active = ‖u‖ > 0
//   which 1: α
//   which 2: β_{j+1} -> rotations, x coefficient, ‖r‖, η; convergence ‖r‖ <= tol ‖u‖
__global__ void __launch_bounds__(256) mr_scalar_kernel(int which, int G, MinresArgs a) {
  if (which != 0 && *a.nactive == 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int ic = warp; ic < (a.presummed ? 0 : a.B); ic += blockDim.x / 32) {
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
  const int c = threadIdx.x;
  if (c < a.B) {
    double* s = a.sc + c * kS;
    const double v = a.sums[c];
    if (which == 0) {
      const double nu = sqrt(v);
      s[0] = s[6] = s[7] = s[8] = nu;
      s[2] = s[3] = 1.0;
      s[4] = s[5] = 0.0;
      s[9] = nu > 0.0 ? 1.0 : 0.0;
      s[13] = 0.0;
      s[15] = 0.0;
    } else if (which == 1) {
      s[1] = v;
    } else {
      const double bn = sqrt(v), al = s[1], be = s[0];
      if (s[9] != 0.0) {
        const double delta = s[3] * al - s[2] * s[5] * be;
        const double rho1 = hypot(delta, bn);
        s[10] = rho1 > 0.0 ? rho1 : 1.0;
        s[11] = s[5] * al + s[2] * s[3] * be;
        s[12] = s[4] * be;
        const double g2 = rho1 > 0.0 ? delta / rho1 : 1.0, s2 = rho1 > 0.0 ? bn / rho1 : 0.0;
        s[13] = g2 * s[6];
        s[7] = fabs(s2) * s[7];
        s[6] = -s2 * s[6];
        s[2] = s[3];
        s[3] = g2;
        s[4] = s[5];
        s[5] = s2;
        s[15] += 1.0;
        if (s[7] <= a.tol * s[8] || bn == 0.0) s[9] = 0.0;  // converged (or exact: invariant subspace)
      } else {
        s[13] = 0.0;
      }
      s[0] = bn;
      s[14] = bn > 0.0 ? 1.0 / bn : 0.0;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int act = 0;
    for (int k = 0; k < a.B; ++k) act += a.sc[k * kS + 9] != 0.0;
    *a.nactive = act;
  }
}

int mr_grid(int64_t n, int B) {
  const int tpb = kThreads / B * B;
  const int64_t need = (n * B + tpb - 1) / tpb;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)num_sms() * 6));
}

}  // namespace

size_t minres_scalar_doubles(int B) { return (size_t)kS * B; }
int minres_grid(int64_t n, int B) { return mr_grid(n, B); }

// vector phases write per-CTA partials (one row per column, minres_grid CTAs); the scalar phase reduces
// them itself (single GPU) or takes a.sums already reduced and allreduced (a.presummed, multi-rank)
void minres_vec(int phase, const MinresArgs& a, cudaStream_t s) {
  WL_LAUNCH("minres_vec");
  const int G = mr_grid(a.n, a.B);
  if (phase == 0) mr_norm_kernel<<<G, kThreads, 0, s>>>(a);
  else if (phase == 1) mr_init_kernel<<<G, kThreads, 0, s>>>(a);
  else if (phase == 2) mr_alpha_kernel<<<G, kThreads, 0, s>>>(a);
  else if (phase == 3) mr_lanczos_kernel<<<G, kThreads, 0, s>>>(a);
  else mr_update_kernel<<<G, kThreads, 0, s>>>(a);
  WL_CUDA(cudaGetLastError());
}

void minres_scalar(int which, const MinresArgs& a, cudaStream_t s) {
  WL_LAUNCH("minres_scalar");
  mr_scalar_kernel<<<1, 256, 0, s>>>(which, mr_grid(a.n, a.B), a);
  WL_CUDA(cudaGetLastError());
}

}  // namespace wl

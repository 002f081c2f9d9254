// block.cu — the tall-skinny block products of XNysTrace-exp's block Krylov bases (Alg. 1 line 4, P:594-625;
// engine.cu wl_xnystrace_exp / wl_xnystrace_exp_rational): block classical Gram–Schmidt and Cholesky QR need
//   gram:  C = X[:, :p]ᵀ Y[:, :q]              (p x q, column-major, ld p)
//   axpy:  Y[:, :q] = β Y[:, :q] + α X[:, :p] C   (C p x q column-major, ld p)
// for row-major n x p / n x q blocks with p <= 1024 basis columns and q <= 64 (2M, M <= 32).  Both are
// HBM streams of X (the basis) with O(q) flops per loaded element: at q = 64 roughly 16 flop/byte, below
// the fp64 FMA rate of the SMs, so plain register-tiled CUDA-core kernels do; no library GEMM.
// gram is deterministic: per-CTA partial tiles over a fixed row split, reduced in CTA order.
#include "wl_internal.cuh"

#include <algorithm>

namespace wl {
namespace {

constexpr int kT = 64;   // output tile (i and j)
constexpr int kR = 32;   // rows per shared-memory chunk
constexpr int kThreads = 256;

// CTA (bx, by): rows [bx * rpc, (bx + 1) * rpc), output rows i in [by * 64, by * 64 + 64), all j < q.
// Thread (ty, tx) of a 16 x 16 grid owns i = i0 + tx + 16a, j = ty + 16b (a, b < 4): X reads are 16 distinct
// consecutive doubles per warp, Y reads a broadcast of two.
__global__ void __launch_bounds__(kThreads) block_gram_kernel(int p, int q, int64_t n, const double* X, int64_t ldx,
                                                              const double* Y, int64_t ldy, int64_t rpc,
                                                              double* part) {
  __shared__ double Xs[kR][kT], Ys[kR][kT];
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
  const int i0 = blockIdx.y * kT;
  const int64_t r0 = (int64_t)blockIdx.x * rpc, r1 = r0 + rpc < n ? r0 + rpc : n;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int64_t rc = r0; rc < r1; rc += kR) {
#pragma unroll
    for (int k = 0; k < kR * kT / kThreads; ++k) {
      const int e = t + k * kThreads, rr = e / kT, c = e % kT;
      const int64_t r = rc + rr;
      Xs[rr][c] = (r < r1 && i0 + c < p) ? X[r * ldx + i0 + c] : 0.0;
      Ys[rr][c] = (r < r1 && c < q) ? Y[r * ldy + c] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int rr = 0; rr < kR; ++rr) {
      double xv[4], yv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) xv[a] = Xs[rr][tx + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) yv[b] = Ys[rr][ty + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] += xv[a] * yv[b];
    }
    __syncthreads();
  }
  double* out = part + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * (kT * kT);
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) out[(tx + 16 * a) * kT + ty + 16 * b] = acc[a][b];
}

// C[j * p + i] = Σ_cta part[(i / 64, cta)][i % 64][j], in CTA order
__global__ void block_gram_reduce(int p, int q, int G, const double* part, double* C) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)p * q) return;
  const int i = (int)(e % p), j = (int)(e / p);
  const double* src = part + (int64_t)(i / kT) * G * (kT * kT) + (i % kT) * kT + j;
  double s = 0.0;
  for (int g = 0; g < G; ++g) s += src[(int64_t)g * (kT * kT)];
  C[e] = s;
}

// CTA: 32 rows; thread t: column j = t % 64 (active if < q) and rows (t / 64) * 8 .. + 7.  C staged in 64-row
// slices, X rows in 32 x 64 slices: Cs reads are consecutive over the warp, Xs reads broadcasts.
__global__ void __launch_bounds__(kThreads) block_axpy_kernel(int p, int q, int64_t n, double alpha, const double* X,
                                                              int64_t ldx, const double* C, double beta, double* Y,
                                                              int64_t ldy) {
  __shared__ double Cs[kT][kT], Xs[kR][kT];
  const int t = threadIdx.x, j = t % kT, rg = t / kT;
  const int64_t r0 = (int64_t)blockIdx.x * kR;
  double acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = 0.0;
  for (int i0 = 0; i0 < p; i0 += kT) {
#pragma unroll
    for (int k = 0; k < kT * kT / kThreads; ++k) {
      const int e = t + k * kThreads, il = e / kT, jj = e % kT;
      Cs[il][jj] = (i0 + il < p && jj < q) ? C[(int64_t)jj * p + i0 + il] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < kR * kT / kThreads; ++k) {
      const int e = t + k * kThreads, rr = e / kT, c = e % kT;
      const int64_t r = r0 + rr;
      Xs[rr][c] = (r < n && i0 + c < p) ? X[r * ldx + i0 + c] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int il = 0; il < kT; ++il) {
      const double c = Cs[il][j];
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] += Xs[rg * 8 + k][il] * c;
    }
    __syncthreads();
  }
  if (j >= q) return;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int64_t r = r0 + rg * 8 + k;
    if (r < n) {
      double* y = Y + r * ldy + j;
      *y = (beta == 0.0 ? 0.0 : beta * *y) + alpha * acc[k];
    }
  }
}

int gram_rows_grid(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(num_sms(), (n + kR - 1) / kR));
}

}  // namespace

size_t block_gram_partials(int64_t n, int p) {
  return (size_t)((p + kT - 1) / kT) * gram_rows_grid(n) * kT * kT;
}

void block_gram(int p, int q, int64_t n, const double* X, int64_t ldx, const double* Y, int64_t ldy, double* C,
                double* partials, cudaStream_t s) {
  if (p < 1 || q < 1 || q > kT) throw Error(WL_EINVAL, "block_gram: need p >= 1 and 1 <= q <= 64");
  WL_LAUNCH("block_gram");
  const int G = gram_rows_grid(n);
  int64_t rpc = (std::max<int64_t>(n, 1) + G - 1) / G;
  rpc = (rpc + kR - 1) / kR * kR;
  const dim3 grid(G, (p + kT - 1) / kT);
  block_gram_kernel<<<grid, kThreads, 0, s>>>(p, q, n, X, ldx, Y, ldy, rpc, partials);
  WL_CUDA(cudaGetLastError());
  note_launch("block_gram_reduce");
  const int64_t nout = (int64_t)p * q;
  block_gram_reduce<<<(int)((nout + 255) / 256), 256, 0, s>>>(p, q, G, partials, C);
  WL_CUDA(cudaGetLastError());
}

void block_axpy(int p, int q, int64_t n, double alpha, const double* X, int64_t ldx, const double* C, double beta,
                double* Y, int64_t ldy, cudaStream_t s) {
  if (p < 1 || q < 1 || q > kT) throw Error(WL_EINVAL, "block_axpy: need p >= 1 and 1 <= q <= 64");
  if (n <= 0) return;
  WL_LAUNCH("block_axpy");
  block_axpy_kernel<<<(int)((n + kR - 1) / kR), kThreads, 0, s>>>(p, q, n, alpha, X, ldx, C, beta, Y, ldy);
  WL_CUDA(cudaGetLastError());
}

}  // namespace wl

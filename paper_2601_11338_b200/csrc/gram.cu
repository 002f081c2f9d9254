// gram.cu — Arnoldi orthogonalisation kernels (step a5): classical Gram-Schmidt, twice.
//
// The Arnoldi process (Saad Alg. 6.1 as cited there) builds an orthonormal basis of
// K_k(Z, u).  The basis lives in HBM as k+1 row-major n x B blocks per half; columns are
// independent Krylov problems that share every pass over memory.  Vectors are stored
// UNNORMALISED with per-(vector, column) scales s_i = 1/||w_i|| ("normalisation lag"), so the
// final rescale never costs a pass: q_i = s_i * Q_i.
//
// Per Arnoldi step (w = Z q_j, nvec = j+1):
//   gram_proj        sums1_i = Q_i . w,  sums1_nvec = w . w               (1 read of the basis)
//   gram_update_proj w' = w - Σ s_i² sums1_i Q_i ;  sums2_i = Q_i . w'    (1 read; Q_i kept in
//                    registers between the update and the second projection)
//   gram_update_norm w'' = w' - Σ s_i² sums2_i Q_i ; sums3 = w'' . w''    (1 read)
// Reductions are deterministic: per-CTA partials, then the last CTA to finish (atomic ticket)
// sums the partials in CTA order.  Threads own one column each (block = B * m threads and
// a grid-stride that is a multiple of B), so column reductions never mix columns.
#include "wl_internal.cuh"
#include <algorithm>

namespace wl {
namespace {

inline int gram_block(int B) { return B * std::max(1, 256 / B); }

// Block-reduce per-thread values v[0..NV) (only the first nv meaningful) by column and write
// this CTA's partial sums to partials[blockIdx.x * nout + i*B + c] (i < nv).
template <int NV>
__device__ inline void block_partials(const double (&v)[NV], int nv, int B, int nout,
                                      double* partials, double* red /* 8 * blockDim */) {
  const int bs = blockDim.x, tid = threadIdx.x, m = bs / B;
#pragma unroll
  for (int i0 = 0; i0 < NV; i0 += 8) {
    if (i0 < nv) {
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (i0 + q < NV) red[q * bs + tid] = v[(i0 + q < NV) ? i0 + q : 0];
      __syncthreads();
      if (tid < 8 * B) {
        const int q = tid / B, c = tid - q * B;
        if (i0 + q < nv) {
          double s = 0.0;
          for (int k = 0; k < m; ++k) s += red[q * bs + c + k * B];
          partials[(int64_t)blockIdx.x * nout + (i0 + q) * B + c] = s;
        }
      }
      __syncthreads();
    }
  }
}

// Last CTA: sums_out[ic] = Σ_cta partials[cta * nout + ic] (fixed order), then reset ticket.
__device__ inline void last_block_reduce(const double* partials, int nout, double* sums_out,
                                         unsigned int* ticket) {
  __shared__ bool am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) am_last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  const int G = gridDim.x;
  for (int ic = threadIdx.x; ic < nout; ic += blockDim.x) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int g = 0;
    for (; g + 3 < G; g += 4) {
      s0 += __ldcg(partials + (int64_t)(g + 0) * nout + ic);
      s1 += __ldcg(partials + (int64_t)(g + 1) * nout + ic);
      s2 += __ldcg(partials + (int64_t)(g + 2) * nout + ic);
      s3 += __ldcg(partials + (int64_t)(g + 3) * nout + ic);
    }
    for (; g < G; ++g) s0 += __ldcg(partials + (int64_t)g * nout + ic);
    sums_out[ic] = (s0 + s1) + (s2 + s3);
  }
  if (threadIdx.x == 0) *ticket = 0u;
}

__device__ inline double load_w(const GramArgs& a, int64_t e, int64_t splitE, double wsc) {
  return e < splitE ? wsc * __ldg(a.wa + e) : __ldg(a.wb + (e - splitE));
}

// Each thread owns column c = tid % B and visits U elements per iteration, e + u*bs
// (u < U): all in column c, each a coalesced warp access, U independent loads per basis vector.
template <int JT, int U>
__global__ void __launch_bounds__(256) gram_proj_kernel(GramArgs a) {
  __shared__ double red[8 * 256];
  const int B = a.B, tid = threadIdx.x, bs = blockDim.x, c = tid % B;
  const int64_t total = a.len * B, splitE = a.split * B;
  const double wsc = a.wscale ? a.wscale[c] : 1.0;
  const int nvec = a.nvec;
  double acc[JT + 1];
#pragma unroll
  for (int i = 0; i <= JT; ++i) acc[i] = 0.0;
  const int64_t step = (int64_t)gridDim.x * bs * U;
  for (int64_t base = (int64_t)blockIdx.x * bs * U + tid; base < total; base += step) {
    double w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = base + (int64_t)u * bs;
      w[u] = e < total ? load_w(a, e, splitE, wsc) : 0.0;
      acc[JT] += w[u] * w[u];
    }
    double q[JT][U];  // all loads of this iteration in flight before any FMA
    const double* qp = a.Q + base;
#pragma unroll
    for (int i = 0; i < JT; ++i) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        q[i][u] = (i < nvec && base + (int64_t)u * bs < total) ? __ldg(qp + (int64_t)u * bs) : 0.0;
      qp += a.vstride;
    }
#pragma unroll
    for (int i = 0; i < JT; ++i) {
      double sum = 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u) sum += q[i][u] * w[u];
      acc[i] += sum;
    }
  }
  double v[JT + 1];
#pragma unroll
  for (int i = 0; i <= JT; ++i) v[i] = (i < nvec) ? acc[i] : (i == nvec ? acc[JT] : 0.0);
  const int nout = (nvec + 1) * B;
  block_partials<JT + 1>(v, nvec + 1, B, nout, a.partials, red);
  last_block_reduce(a.partials, nout, a.sums_out, a.ticket);
}

template <int JT, int U>
__global__ void __launch_bounds__(256) gram_update_proj_kernel(GramArgs a) {
  __shared__ double red[8 * 256];
  __shared__ double coef[JT * kMaxCols];
  const int B = a.B, tid = threadIdx.x, bs = blockDim.x, c = tid % B;
  for (int idx = tid; idx < a.nvec * B; idx += bs) {
    const double si = a.s[idx];
    coef[idx] = si * si * a.sums_in[idx];
  }
  __syncthreads();
  const int64_t total = a.len * B, splitE = a.split * B;
  const double wsc = a.wscale ? a.wscale[c] : 1.0;
  const int nvec = a.nvec;
  double acc[JT];
#pragma unroll
  for (int i = 0; i < JT; ++i) acc[i] = 0.0;
  const int64_t step = (int64_t)gridDim.x * bs * U;
  for (int64_t base = (int64_t)blockIdx.x * bs * U + tid; base < total; base += step) {
    double q[JT][U];
    const double* qp = a.Q + base;
#pragma unroll
    for (int i = 0; i < JT; ++i) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        q[i][u] = (i < nvec && base + (int64_t)u * bs < total) ? __ldg(qp + (int64_t)u * bs) : 0.0;
      qp += a.vstride;
    }
    double w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = base + (int64_t)u * bs;
      w[u] = e < total ? load_w(a, e, splitE, wsc) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < JT; ++i)
      if (i < nvec) {
        const double ci = coef[i * B + c];
#pragma unroll
        for (int u = 0; u < U; ++u) w[u] -= ci * q[i][u];
      }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = base + (int64_t)u * bs;
      if (e < total) a.wout[e] = w[u];
    }
#pragma unroll
    for (int i = 0; i < JT; ++i) {
      double sum = 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u) sum += q[i][u] * w[u];
      acc[i] += sum;
    }
  }
  const int nout = nvec * B;
  block_partials<JT>(acc, nvec, B, nout, a.partials, red);
  last_block_reduce(a.partials, nout, a.sums_out, a.ticket);
}

template <int JT, int U>
__global__ void __launch_bounds__(256) gram_update_norm_kernel(GramArgs a) {
  __shared__ double red[8 * 256];
  __shared__ double coef[JT * kMaxCols];
  const int B = a.B, tid = threadIdx.x, bs = blockDim.x, c = tid % B;
  for (int idx = tid; idx < a.nvec * B; idx += bs) {
    const double si = a.s[idx];
    coef[idx] = si * si * a.sums_in[idx];
  }
  __syncthreads();
  const int64_t total = a.len * B, splitE = a.split * B;
  const double wsc = a.wscale ? a.wscale[c] : 1.0;
  const int nvec = a.nvec;
  double acc[1] = {0.0};
  const int64_t step = (int64_t)gridDim.x * bs * U;
  for (int64_t base = (int64_t)blockIdx.x * bs * U + tid; base < total; base += step) {
    double w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {  // may alias wout: plain loads
      const int64_t e = base + (int64_t)u * bs;
      w[u] = e < total ? (e < splitE ? wsc * a.wa[e] : a.wb[e - splitE]) : 0.0;
    }
    double q[JT][U];
    const double* qp = a.Q + base;
#pragma unroll
    for (int i = 0; i < JT; ++i) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        q[i][u] = (i < nvec && base + (int64_t)u * bs < total) ? __ldg(qp + (int64_t)u * bs) : 0.0;
      qp += a.vstride;
    }
#pragma unroll
    for (int i = 0; i < JT; ++i) {
      const double ci = (i < nvec) ? coef[i * B + c] : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u) w[u] -= ci * q[i][u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = base + (int64_t)u * bs;
      if (e < total) {
        a.wout[e] = w[u];
        acc[0] += w[u] * w[u];
      }
    }
  }
  const int nout = B;
  block_partials<1>(acc, 1, B, nout, a.partials, red);
  last_block_reduce(a.partials, nout, a.sums_out, a.ticket);
}

}  // namespace

int gram_grid(int64_t elems, int B) {
  const int bs = gram_block(B);
  const int64_t blocks = (elems + 4 * bs - 1) / (4 * bs);
  return (int)std::max<int64_t>(1, std::min<int64_t>(blocks, 148 * 4));
}

#define WL_GRAM_DISPATCH(KERNEL, NV, ...)                                                   \
  do {                                                                                      \
    const int bs_ = gram_block(a.B);                                                        \
    if ((NV) <= 8) KERNEL<8, 4><<<a.grid, bs_, 0, s>>>(__VA_ARGS__);                        \
    else if ((NV) <= 16) KERNEL<16, 4><<<a.grid, bs_, 0, s>>>(__VA_ARGS__);                 \
    else if ((NV) <= 32) KERNEL<32, 2><<<a.grid, bs_, 0, s>>>(__VA_ARGS__);                 \
    else KERNEL<64, 1><<<a.grid, bs_, 0, s>>>(__VA_ARGS__);                                 \
  } while (0)

// Bases longer than 64 vectors (outer diffusion Lanczos) are processed in tiles of 64: tile
// [i0, i1) writes its sums at sums_out + i0*B; its trailing w.w slot is overwritten by the next
// tile, and the last tile leaves w.w at index nvec.
void gram_proj(GramArgs a, cudaStream_t s) {
  if (a.nvec > 64) {
    for (int i0 = 0; i0 < a.nvec; i0 += 64) {
      GramArgs t = a;
      t.nvec = std::min(64, a.nvec - i0);
      t.Q = a.Q + (int64_t)i0 * a.vstride;
      t.sums_out = a.sums_out + (int64_t)i0 * a.B;
      gram_proj(t, s);
    }
    return;
  }
  WL_LAUNCH("gram_proj");
  WL_GRAM_DISPATCH(gram_proj_kernel, a.nvec, a);
  WL_CUDA(cudaGetLastError());
}

void gram_update_proj(GramArgs a, cudaStream_t s) {
  if (a.nvec > 32) throw Error(1, "gram_update_proj: nvec > 32 (use the unfused path)");
  WL_LAUNCH("gram_update_proj");
  const int bs_ = gram_block(a.B);
  if (a.nvec <= 8) gram_update_proj_kernel<8, 4><<<a.grid, bs_, 0, s>>>(a);
  else if (a.nvec <= 16) gram_update_proj_kernel<16, 4><<<a.grid, bs_, 0, s>>>(a);
  else gram_update_proj_kernel<32, 2><<<a.grid, bs_, 0, s>>>(a);
  WL_CUDA(cudaGetLastError());
}

void gram_update_norm(GramArgs a, cudaStream_t s) {
  if (a.nvec > 64) {  // tiles of 64 basis vectors; tiles after the first update wout in place
    for (int i0 = 0; i0 < a.nvec; i0 += 64) {
      GramArgs t = a;
      t.nvec = std::min(64, a.nvec - i0);
      t.Q = a.Q + (int64_t)i0 * a.vstride;
      t.s = a.s + (int64_t)i0 * a.B;
      t.sums_in = a.sums_in + (int64_t)i0 * a.B;
      if (i0 > 0) { t.wa = a.wout; t.wscale = nullptr; t.split = a.len; t.wb = nullptr; }
      gram_update_norm(t, s);
    }
    return;
  }
  WL_LAUNCH("gram_update_norm");
  WL_GRAM_DISPATCH(gram_update_norm_kernel, a.nvec, a);
  WL_CUDA(cudaGetLastError());
}

}  // namespace wl

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
//   gram_update_proj w' = w - Σ s_i² sums1_i Q_i ;  sums2_i = Q_i . w'    (1 read: Q_i stays in
//                    registers between the update and the second projection)
//   gram_update_norm w'' = w' - Σ s_i² sums2_i Q_i ; sums3 = w'' . w''    (1 read)
//
// These are pure HBM streams of nvec+2 vectors.  Design (measured, tools/stream_bench.cu on
// B200: register streaming of 32 concurrent vectors reaches 7.3 TB/s, a 1-CTA/SM bulk-TMA ring is
// capped near 4.6 TB/s by the bytes a 227 KB shared memory can keep in flight for 32 streams):
// the basis vectors are split across thread groups — group g owns vectors [8g, 8g+8) — so a
// thread holds at most 8 accumulators and 8 x U loads in flight at full occupancy.  Update
// kernels combine the groups' partial sums Σ c_i Q_i with warp shuffles.  Threads own one column (slot % B, slots a multiple of B), so column
// reductions never mix columns.  Reductions are deterministic: per-CTA partials, then a reduce kernel
// sums them in a fixed order.
#include "wl_internal.cuh"

#include <algorithm>
#include <cstdlib>

namespace wl {
namespace {

constexpr int kVG = 8;             // basis vectors per thread group
constexpr int kMaxGroups = 4;      // => <= 32 vectors per launch (larger sets are tiled)
constexpr int kMaxVecPerLaunch = kVG * kMaxGroups;
constexpr int kBS = 256;

inline int groups_for(int nvec) { return std::max(1, (nvec + kVG - 1) / kVG); }

// sums_out[ic] = Σ_cta partials[ic * G + cta]: one warp per output, lanes stride over the CTAs
// (coalesced), fixed-order shuffle tree — deterministic for a given grid.
__global__ void reduce_partials_kernel(const double* partials, int nout, int G, double* sums_out) {
  const int ic = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (ic >= nout) return;
  const double* p = partials + (int64_t)ic * G;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int g = lane;
  for (; g + 96 < G; g += 128) {
    s0 += __ldcg(p + g);
    s1 += __ldcg(p + g + 32);
    s2 += __ldcg(p + g + 64);
    s3 += __ldcg(p + g + 96);
  }
  for (; g < G; g += 32) s0 += __ldcg(p + g);
  double v = (s0 + s1) + (s2 + s3);
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  if (lane == 0) sums_out[ic] = v;
}

// MODE 0: proj, 1: update_proj, 2: update_norm.
//   block = ES slots x NG groups, interleaved: thread t -> group g = t % NG, slot = t / NG, so the
//   NG groups of a slot are adjacent lanes of one warp and combine by __shfl_xor (an exact,
//   commutative tree: every lane gets bitwise the same sum).  No barrier in the streaming loop.
template <int MODE, int U>
__global__ void __launch_bounds__(kBS) gram_vs_kernel(GramArgs a, int ES, int NG) {
  __shared__ double red[(kVG + 1) * kBS];  // per-thread accumulators for the block reduce
  const int B = a.B, tid = threadIdx.x;
  const int g = tid % NG, slot = tid / NG, c = slot % B;
  const unsigned mask = __activemask();
  const int nvec = a.nvec, i0 = g * kVG;
  const int nv_g = max(0, min(kVG, nvec - i0));
  const int64_t total = a.len * B, splitE = a.split * B;
  const double wsc = a.wscale ? a.wscale[c] : 1.0;
  double cf[kVG];
#pragma unroll
  for (int j = 0; j < kVG; ++j) {
    cf[j] = 0.0;
    if (MODE != 0 && j < nv_g) {
      const double si = a.s[(i0 + j) * B + c];
      cf[j] = si * si * a.sums_in[(i0 + j) * B + c];
    }
  }
  double acc[kVG];
#pragma unroll
  for (int j = 0; j < kVG; ++j) acc[j] = 0.0;
  double accw = 0.0;  // w.w (proj) or w''.w'' (update_norm), group 0 only
  const double* Qg = a.Q + (int64_t)i0 * a.vstride;
  const int64_t step = (int64_t)gridDim.x * ES * U;
  for (int64_t b0 = (int64_t)blockIdx.x * ES * U; b0 < total; b0 += step) {  // block-uniform bound
    double w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = b0 + slot + (int64_t)u * ES;
      w[u] = 0.0;
      if (e < total) {
        if (MODE == 0) w[u] = e < splitE ? wsc * __ldg(a.wa + e) : __ldg(a.wb + (e - splitE));
        else w[u] = e < splitE ? wsc * a.wa[e] : a.wb[e - splitE];  // wa may alias wout
      }
    }
    double q[kVG][U];
#pragma unroll
    for (int j = 0; j < kVG; ++j)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t e = b0 + slot + (int64_t)u * ES;
        q[j][u] = (j < nv_g && e < total) ? __ldg(Qg + j * a.vstride + e) : 0.0;
      }
    if (MODE == 0) {
#pragma unroll
      for (int j = 0; j < kVG; ++j)
#pragma unroll
        for (int u = 0; u < U; ++u) acc[j] += q[j][u] * w[u];
      if (g == 0) {
#pragma unroll
        for (int u = 0; u < U; ++u) accw += w[u] * w[u];
      }
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        double p = 0.0;
#pragma unroll
        for (int j = 0; j < kVG; ++j) p += cf[j] * q[j][u];
        for (int off = 1; off < NG; off <<= 1) p += __shfl_xor_sync(mask, p, off);
        w[u] -= p;  // w' = w - Σ_i c_i Q_i
        const int64_t e = b0 + slot + (int64_t)u * ES;
        if (g == 0 && e < total) {
          a.wout[e] = w[u];
          if (MODE == 2) accw += w[u] * w[u];
        }
      }
      if (MODE == 1) {
#pragma unroll
        for (int j = 0; j < kVG; ++j)
#pragma unroll
          for (int u = 0; u < U; ++u) acc[j] += q[j][u] * w[u];
      }
    }
  }
  // block reduce by (vector, column): out index i*B + c; i = nvec is the w.w slot (proj)
#pragma unroll
  for (int j = 0; j < kVG; ++j) red[j * kBS + tid] = acc[j];
  red[kVG * kBS + tid] = accw;
  __syncthreads();
  const int nrows = (MODE == 0) ? nvec + 1 : (MODE == 1 ? nvec : 1);
  const int nout = nrows * B;
  const int per = ES / B;
  for (int idx = tid; idx < nout; idx += blockDim.x) {
    const int i = idx / B, cc = idx - i * B;
    const bool is_w = (MODE == 0 && i == nvec) || MODE == 2;
    const int gg = is_w ? 0 : i / kVG, j = is_w ? kVG : i % kVG;
    double sum = 0.0;
    for (int k = 0; k < per; ++k) sum += red[j * kBS + (cc + k * B) * NG + gg];
    a.partials[(int64_t)idx * gridDim.x + blockIdx.x] = sum;
  }
}

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

template <int MODE>
void launch_vs(GramArgs a, cudaStream_t s) {
  static const int U = env_int("WL_GRAM_U", 2);           // experiment knobs (defaults tuned)
  static const int target = env_int("WL_GRAM_BS", 256);
  int NG = groups_for(a.nvec);
  if (NG == 3) NG = 4;
  const int ES = std::max(a.B, (target / NG) / a.B * a.B);
  const int64_t total = a.len * a.B;
  const int64_t items = (total + (int64_t)ES * U - 1) / ((int64_t)ES * U);
  a.grid = (int)std::max<int64_t>(1, std::min<int64_t>(items, gram_grid(total, a.B)));
  if (U == 1) gram_vs_kernel<MODE, 1><<<a.grid, ES * NG, 0, s>>>(a, ES, NG);
  else if (U == 4) gram_vs_kernel<MODE, 4><<<a.grid, ES * NG, 0, s>>>(a, ES, NG);
  else gram_vs_kernel<MODE, 2><<<a.grid, ES * NG, 0, s>>>(a, ES, NG);
  WL_CUDA(cudaGetLastError());
  const int nout = (MODE == 0 ? a.nvec + 1 : (MODE == 1 ? a.nvec : 1)) * a.B;
  note_launch("gram_reduce");  // second kernel of this launch scope (counted, timed with it)
  reduce_partials_kernel<<<(nout + 7) / 8, 256, 0, s>>>(a.partials, nout, a.grid, a.sums_out);
  WL_CUDA(cudaGetLastError());
}

}  // namespace

int gram_grid(int64_t elems, int B) {
  (void)elems;
  (void)B;
  return 148 * 6;  // enough resident CTAs for latency hiding; partial buffers are sized for this
}

// Bases longer than 32 vectors are processed in tiles of 32: tile [i0, i1) writes its sums at
// sums_out + i0*B; its trailing w.w slot is overwritten by the next tile, and the last tile
// leaves w.w at index nvec.
void gram_proj(GramArgs a, cudaStream_t s) {
  if (a.nvec > kMaxVecPerLaunch) {
    for (int i0 = 0; i0 < a.nvec; i0 += kMaxVecPerLaunch) {
      GramArgs t = a;
      t.nvec = std::min(kMaxVecPerLaunch, a.nvec - i0);
      t.Q = a.Q + (int64_t)i0 * a.vstride;
      t.sums_out = a.sums_out + (int64_t)i0 * a.B;
      gram_proj(t, s);
    }
    return;
  }
  WL_LAUNCH("gram_proj");
  launch_vs<0>(a, s);
}

void gram_update_proj(GramArgs a, cudaStream_t s) {
  if (a.nvec > kMaxVecPerLaunch) throw Error(1, "gram_update_proj: nvec > 32 (use the unfused path)");
  WL_LAUNCH("gram_update_proj");
  launch_vs<1>(a, s);
}

void gram_update_norm(GramArgs a, cudaStream_t s) {
  if (a.nvec > kMaxVecPerLaunch) {  // tiles of 32 vectors; tiles after the first update wout in place
    for (int i0 = 0; i0 < a.nvec; i0 += kMaxVecPerLaunch) {
      GramArgs t = a;
      t.nvec = std::min(kMaxVecPerLaunch, a.nvec - i0);
      t.Q = a.Q + (int64_t)i0 * a.vstride;
      t.s = a.s + (int64_t)i0 * a.B;
      t.sums_in = a.sums_in + (int64_t)i0 * a.B;
      if (i0 > 0) { t.wa = a.wout; t.wscale = nullptr; t.split = a.len; t.wb = nullptr; }
      gram_update_norm(t, s);
    }
    return;
  }
  WL_LAUNCH("gram_update_norm");
  launch_vs<2>(a, s);
}

void reduce_partials(const double* partials, int nout, int G, double* sums_out, cudaStream_t s) {
  reduce_partials_kernel<<<(nout + 7) / 8, 256, 0, s>>>(partials, nout, G, sums_out);
  WL_CUDA(cudaGetLastError());
}

}  // namespace wl

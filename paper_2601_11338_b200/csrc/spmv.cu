// spmv.cu — fused companion-operator SpMM (step a4 of DESIGN.md).
//
// One application of Z = [[O, I], [μ(μI - D), A]] (eq:Zdef) to a stacked block
// (x; y) needs only its bottom half  A y + μ(μ - d) ⊙ x  — the top half is y itself and is
// never copied (the Gram kernels read it in place).  This is one step of the BTDW three-term
// recurrence eq:qrec.  The seeds q_1 v = A v and q_2 v = A(Av) - μ d⊙v use the same
// kernel with (g0, g1) = (0, 0) / (0, -μ); the Z step uses (g0, g1) = (μ², -μ).  A has unit
// values, so the kernel only adds gathered rows — no value array is read.
//
// Power-law load balance by degree binning (built once per operator, B-independent):
//   small rows  (deg <= 32, incl. isolated rows): one lane group (B lanes, lane c = column c of the
//               row-major n x B blocks) per row, rows in id order so neighbouring groups read
//               neighbouring col_idx ranges;
//   medium rows (32 < deg <= 2048): one warp per row, its lane groups split the nonzeros and are
//               reduced with shuffles;
//   hub rows    (deg > 2048): split into 2048-nonzero chunks, one warp per chunk; each chunk writes
//               a partial and the last chunk to finish (per-row ticket) sums the row's partials in
//               chunk order — deterministic, no second launch.
// Every lane issues up to 8 independent gathers before consuming them (ILP), and all control flow
// is uniform within a lane group.
#include "wl_internal.cuh"

#include <algorithm>
#include <climits>
#include <cstdlib>

namespace wl {
namespace {

constexpr int kThreads = 256;

// Compile-time cache-hint experiment (build with WL_EXTRA_NVCC=-DWL_SPMV_HINTS=n): 1 = evict-first
// ("cache streaming") loads/stores for the col / x / out streams, 2 = also evict-last for gathers of
// the degree-sorted hot rows.  0 (default) = plain loads.
#ifndef WL_SPMV_HINTS
#define WL_SPMV_HINTS 0
#endif
__device__ __forceinline__ int ld_col(const int32_t* p) {
#if WL_SPMV_HINTS >= 1
  return __ldcs(p);
#else
  return __ldg(p);
#endif
}
__device__ __forceinline__ double ld_stream(const double* p) {
#if WL_SPMV_HINTS >= 1
  return __ldcs(p);
#else
  return *p;
#endif
}
__device__ __forceinline__ void st_stream(double* p, double v) {
#if WL_SPMV_HINTS >= 1
  __stcs(p, v);
#else
  *p = v;
#endif
}
constexpr int kWarps = kThreads / 32;

// Per-lane gather context.  Offsets are 32-bit (n_loc * ld < 2^31 is checked on the host), the
// halo select exists only in the HALO instantiation, and only the last round of a range is
// predicated (ncu r3: 18 warp instructions per nonzero before, mostly address/predicate work).
template <int kU, bool HALO>
struct Ctx {
  const SpmvArgs& a;
  int c;
  double g0, g1, sc;
  const double* yc;   // y + c
  const double* yhc;  // yh + c
  int ldy, ldh;
  uint64_t pol = 0;  // L2 evict-last policy (WL_SPMV_HINTS >= 2)
  __device__ double gather(int cl) const {
    if (HALO && cl >= a.n_loc) return __ldg(yhc + (cl - a.n_loc) * ldh);
#if WL_SPMV_HINTS >= 2
    if (cl < a.small_first) {
      double v;
      asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(yc + cl * ldy), "l"(pol));
      return v;
    }
#endif
    return __ldg(yc + cl * ldy);
  }
  // row r of this CSR -> output row a.out_row[r]; the γ term uses d_r from a.degptr when given
  // (the A_loc part of a split operator); the A_halo part accumulates into out
  __device__ void write(int r, int deg, double sum) const {
    const int ro = a.out_row ? __ldg(a.out_row + r) : r;
    double o = sum;
    if (a.x) {
      if (a.degptr) deg = __ldg(a.degptr + ro + 1) - __ldg(a.degptr + ro);
      o += (g0 + g1 * (double)deg) * ld_stream(a.x + (int64_t)ro * a.ldx + c);
    }
    double* dst = a.out + (int64_t)ro * a.ldo + c;
    st_stream(dst, a.accumulate ? *dst + sc * o : sc * o);
  }
  // Σ y[col[z]] for z = z0 + first, z0 + first + step, ... < z1 (step = lane groups sharing the row)
  __device__ double strided_sum(int z0, int z1, int first, int step) const {
    double acc = 0.0;
    int z = z0 + first;
    const int full = z1 - (kU - 1) * step;  // rounds with all kU nonzeros present
    for (; z < full; z += kU * step) {
      int cl[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) cl[u] = ld_col(a.col + z + u * step);
      double v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) v[u] = gather(cl[u]);
#pragma unroll
      for (int u = 0; u < kU; ++u) acc += v[u];
    }
    if (z < z1) {  // predicated tail round
      int cl[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) cl[u] = (z + u * step < z1) ? ld_col(a.col + z + u * step) : -1;
      double v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) v[u] = cl[u] >= 0 ? gather(cl[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < kU; ++u) acc += v[u];
    }
    return acc;
  }
};

// sum of `v` over the lane groups of a warp, result valid in group 0 (lanes 0..B-1)
__device__ inline double group_reduce(double v, int B, int gpw) {
  if ((B & (B - 1)) == 0) {
    for (int off = 16; off >= B; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    return v;
  }
  const int lane = threadIdx.x & 31;
  double s = v;
  for (int g = 1; g < gpw; ++g) {
    const double o = __shfl_sync(0xffffffffu, v, (lane + g * B) & 31);
    s += o;
  }
  return s;
}

template <int kU, bool HALO>
__global__ void __launch_bounds__(kThreads) spmv_binned_kernel(SpmvArgs a) {
  if (a.active && *a.active == 0) return;
  const int B = a.B;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gpw = 32 / B;
  const int gi = lane / B, c = lane - gi * B;
  const bool lane_ok = gi < gpw;
  const int cc = lane_ok ? c : 0;
  Ctx<kU, HALO> ctx{a, cc, a.g0 ? a.g0[cc] : 0.0, a.g1 ? a.g1[cc] : 0.0, a.scale ? a.scale[cc] : 1.0,
                    a.y + cc, a.yh + cc, (int)a.ldy, (int)a.ldh};
#if WL_SPMV_HINTS >= 2
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(ctx.pol));
#endif
  int blk = blockIdx.x;
  if (blk < a.nblk_small) {  // ---- small rows: one lane group per row
    const int idx = (blk * kWarps + warp) * gpw + gi;
    if (!lane_ok || idx >= a.n_small) return;
    const int r = a.small_rows[idx];
    const int z0 = __ldg(a.rowptr + r), z1 = __ldg(a.rowptr + r + 1);
    ctx.write(r, z1 - z0, ctx.strided_sum(z0, z1, 0, 1));
    return;
  }
  blk -= a.nblk_small;
  if (blk < a.nblk_medium) {  // ---- medium rows: one warp per row
    const int idx = blk * kWarps + warp;
    if (idx >= a.n_medium) return;
    const int r = a.medium_rows[idx];
    const int z0 = __ldg(a.rowptr + r), z1 = __ldg(a.rowptr + r + 1);
    const double part = lane_ok ? ctx.strided_sum(z0, z1, gi, gpw) : 0.0;
    const double sum = group_reduce(part, B, gpw);
    if (gi == 0) ctx.write(r, z1 - z0, sum);
    return;
  }
  blk -= a.nblk_medium;
  {  // ---- hub rows: one warp per kHubChunk-nonzero chunk, last chunk of the row reduces in order
    const int idx = blk * kWarps + warp;
    if (idx >= a.n_chunks) return;
    const int4 ch = a.chunks[idx];  // (row, z0, z1, first chunk index of the row)
    const double part = lane_ok ? ctx.strided_sum(ch.y, ch.z, gi, gpw) : 0.0;
    const double sum = group_reduce(part, B, gpw);
    if (gi == 0) a.chunk_part[(int64_t)idx * B + c] = sum;
    __threadfence();
    __syncwarp();
    unsigned ticket = 0;
    const int z0r = __ldg(a.rowptr + ch.x), z1r = __ldg(a.rowptr + ch.x + 1);
    const int nch = (z1r - z0r + kHubChunk - 1) / kHubChunk;
    if (lane == 0) ticket = atomicAdd(a.row_ticket + ch.w, 1u);  // one ticket per hub row
    ticket = __shfl_sync(0xffffffffu, ticket, 0);
    if (ticket != (unsigned)(nch - 1)) return;
    __threadfence();
    if (gi == 0) {
      double tot = 0.0;
      for (int k = 0; k < nch; ++k) tot += __ldcg(a.chunk_part + (int64_t)(ch.w + k) * B + c);
      ctx.write(ch.x, z1r - z0r, tot);
    }
    if (lane == 0) a.row_ticket[ch.w] = 0u;
  }
}

// ---- small rows with contiguous ids (the degree-sorted layout): one warp per batch of 32 rows ----
// The per-row path above pays a chain of dependent memory latencies per row (row id -> rowptr ->
// col -> gather).  Here a warp loads the batch's 33 row starts with one coalesced load, stages the
// batch's nonzero column ids (contiguous) and its x rows in shared memory with a second, and
// each lane group then walks its share of the batch's nonzeros in rounds of kU gathers,
// flushing rows as their ranges end: ~1 latency per kU gathers instead of ~3 per row.  The rounds
// are software-pipelined (round r+1's gathers issue before round r is summed): 39.7 -> 32.0 ms/step
// on C4.  (The same pipelining in the medium/hub path costs registers and occupancy: +38 ms.)
template <int kU, bool HALO>
__global__ void __launch_bounds__(kThreads) spmv_small_batched_kernel(SpmvArgs a) {
  if (a.active && *a.active == 0) return;
  extern __shared__ __align__(16) int s_small[];
  constexpr int kColCap = 32 * kSmallMax;  // max nonzeros of a 32-row batch
  constexpr int kIntsPerWarp = kColCap + 40;
  const int B = a.B, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gpw = 32 / B, gi = lane / B, c = lane - gi * B;
  const bool lane_ok = gi < gpw;
  const int cc = lane_ok ? c : 0;
  int* scol = s_small + warp * kIntsPerWarp;
  int* srow = scol + kColCap;
  double* sx = reinterpret_cast<double*>(s_small + kWarps * kIntsPerWarp) + warp * 32 * B;
  Ctx<kU, HALO> ctx{a, cc, a.g0 ? a.g0[cc] : 0.0, a.g1 ? a.g1[cc] : 0.0, a.scale ? a.scale[cc] : 1.0,
                    a.y + cc, a.yh + cc, (int)a.ldy, (int)a.ldh};
#if WL_SPMV_HINTS >= 2
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(ctx.pol));
#endif
  const int nb = (a.n_small + 31) / 32;
  for (int bt = blockIdx.x * kWarps + warp; bt < nb; bt += gridDim.x * kWarps) {
    const int r0 = a.small_first + bt * 32;
    const int nr = min(32, a.n_small - bt * 32);
    const int zl = __ldg(a.rowptr + r0 + min(lane, nr));
    const int Z1 = __ldg(a.rowptr + r0 + nr);
    const int Z0 = __shfl_sync(0xffffffffu, zl, 0);
    srow[lane] = zl - Z0;  // rows >= nr: empty ranges at the end
    if (lane == 0) srow[32] = Z1 - Z0;
    const int T = Z1 - Z0;
#pragma unroll 4
    for (int p = lane; p < T; p += 32) scol[p] = ld_col(a.col + Z0 + p);
    if (a.x)
      for (int e = lane; e < nr * B; e += 32) sx[e] = ld_stream(a.x + (int64_t)r0 * B + e);
    __syncwarp();
    if (lane_ok) {
      const int ia = gi * nr / gpw, ib = (gi + 1) * nr / gpw;  // this group's rows
      auto flush = [&](int i, double acc) {
        double o = acc;
        if (a.x) {
          const int d = a.degptr ? __ldg(a.degptr + r0 + i + 1) - __ldg(a.degptr + r0 + i) : srow[i + 1] - srow[i];
          o += (ctx.g0 + ctx.g1 * (double)d) * sx[i * B + c];
        }
        st_stream(a.out + (int64_t)(r0 + i) * a.ldo + c, ctx.sc * o);
      };
      int cur = ia, rend = srow[ia + 1];
      const int P1 = srow[ib];
      double acc = 0.0;
      // software pipeline: round r+1's gathers are issued before round r is consumed
      double v[kU];
      {
        const int p = srow[ia];
#pragma unroll
        for (int u = 0; u < kU; ++u) v[u] = p + u < P1 ? ctx.gather(scol[p + u]) : 0.0;
      }
      for (int p = srow[ia]; p < P1; p += kU) {
        double vn[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) vn[u] = p + kU + u < P1 ? ctx.gather(scol[p + kU + u]) : 0.0;
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          if (p + u < P1) {
            while (p + u >= rend) {
              flush(cur, acc);
              acc = 0.0;
              rend = srow[++cur + 1];
            }
            acc += v[u];
          }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) v[u] = vn[u];
      }
      for (; cur < ib; ++cur) {  // the last row with nonzeros and any empty rows after it
        flush(cur, acc);
        acc = 0.0;
      }
    }
    __syncwarp();
  }
}

// ---- small rows, one column (B = 1: diffusion, CG, Markov): one thread per row ----
// At B = 1 a 32-row batch is one row per lane, so the batched kernel's staging buys nothing and its
// per-batch chain (rowptr -> col -> smem -> gather) plus warp syncs dominates.  A thread per row
// keeps the same three dependent loads with ~8x the rows in flight per SM.
template <bool HALO>
__global__ void __launch_bounds__(kThreads) spmv_small_row1_kernel(SpmvArgs a) {
  if (a.active && *a.active == 0) return;
  const int i = blockIdx.x * kThreads + threadIdx.x;
  if (i >= a.n_small) return;
  Ctx<4, HALO> ctx{a, 0, a.g0 ? a.g0[0] : 0.0, a.g1 ? a.g1[0] : 0.0, a.scale ? a.scale[0] : 1.0,
                   a.y, a.yh, (int)a.ldy, (int)a.ldh};
  const int r = a.small_first + i;
  const int z0 = __ldg(a.rowptr + r), z1 = __ldg(a.rowptr + r + 1);
  ctx.write(r, z1 - z0, ctx.strided_sum(z0, z1, 0, 1));
}

size_t small_batched_smem(int B) {
  return (size_t)kWarps * ((32 * kSmallMax + 40) * sizeof(int) + 32 * B * sizeof(double));
}

}  // namespace

void spmv(const SpmvArgs& a0, cudaStream_t s) {
  if (a0.B < 1 || a0.B > kMaxCols) throw Error(1, "spmv: B out of range");
  SpmvArgs a = a0;
  const int gpw = 32 / a.B;
  a.nblk_small = (a.n_small + kWarps * gpw - 1) / (kWarps * gpw);
  a.nblk_medium = (a.n_medium + kWarps - 1) / kWarps;
  const int nblk_hub = (a.n_chunks + kWarps - 1) / kWarps;
  const int grid = a.nblk_small + a.nblk_medium + nblk_hub;
  if (grid <= 0) return;
  static const int U = [] { const char* v = getenv("WL_SPMV_U"); return v ? atoi(v) : 8; }();
  static const bool split = getenv("WL_SPMV_SPLIT") != nullptr;  // per-class timing experiment
  // gather offsets are 32-bit: local rows (col < n_loc) at col * ldy, halo rows at (col - n_loc) * ldh
  if ((int64_t)(a.n_loc + 1) * a.ldy >= INT32_MAX || (a.yh && (int64_t)(a.n_halo + 1) * a.ldh >= INT32_MAX))
    throw Error(8, "spmv: n_loc * ld and n_halo * ldh must be < 2^31 (32-bit gather offsets)");
  const bool halo = a.yh != nullptr;
  auto go = [&](const SpmvArgs& aa, int g) {
    if (halo) {
      if (U >= 16) spmv_binned_kernel<16, true><<<g, kThreads, 0, s>>>(aa);
      else spmv_binned_kernel<8, true><<<g, kThreads, 0, s>>>(aa);
    } else {
      if (U >= 16) spmv_binned_kernel<16, false><<<g, kThreads, 0, s>>>(aa);
      else spmv_binned_kernel<8, false><<<g, kThreads, 0, s>>>(aa);
    }
    WL_CUDA(cudaGetLastError());
  };
  // small rows with contiguous ids (x rows contiguous too): the batched kernel takes them
  static const bool batched_on = [] { const char* v = getenv("WL_SPMV_BATCHED"); return v ? atoi(v) != 0 : true; }();
  const bool batched = batched_on && a.small_first >= 0 && a.n_small > 0 && (a.x == nullptr || a.ldx == a.B);
  static const bool row1_on = [] { const char* v = getenv("WL_SPMV_ROW1"); return v ? atoi(v) != 0 : true; }();
  auto go_small = [&]() {
    if (a.B == 1 && row1_on) {
      const int g = (a.n_small + kThreads - 1) / kThreads;
      if (halo) spmv_small_row1_kernel<true><<<g, kThreads, 0, s>>>(a);
      else spmv_small_row1_kernel<false><<<g, kThreads, 0, s>>>(a);
      WL_CUDA(cudaGetLastError());
      return;
    }
    auto kern = halo ? spmv_small_batched_kernel<8, true> : spmv_small_batched_kernel<8, false>;
    const size_t smem = small_batched_smem(a.B);
    static bool attr[2] = {false, false};
    if (!attr[halo]) {
      WL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)small_batched_smem(kMaxCols)));
      attr[halo] = true;
    }
    int occ = 0;
    WL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, smem));
    const int sms = num_sms();
    const int nb = (a.n_small + 31) / 32;
    const int g = std::max(1, std::min((nb + kWarps - 1) / kWarps, sms * std::max(occ, 1)));
    kern<<<g, kThreads, smem, s>>>(a);
    WL_CUDA(cudaGetLastError());
  };
  if (batched) {
    SpmvArgs t = a;
    t.n_small = 0;
    t.nblk_small = 0;
    if (!split) {
      WL_LAUNCH("spmv_binned");
      go_small();
      if (grid - a.nblk_small > 0) go(t, grid - a.nblk_small);
      return;
    }
    {
      WL_LAUNCH("spmv_small");
      go_small();
    }
    {
      WL_LAUNCH("spmv_medium");
      SpmvArgs m = t;
      m.n_chunks = 0;
      if (m.nblk_medium) go(m, m.nblk_medium);
    }
    {
      WL_LAUNCH("spmv_hub");
      SpmvArgs h = t;
      h.n_medium = 0; h.nblk_medium = 0;
      if (nblk_hub) go(h, nblk_hub);
    }
    return;
  }
  if (!split) {
    WL_LAUNCH("spmv_binned");
    go(a, grid);
    return;
  }
  {
    WL_LAUNCH("spmv_small");
    SpmvArgs t = a;
    t.n_medium = 0; t.nblk_medium = 0; t.n_chunks = 0;
    if (t.nblk_small) go(t, t.nblk_small);
  }
  {
    WL_LAUNCH("spmv_medium");
    SpmvArgs t = a;
    t.n_small = 0; t.nblk_small = 0; t.n_chunks = 0;
    if (t.nblk_medium) go(t, t.nblk_medium);
  }
  {
    WL_LAUNCH("spmv_hub");
    SpmvArgs t = a;
    t.n_small = 0; t.nblk_small = 0; t.n_medium = 0; t.nblk_medium = 0;
    if (nblk_hub) go(t, nblk_hub);
  }
}

}  // namespace wl

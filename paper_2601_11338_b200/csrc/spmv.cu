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
//   small rows  (deg <= 32, incl. isolated rows): one lane group per row; rows with contiguous ids
//               (the degree-sorted layout) go to the batched kernel (a warp per 32 rows);
//   medium rows (32 < deg <= 2048): one warp per row, its lane groups split the nonzeros and are
//               reduced with shuffles;
//   hub rows    (deg > 2048): split into 2048-nonzero chunks, one warp per chunk; each chunk writes
//               a partial and the last chunk to finish (per-row ticket) sums the row's partials in
//               chunk order — deterministic, no second launch.
//
// Lane groups and gather width.  A gathered row of the row-major block y holds B doubles.  A lane
// loads VW consecutive doubles (VW = 1: 8 B; VW = 2: 16 B; VW = 4: 32 B, the sm_100 256-bit load
// LDG.E.ENL2.256), so a row takes W = ceil(B / VW) lanes and one warp instruction gathers
// gpw = 32 / W rows.  On this B200 the rate of random row gathers from L2 depends on it far more
// than on bytes (tools/gather_ceiling.cu, C4 degree distribution, 4e8 rows of 11 columns):
// 8-byte lanes (W = 11, 2 rows per instruction) 8.16 ms; 16-byte lanes 3.34 ms; 32-byte lanes
// (W = 3, 10 rows per instruction) 3.02 ms.  VW > 1 needs ld y (and the halo's ld) a multiple of
// VW and VW-aligned rows: the engine keeps the gathered operand of the TOAR steps in a block padded
// to ld = 4 * ceil(B / 4) (zero phantom columns).  B = 1 uses VW = 1 with a thread per small row.
#include "wl_internal.cuh"

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <type_traits>

// compile-time tuning knobs (tools/build_variants.sh): wide-lane unroll, min CTAs per SM of the rows kernel
#ifndef WL_SPMV_UW
#define WL_SPMV_UW 4
#endif
#ifndef WL_SPMV_MINB
#define WL_SPMV_MINB 6
#endif
#ifndef WL_SPMV_MINB_S
#define WL_SPMV_MINB_S 3
#endif
// 1: the medium rows (several per warp) and the hub chunks of wide-lane kernels load their column ids 4 at a time
#ifndef WL_SPMV_VEC4
#define WL_SPMV_VEC4 0
#endif
// 1: column ids of the next round loaded before the current round's gathers are summed (tools/kernel_variants.sh)
#ifndef WL_SPMV_PREFETCH
#define WL_SPMV_PREFETCH 0
#endif
// fp32 storage (8-float lanes): unroll and min CTAs per SM of the row kernel
#ifndef WL_SPMV_UW_F
#define WL_SPMV_UW_F 4
#endif
#ifndef WL_SPMV_MINB_F
#define WL_SPMV_MINB_F 5  // with float sums: 48 registers (4 CTAs/SM with double sums: 85 -> 78.5 ms/step on C4)
#endif
// fp32 storage: 1 = row sums accumulated in float (half the accumulator registers; the rows are <= 4096-nonzero
// pieces, the output is rounded to float anyway: C4-shaped errors unchanged at 1e-9), 0 = in double
#ifndef WL_SPMV_F_ACC32
#define WL_SPMV_F_ACC32 1
#endif

namespace wl {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// VW values of the storage type T (double; float in the fp32 mode) — sums are always accumulated in double
template <int VW, class T = double>
struct Vec {
  T v[VW];
};

template <int VW, class T = double>
__device__ __forceinline__ Vec<VW, T> vzero() {
  Vec<VW, T> r;
#pragma unroll
  for (int k = 0; k < VW; ++k) r.v[k] = T(0);
  return r;
}
template <int VW, class A, class T>
__device__ __forceinline__ void vadd(Vec<VW, A>& a, const Vec<VW, T>& b) {
#pragma unroll
  for (int k = 0; k < VW; ++k) a.v[k] += (A)b.v[k];
}
template <int VW>
__device__ __forceinline__ void vaddf(Vec<VW, float>& a, const Vec<VW, float>& b) {
#pragma unroll
  for (int k = 0; k < VW; ++k) a.v[k] += b.v[k];
}
// read-only (non-coherent) load of VW consecutive values, VW-aligned (32 bytes at most: the 256-bit LDG)
template <int VW, class T>
__device__ __forceinline__ Vec<VW, T> vload(const T* p) {
  Vec<VW, T> r;
  if constexpr (VW == 1) {
    r.v[0] = __ldg(p);
  } else if constexpr (std::is_same<T, double>::value) {
    if constexpr (VW == 2) {
      const double2 t = __ldg(reinterpret_cast<const double2*>(p));
      r.v[0] = t.x;
      r.v[1] = t.y;
    } else {
      static_assert(VW == 4, "double: VW in {1, 2, 4}");
      asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
          : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3])
          : "l"(p));
    }
  } else {
    static_assert(VW == 8, "float: VW in {1, 8}");
    asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]), "=f"(r.v[6]),
          "=f"(r.v[7])
        : "l"(p));
  }
  return r;
}

// The same with an L2 eviction-priority policy (createpolicy): the hot prefix of the degree-sorted
// gathered block is loaded evict_last, everything streamed once (column ids, cold rows) evict_first.
template <int VW>
__device__ __forceinline__ Vec<VW> vload_hint(const double* p, uint64_t pol) {
  Vec<VW> r;
  if constexpr (VW == 1) {
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r.v[0]) : "l"(p), "l"(pol));
  } else if constexpr (VW == 2) {
    asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(r.v[0]), "=d"(r.v[1]) : "l"(p), "l"(pol));
  } else {
    asm("ld.global.nc.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
        : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3])
        : "l"(p), "l"(pol));
  }
  return r;
}
__device__ __forceinline__ int ld_col_hint(const int32_t* p, uint64_t pol) {
  int v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}

// Per-lane gather context.  Lane group gi of W lanes handles one row at a time; lane (gi, w) owns
// columns c0 = w*VW .. c0+VW-1 (those < B are real).  Offsets are 32-bit (n_loc * ld < 2^31 is
// checked on the host); the halo select exists only in the HALO instantiation, and only the last
// round of a range is predicated.
template <int kU, bool HALO, int VW, bool HINT = false, class T = double>
struct Ctx {
  static_assert(!HINT || std::is_same<T, double>::value, "L2 hints: double storage only");
  using Acc = typename std::conditional<std::is_same<T, float>::value && WL_SPMV_F_ACC32, float, double>::type;
  const SpmvArgs& a;
  uint64_t pol_last = 0, pol_first = 0;  // HINT: L2 policies
  int c0;             // first column of this lane
  int nc;             // real columns of this lane (0..VW)
  const T* yc;        // y + c0
  const T* yhc;       // yh + c0
  int ldy, ldh;
  __device__ Ctx(const SpmvArgs& args, int col0) : a(args), c0(col0) {
    nc = max(0, min(VW, a.B - c0));
    yc = reinterpret_cast<const T*>(a.y) + c0;
    yhc = reinterpret_cast<const T*>(a.yh) + c0;
    ldy = (int)a.ldy;
    ldh = (int)a.ldh;
    if (HINT) {
      asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_last));
      asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
    }
  }
  __device__ Vec<VW, T> gather(int cl) const {
    if constexpr (HINT) {
      if (HALO && cl >= a.n_loc) return vload_hint<VW>(yhc + (cl - a.n_loc) * ldh, pol_first);
      return vload_hint<VW>(yc + cl * ldy, cl < a.hot_rows ? pol_last : pol_first);
    } else {
      if (HALO && cl >= a.n_loc) return vload<VW>(yhc + (cl - a.n_loc) * ldh);
      return vload<VW>(yc + cl * ldy);
    }
  }
  __device__ int col(int z) const {
    if (HINT) return ld_col_hint(a.col + z, pol_first);
    return __ldg(a.col + z);
  }
  // row r of this CSR -> output row a.out_row[r]; the γ term uses d_r from a.degptr when given
  // (the A_loc part of a split operator); the A_halo part accumulates into out.  `x` (the diagonal
  // operand, ld ldx) and out (ld ldo) are unpadded: per-column scalar accesses.
  __device__ void write(int r, int deg, const Vec<VW, Acc>& sum, const double* xrow = nullptr) const {
    const int ro = a.out_row ? __ldg(a.out_row + r) : r;
    if (a.x && a.degptr) deg = __ldg(a.degptr + ro + 1) - __ldg(a.degptr + ro);
    T* dst = reinterpret_cast<T*>(a.out) + (int64_t)ro * a.ldo + c0;
    const T* xs = xrow ? reinterpret_cast<const T*>(xrow) : reinterpret_cast<const T*>(a.x) + (int64_t)ro * a.ldx + c0;
    // per-column constants are read here (L1-resident, B values) rather than held in registers
#pragma unroll
    for (int k = 0; k < VW; ++k) {
      if (k < nc) {
        const int c = c0 + k;
        double o = (double)sum.v[k];
        if (a.x) o += ((a.g0 ? __ldg(a.g0 + c) : 0.0) + (a.g1 ? __ldg(a.g1 + c) : 0.0) * (double)deg) * (double)xs[k];
        const double sc = a.scale ? __ldg(a.scale + c) : 1.0;
        dst[k] = (T)(a.accumulate ? (double)dst[k] + sc * o : sc * o);
      }
    }
  }
  // Σ y[col[z]] for z = z0 + first, z0 + first + step, ... < z1 (step = lane groups sharing the row,
  // 0 <= first < step).  Rounds cover [base, base + kU step); the full-round test depends only on the
  // shared base, so lane groups sharing a row never diverge: all full rounds, then one predicated round.
  __device__ Vec<VW, Acc> strided_sum(int z0, int z1, int first, int step) const {
    Vec<VW, Acc> acc = vzero<VW, Acc>();
    int base = z0;
#if WL_SPMV_PREFETCH
    // the next full round's column ids are loaded before this round's gathers are consumed (one id latency
    // hidden per round)
    if (base + kU * step <= z1) {
      int cl[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) cl[u] = col(base + first + u * step);
      for (;;) {
        const int nb = base + kU * step;
        const bool more = nb + kU * step <= z1;  // warp-uniform (shared base)
        int nx[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) nx[u] = more ? col(nb + first + u * step) : 0;
        Vec<VW, T> v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) v[u] = gather(cl[u]);
        add_round(acc, v);
        base = nb;
        if (!more) break;
#pragma unroll
        for (int u = 0; u < kU; ++u) cl[u] = nx[u];
      }
    }
#else
    for (; base + kU * step <= z1; base += kU * step) {
      int cl[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) cl[u] = col(base + first + u * step);
      Vec<VW, T> v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) v[u] = gather(cl[u]);
      add_round(acc, v);
    }
#endif
    const int z = base + first;
    if (base < z1) {  // predicated tail round
      int cl[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) cl[u] = (z + u * step < z1) ? col(z + u * step) : -1;
      Vec<VW, T> v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) v[u] = cl[u] >= 0 ? gather(cl[u]) : vzero<VW, T>();
      add_round(acc, v);
    }
    return acc;
  }
  // Σ y[col[z]] over [z0, z1) with the column ids of the 4-aligned body loaded 4 at a time (one 16-byte load per
  // 4 gathers: in the medium-row path a warp's id loads touched 5 rows' sectors 4 times per round, a quarter of
  // the L1 wavefronts); group `first` of `step` groups takes the body's 4-id chunks first, first + step, ...; the
  // unaligned head and the tail (< 4 ids each) go through strided_sum.  kU == 4.
  __device__ Vec<VW, Acc> vec4_sum(int z0, int z1, int first, int step) const {
    const int za = min(z1, (z0 + 3) & ~3);
    Vec<VW, Acc> acc = strided_sum(z0, za, first, step);
    const int nch = (z1 - za) >> 2;
    const int4* c4 = reinterpret_cast<const int4*>(a.col + za);
    for (int c = first; c < nch; c += step) {
      const int4 id = __ldg(c4 + c);
      Vec<VW, T> v[kU];
      v[0] = gather(id.x);
      v[1] = gather(id.y);
      v[2] = gather(id.z);
      v[3] = gather(id.w);
      add_round(acc, v);
    }
    vadd(acc, strided_sum(za + 4 * nch, z1, first, step));
    return acc;
  }
  // one round of kU gathered rows into the double accumulator; fp32 storage sums the round in float first
  // (one conversion per round instead of per row: its rounding is that of the stored values)
  __device__ static void add_round(Vec<VW, Acc>& acc, const Vec<VW, T> (&v)[kU]) {
    if constexpr (std::is_same<T, double>::value) {
#pragma unroll
      for (int u = 0; u < kU; ++u) vadd(acc, v[u]);
    } else {
      Vec<VW, T> r = v[0];
#pragma unroll
      for (int u = 1; u < kU; ++u) vaddf(r, v[u]);
      vadd(acc, r);
    }
  }
};

// sum of `v` over the lane groups (W lanes each) of a warp, result valid in group 0 (lanes 0..W-1)
template <int VW, class A>
__device__ inline Vec<VW, A> group_reduce(Vec<VW, A> v, int W, int gpw) {
  if ((W & (W - 1)) == 0) {
#pragma unroll
    for (int k = 0; k < VW; ++k)
      for (int off = 16; off >= W; off >>= 1) v.v[k] += __shfl_down_sync(0xffffffffu, v.v[k], off);
    return v;
  }
  const int lane = threadIdx.x & 31;
  Vec<VW, A> s = v;
  for (int g = 1; g < gpw; ++g) {
#pragma unroll
    for (int k = 0; k < VW; ++k) s.v[k] += __shfl_sync(0xffffffffu, v.v[k], (lane + g * W) & 31);
  }
  return s;
}

template <int VW>
__device__ __forceinline__ int lanes_per_row(int B) { return (B + VW - 1) / VW; }

template <int kU, bool HALO, int VW, bool HINT, class T>
__global__ void __launch_bounds__(kThreads, VW == 1 ? 1 : (sizeof(T) == 4 ? WL_SPMV_MINB_F : WL_SPMV_MINB))
    spmv_binned_kernel(SpmvArgs a) {
  if (a.active && *a.active == 0) return;
  const int W = lanes_per_row<VW>(a.B);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gpw = 32 / W;
  const int gi = lane / W, w = lane - gi * W;
  const bool lane_ok = gi < gpw;
  const Ctx<kU, HALO, VW, HINT, T> ctx(a, lane_ok ? w * VW : 0);
  using Acc = typename Ctx<kU, HALO, VW, HINT, T>::Acc;
  int blk = blockIdx.x;
  if (blk < a.nblk_small) {  // ---- small rows: one lane group per row
    const int idx = (blk * kWarps + warp) * gpw + gi;
    if (!lane_ok || idx >= a.n_small) return;
    const int r = a.small_first >= 0 ? a.small_first + idx : a.small_rows[idx];  // contiguous: no list load
    const int z0 = __ldg(a.rowptr + r), z1 = __ldg(a.rowptr + r + 1);
    ctx.write(r, z1 - z0, ctx.strided_sum(z0, z1, 0, 1));
    return;
  }
  blk -= a.nblk_small;
  if (blk < a.nblk_medium) {  // ---- medium rows: one warp per row (one row per 8 lanes when a row is one lane wide)
    if (W == 1 && a.med_sub) {
      // 32/L rows per warp, L = med_sub lanes each: more rows (independent latency chains) in flight per warp,
      // and the tail round of a ~100-300-nonzero row wastes L lanes instead of 32
      const int L = a.med_sub;
      const int idx = (blk * kWarps + warp) * (32 / L) + lane / L, lg = lane % L;
      const int r = idx < a.n_medium ? (a.medium_first >= 0 ? a.medium_first + idx : a.medium_rows[idx]) : 0;
      const int z0 = idx < a.n_medium ? __ldg(a.rowptr + r) : 0, z1 = idx < a.n_medium ? __ldg(a.rowptr + r + 1) : 0;
      Vec<VW, Acc> part = ctx.strided_sum(z0, z1, lg, L);
#pragma unroll
      for (int k = 0; k < VW; ++k)
        for (int off = L / 2; off > 0; off >>= 1) part.v[k] += __shfl_xor_sync(0xffffffffu, part.v[k], off);
      if (lg == 0 && idx < a.n_medium) ctx.write(r, z1 - z0, part);
      return;
    }
    if (a.med_rpw > 1) {
      // med_rpw rows per warp, gpw / med_rpw lane groups each (B = 11: 2 rows x 5 groups of 3 lanes)
      const int G2 = gpw / a.med_rpw, LR = G2 * W;
      const int rs = lane / LR, base = rs * LR, gi2 = (lane - base) / W;
      const int idx = (blk * kWarps + warp) * a.med_rpw + rs;
      const bool ok = rs < a.med_rpw && idx < a.n_medium;
      const int r = ok ? (a.medium_first >= 0 ? a.medium_first + idx : a.medium_rows[idx]) : 0;
      const int z0 = ok ? __ldg(a.rowptr + r) : 0, z1 = ok ? __ldg(a.rowptr + r + 1) : 0;
      Vec<VW, Acc> part = vzero<VW, Acc>();
      if (ok) {
        if constexpr (WL_SPMV_VEC4 && VW > 1 && kU == 4) part = ctx.vec4_sum(z0, z1, gi2, G2);
        else part = ctx.strided_sum(z0, z1, gi2, G2);
      }
      Vec<VW, Acc> sum = part;
      for (int g = 1; g < G2; ++g) {
        const int src = base + ((lane - base) + g * W) % LR;
#pragma unroll
        for (int k = 0; k < VW; ++k) sum.v[k] += __shfl_sync(0xffffffffu, part.v[k], rs < a.med_rpw ? src : lane);
      }
      if (ok && gi2 == 0) ctx.write(r, z1 - z0, sum);
      return;
    }
    const int idx = blk * kWarps + warp;
    if (idx >= a.n_medium) return;
    const int r = a.medium_first >= 0 ? a.medium_first + idx : a.medium_rows[idx];
    const int z0 = __ldg(a.rowptr + r), z1 = __ldg(a.rowptr + r + 1);
    const Vec<VW, Acc> part = lane_ok ? ctx.strided_sum(z0, z1, gi, gpw) : vzero<VW, Acc>();
    const Vec<VW, Acc> sum = group_reduce<VW>(part, W, gpw);
    if (gi == 0) ctx.write(r, z1 - z0, sum);
    return;
  }
  blk -= a.nblk_medium;
  {  // ---- hub rows: one warp per kHubChunk-nonzero chunk, last chunk of the row reduces in order
    const int idx = blk * kWarps + warp;
    if (idx >= a.n_chunks) return;
    const int4 ch = a.chunks[idx];  // (row, z0, z1, first chunk index of the row)
    Vec<VW, Acc> part = vzero<VW, Acc>();
    if (lane_ok) {
      if constexpr (WL_SPMV_VEC4 && VW > 1 && kU == 4) part = ctx.vec4_sum(ch.y, ch.z, gi, gpw);
      else part = ctx.strided_sum(ch.y, ch.z, gi, gpw);
    }
    const Vec<VW, Acc> sum = group_reduce<VW>(part, W, gpw);
    const int ldp = W * VW;  // partial row: every column slot of the lane group
    if (gi == 0) {
#pragma unroll
      for (int k = 0; k < VW; ++k) a.chunk_part[(int64_t)idx * ldp + w * VW + k] = (double)sum.v[k];
    }
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
      Vec<VW, Acc> tot = vzero<VW, Acc>();
      for (int k = 0; k < nch; ++k)
#pragma unroll
        for (int q = 0; q < VW; ++q) tot.v[q] += (Acc)__ldcg(a.chunk_part + (int64_t)(ch.w + k) * ldp + w * VW + q);
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
// on C4 at VW = 1.
template <int kU, bool HALO, int VW, bool HINT>
__global__ void __launch_bounds__(kThreads, WL_SPMV_MINB_S) spmv_small_batched_kernel(SpmvArgs a) {  // double storage
  if (a.active && *a.active == 0) return;
  extern __shared__ __align__(16) int s_small[];
  constexpr int kColCap = 32 * kSmallMax;  // max nonzeros of a 32-row batch
  constexpr int kIntsPerWarp = kColCap + 40;
  const int B = a.B, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int W = lanes_per_row<VW>(B);
  const int gpw = 32 / W, gi = lane / W, w = lane - gi * W;
  const bool lane_ok = gi < gpw;
  int* scol = s_small + warp * kIntsPerWarp;
  int* srow = scol + kColCap;
  double* sx = reinterpret_cast<double*>(s_small + kWarps * kIntsPerWarp) + warp * 32 * B;
  const Ctx<kU, HALO, VW, HINT> ctx(a, lane_ok ? w * VW : 0);
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
    for (int p = lane; p < T; p += 32) scol[p] = ctx.col(Z0 + p);
    if (a.x)
      for (int e = lane; e < nr * B; e += 32) sx[e] = a.x[(int64_t)r0 * B + e];
    __syncwarp();
    if (lane_ok) {
      const int ia = gi * nr / gpw, ib = (gi + 1) * nr / gpw;  // this group's rows
      auto flush = [&](int i, const Vec<VW>& acc) {
        const int d = a.degptr ? 0 : srow[i + 1] - srow[i];  // (degptr: write() reads d_r itself)
        ctx.write(r0 + i, d, acc, sx + i * B + ctx.c0);
      };
      int cur = ia, rend = srow[ia + 1];
      const int P1 = srow[ib];
      Vec<VW> acc = vzero<VW>();
      // software pipeline: round r+1's gathers are issued before round r is consumed
      Vec<VW> v[kU];
      {
        const int p = srow[ia];
#pragma unroll
        for (int u = 0; u < kU; ++u) v[u] = p + u < P1 ? ctx.gather(scol[p + u]) : vzero<VW>();
      }
      for (int p = srow[ia]; p < P1; p += kU) {
        Vec<VW> vn[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) vn[u] = p + kU + u < P1 ? ctx.gather(scol[p + kU + u]) : vzero<VW>();
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          if (p + u < P1) {
            while (p + u >= rend) {
              flush(cur, acc);
              acc = vzero<VW>();
              rend = srow[++cur + 1];
            }
            vadd(acc, v[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) v[u] = vn[u];
      }
      for (; cur < ib; ++cur) {  // the last row with nonzeros and any empty rows after it
        flush(cur, acc);
        acc = vzero<VW>();
      }
    }
    __syncwarp();
  }
}

// ---- small rows, one column (B = 1: diffusion, CG, Markov): one thread per row ----
// At B = 1 a 32-row batch is one row per lane, so the batched kernel's staging buys nothing and its
// per-batch chain (rowptr -> col -> smem -> gather) plus warp syncs dominates.  A thread per row
// keeps the same three dependent loads with ~8x the rows in flight per SM.
template <bool HALO, bool HINT, class T>
__global__ void __launch_bounds__(kThreads) spmv_small_row1_kernel(SpmvArgs a) {
  if (a.active && *a.active == 0) return;
  const int i = blockIdx.x * kThreads + threadIdx.x;
  if (i >= a.n_small) return;
  const Ctx<4, HALO, 1, HINT, T> ctx(a, 0);
  const int r = a.small_first + i;
  const int z0 = __ldg(a.rowptr + r), z1 = __ldg(a.rowptr + r + 1);
  ctx.write(r, z1 - z0, ctx.strided_sum(z0, z1, 0, 1));
}

// ---- rows without nonzeros at the end of the contiguous small range (isolated vertices: 40% of C4's ids):
// out = scale ⊙ (g0 + g1 d) ⊙ x, a stream over the n_iso x B block (d = 0 unless degptr gives the full degree
// of a split operator's local part)
template <class T>
__global__ void __launch_bounds__(kThreads) spmv_iso_kernel(SpmvArgs a, int r0) {
  if (a.active && *a.active == 0) return;
  const int B = a.B;
  const int64_t total = (int64_t)a.n_iso * B;
  for (int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x; e < total; e += (int64_t)gridDim.x * kThreads) {
    const int64_t i = e / B;
    const int c = (int)(e - i * B);
    const int64_t r = r0 + i;
    double o = 0.0;
    if (a.x) {
      const double d = a.degptr ? (double)(__ldg(a.degptr + r + 1) - __ldg(a.degptr + r)) : 0.0;
      o = ((a.g0 ? __ldg(a.g0 + c) : 0.0) + (a.g1 ? __ldg(a.g1 + c) : 0.0) * d) *
          (double)__ldg(reinterpret_cast<const T*>(a.x) + r * a.ldx + c);
    }
    reinterpret_cast<T*>(a.out)[r * a.ldo + c] = (T)((a.scale ? __ldg(a.scale + c) : 1.0) * o);
  }
}

size_t small_batched_smem(int B) {
  return (size_t)kWarps * ((32 * kSmallMax + 40) * sizeof(int) + 32 * B * sizeof(double));
}

template <int VW>
constexpr int unroll_for() { return VW == 1 ? 8 : VW == 8 ? WL_SPMV_UW_F : WL_SPMV_UW; }  // wide lanes: 4 rounds in flight
template <int VW>
constexpr int unroll_batched() { return VW == 1 ? 8 : VW == 2 ? 4 : 2; }  // pipelined: 2 rounds live

// launch the batched small rows (if any) and the binned kernel (small rows by id list, medium, hub)
template <int VW, bool HINT, class T>
void launch_vw(const SpmvArgs& a, bool halo, bool batched, int grid_rest, cudaStream_t s) {
  constexpr int kU = unroll_for<VW>(), kUb = unroll_batched<VW>();
  static const bool split = getenv("WL_SPMV_SPLIT") != nullptr;  // per-class timing (profiling only)
  SpmvArgs t = a;
  if constexpr (std::is_same<T, double>::value) {  // the batched staging is double only
  if (batched) {
    LaunchScope ls(split ? "spmv_small_batched" : nullptr, s);
    auto kern = halo ? spmv_small_batched_kernel<kUb, true, VW, HINT> : spmv_small_batched_kernel<kUb, false, VW, HINT>;
    const size_t smem = small_batched_smem(a.B);
    static bool attr[2] = {false, false};
    if (!attr[halo]) {
      WL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)small_batched_smem(kMaxCols)));
      attr[halo] = true;
    }
    int occ = 0;
    WL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, smem));
    const int nb = (a.n_small + 31) / 32;
    const int g = std::max(1, std::min((nb + kWarps - 1) / kWarps, num_sms() * std::max(occ, 1)));
    kern<<<g, kThreads, smem, s>>>(a);
    WL_CUDA(cudaGetLastError());
    t.n_small = 0;
    t.nblk_small = 0;
  }
  }
  if (grid_rest <= 0) return;
  LaunchScope ls(split ? "spmv_rows" : nullptr, s);
  if (halo) spmv_binned_kernel<kU, true, VW, HINT, T><<<grid_rest, kThreads, 0, s>>>(t);
  else spmv_binned_kernel<kU, false, VW, HINT, T><<<grid_rest, kThreads, 0, s>>>(t);
  WL_CUDA(cudaGetLastError());
}

template <int VW, class T = double>
void launch_vw(const SpmvArgs& a, bool halo, bool batched, int grid_rest, cudaStream_t s) {
  if constexpr (std::is_same<T, double>::value) {
    if (a.hot_rows > 0) {
      launch_vw<VW, true, T>(a, halo, batched, grid_rest, s);
      return;
    }
  }
  launch_vw<VW, false, T>(a, halo, batched, grid_rest, s);
}

inline bool aligned(const void* p, int bytes) { return (reinterpret_cast<uintptr_t>(p) % bytes) == 0; }

}  // namespace

// widest lane load the gathered operand allows (see the file comment)
int spmv_vector_width(const SpmvArgs& a) {
  if (a.B == 1) return 1;
  const bool halo = a.yh != nullptr;
  if (a.f32) {  // fp32 storage: 32-byte lanes of 8 floats or scalar lanes
    const int vw = 8;
    return (a.ldy % vw == 0 && aligned(a.y, 4 * vw) && (!halo || (a.ldh % vw == 0 && aligned(a.yh, 4 * vw)))) ? vw : 1;
  }
  for (int vw : {4, 2}) {
    if (a.ldy % vw == 0 && aligned(a.y, 8 * vw) && (!halo || (a.ldh % vw == 0 && aligned(a.yh, 8 * vw)))) return vw;
  }
  return 1;
}

void spmv(const SpmvArgs& a0, cudaStream_t s) {
  if (a0.B < 1 || a0.B > kMaxCols) throw Error(1, "spmv: B out of range");
  SpmvArgs a = a0;
  WL_LAUNCH("spmv_binned");
  if (a.small_first >= 0 && a.n_iso > 0 && !a.accumulate) {  // isolated rows: a stream, off the row kernels
    const int r0 = a.small_first + a.n_small - a.n_iso;
    SpmvArgs ai = a;  // rows >= row_limit (the Krylov batches' isolated tail) are not written at all
    if (a.row_limit > 0) ai.n_iso = (int)std::max<int64_t>(0, std::min<int64_t>(a.n_iso, a.row_limit - r0));
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>(((int64_t)ai.n_iso * a.B + kThreads - 1) / kThreads,
                                                            (int64_t)num_sms() * 8));
    if (ai.n_iso > 0) {
      if (a.f32) spmv_iso_kernel<float><<<g, kThreads, 0, s>>>(ai, r0);
      else spmv_iso_kernel<double><<<g, kThreads, 0, s>>>(ai, r0);
      WL_CUDA(cudaGetLastError());
    }
    a.n_small -= a.n_iso;
    a.n_iso = 0;
    if (a.n_small == 0) a.small_first = -1;
  }
  // L2 eviction hints: rows [0, hot_rows) of the degree-sorted gathered block (the most gathered
  // rows) stay, column ids and cold rows go first.  Budget WL_SPMV_HOT_MB of L2 (0 = no hints).
  static const double hot_mb = [] { const char* v = getenv("WL_SPMV_HOT_MB"); return v ? atof(v) : 0.0; }();
  if (a.f32) a.hot_rows = 0;
  else if (hot_mb > 0.0 && a.hot_rows == 0)
    a.hot_rows = (int)std::min<int64_t>(a.n_loc, (int64_t)(hot_mb * 1e6 / (8.0 * a.ldy)));
  static const int vw_cap = [] { const char* v = getenv("WL_SPMV_VW"); return v ? atoi(v) : 4; }();
  int VW = spmv_vector_width(a);
  if (a.f32 ? (VW > 2 * vw_cap) : (VW > vw_cap)) VW = a.f32 ? 1 : vw_cap;  // fp32: 8 or 1
  const int W = (a.B + VW - 1) / VW;
  const int gpw = 32 / W;
  a.nblk_small = (a.n_small + kWarps * gpw - 1) / (kWarps * gpw);
  // lanes per medium row when a row is one lane wide (b = 1): 0 = a warp per row
  static const int med_sub = [] { const char* v = getenv("WL_SPMV_MEDSUB"); return v ? atoi(v) : 4; }();
  a.med_sub = (W == 1 && (med_sub == 4 || med_sub == 8 || med_sub == 16)) ? med_sub : 0;
  // wide rows (W > 1): medium rows per warp (WL_SPMV_MEDRPW; 1 = a warp per row)
  // (defaults measured on C4: 5 with double rows of 3 lanes, 8 with float rows of 2 lanes)
  static const int med_rpw_env = [] { const char* v = getenv("WL_SPMV_MEDRPW"); return v ? atoi(v) : 0; }();
  const int med_rpw = med_rpw_env ? med_rpw_env : (a.f32 ? 8 : 5);
  a.med_rpw = (W > 1 && med_rpw > 1 && gpw / med_rpw >= 1) ? med_rpw : 1;
  const int rows_per_warp = a.med_sub ? 32 / a.med_sub : a.med_rpw;
  // profiling only (wrong results): WL_SPMV_ONLY = any of "s", "m", "h" launches only those row classes
  static const char* only = getenv("WL_SPMV_ONLY");
  if (only) {
    if (!strchr(only, 's')) { a.n_small = 0; a.nblk_small = 0; }
    if (!strchr(only, 'm')) a.n_medium = 0;
    if (!strchr(only, 'h')) a.n_chunks = 0;
  }
  a.nblk_medium = (a.n_medium + kWarps * rows_per_warp - 1) / (kWarps * rows_per_warp);
  const int nblk_hub = (a.n_chunks + kWarps - 1) / kWarps;
  const int grid = a.nblk_small + a.nblk_medium + nblk_hub;
  if (grid <= 0) return;
  // gather offsets are 32-bit: local rows (col < n_loc) at col * ldy, halo rows at (col - n_loc) * ldh
  if ((int64_t)(a.n_loc + 1) * a.ldy >= INT32_MAX || (a.yh && (int64_t)(a.n_halo + 1) * a.ldh >= INT32_MAX))
    throw Error(8, "spmv: n_loc * ld and n_halo * ldh must be < 2^31 (32-bit gather offsets)");
  if (a.out_row && a.small_first >= 0) throw Error(1, "spmv: batched small rows cannot remap output rows");
  const bool halo = a.yh != nullptr;
  if (a.B == 1) {
    if (a.small_first >= 0 && a.n_small > 0) {  // thread per small row
      static const bool split = getenv("WL_SPMV_SPLIT") != nullptr;
      LaunchScope ls(split ? "spmv_small_row1" : nullptr, s);
      const int g = (a.n_small + kThreads - 1) / kThreads;
      if (a.f32) {
        if (halo) spmv_small_row1_kernel<true, false, float><<<g, kThreads, 0, s>>>(a);
        else spmv_small_row1_kernel<false, false, float><<<g, kThreads, 0, s>>>(a);
      } else if (a.hot_rows > 0) {
        if (halo) spmv_small_row1_kernel<true, true, double><<<g, kThreads, 0, s>>>(a);
        else spmv_small_row1_kernel<false, true, double><<<g, kThreads, 0, s>>>(a);
      } else {
        if (halo) spmv_small_row1_kernel<true, false, double><<<g, kThreads, 0, s>>>(a);
        else spmv_small_row1_kernel<false, false, double><<<g, kThreads, 0, s>>>(a);
      }
      WL_CUDA(cudaGetLastError());
      SpmvArgs t = a;
      t.n_small = 0;
      t.nblk_small = 0;
      if (a.f32) launch_vw<1, float>(t, halo, false, grid - a.nblk_small, s);
      else launch_vw<1>(t, halo, false, grid - a.nblk_small, s);
    } else {
      if (a.f32) launch_vw<1, float>(a, halo, false, grid, s);
      else launch_vw<1>(a, halo, false, grid, s);
    }
    return;
  }
  // small rows with contiguous ids (x rows contiguous too): the batched kernel takes them
  static const bool batched_on = [] { const char* v = getenv("WL_SPMV_BATCHED"); return v ? atoi(v) != 0 : true; }();
  // with 8-byte lanes the batch staging pays (round 1: 59 -> 40 ms/step on C4); with 32-byte lanes a warp already
  // walks 10 small rows at once through the row kernel, and the staging costs more than it saves (148 -> 140 ms/step)
  const bool batched = batched_on && !a.f32 && VW == 1 && a.small_first >= 0 && a.n_small > 0 && (a.x == nullptr || a.ldx == a.B);
  const int rest = batched ? grid - a.nblk_small : grid;
  if (a.f32) {
    if (VW == 8) launch_vw<8, float>(a, halo, false, rest, s);
    else launch_vw<1, float>(a, halo, false, rest, s);
    return;
  }
  if (VW == 4) launch_vw<4>(a, halo, batched, rest, s);
  else if (VW == 2) launch_vw<2>(a, halo, batched, rest, s);
  else launch_vw<1>(a, halo, batched, rest, s);
}

}  // namespace wl

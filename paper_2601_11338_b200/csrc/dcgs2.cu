// dcgs2.cu — the two basis passes of the DCGS2 Arnoldi step (step a5): bulk-copy ring kernels.
//
// Per Arnoldi step j (see misc.cu dcgs2_coeffs_kernel for the algebra):
//   pass A (dcgs2_dots):   a_i = q_i.p_j, b_i = q_i.w (i < j), α = p.p, β = p.w, γ = w.w
//   pass B (dcgs2_update): q_j = cq_p p + Σ cq_i q_i      -> spare slot (never aliases p_j)
//                          p_{j+1} = cp_w w + cp_p p + Σ cp_i q_i
// with w = Z p_j = (p_j,bottom ; S), S the SpMM output.  Both passes stream the basis once: they
// are HBM streams of j+2..j+4 vectors, nothing else.
//
// Design (measured on B200, tools/stream_bench.cu): a register-streaming kernel cannot keep the
// ~190 KB per SM in flight that HBM3e needs once 30+ streams each want several loads in flight per
// thread (best register variant: 4.2-4.9 TB/s here).  So both passes run ONE persistent CTA per SM
// in which a producer warp streams every operand of a tile — 16 KB pieces of p_j, w and each basis
// vector — into a 12-stage shared-memory ring with bulk copies (cp.async.bulk, completion on
// per-stage mbarriers) and consumer warps fold each piece into registers and release the stage
// (empty mbarrier, no block-wide barrier).  192 KB per SM are in flight without holding a register.
// Tile = E = tpb * PER elements with tpb = floor(consumers / B) * B: consumer thread t owns the
// elements t + i*tpb (i < PER) of every tile, all of column t % B (row-major n x B blocks), so its
// accumulators never mix columns.  Bulk copies need 16-byte aligned, 16-byte multiple pieces:
// the engine pads each half of a Z vector to an even element count (zero phantom row).
// Basis vectors come from a pointer table in the kernel parameters, which lets the engine rotate
// slots instead of overwriting p_j in place.  Reductions are deterministic: per-CTA partials in a
// fixed order, then reduce_partials (gram.cu).
#include "wl_internal.cuh"

#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace wl {
namespace {

constexpr int kMaxVecPerLaunch = 32;  // longer bases are tiled by the launchers

// pass A keeps 2 x 32 dot accumulators per thread, so it runs 128 consumers x 16 elements (5 warps: 255 registers per thread);
// pass B 512 consumers x 4 elements.
constexpr int kDotsConsumers = 128, kDotsPer = 16;
static_assert(kDotsConsumers * kDotsPer <= 2048, "dots: unpredicated basis loads stay inside one ring stage");
constexpr int kStageElems = 2048;  // double stages (the DCGS2 2n-vector passes)
constexpr int kUpdConsumers = 512, kUpdPer = 4;
// A stage is 16 KB: 2048 doubles, or 4096 floats (opts.fp32 storage), whose consumers own twice the elements per
// thread (PER<T>) — same copies, barriers and bytes in flight (192 KB per SM) per byte for either type.
constexpr int kStages = 12;
constexpr int kRingBytes = kStages * 16384;  // 192 KB per SM
constexpr int kMaxStages = 24;
// a ring of SE-element stages of T: as many as fit kRingBytes (the dots pass keeps 2048-element stages, so float
// storage runs 24 stages of 8 KB; the float update 12 of 16 KB)
template <class T, int SE>
__host__ __device__ constexpr int ring_stages() { return kRingBytes / (SE * (int)sizeof(T)); }
template <class T>
__host__ __device__ constexpr int stage_elems() { return 16384 / (int)sizeof(T); }
// float storage tunables (tools/build_variants.sh): elements per dots thread; update consumers and elements
#ifndef WL_DOTS_F_PER
#define WL_DOTS_F_PER 16
#endif
#ifndef WL_DOTS_F_SPLIT
#define WL_DOTS_F_SPLIT 1  // measured: 2 and 4 chains are slower (registers)
#endif
#ifndef WL_UPD_F_CONSUMERS
#define WL_UPD_F_CONSUMERS 480
#endif
#ifndef WL_UPD_F_PER
#define WL_UPD_F_PER 12  // with 24 KB stages: C4 fp32 update 28.2 -> 26.6 ms/step (0.88 -> 0.93 of HBM)
#endif
#ifndef WL_UPD_F_SE
#define WL_UPD_F_SE 6144
#endif
// double toar_update: 512 consumers x WL_UPD_D_PER elements in WL_UPD_D_SE-element stages
#ifndef WL_UPD_D_PER
#define WL_UPD_D_PER 6  // 24 KB stages: C4 update 50.6 -> 49.5 ms/step (0.98 -> 1.00 of the measured copy bandwidth)
#endif
#ifndef WL_UPD_D_SE
#define WL_UPD_D_SE 3072
#endif
// 1: the float update accumulates in float (coefficients rounded to float: one FFMA per element and output);
// 0: in double (one float -> double conversion per element on the XU pipe, NOUT DFMA)
#ifndef WL_UPD_F_ACC32
#define WL_UPD_F_ACC32 1
#endif
// float dot pass: 192 consumers x 16 elements in 16 KB stages (C4 fp32: 0.78 -> 0.98 of HBM; 128 x 16 in 8 KB
// stages was issue/fetch bound — twice the ring operations per byte of the double pass)
#ifndef WL_DOTS_F_CONSUMERS
#define WL_DOTS_F_CONSUMERS 192
#endif
#ifndef WL_DOTS_F_SE
#define WL_DOTS_F_SE 4096  // float dot-pass stage (elements); the ring holds 192 KB / (4 SE) stages
#endif
template <class T>
__host__ __device__ constexpr int dots_per() { return sizeof(T) == 8 ? kDotsPer : WL_DOTS_F_PER; }
// double dot pass: 192 consumers x 16 elements in 24 KB stages (C4: 45.7 -> 43.1 ms/step; C3 sweep 159 -> 152 ms)
#ifndef WL_DOTS_D_CONSUMERS
#define WL_DOTS_D_CONSUMERS 192
#endif
#ifndef WL_DOTS_D_SE
#define WL_DOTS_D_SE 3072
#endif
static_assert(WL_DOTS_D_CONSUMERS * 16 <= WL_DOTS_D_SE, "double dots tiles fit a stage");
template <class T>
__host__ __device__ constexpr int dots_consumers() { return sizeof(T) == 8 ? WL_DOTS_D_CONSUMERS : WL_DOTS_F_CONSUMERS; }
static_assert(WL_DOTS_F_CONSUMERS * WL_DOTS_F_PER <= WL_DOTS_F_SE, "float dots tiles fit a stage");
// toar_update with float storage: 480 consumers x 12 elements (22 KB tiles in 24 KB stages; 16 warps, up to 128
// registers), double: 512 x 4
template <class T>
__host__ __device__ constexpr int upd_consumers() { return sizeof(T) == 8 ? kUpdConsumers : WL_UPD_F_CONSUMERS; }
template <class T>
__host__ __device__ constexpr int upd_per() { return sizeof(T) == 8 ? WL_UPD_D_PER : WL_UPD_F_PER; }
static_assert(WL_UPD_F_CONSUMERS * WL_UPD_F_PER <= WL_UPD_F_SE && kUpdConsumers * WL_UPD_D_PER <= WL_UPD_D_SE, "update tiles fit a stage");
constexpr int kRedBatch = 24;                       // dots epilogue: values per smem round

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT_%=;\n}" ::"r"(bar),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, int bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// Producer: item sequence per tile = [X0, X1, q_0 .. q_{nq-1}]; X1 may be two-source (wa | wb).
template <class T, int SE>
__device__ __forceinline__ void ring_produce(const Dcgs2Args& a, const T* X0, const T* X1a, const T* X1b,
                             int64_t h, int E, T* ring, uint64_t* full, uint64_t* empty) {
  constexpr int kStages = ring_stages<T, SE>();
  constexpr int sz = (int)sizeof(T);
  const int64_t N = a.len * a.B;
  int s = 0;
  uint32_t ph = 0;
  int64_t it = 0;
  const int nitems = a.nq + (X0 ? 1 : 0) + (X1a ? 1 : 0);
  for (int64_t e0 = (int64_t)blockIdx.x * E; e0 < N; e0 += (int64_t)gridDim.x * E) {
    const int cnt = (int)min((int64_t)E, N - e0);
    for (int item = 0; item < nitems; ++item, ++it) {
      if (it >= kStages) mbar_wait(su32(&empty[s]), ph ^ 1);
      const uint32_t bar = su32(&full[s]);
      const uint32_t dst = su32(ring + (int64_t)s * SE);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(cnt * sz) : "memory");
      const int qi = item - (X0 ? 1 : 0) - (X1a ? 1 : 0);
      if (X0 && item == 0) {
        bulk_g2s(dst, X0 + e0, cnt * sz, bar);
      } else if (qi < 0) {  // X1, possibly straddling the two sources at h
        if (X1b == nullptr || e0 + cnt <= h) {
          bulk_g2s(dst, X1a + e0, cnt * sz, bar);
        } else if (e0 >= h) {
          bulk_g2s(dst, X1b + (e0 - h), cnt * sz, bar);
        } else {
          const int c1 = (int)(h - e0);
          bulk_g2s(dst, X1a + e0, c1 * sz, bar);
          bulk_g2s(dst + c1 * sz, X1b, (cnt - c1) * sz, bar);
        }
      } else {
        bulk_g2s(dst, reinterpret_cast<const T*>(a.Q.p[qi]) + e0, cnt * sz, bar);
      }
      if (++s == kStages) { s = 0; ph ^= 1; }
    }
  }
}

template <class T, int SE>
struct RingCursor {
  static constexpr int kStages = ring_stages<T, SE>();
  int s = 0;
  uint32_t ph = 0;
  __device__ const T* acquire(T* ring, uint64_t* full) {
    mbar_wait(su32(&full[s]), ph);
    return ring + (int64_t)s * SE;
  }
  __device__ void release(uint64_t* empty, int lane) {
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
    if (++s == kStages) { s = 0; ph ^= 1; }
  }
};

__device__ __forceinline__ void ring_init(uint64_t* full, uint64_t* empty, int consumer_warps, int nstages) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < nstages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(consumer_warps));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
}

// pass A: items [P, w?, q_0..q_{nq-1}]; T = the storage type (values are converted and summed in double)
template <class T>
__global__ void __launch_bounds__(dots_consumers<T>() + 32, 1) dcgs2_dots_ring(Dcgs2Args a, int tpb) {
  constexpr int kCons = dots_consumers<T>();
  constexpr int SE = sizeof(T) == 8 ? WL_DOTS_D_SE : WL_DOTS_F_SE;
  constexpr int kStages = ring_stages<T, SE>();
  extern __shared__ __align__(128) double ring_raw[];
  T* ring = reinterpret_cast<T*>(ring_raw);
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, t = threadIdx.x;
  const int B = a.B, nq = a.nq;
  constexpr int PER = dots_per<T>();
  constexpr bool kF32 = sizeof(T) == 4;
  const int E = tpb * PER;
  const int64_t N = a.len * a.B, h = a.split * a.B;
  const bool has_w = a.wa != nullptr;
  ring_init(full, empty, kCons / 32, kStages);
  // the basis loads below carry no bounds predicate (fewer instructions in the 32x-unrolled loop:
  // less icache pressure).  Entries they read past a ragged tile's end, or past E for a lane beyond
  // tpb, meet p = w = 0 and must be finite: zero [E, stage end) of every stage, and the whole ring in
  // the one CTA that owns the ragged last tile (elsewhere the ring only ever holds basis values)
  {
    const int64_t last = (N - 1) / E;
    const bool ragged = N % E != 0 && last % gridDim.x == blockIdx.x;
    for (int st = 0; st < kStages; ++st)
      for (int i = (ragged ? 0 : E) + t; i < SE; i += blockDim.x) ring[(int64_t)st * SE + i] = T(0);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  double acc[2 * kMaxVecPerLaunch], alpha = 0.0, beta = 0.0, gamma = 0.0;
#pragma unroll
  for (int v = 0; v < 2 * kMaxVecPerLaunch; ++v) acc[v] = 0.0;
  if (warp == kCons / 32) {
    if (lane == 0)
      ring_produce<T, SE>(a, reinterpret_cast<const T*>(a.P), has_w ? reinterpret_cast<const T*>(a.wa) : nullptr,
                      reinterpret_cast<const T*>(a.wb), h, E, ring, full, empty);
  } else {
    RingCursor<T, SE> cur;
    const bool act = t < tpb;
    for (int64_t e0 = (int64_t)blockIdx.x * E; e0 < N; e0 += (int64_t)gridDim.x * E) {
      const int cnt = (int)min((int64_t)E, N - e0);
      // the tile's values; with float storage the products of one tile (PER = 32 per thread) are summed in
      // float and each tile partial is added to the double accumulators (one conversion per tile and vector)
      T pv[PER], wv[PER];
      {
        const T* st = cur.acquire(ring, full);
#pragma unroll
        for (int i = 0; i < PER; ++i) pv[i] = (act && t + i * tpb < cnt) ? st[t + i * tpb] : T(0);
        cur.release(empty, lane);
      }
      if (has_w) {
        const T* st = cur.acquire(ring, full);
#pragma unroll
        for (int i = 0; i < PER; ++i) wv[i] = (act && t + i * tpb < cnt) ? st[t + i * tpb] : T(0);
        cur.release(empty, lane);
      } else {
#pragma unroll
        for (int i = 0; i < PER; ++i) wv[i] = T(0);
      }
      {
        T al = kF32 ? T(0) : T(alpha), be = kF32 ? T(0) : T(beta), ga = kF32 ? T(0) : T(gamma);
#pragma unroll
        for (int i = 0; i < PER; ++i) {
          al += pv[i] * pv[i];
          be += pv[i] * wv[i];
          ga += wv[i] * wv[i];
        }
        alpha = kF32 ? alpha + (double)al : (double)al;
        beta = kF32 ? beta + (double)be : (double)be;
        gamma = kF32 ? gamma + (double)ga : (double)ga;
      }
#pragma unroll 32
      for (int j = 0; j < kMaxVecPerLaunch; ++j) {
        if (j < nq) {
          const T* st = cur.acquire(ring, full);
          // double: straight into the running sums (the fp64 path's order); float: per-tile partials in NS
          // independent chains (shorter FFMA dependency chains)
          constexpr int NS = kF32 ? WL_DOTS_F_SPLIT : 1;
          T sa[NS], sb[NS];
#pragma unroll
          for (int u = 0; u < NS; ++u) {
            sa[u] = (kF32 || u) ? T(0) : T(acc[2 * j]);
            sb[u] = (kF32 || u) ? T(0) : T(acc[2 * j + 1]);
          }
#pragma unroll
          for (int i = 0; i < PER; ++i) {
            const T q = st[t + i * tpb];  // t + (PER - 1) tpb < SE for every B
            sa[i % NS] += q * pv[i];
            sb[i % NS] += q * wv[i];
          }
#pragma unroll
          for (int u = 1; u < NS; ++u) {
            sa[0] += sa[u];
            sb[0] += sb[u];
          }
          acc[2 * j] = kF32 ? acc[2 * j] + (double)sa[0] : (double)sa[0];
          acc[2 * j + 1] = kF32 ? acc[2 * j + 1] + (double)sb[0] : (double)sb[0];
          cur.release(empty, lane);
        }
      }
    }
  }
  __syncthreads();  // every copy has landed and been consumed: the ring is free
  // epilogue: per (value, column) sum over the consumer threads of that column, fixed order
  const int nval = 2 * nq + 3;
  double* red = ring_raw;  // [kRedBatch][kCons]
  for (int v0 = 0; v0 < nval; v0 += kRedBatch) {
    if (t < kCons) {
#pragma unroll
      for (int u = 0; u < 2 * kMaxVecPerLaunch; ++u)
        if (u < 2 * nq && u >= v0 && u < v0 + kRedBatch) red[(u - v0) * kCons + t] = acc[u];
      if (2 * nq >= v0 && 2 * nq < v0 + kRedBatch) red[(2 * nq - v0) * kCons + t] = alpha;
      if (2 * nq + 1 >= v0 && 2 * nq + 1 < v0 + kRedBatch) red[(2 * nq + 1 - v0) * kCons + t] = beta;
      if (2 * nq + 2 >= v0 && 2 * nq + 2 < v0 + kRedBatch) red[(2 * nq + 2 - v0) * kCons + t] = gamma;
    }
    __syncthreads();
    const int nv = min(kRedBatch, nval - v0);
    for (int idx = warp; idx < nv * B; idx += blockDim.x / 32) {  // a warp per output, fixed-order tree
      const int vv = idx / B, c = idx - vv * B;
      double sum = 0.0;
      for (int tt = c + lane * B; tt < tpb; tt += 32 * B) sum += red[vv * kCons + tt];
      for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
      if (lane == 0) a.partials[(int64_t)((v0 + vv) * B + c) * gridDim.x + blockIdx.x] = sum;
    }
    __syncthreads();
  }
}

// pass B: items [X0, X1, q_0..q_{nq-1}];  q_j = a0 X0 + Σ cq_i q_i,  p_{j+1} = a1 X0 + a2 X1 + Σ cp_i q_i
// (X0, X1) = (p_j, w) with (a0, a1, a2) = (cq_p, cp_p, cp_w), or (Qout, Pnext) with (1, 0, 1)
// for the vector tiles after the first (accumulate).
__global__ void __launch_bounds__(kUpdConsumers + 32, 1) dcgs2_update_ring(Dcgs2Args a, int tpb) {  // double storage
  extern __shared__ __align__(128) double ring[];
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
  __shared__ double coef[2 * kMaxVecPerLaunch * kMaxCols];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, t = threadIdx.x;
  const int B = a.B, nq = a.nq;
  const int E = tpb * kUpdPer;
  const int64_t N = a.len * a.B, h = a.split * a.B;
  for (int i = t; i < 2 * nq * B; i += blockDim.x) coef[i] = a.coef_v[i];
  ring_init(full, empty, kUpdConsumers / 32, ring_stages<double, kStageElems>());
  __syncthreads();
  if (warp == kUpdConsumers / 32) {
    if (lane == 0) {
      if (a.accumulate) ring_produce<double, kStageElems>(a, a.Qout, a.Pnext, nullptr, h, E, ring, full, empty);
      else ring_produce<double, kStageElems>(a, a.P, a.wa, a.wb, h, E, ring, full, empty);
    }
    return;
  }
  const bool act = t < tpb;
  const int c = t % B;
  double a0, a1, a2;
  bool dead = false;
  if (a.accumulate) { a0 = 1.0; a1 = 0.0; a2 = 1.0; }
  else {
    a0 = a.coef_s[c]; a1 = a.coef_s[B + c]; a2 = a.coef_s[2 * B + c];
    dead = a0 == 0.0;
  }
  RingCursor<double, kStageElems> cur;
  for (int64_t e0 = (int64_t)blockIdx.x * E; e0 < N; e0 += (int64_t)gridDim.x * E) {
    const int cnt = (int)min((int64_t)E, N - e0);
    double sq[kUpdPer], sp[kUpdPer];
    {
      const double* st = cur.acquire(ring, full);
#pragma unroll
      for (int i = 0; i < kUpdPer; ++i) {
        const double x = (act && t + i * tpb < cnt) ? st[t + i * tpb] : 0.0;
        sq[i] = a0 * x;
        sp[i] = a1 * x;
      }
      cur.release(empty, lane);
    }
    {
      const double* st = cur.acquire(ring, full);
#pragma unroll
      for (int i = 0; i < kUpdPer; ++i) sp[i] += a2 * ((act && t + i * tpb < cnt) ? st[t + i * tpb] : 0.0);
      cur.release(empty, lane);
    }
    for (int j = 0; j < nq; ++j) {
      const double cq = coef[(2 * j) * B + c], cp = coef[(2 * j + 1) * B + c];
      const double* st = cur.acquire(ring, full);
#pragma unroll
      for (int i = 0; i < kUpdPer; ++i) {
        const double q = (act && t + i * tpb < cnt) ? st[t + i * tpb] : 0.0;
        sq[i] += cq * q;
        sp[i] += cp * q;
      }
      cur.release(empty, lane);
    }
    if (act) {
#pragma unroll
      for (int i = 0; i < kUpdPer; ++i)
        if (t + i * tpb < cnt) {
          a.Qout[e0 + t + i * tpb] = dead ? 0.0 : sq[i];
          a.Pnext[e0 + t + i * tpb] = dead ? 0.0 : sp[i];
        }
    }
  }
}


// ---- TOAR basis update (engine.cu toar_chunk): out_o = Σ_b cb[b][o] base_b + Σ_i co[o][i] U_i --------
// Items per tile: the bases (y for the first vector tile; the outputs themselves, identity
// coefficients, for later tiles of > 32 vectors) then U_0..U_{m-1}.  Same ring as pass B.
constexpr int kToarMaxOut = 3;
template <int NOUT, class T>
__global__ void __launch_bounds__(upd_consumers<T>() + 32, 1) toar_update_ring(ToarArgs a, int tpb) {
  constexpr int SE = sizeof(T) == 8 ? WL_UPD_D_SE : WL_UPD_F_SE;
  constexpr int kStages = ring_stages<T, SE>();
  constexpr int PER = upd_per<T>();
  extern __shared__ __align__(128) double ring_raw[];
  T* ring = reinterpret_cast<T*>(ring_raw);
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
  __shared__ double coef[NOUT * kMaxVecPerLaunch * kMaxCols];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, t = threadIdx.x;
  const int B = a.B, m = a.m;
  const int E = tpb * PER;
  const int64_t N = a.len * a.B;
  const int nb = a.accumulate ? NOUT : 1;
  for (int i = t; i < NOUT * m * B; i += blockDim.x) {
    const int o = i / (m * B), r = i - o * m * B;
    coef[i] = a.coef_u[(int64_t)(o * a.coef_ld) * B + r];
  }
  ring_init(full, empty, upd_consumers<T>() / 32, kStages);
  __syncthreads();
  if (warp == upd_consumers<T>() / 32) {
    if (lane == 0) {  // producer: items [bases..., U_0..U_{m-1}] per tile
      int s = 0;
      uint32_t ph = 0;
      int64_t it = 0;
      for (int64_t e0 = (int64_t)blockIdx.x * E; e0 < N; e0 += (int64_t)gridDim.x * E) {
        const int cnt = (int)min((int64_t)E, N - e0);
        for (int item = 0; item < nb + m; ++item, ++it) {
          if (it >= kStages) mbar_wait(su32(&empty[s]), ph ^ 1);
          const uint32_t bar = su32(&full[s]);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(cnt * (int)sizeof(T))
                       : "memory");
          const T* src = reinterpret_cast<const T*>(item < nb ? (a.accumulate ? a.out[item] : a.y) : a.U.p[item - nb]);
          bulk_g2s(su32(ring + (int64_t)s * SE), src + e0, cnt * (int)sizeof(T), bar);
          if (++s == kStages) { s = 0; ph ^= 1; }
        }
      }
    }
    return;
  }
  const bool act = t < tpb;
  const int c = t % B;
  // accumulator type: double, or float for float storage with WL_UPD_F_ACC32 (the outputs are rounded to float
  // anyway; the m + 1 <= 33 terms add ~sqrt(m) roundings of the size of the stored inputs' own)
  using Acc = typename std::conditional<sizeof(T) == 4 && WL_UPD_F_ACC32, float, double>::type;
  Acc cy[NOUT];
#pragma unroll
  for (int o = 0; o < NOUT; ++o) cy[o] = (Acc)a.coef_y[o * B + c];
  RingCursor<T, SE> cur;
  for (int64_t e0 = (int64_t)blockIdx.x * E; e0 < N; e0 += (int64_t)gridDim.x * E) {
    const int cnt = (int)min((int64_t)E, N - e0);
    Acc acc[NOUT][PER];
#pragma unroll
    for (int o = 0; o < NOUT; ++o)
#pragma unroll
      for (int i = 0; i < PER; ++i) acc[o][i] = Acc(0);
    for (int b = 0; b < nb; ++b) {
      const T* st = cur.acquire(ring, full);
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const Acc v = (act && t + i * tpb < cnt) ? (Acc)st[t + i * tpb] : Acc(0);
#pragma unroll
        for (int o = 0; o < NOUT; ++o) acc[o][i] += (a.accumulate ? (o == b ? Acc(1) : Acc(0)) : cy[o]) * v;
      }
      cur.release(empty, lane);
    }
    for (int j = 0; j < m; ++j) {
      Acc cj[NOUT];
#pragma unroll
      for (int o = 0; o < NOUT; ++o) cj[o] = (Acc)coef[(o * m + j) * B + c];
      const T* st = cur.acquire(ring, full);
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const Acc v = (act && t + i * tpb < cnt) ? (Acc)st[t + i * tpb] : Acc(0);
#pragma unroll
        for (int o = 0; o < NOUT; ++o) acc[o][i] += cj[o] * v;
      }
      cur.release(empty, lane);
    }
    if (act) {
      // element e = e0 + t + i*tpb is (row e / B, column c); tpb and E are multiples of B, so the row is
      // e0/B + t/B + i*(tpb/B) — outputs with a padded row stride (out_ld) are addressed from it
      const int64_t r0 = e0 / B + t / B;
#pragma unroll
      for (int i = 0; i < PER; ++i)
        if (t + i * tpb < cnt) {
#pragma unroll
          for (int o = 0; o < NOUT; ++o) {
            T* out = reinterpret_cast<T*>(a.out[o]);
            if (a.out_ld[o] > B) {
              T* row = out + (r0 + (int64_t)i * (tpb / B)) * a.out_ld[o];
              row[c] = (T)acc[o][i];
              // the phantom columns too: whole 32-byte sectors reach L2, so DRAM sees no partial-sector writes
              // (spread over the row's threads: column c writes phantoms B + c, B + c + B, ...)
              for (int cc = B + c; cc < pad_vec_t<T>(B); cc += B) row[cc] = T(0);
            } else {
              out[e0 + t + i * tpb] = (T)acc[o][i];
            }
          }
        }
    }
  }
}

size_t ring_smem() { return (size_t)kRingBytes; }  // every ring

VecPtrs shifted(const VecPtrs& v, int i0) {
  VecPtrs r{};
  for (int k = 0; k + i0 < kMaxVecSlots; ++k) r.p[k] = v.p[k + i0];
  return r;
}

}  // namespace

// pass A for nq <= 32 per launch; longer bases tile the vectors: tile [i0, i1) writes its a/b
// pairs at offset 2*i0 and its trailing α/β/γ are overwritten by the next tile.
int dcgs2_dots(Dcgs2Args a, cudaStream_t s) {
  if (a.nq > kMaxVecPerLaunch) {
    if (!a.sums_out) throw Error(1, "dcgs2_dots: tiled passes (> 32 vectors) need sums_out");
    for (int i0 = 0; i0 < a.nq; i0 += kMaxVecPerLaunch) {
      Dcgs2Args t = a;
      t.nq = std::min(kMaxVecPerLaunch, a.nq - i0);
      t.Q = shifted(a.Q, i0);
      t.sums_out = a.sums_out + (int64_t)2 * i0 * a.B;
      dcgs2_dots(t, s);
    }
    return 0;
  }
  WL_LAUNCH("dcgs2_dots");
  {
    if ((a.split * a.B) % 2) throw Error(1, "dcgs2: half length must be even (phantom row)");
    if (a.f32 && (a.split * a.B) % 4) throw Error(1, "dcgs2: fp32 half length must be a multiple of 4 elements");
    auto kern = a.f32 ? dcgs2_dots_ring<float> : dcgs2_dots_ring<double>;
    static bool attr[2] = {false, false};
    if (!attr[a.f32 ? 1 : 0]) {
      WL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ring_smem()));
      attr[a.f32 ? 1 : 0] = true;
    }
    const int nc = a.f32 ? dots_consumers<float>() : dots_consumers<double>();
    const int tpb = nc / a.B * a.B;
    const int64_t N = a.len * a.B;
    // one persistent CTA per SM; an empty rank (N = 0) still launches one CTA so its partials are zeros
    const int E = tpb * (a.f32 ? dots_per<float>() : dots_per<double>());
    a.grid = (int)std::max<int64_t>(1, std::min<int64_t>(num_sms(), (N + E - 1) / E));
    kern<<<a.grid, nc + 32, ring_smem(), s>>>(a, tpb);
    WL_CUDA(cudaGetLastError());
    if (a.sums_out) {  // null: the consumer reduces the partials itself (a.grid of them per output)
      note_launch("gram_reduce");
      reduce_partials(a.partials, (2 * a.nq + 3) * a.B, a.grid, a.sums_out, s);
    }
    return a.grid;
  }
}

void dcgs2_update(Dcgs2Args a, cudaStream_t s) {
  if (a.f32) throw Error(1, "dcgs2_update: double storage only (the fp32 mode runs TOAR)");
  if (a.nq > kMaxVecPerLaunch) {
    for (int i0 = 0; i0 < a.nq; i0 += kMaxVecPerLaunch) {
      Dcgs2Args t = a;
      t.nq = std::min(kMaxVecPerLaunch, a.nq - i0);
      t.Q = shifted(a.Q, i0);
      t.coef_v = a.coef_v + (int64_t)2 * i0 * a.B;
      t.accumulate = i0 > 0 ? 1 : a.accumulate;
      dcgs2_update(t, s);
    }
    return;
  }
  WL_LAUNCH("dcgs2_update");
  {
    if ((a.split * a.B) % 2) throw Error(1, "dcgs2: half length must be even (phantom row)");
    static bool attr = false;
    if (!attr) {
      WL_CUDA(cudaFuncSetAttribute(dcgs2_update_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ring_smem()));
      attr = true;
    }
    const int tpb = kUpdConsumers / a.B * a.B;
    const int64_t N = a.len * a.B;
    const int grid = (int)std::min<int64_t>(num_sms(), (N + tpb * kUpdPer - 1) / (tpb * kUpdPer));
    if (grid == 0) return;  // empty rank
    dcgs2_update_ring<<<grid, kUpdConsumers + 32, ring_smem(), s>>>(a, tpb);
    WL_CUDA(cudaGetLastError());
  }
}

// outputs = linear combinations of one base vector and the basis U (TOAR, engine.cu).  Bases of more
// than 32 vectors are tiled: tiles after the first read the outputs back as their bases.
void toar_update(ToarArgs a, cudaStream_t s) {
  if (a.nout < 1 || a.nout > kToarMaxOut) throw Error(1, "toar_update: 1..3 outputs");
  if (a.m > kMaxVecPerLaunch) {
    for (int o = 0; o < a.nout; ++o)
      if (a.out_ld[o] > a.B) throw Error(1, "toar_update: padded outputs need m <= 32 (tiles read outputs back)");
    for (int i0 = 0; i0 < a.m; i0 += kMaxVecPerLaunch) {
      ToarArgs t = a;
      t.m = std::min(kMaxVecPerLaunch, a.m - i0);
      t.U = shifted(a.U, i0);
      t.coef_u = a.coef_u + (int64_t)i0 * a.B;
      t.accumulate = i0 > 0 ? 1 : a.accumulate;
      toar_update(t, s);
    }
    return;
  }
  WL_LAUNCH("toar_update");
  if ((a.len * a.B) % (a.f32 ? 4 : 2)) throw Error(1, "toar_update: vector length must be a multiple of 16 bytes (phantom rows)");
  static bool attr[2][kToarMaxOut + 1] = {};
  auto kern = a.f32 ? (a.nout == 1 ? toar_update_ring<1, float> : a.nout == 2 ? toar_update_ring<2, float>
                                                                              : toar_update_ring<3, float>)
                    : (a.nout == 1 ? toar_update_ring<1, double> : a.nout == 2 ? toar_update_ring<2, double>
                                                                                : toar_update_ring<3, double>);
  if (!attr[a.f32 ? 1 : 0][a.nout]) {
    WL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ring_smem()));
    attr[a.f32 ? 1 : 0][a.nout] = true;
  }
  const int nc = a.f32 ? upd_consumers<float>() : upd_consumers<double>();
  const int tpb = nc / a.B * a.B;
  const int64_t N = a.len * a.B;
  const int E = tpb * (a.f32 ? upd_per<float>() : upd_per<double>());
  const int grid = (int)std::min<int64_t>(num_sms(), (N + E - 1) / E);
  if (grid == 0) return;  // empty rank
  kern<<<grid, nc + 32, ring_smem(), s>>>(a, tpb);
  WL_CUDA(cudaGetLastError());
}

}  // namespace wl

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
//   medium rows (32 < deg <= 1024): one warp per row, its lane groups split the nonzeros and are
//               reduced with shuffles;
//   hub rows    (deg > 1024): split into 1024-nonzero chunks, one warp per chunk; each chunk writes
//               a partial and the last chunk to finish (per-row ticket) sums the row's partials in
//               chunk order — deterministic, no second launch.
// Every lane issues up to 8 independent gathers before consuming them (ILP), and all control flow
// is uniform within a lane group.
#include "wl_internal.cuh"

namespace wl {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kU = 8;  // gathers in flight per lane

struct Ctx {
  const SpmvArgs& a;
  int c;
  double g0, g1, sc;
  __device__ double gather(int cl) const {
    return cl < a.n_loc ? __ldg(a.y + (int64_t)cl * a.ldy + c)
                        : __ldg(a.yh + (int64_t)(cl - a.n_loc) * a.ldh + c);
  }
  __device__ void write(int r, int deg, double sum) const {
    double o = sum;
    if (a.x) o += (g0 + g1 * (double)deg) * a.x[(int64_t)r * a.ldx + c];
    a.out[(int64_t)r * a.ldo + c] = sc * o;
  }
  // Σ y[col[z]] for z = z0 + first, z0 + first + step, ... < z1 (step = lane groups sharing the row)
  __device__ double strided_sum(int z0, int z1, int first, int step) const {
    double acc = 0.0;
    for (int z = z0 + first; z < z1; z += kU * step) {  // kU predicated gathers in flight
      int cl[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int zz = z + u * step;
        cl[u] = zz < z1 ? __ldg(a.col + zz) : -1;
      }
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

__global__ void __launch_bounds__(kThreads) spmv_binned_kernel(SpmvArgs a) {
  const int B = a.B;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gpw = 32 / B;
  const int gi = lane / B, c = lane - gi * B;
  const bool lane_ok = gi < gpw;
  const int cc = lane_ok ? c : 0;
  Ctx ctx{a, cc, a.g0 ? a.g0[cc] : 0.0, a.g1 ? a.g1[cc] : 0.0, a.scale ? a.scale[cc] : 1.0};
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
  {  // ---- hub rows: one warp per 1024-nonzero chunk, last chunk of the row reduces in order
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
  WL_LAUNCH("spmv_binned");
  spmv_binned_kernel<<<grid, kThreads, 0, s>>>(a);
  WL_CUDA(cudaGetLastError());
}

}  // namespace wl

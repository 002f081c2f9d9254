// spmv.cu — fused companion-operator SpMM (step a4 of DESIGN.md).
//
// One application of Z = [[O, I], [μ(μI - D), A]] (eq:Zdef) to a stacked block
// (x; y) needs only its bottom half  A y + μ(μ - d) ⊙ x  — the top half is y itself and is
// never copied (the Gram kernels read it in place).  This is one step of the BTDW three-term
// recurrence eq:qrec.  The seeds q_1 v = A v and q_2 v = A(Av) - μ d⊙v use the same
// kernel with (g0, g1) = (0, 0) / (0, -μ); the Z step uses (g0, g1) = (μ², -μ).  A has unit
// values, so the kernel only adds gathered rows — no value array is read.
//
// Load balance: merge-path decomposition (Merrill & Garland) of the (row-end, nnz) sequence
// into equal tiles of merge items, so a 300k-degree hub and a million isolated rows cost the
// same per tile.  A CTA (256 threads) handles one tile; it is split into "lane groups" of B
// lanes (lane c owns column c of the row-major n x B blocks), each group walking IPT
// consecutive merge items.  Gathered rows are prefetched into registers (IPT independent loads
// per lane) before the walk.  Rows split across groups are stitched in shared memory; rows
// split across tiles are stitched deterministically by spmv_fixup_kernel.
#include "wl_internal.cuh"
#include <climits>

namespace wl {
namespace {

constexpr int kThreads = 256;

__host__ __device__ inline int groups_per_cta(int B) { return (kThreads / 32) * (32 / B); }
inline int ipt_for(int B) { return B <= 2 ? 8 : (B <= 8 ? 16 : 32); }

// merge-path search on the tile-local sequence: returns rows consumed at diagonal d
__device__ inline int merge_search(int d, const int* s_rp, int nrows, int z0, int nnzt) {
  int lo = max(0, d - nnzt), hi = min(d, nrows);
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (s_rp[mid + 1] <= z0 + (d - mid - 1)) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

template <int IPT>
__global__ void __launch_bounds__(kThreads) spmv_merge_kernel(SpmvArgs a) {
  extern __shared__ int s_dyn[];
  __shared__ double s_carry[kThreads];  // groups * B <= 256
  __shared__ int s_crow[kThreads];
  __shared__ int s_cdone[kThreads];

  const int B = a.B;
  const int T = a.tile_items;
  const int t = blockIdx.x;
  const int2 c0 = a.tiles[t], c1 = a.tiles[t + 1];
  const int r0 = c0.x, z0 = c0.y;
  const int nrows = c1.x - r0, nnzt = c1.y - z0;
  int* s_rp = s_dyn;           // s_rp[i] = rowptr[r0 + i], i in [0, nrows + 1]
  int* s_col = s_dyn + T + 2;  // s_col[k] = col[z0 + k], k < nnzt

  for (int i = threadIdx.x; i <= nrows + 1; i += kThreads)
    s_rp[i] = (r0 + i <= a.n_loc) ? __ldg(a.rowptr + r0 + i) : INT_MAX;
  for (int k = threadIdx.x; k < nnzt; k += kThreads) s_col[k] = __ldg(a.col + z0 + k);
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gpw = 32 / B;
  const int gi = lane / B, c = lane - gi * B;
  const bool lane_ok = gi < gpw;
  const int g = warp * gpw + (lane_ok ? gi : 0);
  const int total = nrows + nnzt;
  const int d0 = min(g * IPT, total), d1 = min(d0 + IPT, total);
  const int x0 = merge_search(d0, s_rp, nrows, z0, nnzt), y0 = d0 - x0;
  const int x1 = merge_search(d1, s_rp, nrows, z0, nnzt), y1 = d1 - x1;

  // prefetch the gathered values of this group's nonzeros (independent loads in flight)
  double v[IPT];
#pragma unroll
  for (int p = 0; p < IPT; ++p) {
    v[p] = 0.0;
    const int k = y0 + p;
    if (lane_ok && k < y1) {
      const int cl = s_col[k];
      v[p] = cl < a.n_loc ? __ldg(a.y + (int64_t)cl * a.ldy + c)
                          : __ldg(a.yh + (int64_t)(cl - a.n_loc) * a.ldh + c);
    }
  }
  const double g0 = a.g0 ? a.g0[min(c, B - 1)] : 0.0;
  const double g1 = a.g1 ? a.g1[min(c, B - 1)] : 0.0;
  const double sc = a.scale ? a.scale[min(c, B - 1)] : 1.0;

  auto write_row = [&](int row, double val) {  // row: tile-local
    const int r = r0 + row;
    double o = val;
    if (a.x) {
      const double deg = (double)(s_rp[row + 1] - s_rp[row]);
      o += (g0 + g1 * deg) * a.x[(int64_t)r * a.ldx + c];
    }
    a.out[(int64_t)r * a.ldo + c] = sc * o;
  };

  // did earlier merge items (this or previous tiles) consume nonzeros of row x0?
  const bool started_mid = lane_ok && (z0 + y0 > s_rp[x0]);
  bool first = true, held = false;
  double hold = 0.0, acc = 0.0;
  int row = x0;
  if (lane_ok) {
#pragma unroll
    for (int p = 0; p < IPT; ++p) {
      if (y0 + p < y1) {
        const int z = z0 + y0 + p;
        while (s_rp[row + 1] <= z) {  // rows (possibly empty) that end before nonzero z
          if (first && started_mid) { hold = acc; held = true; }
          else write_row(row, acc);
          first = false;
          acc = 0.0;
          ++row;
        }
        acc += v[p];
      }
    }
    while (row < x1) {
      if (first && started_mid) { hold = acc; held = true; }
      else write_row(row, acc);
      first = false;
      acc = 0.0;
      ++row;
    }
    s_carry[g * B + c] = acc;  // partial of the row open at the group's end (row x1)
    if (c == 0) { s_crow[g] = x1; s_cdone[g] = (x1 > x0); }
  }
  __syncthreads();

  if (held) {  // stitch the first completed row with the carries of the preceding groups
    double sum = hold;
    for (int gp = g - 1; gp >= 0; --gp) {
      sum += s_carry[gp * B + c];
      if (s_cdone[gp]) break;
    }
    write_row(x0, sum);
  }
  // tile carry-out: the open row at the tile end, accumulated over the trailing groups
  const int G = groups_per_cta(B);
  if (lane_ok && g == G - 1) {
    const int r1 = c1.x;
    int crow = -1;
    double sum = 0.0;
    if (r1 < a.n_loc && c1.y > max(z0, s_rp[nrows])) {
      crow = r1;
      for (int gp = G - 1; gp >= 0; --gp) {
        sum += s_carry[gp * B + c];
        if (s_cdone[gp]) break;
      }
    }
    a.carry_val[(int64_t)t * B + c] = sum;
    if (c == 0) a.carry_row[t] = crow;
  }
}

// rows spanning several tiles: the first tile of each run adds the run's carries in order
__global__ void spmv_fixup_kernel(const int32_t* carry_row, const double* carry_val, int num_tiles,
                                  int B, const double* scale, double* out, int64_t ldo) {
  const int t = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int c = threadIdx.x & 31;
  if (t >= num_tiles || c >= B) return;
  const int r = carry_row[t];
  if (r < 0 || (t > 0 && carry_row[t - 1] == r)) return;
  double sum = 0.0;
  for (int u = t; u < num_tiles && carry_row[u] == r; ++u) sum += carry_val[(int64_t)u * B + c];
  const double sc = scale ? scale[c] : 1.0;
  out[(int64_t)r * ldo + c] += sc * sum;
}

__global__ void spmv_tiles_kernel(const int32_t* rowptr, int32_t n, int32_t nnz, int T, int2* tiles,
                                  int num_tiles) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > num_tiles) return;
  const int64_t d = min((int64_t)t * T, (int64_t)n + nnz);
  int64_t lo = max((int64_t)0, d - nnz), hi = min(d, (int64_t)n);
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)rowptr[mid + 1] <= d - mid - 1) lo = mid + 1;
    else hi = mid;
  }
  tiles[t] = make_int2((int)lo, (int)(d - lo));
}

}  // namespace

int spmv_tile_items(int B) { return groups_per_cta(B) * ipt_for(B); }

void spmv_tiles(const int32_t* rowptr, int32_t n, int32_t nnz, int tile_items, int2* tiles,
                int num_tiles, cudaStream_t s) {
  WL_LAUNCH("spmv_tiles");
  spmv_tiles_kernel<<<(num_tiles + 1 + 255) / 256, 256, 0, s>>>(rowptr, n, nnz, tile_items, tiles,
                                                                 num_tiles);
  WL_CUDA(cudaGetLastError());
}

void spmv(const SpmvArgs& a, cudaStream_t s) {
  if (a.B < 1 || a.B > kMaxCols) throw Error(1, "spmv: B out of range");
  if (a.tile_items != spmv_tile_items(a.B)) throw Error(1, "spmv: tile size mismatch");
  if (a.num_tiles <= 0) return;
  const size_t smem = sizeof(int) * (2 * (size_t)a.tile_items + 2);
  const int ipt = ipt_for(a.B);
  {
    WL_LAUNCH("spmv_merge");
    if (ipt == 8) spmv_merge_kernel<8><<<a.num_tiles, kThreads, smem, s>>>(a);
    else if (ipt == 16) spmv_merge_kernel<16><<<a.num_tiles, kThreads, smem, s>>>(a);
    else spmv_merge_kernel<32><<<a.num_tiles, kThreads, smem, s>>>(a);
    WL_CUDA(cudaGetLastError());
  }
  {
    WL_LAUNCH("spmv_fixup");
    spmv_fixup_kernel<<<(a.num_tiles + 7) / 8, 256, 0, s>>>(a.carry_row, a.carry_val, a.num_tiles, a.B,
                                                            a.scale, a.out, a.ldo);
    WL_CUDA(cudaGetLastError());
  }
}

}  // namespace wl

// gather_bench.cu — ceiling of random row gathers (the SpMM access pattern) on one B200.
// out[r][c] = Σ_{k<D} Y[idx[D r + k]][c],  Y: n rows x ld doubles (B = 11 used columns),
// idx uniform random (worst case: no L2 reuse).  Variants:
//   reg<U>:  lane group of B lanes per output row, U gathers in flight per lane, persistent warps
//   tma:     one producer warp issues TMA gather4 (4 rows x 96 B) into a smem ring, consumer warps sum
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_bench tools/gather_bench.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void init_kernel(double* Y, int64_t ny, int* idx, int64_t nidx, int n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ny; i += (int64_t)gridDim.x * blockDim.x) Y[i] = (double)(i % 7);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nidx; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h = i * 0x9E3779B97F4A7C15ull;
    h ^= h >> 31; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 29;
    idx[i] = (int)(h % (uint64_t)n);
  }
}

template <int U>
__global__ void __launch_bounds__(256) reg_kernel(const double* Y, int ld, const int* idx, int64_t m, int D, int B, double* out) {
  const int lane = threadIdx.x & 31, gpw = 32 / B, gi = lane / B, c = lane - gi * B;
  const bool ok = gi < gpw;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int64_t nw = (int64_t)gridDim.x * blockDim.x / 32;
  for (int64_t r = gw * gpw + gi; r - gi < m; r += nw * gpw) {
    if (!ok || r >= m) continue;
    const int* ix = idx + r * D;
    double acc = 0.0;
    for (int k = 0; k < D; k += U) {
      int cl[U];
#pragma unroll
      for (int u = 0; u < U; ++u) cl[u] = k + u < D ? __ldg(ix + k + u) : -1;
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = cl[u] >= 0 ? __ldg(Y + (int64_t)cl[u] * ld + c) : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u) acc += v[u];
    }
    out[r * B + c] = acc;
  }
}


// double2 variant: rows padded to ld (even), W = ld/2 lanes per row, each lane loads 16 bytes
template <int U>
__global__ void __launch_bounds__(256) reg2_kernel(const double* Y, int ld, const int* idx, int64_t m, int D, int B, double* out) {
  const int W = ld / 2;
  const int lane = threadIdx.x & 31, gpw = 32 / W, gi = lane / W, c = lane - gi * W;
  const bool ok = gi < gpw;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int64_t nw = (int64_t)gridDim.x * blockDim.x / 32;
  for (int64_t r = gw * gpw + gi; r - gi < m; r += nw * gpw) {
    if (!ok || r >= m) continue;
    const int* ix = idx + r * D;
    double2 acc = make_double2(0.0, 0.0);
    for (int k = 0; k < D; k += U) {
      int cl[U];
#pragma unroll
      for (int u = 0; u < U; ++u) cl[u] = k + u < D ? __ldg(ix + k + u) : -1;
      double2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = cl[u] >= 0 ? __ldg(reinterpret_cast<const double2*>(Y + (int64_t)cl[u] * ld) + c) : make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; }
    }
    if (2 * c < B) out[r * B + 2 * c] = acc.x;
    if (2 * c + 1 < B) out[r * B + 2 * c + 1] = acc.y;
  }
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(bar), "r"(ph) : "memory");
}

// stage = 32 rows (8 gather4) of ROWB bytes; consumers: lane group per output row as above but reading smem
template <int S>
__global__ void __launch_bounds__(288, 1) tma_kernel(const __grid_constant__ CUtensorMap tmap, const int* idx, int64_t m, int D, int B, int ldp, double* out) {
  extern __shared__ __align__(1024) double ring[];
  __shared__ __align__(8) uint64_t full[S], empty[S];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int stage_d = 32 * ldp;  // doubles per stage
  // work: this CTA's output rows [r0, r1), nnz range contiguous: items of 32 nnz
  const int64_t per = (m + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * per, r1 = min(m, r0 + per);
  if (r0 >= r1) return;
  const int64_t z0 = r0 * D, z1 = r1 * D;
  const int64_t nitems = (z1 - z0 + 31) / 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(su32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 8) {  // producer warp: lane k loads index k of the item; lanes 0..7 issue one gather4 each
    int s = 0; uint32_t ph = 0;
    int nxt = z0 + lane < z1 ? __ldg(idx + z0 + lane) : 0;
    for (int64_t it = 0; it < nitems; ++it) {
      const int cur = nxt;
      const int64_t zn = z0 + (it + 1) * 32 + lane;
      nxt = zn < z1 ? __ldg(idx + zn) : 0;
      if (it >= S) mbar_wait(su32(&empty[s]), ph ^ 1);
      const uint32_t bar = su32(&full[s]);
      if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(32 * ldp * 8) : "memory");
      int rr[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) rr[q] = __shfl_sync(0xffffffffu, cur, (lane * 4 + q) & 31);
      if (lane < 8) {
        const uint32_t dst = su32(ring + (int64_t)s * stage_d + lane * 4 * ldp);
        asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                     ::"r"(dst), "l"(&tmap), "r"(0), "r"(rr[0]), "r"(rr[1]), "r"(rr[2]), "r"(rr[3]), "r"(bar) : "memory");
      }
      if (++s == S) { s = 0; ph ^= 1; }
    }
    return;
  }
  // consumers: 8 warps; warp w sums nnz of item it for... simple: thread t<B*? accumulate per column over
  // the item's 32 rows, segmenting by output row (D nnz per row)
  int s = 0; uint32_t ph = 0;
  double acc = 0.0;
  for (int64_t it = 0; it < nitems; ++it) {
    mbar_wait(su32(&full[s]), ph);
    // warp w handles rows 4w..4w+3 of the item; lanes: (row q = lane / 8, column c = lane % 8 .. )
    const double* st = ring + (int64_t)s * stage_d;
    if (lane < 4 * 8) {
      const int q = lane >> 3, c0 = lane & 7;
      for (int c = c0; c < B; c += 8) acc += st[(warp * 4 + q) * ldp + c];
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
    if (++s == S) { s = 0; ph ^= 1; }
  }
  if (acc == 1.2345) out[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int n = 10000000, D = 20, B = 11;
  const int64_t nnz = 200000000, m = nnz / D;
  double *Y11, *Y12, *out;
  int* idx;
  CK(cudaMalloc(&Y11, sizeof(double) * (int64_t)n * 11));
  CK(cudaMalloc(&Y12, sizeof(double) * (int64_t)n * 12));
  CK(cudaMalloc(&idx, sizeof(int) * nnz));
  CK(cudaMalloc(&out, sizeof(double) * m * B));
  init_kernel<<<4096, 256>>>(Y11, (int64_t)n * 11, idx, nnz, n);
  init_kernel<<<4096, 256>>>(Y12, (int64_t)n * 12, idx, 0, n);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto report = [&](const char* name, float ms) {
    printf("  %-34s %7.3f ms  useful %6.0f GB/s  (%5.2f Gnnz/s)\n", name, ms, nnz * (double)B * 8 / ms / 1e6, nnz / ms / 1e6);
  };
#define REG(U, ld, Y, G) { reg_kernel<U><<<G, 256>>>(Y, ld, idx, m, D, B, out); cudaEventRecord(a); \
    for (int r = 0; r < 3; ++r) reg_kernel<U><<<G, 256>>>(Y, ld, idx, m, D, B, out); cudaEventRecord(b); CK(cudaEventSynchronize(b)); \
    float ms; cudaEventElapsedTime(&ms, a, b); char nm[64]; snprintf(nm, 64, "reg U=%d ld=%d grid=%d", U, ld, G); report(nm, ms / 3); }
  REG(4, 11, Y11, 148 * 8) REG(8, 11, Y11, 148 * 8) REG(10, 11, Y11, 148 * 8) REG(20, 11, Y11, 148 * 8) REG(20, 11, Y11, 148 * 4)
  REG(8, 12, Y12, 148 * 8) REG(20, 12, Y12, 148 * 8)
#define REG2(U, G) { reg2_kernel<U><<<G, 256>>>(Y12, 12, idx, m, D, B, out); cudaEventRecord(a); \
    for (int r = 0; r < 3; ++r) reg2_kernel<U><<<G, 256>>>(Y12, 12, idx, m, D, B, out); cudaEventRecord(b); CK(cudaEventSynchronize(b)); \
    float ms; cudaEventElapsedTime(&ms, a, b); char nm[64]; snprintf(nm, 64, "reg2 (double2) U=%d ld=12 grid=%d", U, G); report(nm, ms / 3); }
  REG2(4, 148 * 8) REG2(8, 148 * 8) REG2(20, 148 * 8)
  return 0;
  // TMA gather4
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  CUtensorMap tm;
  const int ldp = 12;
  cuuint64_t dims[2] = {(cuuint64_t)ldp, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)ldp * 8};
  cuuint32_t box[2] = {(cuuint32_t)ldp, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, Y12, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
#define TMA(S) { const int smem = S * 32 * ldp * 8; CK(cudaFuncSetAttribute(tma_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); \
    tma_kernel<S><<<148, 288, smem>>>(tm, idx, m, D, B, ldp, out); CK(cudaGetLastError()); CK(cudaDeviceSynchronize()); cudaEventRecord(a); \
    for (int rr = 0; rr < 3; ++rr) tma_kernel<S><<<148, 288, smem>>>(tm, idx, m, D, B, ldp, out); cudaEventRecord(b); CK(cudaEventSynchronize(b)); \
    float ms; cudaEventElapsedTime(&ms, a, b); char nm[64]; snprintf(nm, 64, "tma gather4 stages=%d (%d KB)", S, smem / 1024); report(nm, ms / 3); }
  TMA(16) TMA(32) TMA(64)
  return 0;
}

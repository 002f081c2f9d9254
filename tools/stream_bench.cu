// stream_bench.cu — HBM read bandwidth with many concurrent streams (Gram-kernel design probe).
// Sums NV vectors of LEN doubles (dot with a fixed vector is equivalent traffic) two ways:
//  (a) register loads: each thread reads 8 B from each stream per iteration (U elements)
//  (b) bulk TMA: each CTA copies CHUNK-byte pieces of every stream into a 3-stage smem ring
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_bench tools/stream_bench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int NV, int U>
__global__ void reg_kernel(const double* __restrict__ base, int64_t stride, int64_t len, double* out) {
  double acc = 0.0;
  const int64_t step = (int64_t)gridDim.x * blockDim.x * U;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x * U + threadIdx.x; e < len; e += step) {
    double v[NV][U];
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
      for (int u = 0; u < U; ++u) v[i][u] = (e + u * blockDim.x < len) ? __ldg(base + i * stride + e + u * blockDim.x) : 0.0;
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
      for (int u = 0; u < U; ++u) acc += v[i][u];
  }
  if (acc == 123.456) out[0] = acc;
}

__device__ inline uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void tma_kernel(const double* base, int64_t stride, int64_t len, int nv, int T, double* out) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bars[3];
  const int64_t ntiles = (len + T - 1) / T;
  const int64_t mine = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 3; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto issue = [&](int64_t k, int s) {
    const int64_t e0 = (blockIdx.x + k * gridDim.x) * (int64_t)T;
    const int cnt = (int)min((int64_t)T, len - e0);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bars[s])), "r"(cnt * 8 * nv));
    for (int i = 0; i < nv; ++i)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(sm + ((int64_t)s * nv + i) * T)), "l"(base + i * stride + e0), "r"(cnt * 8), "r"(su32(&bars[s])) : "memory");
  };
  if (threadIdx.x == 0) for (int s = 0; s < 3 && s < mine; ++s) issue(s, s);
  double acc = 0.0;
  for (int64_t k = 0; k < mine; ++k) {
    const int s = k % 3;
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(su32(&bars[s])), "r"((uint32_t)((k / 3) & 1)) : "memory");
    const int64_t e0 = (blockIdx.x + k * gridDim.x) * (int64_t)T;
    const int cnt = (int)min((int64_t)T, len - e0);
    const double* st = sm + (int64_t)s * nv * T;
    for (int idx = threadIdx.x; idx < cnt; idx += blockDim.x)
      for (int i = 0; i < nv; ++i) acc += st[i * T + idx];
    __syncthreads();
    if (threadIdx.x == 0 && k + 3 < mine) { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); issue(k + 3, s); }
  }
  if (acc == 123.456) out[0] = acc;
}


// (c) per-stream ring: items (tile k, stream i) flow through S stages of CH bytes; one producer
// warp issues bulk copies as stages free up (full/empty mbarriers, no block-wide barrier).
__global__ void ring_kernel(const double* base, int64_t stride, int64_t len, int nv, int T, int S, double* out) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t full[32], empty[32];
  const int nwc = blockDim.x / 32 - 1;  // consumer warps
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = (len + T - 1) / T;
  const int64_t mine = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t items = mine * nv;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(nwc));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (warp == nwc) {  // producer
    if (lane == 0) {
      int s = 0, i = 0;
      uint32_t ph = 0;
      int64_t e0 = (int64_t)blockIdx.x * T;
      for (int64_t it = 0; it < items; ++it) {
        if (it >= S)
          asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(su32(&empty[s])), "r"(ph ^ 1) : "memory");
        const int cnt = (int)min((int64_t)T, len - e0);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(cnt * 8));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su32(sm + (int64_t)s * T)), "l"(base + i * stride + e0), "r"(cnt * 8), "r"(su32(&full[s])) : "memory");
        if (++s == S) { s = 0; ph ^= 1; }
        if (++i == nv) { i = 0; e0 += (int64_t)gridDim.x * T; }
      }
    }
    return;
  }
  double acc = 0.0;
  int s = 0, i = 0;
  uint32_t ph = 0;
  int64_t e0 = (int64_t)blockIdx.x * T;
  for (int64_t it = 0; it < items; ++it) {
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(su32(&full[s])), "r"(ph) : "memory");
    const int cnt = (int)min((int64_t)T, len - e0);
    const double* st = sm + (int64_t)s * T;
    for (int idx = threadIdx.x; idx < cnt; idx += nwc * 32) acc += st[idx];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
    if (++s == S) { s = 0; ph ^= 1; }
    if (++i == nv) { i = 0; e0 += (int64_t)gridDim.x * T; }
  }
  if (acc == 123.456) out[0] = acc;
}

template <int NV, int U>
float run_reg(const double* base, int64_t stride, int64_t len, double* out, int grid, int bs) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  reg_kernel<NV, U><<<grid, bs>>>(base, stride, len, out);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) reg_kernel<NV, U><<<grid, bs>>>(base, stride, len, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / 5;
}

int main(int argc, char** argv) {
  // default: 64 Mi doubles = 512 MiB per stream; argv[1] = doubles per stream (e.g. 220000000)
  const int64_t len = argc > 1 ? atoll(argv[1]) : (1 << 26);
  const int maxnv = 32;
  double* base; double* out;
  CK(cudaMalloc(&base, sizeof(double) * len * maxnv));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemset(base, 0, sizeof(double) * len * maxnv));
  printf("register path (GB/s):\n");
#define R(NV, U, G, BS) { float ms = run_reg<NV, U>(base, len, len, out, G, BS); printf("  nv=%2d U=%d grid=%5d bs=%d : %7.0f\n", NV, U, G, BS, NV * len * 8.0 / ms / 1e6); }
  R(1, 4, 148 * 8, 256) R(2, 4, 148 * 8, 256) R(8, 4, 148 * 4, 256) R(8, 2, 148 * 8, 256) R(16, 2, 148 * 4, 256) R(16, 1, 148 * 8, 256) R(32, 1, 148 * 4, 256) R(32, 2, 148 * 2, 256)
  if (argc > 2 && argv[2][0] == 0x72) return 0;  // "r": register path only
  printf("TMA ring path (GB/s):\n");
  CK(cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  for (int nv : {8, 32}) for (int ch : {2048, 4096, 8192, 16384}) for (int kb : {64, 128, 200}) for (int bs : {160, 288, 544}) {
    const int T = ch / 8, S = kb * 1024 / ch;
    if (S < 2 || S > 32) continue;
    const size_t smem = (size_t)S * ch;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    ring_kernel<<<148, bs, smem>>>(base, len, len, nv, T, S, out);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) ring_kernel<<<148, bs, smem>>>(base, len, len, nv, T, S, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
    CK(cudaGetLastError());
    printf("  nv=%2d chunk=%6d B stages=%2d bs=%d : %7.0f\n", nv, ch, S, bs, nv * len * 8.0 / ms / 1e6);
  }
  if (argc > 3) return 0;
  printf("TMA bulk path (GB/s):\n");
  CK(cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  int nvs[] = {1, 2, 8, 16, 32};
  int chunks[] = {1024, 2048, 4096, 8192, 16384, 32768};
  for (int nv : nvs) {
    for (int ch : chunks) {
      const int T = ch / 8;
      const size_t smem = (size_t)3 * nv * ch;
      if (smem > 200 * 1024) continue;
      for (int ctas : {148, 296}) {
        if (ctas == 296 && smem > 100 * 1024) continue;
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        tma_kernel<<<ctas, 128, smem>>>(base, len, len, nv, T, out);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) tma_kernel<<<ctas, 128, smem>>>(base, len, len, nv, T, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
        CK(cudaGetLastError());
        printf("  nv=%2d chunk=%6d B ctas=%d : %7.0f\n", nv, ch, ctas, nv * len * 8.0 / ms / 1e6);
      }
    }
  }
  return 0;
}

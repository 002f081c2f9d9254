// gather_ceiling.cu — how fast can one B200 serve random row gathers from L2 / HBM / shared memory?
// (the SpMM's bound.)  out[i] = Σ_k Y[idx[i*D + k]] over uniform random idx in [0, N),
// for table sizes N·rowbytes from L2-resident to far beyond L2, rows of 8 B (b = 1) and 88/96 B (B = 11).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_ceiling tools/gather_ceiling.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void init_idx(int* idx, int64_t nidx, int64_t N, uint64_t salt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nidx; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h = (i + salt) * 0x9E3779B97F4A7C15ull;
    h ^= h >> 31; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 29;
    idx[i] = (int)(h % (uint64_t)N);
  }
}
__global__ void init_y(double* Y, int64_t ny) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ny; i += (int64_t)gridDim.x * blockDim.x) Y[i] = (double)(i % 7);
}

// b = 1, thread per output (D gathers), U in flight — the spmv_small_row1 pattern
template <int U>
__global__ void __launch_bounds__(256) g1_thread(const double* Y, const int* idx, int64_t m, int D, double* out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int* ix = idx + i * D;
  double acc = 0.0;
  for (int k = 0; k < D; k += U) {
    int cl[U];
#pragma unroll
    for (int u = 0; u < U; ++u) cl[u] = __ldg(ix + k + u);
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(Y + cl[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  out[i] = acc;
}

// b = 1, warp-strided: lanes take consecutive idx (coalesced index loads), U rounds in flight
template <int U>
__global__ void __launch_bounds__(256) g1_warp(const double* Y, const int* idx, int64_t nnz, double* out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, T = (int64_t)gridDim.x * blockDim.x;
  double acc = 0.0;
  for (int64_t z = t; z < nnz; z += T * U) {
    int cl[U];
#pragma unroll
    for (int u = 0; u < U; ++u) cl[u] = z + u * T < nnz ? __ldg(idx + z + u * T) : 0;
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(Y + cl[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  if (acc == 1.2345) out[0] = acc;
}

// index i ~ P(row) ∝ degree (the C4 gather distribution after degree relabelling): a uniform random
// nonzero z, mapped to its row by binary search in the degree-sorted row pointer rp (n + 1 entries)
__global__ void init_idx_skew(int* idx, int64_t nidx, const int* rp, int n, uint64_t salt) {
  const int nnz = rp[n];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nidx; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h = (i + salt) * 0x9E3779B97F4A7C15ull;
    h ^= h >> 31; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 29;
    const int z = (int)(h % (uint64_t)nnz);
    int lo = 0, hi = n;  // rp[lo] <= z < rp[hi]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (rp[mid] <= z) lo = mid; else hi = mid;
    }
    idx[i] = lo;
  }
}

// b = 1, warp-strided with the first NS entries of the table staged in shared memory
template <int U>
__global__ void __launch_bounds__(1024, 1) g1_hot(const double* Y, int NS, const int* idx, int64_t nnz, double* out) {
  extern __shared__ double tab[];
  for (int i = threadIdx.x; i < NS; i += blockDim.x) tab[i] = Y[i];
  __syncthreads();
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, T = (int64_t)gridDim.x * blockDim.x;
  double acc = 0.0;
  for (int64_t z = t; z < nnz; z += T * U) {
    int cl[U];
#pragma unroll
    for (int u = 0; u < U; ++u) cl[u] = z + u * T < nnz ? __ldg(idx + z + u * T) : 0;
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = cl[u] < NS ? tab[cl[u]] : __ldg(Y + cl[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  if (acc == 1.2345) out[0] = acc;
}

// b = 1 from shared memory: the table (first NS doubles of Y) staged per CTA, same warp-strided walk
template <int U>
__global__ void __launch_bounds__(1024, 1) g1_smem(const double* Y, int NS, const int* idx, int64_t nnz, double* out) {
  extern __shared__ double tab[];
  for (int i = threadIdx.x; i < NS; i += blockDim.x) tab[i] = Y[i];
  __syncthreads();
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, T = (int64_t)gridDim.x * blockDim.x;
  double acc = 0.0;
  for (int64_t z = t; z < nnz; z += T * U) {
    int cl[U];
#pragma unroll
    for (int u = 0; u < U; ++u) cl[u] = z + u * T < nnz ? __ldg(idx + z + u * T) : 0;
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = tab[cl[u] % NS];
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  if (acc == 1.2345) out[0] = acc;
}

// B columns: lane group of B lanes per gathered row (gpw = 32 / B rows per LDG), U in flight
template <int U>
__global__ void __launch_bounds__(256) gB_group(const double* Y, int ld, int B, const int* idx, int64_t nnz, double* out) {
  const int lane = threadIdx.x & 31, gpw = 32 / B, gi = lane / B, c = lane - gi * B;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, W = ((int64_t)gridDim.x * blockDim.x) >> 5;
  if (gi >= gpw) return;
  double acc = 0.0;
  for (int64_t z = w * gpw + gi; z < nnz; z += W * gpw * U) {
    int cl[U];
#pragma unroll
    for (int u = 0; u < U; ++u) cl[u] = z + u * W * gpw < nnz ? __ldg(idx + z + u * W * gpw) : 0;
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(Y + (int64_t)cl[u] * ld + c);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  if (acc == 1.2345) out[0] = acc;
}

// B columns flattened over the warp: element e = 11 z + c; lane l takes e = base + l (all 32 lanes busy)
template <int U, int B>
__global__ void __launch_bounds__(256) gB_flat(const double* Y, const int* idx, int64_t nnz, double* out) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, W = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t ne = nnz * B;
  double acc = 0.0;
  for (int64_t e0 = w * 32 * U; e0 < ne; e0 += W * 32 * U) {
    int cl[U], cc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + u * 32 + lane;
      const int64_t z = e / B;
      cc[u] = (int)(e - z * B);
      cl[u] = e < ne ? __ldg(idx + z) : 0;
    }
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(Y + (int64_t)cl[u] * B + cc[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  if (acc == 1.2345) out[0] = acc;
}

// 16-byte lanes: rows padded to ld = 12 (96 B = 6 x 16 B), 6 lanes per row, 5 rows per LDG
template <int U>
__global__ void __launch_bounds__(256) gB_v2(const double* Y, const int* idx, int64_t nnz, double* out) {
  const int lane = threadIdx.x & 31, gi = lane / 6, c = lane - gi * 6;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, W = ((int64_t)gridDim.x * blockDim.x) >> 5;
  if (gi >= 5) return;
  double acc = 0.0;
  for (int64_t z = w * 5 + gi; z < nnz; z += W * 5 * U) {
    int cl[U];
#pragma unroll
    for (int u = 0; u < U; ++u) cl[u] = z + u * W * 5 < nnz ? __ldg(idx + z + u * W * 5) : 0;
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(reinterpret_cast<const double2*>(Y + (int64_t)cl[u] * 12) + c);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y;
  }
  if (acc == 1.2345) out[0] = acc;
}

// 32-byte lanes (sm_100 256-bit loads): ld = 12 rows are 3 x 32 B, 3 lanes per row, 10 rows per LDG
template <int U>
__global__ void __launch_bounds__(256) gB_v4(const double* Y, const int* idx, int64_t nnz, double* out) {
  const int lane = threadIdx.x & 31, gi = lane / 3, c = lane - gi * 3;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, W = ((int64_t)gridDim.x * blockDim.x) >> 5;
  if (gi >= 10) return;
  double acc = 0.0;
  for (int64_t z = w * 10 + gi; z < nnz; z += W * 10 * U) {
    int cl[U];
#pragma unroll
    for (int u = 0; u < U; ++u) cl[u] = z + u * W * 10 < nnz ? __ldg(idx + z + u * W * 10) : 0;
    double v[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u)
      asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[u][0]), "=d"(v[u][1]), "=d"(v[u][2]), "=d"(v[u][3])
                   : "l"(Y + (int64_t)cl[u] * 12 + 4 * c));
#pragma unroll
    for (int u = 0; u < U; ++u) acc += (v[u][0] + v[u][1]) + (v[u][2] + v[u][3]);
  }
  if (acc == 1.2345) out[0] = acc;
}

// 32-byte lanes over rows at stride LD doubles (LD = 16: the power-of-two stride of the round-2 layout)
template <int U, int LD>
__global__ void __launch_bounds__(256) gB_v4ld(const double* Y, const int* idx, int64_t nnz, double* out) {
  const int lane = threadIdx.x & 31, gi = lane / 3, c = lane - gi * 3;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, W = ((int64_t)gridDim.x * blockDim.x) >> 5;
  if (gi >= 10) return;
  double acc = 0.0;
  for (int64_t z = w * 10 + gi; z < nnz; z += W * 10 * U) {
    int cl[U];
#pragma unroll
    for (int u = 0; u < U; ++u) cl[u] = z + u * W * 10 < nnz ? __ldg(idx + z + u * W * 10) : 0;
    double v[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u)
      asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[u][0]), "=d"(v[u][1]), "=d"(v[u][2]), "=d"(v[u][3])
                   : "l"(Y + (int64_t)cl[u] * LD + 4 * c));
#pragma unroll
    for (int u = 0; u < U; ++u) acc += (v[u][0] + v[u][1]) + (v[u][2] + v[u][3]);
  }
  if (acc == 1.2345) out[0] = acc;
}

// fp32 storage: 11 floats per row at a 16-float (64-byte) stride, 2 lanes of 8 floats per row, 16 rows per LDG
template <int U>
__global__ void __launch_bounds__(256) gF_v8(const float* Y, const int* idx, int64_t nnz, double* out) {
  const int lane = threadIdx.x & 31, gi = lane / 2, c = lane - gi * 2;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, W = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float acc = 0.0f;
  for (int64_t z = w * 16 + gi; z < nnz; z += W * 16 * U) {
    int cl[U];
#pragma unroll
    for (int u = 0; u < U; ++u) cl[u] = z + u * W * 16 < nnz ? __ldg(idx + z + u * W * 16) : 0;
    float v[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u)
      asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=f"(v[u][0]), "=f"(v[u][1]), "=f"(v[u][2]), "=f"(v[u][3]), "=f"(v[u][4]), "=f"(v[u][5]),
                     "=f"(v[u][6]), "=f"(v[u][7])
                   : "l"(Y + (int64_t)cl[u] * 16 + 8 * c));
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < 8; ++k) acc += v[u][k];
  }
  if (acc == 1.2345f) out[0] = acc;
}

// L2 -> SM streaming bandwidth: every CTA re-reads an L2-resident buffer with coalesced 32-byte lanes
__global__ void __launch_bounds__(256) l2_stream(const double* Y, int64_t n, int reps, double* out) {
  double acc = 0.0;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, T = (int64_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (int64_t i = t; i < n / 4; i += T) {
      double v0, v1, v2, v3;
      asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v0), "=d"(v1), "=d"(v2), "=d"(v3) : "l"(Y + 4 * ((i + r * 7919) % (n / 4))));
      acc += (v0 + v1) + (v2 + v3);
    }
  if (acc == 1.2345) out[0] = acc;
}

int main() {
  const int64_t nnz = 400000000;
  const int64_t nmax = 10000000;
  double *Y, *out;
  int* idx;
  CK(cudaMalloc(&Y, sizeof(double) * nmax * 16));
  CK(cudaMalloc(&idx, sizeof(int) * nnz));
  CK(cudaMalloc(&out, sizeof(double) * nnz / 16 + 64));
  init_y<<<4096, 256>>>(Y, nmax * 16);
  CK(cudaDeviceSynchronize());
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto&& launch) {
    launch();
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 3;
  };
  for (int64_t mb : {16, 48, 96}) {
    const int64_t n = mb * 1000000 / 8;
    const int reps = 40;
    float t = timeit([&] { l2_stream<<<sms * 8, 256>>>(Y, n, reps, out); });
    printf("L2-resident stream of %lld MB x %d: %.3f ms, %.0f GB/s\n", (long long)mb, reps, t, n * 8.0 * reps / t / 1e6);
  }
  {
    init_idx<<<4096, 256>>>(idx, nnz, 240000, 5);  // 23 MB of 96-byte rows: L2 resident, uniform
    CK(cudaDeviceSynchronize());
    float t = timeit([&] { gB_v4<4><<<sms * 8, 256>>>(Y, idx, nnz, out); });
    printf("uniform random 96-byte rows from 23 MB (L2): v4 lanes %.3f ms, %.0f Grows/s = %.0f GB/s of rows\n", t, nnz / t / 1e6, nnz * 96.0 / t / 1e6);
  }
  const int64_t Ns[] = {4096, 26624, 262144, 1000000, 10000000};
  printf("b=1: %lld random 8-byte gathers, table of N doubles\n", (long long)nnz);
  for (int64_t N : Ns) {
    init_idx<<<4096, 256>>>(idx, nnz, N, 1);
    CK(cudaDeviceSynchronize());
    const int D = 16;
    float t1 = timeit([&] { g1_thread<4><<<(nnz / D + 255) / 256, 256>>>(Y, idx, nnz / D, D, out); });
    float t2 = timeit([&] { g1_thread<8><<<(nnz / D + 255) / 256, 256>>>(Y, idx, nnz / D, D, out); });
    float t3 = timeit([&] { g1_warp<8><<<sms * 8, 256>>>(Y, idx, nnz, out); });
    printf("  N=%9lld (%7.1f MB): thread U4 %.3f ms (%.0f G/s)  thread U8 %.3f ms (%.0f G/s)  warp-strided U8 %.3f ms (%.0f G/s)\n",
           (long long)N, N * 8 / 1e6, t1, nnz / t1 / 1e6, t2, nnz / t2 / 1e6, t3, nnz / t3 / 1e6);
  }
  {
    const int NS = 26624;
    CK(cudaFuncSetAttribute(g1_smem<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, NS * 8));
    init_idx<<<4096, 256>>>(idx, nnz, NS, 1);
    CK(cudaDeviceSynchronize());
    float t = timeit([&] { g1_smem<8><<<sms, 1024, NS * 8>>>(Y, NS, idx, nnz, out); });
    printf("  smem table of %d doubles (1 CTA x 1024 / SM): %.3f ms (%.0f G/s)\n", NS, t, nnz / t / 1e6);
  }
  printf("B=11: %lld random row gathers (rows of 88 B, ld 11 / 96 B, ld 12)\n", (long long)nnz);
  for (int64_t N : {262144LL, 1000000LL, 10000000LL}) {
    init_idx<<<4096, 256>>>(idx, nnz, N, 2);
    CK(cudaDeviceSynchronize());
    float t1 = timeit([&] { gB_group<8><<<sms * 8, 256>>>(Y, 11, 11, idx, nnz, out); });
    float t2 = timeit([&] { gB_group<8><<<sms * 8, 256>>>(Y, 12, 11, idx, nnz, out); });
    float t3 = timeit([&] { gB_flat<8, 11><<<sms * 8, 256>>>(Y, idx, nnz, out); });
    float t4 = timeit([&] { gB_v2<8><<<sms * 8, 256>>>(Y, idx, nnz, out); });
    printf("  N=%9lld (%7.1f MB @88B): group ld11 %.3f ms (%.0f Grows/s)  group ld12 %.3f  flat ld11 %.3f  double2 ld12 %.3f ms (%.0f Grows/s)\n",
           (long long)N, N * 88 / 1e6, t1, nnz / t1 / 1e6, t2, t3, t4, nnz / t4 / 1e6);
  }
  // the C4 distribution (tools/c4_degree_histogram.txt)
  {
    FILE* fh = fopen("tools/c4_degree_histogram.txt", "r");
    if (!fh) { printf("no histogram\n"); return 0; }
    char line[256];
    int* rp = (int*)malloc(sizeof(int) * (nmax + 1));
    int64_t r = 0;
    rp[0] = 0;
    while (fgets(line, sizeof line, fh)) {
      if (line[0] == '#') continue;
      long long d, c;
      if (sscanf(line, "%lld %lld", &d, &c) != 2) continue;
      for (long long k = 0; k < c && r < nmax; ++k, ++r) rp[r + 1] = rp[r] + (int)d;
    }
    fclose(fh);
    int* drp;
    CK(cudaMalloc(&drp, sizeof(int) * (nmax + 1)));
    CK(cudaMemcpy(drp, rp, sizeof(int) * (nmax + 1), cudaMemcpyHostToDevice));
    init_idx_skew<<<4096, 256>>>(idx, nnz, drp, (int)nmax, 3);
    CK(cudaDeviceSynchronize());
    printf("C4-distributed indices (P(row) ~ degree, degree-sorted ids; n = %lld, nnz in rp = %d)\n", (long long)r, rp[r]);
    float t3 = timeit([&] { g1_warp<8><<<sms * 8, 256>>>(Y, idx, nnz, out); });
    printf("  b=1 warp-strided U8: %.3f ms (%.0f G/s)\n", t3, nnz / t3 / 1e6);
    for (int NS : {8192, 16384, 26624}) {
      CK(cudaFuncSetAttribute(g1_hot<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, NS * 8));
      float t4 = timeit([&] { g1_hot<8><<<sms, 1024, NS * 8>>>(Y, NS, idx, nnz, out); });
      printf("  b=1 warp-strided + smem hot %d: %.3f ms (%.0f G/s)\n", NS, t4, nnz / t4 / 1e6);
    }
    float a1 = timeit([&] { gB_group<8><<<sms * 8, 256>>>(Y, 11, 11, idx, nnz, out); });
    float a2 = timeit([&] { gB_group<8><<<sms * 8, 256>>>(Y, 12, 11, idx, nnz, out); });
    float a4 = timeit([&] { gB_v2<8><<<sms * 8, 256>>>(Y, idx, nnz, out); });
    float a5 = timeit([&] { gB_v2<4><<<sms * 8, 256>>>(Y, idx, nnz, out); });
    float a6 = timeit([&] { gB_v4<4><<<sms * 8, 256>>>(Y, idx, nnz, out); });
    float a7 = timeit([&] { gB_v4<8><<<sms * 8, 256>>>(Y, idx, nnz, out); });
    printf("  B=11 group ld11 %.3f ms (%.0f Grows/s)  group ld12 %.3f  double2 ld12 U8 %.3f ms (%.0f Grows/s)  U4 %.3f  v4(32B) ld12 U4 %.3f U8 %.3f\n",
           a1, nnz / a1 / 1e6, a2, a4, nnz / a4 / 1e6, a5, a6, a7);
    float b1 = timeit([&] { gB_v4ld<4, 16><<<sms * 8, 256>>>(Y, idx, nnz, out); });
    float b2 = timeit([&] { gF_v8<4><<<sms * 8, 256>>>(reinterpret_cast<const float*>(Y), idx, nnz, out); });
    float b3 = timeit([&] { gF_v8<8><<<sms * 8, 256>>>(reinterpret_cast<const float*>(Y), idx, nnz, out); });
    printf("  B=11 v4(32B) ld16 U4 %.3f ms;  fp32 rows (11 floats, ld 16, 2 x 32B lanes) U4 %.3f ms  U8 %.3f ms\n", b1, b2, b3);
  }
  return 0;
}

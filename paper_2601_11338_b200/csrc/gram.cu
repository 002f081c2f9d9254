// gram.cu — deterministic reduction of per-CTA partial sums (the Gram passes' second stage).
//
// Every dot-product pass (dcgs2.cu) writes one partial sum per (output, CTA); this kernel sums them
// in a fixed order, so results are bitwise reproducible for a given grid.  (The register-streaming
// CGS2 kernels that used to live here were replaced by the bulk-copy ring passes: DESIGN.md §8.)
#include "wl_internal.cuh"

namespace wl {
namespace {

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

}  // namespace

int gram_grid(int64_t elems, int B) {
  (void)elems;
  (void)B;
  return num_sms() * 6;  // upper bound on the CTAs of a dot pass: partial buffers are sized for it
}

void reduce_partials(const double* partials, int nout, int G, double* sums_out, cudaStream_t s) {
  reduce_partials_kernel<<<(nout + 7) / 8, 256, 0, s>>>(partials, nout, G, sums_out);
  WL_CUDA(cudaGetLastError());
}

}  // namespace wl

// scatter.cu -- a1: the PNG scatter of PAPER.md Alg. 4.
//
//   for p in P:  for p' in P:  for u in N_i^p(p'):  insert SPR[u] into update_bins[p']
//
// One CTA per work item (source partition p, destination groups [j0, j1)).
// The CTA first stages the partition's source values x[p q .. p q + q) in
// shared memory (coalesced 128-bit loads; 128 KB at q = 2^15, the "cache the
// vertex data of p" of P:137), then each warp streams whole (p, j) groups:
// coalesced reads of png_src, random reads of the staged slice, and
// contiguous writes to the group's disjoint range upd[upd_off[p][j] ...]
// (fixed, disjoint write locations -- no atomics).  A pure copy: the
// update bins are bit-identical to the oracle's scatter for the same x.
#include "pcpm_internal.cuh"

namespace pcpm {
namespace {

__global__ void __launch_bounds__(kScatterThreads, 1)
k_scatter(const ScatterItem* __restrict__ items, int n_items, const float* __restrict__ x, int64_t n_src, int b,
          int64_t k_dst, const uint32_t* __restrict__ png_src, const uint32_t* __restrict__ png_off,
          const uint32_t* __restrict__ upd_off, float* __restrict__ upd) {
  extern __shared__ float4 smem_f4[];
  __shared__ uint32_t next_group;
  constexpr int kUnroll = 4;
  float* xs = reinterpret_cast<float*>(smem_f4);
  const int lane = threadIdx.x & 31;
  const int64_t q = int64_t(1) << b;
  for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
    const ScatterItem item = items[it];
    const int64_t base = (int64_t)item.p << b;
    const int64_t len = min(q, n_src - base);
    // stage x[base, base + len) -- 16 B vectors when aligned
    const float* src = x + base;
    if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
      const int64_t n4 = len >> 2;
      const float4* s4 = reinterpret_cast<const float4*>(src);
      for (int64_t i = threadIdx.x; i < n4; i += blockDim.x) smem_f4[i] = __ldg(s4 + i);
      for (int64_t i = (n4 << 2) + threadIdx.x; i < len; i += blockDim.x) xs[i] = __ldg(src + i);
    } else {
      for (int64_t i = threadIdx.x; i < len; i += blockDim.x) xs[i] = __ldg(src + i);
    }
    if (threadIdx.x == 0) next_group = 0;
    __syncthreads();
    const uint32_t* off = png_off + (int64_t)item.p * (k_dst + 1);
    const uint32_t* uo = upd_off + (int64_t)item.p * k_dst;
    const uint32_t ubase = (uint32_t)base;
    for (;;) {
      // groups (p, j) are claimed dynamically: their sizes vary by orders of magnitude
      uint32_t g = 0;
      if (lane == 0) g = atomicAdd(&next_group, 1u);
      const uint32_t j = item.j0 + __shfl_sync(0xffffffffu, g, 0);
      if (j >= item.j1) break;
      const uint32_t s = __ldg(off + j), len = __ldg(off + j + 1) - s;
      const uint32_t dst = __ldg(uo + j);
      for (uint32_t t = lane; t < len; t += 32 * kUnroll) {
        uint32_t src[kUnroll];
#pragma unroll
        for (int k = 0; k < kUnroll; ++k) src[k] = (t + 32 * k < len) ? __ldg(png_src + s + t + 32 * k) : ubase;
#pragma unroll
        for (int k = 0; k < kUnroll; ++k)
          if (t + 32 * k < len) upd[dst + t + 32 * k] = xs[src[k] - ubase];
      }
    }
    __syncthreads();
  }
}

}  // namespace

int prepare_scatter(pcpm_handle* h) {
  PCPM_CK(cudaFuncSetAttribute(k_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 << kMaxBits));
  return PCPM_OK;
}

int launch_scatter(pcpm_handle* h, const float* x, cudaStream_t s) {
  if (h->n_sitems == 0) return PCPM_OK;
  const int smem = (int)(h->q * sizeof(float));
  int grid = std::min(h->n_sitems, h->num_sms);
  k_scatter<<<grid, kScatterThreads, smem, s>>>(h->sitems, h->n_sitems, x, h->n_src, h->b, h->k_dst, h->png_src,
                                                 h->png_off, h->upd_off, h->upd);
  PCPM_CK(cudaGetLastError());
  h->launches += 1;
  return PCPM_OK;
}

}  // namespace pcpm

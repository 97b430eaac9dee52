// scatter.cu -- a1: the PNG scatter of PAPER.md Alg. 4.
//
//   for p in P:  for p' in P:  for u in N_i^p(p'):  insert SPR[u] into update_bins[p']
//
// One CTA per work item (source partition p, destination groups [j0, j1)).
// The CTA stages the partition's source values x[p q .. p q + q) in shared
// memory (coalesced 128-bit loads; 128 KB at q = 2^15 -- the "cache the vertex
// data of p" of P:137) together with the item's rows of png_off / upd_off.
// Warps then claim whole (p, j) groups dynamically and stream them: coalesced
// reads of the PNG sources (2-byte partition-local in the compact layout),
// random reads of the staged slice, and coalesced writes to the group's
// disjoint range upd[upd_off[p][j] ...] (fixed, disjoint write
// locations -- no atomics).  Eight independent loads per lane are kept in
// flight.  A pure copy: the update bins are bit-identical to the oracle's
// scatter for the same x.
#include "pcpm_internal.cuh"

namespace pcpm {
namespace {

constexpr int kUnroll = 8;

template <typename SrcT>
__global__ void __launch_bounds__(kScatterThreads, 1)
k_scatter(const ScatterItem* __restrict__ items, int n_items, const float* __restrict__ x, int64_t n_src, int b,
          int64_t k_dst, const SrcT* __restrict__ png, const uint32_t* __restrict__ png_off,
          const uint32_t* __restrict__ upd_off, float* __restrict__ upd) {
  extern __shared__ float4 smem_f4[];
  __shared__ uint32_t next_group;
  const int64_t q = int64_t(1) << b;
  float* xs = reinterpret_cast<float*>(smem_f4);
  uint32_t* off_s = reinterpret_cast<uint32_t*>(xs + ((q + 3) & ~int64_t(3)));   // [kScatterMaxGroups + 1]
  uint32_t* uo_s = off_s + kScatterMaxGroups + 4;                                  // [kScatterMaxGroups]
  const int lane = threadIdx.x & 31;
  for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
    const ScatterItem item = items[it];
    const int64_t base = (int64_t)item.p << b;
    const int64_t len = min(q, n_src - base);
    const uint32_t ng = item.j1 - item.j0;
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
    const uint32_t* off = png_off + (int64_t)item.p * (k_dst + 1) + item.j0;
    const uint32_t* uo = upd_off + (int64_t)item.p * k_dst + item.j0;
    for (uint32_t g = threadIdx.x; g <= ng; g += blockDim.x) off_s[g] = __ldg(off + g);
    for (uint32_t g = threadIdx.x; g < ng; g += blockDim.x) uo_s[g] = __ldg(uo + g);
    if (threadIdx.x == 0) next_group = 0;
    __syncthreads();
    const uint32_t ubase = sizeof(SrcT) == 2 ? 0u : (uint32_t)base;   // compact sources are local
    for (;;) {
      // groups (p, j) are claimed dynamically: their sizes vary by orders of magnitude
      uint32_t g = 0;
      if (lane == 0) g = atomicAdd(&next_group, 1u);
      g = __shfl_sync(0xffffffffu, g, 0);
      if (g >= ng) break;
      const uint32_t s = off_s[g], glen = off_s[g + 1] - s;
      float* dst = upd + uo_s[g];
      const SrcT* ps = png + s;
      for (uint32_t t = lane; t < glen; t += 32 * kUnroll) {
        uint32_t sv[kUnroll];
#pragma unroll
        for (int k = 0; k < kUnroll; ++k) sv[k] = (t + 32 * k < glen) ? (uint32_t)__ldg(ps + t + 32 * k) : ubase;
#pragma unroll
        for (int k = 0; k < kUnroll; ++k)
          if (t + 32 * k < glen) dst[t + 32 * k] = xs[sv[k] - ubase];
      }
    }
    __syncthreads();
  }
}

int scatter_smem_bytes(int b) {
  const int64_t q = int64_t(1) << b;
  return (int)(((q + 3) & ~int64_t(3)) * 4 + (2 * kScatterMaxGroups + 8) * 4);
}

}  // namespace

int prepare_scatter(pcpm_handle* h) {
  PCPM_CK(cudaFuncSetAttribute(k_scatter<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               scatter_smem_bytes(kMaxBits)));
  PCPM_CK(cudaFuncSetAttribute(k_scatter<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               scatter_smem_bytes(kMaxBits)));
  return PCPM_OK;
}

int launch_scatter(pcpm_handle* h, const float* x, cudaStream_t s) {
  if (h->n_sitems == 0) return PCPM_OK;
  const int smem = scatter_smem_bytes(h->b);
  const int grid = std::min(h->n_sitems, h->num_sms);
  if (h->wide)
    k_scatter<uint32_t><<<grid, kScatterThreads, smem, s>>>(h->sitems, h->n_sitems, x, h->n_src, h->b, h->k_dst,
                                                            h->png_src, h->png_off, h->upd_off, h->upd);
  else
    k_scatter<uint16_t><<<grid, kScatterThreads, smem, s>>>(h->sitems, h->n_sitems, x, h->n_src, h->b, h->k_dst,
                                                            h->png16, h->png_off, h->upd_off, h->upd);
  PCPM_CK(cudaGetLastError());
  h->launches += 1;
  return PCPM_OK;
}

}  // namespace pcpm

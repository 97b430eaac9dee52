// Microbenchmark: shared-memory accumulator throughput on sm_100a -- the design
// evidence behind the gather's accumulator (DESIGN.md §5 "Why fixed point" and §6).
//
// Every CTA (one per SM, 1024 threads) owns a 128 KB shared array -- one destination
// partition of q = 2^15 u32 words (or 2^14 u64 words) -- and performs random-address
// accumulations into it, like Alg. 5's `PR[id] += update` in the PCPM
// gather.  Each thread keeps 8 independent accumulations in flight per loop trip
// (cheap LCG addresses), so the shared-memory pipe, not the issue rate, is the limit.
//
// Variants (op = one accumulation by one thread):
//   atom.u32     atom.shared.add.u32, return value consumed (the gather's fixed-point
//                low word + carry test)
//   red.u32      red.shared.add.u32 (no return)
//   atom.u64     atom.shared.add.u64 into 2^14 u64 words (128 KB)
//   red.u64      red.shared.add.u64
//   atom.f32     atomicAdd(float*) on shared memory
//   red.f32      red.shared.add.f32
//   lds+sts      racy plain load + store (no atomicity): the non-atomic floor
//   atom.u32.cf  atom.u32 with bank-conflict-free addresses (lane l -> bank l): the
//                one-wavefront-per-instruction ceiling
//   dsmem.red    red.shared::cluster.add.u32 into the PEER CTA of a 2-CTA cluster
//                (distributed shared memory, the q = 2^16 split accumulator)
//   dsmem.atom   atom.shared::cluster.add.u32 into the peer CTA (return consumed)
// Address distributions: uniform over the array; "skew": 1/8 of the ops go to 64 hot
// words (RMAT hubs).
//
// Output: one JSON line per (variant, distribution): Gop/s over the GPU, ops per SM
// clock, and the implied shared-memory wavefronts per warp instruction
// (32 / ops-per-clock, assuming one wavefront per SM clock).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atoms_bench atoms_bench.cu
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

constexpr int kWords32 = 1 << 15;
constexpr int kUnroll = 8;

enum Mode { ATOM32, RED32, ATOM64, RED64, ATOMF, REDF, PLAIN, ATOM32_CF, DSMEM_RED, DSMEM_ATOM, NMODES };
static const char* kNames[NMODES] = {"atom.u32", "red.u32", "atom.u64", "red.u64", "atom.f32",
                                     "red.f32", "lds+sts", "atom.u32.cf", "dsmem.red", "dsmem.atom"};

__device__ __forceinline__ uint32_t lcg(uint32_t x) { return x * 1664525u + 1013904223u; }

template <int MODE>
__global__ void __launch_bounds__(1024, 1) k_acc(int iters, int skew, uint32_t* out) {
  extern __shared__ __align__(16) uint32_t acc[];
  for (int i = threadIdx.x; i < kWords32; i += blockDim.x) acc[i] = 0;
  uint32_t peer_base = 0;
  if constexpr (MODE == DSMEM_RED || MODE == DSMEM_ATOM) {
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    const uint32_t me = (uint32_t)__cvta_generic_to_shared(acc);
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(peer_base) : "r"(me), "r"(cl.block_rank() ^ 1u));
  } else {
    __syncthreads();
  }
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(acc);
  const uint32_t lane = threadIdx.x & 31;
  uint32_t s[kUnroll];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) s[u] = lcg((blockIdx.x * 1024u + threadIdx.x) * 2654435761u + u * 40503u);
  uint32_t sink = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      s[u] = lcg(s[u]);
      uint32_t a = s[u] >> 17;                                   // 15 bits: word index
      if (skew && ((s[u] >> 3) & 7) == 0) a = (s[u] >> 6) & 63;  // hot words
      if constexpr (MODE == ATOM32_CF) a = (a & ~31u) | lane;     // lane l -> bank l
      const uint32_t t = (s[u] & 0xFFFFu) | 1u;
      if constexpr (MODE == ATOM32 || MODE == ATOM32_CF) {
        uint32_t old;
        asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(base + 4 * a), "r"(t) : "memory");
        sink += old;
      } else if constexpr (MODE == RED32) {
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(base + 4 * a), "r"(t) : "memory");
      } else if constexpr (MODE == ATOM64) {
        unsigned long long old;
        asm volatile("atom.shared.add.u64 %0, [%1], %2;" : "=l"(old) : "r"(base + 8 * (a >> 1)), "l"((unsigned long long)t)
                     : "memory");
        sink += (uint32_t)old;
      } else if constexpr (MODE == RED64) {
        asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(base + 8 * (a >> 1)), "l"((unsigned long long)t) : "memory");
      } else if constexpr (MODE == ATOMF) {
        sink += __float_as_uint(atomicAdd(reinterpret_cast<float*>(&acc[a]), __uint_as_float(t)));
      } else if constexpr (MODE == REDF) {
        asm volatile("red.shared.add.f32 [%0], %1;" ::"r"(base + 4 * a), "f"(__uint_as_float(t)) : "memory");
      } else if constexpr (MODE == PLAIN) {
        volatile uint32_t* p = acc + a;
        *p = *p + t;
      } else if constexpr (MODE == DSMEM_RED) {
        asm volatile("red.shared::cluster.add.u32 [%0], %1;" ::"r"(peer_base + 4 * a), "r"(t) : "memory");
      } else if constexpr (MODE == DSMEM_ATOM) {
        uint32_t old;
        asm volatile("atom.shared::cluster.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(peer_base + 4 * a), "r"(t)
                     : "memory");
        sink += old;
      }
    }
  }
  if constexpr (MODE == DSMEM_RED || MODE == DSMEM_ATOM) cg::this_cluster().sync();
  else __syncthreads();
  uint32_t x = sink;
  for (int i = threadIdx.x; i < kWords32; i += blockDim.x) x ^= acc[i];
  atomicAdd(out, x);
}

template <int MODE>
float run(int blocks, int iters, int skew, uint32_t* out, int smem) {
  cudaFuncSetAttribute(k_acc<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(1024);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (MODE == DSMEM_RED || MODE == DSMEM_ATOM) ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, k_acc<MODE>, iters, skew, out);   // warm-up
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) cudaLaunchKernelEx(&cfg, k_acc<MODE>, iters, skew, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "%s: %s\n", kNames[MODE], cudaGetErrorString(e));
    return -1.f;
  }
  return ms / reps;
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  uint32_t* out;
  cudaMalloc(&out, 4);
  const int smem = kWords32 * 4;
  const int iters = 2048;
  const int blocks = sms - (sms & 1);   // even, for the 2-CTA clusters
  for (int skew = 0; skew < 2; ++skew)
    for (int mode = 0; mode < NMODES; ++mode) {
      float ms = -1.f;
      switch (mode) {
        case ATOM32: ms = run<ATOM32>(blocks, iters, skew, out, smem); break;
        case RED32: ms = run<RED32>(blocks, iters, skew, out, smem); break;
        case ATOM64: ms = run<ATOM64>(blocks, iters, skew, out, smem); break;
        case RED64: ms = run<RED64>(blocks, iters, skew, out, smem); break;
        case ATOMF: ms = run<ATOMF>(blocks, iters, skew, out, smem); break;
        case REDF: ms = run<REDF>(blocks, iters, skew, out, smem); break;
        case PLAIN: ms = run<PLAIN>(blocks, iters, skew, out, smem); break;
        case ATOM32_CF: ms = run<ATOM32_CF>(blocks, iters, skew, out, smem); break;
        case DSMEM_RED: ms = run<DSMEM_RED>(blocks, iters, skew, out, smem); break;
        case DSMEM_ATOM: ms = run<DSMEM_ATOM>(blocks, iters, skew, out, smem); break;
      }
      if (ms <= 0.f) continue;
      const double ops = (double)blocks * 1024.0 * iters * kUnroll;
      const double per_clk = ops / (ms * 1e-3) / blocks / (clk_khz * 1e3);   // per SM per clock (max clock)
      printf("{\"op\": \"%s\", \"dist\": \"%s\", \"ms\": %.4f, \"gops\": %.2f, \"ops_per_sm_clk\": %.3f, "
             "\"implied_wavefronts_per_warp_instr\": %.2f, \"sm_clk_mhz_max\": %d}\n",
             kNames[mode], skew ? "skew" : "uniform", ms, ops / ms / 1e6, per_clk, 32.0 / per_clk, clk_khz / 1000);
    }
  return 0;
}

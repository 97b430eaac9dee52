// Microbenchmark: shared-memory accumulator throughput on sm_100a.
// Design evidence for the gather accumulator choice.
// Each CTA owns a 2^15-entry smem array (128 KB of u32 / f32) and performs
// random-address accumulations, like the PCPM gather into one destination
// partition. Variants: u32 atomicAdd with returned old value (fixed-point lo
// word + carry check), u32 red (no return), f32 atomicAdd (CAS loop on smem),
// and a racy plain LDS/STS add as the no-atomic floor.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define Q (1 << 15)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

template <int MODE>
__global__ void __launch_bounds__(1024, 1) k_atoms(int iters, uint32_t* out, int skew) {
  extern __shared__ uint32_t acc[];
  for (int i = threadIdx.x; i < Q; i += blockDim.x) acc[i] = 0;
  __syncthreads();
  uint32_t s = hash32(blockIdx.x * 4096 + threadIdx.x);
  uint32_t carry = 0;
  for (int it = 0; it < iters; ++it) {
    s = hash32(s + it);
    uint32_t a = s & (Q - 1);
    if (skew) { // 1/8 of the adds go to 64 hot addresses
      if ((s >> 20 & 7) == 0) a = (s >> 24) & 63;
    }
    uint32_t t = (s >> 8) | 1u;
    if (MODE == 0) {
      uint32_t old = atomicAdd(&acc[a], t);
      carry += (old + t < old);
    } else if (MODE == 1) {
      asm volatile("red.shared.add.u32 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(&acc[a])), "r"(t));
    } else if (MODE == 2) {
      atomicAdd(reinterpret_cast<float*>(&acc[a]), __uint_as_float(t & 0x3fffffff));
    } else {
      acc[a] += t;
    }
  }
  __syncthreads();
  uint32_t x = 0;
  for (int i = threadIdx.x; i < Q; i += blockDim.x) x ^= acc[i];
  atomicAdd(out, x + carry);
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int l2 = 0, smem_optin = 0, smem_sm = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("device %s SMs %d L2 %d B smem/block optin %d smem/SM %d clock %d kHz\n", p.name,
         p.multiProcessorCount, l2, smem_optin, smem_sm, clk);
  uint32_t* out; cudaMalloc(&out, 4);
  const int smem = Q * 4;
  cudaFuncSetAttribute(k_atoms<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_atoms<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_atoms<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_atoms<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[4] = {"u32 atomicAdd+ret", "u32 red", "f32 atomicAdd(CAS)", "plain lds/sts"};
  int threads_list[3] = {256, 512, 1024};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int skew = 0; skew < 2; ++skew)
  for (int mode = 0; mode < 4; ++mode)
  for (int ti = 0; ti < 3; ++ti) {
    int threads = threads_list[ti];
    int blocks = p.multiProcessorCount;
    int iters = 4096;
    auto launch = [&]() {
      if (mode == 0) k_atoms<0><<<blocks, threads, smem>>>(iters, out, skew);
      if (mode == 1) k_atoms<1><<<blocks, threads, smem>>>(iters, out, skew);
      if (mode == 2) k_atoms<2><<<blocks, threads, smem>>>(iters, out, skew);
      if (mode == 3) k_atoms<3><<<blocks, threads, smem>>>(iters, out, skew);
    };
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    double ops = (double)blocks * threads * iters;
    printf("skew=%d %-22s threads=%4d  %.3f ms  %.1f Gop/s  %.3f op/clk/SM@1.9GHz\n", skew, names[mode], threads, ms,
           ops / ms / 1e6, ops / (ms * 1e-3) / p.multiProcessorCount / 1.9e9);
  }
  cudaError_t err = cudaGetLastError();
  printf("err: %s\n", cudaGetErrorString(err));
  return 0;
}

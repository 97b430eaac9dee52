// pull.cu -- PageRank initialisation (R2: PR_0 = 1/n) and the in-house
// comparison kernel: naive pull-direction PageRank, Alg. 1,
// one warp per destination vertex summing SPR over its in-neighbours (CSC) in
// fp64 registers, with the same apply / dangling rule (R1) as the PCPM path.
#include "pcpm_internal.cuh"

namespace pcpm {
namespace {

// spr_scale: 2^F for the PCPM path (the gather converts SPR * 2^F straight to its
// fixed-point grid, R21), 1 for the pull comparison.
__global__ void k_pr_init(int64_t n, const uint32_t* __restrict__ outdeg, int64_t n_dangling, float* pr0,
                          float* spr, double* red, int red_n, double spr_scale) {
  const double inv_n = 1.0 / (double)n;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    pr0[v] = (float)inv_n;
    const uint32_t dg = outdeg[v];
    spr[v] = dg ? (float)(inv_n / (double)dg * spr_scale) : 0.0f;
  }
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < red_n; i += blockDim.x) red[i] = 0.0;
    __syncthreads();
    if (threadIdx.x == 0) red[0] = (double)n_dangling * inv_n;   // D_0
  }
}

// PR_0 = 1/n_global on a destination shard's slice (R2), SPR_0 = PR_0 / outdeg, and the
// slice's dangling count; k_dang0 turns the count into D_0's share (exact: count / n).
__global__ void k_pr_init_slice(int64_t n_local, const uint32_t* __restrict__ outdeg, double inv_n, float* pr0,
                                float* spr, unsigned long long* cnt, double spr_scale) {
  unsigned long long local = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n_local;
       v += (int64_t)gridDim.x * blockDim.x) {
    pr0[v] = (float)inv_n;
    const uint32_t dg = outdeg[v];
    spr[v] = dg ? (float)(inv_n / (double)dg * spr_scale) : 0.0f;
    local += dg == 0;
  }
  for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(cnt, local);
}
__global__ void k_dang0(const unsigned long long* cnt, double inv_n, double* dang0) {
  *dang0 = (double)*cnt * inv_n;
}

__global__ void __launch_bounds__(256) k_pull(int64_t n, const uint32_t* __restrict__ in_ptr,
                                              const uint32_t* __restrict__ in_src, const float* __restrict__ spr_in,
                                              const uint32_t* __restrict__ outdeg, const float* __restrict__ pr_old,
                                              float* pr_new, float* spr_out, const double* red_in, double* red_out,
                                              double d) {
  const int lane = threadIdx.x & 31;
  const double base = (1.0 - d) / (double)n + d * (red_in[0] / (double)n);
  double dang = 0.0, res = 0.0;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < n; v += nw) {
    double s = 0.0;
    for (uint32_t e = in_ptr[v] + lane; e < in_ptr[v + 1]; e += 32) s += (double)__ldg(spr_in + in_src[e]);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      const double prn = base + d * s;
      pr_new[v] = (float)prn;
      const uint32_t dg = outdeg[v];
      spr_out[v] = dg ? (float)(prn / (double)dg) : 0.0f;
      if (dg == 0) dang += prn;
      res += fabs(prn - (double)pr_old[v]);
    }
  }
  if (lane == 0) {
    atomicAdd(&red_out[2], dang);
    atomicAdd(&red_out[1], res);
  }
}

}  // namespace

// Weighted PageRank (R24): PR_0 = 1/n, SPR_0 = f32(PR_0) * 1/W(u) * 2^F (the apply's
// form, R23), D_0 = #{W(u) = 0} / n.
__global__ void k_pr_init_w(int64_t n, const float* __restrict__ inv_w, int64_t n_zero, float* pr0, float* spr,
                            double* red, int red_n, float spr_scale) {
  const double inv_n = 1.0 / (double)n;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    pr0[v] = (float)inv_n;
    spr[v] = (float)inv_n * inv_w[v] * spr_scale;
  }
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < red_n; i += blockDim.x) red[i] = 0.0;
    __syncthreads();
    if (threadIdx.x == 0) red[0] = (double)n_zero * inv_n;   // D_0
  }
}

int launch_pr_init_weighted(pcpm_handle* h, float* pr0, float* spr, double* red, int red_n, float spr_scale,
                            cudaStream_t s) {
  const int grid = (int)std::min<int64_t>((h->n_src + 255) / 256, h->num_sms * 8);
  k_pr_init_w<<<std::max(grid, 1), 256, 0, s>>>(h->n_src, h->inv_wdeg, h->n_wdangling, pr0, spr, red, red_n,
                                                spr_scale);
  PCPM_CK(cudaGetLastError());
  h->launches += 1;
  return PCPM_OK;
}

int launch_pr_init(pcpm_handle* h, float* pr0, float* spr, double* red, int red_n, double spr_scale, cudaStream_t s) {
  int grid = (int)std::min<int64_t>((h->n_src + 255) / 256, h->num_sms * 8);
  k_pr_init<<<std::max(grid, 1), 256, 0, s>>>(h->n_src, h->outdeg, h->n_dangling, pr0, spr, red, red_n,
                                                  spr_scale);
  PCPM_CK(cudaGetLastError());
  h->launches += 1;
  return PCPM_OK;
}

int launch_pr_init_slice(pcpm_handle* h, float* pr0, float* spr, double* dang0, double spr_scale, cudaStream_t s) {
  const int64_t n_local = h->n_dst;
  const double inv_n = 1.0 / (double)h->n_global;
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(h->counters + 4);   // [4..5] scratch
  PCPM_CK(cudaMemsetAsync(cnt, 0, 8, s));
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n_local + 255) / 256, h->num_sms * 8));
  k_pr_init_slice<<<grid, 256, 0, s>>>(n_local, h->outdeg + h->shard_lo, inv_n, pr0, spr, cnt, spr_scale);
  PCPM_CK(cudaGetLastError());
  k_dang0<<<1, 1, 0, s>>>(cnt, inv_n, dang0);
  PCPM_CK(cudaGetLastError());
  PCPM_CK(cudaMemsetAsync(cnt, 0, 8, s));        // counters are kept zero
  h->launches += 2;
  return PCPM_OK;
}

int launch_pull_iteration(pcpm_handle* h, const float* spr_in, const float* pr_old, float* pr_new, float* spr_out,
                          double* red_t, double d, cudaStream_t s) {
  const int grid = h->num_sms * 8;
  k_pull<<<grid, 256, 0, s>>>(h->n_dst, h->in_ptr, h->in_src, spr_in, h->outdeg, pr_old, pr_new, spr_out, red_t,
                              red_t, (double)d);
  PCPM_CK(cudaGetLastError());
  h->launches += 1;
  return PCPM_OK;
}

}  // namespace pcpm

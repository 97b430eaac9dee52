// build.cu -- a0: the one-time, GPU-built PCPM layout (§3.1-3.3).
//
// From a CSR (row u lists its out-neighbours v ascending) build, all on
// the device and integer-only (bit-identical to the oracle's layout):
//   * destID bins: edges stably sorted by destination
//     partition j = v >> b, so bin j lists IDs in (u, v) order; the MSB flags
//     the first ID of each (u, j) run (Alg. 2's prev_bin test);
//   * the PNG: flagged edges (one per (u, j) pair = Eff_1) stably
//     sorted by (p = u >> b, j) -- the per-partition transposition -- so group
//     (p, j) lists its sources u ascending; png_off are the group starts;
//   * write offsets: upd_off[p][j] = bin_upd_start[j] + sum_{p'<p}
//     |group (p', j)|; bin starts are exclusive scans over j;
//   * chunk_base[c] = #flags in ids[0 .. 128 c): the anchors of the global
//     decode identity used by the gather;
//   * out-degrees, dangling count, work lists for the scatter and gather.
// Sorting replaces the paper's two counting scans because a stable
// radix sort is deterministic and bandwidth-bound on B200; the result is the
// same layout.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <type_traits>

#include "pcpm_internal.cuh"

namespace pcpm {
namespace {

constexpr int kT = 256;

inline int grid_for(int64_t n, int threads = kT) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return static_cast<int>(g);
}

inline int bits_for(uint64_t maxval) {  // bits needed to represent values in [0, maxval]
  int bits = 1;
  while (bits < 64 && (maxval >> bits) != 0) ++bits;
  return bits;
}

#define GRID_STRIDE(i, n) \
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

__global__ void k_check_rows(int64_t n, const int64_t* __restrict__ row_ptr, int64_t m, uint32_t* err) {
  GRID_STRIDE(u, n) {
    int64_t a = row_ptr[u], c = row_ptr[u + 1];
    if (a > c || a < 0 || c > m) atomicOr(err, 1u);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (row_ptr[0] != 0 || row_ptr[n] != m) atomicOr(err, 1u);
  }
}

__global__ void k_mark_rows(int64_t n, const int64_t* __restrict__ row_ptr, uint32_t* rowid) {
  GRID_STRIDE(u, n) {
    if (row_ptr[u] < row_ptr[u + 1]) rowid[row_ptr[u]] = static_cast<uint32_t>(u);
  }
}

struct MaxOp {
  __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return a > b ? a : b; }
};

__global__ void k_iota(int64_t n, uint32_t* out) {
  GRID_STRIDE(i, n) out[i] = static_cast<uint32_t>(i);
}

// Per edge: bin j, run flag (Alg. 2 prev_bin / MSB demarcation P:172-173), validation.
__global__ void k_classify(int64_t m, const uint32_t* __restrict__ col, const uint32_t* __restrict__ rowid,
                           int b, int64_t n_dst, bool compress, uint32_t* keyj, uint32_t* enc,
                           uint8_t* flags, uint32_t* err) {
  GRID_STRIDE(e, m) {
    uint32_t u = rowid[e];
    uint32_t v = col[e];
    bool first = (e == 0) || rowid[e - 1] != u;
    uint32_t pv = first ? 0u : col[e - 1];
    if (v >= n_dst) atomicOr(err, 2u);
    if (!first && pv >= v) atomicOr(err, 4u);
    uint32_t j = v >> b;
    bool flag = compress ? (first || (pv >> b) != j) : true;
    keyj[e] = j;
    enc[e] = v | (flag ? 0x80000000u : 0u);
    flags[e] = flag ? 1 : 0;
  }
}

// starts[key] = first position x with sorted_keys[x] >= key, for key in [0, nkeys]
__global__ void k_boundaries(int64_t m, const uint32_t* __restrict__ sorted_keys, int64_t nkeys, uint32_t* starts) {
  GRID_STRIDE(x, m + 1) {
    int64_t kx = x < m ? (int64_t)sorted_keys[x] : nkeys;
    int64_t kp = x > 0 ? (int64_t)sorted_keys[x - 1] : -1;
    for (int64_t k = kp + 1; k <= kx && k <= nkeys; ++k) starts[k] = static_cast<uint32_t>(x);
  }
}

// ids[x] = v | flag << 31 (4-byte form), ids16[x] = (v & (q-1)) | flag << 15 (compact form)
__global__ void k_gather_ids(int64_t m, const uint32_t* __restrict__ perm, const uint32_t* __restrict__ enc,
                             const float* __restrict__ values, uint32_t qmask, uint32_t* ids, uint16_t* ids16,
                             float* w) {
  GRID_STRIDE(x, m) {
    uint32_t e = perm[x];
    const uint32_t id = enc[e];
    ids[x] = id;
    ids16[x] = (uint16_t)((id & qmask) | ((id >> 31) << 15));
    if (w) w[x] = values ? values[e] : 1.0f;
  }
}

// PCPM_COMPACT_SLOTS: one block per destination bin j.  has_in[j q + l] = 1 for every
// local ID l in bin j; then (after a scan) ids16 local indices become slots.
__global__ void k_mark_in(const uint32_t* __restrict__ bin_start, const uint16_t* __restrict__ ids16, int b,
                          uint32_t* has_in) {
  const uint32_t j = blockIdx.x;
  const uint32_t s0 = bin_start[j], s1 = bin_start[j + 1];
  const size_t base = (size_t)j << b;
  for (uint32_t x = s0 + threadIdx.x; x < s1; x += blockDim.x) has_in[base + (ids16[x] & 0x7FFFu)] = 1u;
}
// slot16[v] = rank of v among its partition's vertices with in-edges (0xFFFF: none)
__global__ void k_slots(int64_t n, int b, const uint32_t* __restrict__ has_in, const uint32_t* __restrict__ scan,
                        uint16_t* slot16) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v0 = (v >> b) << b;
    slot16[v] = has_in[v] ? (uint16_t)(scan[v] - scan[v0]) : (uint16_t)0xFFFFu;
  }
}
__global__ void k_slotmap(int64_t nw, const uint32_t* __restrict__ has_in, const uint32_t* __restrict__ scan, int b,
                          uint2* slotmap) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nw; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = w * 32, v0 = (v >> b) << b;
    uint32_t bits = 0;
    for (int i = 0; i < 32; ++i) bits |= (has_in[v + i] ? 1u : 0u) << i;
    slotmap[w] = make_uint2(bits, scan[v] - scan[v0]);
  }
}
__global__ void k_remap_ids(const uint32_t* __restrict__ bin_start, int b, const uint16_t* __restrict__ slot16,
                            uint16_t* ids16) {
  const uint32_t j = blockIdx.x;
  const uint32_t s0 = bin_start[j], s1 = bin_start[j + 1];
  const uint16_t* sl = slot16 + ((size_t)j << b);
  for (uint32_t x = s0 + threadIdx.x; x < s1; x += blockDim.x) {
    const uint16_t id = ids16[x];
    ids16[x] = (uint16_t)((id & 0x8000u) | sl[id & 0x7FFFu]);
  }
}

__global__ void k_ids16(int64_t m, const uint32_t* __restrict__ ids, uint32_t qmask, uint16_t* ids16) {
  GRID_STRIDE(x, m) {
    const uint32_t id = ids[x];
    ids16[x] = (uint16_t)((id & qmask) | ((id >> 31) << 15));
  }
}

__global__ void k_png16(int64_t ep, const uint32_t* __restrict__ png, uint32_t qmask, uint16_t* png16) {
  GRID_STRIDE(i, ep) png16[i] = (uint16_t)(png[i] & qmask);
}

__global__ void k_png_keys(int64_t ep, const uint32_t* __restrict__ sel, const uint32_t* __restrict__ rowid,
                           const uint32_t* __restrict__ col, int b, int64_t k_dst, uint32_t* key, uint32_t* val) {
  GRID_STRIDE(i, ep) {
    uint32_t e = sel[i];
    uint32_t u = rowid[e];
    key[i] = static_cast<uint32_t>((int64_t)(u >> b) * k_dst + (col[e] >> b));
    val[i] = u;
  }
}

// grp_at[c] = flat group (p*k_dst + j) of PNG entry kPngChunk*c (the sorted group keys)
__global__ void k_grp_at(int64_t ep, const uint32_t* __restrict__ keys_sorted, int64_t n, uint32_t* grp_at) {
  GRID_STRIDE(c, n) {
    const int64_t x = c * kPngChunk;
    grp_at[c] = keys_sorted[x < ep ? x : ep - 1];
  }
}

// png_off[p][j] = G[p*k_dst + j] for j <= k_dst
__global__ void k_png_off(int64_t k_src, int64_t k_dst, const uint32_t* __restrict__ G, uint32_t* png_off) {
  GRID_STRIDE(i, k_src * (k_dst + 1)) {
    int64_t p = i / (k_dst + 1), j = i % (k_dst + 1);
    png_off[i] = G[p * k_dst + j];
  }
}

// Column scans of the group sizes: out[p][j] = sum_{p'<p} |(p', j)|, col_tot[j].
// Block = 32 columns x 32 row segments: segment sums, a scan over the segments, then
// each segment's running offsets (coalesced over j).
__global__ void __launch_bounds__(1024) k_col_scan(int64_t k_src, int64_t k_dst, const uint32_t* __restrict__ G,
                                                   uint32_t* out, uint32_t* col_tot) {
  __shared__ uint32_t part[32][33];
  const int64_t j = blockIdx.x * 32 + threadIdx.x;
  const int y = threadIdx.y;
  const int64_t per = (k_src + 31) / 32;
  const int64_t p0 = min(k_src, y * per), p1 = min(k_src, p0 + per);
  uint32_t sum = 0;
  if (j < k_dst)
    for (int64_t p = p0; p < p1; ++p) sum += G[p * k_dst + j + 1] - G[p * k_dst + j];
  part[y][threadIdx.x] = sum;
  __syncthreads();
  if (y == 0) {
    uint32_t run = 0;
    for (int k = 0; k < 32; ++k) {
      const uint32_t t = part[k][threadIdx.x];
      part[k][threadIdx.x] = run;
      run += t;
    }
    if (j < k_dst) col_tot[j] = run;
  }
  __syncthreads();
  uint32_t run = part[y][threadIdx.x];
  if (j < k_dst)
    for (int64_t p = p0; p < p1; ++p) {
      const int64_t g = p * k_dst + j;
      out[g] = run;
      run += G[g + 1] - G[g];
    }
}
inline void col_scan(int64_t k_src, int64_t k_dst, const uint32_t* G, uint32_t* out, uint32_t* col_tot,
                     cudaStream_t s) {
  k_col_scan<<<(unsigned)((k_dst + 31) / 32), dim3(32, 32), 0, s>>>(k_src, k_dst, G, out, col_tot);
}

// starts[g] = base + first x with keys[x] >= g, for g in [g0, g1]; keys (n of them)
// sorted and in [g0, g1).  n and base may come from device memory (n_dev, base_dev).
__global__ void k_bounds_range(int64_t n_max, const int64_t* n_dev, const uint32_t* __restrict__ keys, int64_t g0,
                               int64_t g1, int64_t base, const int64_t* base_dev, uint32_t* starts) {
  const int64_t n = n_dev ? *n_dev : n_max;
  const int64_t b0 = base_dev ? *base_dev : base;
  GRID_STRIDE(x, n + 1) {
    const int64_t kx = x < n ? (int64_t)keys[x] : g1;
    const int64_t kp = x > 0 ? (int64_t)keys[x - 1] : g0 - 1;
    for (int64_t k = kp + 1; k <= kx; ++k) starts[k] = static_cast<uint32_t>(b0 + x);
  }
}

// Scatter work items (p, [j0, j1)) of ~target updates (at most maxg groups), one warp
// per source partition p: count pass (out == nullptr) or fill pass at off[p].
// Partitions p >= p_tail (the last ones claimed) are cut ~tail_split times finer, so the
// final wave of the persistent scatter has small items (less idle tail).
__global__ void k_sitems(int64_t k_src, int64_t k_dst, const uint32_t* __restrict__ G, int64_t target, int maxg,
                         int64_t p_tail, int tail_split, const uint32_t* __restrict__ off, uint32_t* cnt,
                         ScatterItem* out) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t p = w0; p < k_src; p += nw) {
    uint32_t n = 0, j0 = 0;
    int64_t acc = 0;
    const int64_t ep_p = (int64_t)G[(p + 1) * k_dst] - (int64_t)G[p * k_dst];
    const int64_t tgt = (p >= p_tail && tail_split > 1) ? max((int64_t)4096, min(target, ep_p / tail_split + 1)) : target;
    const uint32_t o = out ? off[p] : 0u;
    for (int64_t jb = 0; jb < k_dst; jb += 32) {
      const int64_t jl = jb + lane;
      const uint32_t sz = jl < k_dst ? G[p * k_dst + jl + 1] - G[p * k_dst + jl] : 0u;
      const int nt = (int)(k_dst - jb < 32 ? k_dst - jb : 32);
      for (int t = 0; t < nt; ++t) {
        acc += __shfl_sync(0xffffffffu, sz, t);
        const uint32_t jj = (uint32_t)(jb + t);
        if (acc >= tgt || jj + 1 - j0 >= (uint32_t)maxg) {         // item offsets fit in smem
          if (out && lane == 0) out[o + n] = ScatterItem{(uint32_t)p, j0, jj + 1, (uint32_t)acc};
          ++n;
          acc = 0;
          j0 = jj + 1;
        }
      }
    }
    if (acc > 0) {
      if (out && lane == 0) out[o + n] = ScatterItem{(uint32_t)p, j0, (uint32_t)k_dst, (uint32_t)acc};
      ++n;
    }
    if (!out && lane == 0) cnt[p] = n;
  }
}

__global__ void k_add_bin_start(int64_t k_src, int64_t k_dst, const uint32_t* __restrict__ bin_upd_start,
                                uint32_t* upd_off) {
  GRID_STRIDE(i, k_src * k_dst) upd_off[i] += bin_upd_start[i % k_dst];
}

// flags per kChunkIds-ID chunk from the compact IDs (flag = bit 15): one warp per chunk, 4 IDs per lane
__global__ void k_chunk_counts16(int64_t nchunks, const uint16_t* __restrict__ ids16, uint32_t* cnt) {
  int lane = threadIdx.x & 31;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = warp; c < nchunks; c += nw) {
    uint2 v = reinterpret_cast<const uint2*>(ids16 + c * kChunkIds)[lane];
    uint32_t f = ((v.x >> 15) & 1u) + (v.x >> 31) + ((v.y >> 15) & 1u) + (v.y >> 31);
    for (int o = 16; o; o >>= 1) f += __shfl_xor_sync(0xffffffffu, f, o);
    if (lane == 0) cnt[c] = f;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) cnt[nchunks] = 0;
}

// |N_o(u)| and its fp32 reciprocal (0 for dangling u; the apply multiplies by it)
__global__ void k_outdeg(int64_t u0, int64_t n, const int64_t* __restrict__ row_ptr, uint32_t* outdeg, float* inv_deg,
                         unsigned long long* n_dangling) {
  __shared__ unsigned int s;
  if (threadIdx.x == 0) s = 0;
  __syncthreads();
  unsigned int local = 0;
  GRID_STRIDE(i, n) {
    const int64_t u = u0 + i;
    uint32_t dg = static_cast<uint32_t>(row_ptr[u + 1] - row_ptr[u]);
    outdeg[u] = dg;
    inv_deg[u] = dg ? 1.0f / (float)dg : 0.0f;
    local += dg == 0;
  }
  atomicAdd(&s, local);
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(n_dangling, (unsigned long long)s);
}

__global__ void k_item_f(int n_items, GatherItem* items, const uint32_t* __restrict__ chunk_base,
                         const uint32_t* __restrict__ bin_upd_start, int jshift = 0) {
  GRID_STRIDE(i, n_items) {
    GatherItem it = items[i];
    const uint32_t bj = it.j >> jshift;               // pair handles: item j is a half of bin j >> 1
    it.fx0 = (it.x0 % kChunkIds == 0) ? chunk_base[it.x0 / kChunkIds] : bin_upd_start[bj];
    it.fx1 = (it.x1 % kChunkIds == 0) ? chunk_base[it.x1 / kChunkIds] : bin_upd_start[bj + 1];
    items[i] = it;
  }
}

// CSC for the pull comparison: in_src[x] = rowid[perm[x]]
__global__ void k_gather_u32(int64_t m, const uint32_t* __restrict__ perm, const uint32_t* __restrict__ src,
                             uint32_t* out) {
  GRID_STRIDE(x, m) out[x] = src[perm[x]];
}

// Column slice [lo, hi) of each (sorted) row: a = lower_bound(lo), c = lower_bound(hi).
__global__ void k_slice_count(int64_t n, const int64_t* __restrict__ row_ptr, const uint32_t* __restrict__ col,
                              uint32_t lo, uint32_t hi, int64_t* cnt, int64_t* first) {
  GRID_STRIDE(u, n) {
    int64_t a = row_ptr[u], e = row_ptr[u + 1];
    int64_t l = a, r = e;
    while (l < r) {
      const int64_t mid = (l + r) >> 1;
      if (col[mid] < lo) l = mid + 1; else r = mid;
    }
    const int64_t x0 = l;
    r = e;
    while (l < r) {
      const int64_t mid = (l + r) >> 1;
      if (col[mid] < hi) l = mid + 1; else r = mid;
    }
    cnt[u] = l - x0;
    first[u] = x0;
  }
}

__global__ void k_slice_fill(int64_t n, const int64_t* __restrict__ new_ptr, const int64_t* __restrict__ first,
                             const uint32_t* __restrict__ col, const float* __restrict__ val, uint32_t lo,
                             uint32_t* out_col, float* out_val) {
  // one warp per row
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = w0; u < n; u += nw) {
    const int64_t o = new_ptr[u], len = new_ptr[u + 1] - o, f = first[u];
    for (int64_t i = lane; i < len; i += 32) {
      out_col[o + i] = col[f + i] - lo;
      if (out_val) out_val[o + i] = val[f + i];
    }
  }
}


// ---------------------------------------------------------------------------
// Chunked construction (the default; DESIGN.md §5 "build").  The CSR is cut into
// chunks of whole source partitions [p0, p1).  Each chunk's edges are stably
// sorted by the flat group key g = (u >> b) * k_dst + (v >> b); one payload word
// carries everything else: (v & (q-1)) | flag << 15 | (u & (q-1)) << 16.  Since a
// chunk holds whole partitions and the CSR lists u ascending (v ascending per
// row), the concatenated chunk sorts are sorted by g with edges in (u, v) order
// inside each group (p, j).  Then
//   * destID bin j = groups (0, j), (1, j), ... concatenated: each
//     group is placed at id_off[p][j] = bin_id_start[j] + sum_{p' < p} |(p', j)|;
//   * the PNG = the flagged edges in the same order (Eff_1: one per
//     (u, j) run; transposed: grouped by (p, j), u ascending).
// With host inputs, chunk c+1 is copied (copy stream) while chunk c is sorted.
struct PayW {                // payload of weighted builds: the word above + the fp32 value
  uint32_t x, y;
};
__device__ __forceinline__ uint32_t pay_word(uint32_t p) { return p; }
__device__ __forceinline__ uint32_t pay_word(PayW p) { return p.x; }
__device__ __forceinline__ float pay_value(uint32_t) { return 1.0f; }
__device__ __forceinline__ float pay_value(PayW p) { return __uint_as_float(p.y); }

__global__ void k_check_rows_c(int64_t u0, int64_t nr, const int64_t* __restrict__ row_ptr, int64_t e0, int64_t e1,
                               uint32_t* err) {
  GRID_STRIDE(i, nr) {
    const int64_t a = row_ptr[u0 + i], c = row_ptr[u0 + i + 1];
    if (a > c || a < e0 || c > e1) atomicOr(err, 1u);
  }
}

__global__ void k_mark_rows_c(int64_t u0, int64_t nr, const int64_t* __restrict__ row_ptr, int64_t e0, int64_t e1,
                              uint32_t* mark) {
  GRID_STRIDE(i, nr) {
    const int64_t a = row_ptr[u0 + i], c = row_ptr[u0 + i + 1];
    if (a < c && a >= e0 && a < e1) mark[a - e0] = static_cast<uint32_t>(u0 + i);
  }
}

// Per edge of the chunk: group key, run flag (Alg. 2 prev_bin / MSB demarcation,
// P:172-173), payload; validation (col < n_dst, rows strictly increasing).
template <typename P>
__global__ void k_classify_c(int64_t e0, int64_t mc, const uint32_t* __restrict__ col, const float* __restrict__ val,
                             const uint32_t* __restrict__ rowid, int b, int64_t n_dst, int64_t k_dst, bool compress,
                             uint32_t* key, P* pay, uint32_t* err) {
  const uint32_t qmask = (1u << b) - 1u;
  GRID_STRIDE(i, mc) {
    const uint32_t u = rowid[i];
    const uint32_t v = col[e0 + i];
    const bool first = (i == 0) || rowid[i - 1] != u;
    const uint32_t pv = first ? 0u : col[e0 + i - 1];
    if (v >= n_dst) atomicOr(err, 2u);
    if (!first && pv >= v) atomicOr(err, 4u);
    uint32_t j = v >> b;
    if (j >= (uint32_t)k_dst) j = (uint32_t)k_dst - 1;      // invalid input: keep the key in range
    const bool flag = compress ? (first || (pv >> b) != (v >> b)) : true;
    key[i] = static_cast<uint32_t>((int64_t)(u >> b) * k_dst + j);
    const uint32_t w = (v & qmask) | (flag ? 0x8000u : 0u) | ((u & qmask) << 16);
    if constexpr (std::is_same<P, PayW>::value) pay[i] = PayW{w, __float_as_uint(val[e0 + i])};
    else pay[i] = w;
  }
}

template <typename P>
__global__ void k_run_flags(int64_t n, const P* __restrict__ pay, uint8_t* fl) {
  GRID_STRIDE(i, n) fl[i] = (uint8_t)((pay_word(pay[i]) >> 15) & 1u);
}

// destID bins: sorted edge x of group g goes to id_off[g] + (x - Gs[g]).
template <typename P>
__global__ void k_place_ids(int64_t m, const uint32_t* __restrict__ keys, const P* __restrict__ pay,
                            const uint32_t* __restrict__ Gs, const uint32_t* __restrict__ id_off, int b, int64_t k_dst,
                            uint16_t* ids16, uint32_t* ids32, float* w) {
  const uint32_t qmask = (1u << b) - 1u;
  GRID_STRIDE(x, m) {
    const uint32_t g = keys[x];
    const P pv = pay[x];
    const uint32_t word = pay_word(pv);
    const uint32_t dst = id_off[g] + (uint32_t)(x - Gs[g]);
    ids16[dst] = (uint16_t)(word & 0xFFFFu);
    if (ids32) ids32[dst] = ((uint32_t)(g % (uint32_t)k_dst) << b | (word & qmask)) | ((word >> 15) & 1u) << 31;
    if (w) w[dst] = pay_value(pv);
  }
}

// PNG, per chunk: its n = *n_dev flagged edges (in group order) go to positions
// off .. off + n, off = *off_dev (the flagged edges of the earlier chunks);
// *off_next = off + n.
template <typename P>
__global__ void k_png_place_c(const int64_t* __restrict__ n_dev, const int64_t* off_dev, int64_t* off_next,
                              const uint32_t* __restrict__ fk, const P* __restrict__ fp, int b, int64_t k_dst,
                              uint32_t* pk, uint16_t* png16, uint32_t* png32) {
  const int64_t n = *n_dev, off = *off_dev;
  if (blockIdx.x == 0 && threadIdx.x == 0) *off_next = off + n;
  GRID_STRIDE(i, n) {
    const uint32_t g = fk[i];
    const uint32_t ul = pay_word(fp[i]) >> 16;
    pk[off + i] = g;
    png16[off + i] = (uint16_t)ul;
    if (png32) png32[off + i] = (g / (uint32_t)k_dst) << b | ul;
  }
}


// ---------------------------------------------------------------------------
// Exclusive prefix sum of u32 counts (hand-written; out may alias in): per block of
// kScanTile elements a sum, one block scans the block sums, then every block scans its
// tile from its base.  Used for the bin / group / anchor offsets.
constexpr int kScanThreads = 1024, kScanPer = 4, kScanTile = kScanThreads * kScanPer;

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t* wsum, uint32_t* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t inc = x;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  if (w == 0) {
    const uint32_t ws = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0u;
    uint32_t wi = ws;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    wsum[lane] = wi - ws;
    if (lane == 31) *total = wi;
  }
  __syncthreads();
  return wsum[w] + inc - x;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_sums(const uint32_t* __restrict__ in, int64_t n,
                                                             uint32_t* bsum) {
  __shared__ uint32_t wsum[32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanPer;
  uint32_t x = 0;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) x += base + k < n ? in[base + k] : 0u;
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = x;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t y = wsum[threadIdx.x];
    for (int o = 16; o; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
    if (threadIdx.x == 0) bsum[blockIdx.x] = y;
  }
}

__global__ void __launch_bounds__(kScanThreads) k_scan_top(uint32_t* bsum, int64_t nb) {
  __shared__ uint32_t wsum[32];
  __shared__ uint32_t tot;
  uint32_t carry = 0;
  for (int64_t c = 0; c < nb; c += kScanThreads) {
    const int64_t i = c + threadIdx.x;
    const uint32_t x = i < nb ? bsum[i] : 0u;
    const uint32_t e = block_excl_scan(x, wsum, &tot);
    if (i < nb) bsum[i] = carry + e;
    carry += tot;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(const uint32_t* in, uint32_t* out, int64_t n,
                                                              const uint32_t* __restrict__ bsum) {
  __shared__ uint32_t wsum[32];
  __shared__ uint32_t tot;
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanPer;
  uint32_t v[kScanPer];
  uint32_t x = 0;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    v[k] = base + k < n ? in[base + k] : 0u;
    x += v[k];
  }
  uint32_t run = bsum[blockIdx.x] + block_excl_scan(x, wsum, &tot);
#pragma unroll
  for (int k = 0; k < kScanPer; ++k)
    if (base + k < n) {
      out[base + k] = run;
      run += v[k];
    }
}


// PCPM_BUILD_TIMING=1: synchronise and print the wall time of each build phase (stderr).
struct PhaseTimer {
  bool on = getenv("PCPM_BUILD_TIMING") != nullptr;
  cudaStream_t s;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  explicit PhaseTimer(cudaStream_t st) : s(st) {}
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[pcpm build] %-28s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  }
};

struct Temp {                 // build scratch: stream-ordered pool memory, freed in stream order
  std::vector<void*> ptrs;
  cudaStream_t s = nullptr;
  explicit Temp(cudaStream_t st) : s(st) {}
  ~Temp() {
    for (void* p : ptrs) cudaFreeAsync(p, s);
  }
  template <typename T>
  cudaError_t alloc(T** p, size_t count) {
    void* q = nullptr;
    cudaError_t e = cudaMallocAsync(&q, std::max<size_t>(count, 1) * sizeof(T), s);
    if (e == cudaSuccess) ptrs.push_back(q);
    *p = reinterpret_cast<T*>(q);
    return e;
  }
};

#define TK(call)                                                                 \
  do {                                                                           \
    cudaError_t _e = (call);                                                     \
    if (_e == cudaErrorMemoryAllocation) {                                       \
      cudaGetLastError();                                                        \
      set_error(PCPM_ENOMEM, std::string("device allocation failed: ") + #call); \
      return PCPM_ENOMEM;                                                        \
    }                                                                            \
    if (_e != cudaSuccess) return cuda_fail(_e, #call, __FILE__, __LINE__);     \
  } while (0)

// out[i] = sum of in[0 .. i), i < n (out may alias in)
int scan_excl_u32(Temp& tmp, const uint32_t* in, uint32_t* out, int64_t n, cudaStream_t s) {
  if (n <= 0) return PCPM_OK;
  const int64_t nb = (n + kScanTile - 1) / kScanTile;
  uint32_t* bsum;
  TK(tmp.alloc(&bsum, nb));
  k_scan_sums<<<(unsigned)nb, kScanThreads, 0, s>>>(in, n, bsum);
  k_scan_top<<<1, kScanThreads, 0, s>>>(bsum, nb);
  k_scan_tiles<<<(unsigned)nb, kScanThreads, 0, s>>>(in, out, n, bsum);
  TK(cudaGetLastError());
  return PCPM_OK;
}

template <typename KeyT, typename ValT>
cudaError_t radix_sort_pairs(Temp& tmp, const KeyT* kin, KeyT* kout, const ValT* vin, ValT* vout, int64_t n,
                             int end_bit, cudaStream_t s) {
  size_t bytes = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, n, 0, end_bit, s);
  if (e != cudaSuccess) return e;
  void* t = nullptr;
  e = tmp.alloc(reinterpret_cast<uint8_t**>(&t), bytes);
  if (e != cudaSuccess) return e;
  return cub::DeviceRadixSort::SortPairs(t, bytes, kin, kout, vin, vout, n, 0, end_bit, s);
}


// Weighted out-degrees W(u) = sum of row u's weights (fp64, lanes then a fixed shuffle
// tree: deterministic), 1/W(u) in fp32 (0 when W(u) = 0: dangling under R24), the
// count of such vertices and whether any weight is negative.  One warp per row.
__global__ void k_row_wsum(int64_t n, const int64_t* __restrict__ row_ptr, const float* __restrict__ val,
                           float* inv_w, unsigned long long* n_zero, uint32_t* neg) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = w0; u < n; u += nw) {
    double sum = 0.0;
    bool ng = false;
    for (int64_t e = row_ptr[u] + lane; e < row_ptr[u + 1]; e += 32) {
      const float x = val[e];
      sum += (double)x;
      ng = ng || x < 0.0f;
    }
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (__any_sync(0xffffffffu, ng) && lane == 0) atomicOr(neg, 1u);
    if (lane == 0) {
      inv_w[u] = sum > 0.0 ? (float)(1.0 / sum) : 0.0f;
      if (!(sum > 0.0)) atomicAdd(n_zero, 1ull);
    }
  }
}

int weighted_degrees(pcpm_handle* h, Temp& tmp, const int64_t* d_row_ptr, const float* d_val) {
  cudaStream_t s = h->stream;
  int rc;
  if ((rc = dev_alloc_t(h, &h->inv_wdeg, h->n_src + 4))) return rc;
  unsigned long long* cnt;
  uint32_t* neg;
  TK(tmp.alloc(&cnt, 1));
  TK(tmp.alloc(&neg, 1));
  TK(cudaMemsetAsync(cnt, 0, 8, s));
  TK(cudaMemsetAsync(neg, 0, 4, s));
  k_row_wsum<<<grid_for(h->n_src * 32), kT, 0, s>>>(h->n_src, d_row_ptr, d_val, h->inv_wdeg, cnt, neg);
  TK(cudaGetLastError());
  unsigned long long hc = 0;
  uint32_t hn = 0;
  TK(cudaMemcpyAsync(&hc, cnt, 8, cudaMemcpyDeviceToHost, s));
  TK(cudaMemcpyAsync(&hn, neg, 4, cudaMemcpyDeviceToHost, s));
  TK(cudaStreamSynchronize(s));
  h->n_wdangling = (int64_t)hc;
  h->neg_weights = hn ? 1 : 0;
  return PCPM_OK;
}

// Offsets, decode anchors, work lists and iteration state: the part of the
// build shared by both layout constructions.  G = flat (p, j) PNG group starts.
int finish_layout(pcpm_handle* h, Temp& tmp, PhaseTimer& pt, uint32_t* G, unsigned long long* d_dang) {
  cudaStream_t s = h->stream;
  const int64_t k_src = h->k_src, k_dst = h->k_dst, q = h->q, n_src = h->n_src, n_dst = h->n_dst, m = h->m;
  const int64_t ep = h->e_prime;
  const int64_t nchunks = h->m_pad / kChunkIds;
  int rc;
  // ---- offsets: png_off, column scans, bin update starts
  k_png_off<<<grid_for(k_src * (k_dst + 1)), kT, 0, s>>>(k_src, k_dst, G, h->png_off);
  uint32_t* col_tot;
  TK(tmp.alloc(&col_tot, k_dst + 1));
  col_scan(k_src, k_dst, G, h->upd_off, col_tot, s);
  TK(cudaMemsetAsync(col_tot + k_dst, 0, 4, s));
  if ((rc = scan_excl_u32(tmp, col_tot, h->bin_upd_start, k_dst + 1, s))) return rc;
  k_add_bin_start<<<grid_for(k_src * k_dst), kT, 0, s>>>(k_src, k_dst, h->bin_upd_start, h->upd_off);
  TK(cudaGetLastError());

  // ---- decode anchors: chunk_base[c] = #flags in ids[0 .. c*kChunkIds)
  {
    uint32_t* cnt;
    TK(tmp.alloc(&cnt, nchunks + 1));
    k_chunk_counts16<<<grid_for(nchunks * 32), kT, 0, s>>>(nchunks, h->ids16, cnt);
    TK(cudaGetLastError());
    if ((rc = scan_excl_u32(tmp, cnt, h->chunk_base, nchunks + 1, s))) return rc;
  }

  pt.mark("pull CSC + offsets + anchors");
  // ---- host-side work lists (small copies)
  // scatter items (p, [j0, j1)) holding ~E' / (2 SMs) updates each, counted on the device
  const int64_t target = std::max<int64_t>(8192, ep / (2 * h->num_sms) + 1);
  int tail_split = 4;                                   // PCPM_SCATTER_TAIL=1: no tail split (A/B)
  if (const char* e = getenv("PCPM_SCATTER_TAIL")) tail_split = std::max(1, atoi(e));
  const int64_t p_tail = std::max<int64_t>(0, k_src - h->num_sms);
  uint32_t *si_cnt, *si_off;
  TK(tmp.alloc(&si_cnt, k_src + 1));
  TK(tmp.alloc(&si_off, k_src + 1));
  TK(cudaMemsetAsync(si_cnt + k_src, 0, 4, s));
  k_sitems<<<grid_for(k_src * 32), kT, 0, s>>>(k_src, k_dst, G, target, kScatterMaxGroups, p_tail, tail_split, nullptr,
                                               si_cnt, nullptr);
  TK(cudaGetLastError());
  if ((rc = scan_excl_u32(tmp, si_cnt, si_off, k_src + 1, s))) return rc;
  std::vector<uint32_t> hbin(k_dst + 1);
  unsigned long long hdang = 0;
  uint32_t n_si = 0;
  TK(cudaMemcpyAsync(hbin.data(), h->bin_id_start, sizeof(uint32_t) * (k_dst + 1), cudaMemcpyDeviceToHost, s));
  TK(cudaMemcpyAsync(&hdang, d_dang, 8, cudaMemcpyDeviceToHost, s));
  TK(cudaMemcpyAsync(&n_si, si_off + k_src, 4, cudaMemcpyDeviceToHost, s));
  TK(cudaStreamSynchronize(s));
  h->n_dangling = (int64_t)hdang;
  h->n_sitems = (int)n_si;
  if ((rc = dev_alloc_t(h, &h->sitems, std::max<size_t>(n_si, 1)))) return rc;
  k_sitems<<<grid_for(k_src * 32), kT, 0, s>>>(k_src, k_dst, G, target, kScatterMaxGroups, p_tail, tail_split, si_off,
                                               nullptr,
                                               h->sitems);
  TK(cudaGetLastError());
  if (h->opt_scatter_lpt && (rc = order_scatter_items(h, s))) return rc;

  // gather items: every destination partition gets >= 1 item (its apply runs even
  // when the bin is empty); heavy bins are cut at tile-aligned points so no
  // item exceeds ~m / (2 SMs) IDs; largest first (LPT, the GPU analogue of the
  // paper's dynamic scheduling).
  std::vector<GatherItem> gi;
  // pair handles (q = 2^16): the gather sees 2 k_dst half-partitions of 2^15 vertices; half
  // hf of bin j is the "bin" j' = 2 j + hf: the same ID range, of which its items add only
  // that half's IDs.  Heavy bins are cut into slices per half like any other bin.
  const int64_t k_g = h->pair ? 2 * k_dst : k_dst;
  const int jsh = h->pair ? 1 : 0;
  const int64_t qa = int64_t(1) << h->gb;            // accumulator words = slot-buffer words per slice
  const int64_t m_str = h->pair ? 2 * m : m;         // IDs the gather streams
  std::vector<uint32_t> nsl(k_g, 0), sbase(k_g, 0);
  uint32_t nslots = 0;
  // items per SM the cut aims at: 2 when bin sizes are skewed (the LPT order then has
  // small slices to fill the tail), 1 when every bin is within 2x of the mean (cutting
  // finer only adds slot traffic); PCPM_GATHER_SLICE_DIV overrides (A/B)
  int64_t max_bin = 0;
  for (int64_t j = 0; j < k_dst; ++j) max_bin = std::max<int64_t>(max_bin, (int64_t)hbin[j + 1] - (int64_t)hbin[j]);
  int slice_div = (k_dst > 0 && max_bin * k_dst <= 2 * m) ? 1 : 2;
  if (const char* e = getenv("PCPM_GATHER_SLICE_DIV")) slice_div = std::max(1, atoi(e));
  int64_t slice = std::max<int64_t>(4 * kTileAlign, ((m_str / (slice_div * h->num_sms)) / kTileAlign + 1) * kTileAlign);
  for (int64_t j = 0; j < k_g; ++j) {
    if (h->pair && (j << h->gb) >= n_dst) continue;   // the last partition may have no upper half
    int64_t s0 = hbin[j >> jsh], s1 = hbin[(j >> jsh) + 1], sz = s1 - s0;
    int64_t nslc = sz > 0 ? (sz + slice - 1) / slice : 1;
    int64_t per = (sz + nslc - 1) / nslc;
    std::vector<int64_t> cuts{s0};
    for (int64_t i = 1; i < nslc; ++i) {
      int64_t c = ((s0 + i * per + kTileAlign - 1) / kTileAlign) * kTileAlign;
      if (c > cuts.back() && c < s1) cuts.push_back(c);
    }
    cuts.push_back(s1);
    const uint32_t ns = (uint32_t)(cuts.size() - 1);
    // slices of a split bin each own a slot: a q-word buffer for their low words
    sbase[j] = ns > 1 ? nslots : 0u;
    for (size_t i = 0; i + 1 < cuts.size(); ++i) {
      GatherItem it{};
      it.j = (uint32_t)j;
      it.x0 = (uint32_t)cuts[i];
      it.x1 = (uint32_t)cuts[i + 1];
      it.pad[0] = ns > 1 ? nslots + (uint32_t)i : 0xFFFFFFFFu;
      gi.push_back(it);
    }
    nsl[j] = ns;
    if (ns > 1) nslots += ns;
  }
  std::stable_sort(gi.begin(), gi.end(),
                   [](const GatherItem& a, const GatherItem& c) { return (a.x1 - a.x0) > (c.x1 - c.x0); });
  // cluster gather for few partitions: cs CTAs per bin (one tile-aligned slice each), cs = 2..8
  h->cl_cs = 0;
  if (!h->pair && k_dst >= 1 && 2 * k_dst <= h->num_sms && !getenv("PCPM_NO_CLUSTER_GATHER")) {
    int cs = 1, cs_max = 8;
    if (const char* e = getenv("PCPM_CLUSTER_MAX")) cs_max = std::max(2, std::min(8, atoi(e)));   // A/B
    while (cs * 2 <= cs_max && (int64_t)cs * 2 * k_dst <= h->num_sms) cs *= 2;
    std::vector<GatherItem> gc;
    for (int64_t j = 0; j < k_dst; ++j) {
      const int64_t s0 = hbin[j], s1 = hbin[j + 1], per = ((s1 - s0 + cs - 1) / cs + kTileAlign - 1) / kTileAlign * kTileAlign;
      for (int r = 0; r < cs; ++r) {
        GatherItem it{};
        it.j = (uint32_t)j;
        int64_t a0 = r == 0 ? s0 : std::min(s1, ((s0 + r * per) / kTileAlign) * kTileAlign);
        int64_t a1 = r == cs - 1 ? s1 : std::min(s1, ((s0 + (r + 1) * per) / kTileAlign) * kTileAlign);
        a0 = std::max(a0, s0);
        a1 = std::max(a1, a0);
        it.x0 = (uint32_t)a0;
        it.x1 = (uint32_t)a1;
        it.pad[0] = 0xFFFFFFFFu;
        gc.push_back(it);
      }
    }
    if ((rc = dev_alloc_t(h, &h->gitems_cl, gc.size()))) return rc;
    TK(cudaMemcpyAsync(h->gitems_cl, gc.data(), sizeof(GatherItem) * gc.size(), cudaMemcpyHostToDevice, s));
    h->cl_cs = cs;
  }
  h->n_gitems = (int)gi.size();
  if ((rc = dev_alloc_t(h, &h->gitems, gi.size()))) return rc;
  if ((rc = dev_alloc_t(h, &h->bin_nslices, k_g))) return rc;
  TK(cudaMemcpyAsync(h->gitems, gi.data(), sizeof(GatherItem) * gi.size(), cudaMemcpyHostToDevice, s));
  TK(cudaMemcpyAsync(h->bin_nslices, nsl.data(), sizeof(uint32_t) * k_g, cudaMemcpyHostToDevice, s));
  if ((rc = dev_alloc_t(h, &h->bin_slot_base, k_g))) return rc;
  TK(cudaMemcpyAsync(h->bin_slot_base, sbase.data(), sizeof(uint32_t) * k_g, cudaMemcpyHostToDevice, s));
  h->n_slots = nslots;
  {
    std::vector<uint32_t> sb;
    for (int64_t j = 0; j < k_g; ++j)
      if (nsl[j] > 1) sb.push_back((uint32_t)j);
    h->n_split_bins = (int)sb.size();
    if ((rc = dev_alloc_t(h, &h->split_bins, std::max<size_t>(1, sb.size())))) return rc;
    if (!sb.empty())
      TK(cudaMemcpyAsync(h->split_bins, sb.data(), sizeof(uint32_t) * sb.size(), cudaMemcpyHostToDevice, s));
    // the fused iteration scatters a split partition after k_apply_split: its scatter items
    h->n_sitems_split = 0;
    if (!sb.empty() && k_src == k_dst && h->n_sitems > 0 && !h->pair) {
      std::vector<ScatterItem> si(h->n_sitems), ss;
      TK(cudaMemcpyAsync(si.data(), h->sitems, sizeof(ScatterItem) * si.size(), cudaMemcpyDeviceToHost, s));
      TK(cudaStreamSynchronize(s));
      for (const ScatterItem& it : si)
        if (it.p < (uint32_t)k_dst && nsl[it.p] > 1) ss.push_back(it);
      if (!ss.empty()) {
        if ((rc = dev_alloc_t(h, &h->sitems_split, ss.size()))) return rc;
        TK(cudaMemcpyAsync(h->sitems_split, ss.data(), sizeof(ScatterItem) * ss.size(), cudaMemcpyHostToDevice, s));
        h->n_sitems_split = (int)ss.size();
      }
    }
  }
  if ((rc = dev_alloc_t(h, &h->slot_buf, std::max<size_t>(1, (size_t)nslots * qa)))) return rc;
  k_item_f<<<grid_for(h->n_gitems), kT, 0, s>>>(h->n_gitems, h->gitems, h->chunk_base, h->bin_upd_start,
                                                h->pair ? 1 : 0);
  TK(cudaGetLastError());
  if (h->cl_cs) {
    const int nc = (int)(k_dst * h->cl_cs);
    k_item_f<<<grid_for(nc), kT, 0, s>>>(nc, h->gitems_cl, h->chunk_base, h->bin_upd_start);
    TK(cudaGetLastError());
  }

  // ---- iteration scratch (kept zero between uses by the kernels)
  const int64_t nv = std::max(n_src, n_dst);
  if ((rc = dev_alloc_t(h, &h->pr[0], nv + 8))) return rc;
  if ((rc = dev_alloc_t(h, &h->pr[1], nv + 8))) return rc;
  if ((rc = dev_alloc_t(h, &h->spr, n_src + 8))) return rc;
  if ((rc = dev_alloc_t(h, &h->xbuf, n_src + 8))) return rc;
  if ((rc = dev_alloc_t(h, &h->ybuf, n_dst + 8))) return rc;
  if ((rc = dev_alloc_t(h, &h->hi, n_dst))) return rc;
  if ((rc = dev_alloc_t(h, &h->counters, 8))) return rc;
  if ((rc = dev_alloc_t(h, &h->bin_arrive, k_g))) return rc;
  TK(cudaMemsetAsync(h->bin_arrive, 0, sizeof(uint32_t) * k_g, s));
  if ((rc = dev_alloc_t(h, &h->xmax, 4))) return rc;
  if ((rc = dev_alloc_t(h, &h->red_fx, 2))) return rc;
  TK(cudaMemsetAsync(h->red_fx, 0, sizeof(unsigned long long) * 2, s));
  TK(cudaMemsetAsync(h->hi, 0, sizeof(uint32_t) * n_dst, s));
  TK(cudaMemsetAsync(h->counters, 0, sizeof(uint32_t) * 8, s));
  TK(cudaMemsetAsync(h->spr, 0, sizeof(float) * (n_src + 8), s));
  TK(cudaMemsetAsync(h->xbuf, 0, sizeof(float) * (n_src + 8), s));
  TK(cudaStreamSynchronize(s));
  pt.mark("work lists + iteration state");
  // ---- PCPM_COMPACT_SLOTS: accumulator slots (unweighted, unsplit, compact, non-shard layouts)
  if (h->want_slots && !h->wide && !h->w && !h->shard && h->n_split_bins == 0 && k_dst > 0 && q >= 64) {
    uint32_t *has_in, *scan;
    TK(tmp.alloc(&has_in, k_dst * q + 1));
    TK(tmp.alloc(&scan, k_dst * q + 1));
    TK(cudaMemsetAsync(has_in, 0, sizeof(uint32_t) * (k_dst * q + 1), s));
    k_mark_in<<<(unsigned)k_dst, 256, 0, s>>>(h->bin_id_start, h->ids16, h->b, has_in);
    TK(cudaGetLastError());
    size_t bytes = 0;
    TK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, has_in, scan, k_dst * q + 1, s));
    uint8_t* t;
    TK(tmp.alloc(&t, bytes));
    TK(cub::DeviceScan::ExclusiveSum(t, bytes, has_in, scan, k_dst * q + 1, s));
    std::vector<uint32_t> pc(k_dst + 1);
    TK(cudaMemcpy2DAsync(pc.data(), sizeof(uint32_t), scan, sizeof(uint32_t) * q, sizeof(uint32_t), k_dst + 1,
                         cudaMemcpyDeviceToHost, s));
    TK(cudaStreamSynchronize(s));
    uint32_t mx = 0;
    for (int64_t j = 0; j < k_dst; ++j) mx = std::max(mx, pc[j + 1] - pc[j]);
    const int words = (int)(((mx + 31) / 32) * 32);
    if (words < q && gather_slots_fit(h->b, words)) {
      const int64_t nd = k_dst * q;
      if ((rc = dev_alloc_t(h, &h->slot16, nd))) return rc;
      k_slots<<<grid_for(nd), kT, 0, s>>>(nd, h->b, has_in, scan, h->slot16);
      k_remap_ids<<<(unsigned)k_dst, 256, 0, s>>>(h->bin_id_start, h->b, h->slot16, h->ids16);
      if ((rc = dev_alloc_t(h, &h->slotmap, nd / 32))) return rc;
      k_slotmap<<<grid_for(nd / 32), kT, 0, s>>>(nd / 32, has_in, scan, h->b, h->slotmap);
      TK(cudaGetLastError());
      h->acc_words = words;
      TK(cudaStreamSynchronize(s));
    }
    pt.mark("accumulator slots");
  }
  return PCPM_OK;
}

}  // namespace

int build_layout_legacy(pcpm_handle* h, const pcpm_csr* csr, unsigned flags) {
  cudaStream_t s = h->stream;
  const int64_t n_src = csr->n_src, n_dst = csr->n_dst, m = csr->nnz;
  const int b = h->b;
  const int64_t q = int64_t(1) << b;
  const int64_t k_src = (n_src + q - 1) / q, k_dst = (n_dst + q - 1) / q;
  h->k_src = k_src;
  h->k_dst = k_dst;
  h->q = q;
  h->n_src = n_src;
  h->n_dst = n_dst;
  h->m = m;
  h->compressed = !(flags & PCPM_NO_COMPRESS);
  h->weighted = csr->values != nullptr || (flags & PCPM_KEEP_VALUES);
  h->wide = (flags & PCPM_WIDE_IDS) != 0;
  h->want_slots = (flags & PCPM_COMPACT_SLOTS) != 0;
  h->m_pad = ((m + kTileAlign - 1) / kTileAlign) * kTileAlign;
  if (h->m_pad == 0) h->m_pad = kTileAlign;

  Temp tmp(s);
  PhaseTimer pt(s);
  // ---- inputs on the device
  const int64_t* row_ptr = csr->row_ptr;
  const uint32_t* col = csr->col_idx;
  const float* values = csr->values;
  if (!is_device_ptr(row_ptr)) {
    int64_t* d;
    TK(tmp.alloc(&d, n_src + 1));
    TK(cudaMemcpyAsync(d, row_ptr, sizeof(int64_t) * (n_src + 1), cudaMemcpyHostToDevice, s));
    row_ptr = d;
  }
  if (m > 0 && !is_device_ptr(col)) {
    uint32_t* d;
    TK(tmp.alloc(&d, m));
    TK(cudaMemcpyAsync(d, col, sizeof(uint32_t) * m, cudaMemcpyHostToDevice, s));
    col = d;
  }
  if (m > 0 && values && !is_device_ptr(values)) {
    float* d;
    TK(tmp.alloc(&d, m));
    TK(cudaMemcpyAsync(d, values, sizeof(float) * m, cudaMemcpyHostToDevice, s));
    values = d;
  }

  uint32_t* err;
  TK(tmp.alloc(&err, 4));
  TK(cudaMemsetAsync(err, 0, 16, s));
  k_check_rows<<<grid_for(n_src), kT, 0, s>>>(n_src, row_ptr, m, err);
  TK(cudaGetLastError());
  uint32_t herr[4] = {0, 0, 0, 0};
  TK(cudaMemcpyAsync(herr, err, 16, cudaMemcpyDeviceToHost, s));
  TK(cudaStreamSynchronize(s));
  if (herr[0]) {
    set_error(PCPM_EBADCSR, "row_ptr is not monotone, or row_ptr[0] != 0, or row_ptr[n_src] != nnz");
    return PCPM_EBADCSR;
  }

  pt.mark("inputs + row validation");
  // ---- layout arrays owned by the handle
  int rc;
  uint32_t* ids32 = nullptr;           // 4-byte IDs: handle-owned for wide handles, else scratch
  if (h->wide) {
    if ((rc = dev_alloc_t(h, &h->ids, h->m_pad))) return rc;
    ids32 = h->ids;
  } else {
    TK(tmp.alloc(&ids32, h->m_pad));
  }
  if ((rc = dev_alloc_t(h, &h->ids16, h->m_pad))) return rc;
  TK(cudaMemsetAsync(h->ids16, 0, sizeof(uint16_t) * h->m_pad, s));
  if (h->weighted && (rc = dev_alloc_t(h, &h->w, h->m_pad))) return rc;
  if ((rc = dev_alloc_t(h, &h->png_off, k_src * (k_dst + 1) + 4))) return rc;
  if ((rc = dev_alloc_t(h, &h->upd_off, k_src * k_dst + 4))) return rc;
  if ((rc = dev_alloc_t(h, &h->bin_id_start, k_dst + 1))) return rc;
  if ((rc = dev_alloc_t(h, &h->bin_upd_start, k_dst + 1))) return rc;
  const int64_t nchunks = h->m_pad / kChunkIds;
  if ((rc = dev_alloc_t(h, &h->chunk_base, nchunks + 1))) return rc;
  if ((rc = dev_alloc_t(h, &h->outdeg, n_src))) return rc;
  if ((rc = dev_alloc_t(h, &h->inv_deg, n_src + 4))) return rc;
  TK(cudaMemsetAsync(ids32, 0, sizeof(uint32_t) * h->m_pad, s));
  if (h->w) TK(cudaMemsetAsync(h->w, 0, sizeof(float) * h->m_pad, s));

  // ---- out-degrees and dangling count
  unsigned long long* d_dang;
  TK(tmp.alloc(&d_dang, 1));
  TK(cudaMemsetAsync(d_dang, 0, 8, s));
  k_outdeg<<<grid_for(n_src), kT, 0, s>>>(0, n_src, row_ptr, h->outdeg, h->inv_deg, d_dang);
  TK(cudaGetLastError());

  pt.mark("allocations + outdeg");
  uint32_t* G = nullptr;  // flat (p, j) group starts, k_src*k_dst + 1 entries
  TK(tmp.alloc(&G, k_src * k_dst + 1));
  int64_t ep = 0;
  if (m > 0) {
    // ---- row id of every edge: mark row starts, inclusive max-scan
    uint32_t *rowmark, *rowid;
    TK(tmp.alloc(&rowmark, m));
    TK(tmp.alloc(&rowid, m));
    TK(cudaMemsetAsync(rowmark, 0, sizeof(uint32_t) * m, s));
    k_mark_rows<<<grid_for(n_src), kT, 0, s>>>(n_src, row_ptr, rowmark);
    TK(cudaGetLastError());
    {
      size_t bytes = 0;
      TK(cub::DeviceScan::InclusiveScan(nullptr, bytes, rowmark, rowid, MaxOp(), m, s));
      uint8_t* t;
      TK(tmp.alloc(&t, bytes));
      TK(cub::DeviceScan::InclusiveScan(t, bytes, rowmark, rowid, MaxOp(), m, s));
    }
    pt.mark("row ids");
    // ---- classify + validate
    uint32_t *keyj, *enc;
    uint8_t* fl;
    TK(tmp.alloc(&keyj, m));
    TK(tmp.alloc(&enc, m));
    TK(tmp.alloc(&fl, m));
    k_classify<<<grid_for(m), kT, 0, s>>>(m, col, rowid, b, n_dst, h->compressed, keyj, enc, fl, err);
    TK(cudaGetLastError());
    TK(cudaMemcpyAsync(herr, err, 16, cudaMemcpyDeviceToHost, s));
    TK(cudaStreamSynchronize(s));
    if (herr[0] & 2u) {
      set_error(PCPM_EBADCSR, "col_idx has an entry >= n_dst");
      return PCPM_EBADCSR;
    }
    if (herr[0] & 4u) {
      set_error(PCPM_EBADCSR, "a row's columns are not strictly increasing (sorted, deduplicated) (R6)");
      return PCPM_EBADCSR;
    }
    pt.mark("classify + validate");
    // ---- destID bins: stable sort of edge indices by j
    uint32_t *iota, *keyj_s, *perm;
    TK(tmp.alloc(&iota, m));
    TK(tmp.alloc(&keyj_s, m));
    TK(tmp.alloc(&perm, m));
    k_iota<<<grid_for(m), kT, 0, s>>>(m, iota);
    TK(cudaGetLastError());
    const int jbits = bits_for((uint64_t)std::max<int64_t>(k_dst - 1, 0));
    if (h->w) {
      // weights travel with the IDs: sort edge indices, then gather IDs and weights
      TK(radix_sort_pairs(tmp, keyj, keyj_s, iota, perm, m, jbits, s));
      pt.mark("sort edges by j");
      k_gather_ids<<<grid_for(m), kT, 0, s>>>(m, perm, enc, values, (uint32_t)(q - 1) & 0x7FFFu, ids32, h->ids16, h->w);
    } else {
      // the encoded IDs are the sort's payload: no random gather afterwards
      TK(radix_sort_pairs(tmp, keyj, keyj_s, enc, ids32, m, jbits, s));
      pt.mark("sort edges by j");
      k_ids16<<<grid_for(m), kT, 0, s>>>(m, ids32, (uint32_t)(q - 1) & 0x7FFFu, h->ids16);
    }
    TK(cudaGetLastError());
    k_boundaries<<<grid_for(m + 1), kT, 0, s>>>(m, keyj_s, k_dst, h->bin_id_start);
    TK(cudaGetLastError());

    pt.mark("destID bins");
    // ---- PNG: flagged edges, stable sort by (p, j)
    uint32_t* sel;
    int64_t* d_nsel;
    TK(tmp.alloc(&sel, m));
    TK(tmp.alloc(&d_nsel, 1));
    {
      size_t bytes = 0;
      TK(cub::DeviceSelect::Flagged(nullptr, bytes, iota, fl, sel, d_nsel, m, s));
      uint8_t* t;
      TK(tmp.alloc(&t, bytes));
      TK(cub::DeviceSelect::Flagged(t, bytes, iota, fl, sel, d_nsel, m, s));
    }
    TK(cudaMemcpyAsync(&ep, d_nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    TK(cudaStreamSynchronize(s));
    h->e_prime = ep;
    uint32_t* png32 = nullptr;
    if (h->wide) {
      if ((rc = dev_alloc_t(h, &h->png_src, ep + 8))) return rc;
      png32 = h->png_src;
    } else {
      TK(tmp.alloc(&png32, ep + 8));
    }
    if ((rc = dev_alloc_t(h, &h->png16, ep + 16))) return rc;
    if ((rc = dev_alloc_t(h, &h->upd, ep + 8))) return rc;
    TK(cudaMemsetAsync(h->upd + ep, 0, sizeof(float) * 8, s));   // the scatter writes [0, E') before any read
    TK(cudaMemsetAsync(h->png16, 0, sizeof(uint16_t) * (ep + 16), s));
    uint32_t *pk, *pv, *pk_s;
    TK(tmp.alloc(&pk, ep));
    TK(tmp.alloc(&pv, ep));
    TK(tmp.alloc(&pk_s, ep));
    k_png_keys<<<grid_for(ep), kT, 0, s>>>(ep, sel, rowid, col, b, k_dst, pk, pv);
    TK(cudaGetLastError());
    TK(radix_sort_pairs(tmp, pk, pk_s, pv, png32, ep, bits_for((uint64_t)(k_src * k_dst - 1)), s));
    pt.mark("select + sort PNG");
    k_boundaries<<<grid_for(ep + 1), kT, 0, s>>>(ep, pk_s, k_src * k_dst, G);
    k_png16<<<grid_for(ep), kT, 0, s>>>(ep, png32, (uint32_t)(q - 1), h->png16);
    TK(cudaGetLastError());
    {
      const int64_t nga = ep / kPngChunk + 64;     // the scatter copies aligned supersets
      if ((rc = dev_alloc_t(h, &h->grp_at, nga))) return rc;
      k_grp_at<<<grid_for(nga), kT, 0, s>>>(ep, pk_s, nga, h->grp_at);
      TK(cudaGetLastError());
    }

    pt.mark("PNG arrays");
    // ---- pull comparison: CSC (in-adjacency), sources ascending per destination
    if (flags & PCPM_BUILD_PULL) {
      if ((rc = dev_alloc_t(h, &h->in_ptr, n_dst + 1))) return rc;
      if ((rc = dev_alloc_t(h, &h->in_src, m))) return rc;
      uint32_t *ck, *ck_s, *cperm;
      TK(tmp.alloc(&ck, m));
      TK(tmp.alloc(&ck_s, m));
      TK(tmp.alloc(&cperm, m));
      TK(cudaMemcpyAsync(ck, col, sizeof(uint32_t) * m, cudaMemcpyDeviceToDevice, s));
      TK(radix_sort_pairs(tmp, ck, ck_s, iota, cperm, m, bits_for((uint64_t)std::max<int64_t>(n_dst - 1, 0)), s));
      k_boundaries<<<grid_for(m + 1), kT, 0, s>>>(m, ck_s, n_dst, h->in_ptr);
      TK(cudaGetLastError());
      k_gather_u32<<<grid_for(m), kT, 0, s>>>(m, cperm, rowid, h->in_src);
      TK(cudaGetLastError());
      h->has_pull = true;
    }
    // ---- max|w| (fixed-point range of the signed SpMV accumulator)
    if (values) {
      float* mx;
      TK(tmp.alloc(&mx, 1));
      float hmx = 0.f;
      int rc2 = launch_absmax(h, values, m, mx, s);
      if (rc2) return rc2;
      TK(cudaMemcpyAsync(&hmx, mx, 4, cudaMemcpyDeviceToHost, s));
      TK(cudaStreamSynchronize(s));
      int ex = 0;
      if (hmx > 0.f) frexpf(hmx, &ex);
      h->wexp = ex;
      if ((rc2 = weighted_degrees(h, tmp, row_ptr, values))) return rc2;
    }
  } else {
    h->e_prime = 0;
    if (h->wide && (rc = dev_alloc_t(h, &h->png_src, 8))) return rc;
    if ((rc = dev_alloc_t(h, &h->png16, 16))) return rc;
    if ((rc = dev_alloc_t(h, &h->grp_at, 64))) return rc;
    TK(cudaMemsetAsync(h->grp_at, 0, 256, s));
    if ((rc = dev_alloc_t(h, &h->upd, 8))) return rc;
    TK(cudaMemsetAsync(h->upd, 0, 32, s));
    TK(cudaMemsetAsync(G, 0, sizeof(uint32_t) * (k_src * k_dst + 1), s));
    TK(cudaMemsetAsync(h->bin_id_start, 0, sizeof(uint32_t) * (k_dst + 1), s));
    if (flags & PCPM_BUILD_PULL) {
      if ((rc = dev_alloc_t(h, &h->in_ptr, n_dst + 1))) return rc;
      if ((rc = dev_alloc_t(h, &h->in_src, 1))) return rc;
      TK(cudaMemsetAsync(h->in_ptr, 0, sizeof(uint32_t) * (n_dst + 1), s));
      h->has_pull = true;
    }
  }

  return finish_layout(h, tmp, pt, G, d_dang);
}

namespace {

template <typename P>
int build_layout_chunked(pcpm_handle* h, const pcpm_csr* csr, unsigned flags) {
  cudaStream_t s = h->stream;
  const int64_t n_src = csr->n_src, n_dst = csr->n_dst, m = csr->nnz;
  const int b = h->b;
  const int64_t q = int64_t(1) << b;
  const int64_t k_src = (n_src + q - 1) / q, k_dst = (n_dst + q - 1) / q;
  h->k_src = k_src;
  h->k_dst = k_dst;
  h->q = q;
  h->n_src = n_src;
  h->n_dst = n_dst;
  h->m = m;
  h->compressed = !(flags & PCPM_NO_COMPRESS);
  h->weighted = csr->values != nullptr || (flags & PCPM_KEEP_VALUES);
  h->wide = (flags & PCPM_WIDE_IDS) != 0;
  h->want_slots = (flags & PCPM_COMPACT_SLOTS) != 0;
  h->m_pad = ((m + kTileAlign - 1) / kTileAlign) * kTileAlign;
  if (h->m_pad == 0) h->m_pad = kTileAlign;
  const int64_t ng = k_src * k_dst;             // groups (p, j)
  const int gbits = bits_for((uint64_t)(ng - 1));

  Temp tmp(s);
  PhaseTimer pt(s);
  const int64_t* row_ptr = csr->row_ptr;
  const uint32_t* col = csr->col_idx;
  const float* values = csr->values;
  const bool host_rp = !is_device_ptr(row_ptr);
  const bool host_col = !is_device_ptr(col);
  const bool host_val = values && !is_device_ptr(values);
  const bool copies = host_rp || host_col || host_val;

  // ---- partition boundaries of row_ptr (host): global checks and the chunk plan
  std::vector<int64_t> pb(k_src + 1);
  if (host_rp) {
    for (int64_t p = 0; p < k_src; ++p) pb[p] = row_ptr[p * q];
    pb[k_src] = row_ptr[n_src];
  } else {
    TK(cudaMemcpy2DAsync(pb.data(), sizeof(int64_t), row_ptr, sizeof(int64_t) * q, sizeof(int64_t), k_src,
                         cudaMemcpyDeviceToHost, s));
    TK(cudaMemcpyAsync(&pb[k_src], row_ptr + n_src, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    TK(cudaStreamSynchronize(s));
  }
  bool rp_ok = pb[0] == 0 && pb[k_src] == m;
  for (int64_t p = 0; p < k_src && rp_ok; ++p) rp_ok = pb[p] <= pb[p + 1];
  if (!rp_ok) {
    set_error(PCPM_EBADCSR, "row_ptr is not monotone, or row_ptr[0] != 0, or row_ptr[n_src] != nnz");
    return PCPM_EBADCSR;
  }
  int64_t target = copies ? std::max<int64_t>(m / 24, int64_t(1) << 22) : std::max<int64_t>(m / 4, int64_t(1) << 24);
  if (const char* e = getenv("PCPM_BUILD_CHUNK_EDGES")) target = std::max<int64_t>(1, atoll(e));   // tests: many chunks
  std::vector<int64_t> cp{0};
  for (int64_t p = 0; p < k_src; ++p)
    if (pb[p + 1] - pb[cp.back()] >= target || p + 1 == k_src) cp.push_back(p + 1);
  const int nck = (int)cp.size() - 1;
  int64_t mc_max = 1;
  for (int c = 0; c < nck; ++c) mc_max = std::max(mc_max, pb[cp[c + 1]] - pb[cp[c]]);

  // ---- device copies of host inputs (filled chunk by chunk on a copy stream)
  int64_t* d_rp = const_cast<int64_t*>(row_ptr);
  uint32_t* d_col = const_cast<uint32_t*>(col);
  float* d_val = const_cast<float*>(values);
  if (host_rp) TK(tmp.alloc(&d_rp, n_src + 1));
  if (host_col) TK(tmp.alloc(&d_col, m));
  if (host_val) TK(tmp.alloc(&d_val, m));

  // ---- layout arrays owned by the handle
  int rc;
  uint32_t* ids32 = nullptr;
  if (h->wide) {
    if ((rc = dev_alloc_t(h, &h->ids, h->m_pad))) return rc;
    ids32 = h->ids;
    TK(cudaMemsetAsync(ids32, 0, sizeof(uint32_t) * h->m_pad, s));
  }
  if ((rc = dev_alloc_t(h, &h->ids16, h->m_pad))) return rc;
  TK(cudaMemsetAsync(h->ids16 + m, 0, sizeof(uint16_t) * (h->m_pad - m), s));
  if (h->weighted) {
    if ((rc = dev_alloc_t(h, &h->w, h->m_pad))) return rc;
    TK(cudaMemsetAsync(h->w + m, 0, sizeof(float) * (h->m_pad - m), s));
  }
  if ((rc = dev_alloc_t(h, &h->png_off, k_src * (k_dst + 1) + 4))) return rc;
  if ((rc = dev_alloc_t(h, &h->upd_off, ng + 4))) return rc;
  if ((rc = dev_alloc_t(h, &h->bin_id_start, k_dst + 1))) return rc;
  if ((rc = dev_alloc_t(h, &h->bin_upd_start, k_dst + 1))) return rc;
  if ((rc = dev_alloc_t(h, &h->chunk_base, h->m_pad / kChunkIds + 1))) return rc;
  if ((rc = dev_alloc_t(h, &h->outdeg, n_src))) return rc;
  if ((rc = dev_alloc_t(h, &h->inv_deg, n_src + 4))) return rc;

  // ---- scratch: sorted edges (keys, payloads) and their flagged subsets, per-chunk buffers
  uint32_t *err, *keys_s, *fk, *mark, *rowid, *key_c;
  P *pay_s, *fp, *pay_c;
  uint8_t* fl_c;
  int64_t* d_cnt;
  unsigned long long* d_dang;
  const bool pull = (flags & PCPM_BUILD_PULL) != 0;
  TK(tmp.alloc(&err, 4));
  TK(tmp.alloc(&d_dang, 1));
  TK(tmp.alloc(&d_cnt, 2 * nck + 2));
  TK(tmp.alloc(&keys_s, m));
  TK(tmp.alloc(&pay_s, m));
  TK(tmp.alloc(&fk, m));
  TK(tmp.alloc(&fp, m));
  TK(tmp.alloc(&mark, mc_max));
  TK(tmp.alloc(&rowid, pull ? m : mc_max));
  TK(tmp.alloc(&key_c, mc_max));
  TK(tmp.alloc(&pay_c, mc_max));
  TK(tmp.alloc(&fl_c, mc_max));
  // group starts in sorted-edge order (Gs) and in the PNG (G), PNG arrays at their
  // final positions (exact-size copies at the end), filled chunk by chunk
  uint32_t *Gs, *G, *pk, *png32_t = nullptr;
  uint16_t* png16_t;
  int64_t* d_off;
  TK(tmp.alloc(&Gs, ng + 1));
  TK(tmp.alloc(&G, ng + 1));
  TK(tmp.alloc(&pk, m));
  TK(tmp.alloc(&png16_t, m));
  if (h->wide) TK(tmp.alloc(&png32_t, m));
  TK(tmp.alloc(&d_off, nck + 1));
  TK(cudaMemsetAsync(d_off, 0, sizeof(int64_t) * (nck + 1), s));
  TK(cudaMemsetAsync(err, 0, 16, s));
  TK(cudaMemsetAsync(d_dang, 0, 8, s));
  TK(cudaMemsetAsync(d_cnt, 0, sizeof(int64_t) * (2 * nck + 2), s));
  // CUB scratch, sized once for the largest chunk
  size_t b_scan = 0, b_sort = 0, b_sel = 0, b_sel2 = 0;
  TK(cub::DeviceScan::InclusiveScan(nullptr, b_scan, mark, rowid, MaxOp(), mc_max, s));
  TK(cub::DeviceRadixSort::SortPairs(nullptr, b_sort, key_c, keys_s, pay_c, pay_s, mc_max, 0, gbits, s));
  TK(cub::DeviceSelect::Flagged(nullptr, b_sel, keys_s, fl_c, fk, d_cnt, mc_max, s));
  TK(cub::DeviceSelect::Flagged(nullptr, b_sel2, pay_s, fl_c, fp, d_cnt, mc_max, s));
  uint8_t* cub_tmp;
  const size_t b_cub = std::max(std::max(b_scan, b_sort), std::max(b_sel, b_sel2));
  TK(tmp.alloc(&cub_tmp, b_cub));

  cudaStream_t cs = nullptr;
  std::vector<cudaEvent_t> evs;
  struct Cleanup {
    cudaStream_t& cs;
    std::vector<cudaEvent_t>& evs;
    ~Cleanup() {
      if (cs) cudaStreamSynchronize(cs);          // no copy may outlive the scratch it writes
      for (cudaEvent_t e : evs) cudaEventDestroy(e);
      if (cs) cudaStreamDestroy(cs);
    }
  } cleanup{cs, evs};
  if (copies) {
    TK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    evs.resize(nck + 1);
    for (auto& e : evs) TK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    TK(cudaEventRecord(evs[nck], s));               // the pool allocations above precede the copies
    TK(cudaStreamWaitEvent(cs, evs[nck], 0));
  }
  pt.mark("plan + allocations");

  // ---- per chunk: copy in, validate, out-degrees, row ids, classify, sort, select the PNG
  for (int c = 0; c < nck; ++c) {
    const int64_t p0 = cp[c], p1 = cp[c + 1];
    const int64_t u0 = p0 * q, u1 = std::min(p1 * q, n_src), nr = u1 - u0;
    const int64_t e0 = pb[p0], e1 = pb[p1], mc = e1 - e0;
    if (copies) {
      if (host_rp)
        TK(cudaMemcpyAsync(d_rp + u0, row_ptr + u0, sizeof(int64_t) * (nr + 1), cudaMemcpyHostToDevice, cs));
      if (host_col && mc)
        TK(cudaMemcpyAsync(d_col + e0, col + e0, sizeof(uint32_t) * mc, cudaMemcpyHostToDevice, cs));
      if (host_val && mc)
        TK(cudaMemcpyAsync(d_val + e0, values + e0, sizeof(float) * mc, cudaMemcpyHostToDevice, cs));
      TK(cudaEventRecord(evs[c], cs));
      TK(cudaStreamWaitEvent(s, evs[c], 0));
    }
    k_check_rows_c<<<grid_for(nr), kT, 0, s>>>(u0, nr, d_rp, e0, e1, err);
    k_outdeg<<<grid_for(nr), kT, 0, s>>>(u0, nr, d_rp, h->outdeg, h->inv_deg, d_dang);
    TK(cudaGetLastError());
    const int64_t g0 = p0 * k_dst, g1 = p1 * k_dst;
    if (mc == 0) {
      k_bounds_range<<<1, kT, 0, s>>>(0, nullptr, keys_s, g0, g1, e0, nullptr, Gs);
      k_png_place_c<P><<<1, kT, 0, s>>>(d_cnt + c, d_off + c, d_off + c + 1, fk, fp, b, k_dst, pk, png16_t, png32_t);
      k_bounds_range<<<1, kT, 0, s>>>(0, d_cnt + c, fk, g0, g1, 0, d_off + c, G);
      TK(cudaGetLastError());
      continue;
    }
    uint32_t* rid = pull ? rowid + e0 : rowid;
    TK(cudaMemsetAsync(mark, 0, sizeof(uint32_t) * mc, s));
    k_mark_rows_c<<<grid_for(nr), kT, 0, s>>>(u0, nr, d_rp, e0, e1, mark);
    TK(cudaGetLastError());
    size_t bt = b_cub;
    TK(cub::DeviceScan::InclusiveScan(cub_tmp, bt, mark, rid, MaxOp(), mc, s));
    k_classify_c<P><<<grid_for(mc), kT, 0, s>>>(e0, mc, d_col, d_val, rid, b, n_dst, k_dst, h->compressed, key_c,
                                                 pay_c, err);
    TK(cudaGetLastError());
    bt = b_cub;
    TK(cub::DeviceRadixSort::SortPairs(cub_tmp, bt, key_c, keys_s + e0, pay_c, pay_s + e0, mc, 0, gbits, s));
    k_run_flags<P><<<grid_for(mc), kT, 0, s>>>(mc, pay_s + e0, fl_c);
    TK(cudaGetLastError());
    bt = b_cub;
    TK(cub::DeviceSelect::Flagged(cub_tmp, bt, keys_s + e0, fl_c, fk + e0, d_cnt + c, mc, s));
    bt = b_cub;
    TK(cub::DeviceSelect::Flagged(cub_tmp, bt, pay_s + e0, fl_c, fp + e0, d_cnt + nck + c, mc, s));
    // this chunk's groups: starts among the sorted edges and in the PNG
    k_bounds_range<<<grid_for(mc + 1), kT, 0, s>>>(mc, nullptr, keys_s + e0, g0, g1, e0, nullptr, Gs);
    k_png_place_c<P><<<grid_for(mc), kT, 0, s>>>(d_cnt + c, d_off + c, d_off + c + 1, fk + e0, fp + e0, b, k_dst,
                                                 pk, png16_t, png32_t);
    k_bounds_range<<<grid_for(mc + 1), kT, 0, s>>>(mc, d_cnt + c, fk + e0, g0, g1, 0, d_off + c, G);
    TK(cudaGetLastError());
  }
  std::vector<int64_t> hcnt(nck);
  uint32_t herr[4] = {0, 0, 0, 0};
  if (nck) TK(cudaMemcpyAsync(hcnt.data(), d_cnt, sizeof(int64_t) * nck, cudaMemcpyDeviceToHost, s));
  TK(cudaMemcpyAsync(herr, err, 16, cudaMemcpyDeviceToHost, s));
  TK(cudaStreamSynchronize(s));
  if (herr[0] & 1u) {
    set_error(PCPM_EBADCSR, "row_ptr is not monotone, or row_ptr[0] != 0, or row_ptr[n_src] != nnz");
    return PCPM_EBADCSR;
  }
  if (herr[0] & 2u) {
    set_error(PCPM_EBADCSR, "col_idx has an entry >= n_dst");
    return PCPM_EBADCSR;
  }
  if (herr[0] & 4u) {
    set_error(PCPM_EBADCSR, "a row's columns are not strictly increasing (sorted, deduplicated) (R6)");
    return PCPM_EBADCSR;
  }
  int64_t ep = 0;
  for (int c = 0; c < nck; ++c) ep += hcnt[c];
  h->e_prime = ep;
  pt.mark("chunks: copy + sort");

  // ---- destID bins: group starts in sorted order, column scans, placement
  uint32_t *id_off, *col_tot;
  TK(tmp.alloc(&id_off, ng));
  TK(tmp.alloc(&col_tot, k_dst + 1));
  col_scan(k_src, k_dst, Gs, id_off, col_tot, s);
  TK(cudaGetLastError());
  TK(cudaMemsetAsync(col_tot + k_dst, 0, 4, s));
  {
    size_t bytes = 0;
    TK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, col_tot, h->bin_id_start, k_dst + 1, s));
    uint8_t* t;
    TK(tmp.alloc(&t, bytes));
    TK(cub::DeviceScan::ExclusiveSum(t, bytes, col_tot, h->bin_id_start, k_dst + 1, s));
  }
  k_add_bin_start<<<grid_for(ng), kT, 0, s>>>(k_src, k_dst, h->bin_id_start, id_off);
  k_place_ids<P><<<grid_for(m), kT, 0, s>>>(m, keys_s, pay_s, Gs, id_off, b, k_dst, h->ids16, ids32, h->w);
  TK(cudaGetLastError());
  pt.mark("destID bins");

  // ---- PNG: exact-size copies of the arrays the chunks filled
  if (h->wide) {
    if ((rc = dev_alloc_t(h, &h->png_src, ep + 8))) return rc;
    TK(cudaMemcpyAsync(h->png_src, png32_t, sizeof(uint32_t) * ep, cudaMemcpyDeviceToDevice, s));
    TK(cudaMemsetAsync(h->png_src + ep, 0, sizeof(uint32_t) * 8, s));
  }
  if ((rc = dev_alloc_t(h, &h->png16, ep + 16))) return rc;
  TK(cudaMemcpyAsync(h->png16, png16_t, sizeof(uint16_t) * ep, cudaMemcpyDeviceToDevice, s));
  TK(cudaMemsetAsync(h->png16 + ep, 0, sizeof(uint16_t) * 16, s));
  if ((rc = dev_alloc_t(h, &h->upd, ep + 8))) return rc;
  TK(cudaMemsetAsync(h->upd + ep, 0, sizeof(float) * 8, s));   // the scatter writes [0, E') before any read
  {
    const int64_t nga = ep / kPngChunk + 64;     // the scatter copies aligned supersets
    if ((rc = dev_alloc_t(h, &h->grp_at, nga))) return rc;
    k_grp_at<<<grid_for(nga), kT, 0, s>>>(ep, pk, nga, h->grp_at);
    TK(cudaGetLastError());
  }
  pt.mark("PNG arrays");

  // ---- pull comparison: CSC (in-adjacency), sources ascending per destination
  if (pull) {
    if ((rc = dev_alloc_t(h, &h->in_ptr, n_dst + 1))) return rc;
    if ((rc = dev_alloc_t(h, &h->in_src, m))) return rc;
    uint32_t *ck, *ck_s, *cperm, *iota;
    TK(tmp.alloc(&ck, m));
    TK(tmp.alloc(&ck_s, m));
    TK(tmp.alloc(&cperm, m));
    TK(tmp.alloc(&iota, m));
    k_iota<<<grid_for(m), kT, 0, s>>>(m, iota);
    TK(cudaMemcpyAsync(ck, d_col, sizeof(uint32_t) * m, cudaMemcpyDeviceToDevice, s));
    TK(radix_sort_pairs(tmp, ck, ck_s, iota, cperm, m, bits_for((uint64_t)std::max<int64_t>(n_dst - 1, 0)), s));
    k_boundaries<<<grid_for(m + 1), kT, 0, s>>>(m, ck_s, n_dst, h->in_ptr);
    TK(cudaGetLastError());
    k_gather_u32<<<grid_for(m), kT, 0, s>>>(m, cperm, rowid, h->in_src);
    TK(cudaGetLastError());
    h->has_pull = true;
  }
  // ---- max|w| (fixed-point range of the signed SpMV accumulator)
  if (values) {
    float* mx;
    TK(tmp.alloc(&mx, 1));
    float hmx = 0.f;
    int rc2 = launch_absmax(h, d_val, m, mx, s);
    if (rc2) return rc2;
    TK(cudaMemcpyAsync(&hmx, mx, 4, cudaMemcpyDeviceToHost, s));
    TK(cudaStreamSynchronize(s));
    int ex = 0;
    if (hmx > 0.f) frexpf(hmx, &ex);
    h->wexp = ex;
    if ((rc2 = weighted_degrees(h, tmp, d_rp, d_val))) return rc2;
  }
  return finish_layout(h, tmp, pt, G, d_dang);
}

// ---------------------------------------------------------------------------
// Counting construction (the default for k_dst <= kCountMaxK; DESIGN.md §5 "build").
// The paper builds bins and PNG with two scans per partition; here the same
// two passes run warp-per-segment over the CSR, with no sort:
//   segment = a row range [u0, u1) of one source partition p (heavy partitions are cut
//   into several), processed by ONE warp in CSR order (u ascending, v ascending);
//   pass 1 (count): per (segment, j) the number of IDs and of runs (MSB-flagged IDs,
//     Alg. 2's prev_bin test) -- plus out-degrees and validation;
//   scans: id_base[s][j] = bin_id_start[j] + IDs of earlier segments in bin j;
//     PNG group starts G (groups (p, j) in (p, j) order) and each segment's
//     run offset inside its group;
//   pass 2 (place): the same walk; an edge's slot = its segment's running base for
//     bin j + its rank among the same-j edges of the 32-edge step (match_any), so
//     each bin lists its IDs in (u, v) order and each PNG group its sources in u
//     order -- exactly the oracle's layout, deterministic, no atomics on the output.
// The running bases live in shared memory, one k_dst-entry array pair per warp.
constexpr int kCntWarps = 12;             // warps (segments in flight) per CTA
constexpr int64_t kCountMaxK = 2048;      // counters: 2 x k_dst u32 per warp (16 KB at k = 2048)

struct BSeg {
  uint32_t u0, u1, p, pad;
};

__global__ void k_fill_f32(int64_t n, float v, float* out) {
  GRID_STRIDE(i, n) out[i] = v;
}

template <bool PLACE, bool COMPRESS, bool WIDE, bool WEIGHTED>
__global__ void __launch_bounds__(32 * kCntWarps) k_seg_pass(
    const BSeg* __restrict__ segs, int n_seg, uint32_t* seg_ctr, const int64_t* __restrict__ row_ptr,
    const uint32_t* __restrict__ col, const float* __restrict__ val, int b, int64_t k_dst, int64_t n_dst,
    uint32_t* CI, uint32_t* CR, const uint32_t* __restrict__ G, uint32_t* outdeg, float* inv_deg,
    unsigned long long* n_dang, uint32_t* err, uint16_t* ids16, uint32_t* ids32, float* w, uint16_t* png16,
    uint32_t* png32) {
  extern __shared__ uint32_t csm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* ci = csm + (size_t)warp * 2 * k_dst;    // IDs (count) / running ID slot (place) per bin j
  uint32_t* cr = ci + k_dst;                         // runs (count) / running PNG slot (place) per bin j
  uint8_t* rowlist = reinterpret_cast<uint8_t*>(csm + (size_t)kCntWarps * 2 * k_dst) + warp * 32;
  const uint32_t qmask = (1u << b) - 1u;
  uint32_t lt, le;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  asm("mov.u32 %0, %%lanemask_le;" : "=r"(le));
  constexpr int D = 4;                               // 32-edge steps whose column loads are in flight
  uint32_t errs = 0;
  for (;;) {
    uint32_t sidx = 0;
    if (lane == 0) sidx = atomicAdd(seg_ctr, 1u);
    sidx = __shfl_sync(0xffffffffu, sidx, 0);
    if (sidx >= (uint32_t)n_seg) break;
    const BSeg sg = segs[sidx];
    for (int64_t j = lane; j < k_dst; j += 32) {
      if (PLACE) {
        ci[j] = CI[(int64_t)sidx * k_dst + j];
        cr[j] = CR[(int64_t)sidx * k_dst + j] + G[(int64_t)sg.p * k_dst + j];
      } else {
        ci[j] = 0u;
        cr[j] = 0u;
      }
    }
    __syncwarp();
    uint32_t dang = 0;
    // row bounds of the first 32-row batch; each batch prefetches the next one's
    auto load_rows = [&](uint32_t ub, int64_t& rs, int64_t& re) {
      const uint32_t u = ub + lane;
      const bool ur = u < sg.u1;
      rs = ub < sg.u1 ? row_ptr[ur ? u : sg.u1] : 0;
      re = ub < sg.u1 ? (ur ? row_ptr[u + 1] : rs) : 0;
    };
    int64_t nrs, nre;
    load_rows(sg.u0, nrs, nre);
    for (uint32_t ub = sg.u0; ub < sg.u1; ub += 32) {
      const uint32_t u = ub + lane;
      const bool ur = u < sg.u1;
      const int64_t rs64 = nrs, re64 = nre;
      load_rows(ub + 32, nrs, nre);
      const bool nonempty = ur && re64 > rs64;
      if (!PLACE) {
        if (ur) {
          const int64_t dg = re64 - rs64;
          if (dg < 0) errs |= 1u;
          outdeg[u] = (uint32_t)(dg > 0 ? dg : 0);
          inv_deg[u] = dg > 0 ? 1.0f / (float)dg : 0.0f;
        }
        dang += __popc(__ballot_sync(0xffffffffu, ur && re64 == rs64));
      }
      // the batch's non-empty rows in order: the k-th row start of the batch is row rowlist[k]
      const uint32_t N = __ballot_sync(0xffffffffu, nonempty);
      if (nonempty) rowlist[__popc(N & lt)] = (uint8_t)lane;
      __syncwarp();
      const int64_t bs = __shfl_sync(0xffffffffu, rs64, 0);
      const int64_t be = __shfl_sync(0xffffffffu, re64, 31);
      const uint32_t rs = (uint32_t)(rs64 - bs);         // row starts relative to the batch (m < 2^32)
      uint32_t pv = 0, pj = 0;                           // edge before the step (lane 31 of the previous one)
      uint32_t starts = 0;                               // row starts before the step
      for (int64_t x0 = bs; x0 < be; x0 += 32 * D) {
        uint32_t vv[D];
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const int64_t x = x0 + 32 * d + lane;
          vv[d] = x < be ? __ldcs(col + x) : 0u;
        }
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const int64_t xc = x0 + 32 * d;
          if (xc >= be) break;
          const int64_t x = xc + lane;
          const bool valid = x < be;
          const uint32_t v = vv[d];
          const uint32_t xr = (uint32_t)(xc - bs);
          // row starts inside this step (bit l: a non-empty row starts at edge xc + l)
          const uint32_t Bm = __reduce_or_sync(0xffffffffu, (nonempty && rs - xr < 32u) ? 1u << (rs - xr) : 0u);
          const bool first = (Bm >> lane) & 1u;
          const uint32_t k = starts + __popc(Bm & le);      // row starts at or before x
          starts += __popc(Bm);
          const uint32_t r = k ? rowlist[k - 1] : 0u;
          uint32_t j = v >> b;
          const uint32_t upv = __shfl_up_sync(0xffffffffu, v, 1), upj = __shfl_up_sync(0xffffffffu, j, 1);
          const uint32_t prv = lane ? upv : pv, prj = lane ? upj : pj;
          if (!PLACE && valid) {
            if (v >= (uint32_t)n_dst) errs |= 2u;
            if (!first && prv >= v) errs |= 4u;
          }
          if (j >= (uint32_t)k_dst) j = (uint32_t)k_dst - 1;   // invalid input: keep indices in range
          const bool flag = !COMPRESS || first || prj != j;   // Alg. 2 prev_bin / MSB demarcation
          const uint32_t F = __ballot_sync(0xffffffffu, valid && flag);
          const uint32_t me = __match_any_sync(0xffffffffu, valid ? j : 0xFFFFFFFFu);
          const bool lead = lane == 31 - __clz(me);         // highest lane of the same-j group
          if (!PLACE) {
            if (valid && lead) {
              ci[j] += __popc(me);
              cr[j] += __popc(me & F);
            }
          } else {
            uint32_t bi = 0, br = 0;
            if (valid) {
              bi = ci[j];
              br = cr[j];
            }
            __syncwarp();
            if (valid) {
              const uint32_t pos = bi + __popc(me & lt);
              ids16[pos] = (uint16_t)((v & qmask) | (flag ? 0x8000u : 0u));
              if (WIDE) ids32[pos] = v | (flag ? 0x80000000u : 0u);
              if (WEIGHTED) w[pos] = val[x];
              if (flag) {
                const uint32_t pp = br + __popc(me & F & lt);
                const uint32_t uu = ub + r;
                png16[pp] = (uint16_t)(uu & qmask);
                if (WIDE) png32[pp] = uu;
              }
              if (lead) {
                ci[j] = bi + __popc(me);
                cr[j] = br + __popc(me & F);
              }
            }
            __syncwarp();
          }
          pv = __shfl_sync(0xffffffffu, v, 31);
          pj = __shfl_sync(0xffffffffu, j, 31);
        }
      }
      __syncwarp();
    }
    __syncwarp();
    if (!PLACE) {
      for (int64_t j = lane; j < k_dst; j += 32) {
        CI[(int64_t)sidx * k_dst + j] = ci[j];
        CR[(int64_t)sidx * k_dst + j] = cr[j];
      }
      if (lane == 0 && dang) atomicAdd(n_dang, (unsigned long long)dang);
    }
    __syncwarp();
  }
  if (!PLACE) {
    for (int o = 16; o; o >>= 1) errs |= __shfl_xor_sync(0xffffffffu, errs, o);
    if (lane == 0 && errs) atomicOr(err, errs);
  }
}


// ---------------------------------------------------------------------------
// CTA-tile form of the two passes (the default; DESIGN.md §5 "build").  One CTA owns a
// segment and walks it in tiles of kTileE consecutive CSR edges:
//   prep   : column loads (coalesced, a whole tile in flight), the row of every edge
//            (row starts marked, then a block max-scan), the run flags of Alg. 2;
//   count  : per-bin ID and run counts with shared-memory atomics;
//   place  : a stable block radix sort of the tile by bin j (LSD, 4-bit digits,
//            warp-striped ranking with ballots), then each bin's run of the tile goes
//            to its running slot -- consecutive positions, so the CTA's writes fill
//            whole sectors while they are still in L2 (148 CTAs x k_dst open sectors,
//            ~10 MB, instead of one open sector per (warp, bin)).
constexpr int kTileThreads = 512, kTileWarps = kTileThreads / 32;
#ifndef PCPM_TILE_E
#define PCPM_TILE_E 4096
#endif
#ifndef PCPM_TILE_BUCKET_CTAS
#define PCPM_TILE_BUCKET_CTAS 2      // CTAs per SM of the bucket pass (2 needs PCPM_TILE_E <= 4096)
#endif
constexpr int kTileE = PCPM_TILE_E;                 // edges per tile
constexpr int kTileItems = kTileE / kTileThreads;   // 8 per thread, warp-striped: element w*512 + l + 32 k
constexpr int kTileECnt = 8192;                      // edges per tile of the count pass
constexpr int kRadixBits = 4, kRadixB = 1 << kRadixBits;

struct TileSmem {           // carved from dynamic shared memory (k_dst-sized arrays first)
  uint32_t* ci;             // [k_dst] counts (count) / running ID slot (place)
  uint32_t* cr;             // [k_dst] run counts / running PNG slot
  uint16_t* bstart;         // [k_dst] first sorted index of bin j in the tile
  uint16_t* bfstart;        // [k_dst] flags before that index
  // double buffers as named fields (a runtime-indexed pointer array would live in local
  // memory and lose the shared address space: generic LD/ST on every access, measured)
  uint16_t *key0, *key1;    // [kTileE] bin j
  uint32_t *pay0, *pay1;    // [kTileE] (v & (q-1)) | flag << 15 | (u & (q-1)) << 16; pay1 doubles as the row marks
  uint16_t *idx0, *idx1;    // [kTileE] tile position (weights)
  uint32_t* sbits;          // [kTileE / 32] row-start bits
  uint32_t* wsum;           // [kTileWarps * kRadixB + 64] scan scratch
  uint32_t *colb0, *colb1;  // [kTileE + 8] the tile's columns (bulk-copied one tile ahead)
};

// mode 1 (pass 1, count): the counts, row-start bits, scan scratch and column buffers only;
// mode 2 (bucket pass): 64 bucket slots, keys, payloads, marks, tags, bits, scratch, columns.
// Both fit twice per SM (two CTAs hide each other's barrier waits); mode 0: everything.
size_t tile_smem_bytes(int64_t k_dst, int mode = 0) {
  const size_t kd = (size_t)((k_dst + 3) & ~int64_t(3));
  if (mode == 1)
    return kd * 4 * 2 + kTileECnt / 32 * 4 + (kTileWarps * kRadixB + 64) * 4 + 2 * ((size_t)kTileECnt + 8) * 4 + 64;
  if (mode == 2)
    return 64 * 4 + (size_t)kTileE * (4 + 4 + 2 + 2) + kTileE / 32 * 4 + (kTileWarps * kRadixB + 64) * 4 +
           2 * ((size_t)kTileE + 8) * 4 + 64;
  return kd * 4 * 2 + kd * 2 * 2 + (size_t)kTileE * (2 + 4 + 2) * 2 + kTileE / 32 * 4 +
         (kTileWarps * kRadixB + 64) * 4 + 2 * ((size_t)kTileE + 8) * 4 + 64;
}

__device__ __forceinline__ TileSmem tile_carve(uint8_t* base, int64_t k_dst, int mode = 0) {
  const size_t kd = (size_t)((k_dst + 3) & ~int64_t(3));
  TileSmem t;
  t.ci = reinterpret_cast<uint32_t*>(base);
  if (mode == 2) {
    t.cr = nullptr;
    t.pay0 = t.ci + 64;
    t.pay1 = t.pay0 + kTileE;
    t.sbits = t.pay1 + kTileE;
    t.wsum = t.sbits + kTileE / 32;
    t.colb0 = t.wsum + kTileWarps * kRadixB + 64;
    t.colb1 = t.colb0 + kTileE + 8;
    t.key0 = reinterpret_cast<uint16_t*>(t.colb1 + kTileE + 8);
    t.idx0 = t.key0 + kTileE;
    t.key1 = t.idx1 = t.bstart = t.bfstart = nullptr;
    return t;
  }
  t.cr = t.ci + kd;
  if (mode == 1) {
    t.sbits = t.cr + kd;
    t.wsum = t.sbits + kTileECnt / 32;
    t.colb0 = t.wsum + kTileWarps * kRadixB + 64;
    t.colb1 = t.colb0 + kTileECnt + 8;
    t.pay0 = t.pay1 = nullptr;
    t.key0 = t.key1 = t.idx0 = t.idx1 = t.bstart = t.bfstart = nullptr;
    return t;
  }
  t.pay0 = t.cr + kd;
  t.pay1 = t.pay0 + kTileE;
  t.sbits = t.pay1 + kTileE;
  t.wsum = t.sbits + kTileE / 32;
  t.colb0 = t.wsum + kTileWarps * kRadixB + 64;
  t.colb1 = t.colb0 + kTileE + 8;
  t.key0 = reinterpret_cast<uint16_t*>(t.colb1 + kTileE + 8);
  t.key1 = t.key0 + kTileE;
  t.idx0 = t.key1 + kTileE;
  t.idx1 = t.idx0 + kTileE;
  t.bstart = t.idx1 + kTileE;
  t.bfstart = t.bstart + kd;
  return t;
}

// BUCKET (with PLACE; the two-level placement for k_dst > kBucketMinK): instead of the
// tile sort by bin, each edge's record ((j & 31) << 32 | payload) goes to the scratch
// sub-range of its segment and bucket h = j >> 5 (SB[s][h], stable: tiles in CSR order,
// ranks by (warp, step, lane)); k_bucket_place then places each (segment, bucket).
struct BucketArgs {
  const uint32_t* SB;       // [n_seg][nbk + 1] scratch start of (s, h); [s][nbk] = the segment's end
  int nbk;                  // buckets = ceil(k_dst / 32)
  uint64_t* rec;            // [m] records
  float* recw;              // [m] weights (WEIGHTED)
  const float* xval;        // BV: the scatter input (the record carries x[u] instead of the payload)
  float* upd;               // BV: the update bins
};

// BV (with BUCKET; the BVGAS engine's per-iteration scatter, Alg. 3): the record
// carries the source value x[u] instead of the layout payload; no validation.
template <bool PLACE, bool COMPRESS, bool WIDE, bool WEIGHTED, bool BUCKET = false, bool BV = false>
__global__ void __launch_bounds__(kTileThreads, BUCKET ? PCPM_TILE_BUCKET_CTAS : (PLACE ? 1 : 2)) k_tile_pass(
    const BSeg* __restrict__ segs, int n_seg, uint32_t* seg_ctr, const int64_t* __restrict__ row_ptr,
    const uint32_t* __restrict__ col, const float* __restrict__ val, int b, int64_t k_dst, int64_t n_dst, int kbits,
    uint32_t* CI, uint32_t* CR, const uint32_t* __restrict__ G, uint32_t* outdeg, float* inv_deg,
    unsigned long long* n_dang, uint32_t* err, uint16_t* ids16, uint32_t* ids32, float* w, uint16_t* png16,
    uint32_t* png32, const BucketArgs ba) {
  // the count pass walks 8192-edge tiles (two CTAs per SM), the placing passes kTileE
  constexpr int TE = PLACE ? kTileE : kTileECnt;
  constexpr int TI = TE / kTileThreads;
  extern __shared__ __align__(16) uint8_t tsm[];
  const TileSmem T = tile_carve(tsm, k_dst, !PLACE ? 1 : (BUCKET ? 2 : 0));
  const int tid = threadIdx.x;
  __shared__ uint32_t seg_s;
  __shared__ __align__(8) uint64_t cbar[2];
  // the tile's 16 B-aligned middle [a, c) of col comes in by one bulk copy (TMA engine), issued
  // one tile ahead; its ragged ends are loaded by threads.  Element x of a tile starting at x0
  // lives at colb[x - (x0 & ~3)].
  const bool bulk_ok = (reinterpret_cast<uintptr_t>(col) & 15) == 0;
  auto issue_cols = [&](int bsel, int64_t x0, int64_t x1) {       // thread 0
    const int64_t a = (x0 + 3) & ~int64_t(3), c = x1 & ~int64_t(3);
    if (bulk_ok && c > a) {
      mbar_arrive_expect_tx(&cbar[bsel], (uint32_t)((c - a) * 4));
      bulk_g2s((bsel ? T.colb1 : T.colb0) + (a - (x0 & ~int64_t(3))), col + a, (uint32_t)((c - a) * 4), &cbar[bsel],
               policy_evict_first());
    } else {
      mbar_arrive(&cbar[bsel]);
    }
  };
  if (tid == 0) {
    mbar_init(&cbar[0], 1);
    mbar_init(&cbar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t cphase = 0u;                 // bit b: parity of column buffer b
  const int lane = tid & 31, warp = tid >> 5;
  const uint32_t qmask = (1u << b) - 1u;
  uint32_t lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  uint32_t errs = 0;
  for (;;) {
    if (tid == 0) seg_s = atomicAdd(seg_ctr, 1u);
    __syncthreads();
    const uint32_t sidx = seg_s;
    if (sidx >= (uint32_t)n_seg) break;
    const BSeg sg = segs[sidx];
    if (BUCKET) {
      for (int h = tid; h < ba.nbk; h += kTileThreads) T.ci[h] = ba.SB[(int64_t)sidx * (ba.nbk + 1) + h];
    }
    for (int64_t j = tid; !BUCKET && j < k_dst; j += kTileThreads) {
      if (PLACE) {
        T.ci[j] = CI[(int64_t)sidx * k_dst + j];
        T.cr[j] = CR[(int64_t)sidx * k_dst + j] + G[(int64_t)sg.p * k_dst + j];
      } else {
        T.ci[j] = 0u;
        T.cr[j] = 0u;
      }
    }
    // out-degrees of the segment's rows (count pass)
    if (!PLACE) {
      uint32_t dang = 0;
      for (uint32_t u = sg.u0 + tid; u < sg.u1; u += kTileThreads) {
        const int64_t dg = row_ptr[u + 1] - row_ptr[u];
        if (dg < 0) errs |= 1u;
        outdeg[u] = (uint32_t)(dg > 0 ? dg : 0);
        inv_deg[u] = dg > 0 ? 1.0f / (float)dg : 0.0f;
        dang += dg == 0;
      }
      for (int o = 16; o; o >>= 1) dang += __shfl_xor_sync(0xffffffffu, dang, o);
      if (lane == 0 && dang) atomicAdd(n_dang, (unsigned long long)dang);
    }
    const int64_t e0 = row_ptr[sg.u0], e1 = row_ptr[sg.u1];
    uint32_t rnext = sg.u0;               // first row whose start is >= the tile's first edge
    uint32_t pbase = 0xFFFFFFFFu;         // rows pbase + tid: row starts prefetched in prs / pre
    int64_t prs = 0, pre = 0;
    uint32_t rcur = sg.u0;                // row of the edge before the tile
    uint32_t pj = 0xFFFFFFFFu, pv = 0;    // bin / column of the edge before the tile
    int cb = 0;                           // column buffer of the current tile
    if (tid == 0 && e0 < e1) issue_cols(0, e0, min(e1, e0 + TE));
    __syncthreads();
    for (int64_t x0 = e0; x0 < e1; x0 += TE, cb ^= 1) {
      const int n = (int)min((int64_t)TE, e1 - x0);
      const int64_t x1 = x0 + n;
      // next tile's columns in flight under this tile's work (its buffer was last read by
      // the previous tile, which every thread has finished)
      if (tid == 0 && x1 < e1) issue_cols(cb ^ 1, x1, min(e1, x1 + TE));
      // ---- prep: columns, row marks
      // (the count pass needs only the row-start bits: no per-edge row, no payload)
      uint32_t* mark = T.pay1;
      if (PLACE)
        for (int i = tid; i < TE; i += kTileThreads) mark[i] = 0u;
      for (int i = tid; i < TE / 32; i += kTileThreads) T.sbits[i] = 0u;
      uint32_t* vfull = (cb ? T.colb1 : T.colb0) + (x0 & 3);   // vfull[i] = col[x0 + i]
      {
        const int64_t a = (x0 + 3) & ~int64_t(3), c = x1 & ~int64_t(3);
        if (!bulk_ok || c <= a) {
          for (int i = tid; i < n; i += kTileThreads) vfull[i] = __ldcs(col + x0 + i);
        } else {
          if (tid < a - x0) vfull[tid] = __ldcs(col + x0 + tid);                 // head (< 4)
          if (tid >= 4 && tid - 4 < x1 - c) vfull[c - x0 + tid - 4] = __ldcs(col + c + tid - 4);   // tail (< 4)
        }
      }
      mbar_wait(&cbar[cb], (cphase >> cb) & 1u);
      cphase ^= 1u << cb;
      __syncthreads();
      if (PLACE && tid == 0) mark[0] = rcur + 1;   // edges before the first row start belong to rcur
      for (uint32_t rb = rnext;; rb += kTileThreads) {
        const uint32_t r = rb + tid;
        int64_t rs = x1, re = x1;
        if (r < sg.u1) {
          if (rb == pbase) {                // loaded during the previous tile
            rs = prs;
            re = pre;
          } else {
            rs = row_ptr[r];
            re = row_ptr[r + 1];
          }
        }
        const bool in = r < sg.u1 && rs < x1;
        if (in && re > rs) {              // a non-empty row starting inside the tile
          if (PLACE) atomicMax(&mark[rs - x0], r + 1);
          atomicOr(&T.sbits[(rs - x0) >> 5], 1u << ((rs - x0) & 31));
        }
        const int cnt = __syncthreads_count(in);
        if (cnt < kTileThreads) {
          rnext = rb + cnt;
          break;
        }
      }
      // the next tile's first round of row starts, loaded now (consumed one tile later)
      pbase = rnext;
      if (rnext + tid < sg.u1) {
        prs = row_ptr[rnext + tid];
        pre = row_ptr[rnext + tid + 1];
      }
      __syncthreads();
      // block max-scan of the marks: element i's row (+1); warp-striped, 16 per thread; the 16
      // rounds are scanned independently, then chained by their maxima (ILP instead of a chain)
      if (PLACE) {
        const int base = warp * (TE / kTileWarps);
        uint32_t loc[TI];
#pragma unroll
        for (int k = 0; k < TI; ++k) loc[k] = mark[base + 32 * k + lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1)
#pragma unroll
          for (int k = 0; k < TI; ++k) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, loc[k], o);
            if (lane >= o) loc[k] = max(loc[k], y);
          }
        uint32_t mx = 0;
#pragma unroll
        for (int k = 0; k < TI; ++k) {
          const uint32_t top = __shfl_sync(0xffffffffu, loc[k], 31);
          loc[k] = max(loc[k], mx);
          mx = max(mx, top);
        }
        if (lane == 0) T.wsum[warp] = mx;
        __syncthreads();
        uint32_t before = 0;
        for (int ww = 0; ww < warp; ++ww) before = max(before, T.wsum[ww]);
#pragma unroll
        for (int k = 0; k < TI; ++k) mark[base + 32 * k + lane] = max(loc[k], before);
      }
      __syncthreads();
      // carries for the next tile (the marks are overwritten by the payloads below)
      if (PLACE && tid == 0) T.wsum[kTileWarps * kRadixB + 2] = mark[n - 1] - 1u;
      // ---- per edge: bin, run flag, payload
      for (int i = tid; i < TE; i += kTileThreads) {
        if (i < n) {
          const uint32_t v = vfull[i];
          const uint32_t u = PLACE ? mark[i] - 1u : 0u;
          const bool first = (T.sbits[i >> 5] >> (i & 31)) & 1u;
          const uint32_t prv = i ? vfull[i - 1] : pv;
          uint32_t j = v >> b;
          if (!PLACE) {
            if (v >= (uint32_t)n_dst) errs |= 2u;
            if (!first && prv >= v) errs |= 4u;
          }
          if (j >= (uint32_t)k_dst) j = (uint32_t)k_dst - 1;
          uint32_t prj = i ? (prv >> b) : pj;
          if (i && prj >= (uint32_t)k_dst) prj = (uint32_t)k_dst - 1;
          const bool flag = !COMPRESS || first || prj != j;
          if (PLACE) {
            T.key0[i] = (uint16_t)j;
            if (!BUCKET) T.idx0[i] = (uint16_t)i;
            T.pay0[i] = BV ? __float_as_uint(__ldg(ba.xval + u)) : (v & qmask) | (flag ? 0x8000u : 0u) | ((u & qmask) << 16);
          } else {
            atomicAdd(&T.ci[j], 1u);
            if (flag) atomicAdd(&T.cr[j], 1u);
          }
        } else if (PLACE) {
          T.key0[i] = 0xFFFFu;          // padding sorts last
          T.idx0[i] = 0;
          T.pay0[i] = 0u;
        }
      }
      __syncthreads();
      // carry (every thread needs pj/pv/rcur for the next tile): broadcast through smem
      if (tid == 0) {
        const uint32_t lv = vfull[n - 1];
        uint32_t lj = lv >> b;
        if (lj >= (uint32_t)k_dst) lj = (uint32_t)k_dst - 1;
        T.wsum[kTileWarps * kRadixB] = lv;
        T.wsum[kTileWarps * kRadixB + 1] = lj;
      }
      __syncthreads();
      pv = T.wsum[kTileWarps * kRadixB];
      pj = T.wsum[kTileWarps * kRadixB + 1];
      rcur = T.wsum[kTileWarps * kRadixB + 2];
      if (!PLACE) {
        __syncthreads();
        continue;
      }
      if constexpr (BUCKET) {
        // ---- stable counting placement of the tile's records by bucket h = j >> 5 (< 64):
        // per warp (its 512 elements: steps k, lanes) ranks from 6 ballots of the bucket
        // bits and per-warp counts in registers (lane l counts buckets l and l + 32); then
        // per-bucket bases over the warps (earlier warps = earlier elements); records go to
        // SB's running slot + base + rank.
        constexpr int kWs = 65;                       // padded stride of the per-warp totals
        uint32_t* wc = T.pay1;                        // [kTileWarps][kWs] (the row marks are consumed)
        const int base = warp * (TE / kTileWarps);
        uint32_t rk[TI];
        uint32_t c_lo = 0, c_hi = 0;
#pragma unroll
        for (int k = 0; k < TI; ++k) {
          const int i = base + 32 * k + lane;
          const bool ok = i < n;
          const uint32_t hb = ok ? (uint32_t)(T.key0[i] >> 5) : 0u;
          const uint32_t vm = __ballot_sync(0xffffffffu, ok);
          uint32_t mb = vm;                           // lanes whose bucket is `lane` or `lane` + 32
#pragma unroll
          for (int t = 0; t < 5; ++t)
            mb &= __ballot_sync(0xffffffffu, (hb >> t) & 1u) ^ (((lane >> t) & 1) ? 0u : 0xFFFFFFFFu);
          const uint32_t b5 = __ballot_sync(0xffffffffu, (hb >> 5) & 1u);
          const uint32_t pm = __shfl_sync(0xffffffffu, mb, hb & 31u) & ((hb & 32u) ? b5 : ~b5);
          const uint32_t bl = __shfl_sync(0xffffffffu, c_lo, hb & 31u), bh = __shfl_sync(0xffffffffu, c_hi, hb & 31u);
          rk[k] = ((hb & 32u) ? bh : bl) + __popc(pm & lt);
          c_lo += __popc(mb & ~b5);
          c_hi += __popc(mb & b5);
        }
        wc[warp * kWs + lane] = c_lo;
        wc[warp * kWs + 32 + lane] = c_hi;
        __syncthreads();
        {
          // bucket 4 w + 2 r + (lane >> 4), r = 0, 1: exclusive scan over the 16 warps (lane & 15)
          static_assert(kTileWarps == 16, "two buckets per 32-lane scan");
          const int l16 = lane & 15;
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const int hh = 4 * warp + 2 * r + (lane >> 4);
            const uint32_t a = hh < ba.nbk ? wc[l16 * kWs + hh] : 0u;
            uint32_t ia = a;
#pragma unroll
            for (int o = 1; o < 16; o <<= 1) {
              const uint32_t y = __shfl_up_sync(0xffffffffu, ia, o, 16);
              if (l16 >= o) ia += y;
            }
            const uint32_t bb = hh < ba.nbk ? T.ci[hh] : 0u;
            __syncwarp();
            if (hh < ba.nbk) {
              wc[l16 * kWs + hh] = bb + ia - a;
              if (l16 == 15) T.ci[hh] = bb + ia;
            }
          }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < TI; ++k) {
          const int i = base + 32 * k + lane;
          if (i < n) {
            const uint32_t j = T.key0[i];
            const uint32_t pos = wc[warp * kWs + (j >> 5)] + rk[k];
            ba.rec[pos] = ((uint64_t)(j & 31u) << 32) | T.pay0[i];
            if (WEIGHTED) ba.recw[pos] = val[x0 + i];
          }
        }
        __syncthreads();
        continue;
      }

      // ---- stable LSD radix sort of the tile by bin (kbits bits, 4 per pass)
      int cur = 0;
      for (int sh = 0; sh < kbits; sh += kRadixBits) {
        const uint16_t* kin = cur ? T.key1 : T.key0;
        const uint32_t* pin = cur ? T.pay1 : T.pay0;
        const uint16_t* iin = cur ? T.idx1 : T.idx0;
        uint16_t* kout = cur ? T.key0 : T.key1;
        uint32_t* pout = cur ? T.pay0 : T.pay1;
        uint16_t* iout = cur ? T.idx0 : T.idx1;
        const int base = warp * (TE / kTileWarps);
        uint32_t rnk[TI];
        uint32_t dig[TI];
        uint32_t cnt = 0;                         // lane d < 16: this warp's count of digit d
        const uint32_t dd = lane & (kRadixB - 1);
        // rounds are independent: ballots per round, then lane dd's running count of digit dd
#pragma unroll
        for (int k = 0; k < TI; ++k) {
          const uint32_t d = (kin[base + 32 * k + lane] >> sh) & (kRadixB - 1);
          uint32_t peers = 0xffffffffu, mdd = 0xffffffffu;   // lanes with my digit / with digit dd
#pragma unroll
          for (int bt = 0; bt < kRadixBits; ++bt) {
            const uint32_t bal = __ballot_sync(0xffffffffu, (d >> bt) & 1u);
            peers &= ((d >> bt) & 1u) ? bal : ~bal;
            mdd &= ((dd >> bt) & 1u) ? bal : ~bal;
          }
          dig[k] = d;
          rnk[k] = cnt | (__popc(peers & lt) << 16);        // (count before the round, rank in the round)
          cnt += __popc(mdd);
        }
#pragma unroll
        for (int k = 0; k < TI; ++k)
          rnk[k] = __shfl_sync(0xffffffffu, rnk[k] & 0xFFFFu, dig[k]) + (rnk[k] >> 16);
        if (lane >= kRadixB) cnt = 0;
        // warp totals per digit -> block bases: base(w, d) = sum_{d' < d} total(d') + sum_{w' < w} cnt(w', d)
        if (lane < kRadixB) T.wsum[lane * kTileWarps + warp] = cnt;     // digit-major
        __syncthreads();
        if (warp == 0) {
          // exclusive scan of the kRadixB * kTileWarps (= 256) counts, 8 per lane
          uint32_t v8[8], s8 = 0;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            v8[k] = T.wsum[lane * 8 + k];
            s8 += v8[k];
          }
          uint32_t inc = s8;
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
          }
          uint32_t run = inc - s8;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            T.wsum[lane * 8 + k] = run;
            run += v8[k];
          }
        }
        __syncthreads();
        const int nxt = cur ^ 1;
#pragma unroll
        for (int k = 0; k < TI; ++k) {
          const int src = base + 32 * k + lane;
          const uint32_t dst = T.wsum[dig[k] * kTileWarps + warp] + rnk[k];
          kout[dst] = kin[src];
          pout[dst] = pin[src];
          iout[dst] = iin[src];
        }
        __syncthreads();
        cur = nxt;
      }
      // ---- positions: bin runs of the sorted tile, flag prefix
      {
        const uint16_t* ks = cur ? T.key1 : T.key0;
        const uint32_t* ps = cur ? T.pay1 : T.pay0;
        const uint16_t* is = cur ? T.idx1 : T.idx0;
        const int base = warp * (TE / kTileWarps);
        uint32_t fpre[TI];
        uint32_t fw = 0;
#pragma unroll
        for (int k = 0; k < TI; ++k) {
          const uint32_t f = (ps[base + 32 * k + lane] >> 15) & 1u;
          const uint32_t bal = __ballot_sync(0xffffffffu, f);
          fpre[k] = fw + __popc(bal & lt);
          fw += __popc(bal);
        }
        if (lane == 0) T.wsum[warp] = fw;
        __syncthreads();
        uint32_t fbase = 0;
        for (int ww = 0; ww < warp; ++ww) fbase += T.wsum[ww];
        // run starts: bstart[j] = first sorted index of j, bfstart[j] = flags before it
#pragma unroll
        for (int k = 0; k < TI; ++k) {
          const int i = base + 32 * k + lane;
          if (i < n) {
            const uint32_t j = ks[i];
            if (i == 0 || ks[i - 1] != j) {
              T.bstart[j] = (uint16_t)i;
              T.bfstart[j] = (uint16_t)(fbase + fpre[k]);
            }
          }
        }
        __syncthreads();
        uint32_t nci[TI], ncr[TI];
#pragma unroll
        for (int k = 0; k < TI; ++k) {
          const int i = base + 32 * k + lane;
          nci[k] = ncr[k] = 0xFFFFFFFFu;
          if (i < n) {
            const uint32_t j = ks[i];
            const uint32_t pw = ps[i];
            const bool f = (pw >> 15) & 1u;
            const uint32_t pos = T.ci[j] + (uint32_t)(i - T.bstart[j]);
            const uint32_t fx = fbase + fpre[k];                      // flags before i in the tile
            const uint32_t pp = T.cr[j] + (fx - T.bfstart[j]);
            ids16[pos] = (uint16_t)(pw & 0xFFFFu);
            if (WIDE) ids32[pos] = ((j << b) | (pw & qmask)) | (f ? 0x80000000u : 0u);
            if (WEIGHTED) w[pos] = val[x0 + is[i]];
            if (f) {
              png16[pp] = (uint16_t)(pw >> 16);
              if (WIDE) png32[pp] = (sg.p << b) | (pw >> 16);
            }
            if (i == n - 1 || ks[i + 1] != j) {   // the bin's last element in the tile
              nci[k] = pos + 1;
              ncr[k] = pp + (f ? 1u : 0u);
            }
          }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < TI; ++k)
          if (nci[k] != 0xFFFFFFFFu) {
            const uint32_t j = ks[base + 32 * k + lane];
            T.ci[j] = nci[k];
            T.cr[j] = ncr[k];
          }
        __syncthreads();
      }
    }
    if (!PLACE) {
      __syncthreads();
      for (int64_t j = tid; j < k_dst; j += kTileThreads) {
        CI[(int64_t)sidx * k_dst + j] = T.ci[j];
        CR[(int64_t)sidx * k_dst + j] = T.cr[j];
      }
    }
    __syncthreads();
  }
  if (!PLACE) {
    for (int o = 16; o; o >>= 1) errs |= __shfl_xor_sync(0xffffffffu, errs, o);
    if (lane == 0 && errs) atomicOr(err, errs);
  }
}

using TilePassFn = void (*)(const BSeg*, int, uint32_t*, const int64_t*, const uint32_t*, const float*, int, int64_t,
                            int64_t, int, uint32_t*, uint32_t*, const uint32_t*, uint32_t*, float*,
                            unsigned long long*, uint32_t*, uint16_t*, uint32_t*, float*, uint16_t*, uint32_t*,
                            const BucketArgs);

template <bool PLACE, bool BUCKET = false>
TilePassFn tile_pass_fn(bool compress, bool wide, bool weighted) {
#define PCPM_TILE_FN(C, WI, WE) \
  if (compress == C && wide == WI && weighted == WE) return k_tile_pass<PLACE, C, WI, WE, BUCKET>;
  PCPM_TILE_FN(true, false, false) PCPM_TILE_FN(true, false, true) PCPM_TILE_FN(true, true, false)
  PCPM_TILE_FN(true, true, true) PCPM_TILE_FN(false, false, false) PCPM_TILE_FN(false, false, true)
  PCPM_TILE_FN(false, true, false) PCPM_TILE_FN(false, true, true)
#undef PCPM_TILE_FN
  return nullptr;
}

// ---------------------------------------------------------------------------
// Two-level placement (k_dst > kBucketMinK; DESIGN.md §5 "build").  The one-level place
// pass writes each tile's edges to k_dst bins in runs of ~m/(tiles k_dst) IDs (4 at c4):
// partial sectors, written back to DRAM several times (measured: 11.6 GB written for 3.6 GB
// of layout).  Here the tile pass first moves each edge's record into its segment's
// bucket h = j >> 5 (runs of ~128 records), then k_bucket_place takes one (segment s,
// bucket h) at a time -- its records in CSR order -- and places them into the 32 bins of h
// (runs of ~256 IDs per tile).  Same stable order, so the same layout, bit for bit.
constexpr int64_t kBucketMinK = 64;        // up to 64 bins the one-level pass already writes long runs
constexpr uint32_t kHeavyUnit = 4 * kTileE;

// SB[s][h] = first scratch slot of (segment s, bucket h): the segment's first edge + the
// IDs of its earlier buckets; SB[s][nbk] = the segment's end.  CI holds the absolute ID
// bases per (s, j) (after the column prefix), so the count of (s, j) is the next
// segment's base minus this one (the last segment: the bin's end).  One block per segment.
__global__ void __launch_bounds__(1024) k_seg_buckets(int64_t n_seg, int64_t k_dst, int nbk, const BSeg* segs,
                                                      const int64_t* __restrict__ row_ptr,
                                                      const uint32_t* __restrict__ CI,
                                                      const uint32_t* __restrict__ bin_id_start, uint32_t* SB) {
  __shared__ uint32_t hs[64];
  const int64_t sg = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int h = warp; h < nbk; h += 32) {
    const int64_t j = (int64_t)h * 32 + lane;
    uint32_t c = 0;
    if (j < k_dst) {
      const uint32_t nxt = sg + 1 < n_seg ? CI[(sg + 1) * k_dst + j] : bin_id_start[j + 1];
      c = nxt - CI[sg * k_dst + j];
    }
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) hs[h] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t run = (uint32_t)row_ptr[segs[sg].u0];
    for (int h = 0; h < nbk; ++h) {
      SB[sg * (nbk + 1) + h] = run;
      run += hs[h];
    }
    SB[sg * (nbk + 1) + nbk] = run;
  }
}

// Work list of the (s, h) units with records: heavy ones (> kHeavyUnit) from the front,
// the rest from the back (claim order only; the output does not depend on it).
__global__ void k_bucket_units(int64_t n_units, int nbk, const uint32_t* __restrict__ SB, uint32_t* units,
                               uint32_t* nheavy_nlight) {
  GRID_STRIDE(u, n_units) {
    const int64_t sg = u / nbk, h = u % nbk;
    const uint32_t sz = SB[sg * (nbk + 1) + h + 1] - SB[sg * (nbk + 1) + h];
    if (sz == 0) continue;
    if (sz > kHeavyUnit) units[atomicAdd(&nheavy_nlight[0], 1u)] = (uint32_t)u;
    else units[n_units - 1 - atomicAdd(&nheavy_nlight[1], 1u)] = (uint32_t)u;
  }
}

// Place the records of unit (s, h) into bins j = 32 h + (0..31): destID slot = CI[s][j] +
// rank among the unit's bin-j records, PNG slot = G[p][j] + CR[s][j] + rank among its
// flagged ones (runs, Alg. 2).  Tiles of kTileE records, warp-striped like the tile pass.
// 2 CTAs of 512 threads per SM, 4096-record tiles (8 per thread).  The CTA walks its units'
// tiles as one stream: the records of the next tile (possibly of the next unit, claimed one
// tile ahead by warp 0, which also loads that unit's bin bases) are bulk-copied (TMA) into
// the other half of a double buffer while this tile is ranked and placed.
#ifndef PCPM_BP_CTAS
#define PCPM_BP_CTAS 2
#endif
constexpr int kBpThreads = 1024 / PCPM_BP_CTAS, kBpWarps = kBpThreads / 32, kBpItems = 8;
constexpr int kBpTile = kBpThreads * kBpItems;
struct BpUnit {
  uint32_t r0, r1, p, h;     // records [r0, r1) of bucket h of a segment of partition p
  uint32_t ci[32], cr[32];   // the 32 bins' first ID slot / first PNG slot for this segment
  uint32_t valid, pad[3];
};
// STAGED (compact layout, the default): a tile's destination IDs and PNG sources are first
// written into shared memory grouped by bin (each bin's records contiguous, in rank order),
// then copied out with consecutive threads writing consecutive slots of a bin (coalesced
// 2-byte stores) instead of every lane storing into a different bin's range.
#ifndef PCPM_BP_STAGED
#define PCPM_BP_STAGED 1
#endif
size_t bucket_place_smem(bool weighted) {
  return 2 * ((size_t)kBpTile + 2) * 8 + (weighted ? 2 * ((size_t)kBpTile + 4) * 4 : 0) + 2 * sizeof(BpUnit) + 64 +
         (PCPM_BP_STAGED ? (size_t)kBpTile * (2 + 2 + 1 + 1) : 0);
}

template <bool WIDE, bool WEIGHTED, bool BV = false>
__global__ void __launch_bounds__(kBpThreads, PCPM_BP_CTAS) k_bucket_place(
    const uint32_t* __restrict__ units, const uint32_t* nheavy_nlight, int64_t n_units, uint32_t* ctr,
    const BSeg* __restrict__ segs, int b, int64_t k_dst, const uint32_t* __restrict__ CI,
    const uint32_t* __restrict__ CR, const uint32_t* __restrict__ G, const BucketArgs ba, uint16_t* ids16,
    uint32_t* ids32, float* w, uint16_t* png16, uint32_t* png32) {
  // Per warp and bin, counts are kept in registers (lane l counts bin l): a step's bins come
  // from 5 ballots of the bin bits, so a step has no shared-memory round trip.
  extern __shared__ __align__(16) uint8_t bsm[];
  uint64_t* rbuf = reinterpret_cast<uint64_t*>(bsm);                          // [2][kBpTile + 2]
  float* wbuf = reinterpret_cast<float*>(rbuf + 2 * (kBpTile + 2));           // [2][kBpTile + 4]
  BpUnit* un = reinterpret_cast<BpUnit*>(reinterpret_cast<uint8_t*>(wbuf) + (WEIGHTED ? 2 * (kBpTile + 4) * 4 : 0));
  uint64_t* bar = reinterpret_cast<uint64_t*>(un + 2);                         // [2]
  constexpr bool kStaged = PCPM_BP_STAGED && !WIDE && !BV;
  uint16_t* stI = reinterpret_cast<uint16_t*>(bar + 8);                        // [kBpTile] staged IDs
  uint16_t* stF = stI + kBpTile;                                               // [kBpTile] staged PNG sources
  uint8_t* tgI = reinterpret_cast<uint8_t*>(stF + kBpTile);                    // [kBpTile] bin of staged ID
  uint8_t* tgF = tgI + kBpTile;                                                // [kBpTile] bin of staged PNG
  __shared__ uint32_t offI[33], offF[33], gI[32], gF[32];   // staged: per-bin tile offsets / global starts
  __shared__ uint32_t wI[kBpWarps][33], wF[kBpWarps][33];   // per-warp totals -> per-warp bases
  __shared__ uint32_t ciS[32], crS[32];                      // running ID / PNG slot of bin 32 h + l
  __shared__ uint32_t tile_s[4];                             // next tile: x0, unit slot, first-of-unit, valid
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  uint32_t sel[5];                                 // lane l's bin mask: AND_t (bal_t ^ sel_t)
#pragma unroll
  for (int t = 0; t < 5; ++t) sel[t] = ((lane >> t) & 1) ? 0u : 0xFFFFFFFFu;
  const uint32_t nh = nheavy_nlight[0], nl = nheavy_nlight[1];
  const uint32_t qmask = (1u << b) - 1u;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  // warp 0: claim the next non-empty unit into slot us, with its bin bases
  auto claim = [&](int us) {
    uint32_t u = 0xFFFFFFFFu;
    if (lane == 0) {
      const uint32_t t = atomicAdd(ctr, 1u);
      u = t < nh ? units[t] : (t - nh < nl ? units[n_units - nl + (t - nh)] : 0xFFFFFFFFu);
    }
    u = __shfl_sync(0xffffffffu, u, 0);
    if (u == 0xFFFFFFFFu) {
      if (lane == 0) un[us].valid = 0u;
      return;
    }
    const int64_t sg = u / ba.nbk;
    const int h = (int)(u % ba.nbk);
    const uint32_t p = segs[sg].p;
    const int64_t j = (int64_t)h * 32 + lane;
    un[us].ci[lane] = j < k_dst ? CI[sg * k_dst + j] : 0u;
    un[us].cr[lane] = (!BV && j < k_dst) ? CR[sg * k_dst + j] + G[(int64_t)p * k_dst + j] : 0u;
    if (lane == 0) {
      un[us].r0 = ba.SB[sg * (ba.nbk + 1) + h];
      un[us].r1 = ba.SB[sg * (ba.nbk + 1) + h + 1];
      un[us].p = p;
      un[us].h = (uint32_t)h;
      un[us].valid = 1u;
    }
  };
  // thread 0: bulk copy of the tile [x0, min(x0 + kBpTile, r1)) of unit slot us into buffer bf
  auto issue = [&](int bf, uint32_t x0, uint32_t r1) {
    const uint32_t xe = min(x0 + (uint32_t)kBpTile, r1);
    const uint32_t xa = x0 & ~1u, xb = (xe + 1) & ~1u;           // 16-byte aligned record range
    const uint32_t wa = x0 & ~3u, wb = (xe + 3) & ~3u;
    mbar_arrive_expect_tx(&bar[bf], (xb - xa) * 8 + (WEIGHTED ? (wb - wa) * 4 : 0));
    bulk_g2s(rbuf + bf * (kBpTile + 2), ba.rec + xa, (xb - xa) * 8, &bar[bf], policy_evict_first());
    if (WEIGHTED) bulk_g2s(wbuf + bf * (kBpTile + 4), ba.recw + wa, (wb - wa) * 4, &bar[bf], policy_evict_first());
  };
  // the first tile
  if (warp == 0) {
    claim(0);
    __syncwarp();
    if (lane == 0) {
      tile_s[0] = un[0].r0;
      tile_s[1] = 0;
      tile_s[2] = 1;
      tile_s[3] = un[0].valid;
      if (un[0].valid) issue(0, un[0].r0, un[0].r1);
    }
  }
  __syncthreads();
  uint32_t phase[2] = {0u, 0u};
  int bf = 0;
  for (;;) {
    const uint32_t x0 = tile_s[0], us = tile_s[1], first = tile_s[2];
    if (!tile_s[3]) break;
    const BpUnit& U = un[us];
    const uint32_t r1 = U.r1;
    if (first && tid < 32) {
      ciS[tid] = U.ci[tid];
      crS[tid] = U.cr[tid];
    }
    __syncthreads();                                 // everyone has read tile_s / the unit slot
    // next tile (same unit, or the first tile of a newly claimed unit) into the other buffer
    if (warp == 0) {
      uint32_t nx0 = x0 + kBpTile, nus = us, nfirst = 0, nvalid = 1;
      if (nx0 >= r1) {
        nus = us ^ 1;
        claim((int)nus);
        __syncwarp();
        nx0 = un[nus].r0;
        nfirst = 1;
        nvalid = un[nus].valid;
      }
      if (lane == 0) {
        if (nvalid) issue(bf ^ 1, nx0, un[nus].r1);
        tile_s[0] = nx0;
        tile_s[1] = nus;
        tile_s[2] = nfirst;
        tile_s[3] = nvalid;
      }
    }
    mbar_wait(&bar[bf], phase[bf]);
    phase[bf] ^= 1u;
    const uint64_t* rs = rbuf + bf * (kBpTile + 2) + (x0 & 1u);
    const float* wsv = wbuf + bf * (kBpTile + 4) + (x0 & 3u);
    const int base = warp * (kBpTile / kBpWarps);
    const uint32_t h = U.h, p = U.p;
    const uint32_t j0 = h * 32u;
    uint64_t rc[kBpItems];
    uint32_t rk[kBpItems];                          // rank among the warp's bin-j records | flagged rank << 16
    uint32_t cI = 0, cF = 0;                        // this warp's counts of bin `lane` so far
#pragma unroll
    for (int k = 0; k < kBpItems; ++k) {
      const int e = base + 32 * k + lane;
      const bool ok = x0 + (uint32_t)e < r1;
      rc[k] = ok ? rs[e] : ~0ull;
      const uint32_t jl = ok ? (uint32_t)(rc[k] >> 32) & 31u : 0u;   // invalid lanes: out of vm
      const uint32_t vm = __ballot_sync(0xffffffffu, ok);
      const uint32_t fb = __ballot_sync(0xffffffffu, ok && ((uint32_t)rc[k] & 0x8000u));
      uint32_t mb = vm;                             // lanes of bin `lane`
#pragma unroll
      for (int t = 0; t < 5; ++t) mb &= __ballot_sync(0xffffffffu, (jl >> t) & 1u) ^ sel[t];
      const uint32_t pm = __shfl_sync(0xffffffffu, mb, jl);   // lanes of my bin (lane jl's mask)
      const uint32_t bI = __shfl_sync(0xffffffffu, cI, jl), bF = __shfl_sync(0xffffffffu, cF, jl);
      rk[k] = (bI + __popc(pm & lt)) | ((bF + __popc(pm & fb & lt)) << 16);
      cI += __popc(mb);
      cF += __popc(mb & fb);
    }
    wI[warp][lane] = cI;
    wF[warp][lane] = cF;
    __syncthreads();
    if (kStaged) {
      // warp 0, lane = bin: per-warp bases within the bin's tile run, the bins' offsets in the
      // staging arrays, their global starts; then the running slots advance
      if (warp == 0) {
        uint32_t rI = 0, rF = 0;
#pragma unroll 4
        for (int ww = 0; ww < kBpWarps; ++ww) {
          const uint32_t a = wI[ww][lane], c = wF[ww][lane];
          wI[ww][lane] = rI;
          wF[ww][lane] = rF;
          rI += a;
          rF += c;
        }
        uint32_t sI = rI, sF = rF;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t yI = __shfl_up_sync(0xffffffffu, sI, o), yF = __shfl_up_sync(0xffffffffu, sF, o);
          if (lane >= o) {
            sI += yI;
            sF += yF;
          }
        }
        offI[lane] = sI - rI;
        offF[lane] = sF - rF;
        if (lane == 31) {
          offI[32] = sI;
          offF[32] = sF;
        }
        gI[lane] = ciS[lane];
        gF[lane] = crS[lane];
        ciS[lane] += rI;
        crS[lane] += rF;
      }
    } else {
      // bins kBpB w .. kBpB w + kBpB - 1: exclusive scans of the kBpWarps warps' counts
      // (segments of kBpWarps lanes), plus the bins' running slots
      constexpr int kBpB = 32 / kBpWarps;            // bins per warp
      const int ls = lane % kBpWarps;
      const int bin = kBpB * warp + lane / kBpWarps;
      const uint32_t a = wI[ls][bin], c = wF[ls][bin];
      uint32_t ia = a, ic = c;
#pragma unroll
      for (int o = 1; o < kBpWarps; o <<= 1) {
        const uint32_t ya = __shfl_up_sync(0xffffffffu, ia, o, kBpWarps);
        const uint32_t yc = __shfl_up_sync(0xffffffffu, ic, o, kBpWarps);
        if (ls >= o) {
          ia += ya;
          ic += yc;
        }
      }
      const uint32_t bI = ciS[bin], bF = crS[bin];
      wI[ls][bin] = bI + ia - a;
      wF[ls][bin] = bF + ic - c;
      __syncwarp();
      if (ls == kBpWarps - 1) {
        ciS[bin] = bI + ia;
        crS[bin] = bF + ic;
      }
    }
    __syncthreads();
    if (kStaged) {
#pragma unroll
      for (int k = 0; k < kBpItems; ++k) {
        if (rc[k] != ~0ull) {
          const uint32_t jl = (uint32_t)(rc[k] >> 32), pw = (uint32_t)rc[k];
          const uint32_t si = offI[jl] + wI[warp][jl] + (rk[k] & 0xFFFFu);
          stI[si] = (uint16_t)(pw & 0xFFFFu);
          tgI[si] = (uint8_t)jl;
          if (WEIGHTED) w[gI[jl] + wI[warp][jl] + (rk[k] & 0xFFFFu)] = wsv[base + 32 * k + lane];
          if (pw & 0x8000u) {
            const uint32_t sf = offF[jl] + wF[warp][jl] + (rk[k] >> 16);
            stF[sf] = (uint16_t)(pw >> 16);
            tgF[sf] = (uint8_t)jl;
          }
        }
      }
      __syncthreads();
      const uint32_t nI = offI[32], nF = offF[32];
      for (uint32_t x = tid; x < nI; x += kBpThreads) {
        const uint32_t jl = tgI[x];
        ids16[gI[jl] + (x - offI[jl])] = stI[x];
      }
      for (uint32_t x = tid; x < nF; x += kBpThreads) {
        const uint32_t jl = tgF[x];
        png16[gF[jl] + (x - offF[jl])] = stF[x];
      }
      __syncthreads();                               // staging / wI / wF / this buffer are reused
      bf ^= 1;
      continue;
    }
#pragma unroll
    for (int k = 0; k < kBpItems; ++k) {
      if (rc[k] != ~0ull) {
        const uint32_t jl = (uint32_t)(rc[k] >> 32), pw = (uint32_t)rc[k];
        const uint32_t pos = wI[warp][jl] + (rk[k] & 0xFFFFu);
        if (BV) {                                    // uncompressed bins: update slot = ID slot
          ba.upd[pos] = __uint_as_float(pw);
          continue;
        }
        ids16[pos] = (uint16_t)(pw & 0xFFFFu);
        if (WIDE) ids32[pos] = (((j0 + jl) << b) | (pw & qmask)) | ((pw & 0x8000u) ? 0x80000000u : 0u);
        if (WEIGHTED) w[pos] = wsv[base + 32 * k + lane];
        if (pw & 0x8000u) {
          const uint32_t pp = wF[warp][jl] + (rk[k] >> 16);
          png16[pp] = (uint16_t)(pw >> 16);
          if (WIDE) png32[pp] = (p << b) | (pw >> 16);
        }
      }
    }
    __syncthreads();                                 // wI / wF / this buffer are reused
    bf ^= 1;
  }
}

using BucketPlaceFn = void (*)(const uint32_t*, const uint32_t*, int64_t, uint32_t*, const BSeg*, int, int64_t,
                               const uint32_t*, const uint32_t*, const uint32_t*, const BucketArgs, uint16_t*,
                               uint32_t*, float*, uint16_t*, uint32_t*);
BucketPlaceFn bucket_place_fn(bool wide, bool weighted) {
  if (wide) return weighted ? k_bucket_place<true, true> : k_bucket_place<true, false>;
  return weighted ? k_bucket_place<false, true> : k_bucket_place<false, false>;
}

// Column prefix of a [rows x cols] count matrix, in place: cnt[r][c] <- sum_{r' < r} cnt[r'][c];
// col_tot[c] = the column total.  Block = 32 columns x 32 row slabs (coalesced over c).
__global__ void __launch_bounds__(1024) k_col_prefix(int64_t rows, int64_t cols, uint32_t* cnt, uint32_t* col_tot) {
  __shared__ uint32_t part[32][33];
  const int64_t c = blockIdx.x * 32 + threadIdx.x;
  const int y = threadIdx.y;
  const int64_t per = (rows + 31) / 32;
  const int64_t r0 = min(rows, y * per), r1 = min(rows, r0 + per);
  uint32_t sum = 0;
  if (c < cols)
    for (int64_t r = r0; r < r1; ++r) sum += cnt[r * cols + c];
  part[y][threadIdx.x] = sum;
  __syncthreads();
  if (y == 0) {
    uint32_t run = 0;
    for (int k = 0; k < 32; ++k) {
      const uint32_t t = part[k][threadIdx.x];
      part[k][threadIdx.x] = run;
      run += t;
    }
    if (c < cols) col_tot[c] = run;
  }
  __syncthreads();
  uint32_t run = part[y][threadIdx.x];
  if (c < cols)
    for (int64_t r = r0; r < r1; ++r) {
      const uint32_t t = cnt[r * cols + c];
      cnt[r * cols + c] = run;
      run += t;
    }
}

// Runs of partition p per bin j: RP[p][j] = sum over p's segments of CR[s][j]; CR
// becomes each segment's run offset inside group (p, j) (segments of p in row order).
__global__ void k_part_runs(int64_t k_src, int64_t k_dst, const uint32_t* __restrict__ seg_first, uint32_t* CR,
                            uint32_t* RP) {
  GRID_STRIDE(i, k_src * k_dst) {
    const int64_t p = i / k_dst, j = i % k_dst;
    uint32_t acc = 0;
    for (uint32_t sg = seg_first[p]; sg < seg_first[p + 1]; ++sg) {
      const uint32_t t = CR[(int64_t)sg * k_dst + j];
      CR[(int64_t)sg * k_dst + j] = acc;
      acc += t;
    }
    RP[i] = acc;
  }
}

__global__ void k_add_row_base(int64_t rows, int64_t cols, const uint32_t* __restrict__ base, uint32_t* m) {
  GRID_STRIDE(i, rows * cols) m[i] += base[i % cols];
}

// grp_at[c] = flat group g of PNG entry kPngChunk * c: the last g with G[g] <= x (empty
// groups share their start with the next one)
__global__ void k_grp_at_G(int64_t ep, const uint32_t* __restrict__ G, int64_t ng, int64_t n, uint32_t* grp_at) {
  GRID_STRIDE(c, n) {
    int64_t x = c * kPngChunk;
    if (x >= ep) x = ep - 1;
    int64_t lo = 0, hi = ng;                    // G[lo] <= x < G[hi] (G[ng] = ep > x)
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)G[mid] <= x) lo = mid;
      else hi = mid;
    }
    grp_at[c] = (uint32_t)lo;
  }
}

using SegPassFn = void (*)(const BSeg*, int, uint32_t*, const int64_t*, const uint32_t*, const float*, int, int64_t,
                           int64_t, uint32_t*, uint32_t*, const uint32_t*, uint32_t*, float*, unsigned long long*,
                           uint32_t*, uint16_t*, uint32_t*, float*, uint16_t*, uint32_t*);

template <bool PLACE>
SegPassFn seg_pass_fn(bool compress, bool wide, bool weighted) {
#define PCPM_SEG_FN(C, WI, WE) \
  if (compress == C && wide == WI && weighted == WE) return k_seg_pass<PLACE, C, WI, WE>;
  PCPM_SEG_FN(true, false, false) PCPM_SEG_FN(true, false, true) PCPM_SEG_FN(true, true, false)
  PCPM_SEG_FN(true, true, true) PCPM_SEG_FN(false, false, false) PCPM_SEG_FN(false, false, true)
  PCPM_SEG_FN(false, true, false) PCPM_SEG_FN(false, true, true)
#undef PCPM_SEG_FN
  return nullptr;
}

int build_layout_count(pcpm_handle* h, const pcpm_csr* csr, unsigned flags) {
  cudaStream_t s = h->stream;
  const int64_t n_src = csr->n_src, n_dst = csr->n_dst, m = csr->nnz;
  const int b = h->b;
  const int64_t q = int64_t(1) << b;
  const int64_t k_src = (n_src + q - 1) / q, k_dst = (n_dst + q - 1) / q;
  h->k_src = k_src;
  h->k_dst = k_dst;
  h->q = q;
  h->n_src = n_src;
  h->n_dst = n_dst;
  h->m = m;
  h->compressed = !(flags & PCPM_NO_COMPRESS);
  h->weighted = csr->values != nullptr || (flags & PCPM_KEEP_VALUES);
  h->wide = (flags & PCPM_WIDE_IDS) != 0;
  h->want_slots = (flags & PCPM_COMPACT_SLOTS) != 0;
  h->m_pad = ((m + kTileAlign - 1) / kTileAlign) * kTileAlign;
  if (h->m_pad == 0) h->m_pad = kTileAlign;
  const int64_t ng = k_src * k_dst;
  Temp tmp(s);
  PhaseTimer pt(s);
  int rc;

  // ---- inputs on the device (host CSR: one copy in, the passes need it twice)
  const int64_t* row_ptr = csr->row_ptr;
  const uint32_t* col = csr->col_idx;
  const float* values = csr->values;
  if (!is_device_ptr(row_ptr)) {
    int64_t* d;
    TK(tmp.alloc(&d, n_src + 1));
    TK(cudaMemcpyAsync(d, row_ptr, sizeof(int64_t) * (n_src + 1), cudaMemcpyHostToDevice, s));
    row_ptr = d;
  }
  if (!is_device_ptr(col)) {
    uint32_t* d;
    TK(tmp.alloc(&d, m));
    TK(cudaMemcpyAsync(d, col, sizeof(uint32_t) * m, cudaMemcpyHostToDevice, s));
    col = d;
  }
  if (values && !is_device_ptr(values)) {
    float* d;
    TK(tmp.alloc(&d, m));
    TK(cudaMemcpyAsync(d, values, sizeof(float) * m, cudaMemcpyHostToDevice, s));
    values = d;
  }

  // ---- partition boundaries (host): global checks and the segment plan
  std::vector<int64_t> pb(k_src + 1);
  TK(cudaMemcpy2DAsync(pb.data(), sizeof(int64_t), row_ptr, sizeof(int64_t) * q, sizeof(int64_t), k_src,
                       cudaMemcpyDeviceToHost, s));
  TK(cudaMemcpyAsync(&pb[k_src], row_ptr + n_src, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  TK(cudaStreamSynchronize(s));
  bool rp_ok = pb[0] == 0 && pb[k_src] == m;
  for (int64_t p = 0; p < k_src && rp_ok; ++p) rp_ok = pb[p] <= pb[p + 1];
  if (!rp_ok) {
    set_error(PCPM_EBADCSR, "row_ptr is not monotone, or row_ptr[0] != 0, or row_ptr[n_src] != nnz");
    return PCPM_EBADCSR;
  }
  // warp mode (PCPM_BUILD_COUNT_MODE=warp, A/B): one warp per segment; tile mode (default): one CTA
  const char* cmode = getenv("PCPM_BUILD_COUNT_MODE");
  const bool warp_mode = cmode && !strcmp(cmode, "warp");
  int64_t seg_target = warp_mode ? std::max<int64_t>(int64_t(1) << 16, m / ((int64_t)h->num_sms * kCntWarps * 3) + 1)
                                 : std::max<int64_t>(int64_t(1) << 16, m / ((int64_t)h->num_sms * 6) + 1);
  if (const char* e = getenv("PCPM_BUILD_SEG_EDGES")) seg_target = std::max<int64_t>(1, atoll(e));   // tests
  std::vector<BSeg> segs;
  std::vector<uint32_t> seg_first(k_src + 1);
  for (int64_t p = 0; p < k_src; ++p) {
    seg_first[p] = (uint32_t)segs.size();
    const int64_t u0 = p * q, u1 = std::min(n_src, u0 + q), rows = u1 - u0;
    int64_t ns = std::max<int64_t>(1, std::min<int64_t>((pb[p + 1] - pb[p] + seg_target - 1) / seg_target,
                                                        (rows + 31) / 32));
    const int64_t per = ((rows + ns - 1) / ns + 31) / 32 * 32;      // rows per segment, whole 32-row batches
    for (int64_t a = u0; a < u1; a += per)
      segs.push_back(BSeg{(uint32_t)a, (uint32_t)std::min(u1, a + per), (uint32_t)p, 0u});
  }
  seg_first[k_src] = (uint32_t)segs.size();
  const int64_t n_seg = (int64_t)segs.size();

  // ---- layout arrays owned by the handle
  uint32_t* ids32 = nullptr;
  if (h->wide) {
    if ((rc = dev_alloc_t(h, &h->ids, h->m_pad))) return rc;
    ids32 = h->ids;
    TK(cudaMemsetAsync(ids32 + m, 0, sizeof(uint32_t) * (h->m_pad - m), s));
  }
  if ((rc = dev_alloc_t(h, &h->ids16, h->m_pad))) return rc;
  TK(cudaMemsetAsync(h->ids16 + m, 0, sizeof(uint16_t) * (h->m_pad - m), s));
  if (h->weighted) {
    if ((rc = dev_alloc_t(h, &h->w, h->m_pad))) return rc;
    TK(cudaMemsetAsync(h->w + m, 0, sizeof(float) * (h->m_pad - m), s));
  }
  if ((rc = dev_alloc_t(h, &h->png_off, k_src * (k_dst + 1) + 4))) return rc;
  if ((rc = dev_alloc_t(h, &h->upd_off, ng + 4))) return rc;
  if ((rc = dev_alloc_t(h, &h->bin_id_start, k_dst + 1))) return rc;
  if ((rc = dev_alloc_t(h, &h->bin_upd_start, k_dst + 1))) return rc;
  if ((rc = dev_alloc_t(h, &h->chunk_base, h->m_pad / kChunkIds + 1))) return rc;
  if ((rc = dev_alloc_t(h, &h->outdeg, n_src))) return rc;
  if ((rc = dev_alloc_t(h, &h->inv_deg, n_src + 4))) return rc;

  // ---- scratch
  BSeg* d_segs;
  uint32_t *d_seg_first, *ctr, *err, *CI, *CR, *RP, *G, *col_tot;
  unsigned long long* d_dang;
  TK(tmp.alloc(&d_segs, n_seg));
  TK(tmp.alloc(&d_seg_first, k_src + 1));
  TK(tmp.alloc(&ctr, 4));
  TK(tmp.alloc(&err, 4));
  TK(tmp.alloc(&d_dang, 1));
  TK(tmp.alloc(&CI, n_seg * k_dst));
  TK(tmp.alloc(&CR, n_seg * k_dst));
  TK(tmp.alloc(&RP, ng + 1));
  TK(tmp.alloc(&G, ng + 1));
  TK(tmp.alloc(&col_tot, k_dst + 1));
  TK(cudaMemcpyAsync(d_segs, segs.data(), sizeof(BSeg) * n_seg, cudaMemcpyHostToDevice, s));
  TK(cudaMemcpyAsync(d_seg_first, seg_first.data(), sizeof(uint32_t) * (k_src + 1), cudaMemcpyHostToDevice, s));
  TK(cudaMemsetAsync(ctr, 0, 16, s));
  TK(cudaMemsetAsync(err, 0, 16, s));
  TK(cudaMemsetAsync(d_dang, 0, 8, s));
  pt.mark("count build: plan + allocations");

  const bool weighted_ids = h->weighted && values != nullptr;
  const size_t smem = warp_mode ? (size_t)kCntWarps * 2 * k_dst * sizeof(uint32_t) + kCntWarps * 32
                                : tile_smem_bytes(k_dst);
  const int kbits = std::max(1, bits_for((uint64_t)std::max<int64_t>(k_dst - 1, 0)));
  SegPassFn cnt_fn = seg_pass_fn<false>(h->compressed, h->wide, weighted_ids);
  SegPassFn place_fn = seg_pass_fn<true>(h->compressed, h->wide, weighted_ids);
  TilePassFn tcnt_fn = tile_pass_fn<false>(h->compressed, h->wide, weighted_ids);
  // two-level placement for many bins (PCPM_BUILD_ONE_LEVEL=1 keeps the one-level pass, A/B)
  const bool two_level = (!warp_mode && k_dst > kBucketMinK && !getenv("PCPM_BUILD_ONE_LEVEL")) || h->bvgas;
  TilePassFn tplace_fn = two_level ? tile_pass_fn<true, true>(h->compressed, h->wide, weighted_ids)
                                   : tile_pass_fn<true>(h->compressed, h->wide, weighted_ids);
  if (warp_mode) {
    TK(cudaFuncSetAttribute(cnt_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    TK(cudaFuncSetAttribute(place_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  } else {
    TK(cudaFuncSetAttribute(tcnt_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tile_smem_bytes(k_dst, 1)));
    TK(cudaFuncSetAttribute(tplace_fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)tile_smem_bytes(k_dst, two_level ? 2 : 0)));
  }
  const int grid = warp_mode
                       ? (int)std::max<int64_t>(1, std::min<int64_t>((n_seg + kCntWarps - 1) / kCntWarps, h->num_sms))
                       : (int)std::max<int64_t>(1, std::min<int64_t>(n_seg, h->num_sms));

  // ---- pass 1: counts, out-degrees, validation
  if (warp_mode)
    cnt_fn<<<grid, 32 * kCntWarps, smem, s>>>(d_segs, (int)n_seg, ctr, row_ptr, col, values, b, k_dst, n_dst, CI, CR,
                                              nullptr, h->outdeg, h->inv_deg, d_dang, err, nullptr, nullptr, nullptr,
                                              nullptr, nullptr);
  else
    tcnt_fn<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(n_seg, 2 * h->num_sms)), kTileThreads,
              tile_smem_bytes(k_dst, 1), s>>>(d_segs, (int)n_seg, ctr, row_ptr, col, values, b, k_dst, n_dst, kbits,
                                             CI, CR, nullptr, h->outdeg, h->inv_deg, d_dang, err, nullptr, nullptr,
                                             nullptr, nullptr, nullptr, BucketArgs{});
  TK(cudaGetLastError());
  uint32_t herr = 0;
  TK(cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, s));
  TK(cudaStreamSynchronize(s));
  if (herr & 1u) {
    set_error(PCPM_EBADCSR, "row_ptr is not monotone, or row_ptr[0] != 0, or row_ptr[n_src] != nnz");
    return PCPM_EBADCSR;
  }
  if (herr & 2u) {
    set_error(PCPM_EBADCSR, "col_idx has an entry >= n_dst");
    return PCPM_EBADCSR;
  }
  if (herr & 4u) {
    set_error(PCPM_EBADCSR, "a row's columns are not strictly increasing (sorted, deduplicated) (R6)");
    return PCPM_EBADCSR;
  }
  pt.mark("count build: pass 1 (count)");

  // ---- scans: ID bases per (segment, bin), PNG groups and run offsets
  k_col_prefix<<<(unsigned)((k_dst + 31) / 32), dim3(32, 32), 0, s>>>(n_seg, k_dst, CI, col_tot);
  TK(cudaMemsetAsync(col_tot + k_dst, 0, 4, s));
  if ((rc = scan_excl_u32(tmp, col_tot, h->bin_id_start, k_dst + 1, s))) return rc;
  k_add_row_base<<<grid_for(n_seg * k_dst), kT, 0, s>>>(n_seg, k_dst, h->bin_id_start, CI);
  k_part_runs<<<grid_for(ng), kT, 0, s>>>(k_src, k_dst, d_seg_first, CR, RP);
  TK(cudaMemsetAsync(RP + ng, 0, 4, s));
  if ((rc = scan_excl_u32(tmp, RP, G, ng + 1, s))) return rc;
  TK(cudaGetLastError());
  uint32_t hep = 0;
  TK(cudaMemcpyAsync(&hep, G + ng, 4, cudaMemcpyDeviceToHost, s));
  TK(cudaStreamSynchronize(s));
  const int64_t ep = (int64_t)hep;
  h->e_prime = ep;
  if (h->wide) {
    if ((rc = dev_alloc_t(h, &h->png_src, ep + 8))) return rc;
    TK(cudaMemsetAsync(h->png_src + ep, 0, sizeof(uint32_t) * 8, s));
  }
  if ((rc = dev_alloc_t(h, &h->png16, ep + 16))) return rc;
  TK(cudaMemsetAsync(h->png16 + ep, 0, sizeof(uint16_t) * 16, s));
  pt.mark("count build: scans");

  // ---- pass 2: place IDs (+ weights) and PNG sources
  TK(cudaMemsetAsync(ctr, 0, 4, s));
  BucketArgs ba{};
  if (two_level) {
    // records into (segment, bucket) sub-ranges, then each sub-range into its 32 bins
    const int nbk = (int)((k_dst + 31) / 32);
    const int64_t n_units = n_seg * nbk;
    uint32_t *SB, *units, *nhl;
    if (h->bvgas) {                                // the per-iteration scatter replays this placement
      if ((rc = dev_alloc_t(h, &SB, n_seg * (nbk + 1)))) return rc;
      if ((rc = dev_alloc_t(h, &units, n_units))) return rc;
      if ((rc = dev_alloc_t(h, &nhl, 4))) return rc;
      if ((rc = dev_alloc_t(h, &ba.rec, m + 2))) return rc;
      h->bv_SB = SB;
      h->bv_units = units;
      h->bv_nhl = nhl;
      h->bv_rec = ba.rec;
      h->bv_nbk = nbk;
    } else {
      TK(tmp.alloc(&SB, n_seg * (nbk + 1)));
      TK(tmp.alloc(&units, n_units));
      TK(tmp.alloc(&nhl, 4));
      TK(tmp.alloc(&ba.rec, m + 2));               // the bulk copies read whole 16-byte words
    }
    if (weighted_ids) TK(tmp.alloc(&ba.recw, m + 4));
    ba.SB = SB;
    ba.nbk = nbk;
    TK(cudaMemsetAsync(nhl, 0, 16, s));
    k_seg_buckets<<<(unsigned)n_seg, 1024, 0, s>>>(n_seg, k_dst, nbk, d_segs, row_ptr, CI, h->bin_id_start, SB);
    tplace_fn<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(n_seg, PCPM_TILE_BUCKET_CTAS * h->num_sms)),
                kTileThreads, tile_smem_bytes(k_dst, 2), s>>>(d_segs, (int)n_seg, ctr, row_ptr, col, values, b, k_dst,
                                                              n_dst, kbits,
                                               CI, CR, G, nullptr, nullptr, nullptr, nullptr, h->ids16, ids32, h->w,
                                               h->png16, h->wide ? h->png_src : nullptr, ba);
    TK(cudaGetLastError());
    pt.mark("count build: pass 2a (buckets)");
    k_bucket_units<<<grid_for(n_units), kT, 0, s>>>(n_units, nbk, SB, units, nhl);
    TK(cudaMemsetAsync(ctr, 0, 4, s));
    const size_t bpsm = bucket_place_smem(weighted_ids);
    TK(cudaFuncSetAttribute(bucket_place_fn(h->wide, weighted_ids), cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)bpsm));
    bucket_place_fn(h->wide, weighted_ids)<<<h->num_sms * PCPM_BP_CTAS, kBpThreads, bpsm, s>>>(
        units, nhl, n_units, ctr, d_segs, b, k_dst, CI, CR, G, ba, h->ids16, ids32, h->w, h->png16,
        h->wide ? h->png_src : nullptr);
  } else if (warp_mode)
    place_fn<<<grid, 32 * kCntWarps, smem, s>>>(d_segs, (int)n_seg, ctr, row_ptr, col, values, b, k_dst, n_dst, CI,
                                                CR, G, nullptr, nullptr, nullptr, nullptr, h->ids16, ids32, h->w,
                                                h->png16, h->wide ? h->png_src : nullptr);
  else
    tplace_fn<<<grid, kTileThreads, smem, s>>>(d_segs, (int)n_seg, ctr, row_ptr, col, values, b, k_dst, n_dst, kbits,
                                               CI, CR, G, nullptr, nullptr, nullptr, nullptr, h->ids16, ids32, h->w,
                                               h->png16, h->wide ? h->png_src : nullptr, ba);
  TK(cudaGetLastError());
  if (h->bvgas) {
    // keep what the per-iteration scatter needs: the CSR, the segment plan, the ID bases
    if ((rc = dev_alloc_t(h, &h->bv_rp, n_src + 1))) return rc;
    if ((rc = dev_alloc_t(h, &h->bv_col, m + 4))) return rc;
    if ((rc = dev_alloc(h, &h->bv_segs, sizeof(BSeg) * n_seg))) return rc;
    if ((rc = dev_alloc_t(h, &h->bv_CI, n_seg * k_dst))) return rc;
    TK(cudaMemcpyAsync(h->bv_rp, row_ptr, sizeof(int64_t) * (n_src + 1), cudaMemcpyDeviceToDevice, s));
    TK(cudaMemcpyAsync(h->bv_col, col, sizeof(uint32_t) * m, cudaMemcpyDeviceToDevice, s));
    TK(cudaMemcpyAsync(h->bv_segs, d_segs, sizeof(BSeg) * n_seg, cudaMemcpyDeviceToDevice, s));
    TK(cudaMemcpyAsync(h->bv_CI, CI, sizeof(uint32_t) * n_seg * k_dst, cudaMemcpyDeviceToDevice, s));
    h->bv_nseg = n_seg;
  }
  if (h->weighted && !values) {
    // PCPM_KEEP_VALUES without values: every weight is 1
    k_fill_f32<<<grid_for(m), kT, 0, s>>>(m, 1.0f, h->w);
    TK(cudaGetLastError());
  }
  pt.mark("count build: pass 2 (place)");

  if ((rc = dev_alloc_t(h, &h->upd, ep + 8))) return rc;
  TK(cudaMemsetAsync(h->upd + ep, 0, sizeof(float) * 8, s));   // the scatter writes [0, E') before any read
  {
    const int64_t nga = ep / kPngChunk + 64;     // the scatter copies aligned supersets
    if ((rc = dev_alloc_t(h, &h->grp_at, nga))) return rc;
    k_grp_at_G<<<grid_for(nga), kT, 0, s>>>(ep > 0 ? ep : 1, G, ng, nga, h->grp_at);
    TK(cudaGetLastError());
  }
  if (values) {
    float* mx;
    TK(tmp.alloc(&mx, 1));
    float hmx = 0.f;
    int rc2 = launch_absmax(h, values, m, mx, s);
    if (rc2) return rc2;
    TK(cudaMemcpyAsync(&hmx, mx, 4, cudaMemcpyDeviceToHost, s));
    TK(cudaStreamSynchronize(s));
    int ex = 0;
    if (hmx > 0.f) frexpf(hmx, &ex);
    h->wexp = ex;
    if ((rc2 = weighted_degrees(h, tmp, row_ptr, values))) return rc2;
  }
  return finish_layout(h, tmp, pt, G, d_dang);
}

}  // namespace

// Layout construction: the chunked sort (default) or the two-sort legacy path
// (PCPM_BUILD_LEGACY=1, and graphs without edges).
int build_layout(pcpm_handle* h, const pcpm_csr* csr, unsigned flags) {
  if (flags & PCPM_BVGAS) {
    // the BVGAS engine: uncompressed bins from the counting build, whose placement it replays
    const int64_t q = int64_t(1) << h->b;
    if (csr->n_src != csr->n_dst || csr->values || (flags & (PCPM_WIDE_IDS | PCPM_KEEP_VALUES | PCPM_BUILD_PULL)) ||
        csr->nnz == 0 || (csr->n_dst + q - 1) / q > kCountMaxK) {
      set_error(PCPM_EINVAL, "PCPM_BVGAS needs a square, unweighted graph with edges, the compact layout and "
                             "k <= 2048 partitions");
      return PCPM_EINVAL;
    }
    h->bvgas = true;
    return build_layout_count(h, csr, flags | PCPM_NO_COMPRESS);
  }
  const bool legacy = getenv("PCPM_BUILD_LEGACY") != nullptr;
  // q = 2^16 (pair handles): only the two-sort path carries 16-bit local IDs (its keys and
  // payloads are whole 4-byte IDs; the other builds pack local ID, flag and source in 32 bits)
  if (legacy || h->pair || csr->nnz == 0 || csr->n_src <= 0 || csr->n_dst <= 0) return build_layout_legacy(h, csr, flags);
  // the counting construction (default) unless the pull CSC is wanted or the bins are too many
  const char* mode = getenv("PCPM_BUILD");                   // "sort": the chunked sort (A/B)
  const int64_t q = int64_t(1) << h->b, k_dst = (csr->n_dst + q - 1) / q;
  // host CSRs take the chunked sort, whose chunks sort while the next ones upload (the H2D
  // hides the build); "count" forces the counting construction (A/B, tests)
  const bool host_in = !is_device_ptr(csr->col_idx) || !is_device_ptr(csr->row_ptr);
  const bool force_count = mode && !strcmp(mode, "count");
  if (!(mode && !strcmp(mode, "sort")) && !(flags & PCPM_BUILD_PULL) && k_dst <= kCountMaxK &&
      (!host_in || force_count))
    return build_layout_count(h, csr, flags);
  return csr->values ? build_layout_chunked<PayW>(h, csr, flags) : build_layout_chunked<uint32_t>(h, csr, flags);
}

// BVGAS scatter (Alg. 3 lines 1-5): every edge (u, v) of the kept CSR inserts
// x[u] into bin v >> b at its insertion point -- the counting build's two-level placement
// replayed on values (records carry x[u]; the ranks, hence the slots, are the build's).
int launch_bvgas_scatter(pcpm_handle* h, const float* x, cudaStream_t s) {
  if (!h->bvgas) {
    set_error(PCPM_ESTATE, "not a BVGAS handle");
    return PCPM_ESTATE;
  }
  BucketArgs ba{};
  ba.SB = h->bv_SB;
  ba.nbk = h->bv_nbk;
  ba.rec = h->bv_rec;
  ba.xval = x;
  ba.upd = h->upd;
  const int64_t n_units = h->bv_nseg * h->bv_nbk;
  const int kbits = std::max(1, bits_for((uint64_t)std::max<int64_t>(h->k_dst - 1, 0)));
  const size_t smem = tile_smem_bytes(h->k_dst, 2);
  TilePassFn f = k_tile_pass<true, false, false, false, true, true>;
  PCPM_CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const BSeg* segs = static_cast<const BSeg*>(h->bv_segs);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(h->bv_nseg, PCPM_TILE_BUCKET_CTAS * h->num_sms));
  PCPM_CK(cudaMemsetAsync(h->bv_nhl + 2, 0, 8, s));
  f<<<grid, kTileThreads, smem, s>>>(segs, (int)h->bv_nseg, h->bv_nhl + 2, h->bv_rp, h->bv_col, nullptr, h->b,
                                     h->k_dst, h->n_dst, kbits, nullptr, nullptr, nullptr, nullptr, nullptr,
                                     nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, ba);
  PCPM_CK(cudaGetLastError());
  const size_t bpsm = bucket_place_smem(false);
  auto g = k_bucket_place<false, false, true>;
  PCPM_CK(cudaFuncSetAttribute(g, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bpsm));
  g<<<h->num_sms * PCPM_BP_CTAS, kBpThreads, bpsm, s>>>(h->bv_units, h->bv_nhl, n_units, h->bv_nhl + 3, segs, h->b,
                                                        h->k_dst, h->bv_CI, nullptr, nullptr, ba, nullptr,
                                                        nullptr, nullptr, nullptr, nullptr);
  PCPM_CK(cudaGetLastError());
  h->launches += 2;
  return PCPM_OK;
}

// Claim order of the scatter items.  Default (opt_scatter_lpt = 0): ascending p, so the
// ~148 items in flight are consecutive source partitions that write bin j at about the
// same time -- the boundary sectors between group (p, j) and (p+1, j) are completed in L2
// instead of being written back partially.  1: largest first (LPT).
int order_scatter_items(pcpm_handle* h, cudaStream_t s) {
  std::vector<ScatterItem> si(h->n_sitems);
  if (si.empty()) return PCPM_OK;
  TK(cudaMemcpyAsync(si.data(), h->sitems, sizeof(ScatterItem) * si.size(), cudaMemcpyDeviceToHost, s));
  TK(cudaStreamSynchronize(s));
  // natural order: (p, j0) ascending; LPT: largest first, ties in natural order
  std::sort(si.begin(), si.end(),
            [](const ScatterItem& a, const ScatterItem& c) { return a.p != c.p ? a.p < c.p : a.j0 < c.j0; });
  if (h->opt_scatter_lpt)
    std::stable_sort(si.begin(), si.end(), [](const ScatterItem& a, const ScatterItem& c) { return a.pad > c.pad; });
  if (!si.empty())
    TK(cudaMemcpyAsync(h->sitems, si.data(), sizeof(ScatterItem) * si.size(), cudaMemcpyHostToDevice, s));
  TK(cudaStreamSynchronize(s));
  return PCPM_OK;
}

// Destination shard: the layout of the column slice [lo, hi) of the
// CSR (n_src rows, local columns v - lo), with the GLOBAL out-degrees of the
// sources (the slice's rows hold only the edges into the slice).
int build_shard_layout(pcpm_handle* h, const pcpm_csr* csr, int64_t lo, int64_t hi, unsigned flags) {
  cudaStream_t s = h->stream;
  const int64_t n = csr->n_src, m = csr->nnz;
  Temp tmp(s);
  const int64_t* row_ptr = csr->row_ptr;
  const uint32_t* col = csr->col_idx;
  const float* values = csr->values;
  if (!is_device_ptr(row_ptr)) {
    int64_t* d;
    TK(tmp.alloc(&d, n + 1));
    TK(cudaMemcpyAsync(d, row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s));
    row_ptr = d;
  }
  if (m > 0 && !is_device_ptr(col)) {
    uint32_t* d;
    TK(tmp.alloc(&d, m));
    TK(cudaMemcpyAsync(d, col, sizeof(uint32_t) * m, cudaMemcpyHostToDevice, s));
    col = d;
  }
  if (m > 0 && values && !is_device_ptr(values)) {
    float* d;
    TK(tmp.alloc(&d, m));
    TK(cudaMemcpyAsync(d, values, sizeof(float) * m, cudaMemcpyHostToDevice, s));
    values = d;
  }
  uint32_t* err;
  TK(tmp.alloc(&err, 4));
  TK(cudaMemsetAsync(err, 0, 16, s));
  k_check_rows<<<grid_for(n), kT, 0, s>>>(n, row_ptr, m, err);
  TK(cudaGetLastError());
  uint32_t herr = 0;
  TK(cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, s));
  TK(cudaStreamSynchronize(s));
  if (herr) {
    set_error(PCPM_EBADCSR, "row_ptr is not monotone, or row_ptr[0] != 0, or row_ptr[n_src] != nnz");
    return PCPM_EBADCSR;
  }
  int64_t *cnt, *first, *new_ptr;
  TK(tmp.alloc(&cnt, n + 1));
  TK(tmp.alloc(&first, n + 1));
  TK(tmp.alloc(&new_ptr, n + 1));
  TK(cudaMemsetAsync(cnt + n, 0, 8, s));
  if (m > 0) {
    k_slice_count<<<grid_for(n), kT, 0, s>>>(n, row_ptr, col, (uint32_t)lo, (uint32_t)hi, cnt, first);
    TK(cudaGetLastError());
  } else {
    TK(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * n, s));
  }
  {
    size_t bytes = 0;
    TK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt, new_ptr, n + 1, s));
    uint8_t* t;
    TK(tmp.alloc(&t, bytes));
    TK(cub::DeviceScan::ExclusiveSum(t, bytes, cnt, new_ptr, n + 1, s));
  }
  int64_t ms = 0;
  TK(cudaMemcpyAsync(&ms, new_ptr + n, 8, cudaMemcpyDeviceToHost, s));
  TK(cudaStreamSynchronize(s));
  uint32_t* scol;
  float* sval = nullptr;
  TK(tmp.alloc(&scol, ms));
  if (values) TK(tmp.alloc(&sval, ms));
  if (ms > 0) {
    k_slice_fill<<<grid_for(n * 32), kT, 0, s>>>(n, new_ptr, first, col, values, (uint32_t)lo, scol, sval);
    TK(cudaGetLastError());
  }
  pcpm_csr sub{};
  sub.n_src = n;
  sub.n_dst = hi - lo;
  sub.nnz = ms;
  sub.row_ptr = new_ptr;
  sub.col_idx = scol;
  sub.values = sval;
  int rc = build_layout(h, &sub, flags);
  if (rc) return rc;
  // global out-degrees and dangling count (build_layout saw only the slice's rows)
  unsigned long long* d_dang;
  TK(tmp.alloc(&d_dang, 1));
  TK(cudaMemsetAsync(d_dang, 0, 8, s));
  k_outdeg<<<grid_for(n), kT, 0, s>>>(0, n, row_ptr, h->outdeg, h->inv_deg, d_dang);
  TK(cudaGetLastError());
  unsigned long long hd = 0;
  TK(cudaMemcpyAsync(&hd, d_dang, 8, cudaMemcpyDeviceToHost, s));
  TK(cudaStreamSynchronize(s));
  h->n_dangling = (int64_t)hd;
  h->shard_lo = lo;
  h->n_global = csr->n_dst;
  return PCPM_OK;
}

}  // namespace pcpm

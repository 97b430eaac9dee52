// pcpm_internal.cuh -- shared internals of libpcpm.so (product path only).
// Handle layout, error plumbing, sm_100a PTX helpers (mbarrier, bulk async
// copy), and the launch-side declarations of the kernels in build.cu,
// scatter.cu, gather.cu and pull.cu.  See DESIGN.md for the data layout.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <utility>
#include <cstdio>
#include <string>
#include <vector>

#include "pcpm.h"

// #pragma unroll with a macro argument (A/B build knobs)
#define PCPM_STR_(x) #x
#define PCPM_UNROLL(n) _Pragma(PCPM_STR_(unroll n))

namespace pcpm {

// ---------------------------------------------------------------- constants
// Gather tile: kTileIds destination IDs per pipeline stage (the compact
// PageRank kernel uses 2x that), decoded by 16 or 32 consumer warps, each owning
// one sub-chunk whose update-index base comes from chunk_base (the global
// decode identity).  Bin slices are cut at kTileAlign multiples.
constexpr int kTileIds = 2048;
constexpr int kTileAlign = 4096;
constexpr int kChunkIds = 128;                         // chunk_base granularity
constexpr int kMaxPeers = 8;                           // fused exchange: SPR destinations besides spr_new
constexpr int kMaxBits = 15;                           // q <= 32768: 128 KB accumulator
// q = 2^16 ("pair" handles, DESIGN.md §6 "partition size"): the 256 KB accumulator of a
// destination partition does not fit one SM, so the gather runs every bin twice, as two
// items that each own one 2^15-vertex half of the partition and skip the other half's IDs
// (4-byte IDs only: a 16-bit local ID plus the run flag does not fit the 2-byte format)
constexpr int kMaxBitsPair = 16;
// SpMV fixed point (R22): F = kSpmvHead - ceil(log2 max|w|) - ceil(log2 max|x|), so every
// term |w x| 2^F <= 2^kSpmvHead of the signed 32-bit low word.  22 leaves 9 bits of headroom:
// the low word overflows (a carry into the global high word: a divergent, serialised path) once
// per >= 512 adds even when all terms have one sign; with 30 it overflowed on 0.7% of c5's adds
// and 60% of the 128-ID sub-chunks took the carry path (c5 gather 1.259 -> 0.793 ms).  The grid
// 2^-F is then 2^-23 of max|w| max|x|: the fp32 rounding of the largest products.
#ifndef PCPM_SPMV_HEAD
#define PCPM_SPMV_HEAD 22
#endif
constexpr int kSpmvHead = PCPM_SPMV_HEAD;
constexpr int kScatterThreads = 1024;
constexpr int kScatterMaxGroups = 2048;                // j-range of one scatter item (smem offsets)
constexpr int kPngChunk = 256;                         // grp_at granularity (scatter warp sub-ranges)

struct GatherItem {        // one slice [x0, x1) of destination bin j
  uint32_t j, x0, x1;
  uint32_t fx0, fx1;       // #flags in ids[0..x0), ids[0..x1)  (global decode identity)
  uint32_t pad[3];         // pad[0]: slot of a split bin's slice (0xFFFFFFFF if the bin is whole)
};
static_assert(sizeof(GatherItem) == 32, "GatherItem is 32 B");

struct ScatterItem {       // source partition p, destination groups [j0, j1)
  uint32_t p, j0, j1, pad;
};

// ---------------------------------------------------------------- handle
struct Graph {             // cached CUDA graph of one pcpm_pagerank configuration
  cudaGraphExec_t exec = nullptr;
  int iters = -1;
  double d = 0.0;
  float* out = nullptr;
  int kind = 0;
  int64_t launches = 0;
};

}  // namespace pcpm

struct pcpm_handle {
  int64_t n_src = 0, n_dst = 0, m = 0, m_pad = 0, e_prime = 0;
  int b = 0;
  int gb = 0;                        // partition bits of the gather's accumulator: min(b, kMaxBits)
  bool pair = false;                 // b = 16: two half-partition gather items per bin
  int64_t q = 0, k_src = 0, k_dst = 0, n_dangling = 0;
  bool weighted = false, compressed = true, has_pull = false;
  cudaStream_t stream = nullptr;
  int device = 0, num_sms = 148;
  double build_ms = 0.0;
  int fixed_bits = 0;
  int64_t launches = 0;
  int64_t device_bytes = 0;
  std::vector<void*> allocs;

  // destination shard (pcpm_build_shard): columns [shard_lo, shard_lo + n_dst) of an
  // n_global-column graph; outdeg holds the GLOBAL out-degrees of all n_src sources
  int64_t shard_lo = 0, n_global = 0;
  bool shard = false;

  // layout (device)
  bool wide = false;                // iterate on the 4-byte arrays (PCPM_WIDE_IDS)
  uint32_t* ids = nullptr;          // [m_pad] 4-byte IDs (wide handles only)
  uint16_t* ids16 = nullptr;        // [m_pad] compact IDs: local | flag << 15
  uint16_t* slot16 = nullptr;       // [n_dst] PCPM_COMPACT_SLOTS: accumulator slot of v (0xFFFF: no in-edges)
  int acc_words = 0;                // slots per partition (rounded up), 0 = q (no slots)
  uint2* slotmap = nullptr;         // [k_dst * q/32] per 32 vertices: (in-edge bits, slots before the word)
  bool want_slots = false;
  float* w = nullptr;               // [m_pad] or null
  uint32_t* png_src = nullptr;      // [E' (+pad)] 4-byte PNG sources (wide handles only)
  uint16_t* png16 = nullptr;        // [E' (+pad)] compact PNG sources: u & (q-1)
  uint32_t* png_off = nullptr;      // [k_src*(k_dst+1)]
  uint32_t* grp_at = nullptr;       // [E'/kPngChunk + 8] flat group p*k_dst + j of PNG entry kPngChunk*c
  uint32_t* upd_off = nullptr;      // [k_src*k_dst]
  uint32_t* bin_id_start = nullptr; // [k_dst+1]
  uint32_t* bin_upd_start = nullptr;// [k_dst+1]
  uint32_t* chunk_base = nullptr;   // [m_pad/kChunkIds + 1]
  uint32_t* outdeg = nullptr;       // [n_src]
  float* inv_deg = nullptr;         // [n_src] 1/|N_o(u)| (0 for dangling u), read by the apply
  float* inv_wdeg = nullptr;        // [n_src] 1/W(u), W(u) = sum of u's edge weights (0 if W(u) = 0); weighted
                                    // PageRank (R24), built when values are given
  int64_t n_wdangling = 0;          // #{u : W(u) = 0}
  int neg_weights = 0;              // some weight < 0 (SpMV only)
  float* upd = nullptr;             // [E' + 8]
  float* upd2 = nullptr;            // [E' + 8] second update-bin buffer of the fused iteration (lazy)
  pcpm::ScatterItem* sitems_split = nullptr;  // scatter items of the source partitions whose bin is split
  int n_sitems_split = 0;
  int wexp = 0;                     // max|w| <= 2^wexp (SpMV fixed-point scale)
  float* xmax = nullptr;            // [1] device max|x| of the last pcpm_spmv
  bool last_was_spmv = false;

  // BVGAS comparison engine (PCPM_BVGAS, Alg. 3): uncompressed bins, and a
  // per-iteration vertex-centric scatter over the kept CSR (build.cu launch_bvgas_scatter)
  bool bvgas = false;
  int64_t* bv_rp = nullptr;         // [n_src+1] the CSR (the scatter traverses it every iteration)
  uint32_t* bv_col = nullptr;       // [m]
  void* bv_segs = nullptr;          // [bv_nseg] segment plan of the counting build
  int64_t bv_nseg = 0;
  int bv_nbk = 0;                   // buckets of 32 bins
  uint32_t* bv_CI = nullptr;        // [bv_nseg * k_dst] first ID (= update) slot of (segment, bin)
  uint32_t* bv_SB = nullptr;        // [bv_nseg * (bv_nbk + 1)] record slots of (segment, bucket)
  uint32_t* bv_units = nullptr;     // [bv_nseg * bv_nbk] (segment, bucket) work list
  uint32_t* bv_nhl = nullptr;       // [4] heavy / light unit counts, claim counters
  uint64_t* bv_rec = nullptr;       // [m + 2] records (bucket pass -> bin pass)

  // pull comparison (CSC)
  uint32_t* in_ptr = nullptr;       // [n_dst+1]
  uint32_t* in_src = nullptr;       // [m]

  // work lists
  pcpm::GatherItem* gitems = nullptr;
  int n_gitems = 0;
  uint32_t* bin_nslices = nullptr;  // [k_dst]
  pcpm::ScatterItem* sitems = nullptr;
  int n_sitems = 0;
  // cluster gather (k_dst < SMs / 2): bin j's cl_cs slices are items [j * cl_cs, (j + 1) * cl_cs)
  pcpm::GatherItem* gitems_cl = nullptr;
  int cl_cs = 0;

  // iteration state
  float* pr[2] = {nullptr, nullptr};// [n]
  float* spr = nullptr;             // [n_src (+pad)]
  float* xbuf = nullptr;            // [n_src (+pad)] staging for host x
  float* ybuf = nullptr;            // [n_dst]      staging for host y / out
  uint32_t* slot_buf = nullptr;     // [n_slots * q] low words of the slices of split bins
  uint32_t* bin_slot_base = nullptr;// [k_dst] first slot of bin j's slices
  uint32_t n_slots = 0;
  uint32_t* bin_arrive = nullptr;   // [k_dst] slice arrival counters (kept zero)
  uint32_t* split_bins = nullptr;   // [n_split_bins] bins cut into slices (applied by k_apply_split)
  int n_split_bins = 0;
  uint32_t* hi = nullptr;           // [n_dst] fixed-point carry words (kept zero)
  uint32_t* counters = nullptr;     // [4] work counter, done counter (kept zero)
  unsigned long long* red_fx = nullptr;  // [2] fixed-point dangling mass / residual accumulators (kept zero)
  double* red = nullptr;            // [2*(red_cap)] D_t, res_t
  int red_cap = 0;
  int last_iters = 0;

  // options (pcpm_set_option)
  int opt_use_graph = 1;
  int opt_gather_variant = 1;
  int opt_cluster_gather = 1;       // 1: k_gather_cl for graphs with few partitions (when built), 0: off
  int opt_pdl = 1;                  // 1: scatter / gather / apply launched as programmatic dependents
  int opt_fuse = 0;                 // 1: gather + next scatter fused (PageRank, compact, square, not shard; measured slower), 0: off
  bool last_fused = false;          // the last pcpm_pagerank ran the fused iteration       // 1: in-line epilogue (k_gather), 2: apply overlapped through tensor memory (k_gather2)
  int opt_gather_pf = 2;            // gather: tiles prefetched into L2 ahead of the ring (0 = off)
  int opt_epi_pf = 4;               // gather: L2 prefetch of the apply's vertex arrays, tiles before the item's end (0 = off)
  int opt_scatter_variant = 0;      // 0: TMA-staged PNG stream (k_scatter_tma), 1: warp per group
  int opt_scatter_lpt = 0;          // scatter claim order: 0 ascending p, 1 largest first
  int opt_scatter_pf = 0;           // scatter: PNG stages prefetched into L2 ahead of the ring
  int opt_phase_timing = 0;
  int opt_phase_timing_saved = 0;
  double* res_host = nullptr;       // pinned: the residual read back by pcpm_pagerank_tol
  int opt_weighted_pr = 0;          // pcpm_pagerank uses the edge weights (R24)
  std::vector<cudaEvent_t> events;  // phase-timing events (created on demand)
  int n_events_used = 0;

  pcpm::Graph graph;
};

namespace pcpm {

// ---------------------------------------------------------------- errors
void set_error(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what, const char* file, int line);

#define PCPM_CK(call)                                                          \
  do {                                                                         \
    cudaError_t _e = (call);                                                   \
    if (_e != cudaSuccess) return ::pcpm::cuda_fail(_e, #call, __FILE__, __LINE__); \
  } while (0)

// allocate device memory owned by the handle
int dev_alloc(pcpm_handle* h, void** p, size_t bytes);
template <typename T>
int dev_alloc_t(pcpm_handle* h, T** p, size_t count) {
  return dev_alloc(h, reinterpret_cast<void**>(p), count * sizeof(T));
}
bool is_device_ptr(const void* p);
int launch_bvgas_scatter(pcpm_handle* h, const float* x, cudaStream_t s);   // build.cu

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// shared-memory atomic add at a 32-bit shared address, returning the old value
__device__ __forceinline__ uint32_t atoms_add_u32(uint32_t saddr, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(saddr), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D bulk async copy global -> shared (TMA engine, UBLKCP), completion on mbarrier.
// dst, src 16 B aligned; bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// bulk prefetch of [src, src + bytes) into L2 (TMA engine; no smem, no completion)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// Programmatic dependent launch (PDL): a kernel launched with the programmatic stream
// serialization attribute may start while its predecessor drains; pdl_wait() blocks until
// the predecessor grid has completed and its memory is visible (a no-op otherwise), and
// pdl_trigger() lets this grid's dependents start launching.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ uint32_t lanemask_le() {
  uint32_t r;
  asm("mov.u32 %0, %%lanemask_le;" : "=r"(r));
  return r;
}

// ---------------------------------------------------------------- tensor memory (tcgen05)
// The gather parks a finished partition's accumulator in TMEM (256 KB per SM,
// 128 lanes x 512 columns of 32 bits) so dedicated apply warps can run Eq. 1 on it
// while the decoders accumulate the next partition in shared memory.  A TMEM
// address is (lane << 16) | column; warp w may access lanes 32 (w % 4) .. + 31.
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {   // one whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {    // the allocating warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// 32 lanes x 8 consecutive columns: thread l writes / reads lane (taddr.lane + l), columns c .. c+7
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr)
               : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Fixed-point reductions of the apply (dangling mass, L1 residual): every term is
// rounded once to 2^-62 and summed in u64 (exact, order-free), so the result does
// not depend on which warp or kernel variant applied which vertex.  Terms and sums
// are <= 2 (PR' <= 1), i.e. < 2^63.
constexpr double kRedScale = 4611686018427387904.0;     // 2^62
__device__ __forceinline__ unsigned long long red_fx(double x) { return __double2ull_rn(x * kRedScale); }

// ---------------------------------------------------------------- launchers
// <<<grid, block, smem, s>>>(args...) with the PDL attribute when pdl is set
template <typename... KArgs, typename... Args>
cudaError_t launch_k(bool pdl, void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t s,
                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
struct GatherArgs {
  const void* ids;         // uint16_t* (compact) or uint32_t* (wide)
  const uint16_t* slot16;  // accumulator slots (PCPM_COMPACT_SLOTS) or null
  int acc_words;           // accumulator words (q without slots)
  const uint2* slotmap;    // slots: (in-edge bits, slot prefix) per 32 vertices
  const float* w;
  const float* upd;
  const uint32_t* chunk_base;
  const GatherItem* items;
  int n_items;
  const uint32_t* bin_nslices;
  uint32_t* counters;      // [0] work, [1] done
  uint32_t* slot_buf;      // split bins: slice s of bin j writes its low words to slot_buf[(base_j + s) q ..]
  const uint32_t* bin_slot_base;
  int has_split;           // split bins exist: k_apply_split applies them and writes the reductions
  uint32_t* bin_arrive;    // [k_dst] slices arrived per split bin (reset by the last)
  uint32_t* hi;
  unsigned long long* red_fx;   // [2] dangling mass / residual of this launch, 2^-62 fixed point (kept zero)
  int b;                   // partition bits of the accumulator (h->gb)
  int pair;                // 1: item j is half (j & 1) of bin j >> 1 and adds only that half's IDs (b = 16)
  int64_t n_dst;
  int fbits;
  // PageRank epilogue
  double d, n;
  const double* red_in;    // D_t at red_in[0]
  double* res_out;         // L1 residual of this iteration
  double* dang_out;        // dangling mass of the new vector (D_{t+1})
  const float* inv_deg;    // 1/outdeg of the destinations (0 = dangling)
  const float* pr_old;
  float* pr_new;
  float* spr_new;
  // SpMV epilogue
  float* y;
  const float* xmax;       // device max|x| of this call (fixed-point scale)
  int wexp;                // max|w| <= 2^wexp
  int pf_tiles;            // L2 prefetch distance of the gather producer, in tiles
  int static_items;        // 1: CTA b processes items[b] only (the cluster gather), 0: claim from counters[0]
  // fused scatter (FUSE instantiations, DESIGN.md §5 "fused iteration"): after applying
  // destination partition j, the CTA scatters source partition p = j of the NEXT iteration
  // (Alg. 4) from the SPR values it just computed, into the other update-bin buffer
  float* upd_next;
  const uint16_t* png16;
  const uint32_t* png_off;
  const uint32_t* upd_off;
  const uint32_t* grp_at;
  int64_t k_dst;
  int epi_pf;              // prefetch inv_deg / pr_old of the item's partition this many tiles before its end
  // fused exchange (pcpm_shard_step_peers): SPR_{t+1} of the slice is also stored to
  // these (peer) buffers, indexed like spr_new
  float* spr_peer[kMaxPeers];
  int n_peer;
};
__device__ int spmv_fbits(float xmax, int wexp);
int launch_absmax(pcpm_handle* h, const float* x, int64_t n, float* out, cudaStream_t s);
int launch_gather(pcpm_handle* h, const GatherArgs& a, bool weighted, bool pagerank, cudaStream_t s,
                  bool multi = false, bool fuse = false);
int gather_smem_bytes(int b, bool wide, bool weighted);
bool gather_slots_fit(int b, int acc_words);   // the 6-stage slot kernel fits in shared memory

// x: the source vector; out: the update bins to write (nullptr = h->upd); split_only: only
// the items of source partitions whose destination bin is split (the fused iteration's rest)
int launch_scatter(pcpm_handle* h, const float* x, cudaStream_t s, float* out = nullptr, bool split_only = false);
int read_debug_counters(unsigned long long* out, int cap, bool reset);
int prepare_gather(pcpm_handle* h);
int prepare_scatter(pcpm_handle* h);
int launch_pr_init(pcpm_handle* h, float* pr0, float* spr, double* red, int red_n, double spr_scale, cudaStream_t s);
int launch_pr_init_weighted(pcpm_handle* h, float* pr0, float* spr, double* red, int red_n, float spr_scale,
                            cudaStream_t s);
int launch_pull_iteration(pcpm_handle* h, const float* spr_in, const float* pr_old, float* pr_new,
                          float* spr_out, double* red_t, double d, cudaStream_t s);
int build_layout(pcpm_handle* h, const pcpm_csr* csr, unsigned flags);
int order_scatter_items(pcpm_handle* h, cudaStream_t s);
int build_shard_layout(pcpm_handle* h, const pcpm_csr* csr, int64_t lo, int64_t hi, unsigned flags);
int launch_pr_init_slice(pcpm_handle* h, float* pr0, float* spr, double* dang0, double spr_scale, cudaStream_t s);

}  // namespace pcpm

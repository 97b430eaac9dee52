// gather.cu -- a2 + a3: the branch-avoiding gather of PAPER.md Alg. 5
// with the apply step of Eq. 1 / Alg. 2 fused into its
// epilogue, or the SpMV epilogue of §3.5.
//
// Alg. 5:  update_ptr += MSB(id);  id &= mask;  PR[id] += update_bins[p][update_ptr]
//
// GPU form:
//  * Persistent CTAs (one per SM, 128 KB accumulator = one destination
//    partition of q = 2^15 vertices in shared memory).  Work items are slices
//    of destination bins, largest first, claimed with an atomic counter.
//  * Warps 0 and 1 are the producers (one per consumer group): for each tile a producer
//    issues bulk async copies (TMA engine, cp.async.bulk) into a 4-stage ring:
//    the IDs (4096 2-byte IDs in the compact layout), the window of update
//    values they reference, and the decode anchors.
//  * 30 consumer warps in two groups of 15 that take alternate stages; each
//    warp decodes two 128-ID sub-chunks of a stage (the group rotates the
//    remaining two) in steps of 32 consecutive IDs (lane l takes ID 32 c + l).
//    The producer also prefetches the tiles (and, near an item's end, the
//    apply's vertex arrays) into L2 ahead of the ring.  The update pointer of Alg. 5
//    becomes a warp prefix count of MSB flags:
//    ptr = anchor + (flags of earlier steps) + popc(ballot & lanemask_le) - 1
//    (reading R5's -1 start), with no data-dependent branch; all loads and
//    atomics of a sub-chunk are independent, so they overlap.
//  * PageRank accumulates in 64-bit fixed point (F fractional bits): the low
//    word lives in shared memory and is updated with native 32-bit integer
//    ATOMS.ADD; the rare carries go to a global high word (a coarse smem bitmap
//    marks groups of 32 vertices that have one).  Integer sums are exact and
//    order-independent, so results are bit-reproducible (DESIGN.md
//    "accumulator": fp32 sums fail the 1e-5 bound at the scale-26 hubs, and
//    fp32 smem atomics are CAS loops on sm_100a).  SpMV uses the signed
//    ("balanced") variant of the same accumulator.
//  * Epilogue: PR' = (1-d)/n + d (acc + D/n) in fp64, stored fp32; SPR' =
//    fp32(PR') * fp32(1/outdeg) (<= 3 fp32 roundings, R23); per-item
//    dangling mass and L1 residual, reduced in fixed order by the last CTA.
//    Slices of split (heavy) bins store their low words to per-slice slot
//    buffers; k_apply_split sums the slots and applies those bins afterwards.
//  * Weighted PageRank (R24) and SpMV multiply each update by the edge weight before the
//    fixed-point add.  In the compact layout the decoders read the weights of a
//    sub-chunk straight from global memory (coalesced, addresses known before the IDs are
//    decoded, prefetched into L2 by the producer), so the ring holds the same 4096-ID tiles
//    as unweighted PageRank; with 4-byte IDs the weights are staged beside the IDs.
//  * The decode is bound by the shared-memory pipe (one random ATOMS per ID,
//    ~4.4 wavefronts per warp instruction), see DESIGN.md §6.
//  * q = 2^16 ("pair" handles, 4-byte IDs): the 256 KB accumulator of a partition does not
//    fit one SM, so every bin is gathered as two half bins: item j' = 2 j + h streams the whole
//    bin j, decodes every ID (all flags advance the update pointer) and adds only the IDs
//    whose bit 15 equals h; accumulator, apply and split-bin slices then work on 2 k
//    half-partitions of 2^15 vertices unchanged (a.b = 15, a.pair = 1).
#include <cstdlib>
#include <type_traits>

#include "pcpm_internal.cuh"

namespace pcpm {
namespace {

constexpr uint32_t kFlagLast = 1u, kFlagEmpty = 2u, kFlagStop = 4u, kFlagScatter = 8u;
constexpr int kFusePng = 8192;                // PNG entries per scatter stage of the fused kernel (16 KB)

struct StageMeta {
  int item;
  uint32_t j;            // destination partition of the item
  uint32_t lo, hi;       // valid ID range of this tile [lo, hi)
  uint32_t tile_base;    // first ID position of the tile
  uint32_t win_base;     // update index of win[0]
  uint32_t flags;
  uint32_t pad;
};

#ifndef PCPM_GATHER_TILE_MODE
#define PCPM_GATHER_TILE_MODE 0     // 0: 4096 x 4 stages, 1: 8192 x 2, 2: 2048 x 8 (compact PageRank)
#endif
template <typename IdT, bool W, bool SL = false>
struct Cfg {
  static constexpr bool kCompact = sizeof(IdT) == 2;
  // compact PageRank (the hot configuration): 4096-ID tiles in a 4-stage ring,
  // 31 consumer warps each taking a 128-ID sub-chunk per stage (32 sub-chunks,
  // the extra one rotating; with the producer, 32 warps).  PCPM_GATHER_BIG_TILE
  // = 1 selects 8192-ID tiles double-buffered (2 x 48 KB; measured slower on
  // c4: 2.10 vs 1.98 ms).  Other variants: 2048-ID tiles, 16 warps of 128 IDs.
#ifndef PCPM_GATHER_WG
#define PCPM_GATHER_WG 1             // 0: weights staged in the ring with 2048-ID tiles (the earlier plan, A/B)
#endif
  // kWG: the edge weights are not staged in the ring; the decoders read them from global
  // memory (coalesced 128 B per step, the producer prefetches them into L2), which lets the
  // weighted compact configurations use the same 4096-ID tiles as unweighted PageRank
  static constexpr bool kWG = W && kCompact && PCPM_GATHER_WG != 0;
  static constexpr bool kHot = kCompact && (!W || kWG);
  static constexpr int kMode = kHot ? PCPM_GATHER_TILE_MODE : 0;
  static constexpr int kTile = kHot ? (kMode == 1 ? 4 * kTileIds : (kMode == 2 ? kTileIds : 2 * kTileIds)) : kTileIds;
#ifndef PCPM_GATHER_STAGES
#define PCPM_GATHER_STAGES 4
#endif
  // SL (accumulator slots, PCPM_COMPACT_SLOTS): the smaller accumulator leaves room for 6 stages
  static constexpr int kStages = SL ? 6 : (kMode == 1 ? 2 : (kMode == 2 ? 8 : (kHot ? PCPM_GATHER_STAGES : 4)));
  // Consumer warps form two groups that take alternate stages (group g: stages
  // g, g+2, ...), so each warp decodes two sub-chunks per stage it sees and the
  // per-stage bookkeeping is paid once per 2 sub-chunks; both groups run at once.
#ifndef PCPM_GATHER_COLD_WARPS
#define PCPM_GATHER_COLD_WARPS 31
#endif
  // producer warps: two (each fills the stages of one consumer group); measured against one
  // on the weighted / SpMV / 4-byte-ID configurations too
#ifndef PCPM_GATHER_PRODUCERS
#define PCPM_GATHER_PRODUCERS 2
#endif
#ifndef PCPM_GATHER_COLD_PRODUCERS
#define PCPM_GATHER_COLD_PRODUCERS 2
#endif
  static constexpr int kProducers = kHot ? PCPM_GATHER_PRODUCERS : PCPM_GATHER_COLD_PRODUCERS;
#ifndef PCPM_GATHER_HOT_WARPS
#define PCPM_GATHER_HOT_WARPS (32 - PCPM_GATHER_PRODUCERS)
#endif
  static constexpr int kWarps = kHot ? PCPM_GATHER_HOT_WARPS : (PCPM_GATHER_COLD_WARPS + 1 - PCPM_GATHER_COLD_PRODUCERS);
  static constexpr int kThreads = 32 * (kWarps + kProducers);
  static constexpr int kSub = kHot ? (kTile / 32 < kChunkIds ? kChunkIds : kTile / 32) : kChunkIds;   // IDs per sub-chunk
  static constexpr int kNsc = kTile / kSub;                // sub-chunks per tile
  static constexpr int kGroupA = (kWarps + 1) / 2;          // warps of group 0 (stages 0, 2)
  static constexpr int kGroupB = kWarps - kGroupA;          // warps of group 1 (stages 1, 3)
  static constexpr int kPer = kSub / 32;                   // decode steps of 32 IDs per sub-chunk
  static constexpr int kIdsBytes = kTile * (int)sizeof(IdT);
  static constexpr int kWinCap = kTile + 8;                // >= #flags + 1, 16 B aligned ends
  static constexpr int kWinBytes = kWinCap * 4;
  static constexpr int kWBytes = (W && !kWG) ? kTile * 4 : 0;
  static constexpr int kCbBytes = (kTile / kChunkIds) * 4;
  static constexpr int kStageBytes = kIdsBytes + kWinBytes + kWBytes + kCbBytes;
  static constexpr int kFlagShift = kCompact ? 15 : 31;
  static_assert(kTileAlign % kTile == 0, "slices are cut at tile multiples");
  static_assert(kSub % kChunkIds == 0 && kSub % 32 == 0, "sub-chunks start on decode anchors");
  static_assert(kThreads <= 1024 && kNsc >= kGroupA && kStages % 2 == 0, "launch shape");
  static_assert(kStageBytes % 16 == 0, "bulk copies need 16 B alignment");
};

__device__ __forceinline__ uint32_t ldcg_u32(const uint32_t* p) { return __ldcg(p); }
// streamed once: read-only path, no L1 allocation
__device__ __forceinline__ float ldg_stream_f32(const float* p) {
  float v;
  asm("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
}  // namespace

// Debug timing of the consumer warps (built with -DPCPM_GATHER_PROFILE=1 only):
// [0] cycles waiting for full stages, [1] decoding stages, [2] at the epilogue's
// first barrier, [3] in the epilogue, [4] warp count.  Read by pcpm_get_debug_counters.
__device__ unsigned long long g_gather_prof[24];   // [8..11]: producer (PCPM_GATHER_PROFILE)
#ifndef PCPM_GATHER_PROFILE
#define PCPM_GATHER_PROFILE 0
#endif
// Timing-only experiment builds (results are wrong): NOOP = consumers release
// stages without decoding (the producer's streaming rate); NO_EPI = skip the apply.
#ifndef PCPM_GATHER_NOOP
#define PCPM_GATHER_NOOP 0
#endif
#ifndef PCPM_GATHER_NO_EPI
#define PCPM_GATHER_NO_EPI 0
#endif
#ifndef PCPM_CARRY_CC
#define PCPM_CARRY_CC 1              // carry test with add.cc / addc (A/B: 0 = NOT + compare)
#endif
#ifndef PCPM_FINE_CARRY
#define PCPM_FINE_CARRY 1            // 1: carry bitmap of k_gather with 1 bit per 4 vertices (0: per 32, A/B)
#endif
#ifndef PCPM_APPLY_HI4
#define PCPM_APPLY_HI4 1             // 1: the vector apply reads a carried quad's high words with one 16-byte load (0: A/B)
#endif
#ifndef PCPM_GATHER_MATCH
#define PCPM_GATHER_MATCH 0          // 1: match.any aggregation of same-destination lanes before the ATOMS (A/B)
#endif
#ifndef PCPM_GATHER_ITEM_FENCE
#define PCPM_GATHER_ITEM_FENCE 0     // 1: fence after every item's reduction atomics (round-1 form, A/B)
#endif

__device__ int spmv_fbits(float xmax, int wexp) {
  int ex = 0;
  if (xmax > 0.0f) frexpf(xmax, &ex);          // xmax <= 2^ex
  const int F = kSpmvHead - wexp - ex;
  return F < -120 ? -120 : (F > 62 ? 62 : F);
}

namespace {

// fixed-point (dangling, residual) partials of one warp into the launch's totals (lane 0)
// (fence = false: the caller fences once before its completion count instead of per item;
// a per-item fence stalls each warp until its apply's stores are acknowledged)
__device__ __forceinline__ void warp_red_add(unsigned long long* red, unsigned long long dang, unsigned long long res,
                                             int lane, bool fence = true) {
  for (int o = 16; o; o >>= 1) {
    dang += __shfl_xor_sync(0xffffffffu, dang, o);
    res += __shfl_xor_sync(0xffffffffu, res, o);
  }
  if (lane == 0) {
    if (dang) atomicAdd(red, dang);
    if (res) atomicAdd(red + 1, res);
    if (fence) __threadfence();
  }
}
// after every partial is in: D_{t+1} and the residual as doubles, totals reset to zero
__device__ __forceinline__ void red_finish(const GatherArgs& a) {
  const unsigned long long dg = __ldcg(a.red_fx), rs = __ldcg(a.red_fx + 1);
  *a.dang_out = (double)dg / kRedScale;
  *a.res_out = (double)rs / kRedScale;
  a.red_fx[0] = 0ull;
  a.red_fx[1] = 0ull;
}

__global__ void k_absmax(int64_t n, const float* __restrict__ x, float* out) {
  float mx = 0.0f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    mx = fmaxf(mx, fabsf(x[i]));
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<int*>(out), __float_as_int(mx));  // mx >= 0
}

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ bool mbar_try_wait_hint(uint64_t* bar, uint32_t parity, uint32_t ns) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(ns)
      : "memory");
  return ok != 0;
}

// Producer-side apply (gather_variant 3, DESIGN.md §6 "producer apply"): at an item's end
// the decoders move the finished accumulator into tensor memory -- local vertex
// i = 64 c + 32 h + l in TMEM lane 32 h + l, column c (h = 0, 1: the lane quadrants of
// producer warps 0 and 1) -- zero the shared copy and go on with the next item; the two
// producer warps run Eq. 1 on it from TMEM (tcgen05.ld) whenever they would otherwise
// wait (for an empty ring stage or a claimed item).  One buffer: a handoff waits until
// both producers released the previous one (tempty).
struct PaRec {             // the item parked in TMEM (written by decoder 0)
  uint32_t j, nsl, slot, stop;
  uint32_t bm[32];         // carry bitmap of its accumulator (1 bit per 32 vertices)
};
struct PaCtx {
  PaRec* rec;
  uint64_t* tfull;         // decoders -> producers, 1 arrival
  uint64_t* tempty;        // producers -> decoders, 2 arrivals
  uint32_t tbase;          // TMEM base address (512 columns)
};

// Producer warp(s) of a gather CTA: claim work items and stream their tiles (IDs,
// update window, decode anchors, weights) into the ring of S stages with bulk async
// copies.  With NP = 2 producers, producer pg fills the stages of consumer group pg
// (stages pg, pg + 2, ...): both walk the same sequence of stage pushes and act on their
// own; producer 0 claims the items and hands them to producer 1 through a small shared
// queue (claimq / qbar), so the per-stage issue work (measured ~1.5k cycles per stage,
// DESIGN.md §6) is split over two warps.
template <typename C, typename IdT, bool W, bool PR, bool SL, bool FUSE = false, int NP = 1, bool PA = false>
__device__ __forceinline__ void gather_producer(const GatherArgs& a, const IdT* ids, uint8_t* stage_base,
                                                StageMeta* meta, uint64_t* full, uint64_t* empty, int lane,
                                                int pg = 0, uint32_t* claimq = nullptr, uint64_t* qbar = nullptr,
                                                const PaCtx* px = nullptr) {
  constexpr int S = C::kStages;
  static_assert(!PA || (NP == 2 && !SL && !FUSE), "producer apply: two producers, plain accumulator");
  static_assert(!FUSE || C::kStageBytes >= kFusePng * 2 + 256, "a scatter stage fits in a ring stage");
  static_assert(NP == 1 || (NP == 2 && S % 2 == 0), "two producers split the stages by parity");
  constexpr int kQ = 8;                            // claim queue depth (producers are < 3 items apart)
  // The window of tile t is fixed by two decode anchors (chunk_base at the
  // tile's ends).  Lanes load the anchors of 32 tiles at once, so the issue
  // loop carries no dependent global load per tile.
  const uint64_t pol = policy_evict_first();
  int stage = 0;
  uint32_t phase = 0;
  bool claimed = false;
  uint32_t nclaim = 0;
  unsigned long long pw = 0, pstages = 0, pcopy = 0, ploop = 0, pclaim = 0;   // PCPM_GATHER_PROFILE
  const long long pt0 = PCPM_GATHER_PROFILE ? clock64() : 0;
  // ---- producer apply (PA): state of the TMEM buffer this warp works on
  bool pa_have = false, pa_done = false;
  uint32_t pa_tph = 0, pa_col = 0;
  unsigned long long pa_dang = 0, pa_res = 0;     // 2^-62 fixed point (red_fx)
  double pa_base = 0.0, pa_spinv = 1.0;           // set after pdl_wait
  // one step: the next 8 TMEM columns of this warp's lane quadrant (256 vertices), or
  // nothing when no buffer is ready.  Warp-wide; block = wait for a buffer.
  auto pa_step = [&](bool block) {
    if constexpr (PA) {
      if (!pa_have) {
        if (pa_done) return;
        uint32_t ok = 1;
        if (block) {
          mbar_wait(px->tfull, pa_tph);
        } else {
          if (lane == 0) ok = mbar_test(px->tfull, pa_tph) ? 1u : 0u;
          ok = __shfl_sync(0xffffffffu, ok, 0);
        }
        if (!ok) return;
        tmem_fence_after();
        pa_col = 0;
        if (px->rec->stop) {
          pa_done = true;
          return;
        }
        pa_have = true;
      }
      const PaRec& H = *px->rec;
      const uint32_t q = 1u << a.b;
      const uint32_t v0 = H.j << a.b;
      const uint32_t cnt = (uint32_t)min((int64_t)q, a.n_dst - (int64_t)v0);
      const uint32_t nsl = H.nsl;
      const uint32_t ib = 32u * (uint32_t)pg + (uint32_t)lane;     // i = 64 c + ib
      uint32_t r[8];
      tmem_ld8(px->tbase + ((32u * (uint32_t)pg) << 16) + pa_col, r);
      if (nsl > 1) {
        // a slice of a split bin: its low words to its slot buffer (k_apply_split applies)
        uint32_t* sbuf = a.slot_buf + (size_t)H.slot * (size_t)q;
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 8; ++k) __stcg(sbuf + ((pa_col + k) << 6) + ib, r[k]);
      } else {
        float idg[8], po[8];
        if constexpr (PR) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t i = ((pa_col + k) << 6) + ib;
            idg[k] = i < cnt ? __ldg(a.inv_deg + v0 + i) : 0.0f;
            po[k] = i < cnt ? __ldg(a.pr_old + v0 + i) : 0.0f;
          }
        }
        tmem_wait_ld();
        const float fscale = __uint_as_float((uint32_t)(127 + a.fbits) << 23);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t i = ((pa_col + k) << 6) + ib;
          if (i >= cnt) continue;
          const uint32_t v = v0 + i;
          uint64_t tot = PR ? (uint64_t)r[k] : (uint64_t)(long long)(int32_t)r[k];
          if ((H.bm[i >> 10] >> ((i >> 5) & 31)) & 1u) {
            tot += (uint64_t)ldcg_u32(&a.hi[v]) << 32;
            a.hi[v] = 0u;
          }
          if constexpr (PR) {
            const double prn = pa_base + a.d * ((double)(long long)tot * __longlong_as_double((long long)(1023 - a.fbits) << 52));
            const float pn = (float)prn;
            a.pr_new[v] = pn;
            a.spr_new[v] = pn * idg[k] * fscale;      // SPR * 2^F (R23)
            if (idg[k] == 0.0f) pa_dang += red_fx(prn);
            pa_res += red_fx(fabs(prn - (double)po[k]));
          } else {
            a.y[v] = (float)((double)(long long)tot * pa_spinv);
          }
        }
      }
      pa_col += 8;
      if (pa_col >= (q >> 6) || (nsl <= 1 && (pa_col << 6) >= cnt)) {   // buffer done: release it
        tmem_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(px->tempty);
        pa_have = false;
        pa_tph ^= 1u;
      }
    }
  };
  // warp-wide wait for phase `parity` of bar, applying while it is not complete (PA)
  auto pa_wait = [&](uint64_t* bar, uint32_t parity) {
    if constexpr (PA) {
      for (;;) {
        uint32_t ok = 0;
        // no apply work in hand: suspend on the barrier (up to ~0.5 us) instead of spinning
        // on the decoders' issue slots, then look for a parked item
        if (lane == 0) ok = (pa_have ? mbar_test(bar, parity) : mbar_try_wait_hint(bar, parity, 500u)) ? 1u : 0u;
        if (__shfl_sync(0xffffffffu, ok, 0)) break;
        pa_step(false);
      }
    }
  };
  auto own = [&]() -> bool { return NP == 1 || (stage & 1) == pg; };
  auto advance = [&]() { if (++stage == S) { stage = 0; phase ^= 1; } };
  auto wait_empty = [&]() {
    if (PCPM_GATHER_PROFILE) {
      const long long t = clock64();
      mbar_wait(&empty[stage], phase ^ 1);
      pw += clock64() - t;
      ++pstages;
    } else {
      mbar_wait(&empty[stage], phase ^ 1);
    }
  };
  auto claim = [&]() -> uint32_t {
    const long long tc = PCPM_GATHER_PROFILE ? clock64() : 0;
    uint32_t v = 0;
    if (a.static_items) {                         // cluster gather: CTA b owns item b only
      v = claimed ? (uint32_t)a.n_items : blockIdx.x;
      claimed = true;
    } else {
      if (lane == 0) {
        if (NP == 1 || pg == 0) {
          v = atomicAdd(&a.counters[0], 1u);
          if (NP == 2) {
            claimq[nclaim % kQ] = v;
            mbar_arrive(&qbar[nclaim % kQ]);      // release: producer 1 reads claimq after its wait
          }
        } else if (!PA) {
          mbar_wait(&qbar[nclaim % kQ], (nclaim / kQ) & 1);
          v = claimq[nclaim % kQ];
        }
      }
      if constexpr (PA) {
        if (pg == 1) {                            // wait for producer 0's claim while applying
          pa_wait(&qbar[nclaim % kQ], (nclaim / kQ) & 1);
          if (lane == 0) v = claimq[nclaim % kQ];
        }
      }
      ++nclaim;
      v = __shfl_sync(0xffffffffu, v, 0);
    }
    if (PCPM_GATHER_PROFILE) pclaim += clock64() - tc;
    return v;
  };
  auto push_meta = [&](const StageMeta& m) {      // a stage without data (empty item / stop)
    if (PA && own()) pa_wait(&empty[stage], phase ^ 1);
    if (own() && lane == 0) {
      wait_empty();
      meta[stage] = m;
      mbar_arrive(&full[stage]);
    }
    __syncwarp();
    advance();
  };
  pdl_wait();                                      // the update bins (scatter) are complete
  if constexpr (PA) {
    if constexpr (PR) pa_base = (1.0 - a.d) / a.n + a.d * (a.red_in[0] / a.n);
    else pa_spinv = ldexp(1.0, -spmv_fbits(*a.xmax, a.wexp));
  }
  uint32_t it = claim();
  GatherItem item{};
  if (it < (uint32_t)a.n_items) item = a.items[it];
  for (;;) {
    if (it >= (uint32_t)a.n_items) {
      StageMeta m{};
      m.item = -1;
      m.flags = kFlagStop;
      push_meta(m);                              // one per consumer group
      push_meta(m);
      break;
    }
    // claim the next item now so its descriptor load overlaps this item's issue loop
    const uint32_t it_next = claim();
    GatherItem item_next{};
    if (it_next < (uint32_t)a.n_items) item_next = a.items[it_next];
    if (item.x0 == item.x1) {
      StageMeta m{};
      m.item = (int)it;
      m.j = item.j;
      m.flags = kFlagLast | kFlagEmpty;
      push_meta(m);                              // both groups run the item's epilogue
      push_meta(m);
    } else {
      const uint32_t t0 = item.x0 / C::kTile, t1 = (item.x1 - 1) / C::kTile;
      for (uint32_t tb0 = t0; tb0 <= t1; tb0 += 32) {
        const uint32_t tl = tb0 + lane;
        uint32_t fa = 0, fb = 0;                 // #flags before the tile's first / after its last ID
        if (tl <= t1) {
          const uint32_t tb = tl * C::kTile;
          fa = (tl == t0) ? item.fx0 : __ldg(a.chunk_base + tb / kChunkIds);
          fb = (tl == t1) ? item.fx1 : __ldg(a.chunk_base + (tb + C::kTile) / kChunkIds);
        }
        const uint32_t nb = min(32u, t1 - tb0 + 1);
        const uint32_t pf = (uint32_t)a.pf_tiles;
        // L2 prefetch of the batch's first pf tiles (the ring then loads them from L2)
        if (pf && lane < nb && lane < pf && (NP == 1 || ((stage + lane) & 1) == pg)) {
          const uint32_t alo = (fa > 0 ? fa - 1 : 0) & ~3u, ahi = (fb + 3) & ~3u;
          bulk_prefetch_l2(ids + tl * C::kTile, C::kIdsBytes);
          if (ahi > alo) bulk_prefetch_l2(a.upd + alo, (ahi - alo) * 4);
          if constexpr (C::kWG) bulk_prefetch_l2(a.w + tl * C::kTile, C::kTile * 4);
        }
        for (uint32_t k = 0; k < nb; ++k) {
          if (!own()) {                          // the other producer's stage
            advance();
            continue;
          }
          const long long tk0 = PCPM_GATHER_PROFILE ? clock64() : 0;
          const uint32_t flo = __shfl_sync(0xffffffffu, fa, k);
          const uint32_t fhi = __shfl_sync(0xffffffffu, fb, k);
          // keep the L2 prefetch pf tiles ahead of the ring (within the batch)
          if (pf && lane == k + pf && lane < nb) {
            const uint32_t alo = (fa > 0 ? fa - 1 : 0) & ~3u, ahi = (fb + 3) & ~3u;
            bulk_prefetch_l2(ids + tl * C::kTile, C::kIdsBytes);
            if (ahi > alo) bulk_prefetch_l2(a.upd + alo, (ahi - alo) * 4);
            if constexpr (C::kWG) bulk_prefetch_l2(a.w + tl * C::kTile, C::kTile * 4);
          }
          if constexpr (PR) {
            // the apply's vertex arrays of partition j into L2 a few tiles before the epilogue
            if (a.epi_pf && lane == 0 && tb0 + k == (t1 > t0 + (uint32_t)a.epi_pf ? t1 - (uint32_t)a.epi_pf : t0)) {
              const int64_t v0 = (int64_t)item.j << a.b;
              const uint32_t vb = (uint32_t)(min(int64_t(1) << a.b, a.n_dst - v0) * 4) & ~15u;
              if (vb) {
                bulk_prefetch_l2(a.inv_deg + v0, vb);
                bulk_prefetch_l2(a.pr_old + v0, vb);
                if (SL) bulk_prefetch_l2(a.slotmap + v0 / 32, vb / 16);   // q/32 uint2 = q/4 bytes
              }
            }
          }
          if constexpr (PA) pa_wait(&empty[stage], phase ^ 1);
          if (lane == 0) {
            const uint32_t t = tb0 + k;
            const uint32_t tb = t * C::kTile;
            const uint32_t wlo = flo > 0 ? flo - 1 : 0;   // the first ID may continue the previous run
            const uint32_t alo = wlo & ~3u, ahi = (fhi + 3) & ~3u;
            wait_empty();
            StageMeta m{};
            m.item = (int)it;
            m.j = item.j;
            m.lo = max(tb, item.x0);
            m.hi = min(tb + C::kTile, item.x1);
            m.tile_base = tb;
            m.win_base = alo;
            // the item's final stage of EACH group is flagged Last: tiles t1 and t1 - 1
            m.flags = (t + 1 >= t1 + (t1 > t0 ? 0u : 1u)) ? kFlagLast : 0u;
            meta[stage] = m;
            uint8_t* sb = stage_base + stage * C::kStageBytes;
            const uint32_t win_bytes = (ahi - alo) * 4;
            const long long tc0 = PCPM_GATHER_PROFILE ? clock64() : 0;
            mbar_arrive_expect_tx(&full[stage], C::kIdsBytes + win_bytes + C::kCbBytes + C::kWBytes);
            bulk_g2s(sb, ids + tb, C::kIdsBytes, &full[stage], pol);
            bulk_g2s(sb + C::kIdsBytes, a.upd + alo, win_bytes, &full[stage], pol);
            bulk_g2s(sb + C::kIdsBytes + C::kWinBytes + C::kWBytes, a.chunk_base + tb / kChunkIds, C::kCbBytes,
                     &full[stage], pol);
            if constexpr (W && !C::kWG) bulk_g2s(sb + C::kIdsBytes + C::kWinBytes, a.w + tb, C::kWBytes, &full[stage], pol);
            if (PCPM_GATHER_PROFILE) pcopy += clock64() - tc0;
          }
          __syncwarp();
          if (PCPM_GATHER_PROFILE) ploop += clock64() - tk0;
          advance();
        }
      }
      if (t1 == t0) {                             // single tile: the other group still needs its Last
        StageMeta m{};
        m.item = (int)it;
        m.j = item.j;
        m.flags = kFlagLast | kFlagEmpty;
        push_meta(m);
      }
    }
    if constexpr (FUSE) {
      // the next iteration's scatter of source partition p = j (Alg. 4): its PNG entries
      // [png_off[p][0], png_off[p][k]) in stages of kFusePng, each with the grp_at anchors
      // of its 256-entry chunks; every group's last scatter stage is flagged Last.  Slices
      // of split bins are scattered after k_apply_split instead (no stages here).
      if (a.bin_nslices[item.j] == 1) {
        const uint32_t p = item.j;
        const uint32_t s0 = __ldg(a.png_off + (int64_t)p * (a.k_dst + 1));
        const uint32_t s1 = __ldg(a.png_off + (int64_t)p * (a.k_dst + 1) + a.k_dst);
        const uint32_t base0 = s0 & ~(uint32_t)(kPngChunk - 1);
        const uint32_t nst = s1 > s0 ? (s1 - base0 + kFusePng - 1) / kFusePng : 0u;
        for (uint32_t c = 0; c < nst; ++c) {
          if (own() && lane == 0) {
            const uint32_t base = base0 + c * kFusePng;
            wait_empty();
            StageMeta m{};
            m.item = (int)it;
            m.j = p;
            m.lo = max(base, s0);
            m.hi = min(base + (uint32_t)kFusePng, s1);
            m.tile_base = base;
            const uint32_t c0 = base / kPngChunk, ca = c0 & ~3u;
            const uint32_t nga = ((((m.hi - base) + kPngChunk - 1) / kPngChunk) + (c0 - ca) + 3) & ~3u;
            m.win_base = c0 - ca;                  // grp_at of the stage's chunk 0 at word win_base
            m.flags = kFlagScatter | ((c + 2 >= nst + (nst > 1 ? 0u : 1u)) ? kFlagLast : 0u);
            meta[stage] = m;
            uint8_t* sb = stage_base + stage * C::kStageBytes;
            const uint32_t bytes = (((m.hi - base) * 2u) + 15u) & ~15u;    // png16 is padded
            mbar_arrive_expect_tx(&full[stage], bytes + nga * 4);
            bulk_g2s(sb, a.png16 + base, bytes, &full[stage], pol);
            bulk_g2s(sb + 2 * kFusePng, a.grp_at + ca, nga * 4, &full[stage], pol);   // grp_at padded
          }
          __syncwarp();
          advance();
        }
        for (uint32_t c = nst; c < 2; ++c) {      // empty PNG or a single stage: Last for the other group(s)
          StageMeta m{};
          m.item = (int)it;
          m.j = p;
          m.flags = kFlagScatter | kFlagLast | kFlagEmpty;
          push_meta(m);
        }
      }
    }
    it = it_next;
    item = item_next;
  }
  if constexpr (PA) {
    while (!pa_done) pa_step(true);               // the items still parked in TMEM
    if constexpr (PR) warp_red_add(a.red_fx, pa_dang, pa_res, lane, false);
  }
  if (PCPM_GATHER_PROFILE && lane == 0) {
    atomicAdd(&g_gather_prof[8], pw);
    atomicAdd(&g_gather_prof[9], (unsigned long long)(clock64() - pt0));
    atomicAdd(&g_gather_prof[10], pstages);
    atomicAdd(&g_gather_prof[11], 1ull);
    atomicAdd(&g_gather_prof[12], pcopy);
    atomicAdd(&g_gather_prof[13], ploop);
    atomicAdd(&g_gather_prof[14], pclaim);
  }
}

// Fused scatter: one PNG stage of source partition p (Alg. 4) by one consumer warp of its
// group: sub-ranges gw, gw + gsz, ... of 256 entries (plus its turn of the rotating
// remainder); upd_next[upd_off[p][j] + t] = xs[u] with the partition's SPR values xs in
// shared memory.  Offsets are read through L1 on group crossings.  Out of line so the
// decode loop's register allocation is not disturbed.
__device__ __noinline__ void fused_scatter_stage(const GatherArgs& a, const StageMeta& m, const uint8_t* sb,
                                                 const float* xs, int gw, int gsz, int& rot, int lane) {
  const uint16_t* ps = reinterpret_cast<const uint16_t*>(sb);
  const uint32_t* gs = reinterpret_cast<const uint32_t*>(sb + 2 * kFusePng) + m.win_base;
  const uint32_t p = m.j;
  const uint32_t* offs = a.png_off + (int64_t)p * (a.k_dst + 1);
  const uint32_t* uos = a.upd_off + (int64_t)p * a.k_dst;
  const uint32_t gbase = p * (uint32_t)a.k_dst;
  auto range = [&](const int sr) {
    const uint32_t wb = m.tile_base + (uint32_t)(sr * kPngChunk);
    const uint32_t wlo = max(wb, m.lo), whi = min(wb + (uint32_t)kPngChunk, m.hi);
    if (wlo >= whi) return;
    const int32_t ga = (int32_t)(gs[sr] - gbase);
    uint32_t g = ga > 0 ? (uint32_t)ga : 0u;
    uint32_t gend = __ldg(offs + g + 1);
    uint32_t delta = __ldg(uos + g) - __ldg(offs + g);
#pragma unroll 4
    for (uint32_t e = wlo + lane; e < whi; e += 32) {
      if (e >= gend) {
        do {
          ++g;
          gend = __ldg(offs + g + 1);
        } while (e >= gend);
        delta = __ldg(uos + g) - __ldg(offs + g);
      }
      a.upd_next[e + delta] = xs[ps[e - m.tile_base]];
    }
  };
  constexpr int kNsr = kFusePng / kPngChunk;
  const int nmain = (kNsr / gsz) * gsz;
  for (int sr = gw; sr < nmain; sr += gsz) range(sr);
  int who = rot;
  for (int sr = nmain; sr < kNsr; ++sr) {
    if (gw == who) range(sr);
    who = (who + 1 == gsz) ? 0 : who + 1;
  }
  rot = who;
}

// Carry bitmap: which accumulator words have a nonzero global high word.  Coarse: 1 bit per
// 32 vertices (q / 1024 words); FINE (k_gather): 1 bit per 4 vertices (q / 128 words = 1 KB),
// so the apply, which takes 4 vertices per thread, reads a.hi only for the quads that carried
// -- with the coarse map ~10% of c4's vertices took that latency-bound path.
template <bool FINE>
__device__ __forceinline__ void carry_mark(uint32_t* bitmap, uint32_t li) {
  if (FINE) atomicOr(&bitmap[li >> 7], 1u << ((li >> 2) & 31));
  else atomicOr(&bitmap[li >> 10], 1u << ((li >> 5) & 31));
}
template <bool FINE>
__device__ __forceinline__ bool carry_test(const uint32_t* bitmap, uint32_t i) {
  return FINE ? ((bitmap[i >> 7] >> ((i >> 2) & 31)) & 1u) != 0u : ((bitmap[i >> 10] >> ((i >> 5) & 31)) & 1u) != 0u;
}

// Decode of one full stage by one consumer warp (Alg. 5): the
// warp takes sub-chunks gw, gw + gsz, ... of the stage's tile (plus its turn of the
// rotating remainder) and adds each ID's update into the shared accumulator.
template <typename C, typename IdT, bool W, bool PR, bool FINE = false>
__device__ __forceinline__ void decode_stage(const GatherArgs& a, const StageMeta& m, const uint8_t* sb,
                                             uint32_t* acc, uint32_t* bitmap, const int gw, const int gsz,
                                             int& rot, const uint32_t qmask, const uint32_t lemask, const int lane,
                                             const float sp_scale_f, const uint32_t v0) {
  constexpr int P = C::kPer;
  const IdT* ids_s = reinterpret_cast<const IdT*>(sb);
  const float* win_s = reinterpret_cast<const float*>(sb + C::kIdsBytes);
  const float* w_s = reinterpret_cast<const float*>(sb + C::kIdsBytes + C::kWinBytes);
  const uint32_t* cb_s = reinterpret_cast<const uint32_t*>(sb + C::kIdsBytes + C::kWinBytes + C::kWBytes);
  const uint32_t acc_s = smem_u32(acc);     // 32-bit shared address of the accumulator (ATOMS operand)
    auto body = [&](const int sc, auto WHOLE) {
      constexpr bool kWhole = decltype(WHOLE)::value;
      const uint32_t xs = m.tile_base + sc * C::kSub;      // first ID position of the sub-chunk
      // lane-strided decode: step c covers the 32 consecutive IDs c*32 .. c*32+31
      // of the sub-chunk, so the window reads of a step hit ~32/r consecutive
      // words (one or two smem wavefronts)
      // IDs are read sign-extended: the run flag (MSB) becomes the sign, one
      // compare per ID for the ballot
      using SIdT = typename std::conditional<sizeof(IdT) == 2, int16_t, int32_t>::type;
      const SIdT* sids = reinterpret_cast<const SIdT*>(ids_s);
      float wv[P];                     // kWG: this sub-chunk's weights, loaded first (addresses known up front)
      if constexpr (C::kWG) {
#pragma unroll
        for (int c = 0; c < P; ++c) wv[c] = ldg_stream_f32(a.w + xs + c * 32 + lane);
      }
      uint32_t id[P];
#pragma unroll
      for (int c = 0; c < P; ++c) id[c] = (uint32_t)(int32_t)sids[sc * C::kSub + c * 32 + lane];
      // Alg. 5 update_ptr = #flags in ids[0..x] - 1 (R5), from the sub-chunk's
      // anchor plus a warp prefix count of the MSB flags, step by step
      uint32_t run = cb_s[(sc * C::kSub) / kChunkIds] - 1u - m.win_base;
      float val[P];
      bool ok[P];
#pragma unroll
      for (int c = 0; c < P; ++c) {
        const uint32_t bal = __ballot_sync(0xffffffffu, (int32_t)id[c] < 0);
        const uint32_t ptr = run + __popc(bal & lemask);
        run += __popc(bal);
        const uint32_t x = xs + c * 32 + lane;
        ok[c] = kWhole || (x >= m.lo && x < m.hi);
        // pair handles (q = 2^16, 4-byte IDs): this item owns half (j & 1) of the bin's
        // partition; the other half's IDs only advance the update pointer
        if constexpr (sizeof(IdT) == 4) ok[c] = ok[c] && (!a.pair || ((id[c] >> kMaxBits) & 1u) == (m.j & 1u));
        val[c] = ok[c] ? win_s[ptr] : 0.0f;
      }
      if constexpr (PR) {
        // PageRank: the apply stores SPR * 2^F (a power-of-two scaling, exact in fp32),
        // so one conversion rounds each term to the 2^-F grid
        uint32_t tlo[P], thi[P], old[P];
#pragma unroll
        for (int c = 0; c < P; ++c) {
          // SPR is stored as SPR * 2^F; weighted PageRank (R24) applies w(u,v) here
          const float tv = W ? val[c] * (C::kWG ? wv[c] : w_s[sc * C::kSub + c * 32 + lane]) : val[c];
          const unsigned long long T = __float2ull_rn(tv);
          tlo[c] = (uint32_t)T;
          thi[c] = (uint32_t)(T >> 32);
        }
#if PCPM_GATHER_MATCH
        // A/B (DESIGN.md §6 "hub aggregation"): lanes of a step that hit the same destination
        // are found with match.any; their terms are summed exactly with three redux.sync adds
        // (16-bit halves of the low words, and the high words) and the lowest lane issues one
        // ATOMS for the group.  Exact integer sums: the result is the same bits.
#pragma unroll
        for (int c = 0; c < P; ++c) {
          const uint32_t key = ok[c] ? (id[c] & qmask) : (0x80000000u | (uint32_t)lane);
          const uint32_t peers = __match_any_sync(0xffffffffu, key);
          if (peers != (1u << lane)) {
            const uint32_t slo = __reduce_add_sync(peers, tlo[c] & 0xFFFFu);
            const uint32_t shi = __reduce_add_sync(peers, tlo[c] >> 16);
            const uint32_t sth = __reduce_add_sync(peers, thi[c]);
            const unsigned long long tot = (unsigned long long)slo + ((unsigned long long)shi << 16) +
                                           ((unsigned long long)sth << 32);
            const bool lead = (__ffs(peers) - 1) == lane;
            tlo[c] = lead ? (uint32_t)tot : 0u;
            thi[c] = lead ? (uint32_t)(tot >> 32) : 0u;
            ok[c] = ok[c] && lead;
          }
        }
#endif
#pragma unroll
        for (int c = 0; c < P; ++c) old[c] = ok[c] ? atoms_add_u32(acc_s + ((id[c] & qmask) << 2), tlo[c]) : 0u;
        // carry out of the low word: old + lo wraps  <=>  lo > ~old; lanes with
        // ok = false have lo = hi = 0 (val = 0) and never carry
        uint32_t any = 0;
#if PCPM_CARRY_CC
        // carry-outs of old + lo counted with add.cc / addc (one add and one add-with-carry
        // per step instead of a NOT and a compare), OR-ed with the high parts
        static_assert(P == 4, "four steps per sub-chunk");
        asm("{\n\t.reg .u32 t;\n\t"
            "add.cc.u32 t, %1, %2;\n\taddc.u32 %0, 0, 0;\n\t"
            "add.cc.u32 t, %3, %4;\n\taddc.u32 %0, %0, 0;\n\t"
            "add.cc.u32 t, %5, %6;\n\taddc.u32 %0, %0, 0;\n\t"
            "add.cc.u32 t, %7, %8;\n\taddc.u32 %0, %0, 0;\n\t}"
            : "=r"(any)
            : "r"(old[0]), "r"(tlo[0]), "r"(old[1]), "r"(tlo[1]), "r"(old[2]), "r"(tlo[2]), "r"(old[3]), "r"(tlo[3]));
        any |= thi[0] | thi[1] | thi[2] | thi[3];
#else
#pragma unroll
        for (int c = 0; c < P; ++c) any |= thi[c] | (tlo[c] > ~old[c] ? 1u : 0u);
#endif
        if (any) {                                   // rare: carry into the global high word
#pragma unroll
          for (int c = 0; c < P; ++c) {
            const uint32_t hinc = thi[c] + (tlo[c] > ~old[c] ? 1u : 0u);
            if (hinc) {
              const uint32_t li = id[c] & qmask;
              atomicAdd(&a.hi[v0 + li], hinc);
              carry_mark<FINE>(bitmap, li);
            }
          }
        }
      } else {
        // SpMV: signed 64-bit fixed point in "balanced" form: the smem low
        // word is read as a signed int32, so a running sum that hovers
        // around zero never wraps; only signed overflow of the low word
        // (|partial| >= 2^31 units) carries +-1 into the global high word.
        // w*x is rounded once to fp32 (<= 2^-24 |w x|, R22); F keeps
        // |w x| 2^F <= 2^22 (kSpmvHead), so each term T is an int32 and the high part of the
        // balanced form is zero: only the low word's signed overflow carries.
        uint32_t tlo[P], old[P];
        int32_t thi[P];
#pragma unroll
        for (int c = 0; c < P; ++c) {
          const float tv = W ? val[c] * (C::kWG ? wv[c] : w_s[sc * C::kSub + c * 32 + lane]) : val[c];
          tlo[c] = (uint32_t)__float2int_rn(tv * sp_scale_f);
          thi[c] = 0;
        }
#pragma unroll
        for (int c = 0; c < P; ++c) old[c] = ok[c] ? atoms_add_u32(acc_s + ((id[c] & qmask) << 2), tlo[c]) : 0u;
        uint32_t any = 0;
        int32_t hinc[P];
#pragma unroll
        for (int c = 0; c < P; ++c) {
          const uint32_t nw = old[c] + tlo[c];
          const bool ovf = (int32_t)((old[c] ^ nw) & (tlo[c] ^ nw)) < 0;
          hinc[c] = ok[c] ? thi[c] + (ovf ? ((int32_t)old[c] < 0 ? -1 : 1) : 0) : 0;
          any |= (uint32_t)hinc[c];
        }
        if (any) {
#pragma unroll
          for (int c = 0; c < P; ++c)
            if (hinc[c]) {
              const uint32_t li = id[c] & qmask;
              atomicAdd(&a.hi[v0 + li], (uint32_t)hinc[c]);
              carry_mark<FINE>(bitmap, li);
            }
        }
      }
    };
  auto process = [&](const int sc) {
    const uint32_t xs = m.tile_base + sc * C::kSub;      // first ID position of the sub-chunk
    if (!PCPM_GATHER_NOOP && xs < m.hi && xs + C::kSub > m.lo) {
      const bool whole = xs >= m.lo && xs + C::kSub <= m.hi;   // warp-uniform: no per-ID range test
      if (whole) body(sc, std::true_type{});
      else body(sc, std::false_type{});
    }
  };
  // sub-chunks gw, gw + gsz, ... of the stage; the remaining kNsc mod gsz
  // sub-chunks rotate over the group's warps from stage to stage
  const int nmain = (C::kNsc / gsz) * gsz;
  // a stage inside its item (all but an item's first and last tiles): no range tests
  const bool stage_whole = !PCPM_GATHER_NOOP && m.lo == m.tile_base && m.hi == m.tile_base + (uint32_t)C::kTile;
  if (stage_whole) {
    for (int sc = gw; sc < nmain; sc += gsz) body(sc, std::true_type{});
  } else {
    for (int sc = gw; sc < nmain; sc += gsz) process(sc);
  }
  int who = rot;
  for (int sc = nmain; sc < C::kNsc; ++sc) {
    if (gw == who) process(sc);
    who = (who + 1 == gsz) ? 0 : who + 1;
  }
  rot = who;
}

// MULTI (PageRank shards with a fused exchange, pcpm_shard_step_peers): the apply
// also stores each SPR group to a.spr_peer[0 .. n_peer) -- other ranks' buffers,
// NVLink P2P -- and the kernel ends with a system-scope fence.
// FUSE (PageRank, DESIGN.md §5 "fused iteration"): after the apply of destination
// partition j the SPR values stay in the accumulator's shared memory and the CTA scatters
// source partition j of the next iteration from them (kFlagScatter stages); SPR is not
// written to global memory.
// PA (gather_variant 3, compact PageRank / SpMV without weights): the apply runs in the
// producer warps from tensor memory (PaRec / PaCtx above); the decoders only hand over.
template <typename IdT, bool W, bool PR, bool MULTI = false, bool SL = false, bool FUSE = false, bool PA = false>
__global__ void __launch_bounds__(Cfg<IdT, W, SL>::kThreads, 1) k_gather(const GatherArgs a) {
  using C = Cfg<IdT, W, SL>;
  constexpr int S = C::kStages;
  constexpr int P = C::kPer;
  extern __shared__ __align__(128) uint8_t smem[];
  const int64_t q = int64_t(1) << a.b;
  const int64_t aw = SL ? (int64_t)a.acc_words : q;                         // accumulator words (slots)
  uint32_t* acc = reinterpret_cast<uint32_t*>(smem);                       // aw words (128 B rounded)
  uint32_t* bitmap = acc + ((aw + 31) / 32) * 32;                          // 1 bit per 32 words
  constexpr bool kFine = PCPM_FINE_CARRY != 0 && !PA && !SL;
  const int bm_div = kFine ? 128 : 1024;
  const int bm_words = (int)((aw + bm_div - 1) / bm_div) < 4 ? 4 : (int)((aw + bm_div - 1) / bm_div);
  uint2* smap = reinterpret_cast<uint2*>(bitmap + ((bm_words + 31) / 32) * 32);  // slots: q/32 words
  uint8_t* stage_base = reinterpret_cast<uint8_t*>(smap + (SL ? q / 32 : 0));
  StageMeta* meta = reinterpret_cast<StageMeta*>(stage_base + S * C::kStageBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(meta + S);
  uint64_t* empty = full + S;
  uint64_t* qbar = empty + S;                                              // [8] claim queue (2 producers)
  double* red_s = reinterpret_cast<double*>(qbar + 8);                     // 2*C::kWarps
  uint32_t* flag_s = reinterpret_cast<uint32_t*>(red_s + 2 * C::kWarps);
  uint32_t* claimq = flag_s + 4;                                           // [8]
  uint64_t* tbar = reinterpret_cast<uint64_t*>(claimq + 8);                // PA: [0] tfull, [1] tempty
  uint32_t* tmem_s = reinterpret_cast<uint32_t*>(tbar + 2);                // PA: TMEM base (+ pad)
  PaRec* parec = reinterpret_cast<PaRec*>(tmem_s + 4);                     // PA: the parked item
  const IdT* ids = reinterpret_cast<const IdT*>(a.ids);
  constexpr int NP = C::kProducers;
  static_assert(!PA || (NP == 2 && C::kThreads == 1024 && !MULTI && !SL && !FUSE), "producer apply layout");

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], (s & 1) ? C::kGroupB : C::kGroupA);   // stage s is consumed by group s & 1
    }
    for (int s = 0; s < 8; ++s) mbar_init(&qbar[s], 1);
    if (PA) {
      mbar_init(&tbar[0], 1);
      mbar_init(&tbar[1], 2);
    }
    fence_mbar_init();
  }
  if (PA && warp == 0) tmem_alloc(tmem_s, 512);     // all of TMEM: one CTA per SM
  if (PA) tmem_fence_before();
  __syncthreads();
  if (PA) tmem_fence_after();
  pdl_trigger();
  PaCtx px{parec, &tbar[0], &tbar[1], PA ? *tmem_s : 0u};

  if (warp < NP) {
    gather_producer<C, IdT, W, PR, SL, FUSE, NP, PA>(a, ids, stage_base, meta, full, empty, lane, warp, claimq, qbar,
                                                     &px);
    if constexpr (PA) {
      __threadfence();                              // this warp's apply stores and red_fx atomics
      named_bar_sync(3, C::kThreads);               // with the consumers' completion count below
      if (warp == 0) {
        tmem_fence_after();
        tmem_dealloc(px.tbase, 512);
      }
    }
    return;
  }

  // ================= consumers =================
  const int cw = warp - NP;                 // consumer warp
  const int grp = cw < C::kGroupA ? 0 : 1;  // its group takes stages grp, grp + 2, ...
  const int gw = grp ? cw - C::kGroupA : cw;
  const int gsz = grp ? C::kGroupB : C::kGroupA;
  const int ctid = threadIdx.x - 32 * NP;   // 0 .. 32 * kWarps - 1
  constexpr int kCons = 32 * C::kWarps;
  const uint32_t qmask = (uint32_t)(q - 1);
  const float fscale = __uint_as_float((uint32_t)(127 + a.fbits) << 23);   // 2^F (PageRank)
  const double inv_scale = 1.0 / (double)fscale;
  for (int64_t i = ctid; i < aw; i += kCons) acc[i] = 0u;
  for (int i = ctid; i < bm_words; i += kCons) bitmap[i] = 0u;
  pdl_wait();                                      // D_t (red_in) and the scatter's bins are complete
  double base_pr = 0.0;
  if constexpr (PR) base_pr = (1.0 - a.d) / a.n + a.d * (a.red_in[0] / a.n);
  // SpMV scale: F = 22 - ceil(log2 max|w|) - ceil(log2 max|x|), so |w x| 2^F <= 2^22 (kSpmvHead)
  double sp_inv = 1.0;
  float sp_scale_f = 1.0f;
  if constexpr (!PR) {
    const int F = spmv_fbits(*a.xmax, a.wexp);
    sp_scale_f = ldexpf(1.0f, F);       // 2^F, F in [-120, 62]: a normal fp32
    sp_inv = ldexp(1.0, -F);
  }
  named_bar_sync(1, kCons);
  const uint32_t lemask = lanemask_le();

  // PA: move the finished accumulator into TMEM for the producers (see PaRec): wait until
  // they released the previous item, then the decoders of lane quadrants 0 and 1 (warps
  // 4 + 4 r + h) copy column groups of 8 and zero the shared words, decoder 0 writes the
  // record; stop = no more items.
  uint32_t tpar = 0;
  auto pa_handoff = [&](const StageMeta& m, bool stop) {
    if constexpr (PA) {
      mbar_wait(px.tempty, tpar ^ 1u);
      tpar ^= 1u;
      tmem_fence_after();
      if (!stop) {
        const int h = warp & 3;
        if (h < 2) {
          const uint32_t ngrp = (uint32_t)(q >> 9);  // 8-column groups (q / 64 columns)
          for (uint32_t cg = (uint32_t)((warp >> 2) - 1); cg < ngrp; cg += 7u) {
            uint32_t r[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) r[k] = acc[((cg * 8 + k) << 6) + 32 * h + lane];
#pragma unroll
            for (int k = 0; k < 8; ++k) acc[((cg * 8 + k) << 6) + 32 * h + lane] = 0u;
            tmem_st8(px.tbase + ((uint32_t)(32 * h) << 16) + cg * 8, r);
          }
          tmem_wait_st();
        }
        if (cw == 0) {
          if (lane == 0) {
            px.rec->j = m.j;
            px.rec->nsl = a.bin_nslices[m.j];
            px.rec->slot = a.items[m.item].pad[0];
            px.rec->stop = 0u;
          }
          px.rec->bm[lane] = lane < bm_words ? bitmap[lane] : 0u;
          if (lane < bm_words) bitmap[lane] = 0u;
        }
      } else if (cw == 0 && lane == 0) {
        px.rec->stop = 1u;
      }
      tmem_fence_before();
      named_bar_sync(1, kCons);                      // every share copied and zeroed
      if (cw == 0 && lane == 0) mbar_arrive(px.tfull);
    }
  };
  int stage = grp, rot = 0;
  int srot = 0;                                     // FUSE: rotation of the scatter stages' remainder
  uint32_t phase = 0;
  unsigned long long pt[4] = {0, 0, 0, 0};
  unsigned long long pe[4] = {0, 0, 0, 0};          // epilogue: pre-apply, apply, reductions, closing barrier
  long long tc = PCPM_GATHER_PROFILE ? clock64() : 0;
  for (;;) {
    mbar_wait(&full[stage], phase);
    if (PCPM_GATHER_PROFILE) { const long long t = clock64(); pt[0] += t - tc; tc = t; }
    const StageMeta m = meta[stage];
    if (m.flags & kFlagStop) break;
    if (FUSE && (m.flags & kFlagScatter)) {
      // next iteration's scatter of source partition m.j from the SPR values in acc
      if (!(m.flags & kFlagEmpty))
        fused_scatter_stage(a, m, stage_base + stage * C::kStageBytes, reinterpret_cast<const float*>(acc), gw, gsz,
                            srot, lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      stage += 2;
      if (stage >= S) { stage -= S; phase ^= 1; }
      if (m.flags & kFlagLast) {
        named_bar_sync(1, kCons);                   // both groups are done reading the SPR values
        for (int64_t i = ctid; i < q; i += kCons) acc[i] = 0u;
        named_bar_sync(1, kCons);
      }
      continue;
    }
    const uint32_t v0 = m.j << a.b;
    if (!(m.flags & kFlagEmpty))
      decode_stage<C, IdT, W, PR, kFine>(a, m, stage_base + stage * C::kStageBytes, acc, bitmap, gw, gsz, rot, qmask,
                                         lemask, lane, sp_scale_f, v0);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    stage += 2;
    if (stage >= S) { stage -= S; phase ^= 1; }
    if (PCPM_GATHER_PROFILE) { const long long t = clock64(); pt[1] += t - tc; tc = t; }

    if (m.flags & kFlagLast) {
      // ---------------- epilogue of this item ----------------
      named_bar_sync(1, kCons);
      if (PCPM_GATHER_PROFILE) { const long long t = clock64(); pt[2] += t - tc; tc = t; }
      if constexpr (PA) {
        pa_handoff(m, false);
        if (PCPM_GATHER_PROFILE) { const long long t = clock64(); pt[3] += t - tc; tc = t; }
        continue;
      }
      const int64_t cnt = min(q, a.n_dst - (int64_t)v0);
      const uint32_t nsl = a.bin_nslices[m.j];
      bool run_apply = true;
      if (nsl > 1) {
        // a slice of a split bin: store its low words to its slot (coalesced plain stores);
        // the last slice to arrive sums the bin's slots
        uint32_t* sbuf = a.slot_buf + (size_t)a.items[m.item].pad[0] * (size_t)q;
        for (int64_t i = ctid; i < q; i += kCons) {
          __stcg(sbuf + i, acc[i]);
          acc[i] = 0u;
        }
        __threadfence();
        named_bar_sync(1, kCons);
        if (ctid == 0) {
          const uint32_t old = atomicAdd(&a.bin_arrive[m.j], 1u);
          const bool last = old == nsl - 1;
          if (last) a.bin_arrive[m.j] = 0u;
          *flag_s = last ? 1u : 0u;
        }
        named_bar_sync(1, kCons);
        // with k_apply_split (the default) every slice only flushes; the in-kernel
        // last-arriver apply below is kept for has_split == 0 handles.  (The code
        // shape of this epilogue measurably changes the decode loop's schedule:
        // keep it as is unless re-measured.)
        run_apply = *flag_s != 0u && !a.has_split;
        if (run_apply) __threadfence();
      }
      // exact 64-bit total of local vertex i; resets the state it reads
      auto total = [&](int64_t i) -> uint64_t {
        const uint32_t v = v0 + (uint32_t)i;
        uint64_t tot;
        if (nsl > 1) {
          // PageRank: unsigned low words; SpMV: balanced (signed) low words, sign-extended
          const uint32_t* sb = a.slot_buf + (size_t)a.bin_slot_base[m.j] * (size_t)q + i;
          tot = (uint64_t)ldcg_u32(&a.hi[v]) << 32;
          for (uint32_t sl = 0; sl < nsl; ++sl) {
            const uint32_t w = ldcg_u32(sb + (size_t)sl * (size_t)q);
            tot += PR ? (uint64_t)w : (uint64_t)(long long)(int32_t)w;
          }
          a.hi[v] = 0u;
        } else {
          tot = PR ? (uint64_t)acc[i] : (uint64_t)(long long)(int32_t)acc[i];
          if (carry_test<kFine>(bitmap, (uint32_t)i)) {
            tot += (uint64_t)ldcg_u32(&a.hi[v]) << 32;
            a.hi[v] = 0u;
          }
          acc[i] = 0u;
        }
        return tot;
      };
      unsigned long long dang = 0, res = 0;   // 2^-62 fixed point (red_fx)
      if (PCPM_GATHER_NO_EPI) run_apply = false;
      if constexpr (SL) {
        // accumulator slots: vertex v reads slot16[v] (bins are never split with slots);
        // a vertex without in-edges has a zero sum.  4 consecutive vertices per thread when
        // the partition length and the output pointers allow 16-byte accesses
        run_apply = false;
        const uint2* gmap = a.slotmap + ((size_t)m.j << a.b) / 32;
        for (int64_t w = ctid; w < q / 32; w += kCons) smap[w] = __ldg(gmap + w);
        named_bar_sync(1, kCons);
        auto slot_of = [&](uint32_t i) -> uint32_t {   // local vertex i -> slot (0xFFFF: no in-edges)
          const uint2 e = smap[i >> 5];
          const uint32_t bit = 1u << (i & 31);
          return (e.x & bit) ? e.y + __popc(e.x & (bit - 1u)) : 0xFFFFu;
        };
        auto slot_total = [&](uint32_t sl) -> uint64_t {
          if (sl == 0xFFFFu) return 0;
          uint64_t tot = PR ? (uint64_t)acc[sl] : (uint64_t)(long long)(int32_t)acc[sl];
          if ((bitmap[sl >> 10] >> ((sl >> 5) & 31)) & 1u) {
            tot += (uint64_t)ldcg_u32(&a.hi[v0 + sl]) << 32;
            a.hi[v0 + sl] = 0u;
          }
          acc[sl] = 0u;
          return tot;
        };
        const bool vec4 = (cnt & 3) == 0 &&
                          (PR ? aligned16(a.pr_new + v0) && aligned16(a.spr_new + v0) && aligned16(a.inv_deg + v0) &&
                                    aligned16(a.pr_old + v0)
                              : aligned16(a.y + v0));
        for (int64_t i = ctid; !vec4 && i < cnt; i += kCons) {      // unaligned output / short partition
          const uint32_t v = v0 + (uint32_t)i;
          const uint64_t tot = slot_total(slot_of((uint32_t)i));
          if constexpr (PR) {
            const double prn = base_pr + a.d * ((double)(long long)tot * inv_scale);
            a.pr_new[v] = (float)prn;
            const float idg = __ldg(a.inv_deg + v);
            a.spr_new[v] = (float)prn * idg * fscale;
            if (idg == 0.0f) dang += red_fx(prn);
            res += red_fx(fabs(prn - (double)a.pr_old[v]));
          } else {
            a.y[v] = (float)((double)(long long)tot * sp_inv);
          }
        }
        for (int64_t i4 = ctid; vec4 && i4 < cnt / 4; i4 += kCons) {
          const uint32_t v = v0 + (uint32_t)(4 * i4);
          const uint32_t il = (uint32_t)(4 * i4);
          const uint32_t sl[4] = {slot_of(il), slot_of(il + 1), slot_of(il + 2), slot_of(il + 3)};
          if constexpr (PR) {
            const float4 idg = __ldg(reinterpret_cast<const float4*>(a.inv_deg + v));
            const float4 po = __ldg(reinterpret_cast<const float4*>(a.pr_old + v));
            const float idv[4] = {idg.x, idg.y, idg.z, idg.w};
            const float pov[4] = {po.x, po.y, po.z, po.w};
            float pn[4], sp[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const double prn = base_pr + a.d * ((double)(long long)slot_total(sl[c]) * inv_scale);
              pn[c] = (float)prn;
              sp[c] = pn[c] * idv[c] * fscale;
              dang += idv[c] != 0.0f ? 0ull : red_fx(prn);
              res += red_fx(fabs(prn - (double)pov[c]));
            }
            *reinterpret_cast<float4*>(a.pr_new + v) = make_float4(pn[0], pn[1], pn[2], pn[3]);
            *reinterpret_cast<float4*>(a.spr_new + v) = make_float4(sp[0], sp[1], sp[2], sp[3]);
          } else {
            float yv[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) yv[c] = (float)((double)(long long)slot_total(sl[c]) * sp_inv);
            *reinterpret_cast<float4*>(a.y + v) = make_float4(yv[0], yv[1], yv[2], yv[3]);
          }
        }
      }
      if (PCPM_GATHER_PROFILE) { const long long t = clock64(); pe[0] += t - tc; tc = t; }
      if (run_apply) {
        if constexpr (PR) {
          bool vec = (cnt & 3) == 0 && aligned16(a.pr_new + v0) && aligned16(a.pr_old + v0) &&
                     aligned16(a.spr_new + v0) && aligned16(a.inv_deg + v0) && aligned16(a.hi + v0);
          if constexpr (MULTI)
            for (int r = 0; r < a.n_peer; ++r) vec = vec && aligned16(a.spr_peer[r] + v0);
          if (vec) {
            const float4* id4 = reinterpret_cast<const float4*>(a.inv_deg + v0);
            const float4* po4 = reinterpret_cast<const float4*>(a.pr_old + v0);
            float4* pn4 = reinterpret_cast<float4*>(a.pr_new + v0);
            float4* sp4 = reinterpret_cast<float4*>(a.spr_new + v0);
            // (batching the loads of several float4 groups per thread measured slower:
            // the extra registers cost the decode loop more than the epilogue gains)
#pragma unroll 1
            for (int64_t i4 = ctid; i4 < cnt / 4; i4 += kCons) {
              const float4 idg = __ldg(id4 + i4);
              const float4 po = __ldg(po4 + i4);
#if PCPM_APPLY_HI4
              // a quad that carried (one bitmap bit covers it): its four global high words with
              // ONE 16-byte load issued beside the loads above, and one 16-byte store to clear
              // them -- total() would chain four dependent load/store pairs, and the whole CTA
              // waits at the closing barrier for the threads that hit such quads
              uint32_t hv[4] = {0u, 0u, 0u, 0u};
              const bool whole = nsl == 1;
              if (whole && carry_test<kFine>(bitmap, (uint32_t)(4 * i4))) {
                uint4* h4p = reinterpret_cast<uint4*>(a.hi + v0) + i4;
                const uint4 h4 = __ldcg(h4p);
                *h4p = make_uint4(0u, 0u, 0u, 0u);
                hv[0] = h4.x; hv[1] = h4.y; hv[2] = h4.z; hv[3] = h4.w;
              }
#endif
              const float idv[4] = {idg.x, idg.y, idg.z, idg.w};
              const float pov[4] = {po.x, po.y, po.z, po.w};
              float pn[4], sp[4];
#pragma unroll
              for (int c = 0; c < 4; ++c) {
#if PCPM_APPLY_HI4
                uint64_t tq;
                if (whole) {
                  tq = (uint64_t)acc[4 * i4 + c] + ((uint64_t)hv[c] << 32);
                  acc[4 * i4 + c] = 0u;
                } else {
                  tq = total(4 * i4 + c);
                }
                const double prn = base_pr + a.d * ((double)(long long)tq * inv_scale);
#else
                const double prn = base_pr + a.d * ((double)(long long)total(4 * i4 + c) * inv_scale);
#endif
                pn[c] = (float)prn;
                sp[c] = pn[c] * idv[c] * fscale;        // SPR * 2^F, SPR = PR / |N_o| (0 if dangling)
                dang += idv[c] != 0.0f ? 0ull : red_fx(prn);
                res += red_fx(fabs(prn - (double)pov[c]));
              }
              pn4[i4] = make_float4(pn[0], pn[1], pn[2], pn[3]);
              if (FUSE && nsl == 1)                     // the next scatter's source values stay on chip
                *reinterpret_cast<uint4*>(acc + 4 * i4) =
                    make_uint4(__float_as_uint(sp[0]), __float_as_uint(sp[1]), __float_as_uint(sp[2]),
                               __float_as_uint(sp[3]));
              else
                sp4[i4] = make_float4(sp[0], sp[1], sp[2], sp[3]);
              if constexpr (MULTI)
                for (int r = 0; r < a.n_peer; ++r)
                  reinterpret_cast<float4*>(a.spr_peer[r] + v0)[i4] = make_float4(sp[0], sp[1], sp[2], sp[3]);
            }
          } else {
            for (int64_t i = ctid; i < cnt; i += kCons) {
              const uint32_t v = v0 + (uint32_t)i;
              const double prn = base_pr + a.d * ((double)(long long)total(i) * inv_scale);
              a.pr_new[v] = (float)prn;
              const float idg = __ldg(a.inv_deg + v);
              if (FUSE && nsl == 1) acc[i] = __float_as_uint((float)prn * idg * fscale);
              else a.spr_new[v] = (float)prn * idg * fscale;
              if constexpr (MULTI)
                for (int r = 0; r < a.n_peer; ++r) a.spr_peer[r][v] = (float)prn * idg * fscale;
              if (idg == 0.0f) dang += red_fx(prn);
              res += red_fx(fabs(prn - (double)a.pr_old[v]));
            }
          }
        } else {
          for (int64_t i = ctid; i < cnt; i += kCons)
            a.y[v0 + (uint32_t)i] = (float)((double)(long long)total(i) * sp_inv);
        }
      }
      if (!SL)
        for (int64_t i = cnt + ctid; i < q; i += kCons) acc[i] = 0u;   // tail of a short last partition
      if (PCPM_GATHER_PROFILE) { const long long t = clock64(); pe[1] += t - tc; tc = t; }
      if constexpr (PR) warp_red_add(a.red_fx, dang, res, lane, PCPM_GATHER_ITEM_FENCE != 0);
      if (PCPM_GATHER_PROFILE) { const long long t = clock64(); pe[2] += t - tc; tc = t; }
      named_bar_sync(1, kCons);
      if (PCPM_GATHER_PROFILE) { const long long t = clock64(); pe[3] += t - tc; tc = t; }
      for (int i = ctid; i < bm_words; i += kCons) bitmap[i] = 0u;
      named_bar_sync(1, kCons);
      if (PCPM_GATHER_PROFILE) { const long long t = clock64(); pt[3] += t - tc; tc = t; }
    }
  }
  if (PCPM_GATHER_PROFILE && lane == 0) {
    for (int k = 0; k < 4; ++k) atomicAdd(&g_gather_prof[k], pt[k]);
    for (int k = 0; k < 4; ++k) atomicAdd(&g_gather_prof[19 + k], pe[k]);
    atomicAdd(&g_gather_prof[4], 1ull);
  }

  if constexpr (PA) {
    StageMeta ms{};
    pa_handoff(ms, true);                          // the producers drain the TMEM buffer and stop
  }
  if constexpr (MULTI) __threadfence_system();     // peer stores performed before the kernel completes
  else __threadfence();                            // this warp's red_fx atomics before the completion count
  // ---------------- last CTA: fixed-order reduction, counter reset ----------------
  if constexpr (PA) named_bar_sync(3, C::kThreads);   // the producers' applies are complete
  else named_bar_sync(1, kCons);
  if (ctid == 0) {
    __threadfence();
    const uint32_t done = atomicAdd(&a.counters[1], 1u);
    *flag_s = (done == gridDim.x - 1) ? 1u : 0u;
  }
  named_bar_sync(1, kCons);
  if (*flag_s) {
    __threadfence();
    if constexpr (PR)
      if (ctid == 0 && !a.has_split) red_finish(a);   // with split bins k_apply_split finishes
    if (ctid == 0) {
      a.counters[0] = 0u;
      a.counters[1] = 0u;
    }
  }
}

// ---------------------------------------------------------------------------
// k_gather2 (default, option "gather_variant" = 2): the same decode, with the apply
// of Eq. 1 taken off the decoders' critical path.  Warp roles (1024 threads):
//   warp 0          producer (as in k_gather)
//   warps 1 .. 27   decoders, two groups on alternate stages (14 + 13 warps)
//   warps 28 .. 31  apply warps, one per TMEM lane quadrant (warp % 4)
// When an item's decode ends, the decoders move its 128 KB accumulator from shared
// memory into one of two tensor-memory buffers (256 columns each: local vertex
// i = 128 c + l lives in lane l, column c), zero the shared copy and start the next
// item at once; the apply warps run the apply (or, for a slice of a split bin, the
// flush to its slot buffer) from TMEM while the next item is decoded.  Handoff
// protocol: tfull[b] (decoders -> apply, 1 arrival) / tempty[b] (apply -> decoders,
// 1 arrival) mbarriers per buffer, with tcgen05 fences around the thread syncs.
// timing-only experiment builds: FORCE_INLINE = the decoders apply every item themselves
// (apply warps idle); NOAPPLY = the apply warps skip the work (results are wrong)
#ifndef PCPM_GATHER2_FORCE_INLINE
#define PCPM_GATHER2_FORCE_INLINE 0
#endif
#ifndef PCPM_GATHER2_NOAPPLY
#define PCPM_GATHER2_NOAPPLY 0
#endif
#ifndef PCPM_GATHER2_APPLY
#define PCPM_GATHER2_APPLY 4                     // apply warps (4 or 8: one or two per TMEM lane quadrant)
#endif
template <typename IdT, bool W>
struct Cfg2 : Cfg<IdT, W> {
  static constexpr int kApply = PCPM_GATHER2_APPLY;
  static constexpr int kDec = 31 - kApply;
  static constexpr int kFirstApply = 1 + kDec;
  static constexpr int kThreads = 32 * (1 + kDec + kApply);
  static constexpr int kGroupA = (kDec + 1) / 2;
  static constexpr int kGroupB = kDec - kGroupA;
  static constexpr int kBufCols = 256;           // TMEM columns per accumulator buffer (q <= 2^15)
  static constexpr int kBmWords = 32;            // carry bitmap words (1 bit per 32 vertices, q <= 2^15)
  static_assert(kThreads == 1024 && kFirstApply % 4 == 0 && kApply % 4 == 0,
                "apply warps cover the four lane quadrants in order");
};

struct HandoffRec {        // one TMEM buffer's item (written by decoder 0, read by the apply warps)
  int item;
  uint32_t j, nsl, slot, stop, pad[3];
  uint32_t bm[32];         // carry bitmap of the item's accumulator
};

template <typename IdT, bool W, bool PR>
int smem_bytes2(int b) {
  using C = Cfg2<IdT, W>;
  const int64_t q = int64_t(1) << b;
  const int64_t head = ((q + 31) / 32) * 32 * 4 + C::kBmWords * 4;
  return (int)(head + C::kStages * C::kStageBytes + C::kStages * sizeof(StageMeta) + 2 * C::kStages * 8 + 4 * 8 +
               2 * sizeof(HandoffRec) + 32);
}

// The apply of one item's accumulator straight from shared memory by nthr threads
// (thread t of them): Eq. 1 for a whole bin, or the flush of a split bin's slice to
// its slot buffer; resets the accumulator and carry words it reads.
template <bool PR, bool MULTI>
__device__ __forceinline__ void apply_from_smem(const GatherArgs& a, uint32_t* acc, const uint32_t* bitmap,
                                                uint32_t v0, uint32_t cnt, int64_t q, uint32_t nsl, uint32_t slot,
                                                int t, int nthr, double base_pr, double inv_scale, float fscale,
                                                double sp_inv, unsigned long long& dang, unsigned long long& res) {
  if (nsl > 1) {
    uint32_t* sbuf = a.slot_buf + (size_t)slot * (size_t)q;
    for (int64_t i = t; i < q; i += nthr) {
      __stcg(sbuf + i, acc[i]);
      acc[i] = 0u;
    }
    return;
  }
  for (uint32_t i = t; i < cnt; i += nthr) {
    const uint32_t v = v0 + i;
    uint64_t tot = PR ? (uint64_t)acc[i] : (uint64_t)(long long)(int32_t)acc[i];
    acc[i] = 0u;
    if ((bitmap[i >> 10] >> ((i >> 5) & 31)) & 1u) {
      tot += (uint64_t)ldcg_u32(&a.hi[v]) << 32;
      a.hi[v] = 0u;
    }
    if constexpr (PR) {
      const float idg = __ldg(a.inv_deg + v);
      const double prn = base_pr + a.d * ((double)(long long)tot * inv_scale);
      const float pn = (float)prn;
      const float sp = pn * idg * fscale;
      a.pr_new[v] = pn;
      a.spr_new[v] = sp;
      if constexpr (MULTI)
        for (int rr = 0; rr < a.n_peer; ++rr) a.spr_peer[rr][v] = sp;
      if (idg == 0.0f) dang += red_fx(prn);
      res += red_fx(fabs(prn - (double)__ldg(a.pr_old + v)));
    } else {
      a.y[v] = (float)((double)(long long)tot * sp_inv);
    }
  }
  for (int64_t i = (int64_t)cnt + t; i < q; i += nthr) acc[i] = 0u;   // tail of a short last partition
}

template <typename IdT, bool W, bool PR, bool MULTI = false>
__global__ void __launch_bounds__(1024, 1) k_gather2(const GatherArgs a) {
  using C = Cfg2<IdT, W>;
  constexpr int S = C::kStages;
  extern __shared__ __align__(128) uint8_t smem[];
  const int64_t q = int64_t(1) << a.b;
  uint32_t* acc = reinterpret_cast<uint32_t*>(smem);                       // q words (128 B rounded)
  uint32_t* bitmap = acc + ((q + 31) / 32) * 32;                           // 1 bit per 32 vertices
  uint8_t* stage_base = reinterpret_cast<uint8_t*>(bitmap + C::kBmWords);
  StageMeta* meta = reinterpret_cast<StageMeta*>(stage_base + S * C::kStageBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(meta + S);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  HandoffRec* hrec = reinterpret_cast<HandoffRec*>(tempty + 2);
  uint32_t* tmem_base_s = reinterpret_cast<uint32_t*>(hrec + 2);
  uint32_t* flag_s = tmem_base_s + 1;
  uint32_t* inline_s = tmem_base_s + 2;
  const IdT* ids = reinterpret_cast<const IdT*>(a.ids);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bm_words = (int)((q + 1023) / 1024);
  const uint32_t ncol8 = (uint32_t)((q + 1023) / 1024);                   // 8-column groups per buffer

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], (s & 1) ? C::kGroupB : C::kGroupA);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&tfull[t], 1);
      mbar_init(&tempty[t], 1);
    }
    fence_mbar_init();
  }
  if (warp == C::kFirstApply) tmem_alloc(tmem_base_s, 2 * C::kBufCols);     // all 512 columns
  for (int i = threadIdx.x; i < C::kBmWords; i += blockDim.x) bitmap[i] = 0u;
  for (int64_t i = threadIdx.x; i < q; i += blockDim.x) acc[i] = 0u;
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = *tmem_base_s;

  if (warp == 0) {
    gather_producer<C, IdT, W, PR, false>(a, ids, stage_base, meta, full, empty, lane);
    return;
  }
  const int qd = warp & 3;                          // TMEM lane quadrant this warp may access
  constexpr int kWork = 32 * (C::kDec + C::kApply); // threads of bar 3 (decoders + apply warps)
  const float fscale = __uint_as_float((uint32_t)(127 + a.fbits) << 23);   // 2^F (PageRank)
  const double inv_scale = 1.0 / (double)fscale;
  double base_pr = 0.0, sp_inv = 1.0;
  float sp_scale_f = 1.0f;
  if constexpr (PR) {
    base_pr = (1.0 - a.d) / a.n + a.d * (a.red_in[0] / a.n);
  } else {
    const int F = spmv_fbits(*a.xmax, a.wexp);
    sp_scale_f = ldexpf(1.0f, F);
    sp_inv = ldexp(1.0, -F);
  }
  unsigned long long pt[4] = {0, 0, 0, 0};
  long long tc = PCPM_GATHER_PROFILE ? clock64() : 0;
  auto prof = [&](int k) {
    if (PCPM_GATHER_PROFILE) { const long long t = clock64(); pt[k] += t - tc; tc = t; }
  };

  if (warp < C::kFirstApply) {
    // ================= decoders =================
    const int cw = warp - 1;
    const int grp = cw < C::kGroupA ? 0 : 1;
    const int gw = grp ? cw - C::kGroupA : cw;
    const int gsz = grp ? C::kGroupB : C::kGroupA;
    constexpr int kDecT = 32 * C::kDec;
    // decoders of quadrant qd: warps qd0, qd0 + 4, ... <= kDec (qd0 = qd, or 4 for qd = 0)
    const int qd0 = qd == 0 ? 4 : qd;
    const int qrank = (warp - qd0) / 4, qcount = (C::kDec - qd0) / 4 + 1;
    const uint32_t qmask = (uint32_t)(q - 1);
    const uint32_t lemask = lanemask_le();
    int stage = grp, rot = 0, tb = 0;
    uint32_t phase = 0, tph = 0;
    // item end: move the accumulator into TMEM buffer tb for the apply warps, or --
    // when they are still busy with both buffers -- apply it here (decision taken by
    // decoder 0 before the barrier that ends the item, so every decoder sees it)
    auto item_end = [&](const StageMeta& m, bool stop) {
      if (cw == 0 && lane == 0)
        *inline_s = (!stop && (PCPM_GATHER2_FORCE_INLINE || !mbar_test(&tempty[tb], tph ^ 1))) ? 1u : 0u;
      named_bar_sync(1, kDecT);                      // all atomics of the item are done
      prof(1);
      if (*inline_s) {
        const uint32_t v0 = m.j << a.b;
        const uint32_t cnt = (uint32_t)min(q, a.n_dst - (int64_t)v0);
        unsigned long long dg = 0, rs = 0;
        apply_from_smem<PR, MULTI>(a, acc, bitmap, v0, cnt, q, a.bin_nslices[m.j], a.items[m.item].pad[0],
                                   threadIdx.x - 32, kDecT, base_pr, inv_scale, fscale, sp_inv, dg, rs);
        if constexpr (PR) warp_red_add(a.red_fx, dg, rs, lane);
        named_bar_sync(1, kDecT);                    // accumulator read and zeroed
        for (int i = threadIdx.x - 32; i < C::kBmWords; i += kDecT) bitmap[i] = 0u;
        named_bar_sync(1, kDecT);
        prof(3);
        return;
      }
      mbar_wait(&tempty[tb], tph ^ 1);               // the apply warps released buffer tb
      tmem_fence_after();
      prof(2);
      if (!stop) {
        const uint32_t tb_addr = tbase + (uint32_t)(tb * C::kBufCols) + ((uint32_t)(32 * qd) << 16);
        for (uint32_t cc = (uint32_t)qrank; cc < ncol8; cc += (uint32_t)qcount) {
          uint32_t r[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t i = (cc * 8 + k) * 128 + 32 * qd + lane;
            r[k] = i < (uint32_t)q ? acc[i] : 0u;
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t i = (cc * 8 + k) * 128 + 32 * qd + lane;
            if (i < (uint32_t)q) acc[i] = 0u;
          }
          tmem_st8(tb_addr + cc * 8, r);
        }
        tmem_wait_st();
      }
      if (cw == 0) {
        HandoffRec& H = hrec[tb];
        if (lane == 0) {
          H.stop = stop ? 1u : 0u;
          H.item = m.item;
          H.j = m.j;
          if (!stop) {
            H.nsl = a.bin_nslices[m.j];
            H.slot = a.items[m.item].pad[0];
          }
        }
        for (int i = lane; i < C::kBmWords; i += 32) {
          H.bm[i] = i < bm_words ? bitmap[i] : 0u;
          bitmap[i] = 0u;
        }
      }
      tmem_fence_before();
      named_bar_sync(1, kDecT);                      // every decoder copied + zeroed its share
      if (cw == 0 && lane == 0) mbar_arrive(&tfull[tb]);
      tb ^= 1;
      if (tb == 0) tph ^= 1;
      prof(3);
    };
    for (;;) {
      mbar_wait(&full[stage], phase);
      prof(0);
      const StageMeta m = meta[stage];
      if (m.flags & kFlagStop) break;
      const uint32_t v0 = m.j << a.b;
      if (!(m.flags & kFlagEmpty))
        decode_stage<C, IdT, W, PR>(a, m, stage_base + stage * C::kStageBytes, acc, bitmap, gw, gsz, rot, qmask,
                                    lemask, lane, sp_scale_f, v0);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      stage += 2;
      if (stage >= S) { stage -= S; phase ^= 1; }
      prof(1);
      if (m.flags & kFlagLast) item_end(m, false);
    }
    StageMeta ms{};
    item_end(ms, true);                              // tell the apply warps to stop
    if (PCPM_GATHER_PROFILE && lane == 0) {
      for (int k = 0; k < 4; ++k) atomicAdd(&g_gather_prof[k], pt[k]);
      atomicAdd(&g_gather_prof[4], 1ull);
    }
  } else {
    // ================= apply warps =================
    const int aw_id = warp - C::kFirstApply;         // quadrant qd = aw_id % 4
    const uint32_t aq = (uint32_t)(aw_id >> 2);      // which of the quadrant's apply warps
    constexpr uint32_t kPerQ = C::kApply / 4;
    unsigned long long dang = 0, res = 0;            // 2^-62 fixed point, this warp's share of the launch
    int tb = 0;
    uint32_t tph = 0;
    for (;;) {
      mbar_wait(&tfull[tb], tph);
      tmem_fence_after();
      prof(0);
      const HandoffRec& H = hrec[tb];
      if (H.stop) break;
      const uint32_t v0 = H.j << a.b;
      const uint32_t cnt = PCPM_GATHER2_NOAPPLY ? 0u : (uint32_t)min(q, a.n_dst - (int64_t)v0);
      const uint32_t nsl = H.nsl;
      const uint32_t tb_addr = tbase + (uint32_t)(tb * C::kBufCols) + ((uint32_t)(32 * qd) << 16);
      uint32_t* sbuf = a.slot_buf + (size_t)H.slot * (size_t)q;
      // per column k: vertices v0 + 128 c + 32 qd + lane -- 32 consecutive vertices per
      // warp instruction (coalesced 128-byte loads and stores); the next chunk's
      // vertex-array loads are issued before this chunk's arithmetic
      float nidg[8], npo[8];
      auto load_in = [&](uint32_t cc) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t i = (cc * 8 + k) * 128 + 32 * qd + lane;
          nidg[k] = i < cnt ? __ldg(a.inv_deg + v0 + i) : 0.0f;
          npo[k] = i < cnt ? __ldg(a.pr_old + v0 + i) : 0.0f;
        }
      };
      if (PR && nsl <= 1) load_in(aq);
#pragma unroll 1
      for (uint32_t cc = aq; cc < ncol8; cc += kPerQ) {
        if (cc * 1024 + 32 * qd >= cnt) break;      // columns beyond the partition (short last one)
        uint32_t r[8];
        tmem_ld8(tb_addr + cc * 8, r);
        if (nsl > 1) {
          // a slice of a split bin: its low words to the slot buffer (k_apply_split applies)
          tmem_wait_ld();
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t i = (cc * 8 + k) * 128 + 32 * qd + lane;
            if (i < (uint32_t)q) __stcg(sbuf + i, r[k]);
          }
          continue;
        }
        float idg[8], po[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          idg[k] = nidg[k];
          po[k] = npo[k];
        }
        if (PR && cc + kPerQ < ncol8) load_in(cc + kPerQ);
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t c = cc * 8 + k;
          const uint32_t i = c * 128 + 32 * qd + lane;
          if (i >= cnt) continue;
          const uint32_t v = v0 + i;
          const uint32_t g = c * 4 + qd;            // carry-bitmap group (32 vertices) of i
          uint64_t tot = PR ? (uint64_t)r[k] : (uint64_t)(long long)(int32_t)r[k];
          if ((H.bm[g >> 5] >> (g & 31)) & 1u) {
            tot += (uint64_t)ldcg_u32(&a.hi[v]) << 32;
            a.hi[v] = 0u;
          }
          if constexpr (PR) {
            const double prn = base_pr + a.d * ((double)(long long)tot * inv_scale);
            const float pn = (float)prn;
            const float sp = pn * idg[k] * fscale;    // SPR * 2^F, SPR = PR / |N_o| (0 if dangling)
            a.pr_new[v] = pn;
            a.spr_new[v] = sp;
            if constexpr (MULTI)
              for (int rr = 0; rr < a.n_peer; ++rr) a.spr_peer[rr][v] = sp;
            if (idg[k] == 0.0f) dang += red_fx(prn);
            res += red_fx(fabs(prn - (double)po[k]));
          } else {
            a.y[v] = (float)((double)(long long)tot * sp_inv);
          }
        }
      }
      tmem_fence_before();
      named_bar_sync(2, 32 * C::kApply);             // all apply warps are done with buffer tb
      if (aw_id == 0 && lane == 0) mbar_arrive(&tempty[tb]);
      tb ^= 1;
      if (tb == 0) tph ^= 1;
      prof(1);
    }
    if (PCPM_GATHER_PROFILE && lane == 0) {
      atomicAdd(&g_gather_prof[5], pt[0]);
      atomicAdd(&g_gather_prof[6], pt[1]);
      atomicAdd(&g_gather_prof[7], 1ull);
    }
    if constexpr (PR) warp_red_add(a.red_fx, dang, res, lane);
  }

  if constexpr (MULTI) __threadfence_system();     // peer stores performed before the kernel completes
  // ---------------- last CTA: totals, counter reset ----------------
  named_bar_sync(3, kWork);
  const int wt = threadIdx.x - 32;
  if (wt == 0) {
    __threadfence();
    const uint32_t done = atomicAdd(&a.counters[1], 1u);
    *flag_s = (done == gridDim.x - 1) ? 1u : 0u;
  }
  named_bar_sync(3, kWork);
  if (*flag_s && wt == 0) {
    __threadfence();
    if constexpr (PR)
      if (!a.has_split) red_finish(a);
    a.counters[0] = 0u;
    a.counters[1] = 0u;
  }
  if (warp == C::kFirstApply) {
    tmem_fence_after();
    tmem_dealloc(tbase, 2 * C::kBufCols);
  }
}


// ---------------------------------------------------------------------------
// k_gather_cl: the gather for graphs with few destination partitions (k_dst <
// SMs / 2, e.g. C2: k = 32 on 148 SMs).  Each bin is cut into cs tile-aligned slices
// processed by the cs CTAs of one thread-block cluster (cs = 2..8), each into its own
// shared-memory accumulator; after a cluster barrier every CTA applies 1/cs of the
// bin's vertices, summing the cs partial low words straight out of its peers' shared
// memory (distributed shared memory, ld.shared::cluster) -- no slot buffers in global
// memory and no separate apply launch (the single-CTA path's k_apply_split).
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t dsmem_addr(const void* p, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(p)), "r"(rank));
  return ra;
}
__device__ __forceinline__ uint4 dsmem_ld4(uint32_t ra) {
  uint4 v;
  asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(ra) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t dsmem_ld(uint32_t ra) {
  uint32_t v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(ra) : "memory");
  return v;
}

template <typename IdT, bool W, bool PR>
__global__ void __launch_bounds__(Cfg<IdT, W>::kThreads, 1) k_gather_cl(const GatherArgs a) {
  using C = Cfg<IdT, W>;
  constexpr int S = C::kStages;
  extern __shared__ __align__(128) uint8_t smem[];
  const int64_t q = int64_t(1) << a.b;
  uint32_t* acc = reinterpret_cast<uint32_t*>(smem);
  uint32_t* bitmap = acc + ((q + 31) / 32) * 32;
  const int bm_words = (int)((q + 1023) / 1024) < 4 ? 4 : (int)((q + 1023) / 1024);
  uint8_t* stage_base = reinterpret_cast<uint8_t*>(bitmap + ((bm_words + 31) / 32) * 32);
  StageMeta* meta = reinterpret_cast<StageMeta*>(stage_base + S * C::kStageBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(meta + S);
  uint64_t* empty = full + S;
  uint64_t* qbar = empty + S;                                            // [8] claim queue (2 producers)
  uint32_t* orbm = reinterpret_cast<uint32_t*>(qbar + 8);                // [bm_words] OR of the cluster's bitmaps
  uint32_t* flag_s = orbm + ((bm_words + 3) & ~3);
  uint32_t* claimq = flag_s + 4;                                         // [8]
  const IdT* ids = reinterpret_cast<const IdT*>(a.ids);
  constexpr int NP = C::kProducers;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], (s & 1) ? C::kGroupB : C::kGroupA);
    }
    for (int s = 0; s < 8; ++s) mbar_init(&qbar[s], 1);
    fence_mbar_init();
  }
  for (int64_t i = threadIdx.x; i < q; i += blockDim.x) acc[i] = 0u;
  for (int i = threadIdx.x; i < bm_words; i += blockDim.x) bitmap[i] = 0u;
  __syncthreads();
  pdl_trigger();
  pdl_wait();
  if (warp < NP) {
    gather_producer<C, IdT, W, PR, false, false, NP>(a, ids, stage_base, meta, full, empty, lane, warp, claimq, qbar);
  } else {
    const int cw = warp - NP;
    const int grp = cw < C::kGroupA ? 0 : 1;
    const int gw = grp ? cw - C::kGroupA : cw;
    const int gsz = grp ? C::kGroupB : C::kGroupA;
    const uint32_t qmask = (uint32_t)(q - 1);
    float sp_scale_f = 1.0f;
    if constexpr (!PR) sp_scale_f = ldexpf(1.0f, spmv_fbits(*a.xmax, a.wexp));
    const uint32_t lemask = lanemask_le();
    int stage = grp, rot = 0;
    uint32_t phase = 0;
    for (;;) {
      mbar_wait(&full[stage], phase);
      const StageMeta m = meta[stage];
      if (m.flags & kFlagStop) break;
      if (!(m.flags & kFlagEmpty))
        decode_stage<C, IdT, W, PR>(a, m, stage_base + stage * C::kStageBytes, acc, bitmap, gw, gsz, rot, qmask,
                                    lemask, lane, sp_scale_f, m.j << a.b);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      stage += 2;
      if (stage >= S) { stage -= S; phase ^= 1; }
    }
  }
  __syncthreads();
  cluster_sync_all();                              // every slice of the bin is accumulated
  const uint32_t rank = cluster_rank(), cs = cluster_size();
  const uint32_t j = a.items[blockIdx.x].j;
  const uint32_t v0 = j << a.b;
  const uint32_t cnt = (uint32_t)min(q, a.n_dst - (int64_t)v0);
  for (int i = threadIdx.x; i < bm_words; i += blockDim.x) {
    uint32_t o = 0;
    for (uint32_t r = 0; r < cs; ++r) o |= dsmem_ld(dsmem_addr(bitmap + i, r));
    orbm[i] = o;
  }
  __syncthreads();
  const uint32_t per = ((cnt + cs - 1) / cs + 3) & ~3u;     // this CTA's vertices [i0, i1)
  const uint32_t i0 = min(cnt, rank * per), i1 = min(cnt, i0 + per);
  const float fscale = __uint_as_float((uint32_t)(127 + a.fbits) << 23);
  const double inv_scale = 1.0 / (double)fscale;
  double base_pr = 0.0, sp_inv = 1.0;
  if constexpr (PR) base_pr = (1.0 - a.d) / a.n + a.d * (a.red_in[0] / a.n);
  else sp_inv = ldexp(1.0, -spmv_fbits(*a.xmax, a.wexp));
  unsigned long long dang = 0, res = 0;
  auto carry_of = [&](uint32_t i) -> uint64_t {    // the global high word of local vertex i (reset)
    if (!((orbm[i >> 10] >> ((i >> 5) & 31)) & 1u)) return 0;
    const uint64_t hv = (uint64_t)ldcg_u32(&a.hi[v0 + i]) << 32;
    a.hi[v0 + i] = 0u;
    return hv;
  };
  // 4 consecutive vertices per thread (i0 and per are multiples of 4)
  for (uint32_t i = i0 + 4 * threadIdx.x; i < i1; i += 4 * blockDim.x) {
    uint64_t su[4] = {0, 0, 0, 0};
    long long ss[4] = {0, 0, 0, 0};
    for (uint32_t r = 0; r < cs; ++r) {
      const uint4 w4 = dsmem_ld4(dsmem_addr(acc + i, r));
      const uint32_t wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        su[c] += wv[c];
        ss[c] += (int32_t)wv[c];
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint32_t ii = i + c;
      if (ii >= i1) break;
      const uint32_t v = v0 + ii;
      const uint64_t tot = carry_of(ii) + (PR ? su[c] : (uint64_t)ss[c]);
      if constexpr (PR) {
        const double prn = base_pr + a.d * ((double)(long long)tot * inv_scale);
        const float idg = __ldg(a.inv_deg + v);
        a.pr_new[v] = (float)prn;
        a.spr_new[v] = (float)prn * idg * fscale;
        if (idg == 0.0f) dang += red_fx(prn);
        res += red_fx(fabs(prn - (double)__ldg(a.pr_old + v)));
      } else {
        a.y[v] = (float)((double)(long long)tot * sp_inv);
      }
    }
  }
  if constexpr (PR) warp_red_add(a.red_fx, dang, res, lane);
  __syncthreads();
  cluster_sync_all();                              // the peers are done reading this CTA's accumulator
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t done = atomicAdd(&a.counters[1], 1u);
    *flag_s = (done == gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (*flag_s && threadIdx.x == 0) {
    __threadfence();
    if constexpr (PR) red_finish(a);
    a.counters[0] = 0u;
    a.counters[1] = 0u;
  }
}

template <typename IdT, bool W>
int smem_bytes_cl(int b) {
  using C = Cfg<IdT, W>;
  const int64_t q = int64_t(1) << b;
  const int bm_words = (int)((q + 1023) / 1024) < 4 ? 4 : (int)((q + 1023) / 1024);
  const int64_t head = ((q + 31) / 32) * 32 * 4 + ((bm_words + 31) / 32) * 32 * 4;
  return (int)(head + C::kStages * C::kStageBytes + C::kStages * sizeof(StageMeta) + 2 * C::kStages * 8 + 8 * 8 +
               ((bm_words + 3) & ~3) * 4 + 16 + 8 * 4);
}

// Apply of the split bins (items whose bin was cut into slices): one block per
// (split bin, 1024-vertex chunk); total = sum of the slices' low words + the carry
// word.  The last block reduces the per-item (gather) and per-block (here)
// dangling / residual partials in fixed order.
constexpr int kSplitThreads = 256, kSplitChunk = 1024;

template <bool PR>
__global__ void __launch_bounds__(kSplitThreads) k_apply_split(const GatherArgs a, const uint32_t* split_bins) {
  const int64_t q = int64_t(1) << a.b;
  const int chunks = (int)((q + kSplitChunk - 1) / kSplitChunk);
  const uint32_t j = split_bins[blockIdx.x / chunks];
  const int64_t c0 = (int64_t)(blockIdx.x % chunks) * kSplitChunk;
  const uint32_t v0 = j << a.b;
  const int64_t cnt = min(q, a.n_dst - (int64_t)v0);
  const uint32_t nsl = a.bin_nslices[j];
  const uint32_t* sb = a.slot_buf + (size_t)a.bin_slot_base[j] * (size_t)q;
  double base_pr = 0.0, inv_scale = 0.0, sp_inv = 1.0;
  float fscale = 1.0f;
  if constexpr (PR) {
    base_pr = (1.0 - a.d) / a.n + a.d * (a.red_in[0] / a.n);
    fscale = __uint_as_float((uint32_t)(127 + a.fbits) << 23);
    inv_scale = 1.0 / (double)fscale;
  } else {
    sp_inv = ldexp(1.0, -spmv_fbits(*a.xmax, a.wexp));
  }
  unsigned long long dang = 0, res = 0;   // 2^-62 fixed point (red_fx)
  const int64_t c1 = min(cnt, c0 + kSplitChunk);
  bool vec = PR && (c1 & 3) == 0 && (q & 3) == 0 && aligned16(a.hi + v0) && aligned16(a.pr_new + v0) && aligned16(a.spr_new + v0) &&
             aligned16(a.inv_deg + v0) && aligned16(a.pr_old + v0) && aligned16(sb);
  for (int r = 0; r < a.n_peer; ++r) vec = vec && aligned16(a.spr_peer[r] + v0);
  if (vec) {
    // 4 consecutive vertices per thread: one 16-byte load per slot, all slots' loads
    // independent (the sums are exact integers, so the order is free)
    for (int64_t i4 = c0 / 4 + threadIdx.x; i4 < c1 / 4; i4 += kSplitThreads) {
      const uint32_t v = v0 + (uint32_t)(4 * i4);
      const uint4 h4 = __ldcg(reinterpret_cast<const uint4*>(a.hi + v));
      uint64_t t0 = (uint64_t)h4.x << 32, t1 = (uint64_t)h4.y << 32, t2 = (uint64_t)h4.z << 32,
               t3 = (uint64_t)h4.w << 32;
#pragma unroll 4
      for (uint32_t sl = 0; sl < nsl; ++sl) {
        const uint4 w = __ldcg(reinterpret_cast<const uint4*>(sb + (size_t)sl * (size_t)q) + i4);
        t0 += w.x;
        t1 += w.y;
        t2 += w.z;
        t3 += w.w;
      }
      *reinterpret_cast<uint4*>(a.hi + v) = make_uint4(0u, 0u, 0u, 0u);
      const float4 idg = __ldg(reinterpret_cast<const float4*>(a.inv_deg + v));
      const float4 po = __ldg(reinterpret_cast<const float4*>(a.pr_old + v));
      const uint64_t tv[4] = {t0, t1, t2, t3};
      const float idv[4] = {idg.x, idg.y, idg.z, idg.w};
      const float pov[4] = {po.x, po.y, po.z, po.w};
      float pn[4], sp[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double prn = base_pr + a.d * ((double)(long long)tv[c] * inv_scale);
        pn[c] = (float)prn;
        sp[c] = pn[c] * idv[c] * fscale;
        if (idv[c] == 0.0f) dang += red_fx(prn);
        res += red_fx(fabs(prn - (double)pov[c]));
      }
      *reinterpret_cast<float4*>(a.pr_new + v) = make_float4(pn[0], pn[1], pn[2], pn[3]);
      *reinterpret_cast<float4*>(a.spr_new + v) = make_float4(sp[0], sp[1], sp[2], sp[3]);
      for (int r = 0; r < a.n_peer; ++r)
        *reinterpret_cast<float4*>(a.spr_peer[r] + v) = make_float4(sp[0], sp[1], sp[2], sp[3]);
    }
  }
  for (int64_t i = c0 + threadIdx.x; !vec && i < c1; i += kSplitThreads) {
    const uint32_t v = v0 + (uint32_t)i;
    uint64_t tot = (uint64_t)__ldcg(&a.hi[v]) << 32;
    for (uint32_t sl = 0; sl < nsl; ++sl) {
      const uint32_t w = __ldcg(sb + (size_t)sl * (size_t)q + i);
      tot += PR ? (uint64_t)w : (uint64_t)(long long)(int32_t)w;   // SpMV low words are signed
    }
    a.hi[v] = 0u;
    if constexpr (PR) {
      const double prn = base_pr + a.d * ((double)(long long)tot * inv_scale);
      a.pr_new[v] = (float)prn;
      const float idg = __ldg(a.inv_deg + v);
      a.spr_new[v] = (float)prn * idg * fscale;
      for (int r = 0; r < a.n_peer; ++r) a.spr_peer[r][v] = (float)prn * idg * fscale;   // fused exchange
      if (idg == 0.0f) dang += red_fx(prn);
      res += red_fx(fabs(prn - (double)a.pr_old[v]));
    } else {
      a.y[v] = (float)((double)(long long)tot * sp_inv);
    }
  }
  if constexpr (PR) {
    warp_red_add(a.red_fx, dang, res, threadIdx.x & 31);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(&a.counters[6], 1u) == gridDim.x - 1) {   // last block: all partials are in
        __threadfence();
        red_finish(a);
        a.counters[6] = 0u;
      }
    }
  }
}

template <typename IdT, bool W, bool SL = false>
int smem_bytes_for(int b, int64_t aw = 0) {
  using C = Cfg<IdT, W, SL>;
  const int64_t q = aw > 0 ? aw : int64_t(1) << b;
  const int bm_div = (PCPM_FINE_CARRY != 0 && !SL) ? 128 : 1024;     // fine carry bitmap (k_gather without slots)
  const int bm_words = (int)((q + bm_div - 1) / bm_div) < 4 ? 4 : (int)((q + bm_div - 1) / bm_div);
  const int64_t head = ((q + 31) / 32) * 32 * 4 + ((bm_words + 31) / 32) * 32 * 4 + (SL ? ((int64_t(1) << b) / 32) * 8 : 0);
  return (int)(head + C::kStages * C::kStageBytes + C::kStages * sizeof(StageMeta) + 2 * C::kStages * 8 + 8 * 8 +
               2 * C::kWarps * 8 + 16 + 8 * 4 + 2 * 8 + 16 + sizeof(PaRec));
}

using GatherFn = void (*)(const GatherArgs);

GatherFn gather_fn(bool wide, bool weighted, bool pagerank, bool multi = false, bool slots = false) {
  if (slots) return pagerank ? k_gather<uint16_t, false, true, false, true> : k_gather<uint16_t, false, false, false, true>;
  if (multi) return wide ? k_gather<uint32_t, false, true, true> : k_gather<uint16_t, false, true, true>;
  if (wide)
    return weighted ? (pagerank ? k_gather<uint32_t, true, true> : k_gather<uint32_t, true, false>)
                    : (pagerank ? k_gather<uint32_t, false, true> : k_gather<uint32_t, false, false>);
  return weighted ? (pagerank ? k_gather<uint16_t, true, true> : k_gather<uint16_t, true, false>)
                  : (pagerank ? k_gather<uint16_t, false, true> : k_gather<uint16_t, false, false>);
}

GatherFn gather_pa_fn() { return k_gather<uint16_t, false, true, false, false, false, true>; }

GatherFn gather_fuse_fn(bool weighted) {       // compact PageRank with the next scatter fused in
  return weighted ? k_gather<uint16_t, true, true, false, false, true> : k_gather<uint16_t, false, true, false, false, true>;
}

GatherFn gather2_fn(bool wide, bool weighted, bool pagerank, bool multi) {
  if (multi) return wide ? k_gather2<uint32_t, false, true, true> : k_gather2<uint16_t, false, true, true>;
  if (wide)
    return weighted ? (pagerank ? k_gather2<uint32_t, true, true> : k_gather2<uint32_t, true, false>)
                    : (pagerank ? k_gather2<uint32_t, false, true> : k_gather2<uint32_t, false, false>);
  return weighted ? (pagerank ? k_gather2<uint16_t, true, true> : k_gather2<uint16_t, true, false>)
                  : (pagerank ? k_gather2<uint16_t, false, true> : k_gather2<uint16_t, false, false>);
}

int gather2_smem_bytes(int b, bool wide, bool weighted) {
  if (wide) return weighted ? smem_bytes2<uint32_t, true, true>(b) : smem_bytes2<uint32_t, false, true>(b);
  return weighted ? smem_bytes2<uint16_t, true, true>(b) : smem_bytes2<uint16_t, false, true>(b);
}

}  // namespace

int gather_smem_bytes(int b, bool wide, bool weighted) {
  if (wide) return weighted ? smem_bytes_for<uint32_t, true>(b) : smem_bytes_for<uint32_t, false>(b);
  return weighted ? smem_bytes_for<uint16_t, true>(b) : smem_bytes_for<uint16_t, false>(b);
}

bool gather_slots_fit(int b, int acc_words) {
  int dev = 0, maxsm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return smem_bytes_for<uint16_t, false, true>(b, acc_words) <= maxsm;
}

GatherFn gather_cl_fn(bool wide, bool weighted, bool pagerank);

int prepare_gather(pcpm_handle* h) {
  int maxsm = 0;
  PCPM_CK(cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
  for (int wd = 0; wd < 2; ++wd)
    for (int w = 0; w < 2; ++w) {
      if (gather_smem_bytes(h->gb, wd, w) > maxsm) {
        set_error(PCPM_ECUDA, "gather shared-memory plan exceeds the device limit for this partition size");
        return PCPM_ECUDA;
      }
      for (int p = 0; p < 2; ++p)
        PCPM_CK(cudaFuncSetAttribute(gather_fn(wd, w, p), cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
    }
  for (int wd = 0; wd < 2; ++wd)
    PCPM_CK(cudaFuncSetAttribute(gather_fn(wd, false, true, true), cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
  for (int p = 0; p < 2; ++p)
    PCPM_CK(cudaFuncSetAttribute(gather_fn(false, false, p, false, true), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 maxsm));
  for (int wd = 0; wd < 2; ++wd)
    for (int w = 0; w < 2; ++w) {
      if (gather2_smem_bytes(h->gb, wd, w) > maxsm) {
        set_error(PCPM_ECUDA, "gather (v2) shared-memory plan exceeds the device limit for this partition size");
        return PCPM_ECUDA;
      }
      for (int p = 0; p < 2; ++p)
        PCPM_CK(cudaFuncSetAttribute(gather2_fn(wd, w, p, false), cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
    }
  for (int wd = 0; wd < 2; ++wd)
    PCPM_CK(cudaFuncSetAttribute(gather2_fn(wd, false, true, true), cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
  for (int wd = 0; wd < 2; ++wd)
    for (int w = 0; w < 2; ++w)
      for (int p = 0; p < 2; ++p)
        PCPM_CK(cudaFuncSetAttribute(gather_cl_fn(wd, w, p), cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
  for (int w = 0; w < 2; ++w)
    PCPM_CK(cudaFuncSetAttribute(gather_fuse_fn(w), cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
  PCPM_CK(cudaFuncSetAttribute(gather_pa_fn(), cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
  return PCPM_OK;
}

int launch_absmax(pcpm_handle* h, const float* x, int64_t n, float* out, cudaStream_t s) {
  PCPM_CK(cudaMemsetAsync(out, 0, sizeof(float), s));
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, h->num_sms * 4));
  k_absmax<<<grid, 256, 0, s>>>(n, x, out);
  PCPM_CK(cudaGetLastError());
  h->launches += 1;
  return PCPM_OK;
}

int gather_threads(bool wide, bool weighted) {
  if (wide) return weighted ? Cfg<uint32_t, true>::kThreads : Cfg<uint32_t, false>::kThreads;
  return weighted ? Cfg<uint16_t, true>::kThreads : Cfg<uint16_t, false>::kThreads;
}

int read_debug_counters(unsigned long long* out, int cap, bool reset) {
  unsigned long long v[24];
  PCPM_CK(cudaMemcpyFromSymbol(v, g_gather_prof, sizeof(v)));
  for (int i = 0; i < cap && i < 24; ++i) out[i] = v[i];
  if (reset) {
    unsigned long long z[24] = {};
    PCPM_CK(cudaMemcpyToSymbol(g_gather_prof, z, sizeof(z)));
  }
  return cap < 24 ? cap : 24;
}

int launch_apply_split(pcpm_handle* h, const GatherArgs& a, bool pagerank, cudaStream_t s) {
  if (h->n_split_bins == 0) return PCPM_OK;
  const int chunks = (int)(((int64_t(1) << h->gb) + kSplitChunk - 1) / kSplitChunk);
  const int blocks = h->n_split_bins * chunks;
  if (pagerank)
    k_apply_split<true><<<blocks, kSplitThreads, 0, s>>>(a, h->split_bins);
  else
    k_apply_split<false><<<blocks, kSplitThreads, 0, s>>>(a, h->split_bins);
  PCPM_CK(cudaGetLastError());
  h->launches += 1;
  return PCPM_OK;
}

GatherFn gather_cl_fn(bool wide, bool weighted, bool pagerank) {
  if (wide)
    return weighted ? (pagerank ? k_gather_cl<uint32_t, true, true> : k_gather_cl<uint32_t, true, false>)
                    : (pagerank ? k_gather_cl<uint32_t, false, true> : k_gather_cl<uint32_t, false, false>);
  return weighted ? (pagerank ? k_gather_cl<uint16_t, true, true> : k_gather_cl<uint16_t, true, false>)
                  : (pagerank ? k_gather_cl<uint16_t, false, true> : k_gather_cl<uint16_t, false, false>);
}

int gather_cl_smem_bytes(int b, bool wide, bool weighted) {
  if (wide) return weighted ? smem_bytes_cl<uint32_t, true>(b) : smem_bytes_cl<uint32_t, false>(b);
  return weighted ? smem_bytes_cl<uint16_t, true>(b) : smem_bytes_cl<uint16_t, false>(b);
}

int launch_gather_cl(pcpm_handle* h, const GatherArgs& a0, bool weighted, bool pagerank, cudaStream_t s) {
  GatherArgs a = a0;
  a.items = h->gitems_cl;
  a.n_items = (int)(h->k_dst * h->cl_cs);
  a.static_items = 1;
  a.has_split = 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)a.n_items);
  cfg.blockDim = dim3(gather_threads(h->wide, weighted));
  cfg.dynamicSmemBytes = gather_cl_smem_bytes(a.b, h->wide, weighted);
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)h->cl_cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (h->opt_pdl) {
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.numAttrs = 2;
  }
  if (getenv("PCPM_DEBUG_CLUSTER")) {          // how many clusters fit at once (A/B diagnostics)
    int ncl = 0;
    cudaOccupancyMaxActiveClusters(&ncl, (const void*)gather_cl_fn(h->wide, weighted, pagerank), &cfg);
    cudaGetLastError();
    fprintf(stderr, "[pcpm] cluster gather: %d clusters of %d CTAs, %d can be resident at once\n",
            (int)h->k_dst, h->cl_cs, ncl);
  }
  PCPM_CK(cudaLaunchKernelEx(&cfg, gather_cl_fn(h->wide, weighted, pagerank), a));
  h->launches += 1;
  return PCPM_OK;
}

int launch_gather(pcpm_handle* h, const GatherArgs& a, bool weighted, bool pagerank, cudaStream_t s, bool multi,
                  bool fuse) {
  const bool slots = a.slot16 != nullptr && !weighted && !multi;
  if (fuse) {                                      // PageRank iteration with the next scatter fused in
    const int grid = std::min(h->num_sms, std::max(a.n_items, 1));
    gather_fuse_fn(weighted)<<<grid, gather_threads(false, weighted), gather_smem_bytes(a.b, false, weighted), s>>>(a);
    PCPM_CK(cudaGetLastError());
    h->launches += 1;
    return launch_apply_split(h, a, pagerank, s);
  }
  if (h->cl_cs >= 2 && h->opt_cluster_gather && !slots && !multi) return launch_gather_cl(h, a, weighted, pagerank, s);
  if (!slots && h->opt_gather_variant == 2 && !h->pair) {
    const int grid = std::min(h->num_sms, std::max(a.n_items, 1));
    gather2_fn(h->wide, weighted, pagerank, multi && pagerank && !weighted)<<<grid, 1024,
                                                                           gather2_smem_bytes(a.b, h->wide, weighted), s>>>(a);
    PCPM_CK(cudaGetLastError());
    h->launches += 1;
    return launch_apply_split(h, a, pagerank, s);
  }
  const int smem = slots ? smem_bytes_for<uint16_t, false, true>(a.b, a.acc_words) : gather_smem_bytes(a.b, h->wide, weighted);
  const int grid = std::min(h->num_sms, std::max(a.n_items, 1));
  // gather_variant 3: the apply in the producer warps from tensor memory (compact,
  // unweighted PageRank, 2^9 <= q <= 2^15)
  if (h->opt_gather_variant == 3 && !slots && !multi && !h->wide && !weighted && pagerank && a.b >= 9 && a.b <= 15) {
    PCPM_CK(launch_k(h->opt_pdl != 0, gather_pa_fn(), grid, gather_threads(false, false), smem, s, a));
    h->launches += 1;
    return launch_apply_split(h, a, pagerank, s);
  }
  PCPM_CK(launch_k(h->opt_pdl != 0, gather_fn(h->wide, weighted, pagerank, multi && pagerank && !weighted, slots), grid,
                   gather_threads(h->wide, weighted), smem, s, a));
  h->launches += 1;
  return launch_apply_split(h, a, pagerank, s);     // split bins (small k), if any
}

}  // namespace pcpm

// scatter.cu -- a1: the PNG scatter of PAPER.md Alg. 4.
//
//   for p in P:  for p' in P:  for u in N_i^p(p'):  insert SPR[u] into update_bins[p']
//
// Work items are (source partition p, destination groups [j0, j1)); their PNG
// entries png[png_off[p][j0] .. png_off[p][j1]) are contiguous (groups are
// stored in (p, j) order), and group (p, j) writes the disjoint range
// upd[upd_off[p][j] ...] (fixed, disjoint write locations -- no atomics).
// A pure copy: the update bins are bit-identical to the oracle's scatter for
// the same x.
//
// k_scatter_tma (default):
//  * Persistent CTAs claim items from an atomic counter in source-partition
//    order (neighbouring groups of an update bin are written at about the same
//    time, so their shared sectors complete in L2); the last 148 partitions'
//    items are cut finer so the final wave is short.
//  * Warp 0 is a TMA producer.  Per item it bulk-copies the partition's source
//    values x[p q .. p q + q) (128 KB at q = 2^15 -- "cache the vertex data of
//    p") and the item's rows of png_off / upd_off into shared memory,
//    then streams the item's PNG entries through a 5-stage ring of 16 KB
//    bulk copies with the grp_at anchors of each 256-entry chunk.
//  * 31 consumer warps take 256-entry sub-ranges of each stage.  Lane l
//    handles entries e = base + l + 32 i: consecutive lanes read consecutive
//    PNG entries from smem and write consecutive update slots of the group
//    containing e (dst = upd_off[g] + e - png_off[g]), so global stores are
//    coalesced; the group index is advanced per lane as e crosses group
//    boundaries.
//
// k_scatter_warp (option "scatter_variant" = 1, the round-1 design kept for
// A/B): warps claim whole groups and read the PNG straight from global memory.
#include "pcpm_internal.cuh"

namespace pcpm {
namespace {

// ------------------------------------------------------------------ TMA variant
// consumer warps: 31 for the compact (2-byte) PNG -- 32 sub-ranges of 256 entries per
// 16 KB stage, the extra one rotating -- and 16 for the 4-byte PNG (16 sub-ranges)
#ifndef PCPM_SCATTER_UNROLL
#define PCPM_SCATTER_UNROLL 8
#endif
#ifndef PCPM_SCATTER_WARPS16
#define PCPM_SCATTER_WARPS16 31
#endif
template <typename SrcT> struct ScCfg {
  static constexpr int kW = sizeof(SrcT) == 2 ? PCPM_SCATTER_WARPS16 : 16;
  static constexpr int kThreads = 32 * (kW + 1);
};
constexpr int kScStages = 5;
constexpr int kScStageBytes = 16384;               // PNG bytes per stage
constexpr int kScOffCap = kScatterMaxGroups + 8;   // offsets of one item (+ alignment slack)

struct ScItemMeta {
  uint32_t p, j0, ng;
  uint32_t stop;
  uint32_t off_shift;    // png_off row starts at off_s[off_shift]
  uint32_t uo_shift;     // upd_off row starts at uo_s[uo_shift]
  uint32_t pad[2];
};
struct ScStageMeta {
  uint32_t base;         // PNG position of stage element 0 (a multiple of kPngChunk)
  uint32_t lo, hi;       // valid PNG positions [lo, hi)
  uint32_t last;         // last stage of the item
  uint32_t gshift;       // grp_at[base / kPngChunk] is at stage_grp[gshift]
  uint32_t pad[3];
};
constexpr int kScGrpCap = kScStageBytes / 2 / kPngChunk + 8;   // grp_at entries per stage (+ alignment)

struct ScatterArgs {
  const ScatterItem* items;
  int n_items;
  const float* x;
  int64_t n_src;
  int b;
  int64_t k_dst;
  const void* png;
  const uint32_t* png_off;
  const uint32_t* upd_off;
  const uint32_t* grp_at;
  float* upd;
  uint32_t* counters;    // [2] item counter, [3] done counter (kept zero)
  int pf_stages;         // L2 prefetch distance in stages
};

// XG (scatter_variant 2, the "SPR through L1/L2" A/B of DESIGN.md §6): the source values
// are read with ld.global.nc instead of a 128 KB shared-memory copy of the partition's
// slice per item -- for graphs whose vector is L2-resident and whose items are many
// per source partition (small k), the staging is mostly redundant traffic.
// VEC (scatter_variant 3, north star (2)'s "vectorised 128-bit stores"): each lane writes
// 4 consecutive update slots with one 16-byte store.  A group's slots are contiguous but
// start at any word (upd_off is a running count), so the quads are aligned in
// DESTINATION space per group: group g's segment of the sub-range covers the quads
// floor4(lo + delta_g) .. of upd, its first and last quads partial (scalar stores).  The
// quads of all groups in the sub-range are numbered consecutively and dealt to the lanes
// 32 at a time; a lane finds its group by walking from the round's first group.
template <typename SrcT, bool XG = false, bool VEC = false>
__global__ void __launch_bounds__(ScCfg<SrcT>::kThreads, 1) k_scatter_tma(const ScatterArgs a) {
  constexpr int kScW = ScCfg<SrcT>::kW;
  constexpr int kChunk = kScStageBytes / (int)sizeof(SrcT);   // PNG entries per stage
  constexpr int kSub = kPngChunk;                               // entries per sub-range
  constexpr int kNsr = kChunk / kSub;                           // sub-ranges per stage
  constexpr uint32_t kAlignE = kPngChunk;                       // stage bases: multiples of kPngChunk
  static_assert(kSub % kPngChunk == 0 && kNsr >= kScW, "warp sub-ranges start on grp_at anchors");
  extern __shared__ __align__(128) uint8_t smem[];
  const int64_t q = int64_t(1) << a.b;
  float* xs = reinterpret_cast<float*>(smem);                                        // q floats (none with XG)
  uint32_t* off_s = reinterpret_cast<uint32_t*>(smem + (XG ? int64_t(0) : ((q * 4 + 127) & ~int64_t(127))));
  uint32_t* uo_s = off_s + kScOffCap;
  uint8_t* ring = reinterpret_cast<uint8_t*>(uo_s + kScOffCap);
  uint32_t* grp_s = reinterpret_cast<uint32_t*>(ring + kScStages * kScStageBytes);       // [kScStages][kScGrpCap]
  ScStageMeta* smeta = reinterpret_cast<ScStageMeta*>(grp_s + kScStages * kScGrpCap);
  ScItemMeta* imeta = reinterpret_cast<ScItemMeta*>(smeta + kScStages);
  uint64_t* full = reinterpret_cast<uint64_t*>(imeta + 1);
  uint64_t* empty = full + kScStages;
  uint64_t* ifull = empty + kScStages;
  uint64_t* iempty = ifull + 1;
  uint32_t* flag_s = reinterpret_cast<uint32_t*>(iempty + 1);
  const SrcT* png = reinterpret_cast<const SrcT*>(a.png);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kScStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kScW);
    }
    mbar_init(ifull, 1);
    mbar_init(iempty, kScW);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_trigger();
  pdl_wait();                                      // x (the previous gather's SPR) is complete

  if (warp == 0) {
    // ================= producer =================
    if (lane == 0) {
      const uint64_t pol_stream = policy_evict_first();
      const uint64_t pol_keep = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0, iphase = 0;
      for (;;) {
        const uint32_t it = atomicAdd(&a.counters[2], 1u);
        const bool stop = it >= (uint32_t)a.n_items;
        ScatterItem item{};
        uint32_t s0 = 0, s1 = 0;
        if (!stop) {
          item = a.items[it];
          s0 = __ldg(a.png_off + (int64_t)item.p * (a.k_dst + 1) + item.j0);
          s1 = __ldg(a.png_off + (int64_t)item.p * (a.k_dst + 1) + item.j1);
          if (s0 == s1) continue;                                   // nothing to write
          // warm L2 with the item's first stages and its source slice while the
          // consumers finish the previous item
          const int64_t xb = (int64_t)item.p << a.b;
          const uint32_t xpb = (uint32_t)((min(q, a.n_src - xb) * 4) & ~int64_t(15));
          if (xpb) bulk_prefetch_l2(a.x + xb, xpb);
          const uint32_t ab = s0 & ~(kAlignE - 1);
          for (int c = kScStages; c < kScStages + a.pf_stages; ++c) {
            const uint32_t cb = ab + (uint32_t)c * kChunk;
            if (cb >= s1) break;
            bulk_prefetch_l2(png + cb, kScStageBytes);
          }
        }
        uint32_t cb = 0;
        // issue a stage of the item's PNG entries through the ring
        auto issue = [&](uint32_t c) {
          if (a.pf_stages) {
            const uint32_t pb = c + (uint32_t)a.pf_stages * kChunk;
            if (pb < s1) bulk_prefetch_l2(png + pb, kScStageBytes);
          }
          mbar_wait(&empty[stage], phase ^ 1);
          ScStageMeta sm;
          sm.base = c;
          sm.lo = max(c, s0);
          sm.hi = min(c + (uint32_t)kChunk, s1);
          sm.last = (c + (uint32_t)kChunk >= s1) ? 1u : 0u;
          const uint32_t c0 = c / kPngChunk, ca = c0 & ~3u;
          const uint32_t nga = (((sm.hi - c + kPngChunk - 1) / kPngChunk) + (c0 - ca) + 3) & ~3u;
          sm.gshift = c0 - ca;
          smeta[stage] = sm;
          const uint32_t bytes = (((sm.hi - c) * (uint32_t)sizeof(SrcT)) + 15) & ~15u;   // png is padded
          mbar_arrive_expect_tx(&full[stage], bytes + nga * 4);
          bulk_g2s(ring + stage * kScStageBytes, png + c, bytes, &full[stage], pol_stream);
          bulk_g2s(grp_s + stage * kScGrpCap, a.grp_at + ca, nga * 4, &full[stage], pol_stream);   // grp_at padded
          if (++stage == kScStages) { stage = 0; phase ^= 1; }
        };
        if (!stop) {
          // the first ring stages of this item do not depend on the source slice:
          // issue them while the consumers finish the previous item
          cb = s0 & ~(kAlignE - 1);
          for (int c = 0; c < kScStages && cb < s1; ++c, cb += kChunk) issue(cb);
        }
        mbar_wait(iempty, iphase ^ 1);                              // consumers done with the last item
        iphase ^= 1;
        ScItemMeta im{};
        if (stop) {
          im.stop = 1;
          *imeta = im;
          mbar_arrive(ifull);
          break;
        }
        const int64_t xbase = (int64_t)item.p << a.b;
        const int64_t len = min(q, a.n_src - xbase);
        const uint32_t xbytes = (uint32_t)(((len * 4) + 15) & ~int64_t(15));      // x is padded (launch_scatter)
        const int64_t orow = (int64_t)item.p * (a.k_dst + 1) + item.j0;
        const int64_t urow = (int64_t)item.p * a.k_dst + item.j0;
        const uint32_t ng = item.j1 - item.j0;
        const int64_t oal = orow & ~int64_t(3), ual = urow & ~int64_t(3);
        const uint32_t obytes = (uint32_t)(((orow + ng + 1 - oal) * 4 + 15) & ~int64_t(15));   // offsets padded
        const uint32_t ubytes = (uint32_t)(((urow + ng - ual) * 4 + 15) & ~int64_t(15));
        im.p = item.p;
        im.j0 = item.j0;
        im.ng = ng;
        im.off_shift = (uint32_t)(orow - oal);
        im.uo_shift = (uint32_t)(urow - ual);
        *imeta = im;
        mbar_arrive_expect_tx(ifull, (XG ? 0u : xbytes) + obytes + ubytes);
        if (!XG) bulk_g2s(xs, a.x + xbase, xbytes, ifull, pol_keep);
        bulk_g2s(off_s, a.png_off + oal, obytes, ifull, pol_keep);
        bulk_g2s(uo_s, a.upd_off + ual, ubytes, ifull, pol_keep);
        for (; cb < s1; cb += kChunk) issue(cb);
      }
    }
  } else {
    // ================= consumers =================
    const int cw = warp - 1;
    int stage = 0, rot = 0;
    uint32_t phase = 0, iphase = 0;
    const uint32_t ubase_wide = 0;
    (void)ubase_wide;
    for (;;) {
      mbar_wait(ifull, iphase);
      iphase ^= 1;
      const ScItemMeta im = *imeta;
      if (im.stop) break;
      const uint32_t* offs = off_s + im.off_shift;    // offs[g] = png_off[p][j0 + g], g in [0, ng]
      const uint32_t* uos = uo_s + im.uo_shift;       // uos[g] = upd_off[p][j0 + g]
      const uint32_t ubase = sizeof(SrcT) == 2 ? 0u : (im.p << a.b);   // wide sources are global IDs
      const float* xg = a.x + ((int64_t)im.p << a.b);                   // XG: the slice in global memory
      for (;;) {
        mbar_wait(&full[stage], phase);
        const ScStageMeta sm = smeta[stage];
        const SrcT* ps = reinterpret_cast<const SrcT*>(ring + stage * kScStageBytes);
        // VEC: quads of destination slots, aligned per group (see the kernel's comment)
        auto range_vec = [&](const int sr) {
          const uint32_t wb = sm.base + (uint32_t)(sr * kSub);
          const uint32_t wlo = max(wb, sm.lo), whi = min(wb + (uint32_t)kSub, sm.hi);
          if (wlo >= whi) return;
          const int32_t ga = (int32_t)(grp_s[stage * kScGrpCap + sm.gshift + (wb - sm.base) / kPngChunk] -
                                       (im.p * (uint32_t)a.k_dst + im.j0));
          uint32_t g = ga > 0 ? (uint32_t)ga : 0u;
          while (offs[g + 1] <= wlo) ++g;                 // the group of wlo (the anchor is wb's)
          // quads of group gg inside [wlo, whi): 0 if the segment is empty
          auto nq = [&](uint32_t gg) -> uint32_t {
            const uint32_t slo = max(offs[gg], wlo), shi = min(offs[gg + 1], whi);
            if (slo >= shi) return 0u;
            const uint32_t dl = uos[gg] - offs[gg];
            return ((shi + dl + 3) >> 2) - ((slo + dl) >> 2);
          };
          uint32_t total = 0;
          for (uint32_t gg = g; offs[gg] < whi; ++gg) total += nq(gg);
          uint32_t gcur = g, qcur = 0;                    // the round's first quad: quad qcur of group gcur
          for (uint32_t t0 = 0; t0 < total; t0 += 32) {
            uint32_t gg = gcur, rem = qcur + lane, n = nq(gg);
            while (rem >= n && t0 + lane < total) {
              rem -= n;
              ++gg;
              n = nq(gg);
            }
            if (t0 + lane < total) {
              const uint32_t dl = uos[gg] - offs[gg];
              const uint32_t slo = max(offs[gg], wlo), shi = min(offs[gg + 1], whi);
              const uint32_t dq = (((slo + dl) >> 2) + rem) << 2;          // first slot of the quad
              const int32_t lead = (int32_t)(dq - dl - slo);                // < 0: the quad starts before slo
              const uint32_t elo = lead > 0 ? slo + (uint32_t)lead : slo, ehi = min(dq + 4 - dl, shi);
              const SrcT* pe = ps + (elo - sm.base);
              if (ehi - elo == 4) {
                const uint32_t u0 = (uint32_t)pe[0] - ubase, u1 = (uint32_t)pe[1] - ubase;
                const uint32_t u2 = (uint32_t)pe[2] - ubase, u3 = (uint32_t)pe[3] - ubase;
                *reinterpret_cast<float4*>(a.upd + dq) =
                    XG ? make_float4(__ldg(xg + u0), __ldg(xg + u1), __ldg(xg + u2), __ldg(xg + u3))
                       : make_float4(xs[u0], xs[u1], xs[u2], xs[u3]);
              } else {
                for (uint32_t e = elo; e < ehi; ++e) {
                  const uint32_t u = (uint32_t)ps[e - sm.base] - ubase;
                  a.upd[e + dl] = XG ? __ldg(xg + u) : xs[u];
                }
              }
            }
            // next round starts after lane 31's quad
            const uint32_t g31 = __shfl_sync(0xffffffffu, gg, 31), r31 = __shfl_sync(0xffffffffu, rem, 31);
            gcur = g31;
            qcur = r31 + 1;
          }
        };
        auto range = [&](const int sr) {
          if constexpr (VEC) {
            range_vec(sr);
            return;
          }
        const uint32_t wb = sm.base + (uint32_t)(sr * kSub);
        const uint32_t wlo = max(wb, sm.lo), whi = min(wb + (uint32_t)kSub, sm.hi);
        if (wlo < whi) {
          // group of the sub-range's first entry from its precomputed grp_at anchor
          // (flat group p*k_dst + j), then advanced per lane as e crosses group
          // ends; (gend, delta) stay in registers between crossings
          const int32_t ga = (int32_t)(grp_s[stage * kScGrpCap + sm.gshift + (wb - sm.base) / kPngChunk] -
                                       (im.p * (uint32_t)a.k_dst + im.j0));
          uint32_t g = ga > 0 ? (uint32_t)ga : 0u;
          uint32_t gend = offs[g + 1];
          uint32_t delta = uos[g] - offs[g];                 // dst = e + delta within group g
          PCPM_UNROLL(PCPM_SCATTER_UNROLL)
          for (uint32_t e = wlo + lane; e < whi; e += 32) {
            if (e >= gend) {
              do {
                ++g;
                gend = offs[g + 1];
              } while (e >= gend);
              delta = uos[g] - offs[g];
            }
            const uint32_t u = (uint32_t)ps[e - sm.base] - ubase;
            a.upd[e + delta] = XG ? __ldg(xg + u) : xs[u];
          }
        }
        };
        for (int sr = cw; sr < (kNsr / kScW) * kScW; sr += kScW) range(sr);
        int who = rot;                                 // leftover sub-ranges rotate over the warps
        for (int sr = (kNsr / kScW) * kScW; sr < kNsr; ++sr) {
          if (cw == who) range(sr);
          who = (who + 1 == kScW) ? 0 : who + 1;
        }
        rot = who;
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == kScStages) { stage = 0; phase ^= 1; }
        if (sm.last) break;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(iempty);
    }
  }

  // last CTA resets the work counters (graph replays start from zero)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t done = atomicAdd(&a.counters[3], 1u);
    if (done == gridDim.x - 1) {
      a.counters[2] = 0u;
      a.counters[3] = 0u;
    }
  }
  (void)flag_s;
}

int scatter_tma_smem_bytes(int b, bool xg = false) {
  const int64_t q = xg ? 0 : int64_t(1) << b;          // XG reads the source values from global memory
  return (int)(((q * 4 + 127) & ~int64_t(127)) + 2 * kScOffCap * 4 + kScStages * kScStageBytes +
               kScStages * kScGrpCap * 4 + kScStages * sizeof(ScStageMeta) + sizeof(ScItemMeta) + (2 * kScStages + 2) * 8 + 16);
}

// ------------------------------------------------------------------ warp-per-group variant
constexpr int kUnroll = 8;

template <typename SrcT>
__global__ void __launch_bounds__(kScatterThreads, 1)
k_scatter_warp(const ScatterItem* __restrict__ items, int n_items, const float* __restrict__ x, int64_t n_src,
               int b, int64_t k_dst, const SrcT* __restrict__ png, const uint32_t* __restrict__ png_off,
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

int scatter_warp_smem_bytes(int b) {
  const int64_t q = int64_t(1) << b;
  return (int)(((q + 3) & ~int64_t(3)) * 4 + (2 * kScatterMaxGroups + 8) * 4);
}

}  // namespace

int prepare_scatter(pcpm_handle* h) {
  (void)h;
  PCPM_CK(cudaFuncSetAttribute(k_scatter_tma<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               scatter_tma_smem_bytes(kMaxBits)));
  PCPM_CK(cudaFuncSetAttribute(k_scatter_tma<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               scatter_tma_smem_bytes(kMaxBits)));
  PCPM_CK(cudaFuncSetAttribute(k_scatter_tma<uint16_t, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               scatter_tma_smem_bytes(kMaxBits)));
  PCPM_CK(cudaFuncSetAttribute(k_scatter_tma<uint32_t, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               scatter_tma_smem_bytes(kMaxBits)));
  PCPM_CK(cudaFuncSetAttribute(k_scatter_tma<uint16_t, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               scatter_tma_smem_bytes(kMaxBits)));
  PCPM_CK(cudaFuncSetAttribute(k_scatter_tma<uint32_t, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               scatter_tma_smem_bytes(kMaxBits)));
  PCPM_CK(cudaFuncSetAttribute(k_scatter_warp<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               scatter_warp_smem_bytes(kMaxBits)));
  PCPM_CK(cudaFuncSetAttribute(k_scatter_warp<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               scatter_warp_smem_bytes(kMaxBits)));
  return PCPM_OK;
}

int launch_scatter(pcpm_handle* h, const float* x, cudaStream_t s, float* out, bool split_only) {
  const ScatterItem* items = split_only ? h->sitems_split : h->sitems;
  const int n_items = split_only ? h->n_sitems_split : h->n_sitems;
  float* upd = out ? out : h->upd;
  if (n_items == 0) return PCPM_OK;
  const int grid = std::min(n_items, h->num_sms);
  // q = 2^16 (pair handles): a source partition's 256 KB slice does not fit in shared memory, so
  // the source values are read through L1/L2 (the XG kernel)
  if ((h->opt_scatter_variant == 1 && !h->pair) || h->b < 2) {   // the bulk-copy variant needs 16 B aligned slices
    const int smem = scatter_warp_smem_bytes(h->b);
    if (h->wide)
      k_scatter_warp<uint32_t><<<grid, kScatterThreads, smem, s>>>(items, n_items, x, h->n_src, h->b,
                                                                   h->k_dst, h->png_src, h->png_off, h->upd_off,
                                                                   upd);
    else
      k_scatter_warp<uint16_t><<<grid, kScatterThreads, smem, s>>>(items, n_items, x, h->n_src, h->b,
                                                                   h->k_dst, h->png16, h->png_off, h->upd_off,
                                                                   upd);
  } else {
    // the bulk copy of a source slice reads whole 16 B words: x must be 16 B aligned
    // and readable up to round16(n_src); internal vectors are padded, user vectors
    // that are not go through the padded staging buffer
    if ((reinterpret_cast<uintptr_t>(x) & 15) != 0 ||
        ((h->n_src & 3) != 0 && x != h->spr && x != h->xbuf)) {
      PCPM_CK(cudaMemcpyAsync(h->xbuf, x, sizeof(float) * h->n_src, cudaMemcpyDeviceToDevice, s));
      x = h->xbuf;
    }
    ScatterArgs a{};
    a.items = items;
    a.n_items = n_items;
    a.x = x;
    a.n_src = h->n_src;
    a.b = h->b;
    a.k_dst = h->k_dst;
    a.png = h->wide ? static_cast<const void*>(h->png_src) : static_cast<const void*>(h->png16);
    a.png_off = h->png_off;
    a.upd_off = h->upd_off;
    a.grp_at = h->grp_at;
    a.upd = upd;
    a.counters = h->counters;
    a.pf_stages = h->opt_scatter_pf;
    const bool xg = h->opt_scatter_variant == 2 || h->pair, vec = h->opt_scatter_variant == 3 && !h->pair;
    const int smem = scatter_tma_smem_bytes(h->b, xg);
    if (h->wide)
      PCPM_CK(launch_k(h->opt_pdl != 0,
                       xg ? k_scatter_tma<uint32_t, true> : vec ? k_scatter_tma<uint32_t, false, true> : k_scatter_tma<uint32_t>,
                       grid, ScCfg<uint32_t>::kThreads, smem, s, a));
    else
      PCPM_CK(launch_k(h->opt_pdl != 0,
                       xg ? k_scatter_tma<uint16_t, true> : vec ? k_scatter_tma<uint16_t, false, true> : k_scatter_tma<uint16_t>,
                       grid, ScCfg<uint16_t>::kThreads, smem, s, a));
  }
  PCPM_CK(cudaGetLastError());
  h->launches += 1;
  return PCPM_OK;
}

}  // namespace pcpm

// api.cu -- the C ABI of include/pcpm.h: handle lifecycle, the PageRank
// iteration driver (a4: init -> iters x [scatter -> gather+apply], captured in
// a CUDA graph), SpMV (a5), the pull comparison, and introspection.
#include <cmath>
#include <cstring>
#include <string>

#include "pcpm_internal.cuh"

namespace pcpm {

namespace {
thread_local int g_status = 0;
thread_local std::string g_msg;

int ceil_log2(uint64_t x) {
  int r = 0;
  while ((uint64_t(1) << r) < x) ++r;
  return r;
}
}  // namespace

void set_error(int code, const std::string& msg) {
  g_status = code;
  g_msg = msg;
}

int cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  char buf[512];
  snprintf(buf, sizeof(buf), "%s failed: %s (%s:%d)", what, cudaGetErrorString(e), file, line);
  int code = (e == cudaErrorMemoryAllocation) ? PCPM_ENOMEM : PCPM_ECUDA;
  cudaGetLastError();
  set_error(code, buf);
  return code;
}

// Device memory comes from the stream-ordered default pool (cudaMallocAsync on the
// handle's stream), kept cached between builds: repeated builds (the e2e path) then
// skip the synchronous cudaMalloc/cudaFree of multi-GB buffers.
void pool_setup(int device) {
  static bool done[64] = {false};
  if (device < 0 || device >= 64 || done[device]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  cudaGetLastError();
  done[device] = true;
}

}  // namespace pcpm

extern "C" int pcpm_pool_reserve(int64_t bytes) {
  using namespace pcpm;
  if (bytes < 0) {
    set_error(PCPM_EINVAL, "bytes < 0");
    return PCPM_EINVAL;
  }
  if (bytes == 0) return PCPM_OK;
  int dev = 0;
  PCPM_CK(cudaGetDevice(&dev));
  pool_setup(dev);
  cudaStream_t s;
  PCPM_CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  void* p = nullptr;
  const cudaError_t e = cudaMallocAsync(&p, (size_t)bytes, s);
  if (e != cudaSuccess) {
    cudaGetLastError();
    cudaStreamDestroy(s);
    set_error(PCPM_ENOMEM, "pool reserve of " + std::to_string(bytes) + " bytes failed: " + cudaGetErrorString(e));
    return PCPM_ENOMEM;
  }
  cudaFreeAsync(p, s);
  const cudaError_t e2 = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  PCPM_CK(e2);
  return PCPM_OK;
}

namespace pcpm {

int dev_alloc(pcpm_handle* h, void** p, size_t bytes) {
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMallocAsync(p, bytes, h->stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error(PCPM_ENOMEM, "cudaMalloc of " + std::to_string(bytes) + " bytes failed: " + cudaGetErrorString(e));
    *p = nullptr;
    return PCPM_ENOMEM;
  }
  h->allocs.push_back(*p);
  h->device_bytes += (int64_t)bytes;
  return PCPM_OK;
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes attr;
  cudaError_t e = cudaPointerGetAttributes(&attr, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

namespace {

void free_graph(pcpm_handle* h) {
  if (h->graph.exec) cudaGraphExecDestroy(h->graph.exec);
  h->graph = Graph{};
}

int ensure_red(pcpm_handle* h, int iters) {
  const int need = 2 * (iters + 2);
  if (h->red_cap >= need) return PCPM_OK;
  if (h->red) {
    cudaFreeAsync(h->red, h->stream);
    for (auto& p : h->allocs)
      if (p == h->red) p = nullptr;
    h->red = nullptr;
  }
  free_graph(h);
  int cap = std::max(need, 64);
  int rc = dev_alloc_t(h, &h->red, cap);
  if (rc) return rc;
  h->red_cap = cap;
  return PCPM_OK;
}

int pr_fixed_bits(int64_t n) {
  // F: typical SPR ~ 1/(n*deg) lands near 2^22 in the low word; PR <= 1 so the
  // u64 never overflows; resolution 2^-(F+1) ~ 1e-8 (1-d)/n per term.
#ifndef PCPM_PR_FBASE
#define PCPM_PR_FBASE 26
#endif
  return std::min(60, std::max(30, PCPM_PR_FBASE + ceil_log2((uint64_t)n)));
}

GatherArgs base_args(pcpm_handle* h, int fbits) {
  GatherArgs a{};
  a.ids = h->wide ? static_cast<const void*>(h->ids) : static_cast<const void*>(h->ids16);
  a.slot16 = h->wide ? nullptr : h->slot16;
  a.acc_words = h->slot16 ? h->acc_words : (int)(int64_t(1) << h->gb);
  a.slotmap = h->wide ? nullptr : h->slotmap;
  a.w = h->w;
  a.upd = h->upd;
  a.chunk_base = h->chunk_base;
  a.items = h->gitems;
  a.n_items = h->n_gitems;
  a.bin_nslices = h->bin_nslices;
  a.counters = h->counters;
  a.slot_buf = h->slot_buf;
  a.bin_slot_base = h->bin_slot_base;
  a.has_split = h->n_split_bins > 0;
  a.bin_arrive = h->bin_arrive;
  a.hi = h->hi;
  a.red_fx = h->red_fx;
  a.b = h->gb;
  a.pair = h->pair ? 1 : 0;
  a.n_dst = h->n_dst;
  a.fbits = fbits;
  a.inv_deg = h->inv_deg + h->shard_lo;  // apply: 1 / global out-degree of destination v (shards: lo + v)
  a.epi_pf = h->opt_epi_pf;
  a.pf_tiles = h->opt_gather_pf;
  a.png16 = h->png16;
  a.png_off = h->png_off;
  a.upd_off = h->upd_off;
  a.grp_at = h->grp_at;
  a.k_dst = h->k_dst;
  return a;
}

int mark(pcpm_handle* h, cudaStream_t s) {
  if (!h->opt_phase_timing) return PCPM_OK;
  if ((int)h->events.size() <= h->n_events_used) {
    cudaEvent_t e;
    PCPM_CK(cudaEventCreate(&e));
    h->events.push_back(e);
  }
  // inside stream capture an event record must be an external node to be timeable
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  PCPM_CK(cudaStreamIsCapturing(s, &st));
  const unsigned fl = (st == cudaStreamCaptureStatusActive) ? cudaEventRecordExternal : cudaEventRecordDefault;
  PCPM_CK(cudaEventRecordWithFlags(h->events[h->n_events_used++], s, fl));
  return PCPM_OK;
}

// Iteration t of Eq. 1: scatter (Alg. 4) then gather (Alg. 5) + apply, PR_t in
// pr[t & 1] -> PR_{t+1} in pr_new; red[2t] = D_t in, red[2t+1] = residual, red[2t+2] = D_{t+1}.
int enqueue_iteration(pcpm_handle* h, double d, int t, float* pr_new, cudaStream_t s) {
  int rc;
  const bool wpr = h->opt_weighted_pr && h->inv_wdeg && h->w;      // weighted PageRank (R24)
  if ((rc = h->bvgas ? launch_bvgas_scatter(h, h->spr, s) : launch_scatter(h, h->spr, s))) return rc;   // Alg. 4 / Alg. 3
  if ((rc = mark(h, s))) return rc;
  GatherArgs a = base_args(h, h->fixed_bits);
  a.d = d;
  a.n = (double)h->n_src;
  a.red_in = h->red + 2 * t;
  a.res_out = h->red + 2 * t + 1;
  a.dang_out = h->red + 2 * t + 2;
  a.pr_old = h->pr[t & 1];
  a.pr_new = pr_new;
  a.spr_new = h->spr;
  if (wpr) a.inv_deg = h->inv_wdeg;                              // 1/W(u): the weights' normalisation
  if ((rc = launch_gather(h, a, wpr, true, s))) return rc;        // Alg. 5 (+ weights) + apply
  return mark(h, s);
}

// The fused iteration (gather + apply + the next iteration's scatter in one kernel, DESIGN.md
// §5) applies to square, compact, single-GPU handles on the persistent gather path.
bool fused_ok(const pcpm_handle* h) {
  return h->opt_fuse && !h->bvgas && !h->wide && !h->shard && h->n_src == h->n_dst && h->k_src == h->k_dst && !h->slot16 &&
         !(h->cl_cs >= 2 && h->opt_cluster_gather) && h->opt_gather_variant == 1 && h->e_prime > 0;
}

int enqueue_pagerank(pcpm_handle* h, double d, int iters, float* dst, cudaStream_t s) {
  int rc;
  const int fbits = pr_fixed_bits(h->n_src);
  h->fixed_bits = fbits;
  h->last_was_spmv = false;
  h->n_events_used = 0;
  if ((rc = mark(h, s))) return rc;
  const bool wpr = h->opt_weighted_pr && h->inv_wdeg && h->w;      // weighted PageRank (R24)
  if (wpr) {
    if ((rc = launch_pr_init_weighted(h, h->pr[0], h->spr, h->red, h->red_cap, std::ldexp(1.0f, fbits), s))) return rc;
  } else if ((rc = launch_pr_init(h, h->pr[0], h->spr, h->red, h->red_cap, std::ldexp(1.0, fbits), s))) {
    return rc;
  }
  if ((rc = mark(h, s))) return rc;
  if (iters == 0) {
    PCPM_CK(cudaMemcpyAsync(dst, h->pr[0], sizeof(float) * h->n_src, cudaMemcpyDeviceToDevice, s));
    return PCPM_OK;
  }
  h->last_fused = fused_ok(h) && h->upd2 != nullptr && iters > 1;
  if (!h->last_fused) {
    for (int t = 0; t < iters; ++t)
      if ((rc = enqueue_iteration(h, d, t, (t == iters - 1) ? dst : h->pr[(t + 1) & 1], s))) return rc;
    return PCPM_OK;
  }
  // fused: scatter of SPR_0 (Alg. 4), then per iteration one kernel that gathers the bins of
  // iteration t (buffer t & 1), applies, and scatters SPR_{t+1} into buffer (t + 1) & 1
  float* bins[2] = {h->upd, h->upd2};
  if ((rc = launch_scatter(h, h->spr, s, bins[0]))) return rc;
  if ((rc = mark(h, s))) return rc;
  for (int t = 0; t < iters; ++t) {
    const bool fuse = t < iters - 1;
    GatherArgs a = base_args(h, h->fixed_bits);
    a.d = d;
    a.n = (double)h->n_src;
    a.red_in = h->red + 2 * t;
    a.res_out = h->red + 2 * t + 1;
    a.dang_out = h->red + 2 * t + 2;
    a.pr_old = h->pr[t & 1];
    a.pr_new = (t == iters - 1) ? dst : h->pr[(t + 1) & 1];
    a.spr_new = h->spr;
    a.upd = bins[t & 1];
    a.upd_next = bins[(t + 1) & 1];
    if (wpr) a.inv_deg = h->inv_wdeg;
    if ((rc = launch_gather(h, a, wpr, true, s, false, fuse))) return rc;
    // split partitions: k_apply_split wrote their SPR to global memory; scatter them now
    if (fuse && h->n_sitems_split && (rc = launch_scatter(h, h->spr, s, bins[(t + 1) & 1], true))) return rc;
    if ((rc = mark(h, s))) return rc;
  }
  return PCPM_OK;
}

int enqueue_pull(pcpm_handle* h, double d, int iters, float* dst, cudaStream_t s) {
  int rc;
  float* sprb[2] = {h->spr, h->xbuf};
  h->n_events_used = 0;
  if ((rc = mark(h, s))) return rc;
  if ((rc = launch_pr_init(h, h->pr[0], sprb[0], h->red, h->red_cap, 1.0, s))) return rc;
  if ((rc = mark(h, s))) return rc;
  if (iters == 0) {
    PCPM_CK(cudaMemcpyAsync(dst, h->pr[0], sizeof(float) * h->n_src, cudaMemcpyDeviceToDevice, s));
    return PCPM_OK;
  }
  for (int t = 0; t < iters; ++t) {
    float* pr_new = (t == iters - 1) ? dst : h->pr[(t + 1) & 1];
    if ((rc = launch_pull_iteration(h, sprb[t & 1], h->pr[t & 1], pr_new, sprb[(t + 1) & 1], h->red + 2 * t, d, s)))
      return rc;
    if ((rc = mark(h, s))) return rc;
  }
  return PCPM_OK;
}

int run_captured(pcpm_handle* h, int kind, double d, int iters, float* dst) {
  cudaStream_t s = h->stream;
  auto enq = [&](cudaStream_t st) { return kind == 0 ? enqueue_pagerank(h, d, iters, dst, st)
                                                      : enqueue_pull(h, d, iters, dst, st); };
  h->launches = 0;
  if (!h->opt_use_graph) return enq(s);
  Graph& g = h->graph;
  if (!(g.exec && g.iters == iters && g.d == d && g.out == dst && g.kind == kind)) {
    free_graph(h);
    cudaStream_t cs;
    PCPM_CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaGraph_t graph;
    cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) {
      cudaStreamDestroy(cs);
      return cuda_fail(e, "cudaStreamBeginCapture", __FILE__, __LINE__);
    }
    int rc = enq(cs);
    e = cudaStreamEndCapture(cs, &graph);
    cudaStreamDestroy(cs);
    if (rc) {
      if (e == cudaSuccess) cudaGraphDestroy(graph);
      return rc;
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture", __FILE__, __LINE__);
    e = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate", __FILE__, __LINE__);
    g.iters = iters;
    g.d = d;
    g.out = dst;
    g.kind = kind;
    g.launches = h->launches;
  }
  h->launches = g.launches;
  PCPM_CK(cudaGraphLaunch(g.exec, s));
  return PCPM_OK;
}

int pagerank_common(pcpm_handle* h, double d, int iters, float* out, int kind) {
  if (!h || !out) {
    set_error(PCPM_EINVAL, "NULL handle or output");
    return PCPM_EINVAL;
  }
  if (!(d > 0.0 && d < 1.0) || iters < 0) {
    set_error(PCPM_EINVAL, "d must be in (0,1) and iters >= 0");
    return PCPM_EINVAL;
  }
  if (h->n_src != h->n_dst) {
    set_error(PCPM_ESTATE, "PageRank needs a square matrix (n_src == n_dst)");
    return PCPM_ESTATE;
  }
  if (kind == 1 && !h->has_pull) {
    set_error(PCPM_ESTATE, "pcpm_pull_pagerank needs a handle built with PCPM_BUILD_PULL");
    return PCPM_ESTATE;
  }
  int rc = ensure_red(h, iters);
  if (rc) return rc;
  if (kind == 0 && fused_ok(h) && !h->upd2 && iters > 1) {   // second update-bin buffer of the fused path
    if ((rc = dev_alloc_t(h, &h->upd2, h->e_prime + 8))) return rc;
    PCPM_CK(cudaMemsetAsync(h->upd2, 0, sizeof(float) * (h->e_prime + 8), h->stream));
  }
  // refreshed on every call: a cached graph skips enqueue_pagerank, which also sets them
  h->fixed_bits = kind == 0 ? pr_fixed_bits(h->n_src) : 0;
  h->last_was_spmv = false;
  const bool dev_out = is_device_ptr(out);
  float* dst = dev_out ? out : h->ybuf;
  rc = run_captured(h, kind, d, iters, dst);
  if (rc) return rc;
  h->last_iters = iters;
  if (!dev_out) {
    PCPM_CK(cudaMemcpyAsync(out, dst, sizeof(float) * h->n_src, cudaMemcpyDeviceToHost, h->stream));
    PCPM_CK(cudaStreamSynchronize(h->stream));
  }
  return PCPM_OK;
}

}  // namespace
}  // namespace pcpm

using namespace pcpm;

extern "C" {

static pcpm_handle* build_common(const pcpm_csr* csr, int partition_bits, unsigned flags, void* cuda_stream,
                                 int64_t lo, int64_t hi) {
  set_error(PCPM_OK, "");
  if (!csr || !csr->row_ptr || (csr->nnz > 0 && !csr->col_idx)) {
    set_error(PCPM_EINVAL, "NULL csr / row_ptr / col_idx");
    return nullptr;
  }
  if (partition_bits < 1 || partition_bits > kMaxBitsPair || (partition_bits > kMaxBits && lo >= 0)) {
    set_error(PCPM_EINVAL, "partition_bits must be in [1, 16] (shards: [1, 15])");
    return nullptr;
  }
  // q = 2^16: 4-byte IDs, two half-partition gather items per bin (pcpm.h)
  if (partition_bits > kMaxBits) flags |= PCPM_WIDE_IDS;
  if (csr->n_src < 1 || csr->n_dst < 1 || csr->nnz < 0) {
    set_error(PCPM_EINVAL, "n_src, n_dst must be >= 1 and nnz >= 0");
    return nullptr;
  }
  if (csr->n_src >= (int64_t(1) << 31) || csr->n_dst >= (int64_t(1) << 31)) {
    set_error(PCPM_ETOOBIG, "n >= 2^31: the MSB of a 4-byte ID is the run flag (P:172-173)");
    return nullptr;
  }
  if (csr->nnz >= (int64_t(1) << 32) - kTileIds) {
    set_error(PCPM_ETOOBIG, "nnz >= 2^32: bin positions are 32-bit");
    return nullptr;
  }
  const int64_t q = int64_t(1) << partition_bits;
  const int64_t ks = (csr->n_src + q - 1) / q, kd = (csr->n_dst + q - 1) / q;
  if (ks * kd > (int64_t(1) << 28)) {
    set_error(PCPM_ETOOBIG, "k_src * k_dst > 2^28: the O(k^2) offset matrices (P:148) are too large");
    return nullptr;
  }
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    set_error(PCPM_ECUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    return nullptr;
  }
  pcpm_handle* h = new pcpm_handle();
  h->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
  h->b = partition_bits;
  h->gb = std::min(partition_bits, kMaxBits);
  h->pair = partition_bits > kMaxBits;
  if (h->pair) h->opt_pdl = 0;
  cudaGetDevice(&h->device);
  pool_setup(h->device);
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, h->stream);
  int rc = prepare_gather(h);
  if (rc == PCPM_OK) rc = prepare_scatter(h);
  if (rc == PCPM_OK) {
    if (lo < 0) {
      rc = build_layout(h, csr, flags);
      h->n_global = h->n_dst;
    } else {
      h->shard = true;
      rc = build_shard_layout(h, csr, lo, hi, flags);
    }
  }
  if (rc == PCPM_OK) {
    cudaEventRecord(e1, h->stream);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    h->build_ms = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (rc != PCPM_OK) {
    int st = g_status;
    std::string msg = g_msg;
    pcpm_destroy(h);
    set_error(st ? st : rc, msg);
    return nullptr;
  }
  return h;
}

pcpm_handle* pcpm_build_ex(const pcpm_csr* csr, int partition_bits, unsigned flags, void* cuda_stream) {
  return build_common(csr, partition_bits, flags, cuda_stream, -1, -1);
}

pcpm_handle* pcpm_build_shard(const pcpm_csr* csr, int partition_bits, int64_t v_lo, int64_t v_hi, unsigned flags,
                              void* cuda_stream) {
  set_error(PCPM_OK, "");
  if (!csr || partition_bits < 1 || partition_bits > kMaxBits) {
    set_error(PCPM_EINVAL, "NULL csr or partition_bits not in [1, 15]");
    return nullptr;
  }
  if (v_lo < 0 || v_hi <= v_lo || v_hi > csr->n_dst || (v_lo & ((int64_t(1) << partition_bits) - 1)) != 0) {
    set_error(PCPM_EINVAL, "shard range must satisfy 0 <= v_lo < v_hi <= n_dst with v_lo a multiple of 2^b");
    return nullptr;
  }
  if (flags & (PCPM_BUILD_PULL | PCPM_NO_COMPRESS)) {
    set_error(PCPM_EINVAL, "shard handles take only PCPM_WIDE_IDS / PCPM_KEEP_VALUES");
    return nullptr;
  }
  if (csr->n_dst >= (int64_t(1) << 31)) {
    set_error(PCPM_ETOOBIG, "n >= 2^31: the MSB of a 4-byte ID is the run flag (P:172-173)");
    return nullptr;
  }
  if (csr->n_src != csr->n_dst) {
    // the apply reads the global out-degrees of the slice's vertices (outdeg + v_lo): the
    // graph must be square (PageRank, Eq. 1)
    set_error(PCPM_ESTATE, "pcpm_build_shard needs a square graph (n_src == n_dst)");
    return nullptr;
  }
  return build_common(csr, partition_bits, flags, cuda_stream, v_lo, v_hi);
}

int pcpm_shard_init(pcpm_handle* h, float* pr0, float* spr0, double* dang0) {
  if (!h || !pr0 || !spr0 || !dang0) {
    set_error(PCPM_EINVAL, "NULL handle or output");
    return PCPM_EINVAL;
  }
  if (!is_device_ptr(pr0) || !is_device_ptr(spr0) || !is_device_ptr(dang0)) {
    set_error(PCPM_EINVAL, "pcpm_shard_init takes device pointers");
    return PCPM_EINVAL;
  }
  h->launches = 0;
  return launch_pr_init_slice(h, pr0, spr0, dang0, std::ldexp(1.0, pr_fixed_bits(h->n_global)), h->stream);
}

static int shard_step_common(pcpm_handle* h, double d, const float* spr_in, const double* D_in, const float* pr_old,
                             float* pr_new, float* const* outs, int n_outs, double* red_out, const char* fn) {
  if (!h || !spr_in || !D_in || !pr_old || !pr_new || !outs || !red_out) {
    set_error(PCPM_EINVAL, "NULL handle or argument");
    return PCPM_EINVAL;
  }
  if (n_outs < 1 || n_outs > 1 + kMaxPeers) {
    set_error(PCPM_EINVAL, "n_outs must be in [1, PCPM_MAX_PEERS + 1]");
    return PCPM_EINVAL;
  }
  if (!(d > 0.0 && d < 1.0)) {
    set_error(PCPM_EINVAL, "d must be in (0,1)");
    return PCPM_EINVAL;
  }
  bool dev = is_device_ptr(spr_in) && is_device_ptr(D_in) && is_device_ptr(pr_old) && is_device_ptr(pr_new) &&
             is_device_ptr(red_out);
  for (int i = 0; i < n_outs; ++i) dev = dev && outs[i] && is_device_ptr(outs[i]);
  if (!dev) {
    set_error(PCPM_EINVAL, std::string(fn) + " takes device pointers");
    return PCPM_EINVAL;
  }
  if (!h->shard && h->n_src != h->n_dst) {
    set_error(PCPM_ESTATE, std::string(fn) + " needs a shard handle or a square matrix");
    return PCPM_ESTATE;
  }
  if (n_outs > 1 && h->slot16) {
    // the fused-exchange gather indexes its accumulator by vertex, not by slot
    set_error(PCPM_ESTATE, std::string(fn) + ": handles built with PCPM_COMPACT_SLOTS take n_outs == 1");
    return PCPM_ESTATE;
  }
  cudaStream_t s = h->stream;
  h->launches = 0;
  const int fbits = pr_fixed_bits(h->n_global);
  h->fixed_bits = fbits;
  h->last_was_spmv = false;
  int rc = launch_scatter(h, spr_in, s);                     // Alg. 4 over all source partitions
  if (rc) return rc;
  GatherArgs a = base_args(h, fbits);
  a.d = d;
  a.n = (double)h->n_global;
  a.red_in = D_in;
  a.res_out = red_out;
  a.dang_out = red_out + 1;
  a.pr_old = pr_old;
  a.pr_new = pr_new;
  a.spr_new = outs[0];
  a.n_peer = n_outs - 1;
  for (int i = 1; i < n_outs; ++i) a.spr_peer[i - 1] = outs[i];
  return launch_gather(h, a, false, true, s, n_outs > 1);   // Alg. 5 + apply on the shard's vertices
}

int pcpm_shard_step(pcpm_handle* h, double d, const float* spr_in, const double* D_in, const float* pr_old,
                    float* pr_new, float* spr_out, double* red_out) {
  float* outs[1] = {spr_out};
  return shard_step_common(h, d, spr_in, D_in, pr_old, pr_new, spr_out ? outs : nullptr, 1, red_out,
                           "pcpm_shard_step");
}

int pcpm_shard_step_peers(pcpm_handle* h, double d, const float* spr_in, const double* D_in, const float* pr_old,
                          float* pr_new, float* const* spr_outs, int n_outs, double* red_out) {
  return shard_step_common(h, d, spr_in, D_in, pr_old, pr_new, spr_outs, n_outs, red_out, "pcpm_shard_step_peers");
}

int pcpm_shard_init_peers(pcpm_handle* h, float* pr0, float* const* spr_outs, int n_outs, double* dang0) {
  if (!spr_outs || n_outs < 1 || n_outs > 1 + kMaxPeers) {
    set_error(PCPM_EINVAL, "spr_outs must hold 1 .. PCPM_MAX_PEERS + 1 pointers");
    return PCPM_EINVAL;
  }
  for (int i = 0; i < n_outs; ++i)
    if (!spr_outs[i] || !is_device_ptr(spr_outs[i])) {
      set_error(PCPM_EINVAL, "pcpm_shard_init_peers takes device pointers");
      return PCPM_EINVAL;
    }
  int rc = pcpm_shard_init(h, pr0, spr_outs[0], dang0);
  if (rc) return rc;
  for (int i = 1; i < n_outs; ++i)           // SPR_0 of the slice to the peers (once per run)
    PCPM_CK(cudaMemcpyAsync(spr_outs[i], spr_outs[0], sizeof(float) * h->n_dst, cudaMemcpyDefault, h->stream));
  return PCPM_OK;
}

int pcpm_ipc_handle_bytes(void) { return (int)sizeof(cudaIpcMemHandle_t); }

int pcpm_ipc_alloc(int64_t bytes, void** dev_ptr) {
  if (!dev_ptr || bytes <= 0) {
    set_error(PCPM_EINVAL, "NULL output or bytes <= 0");
    return PCPM_EINVAL;
  }
  *dev_ptr = nullptr;
  const cudaError_t e = cudaMalloc(dev_ptr, (size_t)bytes);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    set_error(PCPM_ENOMEM, "cudaMalloc of an exchange buffer failed");
    return PCPM_ENOMEM;
  }
  PCPM_CK(e);
  PCPM_CK(cudaMemset(*dev_ptr, 0, (size_t)bytes));
  return PCPM_OK;
}

int pcpm_ipc_free(void* dev_ptr) {
  if (dev_ptr) PCPM_CK(cudaFree(dev_ptr));
  return PCPM_OK;
}

int pcpm_ipc_get_handle(void* dev_ptr, void* handle_out) {
  if (!dev_ptr || !handle_out) {
    set_error(PCPM_EINVAL, "NULL pointer or handle buffer");
    return PCPM_EINVAL;
  }
  cudaIpcMemHandle_t hd;
  PCPM_CK(cudaIpcGetMemHandle(&hd, dev_ptr));
  memcpy(handle_out, &hd, sizeof(hd));
  return PCPM_OK;
}

int pcpm_ipc_open(const void* handle, void** dev_ptr_out) {
  if (!handle || !dev_ptr_out) {
    set_error(PCPM_EINVAL, "NULL handle or output");
    return PCPM_EINVAL;
  }
  cudaIpcMemHandle_t hd;
  memcpy(&hd, handle, sizeof(hd));
  PCPM_CK(cudaIpcOpenMemHandle(dev_ptr_out, hd, cudaIpcMemLazyEnablePeerAccess));
  return PCPM_OK;
}

int pcpm_ipc_close(void* dev_ptr) {
  if (dev_ptr) PCPM_CK(cudaIpcCloseMemHandle(dev_ptr));
  return PCPM_OK;
}

pcpm_handle* pcpm_build(const pcpm_csr* csr, int partition_bits) {
  return pcpm_build_ex(csr, partition_bits, 0u, nullptr);
}

int pcpm_pagerank(pcpm_handle* h, double d, int iters, float* out) { return pagerank_common(h, d, iters, out, 0); }

int pcpm_pagerank_tol(pcpm_handle* h, double d, double tol, int max_iters, float* out, int* iters_done) {
  if (!h || !out || !iters_done) {
    set_error(PCPM_EINVAL, "NULL handle, output or iters_done");
    return PCPM_EINVAL;
  }
  if (!(d > 0.0 && d < 1.0) || max_iters < 1 || !(tol >= 0.0)) {
    set_error(PCPM_EINVAL, "d must be in (0,1), max_iters >= 1, tol >= 0");
    return PCPM_EINVAL;
  }
  if (h->n_src != h->n_dst) {
    set_error(PCPM_ESTATE, "PageRank needs a square matrix (n_src == n_dst)");
    return PCPM_ESTATE;
  }
  int rc = ensure_red(h, max_iters);
  if (rc) return rc;
  if (!h->res_host) PCPM_CK(cudaMallocHost(reinterpret_cast<void**>(&h->res_host), sizeof(double) * 2));
  cudaStream_t s = h->stream;
  h->launches = 0;
  h->opt_phase_timing_saved = h->opt_phase_timing;
  h->opt_phase_timing = 0;                     // no event bookkeeping on this path
  const int fbits = pr_fixed_bits(h->n_src);
  h->fixed_bits = fbits;
  h->last_was_spmv = false;
  h->n_events_used = 0;
  const bool wpr = h->opt_weighted_pr && h->inv_wdeg && h->w;
  rc = wpr ? launch_pr_init_weighted(h, h->pr[0], h->spr, h->red, h->red_cap, std::ldexp(1.0f, fbits), s)
           : launch_pr_init(h, h->pr[0], h->spr, h->red, h->red_cap, std::ldexp(1.0, fbits), s);
  // One iteration in flight: iteration t is enqueued before the host looks at the
  // residual of iteration t - 1 (copied to pinned memory behind an event).  If that
  // residual is <= tol the result is PR_t, in pr[t & 1], which iteration t only reads.
  int done = max_iters;
  cudaEvent_t ev = nullptr;
  if (!rc && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) rc = PCPM_ECUDA;
  for (int t = 0; t < max_iters && !rc; ++t) {
    if ((rc = enqueue_iteration(h, d, t, h->pr[(t + 1) & 1], s))) break;
    if (t > 0) {
      if (cudaEventSynchronize(ev) != cudaSuccess) { rc = PCPM_ECUDA; break; }
      if (h->res_host[0] <= tol) {               // sum |PR_t - PR_{t-1}| <= tol
        done = t;
        break;
      }
    }
    if (cudaMemcpyAsync(h->res_host, h->red + 2 * t + 1, sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaEventRecord(ev, s) != cudaSuccess) {
      rc = PCPM_ECUDA;
      break;
    }
  }
  if (ev) cudaEventDestroy(ev);
  h->opt_phase_timing = h->opt_phase_timing_saved;
  if (rc) {
    if (rc == PCPM_ECUDA) set_error(PCPM_ECUDA, "CUDA error in pcpm_pagerank_tol");
    return rc;
  }
  if (done == max_iters) {                       // the last iteration's residual
    PCPM_CK(cudaStreamSynchronize(s));
  }
  h->last_iters = done;
  *iters_done = done;
  PCPM_CK(cudaMemcpyAsync(out, h->pr[done & 1], sizeof(float) * h->n_src, cudaMemcpyDefault, s));
  PCPM_CK(cudaStreamSynchronize(s));
  return PCPM_OK;
}

int pcpm_pull_pagerank(pcpm_handle* h, double d, int iters, float* out) {
  return pagerank_common(h, d, iters, out, 1);
}

int pcpm_spmv(pcpm_handle* h, const float* x, float* y) {
  if (!h || !x || !y) {
    set_error(PCPM_EINVAL, "NULL handle, x or y");
    return PCPM_EINVAL;
  }
  cudaStream_t s = h->stream;
  const bool dev_x = is_device_ptr(x), dev_y = is_device_ptr(y);
  const float* xd = x;
  if (!dev_x) {
    PCPM_CK(cudaMemcpyAsync(h->xbuf, x, sizeof(float) * h->n_src, cudaMemcpyHostToDevice, s));
    xd = h->xbuf;
  }
  float* yd = dev_y ? y : h->ybuf;
  h->launches = 0;
  int rc = launch_absmax(h, xd, h->n_src, h->xmax, s);                    // fixed-point scale of this x
  if (rc) return rc;
  rc = h->bvgas ? launch_bvgas_scatter(h, xd, s) : launch_scatter(h, xd, s);   // Alg. 4 (Alg. 3) on x
  if (rc) return rc;
  h->last_was_spmv = true;
  GatherArgs a = base_args(h, 0);
  a.y = yd;
  a.xmax = h->xmax;
  a.wexp = h->weighted ? h->wexp : 0;
  rc = launch_gather(h, a, h->weighted, false, s);                         // Alg. 5 with weights (§3.5)
  if (rc) return rc;
  if (!dev_y) {
    PCPM_CK(cudaMemcpyAsync(y, yd, sizeof(float) * h->n_dst, cudaMemcpyDeviceToHost, s));
    PCPM_CK(cudaStreamSynchronize(s));
  }
  return PCPM_OK;
}

int pcpm_scatter(pcpm_handle* h, const float* x) {
  if (!h || !x) {
    set_error(PCPM_EINVAL, "NULL handle or x");
    return PCPM_EINVAL;
  }
  const float* xd = x;
  if (!is_device_ptr(x)) {
    PCPM_CK(cudaMemcpyAsync(h->xbuf, x, sizeof(float) * h->n_src, cudaMemcpyHostToDevice, h->stream));
    xd = h->xbuf;
  }
  h->launches = 0;
  return h->bvgas ? launch_bvgas_scatter(h, xd, h->stream) : launch_scatter(h, xd, h->stream);
}

void pcpm_destroy(pcpm_handle* h) {
  if (!h) return;
  if (h->stream) cudaStreamSynchronize(h->stream);
  else cudaDeviceSynchronize();
  free_graph(h);
  for (cudaEvent_t e : h->events) cudaEventDestroy(e);
  for (void* p : h->allocs)
    if (p) cudaFreeAsync(p, h->stream);
  if (h->res_host) cudaFreeHost(h->res_host);
  delete h;
}

int pcpm_set_stream(pcpm_handle* h, void* cuda_stream) {
  if (!h) {
    set_error(PCPM_EINVAL, "NULL handle");
    return PCPM_EINVAL;
  }
  // the handle's scratch (counters, carries, update bins, reductions) is shared by
  // every call: work queued on the old stream completes before the new stream is used
  PCPM_CK(cudaStreamSynchronize(h->stream));
  h->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
  return PCPM_OK;
}

int pcpm_last_error(char* buf, int cap) {
  const int len = (int)g_msg.size();
  if (buf && cap > 0) {
    const int k = std::min(len, cap - 1);
    memcpy(buf, g_msg.data(), k);
    buf[k] = 0;
  }
  return len;
}

int pcpm_last_status(void) { return g_status; }

int pcpm_get_info(const pcpm_handle* h, pcpm_info* out) {
  if (!h || !out) {
    set_error(PCPM_EINVAL, "NULL handle or info");
    return PCPM_EINVAL;
  }
  pcpm_info i{};
  i.n_src = h->n_src;
  i.n_dst = h->n_dst;
  i.nnz = h->m;
  i.partition_bits = h->b;
  i.q = h->q;
  i.k_src = h->k_src;
  i.k_dst = h->k_dst;
  i.e_prime = h->e_prime;
  i.r = h->e_prime ? (double)h->m / (double)h->e_prime : 0.0;
  i.n_dangling = h->n_dangling;
  i.weighted = h->weighted;
  i.compressed = h->compressed;
  i.device_bytes = h->device_bytes;
  i.build_ms = h->build_ms;
  i.gather_items = h->n_gitems;
  i.scatter_items = h->n_sitems;
  i.fixed_point_bits = h->fixed_bits;
  i.compact_slots = h->slot16 ? 1 : 0;
  i.bvgas = h->bvgas ? 1 : 0;
  i.fused_iterations = h->last_fused ? 1 : 0;
  if (h->last_was_spmv && h->xmax) {   // same rule as spmv_fbits() in gather.cu
    float xm = 0.f;
    if (cudaMemcpy(&xm, h->xmax, 4, cudaMemcpyDeviceToHost) == cudaSuccess) {
      int ex = 0;
      if (xm > 0.f) frexpf(xm, &ex);
      const int F = kSpmvHead - (h->weighted ? h->wexp : 0) - ex;
      i.fixed_point_bits = F < -120 ? -120 : (F > 62 ? 62 : F);
    } else {
      cudaGetLastError();
    }
  }
  *out = i;
  return PCPM_OK;
}

int pcpm_export_layout(pcpm_handle* h, pcpm_layout_view* out) {
  if (!h || !out) {
    set_error(PCPM_EINVAL, "NULL handle or view");
    return PCPM_EINVAL;
  }
  pcpm_layout_view v{};
  v.ids = h->ids;
  v.w = h->w;
  v.png_src = h->png_src;
  v.png_off = h->png_off;
  v.upd_off = h->upd_off;
  v.bin_id_start = h->bin_id_start;
  v.bin_upd_start = h->bin_upd_start;
  v.chunk_base = h->chunk_base;
  v.out_degree = h->outdeg;
  v.upd = h->upd;
  v.chunk_ids = kChunkIds;
  v.ids16 = h->ids16;
  v.png_src16 = h->png16;
  v.wide = h->wide ? 1 : 0;
  *out = v;
  return PCPM_OK;
}

int pcpm_get_residuals(pcpm_handle* h, double* host, int cap) {
  if (!h || !host) {
    set_error(PCPM_EINVAL, "NULL handle or buffer");
    return PCPM_EINVAL;
  }
  if (!h->red) return 0;
  const int n = std::min(cap, 2 * (h->last_iters + 1));
  PCPM_CK(cudaMemcpyAsync(host, h->red, sizeof(double) * n, cudaMemcpyDeviceToHost, h->stream));
  PCPM_CK(cudaStreamSynchronize(h->stream));
  return n;
}

int pcpm_set_option(pcpm_handle* h, const char* key, int64_t value) {
  if (!h || !key) {
    set_error(PCPM_EINVAL, "NULL handle or key");
    return PCPM_EINVAL;
  }
  if (!strcmp(key, "phase_timing")) {
    h->opt_phase_timing = (int)value;
    free_graph(h);
    return PCPM_OK;
  }
  if (!strcmp(key, "use_graph")) {
    h->opt_use_graph = (int)value;
    free_graph(h);
    return PCPM_OK;
  }
  if (!strcmp(key, "scatter_variant")) {
    if (value < 0 || value > 3) {
      set_error(PCPM_EINVAL, "scatter_variant must be 0 (TMA stream), 1 (warp per group), 2 (TMA stream, "
                             "source values read through L1/L2) or 3 (TMA stream, 16-byte stores)");
      return PCPM_EINVAL;
    }
    h->opt_scatter_variant = (int)value;
    free_graph(h);
    return PCPM_OK;
  }
  if (!strcmp(key, "gather_variant")) {
    if (value < 1 || value > 3) {
      set_error(PCPM_EINVAL,
                "gather_variant must be 1 (in-line epilogue), 2 (apply warps from tensor memory) or 3 (apply in the "
                "producer warps from tensor memory)");
      return PCPM_EINVAL;
    }
    h->opt_gather_variant = (int)value;
    free_graph(h);
    return PCPM_OK;
  }
  if (!strcmp(key, "fuse_scatter")) {
    h->opt_fuse = value ? 1 : 0;
    free_graph(h);
    return PCPM_OK;
  }
  if (!strcmp(key, "cluster_gather")) {
    h->opt_cluster_gather = value ? 1 : 0;
    free_graph(h);
    return PCPM_OK;
  }
  if (!strcmp(key, "pdl")) {
    // pair handles (q = 2^16) launch plainly: with programmatic dependent launch their
    // iteration measured 30% slower (c3: 2.39 vs 1.83 ms)
    h->opt_pdl = (value && !h->pair) ? 1 : 0;
    free_graph(h);
    return PCPM_OK;
  }
  if (!strcmp(key, "gather_prefetch")) {
    if (value < 0 || value > 16) {
      set_error(PCPM_EINVAL, "gather_prefetch must be in [0, 16]");
      return PCPM_EINVAL;
    }
    h->opt_gather_pf = (int)value;
    free_graph(h);
    return PCPM_OK;
  }
  if (!strcmp(key, "scatter_lpt")) {
    h->opt_scatter_lpt = value ? 1 : 0;
    free_graph(h);
    return order_scatter_items(h, h->stream);
  }
  if (!strcmp(key, "scatter_prefetch")) {
    if (value < 0 || value > 64) {
      set_error(PCPM_EINVAL, "scatter_prefetch must be in [0, 64]");
      return PCPM_EINVAL;
    }
    h->opt_scatter_pf = (int)value;
    free_graph(h);
    return PCPM_OK;
  }
  if (!strcmp(key, "weighted_pagerank")) {
    if (value && (!h->inv_wdeg || !h->w || h->shard)) {
      set_error(PCPM_ESTATE, "weighted_pagerank needs a (non-shard) handle built with edge values");
      return PCPM_ESTATE;
    }
    if (value && h->neg_weights) {
      set_error(PCPM_EINVAL, "weighted_pagerank needs non-negative edge values (R24)");
      return PCPM_EINVAL;
    }
    h->opt_weighted_pr = value ? 1 : 0;
    free_graph(h);
    return PCPM_OK;
  }
    if (!strcmp(key, "epilogue_prefetch")) {
    if (value < 0 || value > 64) {
      set_error(PCPM_EINVAL, "epilogue_prefetch must be in [0, 64] (tiles before the item's end)");
      return PCPM_EINVAL;
    }
    h->opt_epi_pf = (int)value;
    free_graph(h);
    return PCPM_OK;
  }
  set_error(PCPM_EINVAL, std::string("unknown option ") + key);
  return PCPM_EINVAL;
}

int pcpm_get_debug_counters(uint64_t* out, int cap, int reset) {
  if (!out || cap < 0) {
    set_error(PCPM_EINVAL, "NULL output");
    return PCPM_EINVAL;
  }
  return read_debug_counters(reinterpret_cast<unsigned long long*>(out), cap, reset != 0);
}

int64_t pcpm_last_launch_count(const pcpm_handle* h) { return h ? h->launches : 0; }

int pcpm_get_phase_times(pcpm_handle* h, float* ms, int cap) {
  if (!h || !ms) {
    set_error(PCPM_EINVAL, "NULL handle or buffer");
    return PCPM_EINVAL;
  }
  if (!h->opt_phase_timing || h->n_events_used < 2) return 0;
  PCPM_CK(cudaStreamSynchronize(h->stream));
  const int n = std::min(cap, h->n_events_used - 1);
  for (int i = 0; i < n; ++i) PCPM_CK(cudaEventElapsedTime(&ms[i], h->events[i], h->events[i + 1]));
  return n;
}

}  // extern "C"

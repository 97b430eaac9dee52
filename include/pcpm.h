/*
 * pcpm.h -- C ABI of the B200-native Partition-Centric PageRank / SpMV hot path
 * (Lakhotia, Kannan, Prasanna, "Accelerating PageRank using Partition-Centric
 * Processing", arXiv:1709.07122).  "P:<n>" cites /root/reference/PAPER.md
 * line n; readings R1..R19 are listed in DESIGN.md.
 *
 * The library (libpcpm.so, built from paper_1709_07122_b200/csrc/) runs every
 * step on one sm_100a GPU: the one-time layout build (§3.1-3.3), the PNG
 * scatter (Alg. 4), the branch-avoiding gather (Alg. 5) and the apply step
 * (Eq. 1).  There is no CPU fallback: every entry point that needs the GPU
 * returns PCPM_ECUDA when no device is usable.
 *
 * Conventions
 *  - Pointers are plain host or device pointers; the library detects which
 *    with cudaPointerGetAttributes.  Host inputs are copied to the device
 *    inside the call; host outputs are copied back before the call returns.
 *  - All device work is ordered on the handle's stream (pcpm_set_stream;
 *    default: the legacy default stream).  With device outputs the calls are
 *    asynchronous with respect to the host, except pcpm_build which
 *    synchronises once to size E'.
 *  - Return value 0 = success, negative = PCPM_E* code; pcpm_last_error()
 *    gives a thread-local message for the last failure.
 *  - Limits: n_src, n_dst < 2^31 (the MSB of a 4-byte ID is the run flag,
 *    P:172-173); nnz < 2^32 (u32 bin positions); partition_bits in [1, 16]:
 *    up to 15 one destination partition's accumulator (2^b x 4 B) lives in one
 *    CTA's shared memory; 16 (the right end of the paper's partition-size
 *    sweep; not for pcpm_build_shard or PCPM_BVGAS) implies
 *    PCPM_WIDE_IDS -- a 16-bit local ID plus the run flag needs the 4-byte
 *    format -- and the gather streams every bin twice, once per 2^15-vertex
 *    half of its partition, while the scatter reads the source values through
 *    L1/L2 (a 256 KB slice does not fit in shared memory); results are the
 *    same bits as with 15.  k_src * k_dst <= 2^28 (the O(k^2) offset matrices
 *    of P:148 / P:246).
 */
#ifndef PCPM_H
#define PCPM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PCPM_OK 0
#define PCPM_EINVAL -1   /* NULL pointer, partition_bits out of range, d not in (0,1), iters < 0 ... */
#define PCPM_ETOOBIG -2  /* n >= 2^31, nnz >= 2^32, k_src*k_dst > 2^28 */
#define PCPM_EBADCSR -3  /* row_ptr not monotone / row_ptr[0] != 0 / row_ptr[n] != nnz, col >= n_dst,
                            or a row whose columns are not strictly increasing (R6) */
#define PCPM_ENOMEM -4   /* device allocation failed */
#define PCPM_ECUDA -5    /* any other CUDA error (text in pcpm_last_error) */
#define PCPM_ESTATE -6   /* operation not valid for this handle (e.g. PageRank on a non-square matrix) */

/* pcpm_build_ex flags */
#define PCPM_NO_COMPRESS 0x1u  /* uncompressed bins: every ID flagged, one update per edge (E' = m);
                                  the BVGAS-like traffic baseline of P:342-345, measured with our layout */
#define PCPM_BUILD_PULL 0x2u   /* also build the in-adjacency (CSC) for pcpm_pull_pagerank */
#define PCPM_KEEP_VALUES 0x4u  /* keep weight bins even if values == NULL (all ones) */
#define PCPM_COMPACT_SLOTS 0x10u /* accumulator slots: when every destination partition has <= ~20K
                                  vertices with in-edges (and no bin is split), the 2-byte IDs hold the
                                  vertex's rank among its partition's vertices with in-edges, so the
                                  gather's shared-memory accumulator shrinks and its TMA ring gets 6
                                  stages instead of 4.  Results are identical; ignored (layout as
                                  without the flag) for weighted / shard / wide handles or when the
                                  condition fails (pcpm_get_info().compact_slots says which). */
#define PCPM_BVGAS 0x20u       /* the BVGAS comparison engine (Alg. 3; implies PCPM_NO_COMPRESS):
                                  destination IDs written once at build (the paper's own BVGAS,
                                  P:313), and every iteration's scatter traverses the CSR vertex-
                                  centrically, inserting each edge's update (u's value) at its bin's
                                  insertion point -- one update per edge instead of one per (u, j) run.
                                  The handle keeps a copy of the CSR.  Square, unweighted, compact
                                  layout only (else PCPM_EINVAL). */
#define PCPM_WIDE_IDS 0x8u     /* iterate on the paper's 4-byte layout (global 31-bit IDs + MSB flag in
                                  destID bins, 4-byte PNG sources) instead of the default
                                  compact one (2-byte partition-local IDs: 15-bit offset + MSB flag,
                                  2-byte PNG sources; the "smallest number of bits" of P:589).  Both
                                  encode the same bins; the compact one moves half the index bytes. */

/* A CSR matrix M with n_src rows and n_dst columns: row u lists the columns
 * v with M[u][v] != 0, i.e. the out-neighbours of u (push form).
 * For PageRank n_src == n_dst == |V| and M is the 0/1 adjacency A; for SpMV
 * the library computes y = M^T x (Eq. 2 orientation; reading R17). */
typedef struct {
  int64_t n_src;            /* rows (source vertices) */
  int64_t n_dst;            /* columns (destination vertices) */
  int64_t nnz;              /* nonzeros / edges, after deduplication (R10) */
  const int64_t* row_ptr;   /* n_src+1 entries, row_ptr[0] = 0, monotone, row_ptr[n_src] = nnz */
  const uint32_t* col_idx;  /* nnz entries, < n_dst, strictly increasing within each row */
  const float* values;      /* nnz entries or NULL (= all ones); PageRank uses them only with the
                               "weighted_pagerank" option (R24) */
} pcpm_csr;

typedef struct pcpm_handle pcpm_handle;

/* Facts about a built layout (sizes are element counts). */
typedef struct {
  int64_t n_src, n_dst, nnz;
  int32_t partition_bits;   /* b, q = 2^b */
  int64_t q, k_src, k_dst;  /* partitions: P_i = [i q, (i+1) q) */
  int64_t e_prime;          /* |E'| = #distinct (u, floor(v/q)) pairs */
  double r;                 /* compression ratio m / E' (Table 2) */
  int64_t n_dangling;       /* vertices with out-degree 0 */
  int32_t weighted;         /* weight bins present */
  int32_t compressed;       /* 0 when built with PCPM_NO_COMPRESS */
  int64_t device_bytes;     /* device memory held by the handle */
  double build_ms;          /* device time of the build (event-timed) */
  int64_t gather_items, scatter_items;  /* work-list sizes of the two kernels */
  int32_t fixed_point_bits;   /* F of the last pcpm_pagerank / pcpm_spmv call */
  int32_t compact_slots;      /* 1: built with accumulator slots (PCPM_COMPACT_SLOTS applied) */
  int32_t fused_iterations;   /* 1: the last pcpm_pagerank ran the fused iteration (each gather kernel also
                                 scatters the next iteration's updates; phase times then read: init, the
                                 first scatter, one entry per iteration) */
  int32_t bvgas;              /* 1: the BVGAS comparison engine (PCPM_BVGAS) */
} pcpm_info;

/* Device pointers to the built layout, for bit-exact tests (read-only).
 * The compact arrays (ids16, png_src16) always exist; the 4-byte arrays
 * (ids, png_src) only for handles built with PCPM_WIDE_IDS (else NULL). */
typedef struct {
  const uint32_t* ids;           /* [nnz] destID bins concatenated in j order; v | flag<<31 */
  const float* w;                /* [nnz] weights aligned with ids, or NULL */
  const uint32_t* png_src;       /* [E'] PNG sources grouped (p, j), u ascending */
  const uint32_t* png_off;       /* [k_src*(k_dst+1)] start of group (p,j) in png_src; row p ends with
                                    png_off[p][k_dst] = end of partition p */
  const uint32_t* upd_off;       /* [k_src*k_dst] write offset of source partition p into the
                                    concatenated update bins, P:148 */
  const uint32_t* bin_id_start;  /* [k_dst+1] first ID of bin j */
  const uint32_t* bin_upd_start; /* [k_dst+1] first update of bin j */
  const uint32_t* chunk_base;    /* [nnz/128 + 2] #flags in ids[0 .. 128 c) (decode anchors) */
  const uint32_t* out_degree;    /* [n_src] |N_o(u)| */
  float* upd;                    /* [E'] update bins of the last scatter (scratch) */
  int64_t chunk_ids;             /* IDs per chunk_base entry (128) */
  const uint16_t* ids16;         /* [nnz] compact destID bins: (v & (q-1)) | flag<<15 (b = 16: 15 local bits) */
  const uint16_t* png_src16;     /* [E'] compact PNG sources: u & (q-1) (u is in partition p) */
  int32_t wide;                  /* 1 when the kernels iterate on the 4-byte arrays */
} pcpm_layout_view;

/* Build the PCPM layout on the GPU (§3.1-3.3): validation,
 * partitioning into k = ceil(n/q) partitions of q = 2^partition_bits
 * vertices, the k x k write offsets of P:148, the destID bins with MSB run
 * flags, the per-partition transposed PNG and the
 * decode anchors.  Integer work only; the result is bit-identical to the
 * oracle's layout.  csr arrays are borrowed for the duration of the call and
 * may be host or device memory.  Returns NULL on error (see pcpm_last_error;
 * pcpm_last_status gives the code). */
pcpm_handle* pcpm_build(const pcpm_csr* csr, int partition_bits);
pcpm_handle* pcpm_build_ex(const pcpm_csr* csr, int partition_bits, unsigned flags, void* cuda_stream);

/* PageRank, Eq. 1 with PR_0 = 1/n (R2), damping d in (0,1), and the
 * dangling-mass rule R1: PR_{t+1}(v) = (1-d)/n + d*(sum_{u->v} PR_t(u)/|N_o(u)|
 * + D_t/n).  Runs `iters` iterations of scatter (Alg. 4) -> gather (Alg. 5)
 * -> apply, captured in a CUDA graph.  out: n floats (host or device) receive
 * the unscaled PR_iters (R4).  iters = 0 returns 1/n.  PCPM_ESTATE if the
 * handle is not square. */
int pcpm_pagerank(pcpm_handle* h, double d, int iters, float* out);
/* PageRank iterated to convergence: the same iterations as pcpm_pagerank, run
 * until the L1 residual sum_v |PR_t(v) - PR_{t-1}(v)| (computed by the fused apply
 * of every iteration) is <= tol, or max_iters iterations.  out receives PR_t for
 * that t (host or device, n floats); *iters_done = t.  The host reads one residual
 * per iteration while the next iteration already runs (kernels launched directly,
 * no graph).  tol >= 0, max_iters >= 1; returns 0 or PCPM_E*. */
int pcpm_pagerank_tol(pcpm_handle* h, double d, double tol, int max_iters, float* out, int* iters_done);

/* y = M^T x (§3.5): y[v] = sum over CSR entries (u -> v) of
 * w(u,v) * x[u], with w = values given at build (1 if none).  x: n_src floats,
 * y: n_dst floats, host or device. */
int pcpm_spmv(pcpm_handle* h, const float* x, float* y);

/* Same PageRank computed by the naive pull-direction kernel (Alg. 1, P:86-99;
 * the in-house comparison of BASELINE.json).  Needs PCPM_BUILD_PULL. */
int pcpm_pull_pagerank(pcpm_handle* h, double d, int iters, float* out);

/* ---- Multi-GPU: destination shards.
 * Rank r owns the destination vertices [v_lo, v_hi) (v_lo a multiple of q = 2^b,
 * so its bins are whole partitions of the global graph).  Per iteration every
 * rank scatters all source partitions into ITS bins only, gathers and applies
 * its vertices, then the ranks all-gather the SPR slices (one n*4-byte exchange)
 * and all-reduce (residual, dangling mass); paper_1709_07122_b200/dist.py drives
 * the exchange with torch.distributed (NCCL).
 *
 * pcpm_build_shard: layout of the column slice [v_lo, v_hi) of csr (n_src rows,
 * local columns v - v_lo), keeping the GLOBAL out-degrees |N_o(u)| of all
 * sources (P:65's SPR divides by the full out-degree).  csr is borrowed, host or
 * device; only the slice's columns are validated.  flags: PCPM_WIDE_IDS,
 * PCPM_KEEP_VALUES.  NULL on error (PCPM_ESTATE if csr is not square).
 * pcpm_shard_init: PR_0 = 1/n_global on the slice (pr0, spr0: DEVICE f32[v_hi-v_lo])
 * and dang0 (DEVICE f64[1]) = the slice's share of D_0.
 * pcpm_shard_step: one iteration of Eq. 1 with rule R1 for the slice:
 *   spr_in  DEVICE f32[n_src]  SPR_t of ALL vertices (after the all-gather);
 *   D_in    DEVICE f64[1]      D_t, the global dangling mass (after the all-reduce);
 *   pr_old  DEVICE f32[n_loc]  the slice's PR_t;  pr_new / spr_out: its PR_{t+1}, SPR_{t+1}
 *           (spr_out may alias spr_in + v_lo: the scatter has read spr_in before the gather writes);
 *   red_out DEVICE f64[2]      [0] = sum |PR_{t+1} - PR_t| over the slice, [1] = its dangling mass.
 * Stream-ordered on the handle's stream; returns 0 or PCPM_E*. */
pcpm_handle* pcpm_build_shard(const pcpm_csr* csr, int partition_bits, int64_t v_lo, int64_t v_hi,
                              unsigned flags, void* cuda_stream);
int pcpm_shard_init(pcpm_handle* h, float* pr0, float* spr0, double* dang0);
int pcpm_shard_step(pcpm_handle* h, double d, const float* spr_in, const double* D_in, const float* pr_old,
                    float* pr_new, float* spr_out, double* red_out);

/* pcpm_shard_step_peers: pcpm_shard_step with the SPR exchange fused into the apply
 * (DESIGN.md §7).  The gather's epilogue stores every SPR_{t+1} vertex group it
 * produces to all of spr_outs[0 .. n_outs): spr_outs[0] is this rank's own chunk
 * (as pcpm_shard_step's spr_out), spr_outs[1..] the same chunk in the other ranks'
 * full-SPR buffers -- peer device memory opened with pcpm_ipc_open, written over
 * NVLink / NVSwitch as the tiles finish -- so no all-gather follows.  spr_outs is a
 * HOST array of n_outs (1 .. PCPM_MAX_PEERS + 1) DEVICE pointers, each 16-byte
 * aligned for the vector path (n_outs > 1 is PCPM_ESTATE for handles built with
 * PCPM_COMPACT_SLOTS).  The gather ends with a system-scope fence: once the
 * kernel completes its stores are visible to the peers; the caller orders each
 * peer's next iteration after a collective (dist.py: the all-reduce of red_out).
 * Returns 0 or PCPM_E*. */
#define PCPM_MAX_PEERS 8
/* pcpm_shard_init_peers: pcpm_shard_init writing SPR_0 of the slice to spr_outs[0]
 * and copying it to spr_outs[1..] (same layout as pcpm_shard_step_peers). */
int pcpm_shard_init_peers(pcpm_handle* h, float* pr0, float* const* spr_outs, int n_outs, double* dang0);
int pcpm_shard_step_peers(pcpm_handle* h, double d, const float* spr_in, const double* D_in, const float* pr_old,
                          float* pr_new, float* const* spr_outs, int n_outs, double* red_out);
/* CUDA IPC plumbing for the fused exchange (one process per GPU).
 * pcpm_ipc_alloc / _free: a plain cudaMalloc'ed, zeroed exchange buffer (IPC handles
 * need a whole allocation); pcpm_ipc_get_handle writes pcpm_ipc_handle_bytes() bytes
 * describing it; pcpm_ipc_open maps another process's buffer into this one (peer
 * access enabled lazily) and pcpm_ipc_close unmaps it.  0 or PCPM_E*. */
int pcpm_ipc_handle_bytes(void);
int pcpm_ipc_alloc(int64_t bytes, void** dev_ptr);
int pcpm_ipc_free(void* dev_ptr);
int pcpm_ipc_get_handle(void* dev_ptr, void* handle_out);
int pcpm_ipc_open(const void* handle, void** dev_ptr_out);
int pcpm_ipc_close(void* dev_ptr);

void pcpm_destroy(pcpm_handle* h);

/* ---- Job runtime: whole PageRank jobs from HOST memory, pipelined (csrc/jobs.cu).
 * A job is: H2D copy of a square CSR -> pcpm_build_ex(csr, partition_bits, flags) ->
 * pcpm_pagerank(d, iters) -> n floats of PR_iters written to `out` (host or device).
 * One worker thread runs the jobs in submission order on the runtime's compute stream;
 * job k+1's CSR is uploaded on a copy stream while job k builds and iterates, and job
 * k's result is copied out on a third stream, so consecutive jobs overlap their PCIe
 * transfers with GPU work (one layout resident at a time).  Host arrays should be pinned
 * (cudaHostAlloc / cudaHostRegister) for the copies to run asynchronously; they are
 * borrowed until pcpm_job_wait returns for the job.  With values and PCPM_KEEP_VALUES
 * the job runs weighted PageRank (R24).
 * pcpm_runtime_create: NULL on error.  pcpm_job_submit: returns at once (0 or
 * PCPM_EINVAL / PCPM_ECUDA), *job_id identifies the job.  pcpm_job_wait: blocks until
 * the job's result is in `out`; returns the job's status (build / iteration errors
 * included) and forgets the id.  pcpm_runtime_destroy: finishes the queued jobs and
 * releases the runtime (jobs not waited for are discarded). */
typedef struct pcpm_runtime pcpm_runtime;
pcpm_runtime* pcpm_runtime_create(void);
int pcpm_job_submit(pcpm_runtime* rt, const pcpm_csr* csr, int partition_bits, unsigned flags, double d, int iters,
                    float* out, int64_t* job_id);
int pcpm_job_wait(pcpm_runtime* rt, int64_t job_id);
void pcpm_runtime_destroy(pcpm_runtime* rt);

/* Support: stream, errors, introspection. */
/* Memory: handles take their device memory from the current device's stream-ordered
 * default pool (cudaMallocAsync), which keeps freed memory cached.  pcpm_pool_reserve
 * maps `bytes` into that pool once (allocate + free, synchronous), so later builds and
 * two layouts alive at once (pipelined jobs) carve from cached memory instead of
 * mapping new memory mid-run.  0, PCPM_EINVAL (bytes < 0), PCPM_ENOMEM, PCPM_ECUDA. */
int pcpm_pool_reserve(int64_t bytes);
/* pcpm_set_stream: later calls order their device work on cuda_stream (NULL = the
 * legacy default stream).  The handle's scratch is shared by all calls, so the call
 * first synchronises the previous stream: work queued there completes before any
 * work on the new one.  0, PCPM_EINVAL, PCPM_ECUDA. */
int pcpm_set_stream(pcpm_handle* h, void* cuda_stream);
int pcpm_last_error(char* buf, int cap);   /* copies the message, returns its length */
int pcpm_last_status(void);                /* code of the last failure on this thread */
int pcpm_get_info(const pcpm_handle* h, pcpm_info* out);
int pcpm_export_layout(pcpm_handle* h, pcpm_layout_view* out);
/* Per-iteration diagnostics of the last pcpm_pagerank: host[2*t] = D_t (dangling
 * mass of PR_t), host[2*t+1] = sum_v |PR_{t+1}(v) - PR_t(v)|.  Returns the
 * number of doubles written (synchronises the stream). */
int pcpm_get_residuals(pcpm_handle* h, double* host, int cap);
/* Run only the scatter (Alg. 4) of x (n_src floats, device) into the handle's
 * update bins (exported as pcpm_layout_view.upd); for bit-exact tests. */
int pcpm_scatter(pcpm_handle* h, const float* x);
/* Select a kernel variant for A/B experiments.
 * Keys: "phase_timing", "use_graph", "scatter_variant" (0|1|2|3: 3 = 16-byte vector stores of update quads), "gather_variant" (1: the
 * gather applies each finished partition itself, the default; 2: k_gather2, which parks
 * the partition's accumulator in tensor memory and lets 4 dedicated warps apply it
 * while 27 warps decode the next one -- measured slower), "scatter_lpt",
 * "scatter_prefetch", "gather_prefetch", "epilogue_prefetch", "cluster_gather", "pdl"
 * (1, default: the scatter and gather are launched as programmatic dependents, so a
 * kernel's prologue overlaps its predecessor's tail; 0: plain stream order) (kernel variants:
 * every one computes the same result) and "weighted_pagerank" (1: pcpm_pagerank
 * uses the edge values as weights, u passing PR(u) w(u,v) / W(u) to v with
 * W(u) = sum of u's weights (reading R24); needs a non-shard handle
 * built with non-negative values, else PCPM_ESTATE / PCPM_EINVAL).  Every variant
 * computes the same result.  Returns PCPM_EINVAL for unknown keys or
 * out-of-range values. */
int pcpm_set_option(pcpm_handle* h, const char* key, int64_t value);
/* Kernel launches issued by the last pcpm_pagerank / pcpm_spmv call (per call). */
int64_t pcpm_last_launch_count(const pcpm_handle* h);
/* Per-kernel device times (ms, CUDA events on the handle's stream, recorded
 * inside the captured graph) of the last pcpm_pagerank / pcpm_pull_pagerank
 * call when option "phase_timing" is 1: ms[0] = init, then for t = 0..iters-1
 * ms[1+2t] = scatter_t, ms[2+2t] = gather_t (pull: ms[1+t] = pull_t).
 * Returns the number of floats written (synchronises the stream). */
int pcpm_get_phase_times(pcpm_handle* h, float* ms, int cap);
/* Consumer-warp cycle counters of the gather accumulated since the last reset, for
 * builds with -DPCPM_GATHER_PROFILE=1 (all zero otherwise): out[0] waiting for
 * stages, out[1] decoding, out[2] at the epilogue's first barrier, out[3] in the
 * epilogue, out[4] number of warps that reported.  Synchronous; returns the count. */
int pcpm_get_debug_counters(uint64_t* out, int cap, int reset);

#ifdef __cplusplus
}
#endif
#endif /* PCPM_H */

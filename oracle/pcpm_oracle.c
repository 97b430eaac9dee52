/*
 * pcpm_oracle.c -- the CPU oracle for the PCPM PageRank / SpMV hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this
 * library.  The product path (paper_1709_07122_b200/, libpcpm.so) never links,
 * imports or executes anything under oracle/, and this file shares no code,
 * header, table or helper with it.
 *
 * Plain, slow, obviously-correct C in fp64.  Every function follows the
 * passage of /root/reference/PAPER.md ("P:<line>") that defines it, written
 * out in the paper's order and notation with no blocking, fusion or
 * reordering.  Where the paper is silent the reading is named by its
 * DESIGN.md id (R1..Rn); SURVEY.md §8(c) proposed them.
 *
 * Parity pins (tests/test_oracle_pins.py, run with -m "not gpu"):
 *   oracle_pagerank   pinned: directed cycle, complete digraph, edgeless graph,
 *                     n=1 self-loop, 2-cycle, out-star / in-star closed forms
 *                     at every t, dense brute-force power iteration (n<=64),
 *                     stationary vector by linear solve, sum(PR)=1.
 *   oracle_pagerank_weighted  pinned: uniform weights = oracle_pagerank, per-source
 *                     scaling invariance, zero weights = removed edges, dense
 *                     brute-force power iteration of the weighted chain (n<=48).
 *   oracle_spmv_t     pinned: identity, zero, 2x2 hand product, dense numpy
 *                     product on random matrices, Eq. 2 consistency.
 *   oracle_layout     pinned: G_toy hand derivation (tests/golden)
 *                     offsets fragment, a second unrelated algorithm (sort by
 *                     (v>>b, u, v)), brute-force (u, v>>b) pair set, PNG
 *                     monotonicity under q doubling, structural invariants.
 *   oracle_scatter    pinned: hand example on G_toy, gather-mass identity.
 *   oracle_gather     pinned: Alg. 2 branching gather written separately in
 *                     the test (differential), hand examples.
 * No function is "parity unpinned".
 *
 * Index conventions (shared with the product only through the documented
 * C-ABI semantics in include/pcpm.h, never through code):
 *   CSR: row_ptr int64[n_src+1], col uint32[m]; row u lists the out-neighbours
 *   v of u (push form), strictly increasing within a row.
 *   q = 2^b, partition of vertex v is v >> b (reading R9).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_MSB 0x80000000u

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Thread count of the OpenMP loops (bench.py's single-core baseline). */
void oracle_set_threads(int t) {
#ifdef _OPENMP
  omp_set_num_threads(t > 0 ? t : 1);
#else
  (void)t;
#endif
}

/* Neumaier compensated sum of x[0..n) (D_t and checks use a
 * compensated fp64 sum so that sum(PR)=1 holds to ~1e-16 n). */
static double oracle_sum(const double* x, int64_t n) {
  double s = 0.0, c = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double t = s + x[i];
    if (fabs(s) >= fabs(x[i])) c += (s - t) + x[i];
    else c += (x[i] - t) + s;
    s = t;
  }
  return s + c;
}

/* ---------------------------------------------------------------------------
 * In-adjacency (CSC) of a CSR graph: N_i(v) of Table 1, listed in
 * ascending source order.  Used by the pull-form PageRank below (Alg. 1,
 * P:86-99).  in_ptr int64[n+1], in_src uint32[m] are caller-allocated.
 * ------------------------------------------------------------------------- */
int oracle_transpose(int64_t n, const int64_t* row_ptr, const uint32_t* col,
                     int64_t* in_ptr, uint32_t* in_src) {
  int64_t m = row_ptr[n];
  for (int64_t v = 0; v <= n; ++v) in_ptr[v] = 0;
  for (int64_t e = 0; e < m; ++e) {
    if (col[e] >= (uint64_t)n) return -1;
    in_ptr[col[e] + 1] += 1;
  }
  for (int64_t v = 0; v < n; ++v) in_ptr[v + 1] += in_ptr[v];
  int64_t* cursor = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  if (!cursor) return -2;
  for (int64_t v = 0; v < n; ++v) cursor[v] = in_ptr[v];
  for (int64_t u = 0; u < n; ++u)          /* u ascending => in-lists ascending */
    for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e)
      in_src[cursor[col[e]]++] = (uint32_t)u;
  free(cursor);
  return 0;
}

/* ---------------------------------------------------------------------------
 * PageRank by its plain definition, Eq. 1, computed in the pull
 * direction of Alg. 1 in fp64, with:
 *   R1 (dangling): the mass D_t of zero-out-degree vertices is redistributed
 *      uniformly: PR_{t+1}(v) = (1-d)/n + d*( sum_{u in N_i(v)} PR_t(u)/|N_o(u)|
 *      + D_t/n ).  (BASELINE.json config 1 "dangling vertices' mass
 *      redistributed uniformly"; the paper is silent.)
 *   R2 (initial vector): PR_0(v) = 1/n.
 *   R11 (iteration count): iters updates are applied to PR_0.
 * The result is the unscaled PR_iters (reading R4).
 * Arguments: in-adjacency from oracle_transpose, out-degree from the CSR.
 * Output pr int64[n] doubles.  Returns 0, or <0 on bad input.
 * ------------------------------------------------------------------------- */
/* One Eq. 1 update in pull form, PR_t -> PR_{t+1} in place (pr), with caller-owned
 * scratch work[3n] (no allocation: the bench's reference arm times exactly one
 * iteration per step with the buffers allocated outside the timed region). */
int oracle_pagerank_pull_step(int64_t n, const int64_t* row_ptr, const int64_t* in_ptr,
                              const uint32_t* in_src, double d, double* pr, double* work) {
  if (n <= 0 || !(d > 0.0 && d < 1.0) || !work) return -1;
  double* spr = work;
  double* dang = work + n;
  double* next = work + 2 * n;
  /* SPR(u) = PR(u)/|N_o(u)| (Table 1); dangling mass D_t (R1). */
  for (int64_t u = 0; u < n; ++u) {
    int64_t deg = row_ptr[u + 1] - row_ptr[u];
    spr[u] = deg > 0 ? pr[u] / (double)deg : 0.0;
    dang[u] = deg > 0 ? 0.0 : pr[u];
  }
  double D = oracle_sum(dang, n);
  /* Eq. 1: new value = (1-d)/|V| + d * sum over in-neighbours (+ R1 term). */
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t v = 0; v < n; ++v) {
    double temp = 0.0;
    for (int64_t e = in_ptr[v]; e < in_ptr[v + 1]; ++e) temp += spr[in_src[e]];
    next[v] = (1.0 - d) / (double)n + d * (temp + D / (double)n);
  }
  memcpy(pr, next, sizeof(double) * (size_t)n);
  return 0;
}

int oracle_pagerank_pull(int64_t n, const int64_t* row_ptr, const int64_t* in_ptr,
                         const uint32_t* in_src, double d, int iters, double* pr) {
  if (n <= 0 || iters < 0 || !(d > 0.0 && d < 1.0)) return -1;
  double* work = (double*)malloc(sizeof(double) * 3 * (size_t)n);
  if (!work) return -2;
  for (int64_t v = 0; v < n; ++v) pr[v] = 1.0 / (double)n;           /* R2 */
  int rc = 0;
  for (int it = 0; it < iters && rc == 0; ++it)
    rc = oracle_pagerank_pull_step(n, row_ptr, in_ptr, in_src, d, pr, work);
  free(work);
  return rc;
}

/* ---------------------------------------------------------------------------
 * Weighted PageRank (§3.5: edge weights stored with the destination IDs
 * "applied to the source node value before updating the destination node"; the
 * normalisation is reading R24): u passes PR(u) * w(u,v) / W(u) to v, with
 * W(u) = sum_v w(u,v) and w >= 0.  Vertices with W(u) = 0 (out-degree 0, or only
 * zero weights) are dangling and their mass is spread uniformly (R1):
 *   PR_{t+1}(v) = (1-d)/n + d * ( sum_{u->v} PR_t(u) w(u,v) / W(u) + D_t/n ).
 * With every w = 1 this is oracle_pagerank.  Push form, plain loops, fp64.
 * Returns 0, -1 on bad arguments, -3 on a negative weight.
 * ------------------------------------------------------------------------- */
int oracle_pagerank_weighted(int64_t n, const int64_t* row_ptr, const uint32_t* col, const float* w,
                             double d, int iters, double* pr) {
  if (n <= 0 || iters < 0 || !(d > 0.0 && d < 1.0)) return -1;
  int64_t m = row_ptr[n];
  for (int64_t e = 0; e < m; ++e) if (w[e] < 0.0f) return -3;
  double* W = (double*)malloc(sizeof(double) * (size_t)n);
  double* dang = (double*)malloc(sizeof(double) * (size_t)n);
  double* next = (double*)malloc(sizeof(double) * (size_t)n);
  if (!W || !dang || !next) { free(W); free(dang); free(next); return -2; }
  for (int64_t u = 0; u < n; ++u) {
    double s = 0.0;
    for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) s += (double)w[e];
    W[u] = s;
  }
  for (int64_t v = 0; v < n; ++v) pr[v] = 1.0 / (double)n;           /* R2 */
  for (int it = 0; it < iters; ++it) {
    for (int64_t u = 0; u < n; ++u) dang[u] = W[u] > 0.0 ? 0.0 : pr[u];
    double D = oracle_sum(dang, n);                                   /* R1 */
    for (int64_t v = 0; v < n; ++v) next[v] = 0.0;
    for (int64_t u = 0; u < n; ++u) {
      if (!(W[u] > 0.0)) continue;
      for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e)
        next[col[e]] += pr[u] * (double)w[e] / W[u];
    }
    for (int64_t v = 0; v < n; ++v) next[v] = (1.0 - d) / (double)n + d * (next[v] + D / (double)n);
    memcpy(pr, next, sizeof(double) * (size_t)n);
  }
  free(W); free(dang); free(next);
  return 0;
}

/* Convenience: transpose + pull PageRank in one call (tests). */
int oracle_pagerank(int64_t n, const int64_t* row_ptr, const uint32_t* col,
                    double d, int iters, double* pr) {
  int64_t m = row_ptr[n];
  int64_t* in_ptr = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  uint32_t* in_src = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(m > 0 ? m : 1));
  if (!in_ptr || !in_src) { free(in_ptr); free(in_src); return -2; }
  int rc = oracle_transpose(n, row_ptr, col, in_ptr, in_src);
  if (rc == 0) rc = oracle_pagerank_pull(n, row_ptr, in_ptr, in_src, d, iters, pr);
  free(in_ptr); free(in_src);
  return rc;
}

/* ---------------------------------------------------------------------------
 * SpMV of §3.5 in the orientation of Eq. 2:
 *   y[v] = sum over CSR entries (u -> v) of  val(u,v) * x[u]
 * i.e. y = M^T x for the CSR matrix M passed in (reading R17).  val == NULL
 * means the 0/1 adjacency A.  fp32 inputs are promoted to fp64; each y[v]
 * accumulates its terms in ascending u.
 * ------------------------------------------------------------------------- */
int oracle_spmv_t(int64_t n_src, int64_t n_dst, const int64_t* row_ptr, const uint32_t* col,
                  const float* val, const float* x, double* y) {
  for (int64_t v = 0; v < n_dst; ++v) y[v] = 0.0;
  for (int64_t u = 0; u < n_src; ++u)
    for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) {
      if (col[e] >= (uint64_t)n_dst) return -1;
      double a = val ? (double)val[e] : 1.0;
      y[col[e]] += a * (double)x[u];
    }
  return 0;
}

/* ---------------------------------------------------------------------------
 * Layout sizes: k_src = ceil(n_src/q), k_dst = ceil(n_dst/q) (R9) and
 * E' = number of distinct (u, floor(v/q)) pairs (Eff_1).
 * ------------------------------------------------------------------------- */
int oracle_layout_sizes(int64_t n_src, int64_t n_dst, const int64_t* row_ptr,
                        const uint32_t* col, int b, int64_t* k_src, int64_t* k_dst,
                        int64_t* e_prime) {
  int64_t q = (int64_t)1 << b;
  *k_src = (n_src + q - 1) / q;
  *k_dst = (n_dst + q - 1) / q;
  int64_t ep = 0;
  for (int64_t u = 0; u < n_src; ++u) {
    int64_t prev_bin = -1;                          /* Alg. 2 "prev_bin <- inf" */
    for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) {
      int64_t bin = (int64_t)(col[e] >> b);
      if (bin != prev_bin) { ++ep; prev_bin = bin; }
    }
  }
  *e_prime = ep;
  return 0;
}

/* ---------------------------------------------------------------------------
 * The PCPM layout by plain definition.
 *
 * destID bins (Alg. 2): walk u ascending,
 * and the out-neighbours v of u ascending (R6/R7); j = v >> b; the ID is
 * flagged (MSB set) when it is the first ID of u's run in partition j
 * ("prev_bin" test of Alg. 2).  The ID (global v, reading R8) is appended to
 * bin j.  On a flag, u is appended to the PNG group (p = u>>b, j) (Eff_1/Eff_2
 * and the per-partition transposition of P:227-246) and one update slot is
 * reserved in update bin j.
 *
 * Offsets: partitions write to bins in the order of their IDs, so the
 * offset of partition p into bin j is the sum of what partitions p' < p write
 * into bin j.  Bins are concatenated in j order into one array each:
 *   bin_id_start[j]  = sum_{j'<j} (IDs in bin j')            (k_dst+1 entries)
 *   bin_upd_start[j] = sum_{j'<j} (updates in bin j')        (k_dst+1 entries)
 *   upd_off[p][j]    = bin_upd_start[j] + sum_{p'<p} cnt_upd[p'][j]
 *   png_off[p][j]    = global start of PNG group (p, j) in png_src; groups are
 *                      stored in (p, j) order, png_off[p][k_dst] = end of p.
 * w (optional): the CSR value of the edge behind each ID, aligned with ids
 * (§3.5 P:288 "storing the edge weights along with destination IDs").
 * All outputs are caller-allocated: ids[m], png_src[E'], png_off[k_src*(k_dst+1)],
 * upd_off[k_src*k_dst], bin_id_start[k_dst+1], bin_upd_start[k_dst+1], w[m].
 * ------------------------------------------------------------------------- */
int oracle_layout(int64_t n_src, int64_t n_dst, const int64_t* row_ptr, const uint32_t* col,
                  const float* val, int b,
                  uint32_t* ids, uint32_t* png_src, uint64_t* png_off, uint64_t* upd_off,
                  uint64_t* bin_id_start, uint64_t* bin_upd_start, float* w) {
  int64_t k_src, k_dst, ep;
  oracle_layout_sizes(n_src, n_dst, row_ptr, col, b, &k_src, &k_dst, &ep);
  int64_t K = k_src * k_dst;
  uint64_t* cnt_upd = (uint64_t*)calloc((size_t)(K > 0 ? K : 1), sizeof(uint64_t));
  uint64_t* cnt_ids = (uint64_t*)calloc((size_t)(K > 0 ? K : 1), sizeof(uint64_t));
  if (!cnt_upd || !cnt_ids) { free(cnt_upd); free(cnt_ids); return -2; }

  /* Scan 1: per (p, j) count runs (updates) and IDs. */
  for (int64_t u = 0; u < n_src; ++u) {
    int64_t p = u >> b, prev_bin = -1;
    for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) {
      if (col[e] >= (uint64_t)n_dst) { free(cnt_upd); free(cnt_ids); return -1; }
      int64_t j = (int64_t)(col[e] >> b);
      if (j != prev_bin) { cnt_upd[p * k_dst + j] += 1; prev_bin = j; }
      cnt_ids[p * k_dst + j] += 1;
    }
  }
  /* Bin starts: exclusive scans over j of the column sums. */
  bin_id_start[0] = 0; bin_upd_start[0] = 0;
  for (int64_t j = 0; j < k_dst; ++j) {
    uint64_t si = 0, su = 0;
    for (int64_t p = 0; p < k_src; ++p) { si += cnt_ids[p * k_dst + j]; su += cnt_upd[p * k_dst + j]; }
    bin_id_start[j + 1] = bin_id_start[j] + si;
    bin_upd_start[j + 1] = bin_upd_start[j] + su;
  }
  /* Write offsets of P:148 for updates and IDs; PNG group starts. */
  uint64_t* id_cur = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(K > 0 ? K : 1));
  uint64_t* png_cur = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(K > 0 ? K : 1));
  if (!id_cur || !png_cur) { free(cnt_upd); free(cnt_ids); free(id_cur); free(png_cur); return -2; }
  for (int64_t j = 0; j < k_dst; ++j) {
    uint64_t ou = bin_upd_start[j], oi = bin_id_start[j];
    for (int64_t p = 0; p < k_src; ++p) {
      upd_off[p * k_dst + j] = ou;
      id_cur[p * k_dst + j] = oi;
      ou += cnt_upd[p * k_dst + j];
      oi += cnt_ids[p * k_dst + j];
    }
  }
  uint64_t g = 0;
  for (int64_t p = 0; p < k_src; ++p) {
    for (int64_t j = 0; j < k_dst; ++j) {
      png_off[p * (k_dst + 1) + j] = g;
      png_cur[p * k_dst + j] = g;
      g += cnt_upd[p * k_dst + j];
    }
    png_off[p * (k_dst + 1) + k_dst] = g;
  }
  /* Scan 2: fill IDs (MSB on the first of each run) and PNG sources. */
  for (int64_t u = 0; u < n_src; ++u) {
    int64_t p = u >> b, prev_bin = -1;
    for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) {
      uint32_t v = col[e];
      int64_t j = (int64_t)(v >> b);
      uint32_t flag = 0;
      if (j != prev_bin) {
        flag = ORACLE_MSB;
        png_src[png_cur[p * k_dst + j]++] = (uint32_t)u;
        prev_bin = j;
      }
      uint64_t x = id_cur[p * k_dst + j]++;
      ids[x] = v | flag;
      if (w) w[x] = val ? val[e] : 1.0f;
    }
  }
  free(cnt_upd); free(cnt_ids); free(id_cur); free(png_cur);
  return 0;
}

/* ---------------------------------------------------------------------------
 * Scatter, Alg. 4: for p, for p', for u in N_i^p(p'):
 *   insert x[u] into update_bins[p'] -- i.e.
 *   upd[upd_off[p][j] + t] = x[png_src[png_off[p][j] + t]].
 * A pure copy of fp32 values (bit-exact reference for the GPU scatter).
 * ------------------------------------------------------------------------- */
int oracle_scatter(int64_t k_src, int64_t k_dst, const uint32_t* png_src, const uint64_t* png_off,
                   const uint64_t* upd_off, const float* x, float* upd) {
  for (int64_t p = 0; p < k_src; ++p)
    for (int64_t j = 0; j < k_dst; ++j) {
      uint64_t s = png_off[p * (k_dst + 1) + j], e = png_off[p * (k_dst + 1) + j + 1];
      for (uint64_t t = 0; t < e - s; ++t) upd[upd_off[p * k_dst + j] + t] = x[png_src[s + t]];
    }
  return 0;
}

/* ---------------------------------------------------------------------------
 * Branch-avoiding gather, Alg. 5, fp64 accumulation:
 *   for each bin j: update_ptr <- -1 (reading R5: Alg. 5 increments before
 *   the read and every bin starts with a flagged ID);
 *   id <- bin[ptr++]; update_ptr += MSB(id); id &= mask; acc[id] += upd[update_ptr]
 *   (times w[x] for the weighted form of §3.5).
 * acc is double[n_dst], zeroed here ("PR[:] = 0", Alg. 5 line 1).
 * ------------------------------------------------------------------------- */
int oracle_gather(int64_t k_dst, int64_t n_dst, const uint32_t* ids, const float* upd,
                  const float* w, const uint64_t* bin_id_start, const uint64_t* bin_upd_start,
                  double* acc) {
  for (int64_t v = 0; v < n_dst; ++v) acc[v] = 0.0;
  for (int64_t j = 0; j < k_dst; ++j) {
    int64_t update_ptr = (int64_t)bin_upd_start[j] - 1;
    for (uint64_t x = bin_id_start[j]; x < bin_id_start[j + 1]; ++x) {
      uint32_t id = ids[x];
      update_ptr += (int64_t)(id >> 31);
      id &= 0x7FFFFFFFu;
      if (id >= (uint64_t)n_dst) return -1;
      double term = (double)upd[update_ptr];
      if (w) term *= (double)w[x];
      acc[id] += term;
    }
  }
  return 0;
}

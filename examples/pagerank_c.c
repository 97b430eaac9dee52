/*
 * pagerank_c.c -- the C ABI used from plain C (no CUDA headers, no Python): a
 * seeded random digraph in host memory, PCPM layout build, PageRank (Eq. 1 with
 * the dangling rule R1) and one SpMV through include/pcpm.h with HOST pointers
 * (the library copies in and out).
 *
 *   gcc -O2 -I include examples/pagerank_c.c -L paper_1709_07122_b200 -lpcpm \
 *       -Wl,-rpath,$PWD/paper_1709_07122_b200 -o pagerank_c && ./pagerank_c
 *
 * Prints n, m, E', the sum of PR (1 up to fp32 rounding) and PR of a few vertices;
 * exits non-zero on any library error.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "pcpm.h"

static uint64_t splitmix64(uint64_t* s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : (x > y);
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 100000;   /* vertices */
  const int deg = 8;                                        /* out-edges drawn per vertex */
  int64_t* row_ptr = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  uint32_t* col = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(n * deg));
  float* pr = (float*)malloc(sizeof(float) * (size_t)n);
  float* x = (float*)malloc(sizeof(float) * (size_t)n);
  float* y = (float*)malloc(sizeof(float) * (size_t)n);
  if (!row_ptr || !col || !pr || !x || !y) return 2;
  uint64_t seed = 42;
  int64_t m = 0;
  row_ptr[0] = 0;
  for (int64_t u = 0; u < n; ++u) {
    const int d = (int)(splitmix64(&seed) % (deg + 1));     /* 0..deg: some vertices dangle */
    uint32_t* row = col + m;
    for (int i = 0; i < d; ++i) row[i] = (uint32_t)(splitmix64(&seed) % (uint64_t)n);
    qsort(row, (size_t)d, sizeof(uint32_t), cmp_u32);      /* rows sorted, deduplicated (R6) */
    int k = 0;
    for (int i = 0; i < d; ++i)
      if (k == 0 || row[i] != row[k - 1]) row[k++] = row[i];
    m += k;
    row_ptr[u + 1] = m;
  }
  pcpm_csr csr = {n, n, m, row_ptr, col, NULL};
  pcpm_handle* h = pcpm_build(&csr, 15);
  if (!h) {
    char msg[256];
    pcpm_last_error(msg, (int)sizeof msg);
    fprintf(stderr, "pcpm_build failed: %s\n", msg);
    return 1;
  }
  pcpm_info info;
  if (pcpm_get_info(h, &info) || pcpm_pagerank(h, 0.85, 20, pr)) {
    char msg[256];
    pcpm_last_error(msg, (int)sizeof msg);
    fprintf(stderr, "pcpm_pagerank failed: %s\n", msg);
    return 1;
  }
  double sum = 0.0;
  for (int64_t v = 0; v < n; ++v) sum += pr[v];
  for (int64_t v = 0; v < n; ++v) x[v] = 1.0f;
  if (pcpm_spmv(h, x, y)) return 1;                          /* y = A^T 1 = in-degrees */
  int64_t indeg_sum = 0;
  for (int64_t v = 0; v < n; ++v) indeg_sum += (int64_t)(y[v] + 0.5f);
  printf("n=%lld m=%lld e_prime=%lld r=%.3f sum_pr=%.7f pr0=%.6e pr1=%.6e spmv_sum=%lld\n", (long long)n,
         (long long)m, (long long)info.e_prime, info.r, sum, pr[0], pr[1], (long long)indeg_sum);
  pcpm_destroy(h);
  free(row_ptr); free(col); free(pr); free(x); free(y);
  return (indeg_sum == m && sum > 0.999 && sum < 1.001) ? 0 : 3;
}

/*
 * bfs_order.c -- locality labelling for the C4-BFS input (BASELINE.json
 * configs[3] "locality labelling (BFS order from highest-out-degree vertex)";
 * DESIGN.md reading R16).  Input generation only: no PCPM arithmetic.
 *
 *   start  = the vertex of highest out-degree (ties -> smaller ID);
 *   BFS over out-edges, each row's neighbours visited in ascending ID order
 *   (CSR rows are sorted), new ID = visit rank (order of first discovery);
 *   when the queue empties, restart from the unvisited vertex of highest
 *   out-degree (ties -> smaller ID).
 *
 * new_id[v] receives the label of old vertex v.  Single-threaded, O(n + m).
 */
#include <stdint.h>
#include <stdlib.h>

int inputs_bfs_order(int64_t n, const int64_t* row_ptr, const uint32_t* col, int64_t* new_id) {
  /* restart order: out-degree descending, ID ascending (stable counting sort) */
  int64_t maxdeg = 0;
  for (int64_t u = 0; u < n; ++u) {
    int64_t dg = row_ptr[u + 1] - row_ptr[u];
    if (dg > maxdeg) maxdeg = dg;
  }
  int64_t* bucket = (int64_t*)calloc((size_t)maxdeg + 2, sizeof(int64_t));
  int64_t* order = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
  int64_t* queue = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
  if (!bucket || !order || !queue) {
    free(bucket); free(order); free(queue);
    return -1;
  }
  /* bucket index = maxdeg - deg, so the scan order is degree descending */
  for (int64_t u = 0; u < n; ++u) bucket[maxdeg - (row_ptr[u + 1] - row_ptr[u]) + 1]++;
  for (int64_t i = 1; i <= maxdeg + 1; ++i) bucket[i] += bucket[i - 1];
  for (int64_t u = 0; u < n; ++u) order[bucket[maxdeg - (row_ptr[u + 1] - row_ptr[u])]++] = u;

  for (int64_t u = 0; u < n; ++u) new_id[u] = -1;
  int64_t next = 0;
  for (int64_t s = 0; s < n; ++s) {
    int64_t src = order[s];
    if (new_id[src] >= 0) continue;
    int64_t head = 0, tail = 0;
    new_id[src] = next++;
    queue[tail++] = src;
    while (head < tail) {
      int64_t u = queue[head++];
      for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) {
        int64_t v = col[e];
        if (new_id[v] < 0) {
          new_id[v] = next++;
          queue[tail++] = v;
        }
      }
    }
  }
  free(bucket); free(order); free(queue);
  return 0;
}

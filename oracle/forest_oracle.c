/*
 * C restatement of the ForestColl allgather data plane — TEST INFRASTRUCTURE
 * ONLY (the multi-threaded CPU baseline of bench.py and a cross-check of the
 * numpy oracle).  The product never links or calls it.
 *
 * Semantics (identical to oracle/forest_oracle.py): tree
 * (root r, batch j) carries shard elements [floor(S*lo/k), floor(S*hi/k)) of
 * root r ("a 1/k shard of data is broadcast along each out-tree",
 * PAPER.md:478; batches: pkg/src/collsched/schedule.py:55-65); the root copies
 * its own slice in, and every tree edge u->v copies the slice from u's output
 * into v's output at offset r*S, in BFS order from the root (delivery order,
 * verify.py:266-283).  Trees touch disjoint output ranges, so they run in
 * parallel.
 */
#include <stddef.h>
#include <string.h>

void fo_allgather(int n, int ntrees, int k, const int* root, const int* mlo, const int* mhi,
                  const int* order, const int* parent, const char* const* sends,
                  char* const* recvs, long long S, int esize, int threads) {
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
  for (int t = 0; t < ntrees; ++t) {
    const int r = root[t];
    const long long a = S * mlo[t] / k, b = S * mhi[t] / k;
    const size_t off = (size_t)(r * S + a) * esize, len = (size_t)(b - a) * esize;
    if (len == 0) continue;
    memcpy(recvs[r] + off, sends[r] + (size_t)a * esize, len);
    for (int i = 0; i < n; ++i) {
      const int v = order[t * n + i];
      const int p = parent[t * n + v];
      if (p >= 0) memcpy(recvs[v] + off, recvs[p] + off, len);
    }
  }
}

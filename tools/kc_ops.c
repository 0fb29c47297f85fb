/* Measurement harness (not product, not oracle): the algorithmic integer
 * work OPS(k) of SURVEY.md §8(d) for the k >= 5 issue roofline.
 *
 *   OPS(k) = 2 * sum_{e : s_e >= k-2} ceil(s_e / 32) * X_e
 *
 * s_e = |N+(v) ∩ N+(u)| for the directed edge e = (v, u); X_e = 1 + the
 * number of iterations of the candidate loop (clique_rec.hpp:49-60) that
 * the reference's EDGE engine (counting.cpp:158-187) executes under e, each
 * iteration being one intersection cands ∩ N+(x), with the reference's own
 * pruning (clique_rec.hpp:30,53).  The recursion is the one restated in
 * oracle/kc_oracle.c (kco_rec), instrumented; its clique total is returned
 * as the cross-check against count_total.  OpenMP over source vertices.
 */
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  const uint64_t* off;
  const uint32_t* adj;
  uint64_t* stamp;
  uint32_t** bufs;
  uint64_t iters;
} ctx_t;

static uint64_t rec(ctx_t* c, const uint32_t* cands, uint64_t ncand, int remaining, int depth,
                    uint64_t token_base) {
  if (ncand < (uint64_t)remaining) return 0;
  if (remaining == 1) return ncand;
  const uint64_t token = token_base + (uint64_t)depth;
  uint64_t total = 0;
  uint32_t* next = c->bufs[depth + 1];
  for (uint64_t i = 0; i < ncand; i++) {
    uint32_t u = cands[i];
    c->iters++;
    uint64_t nn = 0;
    for (uint64_t p = c->off[u]; p < c->off[u + 1]; p++)
      if (c->stamp[c->adj[p]] == token) next[nn++] = c->adj[p];
    if (nn + 1 < (uint64_t)remaining) continue;
    for (uint64_t j = 0; j < nn; j++) c->stamp[next[j]] = token + 1;
    total += rec(c, next, nn, remaining - 1, depth + 1, token_base);
    for (uint64_t j = 0; j < nn; j++) c->stamp[next[j]] = token;
  }
  return total;
}

/* returns 0; *ops and *total out; k >= 3 */
int kc_ops(uint32_t n, const uint64_t* off, const uint32_t* adj, int k, uint64_t* ops_out,
           uint64_t* total_out) {
  uint64_t maxd = 0;
  for (uint32_t v = 0; v < n; v++)
    if (off[v + 1] - off[v] > maxd) maxd = off[v + 1] - off[v];
  uint64_t ops = 0, total = 0;
#pragma omp parallel reduction(+ : ops, total)
  {
    ctx_t c;
    c.off = off;
    c.adj = adj;
    c.stamp = calloc((size_t)n + 1, 8);
    c.bufs = malloc(((size_t)k + 3) * sizeof(uint32_t*));
    for (int i = 0; i < k + 3; i++) c.bufs[i] = malloc((maxd + 1) * 4);
    uint64_t next_token = 1;
#pragma omp for schedule(dynamic, 256)
    for (uint32_t v = 0; v < n; v++) {
      for (uint64_t e = off[v]; e < off[v + 1]; e++) {
        const uint32_t u = adj[e];
        uint32_t* both = c.bufs[2];
        uint64_t nb = 0, a = off[v], b = off[u];
        while (a < off[v + 1] && b < off[u + 1]) {
          if (adj[a] < adj[b]) a++;
          else if (adj[b] < adj[a]) b++;
          else { both[nb++] = adj[a]; a++; b++; }
        }
        if (nb + 2 < (uint64_t)k) continue;
        const uint64_t tb = next_token;
        next_token += (uint64_t)k + 2;
        for (uint64_t i = 0; i < nb; i++) c.stamp[both[i]] = tb + 2;
        c.iters = 0;
        total += rec(&c, both, nb, k - 2, 2, tb);
        ops += 2 * ((nb + 31) / 32) * (1 + c.iters);
      }
    }
    for (int i = 0; i < k + 3; i++) free(c.bufs[i]);
    free(c.bufs);
    free(c.stamp);
  }
  *ops_out = ops;
  *total_out = total;
  return 0;
}

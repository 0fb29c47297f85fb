/* TEST INFRASTRUCTURE ONLY — the CPU restatement ("port") oracle.
 *
 * Plain-C restatement of the reference's arb-count path, used by tests/ as
 * the checker and by bench.py's cpu_baseline leg when the compiled
 * reference (oracle/_ref/libkclique_ref.so) is absent.  Nothing in the
 * product links, loads or calls this file.
 *
 * Pinned by tests/test_oracle_pin.py against (1) the compiled reference
 * itself on hundreds of seeded graphs, and (2) the reference's own known
 * answers (proj/tests/test_counting.cpp:30-46, test_orientation.cpp:54-185).
 *
 * Each function cites the reference file:line it restates; paths are
 * relative to /root/reference/proj.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- ranking -------------------------------------------------------- */

/* rank_by_degree, src/orientation.cpp:10-17: stable sort of ids by degree
 * (ties keep id order), restated as a counting sort. */
int kco_rank_degree(uint32_t n, const uint64_t* off, uint32_t* rank) {
  uint64_t maxd = 0;
  for (uint32_t v = 0; v < n; v++)
    if (off[v + 1] - off[v] > maxd) maxd = off[v + 1] - off[v];
  uint64_t* start = calloc(maxd + 2, sizeof(uint64_t));
  if (!start) return 3;
  for (uint32_t v = 0; v < n; v++) start[off[v + 1] - off[v] + 1]++;
  for (uint64_t d = 0; d <= maxd; d++) start[d + 1] += start[d];
  for (uint32_t v = 0; v < n; v++) rank[v] = (uint32_t)start[off[v + 1] - off[v]]++;
  free(start);
  return 0;
}

/* estimate_arboricity, src/orientation.cpp:124-155.  Batch members are
 * processed in id order; each one's alive neighbours lose a degree and an
 * edge before the member itself dies, so intra-batch edges count once. */
int kco_estimate_arboricity(uint32_t n, uint64_t m, const uint64_t* off,
                            const uint32_t* adj, double eps, uint64_t* out) {
  if (!(eps > 0)) return 1;
  uint64_t* deg = malloc((size_t)n * 8 + 8);
  uint8_t* alive = malloc((size_t)n + 1);
  uint32_t* rem = malloc((size_t)n * 4 + 4);
  uint32_t* batch = malloc((size_t)n * 4 + 4);
  if (!deg || !alive || !rem || !batch) return 3;
  for (uint32_t v = 0; v < n; v++) {
    deg[v] = off[v + 1] - off[v];
    alive[v] = 1;
    rem[v] = v;
  }
  uint64_t nrem = n, edges_left = m;
  double peak = 0;
  while (nrem) {
    double density = (double)edges_left / (double)nrem;
    if (density > peak) peak = density;
    double cutoff = 2 * (1 + eps) * density;
    uint64_t nb = 0;
    for (uint64_t i = 0; i < nrem; i++)
      if ((double)deg[rem[i]] <= cutoff) batch[nb++] = rem[i];
    for (uint64_t i = 0; i < nb; i++) {
      uint32_t v = batch[i];
      for (uint64_t p = off[v]; p < off[v + 1]; p++)
        if (alive[adj[p]]) {
          deg[adj[p]]--;
          edges_left--;
        }
      alive[v] = 0;
    }
    uint64_t w = 0;
    for (uint64_t i = 0; i < nrem; i++)
      if (alive[rem[i]]) rem[w++] = rem[i];
    nrem = w;
  }
  uint64_t a = (uint64_t)ceil(peak);
  *out = a < 1 ? 1 : a;
  free(deg), free(alive), free(rem), free(batch);
  return 0;
}

/* rank_barenboim_elkin, src/orientation.cpp:86-122: each round removes
 * every remaining vertex with double(deg) < threshold, in id order; an
 * empty round doubles the threshold and still counts as a round;
 * decrements apply only to survivors of the round. */
int kco_rank_be(uint32_t n, const uint64_t* off, const uint32_t* adj,
                double eps, uint64_t alpha_hat, uint32_t* rank,
                uint64_t* rounds_out) {
  if (!(eps > 0)) return 1;
  if (alpha_hat < 1) return 1;
  uint64_t* deg = malloc((size_t)n * 8 + 8);
  uint8_t* alive = malloc((size_t)n + 1);
  uint32_t* rem = malloc((size_t)n * 4 + 4);
  uint32_t* batch = malloc((size_t)n * 4 + 4);
  if (!deg || !alive || !rem || !batch) return 3;
  for (uint32_t v = 0; v < n; v++) {
    deg[v] = off[v + 1] - off[v];
    alive[v] = 1;
    rem[v] = v;
  }
  double threshold = (2 + eps) * (double)alpha_hat;
  uint64_t nrem = n, rounds = 0, placed = 0;
  while (nrem) {
    rounds++;
    uint64_t nb = 0;
    for (uint64_t i = 0; i < nrem; i++)
      if ((double)deg[rem[i]] < threshold) batch[nb++] = rem[i];
    if (nb == 0) {
      threshold *= 2;
      continue;
    }
    for (uint64_t i = 0; i < nb; i++) {
      rank[batch[i]] = (uint32_t)placed++;
      alive[batch[i]] = 0;
    }
    for (uint64_t i = 0; i < nb; i++)
      for (uint64_t p = off[batch[i]]; p < off[batch[i] + 1]; p++)
        if (alive[adj[p]]) deg[adj[p]]--;
    uint64_t w = 0;
    for (uint64_t i = 0; i < nrem; i++)
      if (alive[rem[i]]) rem[w++] = rem[i];
    nrem = w;
  }
  if (rounds_out) *rounds_out = rounds;
  free(deg), free(alive), free(rem), free(batch);
  return 0;
}

/* rank_by_kcore, src/orientation.cpp:23-46: lazy-deletion min-heap on
 * (induced degree, id); pops one vertex at a time. */
typedef struct { uint64_t d; uint32_t v; } kco_entry;
static int entry_less(kco_entry a, kco_entry b) {
  return a.d < b.d || (a.d == b.d && a.v < b.v);
}
int kco_rank_kcore(uint32_t n, const uint64_t* off, const uint32_t* adj,
                   uint32_t* rank) {
  uint64_t cap = (uint64_t)n + (n ? off[n] : 0) + 1, size = 0;
  kco_entry* heap = malloc(cap * sizeof(kco_entry));
  uint64_t* deg = malloc((size_t)n * 8 + 8);
  uint8_t* done = calloc((size_t)n + 1, 1);
  if (!heap || !deg || !done) return 3;
#define KCO_PUSH(D, V)                                                  \
  do {                                                                  \
    kco_entry e_ = {(D), (V)};                                          \
    uint64_t i_ = size++;                                               \
    while (i_ && entry_less(e_, heap[(i_ - 1) / 2])) {                  \
      heap[i_] = heap[(i_ - 1) / 2];                                    \
      i_ = (i_ - 1) / 2;                                                \
    }                                                                   \
    heap[i_] = e_;                                                      \
  } while (0)
  for (uint32_t v = 0; v < n; v++) {
    deg[v] = off[v + 1] - off[v];
    KCO_PUSH(deg[v], v);
  }
  uint32_t placed = 0;
  while (size) {
    kco_entry top = heap[0];
    kco_entry last = heap[--size];
    uint64_t i = 0;
    for (;;) {
      uint64_t c = 2 * i + 1;
      if (c >= size) break;
      if (c + 1 < size && entry_less(heap[c + 1], heap[c])) c++;
      if (!entry_less(heap[c], last)) break;
      heap[i] = heap[c];
      i = c;
    }
    if (size) heap[i] = last;
    if (done[top.v] || top.d != deg[top.v]) continue;
    done[top.v] = 1;
    rank[top.v] = placed++;
    for (uint64_t p = off[top.v]; p < off[top.v + 1]; p++) {
      uint32_t u = adj[p];
      if (!done[u]) {
        deg[u]--;
        KCO_PUSH(deg[u], u);
      }
    }
  }
#undef KCO_PUSH
  free(heap), free(deg), free(done);
  return 0;
}

/* ---- orientation ---------------------------------------------------- */

/* direct_by_ranking, src/graph.cpp:94-114: keep u->v iff rank(v) >
 * rank(u); slices keep the undirected slice's ascending id order.
 * out_off has n+1 entries, out_adj m entries. */
int kco_direct(uint32_t n, const uint64_t* off, const uint32_t* adj,
               const uint32_t* rank, uint64_t* out_off, uint32_t* out_adj) {
  out_off[0] = 0;
  uint64_t pos = 0;
  for (uint32_t u = 0; u < n; u++) {
    for (uint64_t p = off[u]; p < off[u + 1]; p++)
      if (rank[adj[p]] > rank[u]) out_adj[pos++] = adj[p];
    out_off[u + 1] = pos;
  }
  return 0;
}

/* ---- counting ------------------------------------------------------- */

typedef struct {
  const uint64_t* off;
  const uint32_t* adj;
  uint64_t* stamp;   /* per-vertex token marks (clique_rec.hpp:24-62) */
  uint32_t** bufs;   /* candidate buffers per depth */
  uint64_t* pv;      /* may be NULL */
  uint32_t* chain;
  int chain_len;
} kco_ctx;

/* clique_rec, src/clique_rec.hpp:24-62, in global id space with the
 * stamp array (edge engine, src/counting.cpp:174-186). */
static uint64_t kco_rec(kco_ctx* c, const uint32_t* cands, uint64_t ncand,
                        int remaining, int depth, uint64_t token_base) {
  if (ncand < (uint64_t)remaining) return 0;
  if (remaining == 1) {
    if (c->pv) {
      for (uint64_t i = 0; i < ncand; i++) c->pv[cands[i]]++;
      for (int i = 0; i < c->chain_len; i++) c->pv[c->chain[i]] += ncand;
    }
    return ncand;
  }
  const uint64_t token = token_base + (uint64_t)depth;
  uint64_t total = 0;
  uint32_t* next = c->bufs[depth + 1];
  for (uint64_t i = 0; i < ncand; i++) {
    uint32_t u = cands[i];
    uint64_t nn = 0;
    for (uint64_t p = c->off[u]; p < c->off[u + 1]; p++)
      if (c->stamp[c->adj[p]] == token) next[nn++] = c->adj[p];
    if (nn + 1 < (uint64_t)remaining) continue;
    for (uint64_t j = 0; j < nn; j++) c->stamp[next[j]] = token + 1;
    c->chain[c->chain_len++] = u;
    total += kco_rec(c, next, nn, remaining - 1, depth + 1, token_base);
    c->chain_len--;
    for (uint64_t j = 0; j < nn; j++) c->stamp[next[j]] = token;
  }
  return total;
}

/* count_impl edge engine, src/counting.cpp:138-189 (serial): one task per
 * directed edge (v,u); candidates = N+(v) ∩ N+(u) by sorted merge; k==2
 * special case.  pv (n entries) may be NULL.  Returns 1 for k < 2. */
int kco_count(uint32_t n, const uint64_t* out_off, const uint32_t* out_adj,
              int k, uint64_t* total_out, uint64_t* pv) {
  if (k < 2) return 1;
  uint64_t maxd = 0;
  for (uint32_t v = 0; v < n; v++)
    if (out_off[v + 1] - out_off[v] > maxd) maxd = out_off[v + 1] - out_off[v];
  kco_ctx c;
  c.off = out_off;
  c.adj = out_adj;
  c.pv = pv;
  c.stamp = calloc((size_t)n + 1, 8);
  c.chain = malloc(((size_t)k + 2) * 4);
  c.bufs = malloc(((size_t)k + 3) * sizeof(uint32_t*));
  if (!c.stamp || !c.chain || !c.bufs) return 3;
  for (int i = 0; i < k + 3; i++) {
    c.bufs[i] = malloc((maxd + 1) * 4);
    if (!c.bufs[i]) return 3;
  }
  if (pv) memset(pv, 0, (size_t)n * 8);
  uint64_t total = 0, next_token = 1;
  for (uint32_t v = 0; v < n; v++) {
    for (uint64_t e = out_off[v]; e < out_off[v + 1]; e++) {
      uint32_t u = out_adj[e];
      if (k == 2) {
        total++;
        if (pv) pv[v]++, pv[u]++;
        continue;
      }
      /* std::set_intersection of two id-sorted slices (counting.cpp:178) */
      uint32_t* both = c.bufs[2];
      uint64_t nb = 0, a = out_off[v], b = out_off[u];
      while (a < out_off[v + 1] && b < out_off[u + 1]) {
        if (out_adj[a] < out_adj[b]) a++;
        else if (out_adj[b] < out_adj[a]) b++;
        else { both[nb++] = out_adj[a]; a++; b++; }
      }
      if (nb + 2 < (uint64_t)k) continue;
      uint64_t tb = next_token;
      next_token += (uint64_t)k + 2;
      for (uint64_t i = 0; i < nb; i++) c.stamp[both[i]] = tb + 2;
      c.chain[0] = v;
      c.chain[1] = u;
      c.chain_len = 2;
      total += kco_rec(&c, both, nb, k - 2, 2, tb);
    }
  }
  *total_out = total;
  for (int i = 0; i < k + 3; i++) free(c.bufs[i]);
  free(c.bufs), free(c.chain), free(c.stamp);
  return 0;
}

/* Closed-form algorithmic staging bytes of the paper's per-source scheme
 * (SURVEY.md §8(d)): 16n + 20m + 4 * sum_w indeg(w) * outdeg(w). */
uint64_t kco_alg_bytes(uint32_t n, const uint64_t* out_off, const uint32_t* out_adj) {
  uint64_t m = n ? out_off[n] : 0;
  uint64_t* indeg = calloc((size_t)n + 1, 8);
  for (uint64_t e = 0; e < m; e++) indeg[out_adj[e]]++;
  uint64_t s = 0;
  for (uint32_t w = 0; w < n; w++) s += indeg[w] * (out_off[w + 1] - out_off[w]);
  free(indeg);
  return 16 * (uint64_t)n + 20 * m + 4 * s;
}

/* The multi-GPU split, restated for the CPU tests: only
 * the cliques whose lowest-ranked vertex v passes the source filter -- the
 * edge tasks (v,u) of counting.cpp:158-187 with such a source v.
 * mode 0: rank[v] % nparts == part (kco_count_part);
 * mode 1: lo <= rank[v] < hi (kco_count_range, the contiguous ranges of
 * kcg_partition_plan / shard.plan). */
static int kco_count_sources(uint32_t n, const uint64_t* out_off, const uint32_t* out_adj,
                             const uint32_t* rank, int k, int mode, uint32_t a0, uint32_t a1,
                             uint64_t* total_out, uint64_t* pv) {
  uint64_t total = 0;
  if (pv) memset(pv, 0, (size_t)n * 8);
  uint64_t maxd = 0;
  for (uint32_t v = 0; v < n; v++)
    if (out_off[v + 1] - out_off[v] > maxd) maxd = out_off[v + 1] - out_off[v];
  kco_ctx c;
  c.off = out_off;
  c.adj = out_adj;
  c.pv = pv;
  c.stamp = calloc((size_t)n + 1, 8);
  c.chain = malloc(((size_t)k + 2) * 4);
  c.bufs = malloc(((size_t)k + 3) * sizeof(uint32_t*));
  if (!c.stamp || !c.chain || !c.bufs) return 3;
  for (int i = 0; i < k + 3; i++) c.bufs[i] = malloc((maxd + 1) * 4);
  uint64_t next_token = 1;
  for (uint32_t v = 0; v < n; v++) {
    if (mode == 0 ? rank[v] % a1 != a0 : (rank[v] < a0 || rank[v] >= a1)) continue;
    for (uint64_t e = out_off[v]; e < out_off[v + 1]; e++) {
      uint32_t u = out_adj[e];
      if (k == 2) {
        total++;
        if (pv) pv[v]++, pv[u]++;
        continue;
      }
      uint32_t* both = c.bufs[2];
      uint64_t nb = 0, a = out_off[v], b = out_off[u];
      while (a < out_off[v + 1] && b < out_off[u + 1]) {
        if (out_adj[a] < out_adj[b]) a++;
        else if (out_adj[b] < out_adj[a]) b++;
        else { both[nb++] = out_adj[a]; a++; b++; }
      }
      if (nb + 2 < (uint64_t)k) continue;
      uint64_t tb = next_token;
      next_token += (uint64_t)k + 2;
      for (uint64_t i = 0; i < nb; i++) c.stamp[both[i]] = tb + 2;
      c.chain[0] = v;
      c.chain[1] = u;
      c.chain_len = 2;
      total += kco_rec(&c, both, nb, k - 2, 2, tb);
    }
  }
  *total_out = total;
  for (int i = 0; i < k + 3; i++) free(c.bufs[i]);
  free(c.bufs), free(c.chain), free(c.stamp);
  return 0;
}

int kco_count_part(uint32_t n, const uint64_t* out_off, const uint32_t* out_adj,
                   const uint32_t* rank, int k, uint32_t part, uint32_t nparts,
                   uint64_t* total_out, uint64_t* pv) {
  if (k < 2 || nparts == 0 || part >= nparts) return 1;
  return kco_count_sources(n, out_off, out_adj, rank, k, 0, part, nparts, total_out, pv);
}

int kco_count_range(uint32_t n, const uint64_t* out_off, const uint32_t* out_adj,
                    const uint32_t* rank, int k, uint32_t r_lo, uint32_t r_hi,
                    uint64_t* total_out, uint64_t* pv) {
  if (k < 2 || r_lo > r_hi) return 1;
  return kco_count_sources(n, out_off, out_adj, rank, k, 1, r_lo, r_hi, total_out, pv);
}

/* ---- peeling --------------------------------- */

/* Per-vertex k-clique counts of the subgraph induced by the live vertices
 * (dead ones isolated), by recounting from scratch: the residual graph is
 * degree-ordered and counted with kco_count.  This is the "sequential
 * recounting reference" the reference's own peeling tests compare against
 * (proj/tests/test_peeling.cpp:23-52, testutil.hpp reference_peel). */
static int kco_residual(uint32_t n, const uint64_t* off, const uint32_t* adj,
                        const uint8_t* live, int k, uint64_t* total, uint64_t* pv) {
  uint64_t* roff = calloc((size_t)n + 1, sizeof(uint64_t));
  uint64_t two_m = off[n];
  uint32_t* radj = malloc((two_m ? two_m : 1) * sizeof(uint32_t));
  uint32_t* rank = malloc(((size_t)n + 1) * sizeof(uint32_t));
  uint64_t* doff = malloc(((size_t)n + 1) * sizeof(uint64_t));
  uint32_t* dadj = malloc((two_m ? two_m : 1) * sizeof(uint32_t));
  int rc = 3;
  if (!roff || !radj || !rank || !doff || !dadj) goto out;
  for (uint32_t v = 0; v < n; v++) {
    roff[v + 1] = roff[v];
    if (!live[v]) continue;
    for (uint64_t p = off[v]; p < off[v + 1]; p++)
      if (live[adj[p]]) radj[roff[v + 1]++] = adj[p];
  }
  if ((rc = kco_rank_degree(n, roff, rank))) goto out;
  if ((rc = kco_direct(n, roff, radj, rank, doff, dadj))) goto out;
  rc = kco_count(n, doff, dadj, k, total, pv);
out:
  free(roff);
  free(radj);
  free(rank);
  free(doff);
  free(dadj);
  return rc;
}

/* update_counts, src/peeling.cpp:114-200, restated as recount differencing
 * (test_peeling.cpp:101-148 checks the reference against exactly this):
 * every survivor u loses pv_A[u] - pv_{A\B}[u] cliques, removed =
 * tot_A - tot_{A\B}.  Status 1 for a peeled / out-of-range batch vertex
 * (peeling.cpp:133-136), 4 when a count would go negative (159-161).
 * changed (n capacity) receives the survivors whose count dropped,
 * ascending. */
int kco_update_counts(uint32_t n, const uint64_t* off, const uint32_t* adj, int k,
                      uint64_t* counts, const uint32_t* batch, uint64_t nb,
                      const uint8_t* peeled, uint64_t* removed, uint32_t* changed,
                      uint64_t* nchanged) {
  if (k < 2) return 1;
  for (uint64_t i = 0; i < nb; i++)
    if (batch[i] >= n || peeled[batch[i]]) return 1;
  uint8_t* live = malloc((size_t)n + 1);
  uint64_t* pa = malloc(((size_t)n + 1) * sizeof(uint64_t));
  uint64_t* pb = malloc(((size_t)n + 1) * sizeof(uint64_t));
  int rc = 3;
  if (!live || !pa || !pb) goto out;
  for (uint32_t v = 0; v < n; v++) live[v] = !peeled[v];
  uint64_t ta = 0, tb = 0;
  if ((rc = kco_residual(n, off, adj, live, k, &ta, pa))) goto out;
  for (uint64_t i = 0; i < nb; i++) live[batch[i]] = 0;
  if ((rc = kco_residual(n, off, adj, live, k, &tb, pb))) goto out;
  int under = 0;
  *nchanged = 0;
  for (uint32_t v = 0; v < n; v++) {
    if (!live[v]) continue;
    uint64_t d = pa[v] - pb[v];
    if (d > counts[v]) under = 1;
    counts[v] -= d;
    if (d) changed[(*nchanged)++] = v;
  }
  *removed = ta - tb;
  rc = under ? 4 : 0;
out:
  free(live);
  free(pa);
  free(pb);
  return rc;
}

/* peel_exact / peel_approx, src/peeling.cpp:202-320: rounds extract every
 * live vertex of minimum count (exact; core = running max of the extracted
 * values) or every live vertex with double(count) <= k (1+eps) rem / alive
 * (approx), counts recomputed from scratch on the residual graph each
 * round; best density compared as exact fractions (peeling.cpp:196-211).
 * res = {rounds, total, best_round, num_dense}; core (n, exact only) and
 * dense (n) are outputs. */
int kco_peel(uint32_t n, const uint64_t* off, const uint32_t* adj, int k, int exact,
             double eps, uint64_t* res, double* density, uint64_t* core, uint32_t* dense) {
  if (k < 2) return 1;
  if (!exact && !(eps > 0)) return 1;
  memset(res, 0, 4 * sizeof(uint64_t));
  *density = 0.0;
  if (n == 0) return 0;
  uint8_t* live = malloc(n);
  uint64_t* cur = malloc((size_t)n * sizeof(uint64_t));
  uint64_t* round_of = malloc((size_t)n * sizeof(uint64_t));
  int rc = 3;
  if (!live || !cur || !round_of) goto out;
  memset(live, 1, n);
  uint64_t total = 0;
  if ((rc = kco_residual(n, off, adj, live, k, &total, cur))) goto out;
  res[1] = total;
  uint64_t best_c = 0, best_a = 1, best_r = 0;
  if ((unsigned __int128)total * best_a > (unsigned __int128)best_c * n) {
    best_c = total;
    best_a = n;
  }
  uint64_t rem = total, alive = n, round = 0, level = 0;
  while (alive > 0) {
    round++;
    uint64_t mn = UINT64_MAX;
    double cutoff = 0;
    if (exact) {
      for (uint32_t v = 0; v < n; v++)
        if (live[v] && cur[v] < mn) mn = cur[v];
      if (mn > level) level = mn;
    } else {
      cutoff = (double)k * (1.0 + eps) * ((double)rem / (double)alive);
    }
    uint64_t nb = 0;
    for (uint32_t v = 0; v < n; v++) {
      if (!live[v]) continue;
      if (exact ? cur[v] == mn : (double)cur[v] <= cutoff) {
        live[v] = 0;
        round_of[v] = round;
        if (exact) core[v] = level;
        nb++;
      }
    }
    if (nb == 0) {
      rc = 4;
      goto out;
    }
    alive -= nb;
    if ((rc = kco_residual(n, off, adj, live, k, &rem, cur))) goto out;
    if (alive && (unsigned __int128)rem * best_a > (unsigned __int128)best_c * alive) {
      best_c = rem;
      best_a = alive;
      best_r = round;
    }
  }
  res[0] = round;
  res[2] = best_r;
  res[3] = 0;
  for (uint32_t v = 0; v < n; v++)
    if (round_of[v] > best_r) dense[res[3]++] = v;
  *density = best_a ? (double)best_c / (double)best_a : 0.0;
  rc = 0;
out:
  free(live);
  free(cur);
  free(round_of);
  return rc;
}

/* ---- colour sparsification ------------------- */

static uint64_t kco_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* color_of, src/sampling.cpp:17-24 */
uint64_t kco_color(uint64_t seed, uint32_t v, uint64_t colors) {
  uint64_t h = kco_splitmix64(kco_splitmix64(seed) + 0x9e3779b97f4a7c15ULL * ((uint64_t)v + 1));
  return (uint64_t)(((unsigned __int128)h * colors) >> 64);
}

/* colorful_sparsify, src/sampling.cpp:28-40: the monochromatic edges of the
 * CSR, written as a CSR (out_off n+1, out_adj up to 2m).  Slices stay
 * ascending, which is Graph::from_edges of the kept pairs. */
int kco_sparsify(uint32_t n, const uint64_t* off, const uint32_t* adj, uint64_t colors,
                 uint64_t seed, uint64_t* out_off, uint32_t* out_adj) {
  if (colors < 1) return 1;
  uint64_t* col = malloc(((size_t)n + 1) * sizeof(uint64_t));
  if (!col) return 3;
  for (uint32_t v = 0; v < n; v++) col[v] = colors == 1 ? 0 : kco_color(seed, v, colors);
  out_off[0] = 0;
  for (uint32_t v = 0; v < n; v++) {
    out_off[v + 1] = out_off[v];
    for (uint64_t p = off[v]; p < off[v + 1]; p++)
      if (col[adj[p]] == col[v]) out_adj[out_off[v + 1]++] = adj[p];
  }
  free(col);
  return 0;
}

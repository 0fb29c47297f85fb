// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" wrapper around the UNMODIFIED reference library, compiled from
// the sources where they lie under /root/reference/proj/src by
// oracle/Makefile into oracle/_ref/libkclique_ref.so.  Used by tests/ as the
// pinning oracle, and by bench.py --impl reference as the CPU arm.
//
// Every entry point maps the reference's exceptions onto the same status
// codes as the product C ABI (include/kcg.h): 0 ok, 1 invalid argument,
// 2 runtime error, 3 out of memory, 4 logic error.
#include <omp.h>

#include <chrono>
#include <cstdint>
#include <cstring>
#include <new>
#include <span>
#include <stdexcept>
#include <vector>

#include "kclique/counting.hpp"
#include "kclique/graph.hpp"
#include "kclique/oracle.hpp"
#include "kclique/orientation.hpp"
#include "kclique/peeling.hpp"
#include "kclique/sampling.hpp"

using namespace kclique;

namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (const std::logic_error&) {
    return 4;
  } catch (const std::bad_alloc&) {
    return 3;
  } catch (...) {
    return 2;
  }
}

double now_s() {
  return std::chrono::duration<double>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

}  // namespace

extern "C" {

void ref_set_threads(int t) {
  if (t > 0) omp_set_num_threads(t);
}
int ref_max_threads(void) { return omp_get_max_threads(); }

// Builds a reference Graph from a symmetric CSR (only u<v entries used).
int ref_graph_create(uint32_t n, const uint64_t* off, const uint32_t* adj,
                     void** out) {
  return guarded([&] {
    std::vector<std::pair<VertexId, VertexId>> edges;
    edges.reserve(n ? off[n] / 2 : 0);
    for (uint32_t u = 0; u < n; u++)
      for (uint64_t p = off[u]; p < off[u + 1]; p++)
        if (adj[p] > u) edges.emplace_back(u, adj[p]);
    *out = new Graph(Graph::from_edges(n, std::move(edges)));
  });
}

int ref_graph_from_edge_list(uint32_t n, const uint32_t* us,
                             const uint32_t* vs, uint64_t cnt, void** out) {
  return guarded([&] {
    std::vector<std::pair<VertexId, VertexId>> edges(cnt);
    for (uint64_t i = 0; i < cnt; i++) edges[i] = {us[i], vs[i]};
    *out = new Graph(Graph::from_edges(n, std::move(edges)));
  });
}

void ref_graph_destroy(void* g) { delete static_cast<Graph*>(g); }

uint64_t ref_graph_m(void* g) { return static_cast<Graph*>(g)->num_edges(); }

int ref_graph_csr(void* g, uint64_t* off, uint32_t* adj) {
  const Graph& G = *static_cast<Graph*>(g);
  std::memcpy(off, G.offsets().data(), G.offsets().size() * 8);
  std::memcpy(adj, G.adjacency().data(), G.adjacency().size() * 4);
  return 0;
}

// strategy: 0 degree, 1 original, 2 kcore, 3 goodrich_pszona,
// 4 barenboim_elkin (alpha_hat == 0 -> estimated, as make_ranking does)
int ref_rank(void* g, int strategy, double eps, uint64_t alpha_hat,
             uint32_t* rank_out, uint64_t* rounds_out, double* seconds) {
  return guarded([&] {
    const Graph& G = *static_cast<Graph*>(g);
    double t0 = now_s();
    Ranking r;
    uint64_t rounds = 0;
    switch (strategy) {
      case 0: r = rank_by_degree(G); break;
      case 1: r = rank_original(G); break;
      case 2: r = rank_by_kcore(G); break;
      case 3: r = rank_goodrich_pszona(G, eps, &rounds); break;
      case 4: {
        uint64_t a = alpha_hat ? alpha_hat : estimate_arboricity(G, eps);
        r = rank_barenboim_elkin(G, eps, a, &rounds);
        break;
      }
      case 5: {  // make_ranking dispatch for barenboim_elkin
        OrientConfig cfg{OrientStrategy::barenboim_elkin, eps, {}};
        if (alpha_hat) cfg.alpha_hat = alpha_hat;
        r = make_ranking(G, cfg);
        break;
      }
      default: throw std::invalid_argument("strategy");
    }
    if (seconds) *seconds = now_s() - t0;
    std::memcpy(rank_out, r.ranks().data(), size_t(r.size()) * 4);
    if (rounds_out) *rounds_out = rounds;
  });
}

int ref_estimate_arboricity(void* g, double eps, uint64_t* out) {
  return guarded([&] { *out = estimate_arboricity(*static_cast<Graph*>(g), eps); });
}

int ref_direct(void* g, const uint32_t* rank, void** out, double* seconds) {
  return guarded([&] {
    const Graph& G = *static_cast<Graph*>(g);
    std::vector<VertexId> rv(rank, rank + G.num_vertices());
    Ranking r(std::move(rv));
    double t0 = now_s();
    auto* dg = new DirectedGraph(direct_by_ranking(G, r));
    if (seconds) *seconds = now_s() - t0;
    *out = dg;
  });
}

int ref_direct_sized(void* g, const uint32_t* rank, uint32_t rank_len, void** out) {
  return guarded([&] {
    const Graph& G = *static_cast<Graph*>(g);
    std::vector<VertexId> rv(rank, rank + rank_len);
    *out = new DirectedGraph(direct_by_ranking(G, Ranking(std::move(rv))));
  });
}

void ref_dg_destroy(void* dg) { delete static_cast<DirectedGraph*>(dg); }

int ref_dg_csr(void* dgp, uint64_t* off, uint32_t* adj) {
  const DirectedGraph& dg = *static_cast<DirectedGraph*>(dgp);
  for (uint32_t v = 0; v <= dg.num_vertices(); v++)
    off[v] = v < dg.num_vertices() ? dg.out_offset(v) : dg.num_edges();
  std::memcpy(adj, dg.out_targets().data(), dg.out_targets().size() * 4);
  return 0;
}

uint64_t ref_dg_max_out_degree(void* dgp) {
  return static_cast<DirectedGraph*>(dgp)->max_out_degree();
}

// parallelism: 0 node, 1 edge, 2 default_parallelism(k)
int ref_count(void* dgp, int k, int parallelism, int build_induced,
              int want_pv, uint64_t* total, uint64_t* pv, double* seconds) {
  return guarded([&] {
    const DirectedGraph& dg = *static_cast<DirectedGraph*>(dgp);
    CountConfig cfg;
    cfg.parallelism = parallelism == 0   ? Parallelism::node
                      : parallelism == 1 ? Parallelism::edge
                                         : default_parallelism(k);
    cfg.build_induced = build_induced != 0;
    double t0 = now_s();
    CliqueCounts c = want_pv ? count_per_vertex(dg, k, cfg) : count_total(dg, k, cfg);
    if (seconds) *seconds = now_s() - t0;
    *total = c.total;
    if (want_pv && pv) std::memcpy(pv, c.per_vertex.data(), c.per_vertex.size() * 8);
  });
}

int ref_brute_force(void* g, int k, uint64_t* total, uint64_t* pv) {
  return guarded([&] {
    CliqueCounts c = oracle::brute_force_count(*static_cast<Graph*>(g), k);
    *total = c.total;
    if (pv) std::memcpy(pv, c.per_vertex.data(), c.per_vertex.size() * 8);
  });
}

int ref_exact_arboricity(void* g, uint64_t* out) {
  return guarded([&] { *out = oracle::exact_arboricity(*static_cast<Graph*>(g)); });
}

// update_counts (peeling.cpp:194-200): counts in/out (n), changed out (n
// capacity).
int ref_update_counts(void* g, void* dg, int k, uint64_t* counts, const uint32_t* batch,
                      uint64_t batch_len, const uint8_t* peeled, uint64_t* removed,
                      uint32_t* changed, uint64_t* changed_len) {
  return guarded([&] {
    const Graph& G = *static_cast<Graph*>(g);
    const uint32_t n = G.num_vertices();
    UpdateResult r = update_counts(G, *static_cast<DirectedGraph*>(dg), k,
                                   std::span<uint64_t>(counts, n),
                                   std::span<const VertexId>(batch, batch_len),
                                   std::span<const uint8_t>(peeled, n));
    *removed = r.removed;
    *changed_len = r.changed.size();
    if (!r.changed.empty()) std::memcpy(changed, r.changed.data(), r.changed.size() * 4);
  });
}

// peel_exact / peel_approx (peeling.cpp:202-320).  res = {rounds, total,
// best_round, num_dense}; core (n, exact only) and dense (n) may be null.
int ref_peel(void* g, void* dg, int k, int exact, double eps, uint64_t* res, double* density,
             uint64_t* core, uint32_t* dense, double* seconds) {
  return guarded([&] {
    const Graph& G = *static_cast<Graph*>(g);
    const double t0 = now_s();
    PeelOutcome o = exact ? peel_exact(G, *static_cast<DirectedGraph*>(dg), k)
                          : peel_approx(G, *static_cast<DirectedGraph*>(dg), k, eps);
    if (seconds) *seconds = now_s() - t0;
    res[0] = o.rounds;
    res[1] = o.total_cliques;
    res[2] = o.best_round;
    res[3] = o.dense_vertices.size();
    *density = o.best_density;
    if (core && !o.core.empty()) std::memcpy(core, o.core.data(), o.core.size() * 8);
    if (dense && !o.dense_vertices.empty())
      std::memcpy(dense, o.dense_vertices.data(), o.dense_vertices.size() * 4);
  });
}

// colorful_sparsify (sampling.cpp:28-40) -> a new reference Graph
int ref_colorful_sparsify(void* g, uint64_t colors, uint64_t seed, void** out) {
  return guarded([&] {
    *out = new Graph(colorful_sparsify(*static_cast<Graph*>(g), colors, seed));
  });
}

// approx_count (sampling.cpp:42-57); res = {sub_count}, dres = {p, estimate}
int ref_approx_count(void* g, int k, uint64_t colors, uint64_t seed, int strategy, double eps,
                     uint64_t* sub_count, double* p, double* estimate) {
  return guarded([&] {
    OrientConfig oc;
    oc.strategy = static_cast<OrientStrategy>(strategy);
    oc.epsilon = eps;
    SampleEstimate e = approx_count(*static_cast<Graph*>(g), k, colors, seed, oc);
    *sub_count = e.sub_count;
    *p = e.p;
    *estimate = e.estimate;
  });
}

double ref_analytic_variance(uint64_t true_count, double p, int k, const uint64_t* pairs,
                             uint64_t npairs) {
  return analytic_variance(true_count, p, k, std::span<const uint64_t>(pairs, npairs));
}

}  // extern "C"

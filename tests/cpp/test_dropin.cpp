// Drop-in check: compiled against the repo's include/kclique/*.hpp and
// linked against libkclique_b200.so (which runs on the B200), exercising
// the reference API the way the reference's own unit tests do
// (proj/tests/test_counting.cpp, test_orientation.cpp, test_graph.cpp,
// test_peeling.cpp, test_bucket_queue.cpp, test_sampling.cpp).
// The expected values are the reference's known answers; the brute-force
// checker below is an independent exhaustive enumeration.
//
// Prints one line per case and "DROPIN OK <n>" / "DROPIN FAIL <n>" last;
// exit status 0 iff every check passed.
#include <algorithm>
#include <cstdio>
#include <functional>
#include <numeric>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "kclique/counting.hpp"
#include "kclique/graph.hpp"
#include "kclique/orientation.hpp"
#include "kclique/peeling.hpp"
#include "kclique/sampling.hpp"

using namespace kclique;

static int g_checks = 0, g_fail = 0;
#define CHECK(cond)                                                      \
  do {                                                                   \
    g_checks++;                                                          \
    if (!(cond)) {                                                       \
      g_fail++;                                                          \
      std::printf("  FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond);    \
    }                                                                    \
  } while (0)
#define CHECK_THROWS_AS(expr, exc)                                       \
  do {                                                                   \
    g_checks++;                                                          \
    bool ok_ = false;                                                    \
    try {                                                                \
      (void)(expr);                                                      \
    } catch (const exc&) {                                               \
      ok_ = true;                                                        \
    } catch (...) {                                                      \
    }                                                                    \
    if (!ok_) {                                                          \
      g_fail++;                                                          \
      std::printf("  FAILED %s:%d: %s throws %s\n", __FILE__, __LINE__,  \
                  #expr, #exc);                                          \
    }                                                                    \
  } while (0)

namespace {

// Fixture graphs with the reference's generator semantics
// (proj/tests/testutil.hpp:39-71): mt19937_64 raw bits, uniform = x>>11
// scaled by 2^-53, edge iff uniform < p.
Graph gnp(VertexId n, double p, uint64_t seed) {
  std::mt19937_64 eng(seed);
  std::vector<std::pair<VertexId, VertexId>> e;
  for (VertexId u = 0; u < n; u++)
    for (VertexId v = u + 1; v < n; v++)
      if (double(eng() >> 11) * 0x1.0p-53 < p) e.emplace_back(u, v);
  return Graph::from_edges(n, std::move(e));
}
Graph complete(VertexId n) { return gnp(n, 1.1, 1); }
Graph path_graph(VertexId n) {
  std::vector<std::pair<VertexId, VertexId>> e;
  for (VertexId v = 0; v + 1 < n; v++) e.emplace_back(v, v + 1);
  return Graph::from_edges(n, std::move(e));
}
Graph star(VertexId leaves) {
  std::vector<std::pair<VertexId, VertexId>> e;
  for (VertexId v = 1; v <= leaves; v++) e.emplace_back(0, v);
  return Graph::from_edges(leaves + 1, std::move(e));
}
Graph two_clumps() {
  std::vector<std::pair<VertexId, VertexId>> e;
  for (VertexId u = 0; u < 4; u++)
    for (VertexId v = u + 1; v < 4; v++) e.emplace_back(u, v);
  for (VertexId u = 3; u < 7; u++)
    for (VertexId v = u + 1; v < 7; v++) e.emplace_back(u, v);
  e.emplace_back(0, 7);
  return Graph::from_edges(8, std::move(e));
}

// Independent exhaustive count (ascending-id backtracking on the
// undirected graph) with per-vertex participation.
struct Brute {
  uint64_t total = 0;
  std::vector<uint64_t> pv;
};
Brute brute(const Graph& g, int k) {
  Brute b;
  b.pv.assign(g.num_vertices(), 0);
  std::vector<VertexId> cl;
  std::function<void(const std::vector<VertexId>&)> rec = [&](const std::vector<VertexId>& c) {
    if (int(cl.size()) == k) {
      b.total++;
      for (VertexId v : cl) b.pv[v]++;
      return;
    }
    for (VertexId x : c) {
      std::vector<VertexId> nx;
      for (VertexId y : c)
        if (y > x && g.has_edge(x, y)) nx.push_back(y);
      cl.push_back(x);
      rec(nx);
      cl.pop_back();
    }
  };
  std::vector<VertexId> all(g.num_vertices());
  std::iota(all.begin(), all.end(), 0);
  rec(all);
  return b;
}

DirectedGraph oriented(const Graph& g, OrientStrategy s = OrientStrategy::degree) {
  return direct_by_ranking(g, make_ranking(g, {s, 1.0, {}}));
}

uint64_t degeneracy(const Graph& g) {
  const VertexId n = g.num_vertices();
  std::vector<uint64_t> deg(n);
  std::vector<char> gone(n, 0);
  for (VertexId v = 0; v < n; v++) deg[v] = g.degree(v);
  uint64_t best = 0;
  for (VertexId s = 0; s < n; s++) {
    VertexId pick = n;
    for (VertexId v = 0; v < n; v++)
      if (!gone[v] && (pick == n || deg[v] < deg[pick])) pick = v;
    best = std::max(best, deg[pick]);
    gone[pick] = 1;
    for (VertexId u : g.neighbors(pick))
      if (!gone[u]) deg[u]--;
  }
  return best;
}

void case_fixed_counts() {
  CHECK(count_total(oriented(complete(6)), 4).total == 15);
  CHECK(count_total(oriented(complete(6)), 6).total == 1);
  CHECK(count_total(oriented(complete(6)), 7).total == 0);
  CHECK(count_total(oriented(two_clumps()), 3).total == 8);
  CHECK(count_total(oriented(path_graph(9)), 3).total == 0);
  CHECK_THROWS_AS(count_total(oriented(complete(3)), 1), std::invalid_argument);
  CHECK(count_total(oriented(complete(5)), 3).per_vertex.empty());
}

void case_k2() {
  for (uint64_t seed = 0; seed < 6; seed++) {
    Graph g = gnp(25, 0.3, seed);
    CHECK(count_total(oriented(g), 2).total == g.num_edges());
    auto pv = count_per_vertex(oriented(g), 2);
    for (VertexId v = 0; v < g.num_vertices(); v++) CHECK(pv.per_vertex[v] == g.degree(v));
  }
}

void case_orderings_agree() {
  const OrientStrategy all[] = {OrientStrategy::degree, OrientStrategy::original,
                                OrientStrategy::kcore, OrientStrategy::goodrich_pszona,
                                OrientStrategy::barenboim_elkin};
  for (uint64_t seed = 0; seed < 12; seed++) {
    Graph g = gnp(VertexId(8 + seed), 0.45, seed + 400);
    for (int k = 3; k <= 6; k++) {
      uint64_t want = brute(g, k).total;
      for (auto s : all) {
        DirectedGraph dg = oriented(g, s);
        for (Parallelism p : {Parallelism::node, Parallelism::edge})
          CHECK(count_total(dg, k, {p, true}).total == want);
      }
    }
  }
}

void case_per_vertex() {
  for (uint64_t seed = 0; seed < 8; seed++) {
    Graph g = gnp(14, 0.5, seed + 900);
    for (int k : {3, 4, 5}) {
      Brute want = brute(g, k);
      CliqueCounts got = count_per_vertex(oriented(g), k);
      CHECK(got.total == want.total);
      CHECK(got.per_vertex == want.pv);
      uint64_t s = std::accumulate(got.per_vertex.begin(), got.per_vertex.end(), uint64_t(0));
      CHECK(s == uint64_t(k) * got.total);
    }
  }
}

void case_degree_ranking() {
  Graph p3 = path_graph(3);
  Ranking r = rank_by_degree(p3);
  CHECK(r.rank_of(0) < r.rank_of(1));
  CHECK(r.rank_of(2) < r.rank_of(1));
  CHECK(rank_by_degree(complete(5)) == Ranking::identity(5));
  for (uint64_t seed = 0; seed < 8; seed++) {
    Graph g = gnp(18, 0.3, seed);
    DirectedGraph dg = direct_by_ranking(g, rank_by_degree(g));
    for (VertexId v = 0; v < g.num_vertices(); v++)
      for (VertexId u : dg.out_neighbors(v)) CHECK(g.degree(u) >= g.degree(v));
  }
}

void case_original_and_direct() {
  CHECK(rank_original(gnp(9, 0.4, 3)) == Ranking::identity(9));
  Graph tri = Graph::from_edges(3, {{0, 1}, {1, 2}, {0, 2}});
  DirectedGraph dg = direct_by_ranking(tri, rank_original(tri));
  CHECK(dg.out_degree(0) == 2);
  CHECK(dg.out_degree(1) == 1);
  CHECK(dg.out_degree(2) == 0);
  CHECK_THROWS_AS(direct_by_ranking(tri, Ranking::identity(2)), std::invalid_argument);
}

void case_kcore() {
  Graph p10 = path_graph(10);
  CHECK(direct_by_ranking(p10, rank_by_kcore(p10)).max_out_degree() == 1);
  Graph k5 = complete(5);
  DirectedGraph dg = direct_by_ranking(k5, rank_by_kcore(k5));
  std::vector<uint64_t> outs;
  for (VertexId v = 0; v < 5; v++) outs.push_back(dg.out_degree(v));
  std::sort(outs.begin(), outs.end());
  CHECK((outs == std::vector<uint64_t>{0, 1, 2, 3, 4}));
  for (uint64_t seed = 0; seed < 20; seed++) {
    Graph g = gnp(20, 0.25, seed);
    CHECK(direct_by_ranking(g, rank_by_kcore(g)).max_out_degree() == degeneracy(g));
  }
}

void case_be_and_gp() {
  uint64_t rounds = 0;
  Ranking r = rank_barenboim_elkin(complete(4), 1.0, 2, &rounds);
  CHECK(rounds == 1);
  CHECK(r == Ranking::identity(4));
  Graph s9 = star(9);
  r = rank_barenboim_elkin(s9, 1.0, 1, &rounds);
  CHECK(rounds == 2);
  CHECK(r.rank_of(0) == 9);
  CHECK(direct_by_ranking(s9, r).out_degree(0) == 0);
  CHECK(rank_barenboim_elkin(complete(8), 0.1, 1, &rounds).size() == 8);
  CHECK_THROWS_AS(rank_barenboim_elkin(s9, -1.0, 1), std::invalid_argument);
  CHECK_THROWS_AS(rank_barenboim_elkin(s9, 1.0, 0), std::invalid_argument);

  r = rank_goodrich_pszona(complete(4), 1.0, &rounds);
  CHECK(rounds == 4);
  CHECK(direct_by_ranking(star(9), rank_goodrich_pszona(star(9), 1.0)).max_out_degree() <= 3);
  CHECK_THROWS_AS(rank_goodrich_pszona(complete(3), 0.0), std::invalid_argument);
}

void case_arboricity() {
  CHECK(estimate_arboricity(path_graph(12), 1.0) == 1);
  CHECK(estimate_arboricity(Graph{}, 1.0) == 1);
  uint64_t k5 = estimate_arboricity(complete(5), 1.0);
  CHECK(k5 >= 2 && k5 <= 3);
  CHECK_THROWS_AS(estimate_arboricity(complete(3), 0.0), std::invalid_argument);
}

void case_dispatch() {
  Graph g = gnp(16, 0.4, 9);
  CHECK(make_ranking(g, {OrientStrategy::degree, 1.0, {}}) == rank_by_degree(g));
  CHECK(make_ranking(g, {OrientStrategy::original, 1.0, {}}) == Ranking::identity(16));
  CHECK(make_ranking(g, {OrientStrategy::kcore, 1.0, {}}) == rank_by_kcore(g));
  CHECK(make_ranking(g, {OrientStrategy::goodrich_pszona, 1.0, {}}) ==
        rank_goodrich_pszona(g, 1.0));
  uint64_t est = estimate_arboricity(g, 1.0);
  CHECK(make_ranking(g, {OrientStrategy::barenboim_elkin, 1.0, {}}) ==
        rank_barenboim_elkin(g, 1.0, est));
  CHECK(make_ranking(g, {OrientStrategy::barenboim_elkin, 1.0, 3}) ==
        rank_barenboim_elkin(g, 1.0, 3));
}

void case_dag_properties() {
  for (uint64_t seed = 0; seed < 10; seed++) {
    Graph g = gnp(20, 0.3, seed);
    std::vector<VertexId> order(g.num_vertices());
    std::iota(order.begin(), order.end(), 0);
    std::mt19937_64 eng(seed * 31 + 7);
    for (size_t i = order.size(); i > 1; i--) std::swap(order[i - 1], order[eng() % i]);
    Ranking r = Ranking::from_order(order);
    DirectedGraph dg = direct_by_ranking(g, r);
    uint64_t out_sum = 0;
    std::vector<std::pair<VertexId, VertexId>> sym;
    for (VertexId v = 0; v < g.num_vertices(); v++) {
      out_sum += dg.out_degree(v);
      auto s = dg.out_neighbors(v);
      for (size_t i = 0; i < s.size(); i++) {
        CHECK(r.rank_of(s[i]) > r.rank_of(v));
        if (i) CHECK(s[i - 1] < s[i]);
        CHECK(g.has_edge(v, s[i]));
        sym.emplace_back(v, s[i]);
      }
    }
    CHECK(out_sum == g.num_edges());
    CHECK(Graph::from_edges(g.num_vertices(), std::move(sym)) == g);
  }
}

void case_graph_io() {
  Graph g = Graph::from_edges(4, {{1, 0}, {0, 1}, {2, 2}, {3, 1}, {1, 3}});
  CHECK(g.num_edges() == 2 && g.has_edge(0, 1) && g.has_edge(1, 3) && g.degree(2) == 0);
  CHECK_THROWS_AS(Graph::from_edges(2, {{0, 2}}), std::invalid_argument);
  std::istringstream in("# header\n\n500 7\n7 9000000000\n");
  ParsedGraph pg = parse_edge_list(in);
  CHECK(pg.graph.num_vertices() == 3 && pg.graph.num_edges() == 2);
  CHECK((pg.original_ids == std::vector<uint64_t>{500, 7, 9000000000ULL}));
  std::istringstream bad("0 1\nfoo bar\n");
  uint64_t line = 0;
  try {
    parse_edge_list(bad);
  } catch (const ParseError& e) {
    line = e.line();
  }
  CHECK(line == 2);
  std::ostringstream out;
  serialize_edge_list(Graph::from_edges(4, {{2, 0}, {0, 1}, {3, 2}}), out);
  CHECK(out.str() == "0 1\n0 2\n2 3\n");
  CHECK_THROWS_AS(Ranking({0, 0}), std::invalid_argument);
  CHECK_THROWS_AS(Ranking::from_order(std::vector<VertexId>{1, 1}), std::invalid_argument);
  Ranking r({2, 0, 1});
  CHECK((r.order() == std::vector<VertexId>{1, 2, 0}));
}

void case_default_parallelism() {
  CHECK(default_parallelism(3) == Parallelism::node);
  CHECK(default_parallelism(7) == Parallelism::node);
  CHECK(default_parallelism(8) == Parallelism::edge);
}

// ---- peeling (proj/tests/test_peeling.cpp, test_bucket_queue.cpp) ----

void case_bucket_queue() {
  std::vector<uint64_t> vals = {5, 3, 9, 3, 5, 0};
  BucketQueue q(vals);
  CHECK(q.size() == 6);
  auto [v0, b0] = q.extract_min();
  CHECK(v0 == 0 && b0 == std::vector<VertexId>{5});
  auto [v1, b1] = q.extract_min();
  CHECK(v1 == 3 && (b1 == std::vector<VertexId>{1, 3}));
  auto [v2, b2] = q.extract_min();
  CHECK(v2 == 5 && (b2 == std::vector<VertexId>{0, 4}));
  auto [v3, b3] = q.extract_min();
  CHECK(v3 == 9 && b3 == std::vector<VertexId>{2});
  CHECK(q.empty());
  CHECK_THROWS_AS(q.extract_min(), std::logic_error);
  std::vector<uint64_t> v2s = {10, 20, 30};
  BucketQueue r(v2s);
  r.update(2, 1);
  CHECK(r.extract_min().first == 1);
  r.update(0, 500);
  CHECK(r.extract_min().first == 20);
  r.update(0, 499);
  r.update(0, 7);
  auto [w, bw] = r.extract_min();
  CHECK(w == 7 && bw == std::vector<VertexId>{0});
  CHECK_THROWS_AS(r.update(0, 3), std::logic_error);
  std::vector<uint64_t> v3s = {8, 8, 8};
  BucketQueue s3(v3s);
  s3.update(1, 3);
  CHECK(s3.value(1) == 3);
}

void case_update_counts() {
  Graph g = complete(4);
  DirectedGraph dg = oriented(g);
  std::vector<uint64_t> counts(4, 3);
  std::vector<uint8_t> peeled(4, 0);
  std::vector<VertexId> batch = {0};
  UpdateResult res = update_counts(g, dg, 3, counts, batch, peeled);
  CHECK(res.removed == 3);
  CHECK((res.changed == std::vector<VertexId>{1, 2, 3}));
  CHECK(counts[1] == 1 && counts[2] == 1 && counts[3] == 1);
  std::vector<uint64_t> c2(4, 3);
  std::vector<VertexId> all = {0, 1, 2, 3};
  res = update_counts(g, dg, 3, c2, all, peeled);
  CHECK(res.removed == 4 && res.changed.empty());
  peeled[2] = 1;
  std::vector<VertexId> b2 = {1, 2};
  CHECK_THROWS_AS(update_counts(g, dg, 3, c2, b2, peeled), std::invalid_argument);
  std::vector<uint8_t> none(4, 0);
  std::vector<uint64_t> zeros(4, 0);
  CHECK_THROWS_AS(update_counts(g, dg, 3, zeros, batch, none), std::logic_error);
  // recount differencing on random residual graphs (test_peeling.cpp:101-148)
  std::mt19937_64 rng(5);
  for (uint64_t seed = 0; seed < 6; seed++) {
    Graph h = gnp(12, 0.45, seed + 2200);
    DirectedGraph dh = oriented(h);
    for (int k : {3, 4}) {
      std::vector<uint8_t> pe(12, 0);
      std::vector<uint64_t> cur = brute(h, k).pv;
      std::vector<VertexId> alive(12);
      std::iota(alive.begin(), alive.end(), 0);
      while (!alive.empty()) {
        std::shuffle(alive.begin(), alive.end(), rng);
        size_t take = 1 + rng() % std::min<size_t>(alive.size(), 4);
        std::vector<VertexId> bt(alive.begin(), alive.begin() + take);
        std::sort(bt.begin(), bt.end());
        // residual before/after by exhaustive count
        auto residual = [&](const std::vector<uint8_t>& dead) {
          std::vector<std::pair<VertexId, VertexId>> e;
          for (VertexId v = 0; v < 12; v++)
            for (VertexId u : h.neighbors(v))
              if (v < u && !dead[v] && !dead[u]) e.emplace_back(v, u);
          return brute(Graph::from_edges(12, std::move(e)), k);
        };
        Brute before = residual(pe);
        UpdateResult ur = update_counts(h, dh, k, cur, bt, pe);
        for (VertexId v : bt) pe[v] = 1;
        alive.erase(alive.begin(), alive.begin() + take);
        Brute after = residual(pe);
        CHECK(ur.removed == before.total - after.total);
        std::vector<VertexId> ch;
        for (VertexId v = 0; v < 12; v++) {
          if (pe[v]) continue;
          CHECK(cur[v] == after.pv[v]);
          if (after.pv[v] != before.pv[v]) ch.push_back(v);
        }
        CHECK(ur.changed == ch);
      }
    }
  }
}

void case_peel() {
  Graph k5 = complete(5);
  PeelOutcome out = peel_exact(k5, oriented(k5), 3);
  CHECK(out.total_cliques == 10 && out.rounds == 1 && out.best_density == 2.0);
  CHECK(out.best_round == 0 && out.core == std::vector<uint64_t>(5, 6));
  CHECK((out.dense_vertices == std::vector<VertexId>{0, 1, 2, 3, 4}));
  Graph two = Graph::from_edges(6, {{0, 1}, {1, 2}, {0, 2}, {3, 4}, {4, 5}, {3, 5}});
  out = peel_exact(two, oriented(two), 3);
  CHECK(out.total_cliques == 2 && out.rounds == 1 && out.best_density == 2.0 / 6.0);
  CHECK(out.core == std::vector<uint64_t>(6, 1) && out.dense_vertices.size() == 6);
  out = peel_approx(k5, oriented(k5), 3, 0.5);
  CHECK(out.rounds == 1 && out.best_density == 2.0 && out.dense_vertices.size() == 5);
  Graph p = path_graph(8);
  out = peel_approx(p, oriented(p), 3, 0.5);
  CHECK(out.total_cliques == 0 && out.rounds == 1 && out.best_density == 0.0);
  CHECK_THROWS_AS(peel_exact(k5, oriented(k5), 1), std::invalid_argument);
  CHECK_THROWS_AS(peel_approx(k5, oriented(k5), 3, 0.0), std::invalid_argument);
  // exact peeling == sequential recounting (test_peeling.cpp:173-192)
  for (uint64_t seed = 0; seed < 10; seed++) {
    Graph g = gnp(VertexId(8 + seed % 7), 0.5, seed + 5100);
    const VertexId n = g.num_vertices();
    for (int k : {3, 4}) {
      PeelOutcome ex = peel_exact(g, oriented(g), k);
      std::vector<uint8_t> dead(n, 0);
      std::vector<uint64_t> core(n, 0), when(n, 0);
      uint64_t level = 0, rounds = 0, alive = n, bc = 0, ba = 1, br = 0;
      Brute b = brute(g, k);
      if (b.total * ba > bc * n) bc = b.total, ba = n;
      while (alive) {
        rounds++;
        uint64_t mn = UINT64_MAX;
        for (VertexId v = 0; v < n; v++)
          if (!dead[v]) mn = std::min(mn, b.pv[v]);
        level = std::max(level, mn);
        std::vector<VertexId> bt;
        for (VertexId v = 0; v < n; v++)
          if (!dead[v] && b.pv[v] == mn) bt.push_back(v);
        for (VertexId v : bt) dead[v] = 1, core[v] = level, when[v] = rounds;
        alive -= bt.size();
        std::vector<std::pair<VertexId, VertexId>> e;
        for (VertexId v = 0; v < n; v++)
          for (VertexId u : g.neighbors(v))
            if (v < u && !dead[v] && !dead[u]) e.emplace_back(v, u);
        b = brute(Graph::from_edges(n, std::move(e)), k);
        if (alive && b.total * ba > bc * alive) bc = b.total, ba = alive, br = rounds;
      }
      std::vector<VertexId> dense;
      for (VertexId v = 0; v < n; v++)
        if (when[v] > br) dense.push_back(v);
      CHECK(ex.core == core);
      CHECK(ex.rounds == rounds);
      CHECK(ex.best_round == br);
      CHECK(ex.best_density == double(bc) / double(ba));
      CHECK(ex.dense_vertices == dense);
    }
  }
}

// ---- list_cliques (proj/tests/test_counting.cpp:103-128) ----
void case_list_cliques() {
  for (uint64_t seed = 0; seed < 6; seed++) {
    Graph g = gnp(16, 0.55, seed + 900);
    for (auto s : {OrientStrategy::degree, OrientStrategy::original}) {
      Ranking r = make_ranking(g, {s, 1.0, {}});
      DirectedGraph dg = direct_by_ranking(g, r);
      for (int k : {2, 3, 4, 5}) {
        std::vector<std::vector<VertexId>> got;
        CliqueCounts c = list_cliques(dg, k, {}, [&](std::span<const VertexId> cl) {
          CHECK(cl.size() == size_t(k));
          for (size_t i = 1; i < cl.size(); i++) CHECK(r.rank_of(cl[i - 1]) < r.rank_of(cl[i]));
          std::vector<VertexId> ids(cl.begin(), cl.end());
          std::sort(ids.begin(), ids.end());
          for (size_t i = 0; i < ids.size(); i++)
            for (size_t j = i + 1; j < ids.size(); j++) CHECK(g.has_edge(ids[i], ids[j]));
          got.push_back(std::move(ids));
        });
        CHECK(c.total == brute(g, k).total);
        CHECK(got.size() == c.total);
        std::sort(got.begin(), got.end());
        CHECK(std::adjacent_find(got.begin(), got.end()) == got.end());
      }
    }
  }
  CHECK_THROWS_AS(list_cliques(oriented(complete(4)), 1, {}, [](std::span<const VertexId>) {}),
                  std::invalid_argument);
  bool thrown = false;
  try {
    list_cliques(oriented(complete(6)), 3, {},
                 [](std::span<const VertexId>) { throw std::out_of_range("stop"); });
  } catch (const std::out_of_range&) {
    thrown = true;
  }
  CHECK(thrown);
}

// ---- sampling (proj/tests/test_sampling.cpp) ----
void case_sampling() {
  Graph g = gnp(30, 0.3, 5);
  CHECK(colorful_sparsify(g, 1, 42) == g);
  SampleEstimate est = approx_count(g, 3, 1, 42);
  CHECK(est.p == 1.0 && est.sub_count == brute(g, 3).total);
  CHECK(est.estimate == double(est.sub_count));
  for (uint64_t seed : {1u, 2u, 3u}) {
    Graph h = gnp(40, 0.25, seed + 60);
    for (uint32_t colors : {2u, 3u, 5u}) {
      Graph sub = colorful_sparsify(h, colors, seed);
      CHECK(sub.num_vertices() == h.num_vertices() && sub.num_edges() <= h.num_edges());
      CHECK(sub == colorful_sparsify(h, colors, seed));
      for (VertexId v = 0; v < sub.num_vertices(); v++)
        for (VertexId u : sub.neighbors(v)) CHECK(h.has_edge(v, u));
      // exact count of the sparsified graph == approx_count's sub_count
      CHECK(approx_count(h, 3, colors, seed).sub_count == brute(sub, 3).total);
    }
  }
  Graph g24 = gnp(24, 0.4, 99);
  SampleEstimate e4 = approx_count(g24, 4, 3, 7);
  CHECK(e4.k == 4 && e4.colors == 3 && e4.p == 1.0 / 3.0);
  CHECK(e4.estimate == double(e4.sub_count) * 27.0);
  CHECK(approx_count(g24, 4, 3, 7).estimate == e4.estimate);
  CHECK_THROWS_AS(colorful_sparsify(complete(4), 0, 1), std::invalid_argument);
  CHECK_THROWS_AS(approx_count(complete(4), 1, 2, 1), std::invalid_argument);
  std::vector<uint64_t> none(3, 0);
  CHECK(analytic_variance(10, 1.0, 3, none) == 0.0);
  CHECK(analytic_variance(1, 0.5, 3, none) == 3.0);
}

}  // namespace

int main() {
  struct {
    const char* name;
    void (*fn)();
  } cases[] = {
      {"fixed counts", case_fixed_counts},
      {"k=2 counts edges", case_k2},
      {"orderings agree with exhaustive count", case_orderings_agree},
      {"per-vertex counts", case_per_vertex},
      {"degree ranking", case_degree_ranking},
      {"original ranking / direct_by_ranking", case_original_and_direct},
      {"kcore realizes degeneracy", case_kcore},
      {"barenboim-elkin / goodrich-pszona shapes", case_be_and_gp},
      {"arboricity estimate", case_arboricity},
      {"make_ranking dispatch", case_dispatch},
      {"directed graph properties", case_dag_properties},
      {"graph construction and text io", case_graph_io},
      {"default parallelism", case_default_parallelism},
      {"bucket queue", case_bucket_queue},
      {"update_counts", case_update_counts},
      {"peel_exact / peel_approx", case_peel},
      {"colour sparsification / approx_count", case_sampling},
      {"list_cliques", case_list_cliques},
  };
  for (auto& c : cases) {
    int before = g_fail;
    try {
      c.fn();
    } catch (const std::exception& e) {
      g_fail++;
      std::printf("  EXCEPTION %s\n", e.what());
    }
    std::printf("%s %s\n", g_fail == before ? "PASS" : "FAIL", c.name);
  }
  std::printf("DROPIN %s %d checks, %d failed\n", g_fail ? "FAIL" : "OK", g_checks, g_fail);
  return g_fail ? 1 : 0;
}

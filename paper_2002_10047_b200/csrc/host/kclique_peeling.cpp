// Drop-in peeling entry points (include/kclique/peeling.hpp).  The graph
// stays resident (kcg_cache.hpp); when its device DAG is not already dg's,
// dg's ranking is installed and the DAG rebuilt on the device
// (direct_by_ranking is a function of the two, graph.cpp:94-114); the
// rounds run in kcg_peel.cu.  BucketQueue is host bookkeeping with
// the reference's observable behaviour (peeling.hpp:12-53).
#include <stdexcept>

#include "kcg_cache.hpp"
#include "kcg_handle.hpp"
#include "kclique/peeling.hpp"

namespace kclique {

BucketQueue::BucketQueue(std::span<const uint64_t> values, uint64_t)
    : value_(values.begin(), values.end()), extracted_(values.size(), 0) {
  for (VertexId v = 0; v < value_.size(); v++) order_.emplace(value_[v], v);
}

std::pair<uint64_t, std::vector<VertexId>> BucketQueue::extract_min() {
  if (order_.empty()) throw std::logic_error("extract_min on an empty BucketQueue");
  const uint64_t val = order_.begin()->first;
  std::vector<VertexId> out;
  while (!order_.empty() && order_.begin()->first == val) {
    const VertexId v = order_.begin()->second;
    order_.erase(order_.begin());
    extracted_[v] = 1;
    out.push_back(v);
  }
  return {val, std::move(out)};
}

void BucketQueue::update(VertexId v, uint64_t value) {
  if (v >= value_.size() || extracted_[v])
    throw std::logic_error("BucketQueue::update on an extracted vertex");
  order_.erase({value_[v], v});
  value_[v] = value;
  order_.emplace(value, v);
}

namespace {

PeelOutcome outcome(const kcg_peel_result& r, std::vector<VertexId> dense,
                    std::vector<uint64_t> core) {
  PeelOutcome o;
  o.rounds = r.rounds;
  o.total_cliques = r.total_cliques;
  o.best_density = r.best_density;
  o.best_round = r.best_round;
  dense.resize(r.num_dense);
  o.dense_vertices = std::move(dense);
  o.core = std::move(core);
  return o;
}

}  // namespace

UpdateResult update_counts(const Graph& g, const DirectedGraph& dg, int k,
                           std::span<uint64_t> counts, std::span<const VertexId> batch,
                           std::span<const uint8_t> peeled) {
  if (k < 2) throw std::invalid_argument("k must be at least 2");
  const VertexId n = g.num_vertices();
  if (counts.size() < n || peeled.size() < n)
    throw std::invalid_argument("counts and peeled must cover every vertex");
  auto dev = b200::resident_for_graph(g);
  std::lock_guard<std::mutex> lk(dev->mu);
  b200::ensure_oriented(*dev, g, dg);
  UpdateResult res;
  std::vector<VertexId> changed(n);
  uint64_t nch = 0;
  b200::check(kcg_update_counts(dev->h, k, counts.data(), batch.data(), batch.size(),
                                peeled.data(), &res.removed, changed.data(), &nch));
  changed.resize(nch);
  res.changed = std::move(changed);
  return res;
}

PeelOutcome peel_exact(const Graph& g, const DirectedGraph& dg, int k) {
  if (k < 2) throw std::invalid_argument("k must be at least 2");
  const VertexId n = g.num_vertices();
  if (n == 0) return PeelOutcome{};
  auto res = b200::resident_for_graph(g);
  std::lock_guard<std::mutex> lk(res->mu);
  b200::ensure_oriented(*res, g, dg);
  kcg_peel_result r{};
  std::vector<uint64_t> core(n);
  std::vector<VertexId> dense(n);
  b200::check(kcg_peel_exact(res->h, k, &r, core.data(), dense.data()));
  return outcome(r, std::move(dense), std::move(core));
}

PeelOutcome peel_approx(const Graph& g, const DirectedGraph& dg, int k, double epsilon) {
  if (k < 2) throw std::invalid_argument("k must be at least 2");
  if (epsilon <= 0) throw std::invalid_argument("epsilon must be positive");
  const VertexId n = g.num_vertices();
  if (n == 0) return PeelOutcome{};
  auto res = b200::resident_for_graph(g);
  std::lock_guard<std::mutex> lk(res->mu);
  b200::ensure_oriented(*res, g, dg);
  kcg_peel_result r{};
  std::vector<VertexId> dense(n);
  b200::check(kcg_peel_approx(res->h, k, epsilon, &r, dense.data()));
  return outcome(r, std::move(dense), {});
}

}  // namespace kclique

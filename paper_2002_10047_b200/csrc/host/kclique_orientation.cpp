// Drop-in ranking entry points (include/kclique/orientation.hpp): the graph
// stays resident on the B200 across calls (kcg_cache.hpp) and the peeling
// rounds run there (kcg_rank); the returned Ranking is remembered as the
// one installed, so direct_by_ranking(g, r) uploads nothing.
#include "kcg_cache.hpp"
#include "kcg_handle.hpp"
#include "kclique/orientation.hpp"

namespace kclique {
namespace {

Ranking run(const Graph& g, int strategy, double eps, uint64_t alpha_hat, uint64_t* rounds,
            uint64_t* alpha_out = nullptr) {
  std::vector<VertexId> rank;
  b200::resize_huge(rank, g.num_vertices());
  uint64_t r = 0, a = 0;
  if (g.num_vertices() == 0) {
    // keep the reference's argument checks for the empty graph
    if ((strategy == KCG_GOODRICH_PSZONA || strategy == KCG_BARENBOIM_ELKIN) && !(eps > 0))
      throw std::invalid_argument("epsilon must be positive");
    if (rounds) *rounds = r;
    if (alpha_out) *alpha_out = a;
    return Ranking(std::move(rank));
  }
  auto res = b200::resident_for_graph(g);
  std::lock_guard<std::mutex> lk(res->mu);
  b200::set_keys(*res, {}, {});
  b200::check(kcg_rank(res->h, strategy, eps, alpha_hat, rank.data(), &r, &a));
  if (rounds) *rounds = r;
  if (alpha_out) *alpha_out = a;
  Ranking out(std::move(rank));  // the buffer moves with the returned value
  b200::set_keys(*res, b200::key_of(out), {});
  return out;
}

}  // namespace

Ranking rank_by_degree(const Graph& g) { return run(g, KCG_DEGREE, 1.0, 0, nullptr); }
Ranking rank_original(const Graph& g) { return Ranking::identity(g.num_vertices()); }
Ranking rank_by_kcore(const Graph& g) { return run(g, KCG_KCORE, 1.0, 0, nullptr); }

Ranking rank_goodrich_pszona(const Graph& g, double epsilon, uint64_t* rounds_out) {
  if (!(epsilon > 0)) throw std::invalid_argument("epsilon must be positive");
  return run(g, KCG_GOODRICH_PSZONA, epsilon, 0, rounds_out);
}

Ranking rank_barenboim_elkin(const Graph& g, double epsilon, uint64_t alpha_hat,
                             uint64_t* rounds_out) {
  if (!(epsilon > 0)) throw std::invalid_argument("epsilon must be positive");
  if (alpha_hat < 1) throw std::invalid_argument("alpha_hat must be >= 1");
  return run(g, KCG_BARENBOIM_ELKIN, epsilon, alpha_hat, rounds_out);
}

uint64_t estimate_arboricity(const Graph& g, double epsilon) {
  if (!(epsilon > 0)) throw std::invalid_argument("epsilon must be positive");
  if (g.num_vertices() == 0) return 1;
  auto res = b200::resident_for_graph(g);
  std::lock_guard<std::mutex> lk(res->mu);
  uint64_t a = 0;
  b200::check(kcg_estimate_arboricity(res->h, epsilon, &a));
  return a;
}

Ranking make_ranking(const Graph& g, const OrientConfig& cfg) {
  switch (cfg.strategy) {
    case OrientStrategy::degree:
      return rank_by_degree(g);
    case OrientStrategy::original:
      return rank_original(g);
    case OrientStrategy::kcore:
      return rank_by_kcore(g);
    case OrientStrategy::goodrich_pszona:
      return rank_goodrich_pszona(g, cfg.epsilon);
    case OrientStrategy::barenboim_elkin: {
      if (!(cfg.epsilon > 0)) throw std::invalid_argument("epsilon must be positive");
      // alpha_hat 0 asks kcg_rank to estimate it on the device
      uint64_t a = cfg.alpha_hat ? *cfg.alpha_hat : 0;
      if (cfg.alpha_hat && a < 1) throw std::invalid_argument("alpha_hat must be >= 1");
      return run(g, KCG_BARENBOIM_ELKIN, cfg.epsilon, a, nullptr);
    }
  }
  throw std::invalid_argument("unknown orientation strategy");
}

}  // namespace kclique
